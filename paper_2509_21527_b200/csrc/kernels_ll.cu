// kernels_ll.cu — default ("LL") protocol of the hot path.
//
// The paper signals each pulse with one system-scope release flag issued by
// the last CTA after a completion counter (Alg. 5).  On B200 each
// such hop costs a MEMBAR.SYS per CTA + an atomic + a release store + the
// remote poll.  Here every 8-byte store that crosses between GPUs carries its
// own 32-bit sequence tag next to one fp32 value (single-copy atomic), so:
//   * no fences, counters or flags on the data path;
//   * forwarding is row-level: a forwarded row leaves as soon as its own unit
//     arrived (Alg. 4's dependency wait shrinks to the rows actually read);
//   * the force halo is a deterministic fold in the oracle's order (R15), no
//     atomics, and a row is pushed back as soon as it is final (Alg. 5
//     DEP_MGMT at row granularity).
//
// Hop groups: the DD ranks a process drives share one GPU's
// memory, so a pulse between two of them is not a transport hop.  The plan
// (runtime.cu, at the NS step) resolves such pulses: every halo row an x item
// writes names its origin — a home row, or the LL unit in which the row crossed
// from another group — and the +L shifts it picked up on the way (applied in
// pulse order: the oracle's fp32 adds, bit for bit); the force halo of a group
// is a set of trees, each folded by one thread per component with children in
// descending pulse order.  Only pulses between groups wait.  With one DD rank
// per GPU (the paper's setup) every pulse is a hop and this is the paper's
// staged schedule; HALO_COLLAPSE=0 makes every rank its own group on any GPU
// count (the staged schedule on one GPU: the cross-GPU code paths under test).
//
// One kernel body serves three launches (kMode): the x halo, the f halo, and
// both in ONE launch (halo_exchange_xf; "a single kernel for
// x+f when no compute sits between them") in which the tree items start once
// every halo row of the process is complete (a launch-wide item counter, the
// place of the non-bonded kernel between the two exchanges, Alg. 2).
//
// Each CTA runs a static list of work items; every item is one fixed-size block
// in HBM.  A ring of kRing shared-memory slots is filled by bulk (TMA) copies
// completing on mbarriers: the first blocks are requested before
// griddepcontrol.wait (static plan data, overlapped with the previous kernel's
// drain), and the block of item j+ring is requested as soon as item j is done.
// Items are ordered by dependency class (a wait only targets an item of a lower
// class on another GPU).  Progress needs every CTA of the grid to
// be resident at once: the grid never exceeds the occupancy-computed capacity of
// the device, which holds when this context may use every SM (launches are not
// cooperative by default: a cooperative launch disables programmatic dependent
// launch).  Where that is not guaranteed — MPS with an active-thread percentage,
// green contexts, a persistent kernel holding SMs — the launch is cooperative
// (HALO_COOP=1; the default under MPS), and the driver refuses a grid that cannot
// be co-resident instead of letting it spin until the timeout.
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>

#include "halo_internal.h"
#include "ptx.cuh"

namespace halo {

__device__ __forceinline__ uint64_t ll_pack(float v, uint32_t tag) {
  return ((uint64_t)tag << 32) | (uint64_t)__float_as_uint(v);
}

// Slow path: poll one LL unit until it carries `tag`; bounded like every wait.
// Tight polling for the first ~kTightNs of the wait (the latency regime: data
// arrives within a few us, and every poll counts), then exponential __nanosleep
// backoff up to ~2 us per poll: a wait that lasts because the peer's grid is not
// yet resident (it shares the SMs with a concurrent compute kernel, Alg. 2) must
// not steal that kernel's issue slots and L2 bandwidth.  The clock is read every
// 16 polls.  sleep_ns > 0 (HALO_POLL_NS) forces a fixed sleep; kPollTight
// (HALO_POLL_NS=-1) never sleeps.
__device__ __forceinline__ uint64_t ll_spin(const uint64_t* u, uint32_t tag, uint64_t timeout_ns, int* err_host,
                                         int code, uint32_t sleep_ns) {
  constexpr uint64_t kTightNs = 20000;
  const uint64_t t0 = gtimer();
  uint32_t backoff = 0;  // 0 = tight; else the current sleep in ns
  for (uint32_t it = 1;; ++it) {
    if (sleep_ns) {
      if (sleep_ns != kPollTight) __nanosleep(sleep_ns);
    } else if (backoff) {
      __nanosleep(backoff);
      if (backoff < 2048u && (it & 7u) == 0) backoff <<= 1;
    }
    const uint64_t v = ld_relaxed_sys(u);
    if ((uint32_t)(v >> 32) == tag) return v;
    if ((it & 15u) == 0) {
      const uint64_t el = gtimer() - t0;
      if (!backoff && el > kTightNs) backoff = 128u;
      if ((it & 1023u) == 0) {
        if (el > timeout_ns) {
          report_timeout(err_host, code);
          return v;
        }
        if (*(volatile int*)err_host != 0) return v;
      }
    }
  }
}

// Checked build (-DHALO_BOUNDS_CHECK, tests/bounds_check_run.py; compute-sanitizer is closed
// on this GPU pool): every global index the kernel derives from a plan record is checked
// against its buffer; a failed check reports kErrKindBounds (local rank, check number),
// and the access goes to index 0 instead.  The production build compiles the checks out.
#ifdef HALO_BOUNDS_CHECK
__device__ __noinline__ bool bc_fail(const ExParams& P, int code, int lr) {
  report_timeout(P.err_host, tcode(kErrKindBounds, lr & 0xff, code));
  return false;
}
#define HALO_BC(cond, code, lr) ((cond) ? true : bc_fail(P, (code), (lr)))
#else
#define HALO_BC(cond, code, lr) true
#endif

// An item of another NS epoch's plan (a stale graph replay): report once, do nothing.
__device__ __noinline__ uint32_t stale_item(const ExParams& P) {
  if (threadIdx.x == 0) report_timeout(P.err_host, tcode(kErrKindStalePlan, 0, 0));
  return 0;
}

__device__ __forceinline__ float ll_wait(const uint64_t* u, uint32_t tag, uint64_t timeout_ns, int* err_host,
                                         int code, uint32_t sleep_ns) {
  uint64_t v = ld_relaxed_sys(u);
  if ((uint32_t)(v >> 32) != tag) v = ll_spin(u, tag, timeout_ns, err_host, code, sleep_ns);
  return __uint_as_float((uint32_t)v);
}


// ---------------------------------------------------------------- x items
// kU = units per thread per batch: 1 for the latency regime (64-row items, at
// most one unit per thread), 4 for large items (bandwidth regime: every load of
// a batch is issued before any store — the stores are asm volatile with a
// memory clobber, so one unit at a time would serialise a memory latency each).
// kLocal: every item of the plan stays in this hop group (one process hosts every DD
// rank: no LL units anywhere) — the LL paths are compiled out (less code to fetch cold).
template <int W, int kU, bool kChk, bool kLocal = false>
__device__ __forceinline__ void x_item(const XRec& r, const XEnt* ent, const LocalBase* lb, const ExParams& P,
                                       uint32_t tag) {
  // a CUDA graph captured before the last NS step replays with this epoch: every item of
  // a replaced (or zeroed) plan carries another one and is treated as empty
  const uint32_t n = !kChk || r.epoch == P.plan_epoch ? r.n_units : stale_item(P);
  const uint32_t B = blockDim.x;
  if (!kLocal && r.kind == kItemXWait) {
    // a bulk pulse: the x-sender stored this rank's rows straight into
    // x and counts them here (one release add per send item); wait for all n, then take
    // them back off so the word is 0 for the next launch
    if (threadIdx.x == 0 && n != 0 &&
        wait_geq<true>(r.bulk, n, P.timeout_ns, P.err_host, tcode(10, r.lrank, r.pulse), P.poll_ns))
      red_add_relaxed_sys(r.bulk, (uint64_t)0 - n);
    return;
  }
  if (!kLocal && r.kind == kItemXRecv) {
    // this rank's halo rows of one pulse from another group: LL units -> x rows;
    // 4 units per thread per batch: the polls of a batch are in flight together
    constexpr int kR = 4;
    if (!HALO_BC((uint64_t)r.begin * W + n <= P.ll_stride && r.begin + n / W <= (uint32_t)P.cap_rows, 7, r.lrank))
      return;
    for (uint32_t base = threadIdx.x; base < n; base += kR * B) {
      uint64_t w[kR];
#pragma unroll
      for (int k = 0; k < kR; ++k)
        if (base + k * B < n) w[k] = ld_relaxed_sys(r.ll + base + k * B);
#pragma unroll
      for (int k = 0; k < kR; ++k) {
        const uint32_t u = base + k * B;
        if (u >= n) continue;
        if ((uint32_t)(w[k] >> 32) != tag)
          w[k] = ll_spin(r.ll + u, tag, P.timeout_ns, P.err_host, tcode(10, r.lrank, r.pulse), P.poll_ns);
        r.xdst[u] = __uint_as_float((uint32_t)w[k]);
      }
    }
    return;
  }
  // SEND (Alg. 3 + Alg. 4): per halo row, its origin (home row, or the LL unit in
  // which it entered this group: a row-level dependency wait) + its shifts (R25)
  for (uint32_t base = threadIdx.x; base < n; base += kU * B) {
    uint64_t w[kU];
    const uint64_t* src[kU];
    uint32_t mask[kU];
#pragma unroll
    for (int k = 0; k < kU; ++k) {
      const uint32_t u = base + k * B;
      src[k] = nullptr;
      if (u < n) {
        const uint32_t e = u / W;
        const int c = (int)(u - e * W);
        XEnt E = ent[e];
        if (!HALO_BC(E.l < (uint32_t)P.n_local, 1, r.lrank)) E.l = 0;
        const LocalBase& L = lb[E.l];
        mask[k] = E.mask;
        if (kLocal || !(E.kq & 0x80u)) {
          // a home row: never written during the kernel
          if (!HALO_BC(E.row < (uint32_t)P.cap_rows, 2, r.lrank)) E.row = 0;
          w[k] = ((uint64_t)tag << 32) | __float_as_uint(__ldg(L.x + (size_t)E.row * W + c));
        } else {
          const int q = E.kq & 7;
          if (!HALO_BC(q < P.P && (uint64_t)E.row * W + c < P.ll_stride &&
                           (uint32_t)L.recv_off[q] + E.row < (uint32_t)P.cap_rows, 3, r.lrank))
            E.row = 0;
          if (q < P.p_lo || (P.debug & kMutateXNoWait)) {
            // arrived in an earlier launch (set_maps' per-pulse exchanges): final in x.
            // kMutateXNoWait: the protocol mutation the sentinel tests must catch —
            // forward the row from x without waiting for its arrival
            w[k] = ((uint64_t)tag << 32) | __float_as_uint(__ldcg(L.x + (size_t)(L.recv_off[q] + E.row) * W + c));
          } else {
            src[k] = L.xll + (size_t)q * P.ll_stride + (size_t)E.row * W + c;
            w[k] = ld_relaxed_sys(src[k]);
          }
        }
      }
    }
#pragma unroll
    for (int k = 0; k < kU; ++k) {
      const uint32_t u = base + k * B;
      if (u >= n) continue;
      const uint32_t e = u / W;
      const int c = (int)(u - e * W);
      if (!kLocal && src[k] != nullptr && (uint32_t)(w[k] >> 32) != tag)
        w[k] = ll_spin(src[k], tag, P.timeout_ns, P.err_host, tcode(11, r.lrank, r.pulse), P.poll_ns);
      float v = __uint_as_float((uint32_t)w[k]);
      if (c < 3) {
#pragma unroll
        for (int q = 0; q < kMaxP; ++q)
          if (mask[k] >> q & 1u) v = __fadd_rn(v, c == r.pdim[q] ? r.shiftL[q] : 0.0f);
      }
      size_t o = (size_t)(r.begin + e) * W + c;
      if (!HALO_BC(kLocal || r.dst_x != nullptr ? r.begin + e < (uint32_t)P.cap_rows : o < P.ll_stride, 4, r.lrank))
        o = 0;
      if (kLocal || r.dst_x != nullptr) r.dst_x[o] = v;  // a rank of this group: its halo row directly
      else st_relaxed_sys(r.dst_ll + o, ll_pack(v, tag));
    }
  }
  // experiment (HALO_DEBUG=128): drain this thread's peer stores inside the item
  if (P.debug & kFenceAfterPeerStores) fence_sys();
}

// Two send items at once (the fused launch: its x phase runs at the f kernel's 4 CTAs
// per SM, so a CTA holds ~1.6 x items; processing two together keeps one load of each
// in flight per thread instead of two dependent rounds).  Same arithmetic as x_item.
template <int W, bool kChk, bool kLocal = false>
__device__ __forceinline__ void x_send_pair(const XRec& r0, const XEnt* e0, const XRec& r1, const XEnt* e1,
                                            const LocalBase* lb, const ExParams& P, uint32_t tag) {
  const XRec* rr[2] = {&r0, &r1};
  const XEnt* ee[2] = {e0, e1};
  uint32_t n[2];
#pragma unroll
  for (int i = 0; i < 2; ++i) n[i] = !kChk || rr[i]->epoch == P.plan_epoch ? rr[i]->n_units : stale_item(P);
  const uint32_t B = blockDim.x;
  for (uint32_t u = threadIdx.x; u < max(n[0], n[1]); u += B) {
    uint64_t w[2];
    const uint64_t* src[2];
    uint32_t mask[2];
#pragma unroll
    for (int i = 0; i < 2; ++i) {
      src[i] = nullptr;
      if (u < n[i]) {
        const uint32_t e = u / W;
        const int c = (int)(u - e * W);
        XEnt E = ee[i][e];
        if (!HALO_BC(E.l < (uint32_t)P.n_local, 1, rr[i]->lrank)) E.l = 0;
        if (!HALO_BC(E.row < (uint32_t)P.cap_rows, 2, rr[i]->lrank)) E.row = 0;
        const LocalBase& L = lb[E.l];
        mask[i] = E.mask;
        if (kLocal || !(E.kq & 0x80u)) {
          w[i] = ((uint64_t)tag << 32) | __float_as_uint(__ldg(L.x + (size_t)E.row * W + c));
        } else {
          const int q = E.kq & 7;
          if (q < P.p_lo || (P.debug & kMutateXNoWait)) {
            w[i] = ((uint64_t)tag << 32) | __float_as_uint(__ldcg(L.x + (size_t)(L.recv_off[q] + E.row) * W + c));
          } else {
            src[i] = L.xll + (size_t)q * P.ll_stride + (size_t)E.row * W + c;
            w[i] = ld_relaxed_sys(src[i]);
          }
        }
      }
    }
#pragma unroll
    for (int i = 0; i < 2; ++i) {
      if (u >= n[i]) continue;
      const XRec& r = *rr[i];
      const uint32_t e = u / W;
      const int c = (int)(u - e * W);
      if (!kLocal && src[i] != nullptr && (uint32_t)(w[i] >> 32) != tag)
        w[i] = ll_spin(src[i], tag, P.timeout_ns, P.err_host, tcode(11, r.lrank, r.pulse), P.poll_ns);
      float v = __uint_as_float((uint32_t)w[i]);
      if (c < 3) {
#pragma unroll
        for (int q = 0; q < kMaxP; ++q)
          if (mask[i] >> q & 1u) v = __fadd_rn(v, c == r.pdim[q] ? r.shiftL[q] : 0.0f);
      }
      size_t o = (size_t)(r.begin + e) * W + c;
      if (!HALO_BC(kLocal || r.dst_x != nullptr ? r.begin + e < (uint32_t)P.cap_rows : o < P.ll_stride, 4, r.lrank))
        o = 0;
      if (kLocal || r.dst_x != nullptr) r.dst_x[o] = v;
      else st_relaxed_sys(r.dst_ll + o, ll_pack(v, tag));
    }
  }
}

// ---------------------------------------------------------------- f items
// Fused launch: thread 0 waits until the last x item of this launch released
// xf_done = seq (polling one word, with a short sleep between polls so that ~600
// waiting CTAs do not flood the line the x items' counter shares the L2 with).
// Bounded like every wait.
__device__ __noinline__ void xdone_wait(Ctrl* ctrl, uint64_t seq, const ExParams& P) {
  const uint64_t t0 = gtimer();
  for (uint32_t it = 1;; ++it) {
    if (ld_acquire_gpu(&ctrl->xf_done) >= seq) return;  // the counted items' stores happen-before
    __nanosleep(it < 8 ? 32 : 128);
    if ((it & 255u) == 0) {
      if (gtimer() - t0 > P.timeout_ns) {
        report_timeout(P.err_host, tcode(15, 0, 0));
        return;
      }
      if (*(volatile int*)P.err_host != 0) return;
    }
  }
}

// Shift forces (R13; north_star): the value of every edge whose parent's rank
// wrapped in the edge's pulse goes to fshift[rank][dim].  Each thread adds its
// edges' values into its own column of the item's buckets (fp64, shared memory,
// no atomics); after the item a fixed-order reduction per (bucket, component)
// and ONE fp64 atomic add per (bucket, component) into fshift.  Edges of a tree
// with more distinct targets than kMaxBuckets add directly (kFsDirect).
__device__ __forceinline__ void fs_bucket_add(double (*s_v)[kThreads], int b, float v, const ExParams& P) {
  double& a = s_v[b][threadIdx.x];
  a = (P.debug & kMutateFshiftF32) ? (double)((float)a + v) : a + (double)v;  // mutation: fp32 accumulation
}
__device__ __forceinline__ void fs_add(double (*s_v)[kThreads], const TNode& nd, int c, float v,
                                       const ExParams& P) {
  const int b = (nd.kq >> 3) & 15;
  if (b == kFsNone || c >= 3) return;
  if (b == kFsDirect) atomicAdd(P.fshift + 3 * nd.fs + c, (double)v);
  else fs_bucket_add(s_v, b, v, P);
}

__device__ __forceinline__ float ll_value(uint64_t w, const uint64_t* src, const ExParams& P, uint32_t tag,
                                          int lrank, int q) {
  if ((uint32_t)(w >> 32) != tag && !(P.debug & kMutateFNoWait))
    w = ll_spin(src, tag, P.timeout_ns, P.err_host, tcode(12, lrank, q), P.poll_ns);
  return __uint_as_float((uint32_t)w);
}

// Large trees (> kFastNodes nodes, P > 3): depth-first fold with an explicit
// stack of open levels, one node at a time.
template <int W>
__device__ __noinline__ float tree_fold_generic(const TNode* nd, int nn, const LocalBase* lb, const ExParams& P,
                                                int c, uint32_t tag, int lrank, double (*s_v)[kThreads], bool fs_on) {
  float acc[kMaxDepth];
  int stk[kMaxDepth];
  int top = 0;
  auto load = [&](const TNode& m) -> float {
    const LocalBase& L = lb[m.il >> 24];
    const uint32_t idx = m.il & (kMaxRows - 1);
    if (!(m.kq & 0x80u)) return __ldcg(L.f + (size_t)idx * W + c);
    const uint64_t* a = L.fll + (size_t)(m.kq & 7) * P.ll_stride + (size_t)idx * W + c;
    return ll_value(ld_relaxed_sys(a), a, P, tag, lrank, m.kq & 7);
  };
  auto close_to = [&](int d) {
    for (int t = top; t >= d && t >= 1; --t) {
      const TNode& m = nd[stk[t]];
      if (m.flags & 1u) lb[m.il >> 24].f[(size_t)(m.il & (kMaxRows - 1)) * W + c] = acc[t];
      if (fs_on) fs_add(s_v, m, c, acc[t], P);
      acc[t - 1] = P.accumulate ? __fadd_rn(acc[t - 1], acc[t]) : acc[t];
    }
    top = min(top, d - 1);
  };
  acc[0] = load(nd[0]);
  stk[0] = 0;
  for (int k = 1; k < nn; ++k) {
    const int d = nd[k].flags >> 1;
    close_to(d);
    acc[d] = load(nd[k]);
    stk[d] = k;
    top = d;
  }
  close_to(1);
  if (nd[0].flags & 1u) lb[nd[0].il >> 24].f[(size_t)(nd[0].il & (kMaxRows - 1)) * W + c] = acc[0];
  return acc[0];
}

// After an item: the fixed-order reduction of its shift-force buckets; output
// (b, comp) by warp (b*3 + comp) mod warps, lanes over the threads of that
// component in a fixed order, then a fixed xor-shuffle tree, one fp64 atomic.
template <int W>
__device__ __forceinline__ void fs_flush(const GRec& g, double (*s_v)[kThreads], uint32_t S, const ExParams& P) {
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = (int)(blockDim.x >> 5);
  for (int o = warp; o < 3 * g.n_buckets; o += nw) {
    const int b = o / 3, cc = o % 3;
    double a = 0.0;
    for (uint32_t t = cc + W * lane; t < S; t += 32 * W) a += s_v[b][t];
#pragma unroll
    for (int m = 16; m > 0; m >>= 1) a += __shfl_xor_sync(0xffffffffu, a, m);
    if (P.debug & kMutateFshiftF32) a = (double)(float)a;  // mutation: fp32 partials
    if (lane == 0 && a != 0.0) atomicAdd(P.fshift + 3 * g.bucket_fs[b] + cc, a);
  }
}

// The LL nodes of a small tree: every unit requested, then each one checked for
// this launch's tag (spinning until the remote push lands) into shared memory.
template <int W>
__device__ __noinline__ void tree_ll_nodes(const TRoot R, const uint32_t* il, const LocalBase* lb,
                                           const ExParams& P, uint32_t tag, int lrank, float (*s_val)[kThreads]) {
  const int c = (int)(threadIdx.x % W);
  const uint64_t* a[kFastNodes];
  uint64_t w[kFastNodes];
#pragma unroll
  for (int k = 0; k < kFastNodes; ++k)
    if (k < R.nn && (R.llmask >> k & 1u)) {
      a[k] = lb[il[k] >> 24].fll + (size_t)(R.q >> (4 * k) & 15u) * P.ll_stride + (size_t)(il[k] & (kMaxRows - 1)) * W + c;
      w[k] = ld_relaxed_sys(a[k]);
    }
  for (int k = 0; k < kFastNodes; ++k)
    if (k < R.nn && (R.llmask >> k & 1u)) {
      uint64_t x = 0;
#pragma unroll
      for (int m = 0; m < kFastNodes; ++m)
        if (m == k) x = w[m];
      if ((uint32_t)(x >> 32) != tag && !(P.debug & kMutateFNoWait)) {
        const uint64_t* ak = lb[il[k] >> 24].fll + (size_t)(R.q >> (4 * k) & 15u) * P.ll_stride +
                             (size_t)(il[k] & (kMaxRows - 1)) * W + c;
        x = ll_spin(ak, tag, P.timeout_ns, P.err_host, tcode(12, lrank, R.q >> (4 * k) & 15u), P.poll_ns);
      }
      s_val[k][threadIdx.x] = __uint_as_float((uint32_t)x);
    }
}

// One small-tree item: each (root, component) is folded by one thread.  All node
// values are loaded first (every load in flight) into the thread's column of
// shared memory, then one add per edge in POSTORDER (the root record's 4-bit
// fields): a node's children finish before it, in preorder = descending pulse
// order, so its parent receives f[parent] + children in the oracle's order (R15:
// one fp32 RNE add per child, the bits match).  A node's value is final when it
// is reached: stored (F nodes with children), added to its shift-force bucket,
// then added into its parent.  A root whose parent is in another group pushes
// its value there.  ~10 instructions per edge, none for absent nodes.
template <int W, bool kChk, bool kLocal = false>
__device__ __forceinline__ void tree_item(const GRec& g, const TRoot* roots, const uint4* nodes, const LocalBase* lb,
                                          const ExParams& P, uint32_t tag, double (*s_v)[kThreads],
                                          float (*s_val)[kThreads], uint64_t* tdet) {
  const uint32_t n = !kChk || g.epoch == P.plan_epoch ? g.n_units : stale_item(P);  // (as x_item)
  const uint32_t S = (blockDim.x / W) * W;  // stride: a multiple of W, every thread keeps one component
  const int c = (int)(threadIdx.x % W);
  const int tid = threadIdx.x;
  const bool fs_on = P.fshift != nullptr && g.n_buckets > 0 && n > 0;
  if (fs_on)
    for (int b = 0; b < g.n_buckets; ++b) s_v[b][tid] = 0.0;
  for (uint32_t u = tid; u < n && (uint32_t)tid < S; u += S) {
    const uint32_t j = u / W;
    const TRoot R = roots[j];
    const uint32_t* il = reinterpret_cast<const uint32_t*>(nodes + 2 * j);
    const int nn = R.nn;
#ifdef HALO_BOUNDS_CHECK
    if (!HALO_BC(nn >= 1 && nn <= kFastNodes && j < (uint32_t)P.tree_rows, 9, g.lrank)) continue;
    {
      bool bad = false;
      for (int k = 0; k < nn; ++k) {
        const uint32_t l = il[k] >> 24, i = il[k] & (kMaxRows - 1);
        bad |= l >= (uint32_t)P.n_local;
        bad |= (R.llmask >> k & 1u) ? (uint64_t)i * W + c >= P.ll_stride || (int)(R.q >> (4 * k) & 15u) >= P.P
                                   : i >= (uint32_t)P.cap_rows;
      }
      if (!HALO_BC(!bad, 10, g.lrank)) continue;
    }
#endif
    if (tdet && u == 0) tdet[0] = gtimer() + (il[0] == 0xffffffffu ? 1 : 0);  // records read
    // F node values straight into this thread's shared-memory column (LDGSTS: every
    // load in flight, no registers held); LL nodes out of line (they wait for a
    // remote push anyway)
#pragma unroll
    for (int k = 0; k < kFastNodes; ++k)
      if (k < nn && !(R.llmask >> k & 1u))
        cp_async4(&s_val[k][tid], lb[il[k] >> 24].f + (size_t)(il[k] & (kMaxRows - 1)) * W + c);
    cp_async_commit();
    if (!kLocal && R.llmask) tree_ll_nodes<W>(R, il, lb, P, tag, g.lrank, s_val);
    cp_async_wait_all();
    if (tdet && u == 0) tdet[1] = gtimer() + (__float_as_uint(s_val[0][tid]) == 0x7fc00001u ? 1 : 0);  // loads landed
    const uint32_t* ilr = il;
    for (int e = 0; e < nn - 1; ++e) {
      const int m = R.post >> (4 * e) & 15u;
      const int pm = R.par >> (4 * m) & 15u;
      const float vm = s_val[m][tid];
      if (R.stmask >> m & 1u) lb[ilr[m] >> 24].f[(size_t)(ilr[m] & (kMaxRows - 1)) * W + c] = vm;
      if (fs_on && c < 3) {
        const int b = R.bucket >> (4 * m) & 15u;
        if (b != kFsNone) fs_bucket_add(s_v, b, vm, P);
      }
      s_val[pm][tid] = P.accumulate ? __fadd_rn(s_val[pm][tid], vm) : vm;
    }
    const float root = s_val[0][tid];
    if (R.stmask & 1u) lb[il[0] >> 24].f[(size_t)(il[0] & (kMaxRows - 1)) * W + c] = root;
    if (!kLocal && R.push != nullptr) st_relaxed_sys(R.push + c, ll_pack(root, tag));
    if (tdet && u == 0) tdet[2] = gtimer();  // folded and stored
  }
  if (fs_on) fs_flush<W>(g, s_v, S, P);
  if (tdet) tdet[3] = gtimer();
}

// One large-tree item (kItemTreeG): the generic fold, one (root, component) per thread.
template <int W, bool kChk>
__device__ __noinline__ void tree_item_generic(const GRec& g, const TRootG* roots, const TNode* nodes,
                                                  const LocalBase* lb, const ExParams& P, uint32_t tag,
                                                  double (*s_v)[kThreads]) {
  const uint32_t n = !kChk || g.epoch == P.plan_epoch ? g.n_units : stale_item(P);  // (as x_item)
  const uint32_t S = (blockDim.x / W) * W;
  const int c = (int)(threadIdx.x % W);
  const bool fs_on = P.fshift != nullptr && n > 0;
  if (fs_on)
    for (int b = 0; b < g.n_buckets; ++b) s_v[b][threadIdx.x] = 0.0;
  for (uint32_t u = threadIdx.x; u < n && threadIdx.x < S; u += S) {
    const TRootG R = roots[u / W];
    const float root = tree_fold_generic<W>(nodes + R.node_begin, R.n_nodes, lb, P, c, tag, g.lrank, s_v, fs_on);
    if (R.push != nullptr) st_relaxed_sys(R.push + c, ll_pack(root, tag));
  }
  if (fs_on && g.n_buckets > 0) fs_flush<W>(g, s_v, S, P);
}

// ---------------------------------------------------------------- kernel
enum : int { kModeX = 0, kModeF = 1, kModeXF = 2 };

// Item block sizes: x = record + item_rows entries; f = record + tree_rows small
// tree roots (32 B) and their nodes (32 B) — a large-tree block has the same size.
__host__ __device__ __forceinline__ uint32_t xblk_bytes(uint32_t R) { return 128u + 8u * R; }
__host__ __device__ __forceinline__ uint32_t fblk_bytes(uint32_t R) { return 128u + 64u * R; }

// Items of this CTA: [0, n_main) round-robin over CTAs [0, G - n_tail) (fused:
// the x items first, then the tree items); n_tail trailing items would get one
// dedicated CTA each (none in the current plan).
// CTA size: 256 threads, except the experimental x variant kU = 3 (64-thread CTAs, meant
// to leave SM room for the f launch's CTAs under PDL; measured slower, see ll_fn_c).
template <int kU, int kMode>
__host__ __device__ constexpr int ll_threads() {
  return kMode == 0 && kU == 3 ? 64 : kThreads;
}

#ifndef HALO_XF_MIN_BLOCKS
#define HALO_XF_MIN_BLOCKS 3  // fused launch with LL paths: CTAs per SM the registers are budgeted for (3: no spills)
#endif
#ifndef HALO_F_MIN_BLOCKS
#define HALO_F_MIN_BLOCKS 3   // f launch with LL paths (N > 1): CTAs per SM the registers are budgeted for
                              // (3: no spills; C3 2 GPUs 28.7 -> 27.0, C4-1D 30.9 -> 30.1 us vs 4; the
                              // hop-group-local variants keep 4: fewer registers, and 3 costs them ~1.8 us fused)
#endif
// kChk: the launch is being captured into a CUDA graph, whose replays may outlive the
// plan (the next NS step): every item's epoch is checked.  Eager launches take their
// parameters from the current plan and skip the check (measured: ~0.2 us per step).
template <int W, int kU, int kMode, bool kChk, bool kLocal = false>
__global__ void __launch_bounds__(ll_threads<kU, kMode>(), kMode == kModeX ? (kU == 1 || kU == 3 ? 8 : 4)
                                                           : kLocal           ? 4
                                                           : kMode == kModeXF ? HALO_XF_MIN_BLOCKS
                                                                              : HALO_F_MIN_BLOCKS) k_exchange_ll(
    const __grid_constant__ ExParams P) {
  extern __shared__ __align__(128) unsigned char s_blk[];
  __shared__ uint64_t s_seq[2];
  __shared__ __align__(8) uint64_t s_bar[kRing];
  __shared__ __align__(16) LocalBase s_lb[kMaxLocal];
  __shared__ double s_v[kMode == kModeX ? 1 : kMaxBuckets][kThreads];  // shift-force buckets of an f item
  __shared__ float s_val[kMode == kModeX ? 1 : kFastNodes][kThreads];   // tree node values, one column per thread
  const uint32_t R = (uint32_t)P.item_rows, RT = (uint32_t)P.tree_rows;
  const uint32_t XB = xblk_bytes(R), FB = fblk_bytes(RT);
  const uint32_t SB = kMode == kModeX ? XB : FB;  // ring slot size
  const int nx = kMode == kModeF ? 0 : P.n_items_x;
  const int ring = P.ring;
  Ctrl* ctrl = P.ctrl;
  const int tslot = kMode == kModeF ? 1 : 0;
  const bool trace = (P.flags & HALO_F_TIMERS) && threadIdx.x == 0 && blockIdx.x < kTraceCTAs;
  if (trace) ctrl->trace[tslot][blockIdx.x][0] = gtimer();
  pdl_launch_dependents();
  const int n_main = P.n_items - P.n_tail;
  const int Gm = (int)gridDim.x - P.n_tail;
  const bool tailcta = (int)blockIdx.x >= Gm;
  const int first = tailcta ? n_main + ((int)blockIdx.x - Gm) : (int)blockIdx.x;
  const int stride = tailcta ? P.n_items : Gm;
  const int end = tailcta ? first + 1 : n_main;
  auto blk_of = [&](int i) -> const char* {
    return i < nx ? P.xblk + (size_t)i * XB : P.fblk + (size_t)(i - nx) * FB;
  };
  auto bytes_of = [&](int i) -> uint32_t { return i < nx ? XB : FB; };
  // static plan data, read while the previous kernel of the stream drains (PDL):
  // the first `ring` item blocks (bulk copies) and the local-rank base table;
  // x, f and the LL areas are touched after the wait
  if (threadIdx.x == 0) {
    for (int k = 0; k < ring; ++k) mbar_init(&s_bar[k], 1);
    fence_mbar_init();
    for (int k = 0, i = first; k < ring && i < end; ++k, i += stride)
      bulk_load(s_blk + (size_t)k * SB, blk_of(i), bytes_of(i), &s_bar[k]);
  }
  for (int t = threadIdx.x; t < P.n_local * 4; t += blockDim.x)
    reinterpret_cast<int4*>(s_lb)[t] = __ldg(reinterpret_cast<const int4*>(P.lbase) + t);
#ifdef HALO_EXP_PREFETCH  // measured slower; the call site alone costs ~0.2 us
  if (kMode == kModeX && (P.pf_f_bytes | (uint64_t)P.pf_x) != 0 && threadIdx.x == 32) prefetch_l2<W>(P);
#endif
  pdl_wait();  // everything below may depend on earlier work of the stream
#ifdef HALO_EXP_PREFETCH
  if (trace && (P.debug & kTraceDetail)) ctrl->trace[tslot][blockIdx.x][14] = gtimer();  // wait released
#endif
  // by value when the host knows them (no cold dependent load on the critical path)
  if (threadIdx.x == 0) {
    if (kMode != kModeF) s_seq[0] = P.seq ? P.seq : ll_seq_next(ld_relaxed_gpu(&ctrl->seq_x));
    if (kMode != kModeX) s_seq[1] = P.seq_f ? P.seq_f : ll_seq_next(ld_relaxed_gpu(&ctrl->seq_f));
  }
  timer_start(P.flags, kMode == kModeF ? &ctrl->t_start_f : &ctrl->t_start_x);
  __syncthreads();  // barrier init, base table and sequence numbers visible to every thread
#ifdef HALO_EXP_PREFETCH
  if (trace && (P.debug & kTraceDetail)) ctrl->trace[tslot][blockIdx.x][15] = gtimer();  // prologue done
#endif
  // arrive early: the atomic's latency hides behind the items (launch_arrive)
  const uint32_t arrived = launch_arrive(kMode == kModeF ? &ctrl->done_f : &ctrl->done_x);
  const uint32_t tag_x = (uint32_t)s_seq[0], tag_f = (uint32_t)s_seq[1];
  bool xin_seen = false;
  bool tdet_free = true;  // HALO_DEBUG kTraceDetail: stamps of the first tree item in trace slots 10-13
  int j = 0;
  for (int it = first; it < end; it += stride, ++j) {
    const int slot = j % ring;
    unsigned char* blk = s_blk + (size_t)slot * SB;
    mbar_wait(&s_bar[slot], (uint32_t)(j / ring) & 1u);
    if (trace && j == 0) ctrl->trace[tslot][blockIdx.x][1] = gtimer();
    if (kMode == kModeXF && kLocal && it < nx && it + stride < nx && ring >= 2 && !(P.debug & kTraceDetail)) {
      // two send items of this CTA at once (their blocks are both in the ring)
      const int slot2 = (j + 1) % ring;
      unsigned char* blk2 = s_blk + (size_t)slot2 * SB;
      mbar_wait(&s_bar[slot2], (uint32_t)((j + 1) / ring) & 1u);
      const XRec& r0 = *reinterpret_cast<const XRec*>(blk);
      const XRec& r1 = *reinterpret_cast<const XRec*>(blk2);
      if (!kLocal && (r0.kind == kItemXRecv || r1.kind == kItemXRecv)) {
        x_item<W, kU, kChk>(r0, reinterpret_cast<const XEnt*>(blk + 128), s_lb, P, tag_x);
        x_item<W, kU, kChk>(r1, reinterpret_cast<const XEnt*>(blk2 + 128), s_lb, P, tag_x);
      } else {
        x_send_pair<W, kChk, kLocal>(r0, reinterpret_cast<const XEnt*>(blk + 128), r1,
                                     reinterpret_cast<const XEnt*>(blk2 + 128), s_lb, P, tag_x);
      }
      __syncthreads();  // both items' rows are stored before their count; both slots are free
      if (threadIdx.x == 0) {
        if (atom_add_acqrel_gpu(&ctrl->xf_cnt, 2u) == (uint32_t)nx - 2u) {
          ctrl->xf_cnt = 0;  // (the next fused launch's x items start after this launch completes)
          st_release_gpu(&ctrl->xf_done, s_seq[0]);
        }
        fence_proxy_async_smem();
        for (int k2 = 0; k2 < 2; ++k2) {  // refill both slots (items it + ring*stride, it + (ring+1)*stride)
          const int nxt = it + (ring + k2) * stride;
          if (nxt < end) bulk_load(k2 ? blk2 : blk, blk_of(nxt), bytes_of(nxt), &s_bar[k2 ? slot2 : slot]);
        }
      }
      it += stride;
      ++j;
      continue;
    }
    if (kMode != kModeF && it < nx) {
      x_item<W, kU, kChk, kLocal>(*reinterpret_cast<const XRec*>(blk), reinterpret_cast<const XEnt*>(blk + 128), s_lb,
                                  P, tag_x);
      __syncthreads();  // the item's rows are stored (fused: before its count) and the slot is free
      if constexpr (!kLocal) {
        // a bulk pulse's send item: its rows (every thread's stores, ordered by the barrier)
        // are counted; the receiver's wait item acquires the total
        const XRec& r = *reinterpret_cast<const XRec*>(blk);
        if (threadIdx.x == 0 && r.bulk != nullptr && r.kind == kItemXSend && (!kChk || r.epoch == P.plan_epoch)) {
          // counted at gpu scope; the pulse's last item issues the one system-scope release
          // (a release per item measured 1.5x slower: every CTA stalls on its NVLink stores)
          const uint32_t rows = r.n_units / W;
          uint32_t* c = &ctrl->bulk_rows[r.lrank][r.pulse];
          if (atom_add_acqrel_gpu(c, rows) + rows == r.bulk_total) {
            *c = 0;  // (the next launch's items start after this launch completes)
            red_add_release_sys(r.bulk, r.bulk_total);
          }
        }
      }
      if (kMode == kModeXF && threadIdx.x == 0) {  // the launch's last x item releases xf_done
        if (atom_add_acqrel_gpu(&ctrl->xf_cnt, 1u) == (uint32_t)nx - 1u) {
          ctrl->xf_cnt = 0;  // (the next fused launch's x items start after this launch completes)
          st_release_gpu(&ctrl->xf_done, s_seq[0]);
        }
      }
    } else if constexpr (kMode != kModeX) {
      const GRec& g = *reinterpret_cast<const GRec*>(blk);
      if (kMode == kModeXF && !xin_seen) {  // every halo row of this process is complete (the NB kernel's slot)
        if (threadIdx.x == 0 && nx > 0) xdone_wait(ctrl, s_seq[0], P);
        __syncthreads();
        xin_seen = true;
      }
      if (g.kind == kItemTree)
        tree_item<W, kChk, kLocal>(g, reinterpret_cast<const TRoot*>(blk + 128), reinterpret_cast<const uint4*>(blk + 128 + 32 * RT),
                     s_lb, P, tag_f, s_v, s_val,
                     (trace && (P.debug & kTraceDetail) && tdet_free) ? &ctrl->trace[tslot][blockIdx.x][10] : nullptr);
      else
        tree_item_generic<W, kChk>(g, reinterpret_cast<const TRootG*>(blk + 128),
                             reinterpret_cast<const TNode*>(blk + 128 + 16 * (RT / 8 > 0 ? RT / 8 : 1)), s_lb, P,
                             tag_f, s_v);
      __syncthreads();  // everyone is done with this slot
      if (g.kind == kItemTree) tdet_free = false;
    }
    if (trace && j < ((P.debug & kTraceDetail) ? 3 : (kTraceW - 4) / 2)) {
      const uint8_t* b8 = reinterpret_cast<const uint8_t*>(blk);  // kind, pulse/level, lrank: same offsets in XRec/GRec
      ctrl->trace[tslot][blockIdx.x][4 + 2 * j] =
          ((uint64_t)b8[0] << 16) | ((uint64_t)(*reinterpret_cast<const uint16_t*>(b8 + 2)) << 8) | b8[1];
      ctrl->trace[tslot][blockIdx.x][5 + 2 * j] = gtimer();
    }
    if (threadIdx.x == 0 && it + ring * stride < end) {  // refill the slot with the block of item j + ring
      fence_proxy_async_smem();  // generic reads of the slot (this item) before the async write
      const int nxt = it + ring * stride;
      bulk_load(blk, blk_of(nxt), bytes_of(nxt), &s_bar[slot]);
    }
  }
  if (trace) ctrl->trace[tslot][blockIdx.x][2] = gtimer();
  if (threadIdx.x == 0) {
    if (P.flags & HALO_F_TIMERS) atomicMax((unsigned long long*)(kMode == kModeF ? &ctrl->t_end_f : &ctrl->t_end_x), gtimer());
    if (arrived == gridDim.x - 1) {  // every CTA has read the sequence numbers: publish them
      uint32_t* done = kMode == kModeF ? &ctrl->done_f : &ctrl->done_x;
      *done = 0;
      if (kMode != kModeF) st_relaxed_gpu(&ctrl->seq_x, s_seq[0]);
      if (kMode != kModeX) st_relaxed_gpu(&ctrl->seq_f, s_seq[1]);
      if (P.flags & HALO_F_TIMERS) {  // approximate (the last arriver's exit); halo_get_timers uses the trace
        uint64_t* ts = kMode == kModeF ? &ctrl->t_start_f : &ctrl->t_start_x;
        (kMode == kModeF ? ctrl->span_f : ctrl->span_x) = gtimer() - *ts;
        *ts = ~0ull;
        (kMode == kModeF ? ctrl->t_end_f : ctrl->t_end_x) = 0;
      }
    }
  }
  if (trace) ctrl->trace[tslot][blockIdx.x][3] = gtimer();
}

// ------------------------------------------------------------- launchers
cudaError_t launch_coop_kernel_ex(const void* fn, int grid, int block, void** args, cudaStream_t st, bool pdl,
                                  size_t smem, const cudaAccessPolicyWindow* win);

// Narrow x variant (HALO_X_VARIANT): 0 = automatic (one unit per thread for items of
// <= 64 rows, two for larger ones: every load of an item in flight together); 1 = two
// units per thread always; 2 = 64-thread CTAs with 3 units (experiment: the smaller x
// CTAs were meant to let the f launch's CTAs become resident during x, but the register
// file — 64 regs x 256 threads per f CTA — admits only one of them beside the x CTAs;
// measured at C3 1 GPU, A/B: 128-thread CTAs 17.62, 64-thread 18.67 vs 17.36 us/step).
// The fused launch's x items use two units per thread (items of up to 128 rows).
static int g_x_variant = 0;
void ll_set_x_variant(int v) { g_x_variant = v < 0 || v > 2 ? 0 : v; }
template <int W, bool C>
static const void* ll_fn_c(int mode, bool wide, int rows, bool local) {
  if (mode == kModeX && !wide) {
    if (g_x_variant == 2) return (const void*)k_exchange_ll<W, 3, kModeX, C>;
    if (g_x_variant == 1 || rows > 64) return (const void*)k_exchange_ll<W, 2, kModeX, C>;
    return local ? (const void*)k_exchange_ll<W, 1, kModeX, C, true> : (const void*)k_exchange_ll<W, 1, kModeX, C>;
  }
  if (mode == kModeX) return (const void*)k_exchange_ll<W, 4, kModeX, C>;
  if (mode == kModeF && !wide)
    return local ? (const void*)k_exchange_ll<W, 1, kModeF, C, true> : (const void*)k_exchange_ll<W, 1, kModeF, C>;
  if (mode == kModeF) return (const void*)k_exchange_ll<W, 4, kModeF, C>;
  if (wide) return (const void*)k_exchange_ll<W, 4, kModeXF, C>;
  // (pairs of x items only in the local variant: with the LL paths they cost the tree code
  // its registers — 236 B of spills)
  return local ? (const void*)k_exchange_ll<W, 2, kModeXF, C, true> : (const void*)k_exchange_ll<W, 1, kModeXF, C>;
}
template <int W>
static const void* ll_fn(int mode, bool wide, bool chk, int rows, bool local) {
  return chk ? ll_fn_c<W, true>(mode, wide, rows, local) : ll_fn_c<W, false>(mode, wide, rows, local);
}
static const void* ll_fn(int layout, int mode, bool wide, bool chk = false, int rows = 64, bool local = false) {
  return layout == 4 ? ll_fn<4>(mode, wide, chk, rows, local) : ll_fn<3>(mode, wide, chk, rows, local);
}

int ll_block(int mode, bool wide) {
  if (mode != kModeX || wide) return kThreads;
  return g_x_variant == 2 ? 64 : kThreads;
}

// Ring slots (item blocks in flight per CTA) and dynamic shared memory.
// Item blocks in flight per CTA: kRing, two in the wide (bandwidth-regime) variants,
// whose blocks are larger (x 4.2 KiB; f up to 11 KiB with kMaxTreeRows roots): the
// dynamic shared memory stays what the co-resident grid was computed for
// (HALO_RING_F: the f / fused launches' ring, A/B; measured at C4-bw8: 4 is not faster).
static int g_ring_f = 0;
void ll_set_ring_f(int r) { g_ring_f = r <= 0 ? 0 : r < 2 ? 2 : r > kRing ? kRing : r; }
int ll_ring(int mode, bool wide) {
  if (mode != kModeX && g_ring_f) return g_ring_f;
  return wide ? 2 : kRing;
}
size_t ll_smem_bytes(int mode, int rows, int tree_rows, bool wide) {
  const size_t sb = mode == kModeX ? xblk_bytes((uint32_t)rows) : fblk_bytes((uint32_t)tree_rows);
  return (size_t)ll_ring(mode, wide) * sb;
}
uint32_t ll_xblk_bytes(int rows) { return xblk_bytes((uint32_t)rows); }
uint32_t ll_fblk_bytes(int tree_rows) { return fblk_bytes((uint32_t)tree_rows); }

// mode: 0 = x, 1 = f, 2 = fused x+f.  wide = the plan's work items are large
// (bandwidth regime): batched variants.
// chk: the launch is being captured (the epoch-checking variant, kChk).
cudaError_t launch_exchange_ll(const ExParams& p, int mode, int layout, int grid, bool wide,
                               const cudaAccessPolicyWindow* win, cudaStream_t st, bool chk) {
  void* args[] = {(void*)&p};
  return launch_coop_kernel_ex(ll_fn(layout, mode, wide, chk, p.item_rows, p.all_local != 0), grid, ll_block(mode, wide),
                               args, st, true,
                               ll_smem_bytes(mode, p.item_rows, p.tree_rows, wide), win);
}

// Co-resident CTAs per GPU of each mode for the narrow (items <= 128 rows) or
// wide (<= 512) variants, at the largest item size each runs with (a smaller
// launch only fits more).  Also opts the kernels into their dynamic shared memory.
// local_sel: -1 every variant, 0 the variants with LL paths, 1 the hop-group-local ones
// (their register budgets differ: HALO_F_MIN_BLOCKS / HALO_XF_MIN_BLOCKS)
cudaError_t max_coresident_ll(int layout, bool wide, int* blocks /* [4]: x, f, xf, x with 128-row items */,
                              int local_sel) {
  int dev = 0, sms = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  if (e != cudaSuccess) return e;
  const int rows = wide ? kMaxItemRows : 128;
  for (int mode = 0; mode < 4; ++mode) {
    int bmin = 1 << 30;
    const int m = mode == 3 ? 0 : mode, irows = mode == 3 ? 128 : 64;
    for (int v = 0; v < 4; ++v) {  // the grid must fit every variant (eager / captured[, hop-group-local])
      if (local_sel >= 0 && ((v & 2) != 0) != (local_sel == 1)) continue;
      const int chk = v & 1;
      const void* fn = ll_fn(layout, m, wide, chk != 0, irows, (v & 2) != 0);
      e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               (int)ll_smem_bytes(m, kMaxItemRows, kMaxTreeRows, wide));
      if (e != cudaSuccess) return e;
      int b = 0;
      e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, fn, ll_block(m, wide),
                                                        ll_smem_bytes(m, rows, wide ? kMaxTreeRows : kTreeRowsOcc, wide));
      if (e != cudaSuccess) return e;
      bmin = std::min(bmin, b);
    }
    blocks[mode] = bmin * sms;
  }
  return cudaSuccess;
}

}  // namespace halo
