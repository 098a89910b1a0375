// kernels_ll.cu — default ("LL") protocol of the hot path.
//
// The paper signals each pulse with one system-scope release flag issued by
// the last CTA after a completion counter (Alg. 5).  On B200 each
// such hop costs a MEMBAR.SYS per CTA + an atomic + a release store + the
// remote poll.  Here every 8-byte store carries its own 32-bit sequence tag
// next to one fp32 value (single-copy atomic), so:
//   * no fences, counters or flags on the data path;
//   * forwarding is row-level: a dependent row is re-sent as soon as its
//     units arrive (Alg. 4's dependency wait shrinks to the rows actually read);
//   * the force halo is a deterministic GATHER: every target row adds its
//     contributions in descending pulse order (R15) from the LL force buffers,
//     and a halo slice row is pushed back as soon as it is final (Alg. 5
//     DEP_MGMT at row granularity).  Bit-exact with the oracle, no atomics.
//
//   * a receiver on the same GPU (a DD rank of this process) gets its halo
//     rows stored directly by the sender; only rows from other GPUs go through
//     receive items (LL units -> x);
//   * shift forces: per-item fp64 partials of the pushers, one deterministic
//     combine per (rank, wrapped dim) in its own CTA.
//
// One kernel body serves three launches (kMode): the x halo, the f halo, and
// both in ONE launch (halo_exchange_xf; "a single kernel for
// x+f when no compute sits between them") in which the f items of a DD rank
// start once that rank's halo rows are complete (per-rank item counter, the
// place of the non-bonded kernel between the two exchanges, Alg. 2).
//
// Each CTA runs a static list of work items; every item is one contiguous
// block in HBM (128-B XRec / GRec + map slice / task records).  A ring of
// kRing shared-memory slots is filled by bulk (TMA) copies completing on
// mbarriers: the first blocks are requested before griddepcontrol.wait (static
// plan data, overlapped with the previous kernel's drain), and the block of
// item j+ring is requested as soon as item j is done, so a CTA that runs
// several items pays the cold-HBM round trip for its plan once.  Items are
// processed in a static order in which every wait targets an earlier item
// (DESIGN.md §6); the grid never exceeds the co-resident CTA count.
#include <cuda_runtime.h>
#include <stdint.h>

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
template <int W, int kU>
__device__ __forceinline__ void x_item(const XRec& r, const int32_t* s_map, const ExParams& P, uint32_t tag) {
  const uint32_t n = r.n_units;
  const uint32_t B = blockDim.x;
  if (r.kind == kItemXRecv) {
    // this rank's halo rows of one pulse from another GPU: LL units -> x rows;
    // 4 units per thread per batch: the polls of a batch are in flight together
    constexpr int kR = 4;
    for (uint32_t base = threadIdx.x; base < n; base += kR * B) {
      uint64_t w[kR];
#pragma unroll
      for (int k = 0; k < kR; ++k)
        if (base + k * B < n) w[k] = ld_relaxed_sys(r.ll + base + k * B);
#pragma unroll
      for (int k = 0; k < kR; ++k) {
        const uint32_t u = base + k * B;
        if (u >= n) continue;
        if ((uint32_t)(w[k] >> 32) != tag && !(P.debug & kLocalSink))
          w[k] = ll_spin(r.ll + u, tag, P.timeout_ns, P.err_host, tcode(10, r.lrank, r.pulse), P.poll_ns);
        r.xdst[u] = __uint_as_float((uint32_t)w[k]);
      }
    }
  } else if (r.kind == kItemXIndep) {
    // SEND of home rows: gather through the map, shift (R25), tag, store into the receiver's LL slot
    for (uint32_t base = threadIdx.x; base < n; base += kU * B) {
      float v[kU];
#pragma unroll
      for (int k = 0; k < kU; ++k) {
        const uint32_t u = base + k * B;
        if (u < n) {
          const uint32_t i = u / W;
          v[k] = __ldg(r.x + (size_t)s_map[i] * W + (u - i * W));  // home row: never written during the kernel
        }
      }
#pragma unroll
      for (int k = 0; k < kU; ++k) {
        const uint32_t u = base + k * B;
        if (u >= n) continue;
        const int c = (int)(u % W);
        const float o = (r.has_shift && c < 3) ? __fadd_rn(v[k], r.shift[c]) : v[k];
        uint64_t* dst = (P.debug & kLocalSink) ? const_cast<uint64_t*>(r.xll_own) + (size_t)r.pulse * P.ll_stride + u
                                               : r.ll + u;
        st_relaxed_sys(dst, ll_pack(o, tag));
        if (r.xdst) r.xdst[u] = o;  // same-process receiver: its halo row directly (kernel end publishes it)
      }
    }
  } else {
    // SEND of forwarded rows: the pulse each arrived in (Alg. 4 dependent part, R8/R9);
    // the row-level wait is the LL tag of the source unit
    for (uint32_t base = threadIdx.x; base < n; base += kU * B) {
      uint64_t w[kU];
      const uint64_t* src[kU];
#pragma unroll
      for (int k = 0; k < kU; ++k) {
        const uint32_t u = base + k * B;
        src[k] = nullptr;
        if (u < n) {
          const uint32_t i = u / W;
          const int c = (int)(u - i * W);
          const int idx = s_map[i];
          int q = 0;
          while (q < P.P - 1 && (unsigned)(idx - r.recv_off[q]) >= (unsigned)r.recv_size[q]) ++q;
          if (q < P.p_lo || (P.debug & kMutateXNoWait)) {
            // arrived in an earlier launch (set_maps); kMutateXNoWait: the protocol
            // mutation the sentinel tests must catch (forward without waiting)
            w[k] = ((uint64_t)tag << 32) | __float_as_uint(__ldcg(r.x + (size_t)idx * W + c));
          } else {
            src[k] = r.xll_own + (size_t)q * P.ll_stride + (size_t)(idx - r.recv_off[q]) * W + c;
            w[k] = ld_relaxed_sys(src[k]);
          }
        }
      }
#pragma unroll
      for (int k = 0; k < kU; ++k) {
        const uint32_t u = base + k * B;
        if (u >= n) continue;
        if (src[k] != nullptr && (uint32_t)(w[k] >> 32) != tag && !(P.debug & kLocalSink))
          w[k] = ll_spin(src[k], tag, P.timeout_ns, P.err_host, tcode(11, r.lrank, r.pulse), P.poll_ns);
        const int c = (int)(u % W);
        float v = __uint_as_float((uint32_t)w[k]);
        if (r.has_shift && c < 3) v = __fadd_rn(v, r.shift[c]);
        uint64_t* dst = (P.debug & kLocalSink) ? const_cast<uint64_t*>(r.xll_own) + (size_t)r.pulse * P.ll_stride + u
                                               : r.ll + u;
        st_relaxed_sys(dst, ll_pack(v, tag));
        if (r.xdst) r.xdst[u] = v;
      }
    }
  }
  // experiment (HALO_DEBUG=128): drain this thread's peer stores inside the item
  if ((P.debug & kFenceAfterPeerStores) && r.kind != kItemXRecv) fence_sys();
}

// ---------------------------------------------------------------- f items
__device__ __forceinline__ double warp_sum_d(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// threads per CTA of the LL kernels (HALO_F_THREADS build switch for the A/B)
#ifndef HALO_F_THREADS
#define HALO_F_THREADS 256
#endif
constexpr int kThreadsF = HALO_F_THREADS;
static_assert(kThreadsF == kThreads || HALO_F_THREADS != 256, "LL CTA size");

// Deterministic CTA reduction of N outputs held per thread in s_red[j][tid]:
// output j is summed by warp (j mod warps), each lane over a fixed strided slice
// of the threads, then a fixed xor-shuffle tree; threads j < N return output j.
// Every thread has passed the __syncthreads before any shuffle, so no lane
// waits for another's polling loop (a full-mask SHFL right after the divergent
// polling loop had cost ~10 us per level at C3); 2 barriers instead of the 9 of
// a pairwise shared-memory tree.
template <int N>
__device__ __noinline__ double cta_reduce(double (*s_red)[kThreadsF], int j_out) {
  __shared__ double s_out[9];
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = (int)(blockDim.x >> 5);
  for (int j = warp; j < N; j += nw) {
    double v = 0.0;
    for (int t = lane; t < kThreadsF; t += 32) v += s_red[j][t];
    v = warp_sum_d(v);
    if (lane == 0) s_out[j] = v;
  }
  __syncthreads();
  const double tot = (j_out < N) ? s_out[j_out] : 0.0;
  __syncthreads();
  return tot;
}

// Combine item of one rank (R13): the pushers of its wrapping pulses summed,
// per work item, the forces they pushed back to it (3 doubles per slot as tagged
// LL units: no flag, no fence).  One thread per (pulse, slot, component) triple
// in a fixed assignment, then a fixed tree: deterministic, no atomics; only this
// CTA writes the rank's fshift[dim].
__device__ __noinline__ void fshift_combine(const GRec& g, const ExParams& P, uint32_t tag, double (*s_red)[kThreadsF],
                                            uint32_t fsp_slots) {
  const int dim = g.level;
  const bool f32 = (P.debug & kMutateFshiftF32) != 0;  // mutation: fp32 accumulation
  const double fs_old = (threadIdx.x < 3) ? P.fshift[9 * g.lrank + 3 * dim + threadIdx.x] : 0.0;
#pragma unroll
  for (int j = 0; j < 3; ++j) s_red[j][threadIdx.x] = 0.0;
  // one flat index space over (pulse, slot, component) triples; every load of a
  // thread is issued before any wait is resolved
  uint32_t off[kMaxP + 1];
  off[0] = 0;
#pragma unroll
  for (int q = 0; q < kMaxP; ++q) off[q + 1] = off[q] + (q < P.P ? g.nslot[q] * 3 : 0u);
  const uint32_t n = off[kMaxP];
  constexpr int kB = 4;
  for (uint32_t base = threadIdx.x; base < n; base += kB * blockDim.x) {
    const uint64_t* ptr[kB];
    uint64_t hv[kB], lv[kB];
    int dc[kB];
#pragma unroll
    for (int k = 0; k < kB; ++k) {
      const uint32_t e = base + k * blockDim.x;
      ptr[k] = nullptr;
      if (e < n) {
        int q = 0;
        while (e >= off[q + 1]) ++q;
        const uint32_t pp = e - off[q];  // slot * 3 + component
        ptr[k] = g.part + (size_t)q * fsp_slots * 6 + 2 * (size_t)pp;
        dc[k] = (int)(pp % 3);  // component (the item's pulses all shift along `dim`)
        hv[k] = ld_relaxed_sys(ptr[k]);
        lv[k] = ld_relaxed_sys(ptr[k] + 1);
      }
    }
#pragma unroll
    for (int k = 0; k < kB; ++k) {
      if (ptr[k] == nullptr) continue;
      if ((uint32_t)(hv[k] >> 32) != tag) hv[k] = ll_spin(ptr[k], tag, P.timeout_ns, P.err_host, tcode(13, g.lrank, 0), 0);
      if ((uint32_t)(lv[k] >> 32) != tag) lv[k] = ll_spin(ptr[k] + 1, tag, P.timeout_ns, P.err_host, tcode(13, g.lrank, 1), 0);
      const double v = __hiloint2double((int)(uint32_t)hv[k], (int)(uint32_t)lv[k]);
      double& a = s_red[dc[k]][threadIdx.x];
      a = f32 ? (double)((float)a + (float)v) : a + v;
    }
  }
  const double tot = cta_reduce<3>(s_red, threadIdx.x);
  if (threadIdx.x < 3)
    P.fshift[9 * g.lrank + 3 * dim + threadIdx.x] = f32 ? (double)((float)fs_old + (float)tot) : fs_old + tot;
}

// One gather item: every task row adds its contributions from the force LL
// buffers in descending pulse order (R15: bit-exact with the oracle), is
// written back, and — slice rows — pushed to the x-sender's force LL buffer at
// once (Alg. 5 DEP_MGMT at row granularity).  The pushers of a slice whose
// x-sender shifted also sum what they push (fixed tree) into its slot (R13).
// kF = units per thread per batch (1: latency regime, 2: large items).
template <int W, int kF>
__device__ __forceinline__ void f_item(const GRec& g, const int4* tasks, const ExParams& P, uint32_t tag,
                                       double (*s_fs)[kThreadsF]) {
  const uint32_t n = g.n_units;
  const bool push = g.level != kHomeLevel;
  const bool part = (P.fshift != nullptr) && (g.part != nullptr) && !(P.debug & kLocalSink);
  // stride = a multiple of W: every thread keeps one component c
  const uint32_t S = (blockDim.x / W) * W;
  const int c = (int)(threadIdx.x % W);
  double acc = 0.0;
  if (threadIdx.x < S) {
    // task records, f and the contributions of a batch are loaded before any
    // wait or store
    for (uint32_t base = threadIdx.x; base < n; base += kF * S) {
      int4 a[kF], b[kF];
#pragma unroll
      for (int k = 0; k < kF; ++k) {
        const uint32_t u = base + k * S;
        if (u >= n) continue;
        a[k] = tasks[2 * (u / W)];
        b[k] = tasks[2 * (u / W) + 1];
      }
      // contributions j < kPre are loaded with the batch, any further ones (more
      // than kPre pulses touching one row) when resolved
      constexpr int kPre = 3;
      float v[kF];
      uint64_t w[kF][kPre];
#pragma unroll
      for (int k = 0; k < kF; ++k) {
        const uint32_t u = base + k * S;
        if (u >= n) continue;
        const uint32_t cc[kMaxP] = {(uint32_t)a[k].z, (uint32_t)a[k].w, (uint32_t)b[k].x,
                                    (uint32_t)b[k].y, (uint32_t)b[k].z, (uint32_t)b[k].w};
        v[k] = g.f[(size_t)a[k].x * W + c];
#pragma unroll
        for (int j = 0; j < kPre; ++j)
          if (j < a[k].y)
            w[k][j] = ld_relaxed_sys(g.fll_own + (size_t)(cc[j] >> 24) * P.ll_stride + (size_t)(cc[j] & 0xffffffu) * W + c);
      }
#pragma unroll
      for (int k = 0; k < kF; ++k) {
        const uint32_t u = base + k * S;
        if (u >= n) continue;
        const int t = a[k].x, m = a[k].y;
        const uint32_t cc[kMaxP] = {(uint32_t)a[k].z, (uint32_t)a[k].w, (uint32_t)b[k].x,
                                    (uint32_t)b[k].y, (uint32_t)b[k].z, (uint32_t)b[k].w};
        float vv = v[k];
#pragma unroll
        for (int j = 0; j < kMaxP; ++j) {
          if (j < m) {  // pulses descending (R15): one fp32 RNE add per (entry, pulse)
            const int q = (int)(cc[j] >> 24);
            const uint64_t* src = g.fll_own + (size_t)q * P.ll_stride + (size_t)(cc[j] & 0xffffffu) * W + c;
            uint64_t wj = j < kPre ? w[k][j < kPre ? j : 0] : ld_relaxed_sys(src);
            if ((uint32_t)(wj >> 32) != tag && !(P.debug & (kMutateFNoWait | kLocalSink)))
              wj = ll_spin(src, tag, P.timeout_ns, P.err_host, tcode(12, g.lrank, q), P.poll_ns);
            const float val = __uint_as_float((uint32_t)wj);
            vv = P.accumulate ? __fadd_rn(vv, val) : val;
          }
        }
        g.f[(size_t)t * W + c] = vv;
        if (push)
          st_relaxed_sys((P.debug & kLocalSink) ? const_cast<uint64_t*>(g.fll_own) + (size_t)t * W + c
                                                : g.push + (size_t)t * W + c,
                         ll_pack(vv, tag));
        if (part) acc += (double)vv;
      }
    }
  }
  if ((P.debug & kFenceAfterPeerStores) && push) fence_sys();  // experiment (HALO_DEBUG=128)
  if (part) {  // fixed-tree CTA sum of the pushed forces per component -> the x-sender's slot
#pragma unroll
    for (int j = 0; j < 3; ++j) s_fs[j][threadIdx.x] = (threadIdx.x < S && c == j) ? acc : 0.0;
    double tot = cta_reduce<3>(s_fs, threadIdx.x);
    if (P.debug & kMutateFshiftF32) tot = (double)(float)tot;  // mutation: fp32 partials
    if (threadIdx.x < 3) {
      st_relaxed_sys(g.part + 2 * threadIdx.x, ll_pack(__uint_as_float((uint32_t)__double2hiint(tot)), tag));
      st_relaxed_sys(g.part + 2 * threadIdx.x + 1, ll_pack(__uint_as_float((uint32_t)__double2loint(tot)), tag));
    }
  }
}

// Fused launch: a gather item of rank l waits until every x item that completes
// l's halo rows (same-GPU senders' direct rows, receive items) has finished in
// this launch — the position of the non-bonded kernel between exchange_x and
// exchange_f (Alg. 2).  Counters are monotonic within an NS epoch (zeroed by
// set_maps; every LL x launch of the epoch adds its items), so the target of
// this launch is xin_n * (x launches of the epoch up to this one).  Bounded.
__device__ __noinline__ void xin_wait(const uint64_t* cnt, uint64_t target, const ExParams& P, int lrank) {
  const uint64_t t0 = gtimer();
  for (uint32_t it = 1;; ++it) {
    if (ld_relaxed_gpu(cnt) >= target) return;
    if ((it & 15u) == 0) {
      const uint64_t el = gtimer() - t0;
      if (el > 20000) __nanosleep(256);
      if ((it & 1023u) == 0) {
        if (el > P.timeout_ns) {
          report_timeout(P.err_host, tcode(15, lrank, 0));
          return;
        }
        if (*(volatile int*)P.err_host != 0) return;
      }
    }
  }
}

__device__ __forceinline__ void red_add_gpu(uint64_t* p, uint64_t v) {
  asm volatile("red.relaxed.gpu.global.add.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

// ---------------------------------------------------------------- kernel
enum : int { kModeX = 0, kModeF = 1, kModeXF = 2 };

// Items of this CTA: [0, n_main) round-robin over CTAs [0, G - n_tail) (fused:
// the x items first, then the f items), the n_tail shift-force combines (last in
// the item order) one dedicated CTA each, so they start polling at once.
template <int W, int kU, int kF, int kMode>
__global__ void __launch_bounds__(kThreads, kMode == kModeX ? (kU == 1 ? 8 : 4) : (kF == 1 ? 5 : 4)) k_exchange_ll(
    const __grid_constant__ ExParams P) {
  extern __shared__ __align__(128) unsigned char s_blk[];
  __shared__ uint64_t s_seq[2];
  __shared__ __align__(8) uint64_t s_bar[kRing];
  __shared__ double s_fs[kMode == kModeX ? 1 : 3][kMode == kModeX ? 1 : kThreadsF];
  const uint32_t R = (uint32_t)P.item_rows;
  const uint32_t XB = 128u + 4u * R, FB = 128u + 32u * R;
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
  // the first `ring` blocks are static plan data: bulk copies issued while the
  // previous kernel of the stream drains (PDL); x, f, LL are touched after the wait
  if (threadIdx.x == 0) {
    for (int k = 0; k < ring; ++k) mbar_init(&s_bar[k], 1);
    fence_mbar_init();
    for (int k = 0, i = first; k < ring && i < end; ++k, i += stride)
      bulk_load(s_blk + (size_t)k * SB, blk_of(i), bytes_of(i), &s_bar[k]);
  }
  pdl_wait();  // everything below may depend on earlier work of the stream
  // by value when the host knows them (no cold dependent load on the critical path)
  if (threadIdx.x == 0) {
    if (kMode != kModeF) s_seq[0] = P.seq ? P.seq : ld_relaxed_gpu(&ctrl->seq_x) + 1;
    if (kMode != kModeX) s_seq[1] = P.seq_f ? P.seq_f : ld_relaxed_gpu(&ctrl->seq_f) + 1;
  }
  timer_start(P.flags, kMode == kModeF ? &ctrl->t_start_f : &ctrl->t_start_x);
  __syncthreads();  // barrier init and sequence numbers visible to every thread
  // arrive early: the atomic's latency hides behind the items (launch_arrive)
  const uint32_t arrived = launch_arrive(kMode == kModeF ? &ctrl->done_f : &ctrl->done_x);
  const uint32_t tag_x = (uint32_t)s_seq[0], tag_f = (uint32_t)s_seq[1];
  int j = 0;
  for (int it = first; it < end; it += stride, ++j) {
    const int slot = j % ring;
    unsigned char* blk = s_blk + (size_t)slot * SB;
    mbar_wait(&s_bar[slot], (uint32_t)(j / ring) & 1u);
    if (trace && j == 0) ctrl->trace[tslot][blockIdx.x][1] = gtimer();
    if (kMode != kModeF && it < nx) {
      const XRec& r = *reinterpret_cast<const XRec*>(blk);
      x_item<W, kU>(r, reinterpret_cast<const int32_t*>(blk + 128), P, tag_x);
      __syncthreads();  // the item's rows are stored (fused: before its count) and the slot is free
      if (threadIdx.x == 0 && r.xin != nullptr) red_add_gpu(r.xin, 1u);
    } else if constexpr (kMode != kModeX) {
      const GRec& g = *reinterpret_cast<const GRec*>(blk);
      if (kMode == kModeXF && g.xin != nullptr) {  // this rank's halo is complete (the NB kernel's slot)
        if (threadIdx.x == 0) xin_wait(g.xin, (uint64_t)g.xin_n * (s_seq[0] - P.seq_x0), P, g.lrank);
        __syncthreads();
      }
      if (g.kind == kItemFshift) {
        if (P.fshift != nullptr) fshift_combine(g, P, tag_f, s_fs, P.fsp_slots);
      } else {
        f_item<W, kF>(g, reinterpret_cast<const int4*>(blk + 128), P, tag_f, s_fs);
      }
      __syncthreads();  // everyone is done with this slot
    }
    if (trace && j < (kTraceW - 4) / 2) {
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

template <int W>
static const void* ll_fn(int mode, bool wide) {
  if (mode == kModeX) return wide ? (const void*)k_exchange_ll<W, 4, 2, kModeX> : (const void*)k_exchange_ll<W, 1, 1, kModeX>;
  if (mode == kModeF) return wide ? (const void*)k_exchange_ll<W, 4, 2, kModeF> : (const void*)k_exchange_ll<W, 1, 1, kModeF>;
  return wide ? (const void*)k_exchange_ll<W, 4, 2, kModeXF> : (const void*)k_exchange_ll<W, 1, 1, kModeXF>;
}
static const void* ll_fn(int layout, int mode, bool wide) { return layout == 4 ? ll_fn<4>(mode, wide) : ll_fn<3>(mode, wide); }

// Ring slots (item blocks in flight per CTA) and dynamic shared memory.
int ll_ring(bool wide) { return wide ? 2 : kRing; }
size_t ll_smem_bytes(int mode, int rows, bool wide) {
  const size_t sb = mode == kModeX ? 128 + 4 * (size_t)rows : 128 + 32 * (size_t)rows;
  return (size_t)ll_ring(wide) * sb;
}

// mode: 0 = x, 1 = f, 2 = fused x+f.  wide = the plan's work items are large
// (bandwidth regime): batched variants.
cudaError_t launch_exchange_ll(const ExParams& p, int mode, int layout, int grid, bool wide,
                               const cudaAccessPolicyWindow* win, cudaStream_t st) {
  void* args[] = {(void*)&p};
  return launch_coop_kernel_ex(ll_fn(layout, mode, wide), grid, kThreads, args, st, true,
                               ll_smem_bytes(mode, p.item_rows, wide), win);
}

// Co-resident CTAs per GPU of each mode for the narrow (items <= 128 rows) or
// wide (<= 512) variants, at the largest item size each runs with (a smaller
// launch only fits more).  Also opts the kernels into their dynamic shared memory.
cudaError_t max_coresident_ll(int layout, bool wide, int* blocks /* [3]: x, f, xf */) {
  int dev = 0, sms = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  if (e != cudaSuccess) return e;
  const int rows = wide ? kMaxItemRows : 128;
  for (int mode = 0; mode < 3; ++mode) {
    const void* fn = ll_fn(layout, mode, wide);
    e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)ll_smem_bytes(mode, kMaxItemRows, wide));
    if (e != cudaSuccess) return e;
    int b = 0;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, fn, kThreads, ll_smem_bytes(mode, rows, wide));
    if (e != cudaSuccess) return e;
    blocks[mode] = b * sms;
  }
  return cudaSuccess;
}

}  // namespace halo
