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
// Each CTA loads one work-item block (128-B XRec / GRec + map slice / task
// records) per item with one bulk (TMA) copy on an mbarrier, the next one
// while it processes the current: after an L2 flush the plan costs one memory
// round trip, not a chain of dependent loads.  Items are processed in a static
// order in which every wait targets an earlier item, every CTA
// of the grid is co-resident, and launches use programmatic dependent launch.
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

// ---------------------------------------------------------------- x (LL)
// kU = units per thread per batch: 1 for the latency regime (64-row items, at
// most one unit per thread; fewest registers = most co-resident CTAs), 4 for
// large items (bandwidth regime: every load of a batch is issued before any
// store — the stores are asm volatile with a memory clobber, so one unit at a
// time would serialise a full memory latency per unit).
template <int W, int kU>
__global__ void __launch_bounds__(kThreads) k_exchange_x_ll(const __grid_constant__ ExParams P) {
  // two item blocks [XRec | map slice of item_rows ints], double-buffered: the
  // next item's block is fetched (cp.async) while the current one is processed
  extern __shared__ __align__(128) unsigned char s_blk[];
  __shared__ uint64_t s_seq;
  __shared__ __align__(8) uint64_t s_bar[2];  // one mbarrier per item-block buffer
  const uint32_t XB = 128u + 4u * (uint32_t)P.item_rows;
  Ctrl* ctrl = P.ctrl;
  const bool trace = (P.flags & HALO_F_TIMERS) && threadIdx.x == 0 && blockIdx.x < kTraceCTAs;
  if (trace) ctrl->trace[0][blockIdx.x][0] = gtimer();
  pdl_launch_dependents();
  // the first block is static plan data: one bulk (TMA) copy, issued while the
  // previous kernel drains (PDL)
  if (threadIdx.x == 0) {
    mbar_init(&s_bar[0], 1);
    mbar_init(&s_bar[1], 1);
    fence_mbar_init();
    if ((int)blockIdx.x < P.n_items) bulk_load(s_blk, P.xblk + (size_t)blockIdx.x * XB, XB, &s_bar[0]);
  }
  uint32_t phase = 0u;  // bit b = the parity to wait for on s_bar[b] (a register, not an indexed array)
  pdl_wait();  // everything below may depend on earlier work of the stream
  // by value when the host knows it (no cold dependent load on the critical path)
  if (threadIdx.x == 0) s_seq = P.seq ? P.seq : ld_relaxed_gpu(&ctrl->seq_x) + 1;
  timer_start(P.flags, &ctrl->t_start_x);
  __syncthreads();  // barrier init visible to every thread
  if ((int)blockIdx.x < P.n_items) {
    mbar_wait(&s_bar[0], phase & 1u);
    phase ^= 1u;
  }
  // arrive early: the atomic's latency hides behind the items (launch_arrive)
  const uint32_t arrived = launch_arrive(&ctrl->done_x);
  uint64_t seq = 0;
  int cur = 0;
  for (int it = blockIdx.x; it < P.n_items; it += gridDim.x) {
    const bool more = it + (int)gridDim.x < P.n_items;
    if (more && threadIdx.x == 0) {
      fence_proxy_async_smem();  // generic reads of that buffer (previous item) before the async write
      bulk_load(s_blk + (cur ^ 1) * XB, P.xblk + (size_t)(it + gridDim.x) * XB, XB, &s_bar[cur ^ 1]);
    }
    const XRec& r = *reinterpret_cast<const XRec*>(s_blk + cur * XB);
    const int32_t* s_map = reinterpret_cast<const int32_t*>(s_blk + cur * XB + 128);
    if (trace && seq == 0) ctrl->trace[0][blockIdx.x][1] = gtimer();
    seq = s_seq;
    const uint32_t tag = (uint32_t)seq;
    const uint32_t n = r.n_units;
    const uint32_t B = blockDim.x;
    if (r.kind == kItemXRecv) {
      // this rank's halo rows of one pulse from another GPU: LL units -> x rows
      // (HALO_RECV_MULT x the send item rows, default 1); 4 units per thread per
      // batch: the polls of a batch are in flight together.
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
    if (trace) {
      const int slot = (it - (int)blockIdx.x) / (int)gridDim.x;
      if (slot < 2) {
        ctrl->trace[0][blockIdx.x][4 + 2 * slot] = ((uint64_t)r.kind << 16) | ((uint64_t)r.lrank << 8) | r.pulse;
        ctrl->trace[0][blockIdx.x][5 + 2 * slot] = gtimer();
      }
    }
    if (more) {  // the next block has landed
      mbar_wait(&s_bar[cur ^ 1], (phase >> (cur ^ 1)) & 1u);
      phase ^= 1u << (cur ^ 1);
    }
    __syncthreads();  // everyone is done with this block before it is refilled
    cur ^= 1;
  }
  seq = s_seq;
  if (trace) ctrl->trace[0][blockIdx.x][2] = gtimer();
  launch_depart(P.flags, arrived, &ctrl->done_x, &ctrl->seq_x, seq, &ctrl->t_start_x, &ctrl->t_end_x, &ctrl->span_x);
  if (trace) ctrl->trace[0][blockIdx.x][3] = gtimer();
}

// ---------------------------------------------------------------- f (LL)
__device__ __forceinline__ double warp_sum_d(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Deterministic CTA reduction of N outputs held per thread in s_red[j][tid]:
// output j is summed by warp (j mod warps), each lane over a fixed strided slice
// of the threads, then a fixed xor-shuffle tree; threads j < N return output j.
// Every thread has passed the __syncthreads before any shuffle, so no lane
// waits for another's polling loop (a full-mask SHFL right after the divergent
// polling loop had cost ~10 us per level at C3); 2 barriers instead of the 9 of
// a pairwise shared-memory tree.
// threads per CTA of the f kernel (HALO_F_THREADS_128 build switch for the A/B)
#ifndef HALO_F_THREADS
#define HALO_F_THREADS 256
#endif
constexpr int kThreadsF = HALO_F_THREADS;

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
// CTA writes the rank's fshift.
__device__ __noinline__ void fshift_combine(const GRec& g, const ExParams& P, uint32_t tag, double (*s_red)[kThreadsF],
                                            uint32_t fsp_slots) {
  // one combine per (rank, dim g.level): only this CTA writes fshift[dim][0..2]:
  // read it now, off the tail
  const int dim = g.level;
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
      s_red[dc[k]][threadIdx.x] = (P.debug & kMutateFshiftF32) ? (double)((float)s_red[dc[k]][threadIdx.x] + (float)v)
                                                                : s_red[dc[k]][threadIdx.x] + v;
    }
  }
  const double tot = cta_reduce<3>(s_red, threadIdx.x);
  if (threadIdx.x < 3)
    P.fshift[9 * g.lrank + 3 * dim + threadIdx.x] =
        (P.debug & kMutateFshiftF32) ? (double)((float)fs_old + (float)tot) : fs_old + tot;
}

// kF = units per thread per batch (1: latency regime, 2: large items), as kU above.
template <int W, int kF>
__global__ void __launch_bounds__(kThreadsF, kF == 1 ? 5 * 256 / kThreadsF : 4 * 256 / kThreadsF) k_exchange_f_ll(
    const __grid_constant__ ExParams P) {
  // two item blocks [GRec | task records of item_rows rows (32 B each)], double-
  // buffered like the x kernel's
  extern __shared__ __align__(128) unsigned char s_blk[];
  __shared__ uint64_t s_seq;
  __shared__ __align__(8) uint64_t s_bar[2];  // one mbarrier per item-block buffer
  __shared__ double s_fs[3][kThreadsF];
  const uint32_t FB = 128u + 32u * (uint32_t)P.item_rows;
  Ctrl* ctrl = P.ctrl;
  const bool trace = (P.flags & HALO_F_TIMERS) && threadIdx.x == 0 && blockIdx.x < kTraceCTAs;
  if (trace) ctrl->trace[1][blockIdx.x][0] = gtimer();
  pdl_launch_dependents();
  // items [0, n_main) round-robin over CTAs [0, G - n_tail); the n_tail shift-force
  // combines (last in the item order) get one dedicated CTA each, so they start
  // polling at once instead of behind their CTA's earlier items
  const int n_main = P.n_items - P.n_tail;
  const int Gm = (int)gridDim.x - P.n_tail;
  const int first = ((int)blockIdx.x < Gm) ? (int)blockIdx.x : n_main + ((int)blockIdx.x - Gm);
  const int stride = ((int)blockIdx.x < Gm) ? Gm : P.n_items;
  const int end = ((int)blockIdx.x < Gm) ? n_main : P.n_items;
  // the first block is static plan data: fetched while the previous kernel of the
  // stream drains (PDL); f itself is read after the wait
  if (threadIdx.x == 0) {
    mbar_init(&s_bar[0], 1);
    mbar_init(&s_bar[1], 1);
    fence_mbar_init();
    if (first < end) bulk_load(s_blk, P.fblk + (size_t)first * FB, FB, &s_bar[0]);
  }
  uint32_t phase = 0u;  // bit b = the parity to wait for on s_bar[b] (a register, not an indexed array)
  pdl_wait();
  if (threadIdx.x == 0) s_seq = P.seq ? P.seq : ld_relaxed_gpu(&ctrl->seq_f) + 1;
  timer_start(P.flags, &ctrl->t_start_f);
  __syncthreads();
  if (first < end) {
    mbar_wait(&s_bar[0], phase & 1u);
    phase ^= 1u;
  }
  const uint32_t arrived = launch_arrive(&ctrl->done_f);
  uint64_t seq = 0;
  int cur = 0;
  for (int it = first; it < end; it += stride) {
    const bool more = it + stride < end;
    if (more && threadIdx.x == 0) {
      fence_proxy_async_smem();
      bulk_load(s_blk + (cur ^ 1) * FB, P.fblk + (size_t)(it + stride) * FB, FB, &s_bar[cur ^ 1]);
    }
    const GRec& g = *reinterpret_cast<const GRec*>(s_blk + cur * FB);
    const int4* tasks = reinterpret_cast<const int4*>(s_blk + cur * FB + 128);
    if (trace && seq == 0) ctrl->trace[1][blockIdx.x][1] = gtimer();
    seq = s_seq;
    const uint32_t tag = (uint32_t)seq;
    if (g.kind == kItemFshift) {
      if (P.fshift != nullptr) fshift_combine(g, P, tag, s_fs, P.fsp_slots);
      if (trace) {
        const int slot = (it - first) / stride;
        if (slot < 2) {
          ctrl->trace[1][blockIdx.x][4 + 2 * slot] = ((uint64_t)g.kind << 16) | ((uint64_t)g.lrank << 8) | g.level;
          ctrl->trace[1][blockIdx.x][5 + 2 * slot] = gtimer();
        }
      }
      if (more) {
        mbar_wait(&s_bar[cur ^ 1], (phase >> (cur ^ 1)) & 1u);
        phase ^= 1u << (cur ^ 1);
      }
      __syncthreads();
      cur ^= 1;
      continue;
    }
    const uint32_t n = g.n_units;
    const bool push = g.level != kHomeLevel;
    // this item also sums what it pushes when the receiving x-sender shifted (R13)
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
    if (trace) {
      const int slot = (it - first) / stride;
      if (slot < 2) {
        ctrl->trace[1][blockIdx.x][4 + 2 * slot] = ((uint64_t)g.kind << 16) | ((uint64_t)g.lrank << 8) | g.level;
        ctrl->trace[1][blockIdx.x][5 + 2 * slot] = gtimer();
      }
    }
    if (more) {
      mbar_wait(&s_bar[cur ^ 1], (phase >> (cur ^ 1)) & 1u);
      phase ^= 1u << (cur ^ 1);
    }
    __syncthreads();
    cur ^= 1;
  }
  seq = s_seq;
  if (trace) ctrl->trace[1][blockIdx.x][2] = gtimer();
  launch_depart(P.flags, arrived, &ctrl->done_f, &ctrl->seq_f, seq, &ctrl->t_start_f, &ctrl->t_end_f, &ctrl->span_f);
  if (trace) ctrl->trace[1][blockIdx.x][3] = gtimer();
}

// ------------------------------------------------------------- launchers
cudaError_t launch_coop_kernel_ex(const void* fn, int grid, int block, void** args, cudaStream_t st, bool pdl,
                                  size_t smem, const cudaAccessPolicyWindow* win);

template <int W>
static const void* x_fn(bool wide) {
  return wide ? (const void*)k_exchange_x_ll<W, 4> : (const void*)k_exchange_x_ll<W, 1>;
}
template <int W>
static const void* f_fn(bool wide) {
  return wide ? (const void*)k_exchange_f_ll<W, 2> : (const void*)k_exchange_f_ll<W, 1>;
}

// Dynamic shared memory of the LL kernels: two item blocks.
size_t x_smem_bytes(int rows) { return 2 * (128 + 4 * (size_t)rows); }
size_t f_smem_bytes(int rows) { return 2 * (128 + 32 * (size_t)rows); }

// wide = the plan's work items are large (bandwidth regime): batched variants
cudaError_t launch_exchange_x_ll(const ExParams& p, int layout, int grid, bool wide, const cudaAccessPolicyWindow* win,
                                 cudaStream_t st) {
  void* args[] = {(void*)&p};
  return launch_coop_kernel_ex(layout == 4 ? x_fn<4>(wide) : x_fn<3>(wide), grid, kThreads, args, st, true,
                               x_smem_bytes(p.item_rows), win);
}

cudaError_t launch_exchange_f_ll(const ExParams& p, int layout, int grid, bool wide, const cudaAccessPolicyWindow* win,
                                 cudaStream_t st) {
  void* args[] = {(void*)&p};
  return launch_coop_kernel_ex(layout == 4 ? f_fn<4>(wide) : f_fn<3>(wide), grid, kThreadsF, args, st, true,
                               f_smem_bytes(p.item_rows), win);
}

// Co-resident CTAs per GPU for the narrow (items <= 128 rows) or wide (<= 512)
// variants, at the largest item size each runs with (a smaller launch only fits
// more).  Also opts the kernels into their dynamic shared memory.
cudaError_t max_coresident_ll(int layout, bool wide, int* x_blocks, int* f_blocks) {
  int dev = 0, sms = 0, bx = 0, bf = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  if (e != cudaSuccess) return e;
  const int rows = wide ? kMaxItemRows : 128;
  const void* fx = layout == 4 ? x_fn<4>(wide) : x_fn<3>(wide);
  const void* ff = layout == 4 ? f_fn<4>(wide) : f_fn<3>(wide);
  e = cudaFuncSetAttribute(fx, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)x_smem_bytes(kMaxItemRows));
  if (e != cudaSuccess) return e;
  e = cudaFuncSetAttribute(ff, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)f_smem_bytes(kMaxItemRows));
  if (e != cudaSuccess) return e;
  e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bx, fx, kThreads, x_smem_bytes(rows));
  if (e != cudaSuccess) return e;
  e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bf, ff, kThreadsF, f_smem_bytes(rows));
  if (e != cudaSuccess) return e;
  *x_blocks = bx * sms;
  *f_blocks = bf * sms;
  return cudaSuccess;
}

}  // namespace halo
