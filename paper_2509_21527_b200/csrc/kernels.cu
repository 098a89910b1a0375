// kernels.cu — sm_100a kernels of libhalo.
//
//   k_exchange_x   fused gather + periodic shift + NVLink peer store + per-pulse
//                  completion + system-scope release flag (Alg. 3 FusedPackCommX,
//                  Alg. 4 packWithDeps, Alg. 5 syncAndCommWithDeps DATA)
//   k_exchange_f   dependency-gated push of halo force slices + flag-gated
//                  ordered scatter-add + fp64 shift forces (Alg. 6
//                  FusedCommUnpackF, Alg. 5 DEP_MGMT), push variant (R18/R23)
//   k_select       set_maps: fp64 slab predicate + order-preserving compaction (R2, R3, R11)
//   k_handshake    set_maps: send size -> receiver, atomOffset -> sender (device flags)
//   k_depmask      set_maps: wait set of each pulse (R9) and depOffset split (R8)
//   k_status       set_maps: all-to-all error agreement
//   k_pack_x / k_unpack_f   per-pulse kernels of the NCCL baseline schedule
//   k_pingpong     one-way peer flag latency floor
//
// All cross-rank synchronisation is release/acquire on 64-bit monotonic
// sequence numbers (R17).  Every spin is bounded by %globaltimer (timeout ->
// host-mapped error word, HALO_ERR_TIMEOUT on the next call).
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdlib.h>

#include <algorithm>
#include "halo_internal.h"
#include "ptx.cuh"

namespace halo {

// ------------------------------------------------------------ exchange x (hot)
template <int W>
__device__ __forceinline__ void x_rows(const PulseDev& pd, const float* __restrict__ x, uint32_t b, uint32_t e,
                                       bool dep) {
  const int32_t* __restrict__ map = pd.map;
  float* __restrict__ dst = pd.x_dst;
  const bool sh = pd.has_shift != 0;
  const float s0 = pd.shift[0], s1 = pd.shift[1], s2 = pd.shift[2];
  for (uint32_t i = b + threadIdx.x; i < e; i += blockDim.x) {
    const int idx = __ldg(map + i);
    if constexpr (W == 4) {
      const float4* src = reinterpret_cast<const float4*>(x) + idx;
      // dependent rows were written by a peer during this kernel: bypass L1 (.cg)
      float4 v = dep ? __ldcg(src) : __ldg(src);
      if (sh) {  // float32 add of the full 3-vector; w is never shifted (R25)
        v.x = __fadd_rn(v.x, s0);
        v.y = __fadd_rn(v.y, s1);
        v.z = __fadd_rn(v.z, s2);
      }
      reinterpret_cast<float4*>(dst)[i] = v;
    } else {
      const float* src = x + 3 * (size_t)idx;
      float a, bb, c;
      if (dep) {
        a = __ldcg(src); bb = __ldcg(src + 1); c = __ldcg(src + 2);
      } else {
        a = __ldg(src); bb = __ldg(src + 1); c = __ldg(src + 2);
      }
      if (sh) {
        a = __fadd_rn(a, s0);
        bb = __fadd_rn(bb, s1);
        c = __fadd_rn(c, s2);
      }
      float* o = dst + 3 * (size_t)i;
      o[0] = a; o[1] = bb; o[2] = c;
    }
  }
}

// HALO_F_TMA_STORE: the paper's NVLink put (Alg. 3): each warp
// packs a 32-row chunk (gather + shift) into its own shared-memory buffer and the
// warp leader issues one asynchronous bulk (TMA) store of the chunk into the
// receiver's x; the other warps keep packing.  Bulk stores need 16-B aligned
// addresses and sizes: the chunk is staged at the destination's offset mod 16, the
// aligned body goes by TMA, the unaligned head/tail floats (float3 rows only) by
// lane stores.  Double-buffered per warp; before the CTA's completion
// notification every leader waits for its stores to be performed.
constexpr int kStageFloats = 32 * 4 + 4;  // one chunk of 32 rows (<= 16 B each) + 16 B of alignment slack
template <int W>
__device__ __forceinline__ void x_rows_tma(const PulseDev& pd, const float* __restrict__ x, uint32_t b, uint32_t e,
                                           bool dep, float (*stage)[2][kStageFloats]) {
  const int32_t* __restrict__ map = pd.map;
  const bool sh = pd.has_shift != 0;
  const float s0 = pd.shift[0], s1 = pd.shift[1], s2 = pd.shift[2];
  const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  uint32_t k = 0;
  for (uint32_t r0 = b + 32 * warp; r0 < e; r0 += 32 * nw, ++k) {
    float* buf = stage[warp][k & 1];
    if (k >= 2) {  // the store issued from this buffer two chunks ago has read it
      if (lane == 0) bulk_wait_read<1>();
      __syncwarp();
    }
    const uint32_t n = min(32u, e - r0);
    float* gdst = pd.x_dst + (size_t)r0 * W;
    const uint32_t mis = (uint32_t)(((uintptr_t)gdst & 15u) >> 2);  // floats before the next 16-B boundary's origin
    if (lane < n) {
      const int idx = __ldg(map + r0 + lane);
      float v[4];
      if constexpr (W == 4) {
        const float4* src = reinterpret_cast<const float4*>(x) + idx;
        const float4 t = dep ? __ldcg(src) : __ldg(src);
        v[0] = t.x; v[1] = t.y; v[2] = t.z; v[3] = t.w;
      } else {
        const float* src = x + 3 * (size_t)idx;
#pragma unroll
        for (int c = 0; c < 3; ++c) v[c] = dep ? __ldcg(src + c) : __ldg(src + c);
      }
      if (sh) {  // float32 add of the full 3-vector; w is never shifted (R25)
        v[0] = __fadd_rn(v[0], s0);
        v[1] = __fadd_rn(v[1], s1);
        v[2] = __fadd_rn(v[2], s2);
      }
#pragma unroll
      for (int c = 0; c < W; ++c) buf[mis + lane * W + c] = v[c];
    }
    fence_proxy_async_smem();  // this lane's generic smem writes -> visible to the bulk copy
    __syncwarp();
    const uint32_t total = n * W;
    const uint32_t head = mis ? min(4u - mis, total) : 0u;
    const uint32_t body = ((total - head) >> 2) << 2;
    if (lane == 0 && body) {
      bulk_store(gdst + head, buf + mis + head, body * 4u);
      bulk_commit();
    }
    if (lane < head) gdst[lane] = buf[mis + lane];
    if (lane < total - head - body) gdst[head + body + lane] = buf[mis + head + body + lane];
  }
  if (lane == 0 && k) {
    bulk_wait_all();            // this warp's bulk stores are performed ...
    fence_proxy_async_global();  // ... and ordered before the generic release that notifies the peer
  }
}

// Notify the receiver once per pulse: every CTA fences its peer stores and
// increments the pulse's completion counter; the last CTA stores the flag
// (Alg. 5: "only threadIdx.x = 0 proceeds to notify").
__device__ __forceinline__ void pulse_complete_sys(unsigned flags, uint32_t* cnt, int n_items, uint64_t* flag_dst,
                                                   uint64_t seq, uint32_t* notify_count, bool relaxed = false) {
  uint32_t old;
  if (relaxed) {  // G3 (ii) mutation: no release anywhere on the notification path
    asm volatile("atom.relaxed.gpu.global.add.u32 %0, [%1], 1;" : "=r"(old) : "l"(cnt) : "memory");
  } else {
    if (flags & HALO_F_GPU_FENCE) fence_gpu(); else fence_sys();
    old = atom_add_acqrel_gpu(cnt, 1u);
  }
  if (old == (uint32_t)n_items - 1) {
    *cnt = 0;  // no other CTA of this launch touches it again
    if (relaxed) st_relaxed_sys(flag_dst, seq); else st_release_sys(flag_dst, seq);
    if (notify_count) atomicAdd(notify_count, 1u);  // debug (pin G4): one notification per pulse per step
  }
}

template <int W, bool kTma>
__global__ void __launch_bounds__(kThreads) k_exchange_x(const __grid_constant__ ExParams P) {
  __shared__ uint64_t s_seq;
  __shared__ __align__(16) float s_stage[kTma ? kThreads / 32 : 1][2][kStageFloats];  // HALO_F_TMA_STORE chunks
  Ctrl* ctrl = P.ctrl;
  if (threadIdx.x == 0) s_seq = ld_relaxed_gpu(&ctrl->seq_x) + 1;
  timer_start(P.flags, &ctrl->t_start_x);
  __syncthreads();
  const uint64_t seq = s_seq;
  const uint32_t lo_mask = (P.p_lo > 0) ? ((1u << P.p_lo) - 1u) : 0u;

  for (int it = blockIdx.x; it < P.n_items; it += gridDim.x) {
    const Item w = P.items[it];
    const PulseDev& pd = P.pulses[w.lrank * P.P + w.pulse];
    const RankDev& rd = P.ranks[w.lrank];
    const bool dep = (w.kind == kItemXDep);
    if (dep) {
      // Alg. 4: leader acquire-waits exactly the pulses the dependent entries came
      // from (R9; pulses below p_lo completed in earlier launches), then a barrier.
      if (threadIdx.x == 0) {
        uint32_t m = pd.dep_x & ~lo_mask;
        if (P.debug & kMutatePaperQ9) m &= (1u << w.pulse) >> 1;  // G3 (iv): only firstDependentPulse = p-1
        while (m) {
          const int q = __ffs(m) - 1;
          m &= m - 1;
          wait_geq<true>(&rd.hdr->flag_x[q], seq, P.timeout_ns, P.err_host, tcode(1, w.lrank, q), P.poll_ns);
        }
      }
      __syncthreads();
    }
    if ((P.debug & kDelayPulse0) && w.pulse == 0 && rd.rank == P.delay_rank) {  // slow producer (G3)
      const uint64_t t0 = gtimer();
      while (gtimer() - t0 < 20000) __nanosleep(1000);
    }
    if constexpr (kTma)
      x_rows_tma<W>(pd, rd.x, w.begin, w.end, dep, s_stage);
    else
      x_rows<W>(pd, rd.x, w.begin, w.end, dep);
    __syncthreads();
    if (threadIdx.x == 0)
      pulse_complete_sys(P.flags, &ctrl->cnt_x[w.lrank][w.pulse], pd.n_items_x, pd.flag_x_dst, seq,
                         (P.debug & kCountNotify) ? &ctrl->notify[0][w.lrank][w.pulse] : nullptr,
                         (P.debug & kMutateRelaxedFlags) != 0);
  }
  // The launch completes only when this process's halos are complete, so that
  // stream-ordered consumers (non-local NB) see them.
  if (blockIdx.x < P.n_local && threadIdx.x == 0) {
    const int lr = blockIdx.x;
    const RankDev& rd = P.ranks[lr];
    for (int p = P.p_lo; p < P.p_hi; ++p) {
      if (P.pulses[lr * P.P + p].recv_size > 0)
        wait_geq<true>(&rd.hdr->flag_x[p], seq, P.timeout_ns, P.err_host, tcode(2, lr, p), P.poll_ns);
    }
  }
  __syncthreads();
  finish_launch(P.flags, &ctrl->done_x, &ctrl->seq_x, seq, &ctrl->t_start_x, &ctrl->t_end_x, &ctrl->span_x);
}

// ------------------------------------------------------------ exchange f (hot)
template <int W>
__device__ __forceinline__ void push_rows(const PulseDev& pd, const float* __restrict__ f, uint32_t b, uint32_t e) {
  // slice rows [atom_offset + b, atom_offset + e) -> peer fbuf rows [b, e): contiguous
  const float* src = f + (size_t)(pd.atom_offset + b) * W;
  float* dst = pd.fbuf_dst + (size_t)b * W;
  const uint32_t n = (e - b) * W;
  if constexpr (W == 4) {
    const float4* s4 = reinterpret_cast<const float4*>(src);
    float4* d4 = reinterpret_cast<float4*>(dst);
    for (uint32_t i = threadIdx.x; i < (e - b); i += blockDim.x) d4[i] = __ldcg(s4 + i);
  } else {
    for (uint32_t i = threadIdx.x; i < n; i += blockDim.x) dst[i] = __ldcg(src + i);
  }
}

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// buf: row i of the pulse at buf + i*W — the own receive buffer (push; written by
// a peer during this kernel: .cg loads) or, kSmem, the chunk just bulk-loaded
// into shared memory (HALO_F_TMA_GET).
template <int W, bool kSmem>
__device__ __forceinline__ void unpack_rows(const PulseDev& pd, const float* buf, float* __restrict__ f, uint32_t b,
                                            uint32_t e, bool atomic, bool accumulate, double* fshift_rank,
                                            bool f32 = false) {
  const int32_t* __restrict__ map = pd.map;
  const bool do_shift = (fshift_rank != nullptr) && pd.has_shift;
  double a0 = 0.0, a1 = 0.0, a2 = 0.0;
  for (uint32_t i = b + threadIdx.x; i < e; i += blockDim.x) {
    const int t = __ldg(map + i);
    float v[4];
    if constexpr (kSmem) {
#pragma unroll
      for (int c = 0; c < W; ++c) v[c] = buf[(size_t)i * W + c];
    } else if constexpr (W == 4) {
      float4 q = __ldcg(reinterpret_cast<const float4*>(buf) + i);
      v[0] = q.x; v[1] = q.y; v[2] = q.z; v[3] = q.w;
    } else {
      v[0] = __ldcg(buf + 3 * (size_t)i); v[1] = __ldcg(buf + 3 * (size_t)i + 1); v[2] = __ldcg(buf + 3 * (size_t)i + 2);
    }
    float* dst = f + (size_t)t * W;
    if (!accumulate) {
#pragma unroll
      for (int c = 0; c < W; ++c) dst[c] = v[c];
    } else if (atomic) {
#pragma unroll
      for (int c = 0; c < W; ++c) atomicAdd(dst + c, v[c]);
    } else {
      if constexpr (W == 4) {
        float4 o = __ldcg(reinterpret_cast<const float4*>(dst));
        o.x = __fadd_rn(o.x, v[0]); o.y = __fadd_rn(o.y, v[1]); o.z = __fadd_rn(o.z, v[2]); o.w = __fadd_rn(o.w, v[3]);
        *reinterpret_cast<float4*>(dst) = o;
      } else {
#pragma unroll
        for (int c = 0; c < 3; ++c) dst[c] = __fadd_rn(__ldcg(dst + c), v[c]);
      }
    }
    if (do_shift) { a0 += (double)v[0]; a1 += (double)v[1]; a2 += (double)v[2]; }
  }
  if (do_shift) {
    a0 = warp_sum(a0); a1 = warp_sum(a1); a2 = warp_sum(a2);
    if (f32) { a0 = (double)(float)a0; a1 = (double)(float)a1; a2 = (double)(float)a2; }  // mutation: fp32 partials
    if ((threadIdx.x & 31) == 0) {
      double* fs = fshift_rank + 3 * pd.dim;
      atomicAdd(fs + 0, a0); atomicAdd(fs + 1, a1); atomicAdd(fs + 2, a2);
    }
  }
}

// kGet (HALO_F_TMA_GET): the paper's receiver-driven force transport (Alg. 6
// P:394-398): push items only signal that slice p is final (no data), unpack
// items bulk-load (TMA) their chunk of the slice from the peer's f into shared
// memory after the acquire-wait and scatter-add it from there; the last unpack
// CTA of a pulse acks the read (consumed flag), and the launch completes only
// when this process's slices were read by their consumers (R26).
constexpr int kGetFloats = kMaxItemRows * 4 + 8;  // largest item (16-B rows) + 16 B of alignment slack each side
template <int W, bool kGet>
__global__ void __launch_bounds__(kThreads) k_exchange_f(const __grid_constant__ ExParams P) {
  __shared__ uint64_t s_seq;
  __shared__ __align__(16) float s_get[kGet ? kGetFloats : 4];
  __shared__ __align__(8) uint64_t s_bar;
  uint32_t phase = 0;
  Ctrl* ctrl = P.ctrl;
  if (threadIdx.x == 0) {
    s_seq = ld_relaxed_gpu(&ctrl->seq_f) + 1;
    if constexpr (kGet) {
      mbar_init(&s_bar, 1);
      fence_mbar_init();
    }
  }
  timer_start(P.flags, &ctrl->t_start_f);
  __syncthreads();
  const uint64_t seq = s_seq;
  const bool atomic = (P.flags & HALO_F_ATOMIC_UNPACK) != 0;

  for (int it = blockIdx.x; it < P.n_items; it += gridDim.x) {
    const Item w = P.items[it];
    const PulseDev& pd = P.pulses[w.lrank * P.P + w.pulse];
    const RankDev& rd = P.ranks[w.lrank];
    if (w.kind == kItemPush) {
      // DEP_MGMT (Alg. 5): slice p is final once every later pulse that
      // forwarded rows of it has been unpacked here.
      if (threadIdx.x == 0) {
        uint32_t m = pd.fdep;
        while (m) {
          const int q = __ffs(m) - 1;
          m &= m - 1;
          wait_geq<false>(&ctrl->unpacked[w.lrank][q], seq, P.timeout_ns, P.err_host, tcode(3, w.lrank, q), P.poll_ns);
        }
      }
      __syncthreads();
      if constexpr (!kGet) push_rows<W>(pd, rd.f, w.begin, w.end);  // get: the flag alone says "slice p is final"
      __syncthreads();
      if (threadIdx.x == 0)
        pulse_complete_sys(P.flags, &ctrl->cnt_push[w.lrank][w.pulse], pd.n_items_push, pd.flag_f_dst, seq,
                           (P.debug & kCountNotify) ? &ctrl->notify[1][w.lrank][w.pulse] : nullptr,
                           (P.debug & kMutateRelaxedFlags) != 0);
    } else {  // kItemUnpack
      if (threadIdx.x == 0) {
        wait_geq<true>(&rd.hdr->flag_f[w.pulse], seq, P.timeout_ns, P.err_host, tcode(4, w.lrank, w.pulse), P.poll_ns);
        if (!atomic) {  // deterministic: pulses descending (R15)
          uint32_t m = pd.chain;
          while (m) {
            const int q = __ffs(m) - 1;
            m &= m - 1;
            wait_geq<false>(&ctrl->unpacked[w.lrank][q], seq, P.timeout_ns, P.err_host, tcode(5, w.lrank, q), P.poll_ns);
          }
        }
      }
      // get: one bulk load of the chunk's 16-B aligned cover (at most 12 B on each
      // side that are not used) from the peer's f, issued after the acquire
      const float* buf = pd.fbuf_own;
      if constexpr (kGet) {
        const uintptr_t src = (uintptr_t)(pd.f_src + (size_t)w.begin * W);
        const uintptr_t a0 = src & ~(uintptr_t)15;
        const uintptr_t a1 = (src + (size_t)(w.end - w.begin) * W * 4 + 15) & ~(uintptr_t)15;
        if (threadIdx.x == 0) {
          fence_proxy_async_global();  // the acquire above orders the async-proxy read
          bulk_load(s_get, (const void*)a0, (uint32_t)(a1 - a0), &s_bar);
        }
        buf = reinterpret_cast<const float*>(reinterpret_cast<const char*>(s_get) + (src - a0)) - (size_t)w.begin * W;
      }
      __syncthreads();
      double* fs = P.fshift ? P.fshift + 9 * w.lrank : nullptr;
      if constexpr (kGet) {
        mbar_wait(&s_bar, phase);
        phase ^= 1u;
        unpack_rows<W, true>(pd, buf, rd.f, w.begin, w.end, atomic, P.accumulate != 0, fs,
                             (P.debug & kMutateFshiftF32) != 0);
      } else {
        unpack_rows<W, false>(pd, buf, rd.f, w.begin, w.end, atomic, P.accumulate != 0, fs,
                              (P.debug & kMutateFshiftF32) != 0);
      }
      __syncthreads();
      if (threadIdx.x == 0) {
        fence_gpu();
        uint32_t old = atom_add_acqrel_gpu(&ctrl->cnt_unpack[w.lrank][w.pulse], 1u);
        if (old == (uint32_t)pd.n_items_unpack - 1) {
          ctrl->cnt_unpack[w.lrank][w.pulse] = 0;
          st_release_gpu(&ctrl->unpacked[w.lrank][w.pulse], seq);
          if constexpr (kGet) st_release_sys(pd.consumed_dst, seq);  // every chunk of slice p was read
        }
      }
    }
  }
  if constexpr (kGet) {
    // the peers have read this process's halo slices: f may be overwritten after the launch
    if (blockIdx.x < P.n_local && threadIdx.x == 0) {
      const int lr = blockIdx.x;
      for (int p = 0; p < P.P; ++p)
        if (P.pulses[lr * P.P + p].recv_size > 0)
          wait_geq<true>(&P.ranks[lr].hdr->consumed[p], seq, P.timeout_ns, P.err_host, tcode(14, lr, p), P.poll_ns);
    }
  }
  __syncthreads();
  finish_launch(P.flags, &ctrl->done_f, &ctrl->seq_f, seq, &ctrl->t_start_f, &ctrl->t_end_f, &ctrl->span_f);
}

// ------------------------------------------------------------- set_maps kernels
// One CTA (1024 threads) per local rank: ordered compaction of the candidate
// rows [cand0, cand1) with the fp64 slab predicate (R2, R3).  Also checks, on
// the first pulse, that home atoms lie in the rank's cell.
// The slab predicate of candidate row i (R2, R3) and, with rounded zones, R31.
__device__ __forceinline__ bool select_row(const SelParams& S, const RankDev& rd, int lr, int i, double blo) {
  const float* row = rd.x + (size_t)i * S.layout;
  const double dd = __dsub_rn((double)row[S.dim], blo);
  bool sel = dd < S.rc;
  if (sel && S.b_up != nullptr) {
    // rounded zones (R31): a row beyond this rank's upper face in another dim
    // is sent only if its distance to the receiver's cell is < rc (fixed op
    // order, no FMA contraction: the oracle's float64 ops)
    double r2 = __dmul_rn(dd, dd);
    bool beyond = false;
    for (int d2 = 0; d2 < 3; ++d2) {
      if (d2 == S.dim) continue;
      const double t = __dsub_rn((double)row[d2], S.b_up[3 * lr + d2]);
      if (t > 0.0) {
        r2 = __dadd_rn(r2, __dmul_rn(t, t));
        beyond = true;
      }
    }
    sel = !beyond || r2 < S.rc2;
  }
  return sel;
}

__device__ __forceinline__ void select_range(const SelParams& S, int lr, int& c0, int& c1) {
  if (S.cand != nullptr) {
    c0 = S.cand[2 * lr];
    c1 = S.cand[2 * lr + 1];
  } else if (S.kfirst) {  // every row present before the dim's first pulse
    c0 = 0;
    c1 = S.ctrl->n_total[lr];
  } else {  // the rows received in the previous pulse of the dim
    c0 = S.ctrl->atom_offset[lr][S.p - 1];
    c1 = c0 + S.ctrl->recv_size[lr][S.p - 1];
  }
}

// Order-preserving compaction of the candidate rows [c0, c1) with the fp64 slab
// predicate, over many CTAs per local rank (blockIdx.y): kWrite = false counts each
// CTA's selected rows (sel_cnt) and checks, on the first pulse, that home atoms lie in
// the rank's cell; kWrite = true sums the counts of the CTAs before it (its output
// offset; the map stays in ascending row order, R11) and writes its rows; its last CTA
// writes send_size.  CTA c covers rows c0 + [c*1024, (c+1)*1024).
template <bool kWrite>
__global__ void __launch_bounds__(1024) k_select(const __grid_constant__ SelParams S) {
  const int lr = blockIdx.y;
  const RankDev& rd = S.ranks[lr];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  __shared__ int s_cnt[32];
  __shared__ int s_total, s_base;
  if (!kWrite && threadIdx.x == 0) {
    // rows that came from another process in earlier pulses: wait for their arrival
    for (uint32_t m = S.wait_mask[lr]; m; m &= m - 1)
      (void)wait_epoch(&rd.hdr->ns_x[__ffs(m) - 1], S.epoch, S.timeout_ns, S.err_host, tcode(9, lr, __ffs(m) - 1));
  }
  __syncthreads();
  if (!kWrite && S.home_lo != nullptr) {
    bool bad = false;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < rd.n_home; i += gridDim.x * blockDim.x)
      for (int d = 0; d < 3; ++d) {
        if (!(S.decomposed_mask & (1 << d))) continue;
        const double v = (double)rd.x[(size_t)i * S.layout + d];
        bad |= !(v >= S.home_lo[3 * lr + d] && v < S.home_hi[3 * lr + d]);
      }
    if (bad) atomicOr(&S.ctrl->err[lr], kErrGeometry);
  }
  int c0, c1;
  select_range(S, lr, c0, c1);
  const int nchunk = (c1 - c0 + (int)blockDim.x - 1) / (int)blockDim.x;
  const int i = c0 + blockIdx.x * blockDim.x + threadIdx.x;
  const bool sel = blockIdx.x < nchunk && i < c1 && select_row(S, rd, lr, i, S.b_lo[3 * lr + S.dim]);
  const unsigned bal = __ballot_sync(0xffffffffu, sel);
  if (lane == 0) s_cnt[warp] = __popc(bal);
  if (kWrite && warp == 1) {  // this CTA's output offset: the rows of the CTAs before it
    int b = 0;
    for (int k = lane; k < (int)blockIdx.x && k < nchunk; k += 32) b += S.sel_cnt[lr * S.max_chunks + k];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) b += __shfl_xor_sync(0xffffffffu, b, o);
    if (lane == 0) s_base = b;
  }
  __syncthreads();
  if (warp == 0) {
    const int c = (lane < (int)(blockDim.x >> 5)) ? s_cnt[lane] : 0;
    int incl = c;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += y;
    }
    s_cnt[lane] = incl - c;
    if (lane == 31) s_total = incl;
  }
  __syncthreads();
  if (!kWrite) {
    if (threadIdx.x == 0) S.sel_cnt[lr * S.max_chunks + blockIdx.x] = s_total;
    return;
  }
  int32_t* out = rd.maps + (size_t)S.p * S.map_stride;
  const int slot = s_base + s_cnt[warp] + __popc(bal & ((1u << lane) - 1u));
#ifdef HALO_BOUNDS_CHECK  // a map entry beyond the pulse's map slot
  if (sel && (slot < 0 || slot >= S.map_stride)) {
    report_timeout(S.err_host, tcode(kErrKindBounds, lr, 30));
    return;
  }
#endif
  if (sel) out[slot] = i;
  if (threadIdx.x == 0 && (int)blockIdx.x == max(nchunk, 1) - 1) S.ctrl->send_size[lr][S.p] = s_base + s_total;
}

// One warp per local rank (lane 0): size -> receiver, wait own size, grant
// atomOffset -> sender, wait own grant.  All local ranks are co-resident.
__global__ void k_handshake(const __grid_constant__ HsParams H) {
  if (threadIdx.x != 0) return;
  const int lr = blockIdx.x;
  Ctrl* c = H.ctrl;
  const int p = H.p;
  const uint64_t ep = (uint64_t)H.epoch << 32;
  const uint32_t sz = (uint32_t)c->send_size[lr][p];
  // a neighbour in this process reads at gpu scope: no system-scope fence (NS-step latency)
  if (H.sys_mask >> lr & 1u) st_release_sys(H.size_dst[lr], ep | sz);
  else st_release_gpu(H.size_dst[lr], ep | sz);
  uint32_t recv = wait_epoch(&H.own[lr]->meta_size[p], H.epoch, H.timeout_ns, H.err_host, tcode(6, lr, p));
  if (recv == 0xffffffffu) recv = 0;
  const int off = c->n_total[lr];
  uint32_t grant = (uint32_t)off;
  if ((long long)off + (long long)recv > (long long)H.capacity) {
    c->err[lr] |= kErrCapacity;
    grant = 0xffffffffu;
    recv = 0;
  }
  if (H.sys_mask >> (16 + lr) & 1u) st_release_sys(H.off_dst[lr], ep | grant);
  else st_release_gpu(H.off_dst[lr], ep | grant);
  const uint32_t roff = wait_epoch(&H.own[lr]->meta_off[p], H.epoch, H.timeout_ns, H.err_host, tcode(7, lr, p));
  if (roff == 0xffffffffu) {  // receiver out of capacity (or timeout): send nothing
    c->send_size[lr][p] = 0;
    c->remote_off[lr][p] = 0;
  } else {
    c->remote_off[lr][p] = (int)roff;
  }
  c->recv_size[lr][p] = (int)recv;
  c->atom_offset[lr][p] = off;
  c->n_total[lr] = off + (int)recv;
}

// One CTA per local rank: dep mask of pulse p (which earlier receive ranges the
// map reads, R9) and the number of entries < n_home (depOffset split, R8).
__global__ void __launch_bounds__(256) k_depmask(const RankDev* ranks, Ctrl* ctrl, int p, int map_stride) {
  const int lr = blockIdx.x;
  const RankDev& rd = ranks[lr];
  __shared__ unsigned s_mask;
  __shared__ int s_indep;
  __shared__ int s_bad;
  if (threadIdx.x == 0) { s_mask = 0; s_indep = 0; s_bad = 0; }
  __syncthreads();
  const int n = ctrl->send_size[lr][p];
  const int32_t* map = rd.maps + (size_t)p * map_stride;
  unsigned m = 0;
  int indep = 0;
  bool bad = false;
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    const int idx = map[i];
    if (idx < rd.n_home) { ++indep; continue; }
    bool found = false;
    for (int q = 0; q < p; ++q) {
      const int a = ctrl->atom_offset[lr][q], r = ctrl->recv_size[lr][q];
      if (idx >= a && idx < a + r) { m |= 1u << q; found = true; break; }
    }
    bad |= !found;
  }
  if (m) atomicOr(&s_mask, m);
  if (indep) atomicAdd(&s_indep, indep);
  if (bad) s_bad = 1;
  __syncthreads();
  if (threadIdx.x == 0) {
    ctrl->dep[lr][p] = s_mask;
    ctrl->n_indep[lr][p] = s_indep;
    if (s_bad) ctrl->err[lr] |= kErrMap;
  }
}

// set_maps, pulse p: x[map_p] (+shift) -> the receiver's x at remote_off (R12),
// sizes and offsets from the handshake results in device memory.  blockIdx.y =
// local rank, rows grid-strided.  Same-process receivers are covered by stream
// order; k_ns_flag then releases the others' ns_x[p].
template <int W>
__global__ void __launch_bounds__(256) k_ns_x(const __grid_constant__ NsXParams X) {
  const int lr = blockIdx.y;
  const RankDev& rd = X.ranks[lr];
  if (X.wait_mask[lr]) {  // forwarded rows that came from another process: arrived
    if (threadIdx.x == 0)
      for (uint32_t m = X.wait_mask[lr]; m; m &= m - 1)
        (void)wait_epoch(&rd.hdr->ns_x[__ffs(m) - 1], X.epoch, X.timeout_ns, X.err_host, tcode(9, lr, __ffs(m) - 1));
    __syncthreads();
  }
  const int n = X.ctrl->send_size[lr][X.p];
  const int ro = X.ctrl->remote_off[lr][X.p];
  const int32_t* map = rd.maps + (size_t)X.p * X.map_stride;
  float* dst = X.dst_x[lr] + (size_t)ro * W;
  const bool sh = X.has_shift[lr] != 0;
  // the dependency mask of the pulse (which earlier receive ranges the map reads, R9)
  // and the entries < n_home (depOffset split, R8), on the way
  unsigned dm = 0;
  int indep = 0;
  bool bad = false;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const int idx = map[i];
#ifdef HALO_BOUNDS_CHECK  // the source row, the destination row
    if (idx < 0 || idx >= X.cap || ro < 0 || ro + i >= X.cap || i >= X.map_stride) {
      report_timeout(X.err_host, tcode(kErrKindBounds, lr, 31));
      continue;
    }
#endif
    if (idx < rd.n_home) {
      ++indep;
    } else {
      bool found = false;
      for (int q = 0; q < X.p; ++q) {
        const int a0 = X.ctrl->atom_offset[lr][q], r0 = X.ctrl->recv_size[lr][q];
        if (idx >= a0 && idx < a0 + r0) { dm |= 1u << q; found = true; break; }
      }
      bad |= !found;
    }
    const float* src = rd.x + (size_t)idx * W;
    float v[W];
#pragma unroll
    for (int c = 0; c < W; ++c) v[c] = src[c];
    if (sh) {  // the full 3-vector (R25); float4 w is never shifted
#pragma unroll
      for (int c = 0; c < 3; ++c) v[c] = __fadd_rn(v[c], c == X.dim ? X.shift[lr] : 0.0f);
    }
#pragma unroll
    for (int c = 0; c < W; ++c) dst[(size_t)i * W + c] = v[c];
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    dm |= __shfl_xor_sync(0xffffffffu, dm, o);
    indep += __shfl_xor_sync(0xffffffffu, indep, o);
  }
  const bool anybad = __any_sync(0xffffffffu, bad);
  if ((threadIdx.x & 31) == 0) {
    if (dm) atomicOr(&X.ctrl->dep[lr][X.p], dm);
    if (indep) atomicAdd(&X.ctrl->n_indep[lr][X.p], indep);
    if (anybad) atomicOr(&X.ctrl->err[lr], kErrMap);
  }
}

// set_maps start: zero the LL receive areas of every local rank (one launch).
__global__ void k_zero_ll(uint64_t* const* base, size_t units, int n) {
  const int l = blockIdx.y;
  if (l >= n) return;
  uint4* p = reinterpret_cast<uint4*>(base[l]);
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < units / 2; i += (size_t)gridDim.x * blockDim.x)
    p[i] = make_uint4(0, 0, 0, 0);
}

cudaError_t launch_zero_ll(uint64_t* const* base_dev, size_t units, int n, cudaStream_t st) {
  if (n <= 0 || units == 0) return cudaSuccess;
  k_zero_ll<<<dim3(64, n), 256, 0, st>>>(base_dev, units, n);
  return cudaGetLastError();
}

__global__ void k_ns_flag(const __grid_constant__ NsXParams X) {
  const int lr = threadIdx.x;
  if (lr >= X.n_local || X.flag_dst[lr] == nullptr) return;
  fence_sys();  // k_ns_x's peer stores (stream order) before the flag
  st_release_sys(X.flag_dst[lr], ((uint64_t)X.epoch << 32) | 1u);
}

// set_maps end: every local rank acquires the ns_x flags of its pulses from other processes.
__global__ void k_ns_wait(const __grid_constant__ NsWaitParams W) {
  const int lr = threadIdx.x;
  if (lr >= W.n_local) return;
  for (uint32_t m = W.mask[lr]; m; m &= m - 1)
    (void)wait_epoch(&W.own[lr]->ns_x[__ffs(m) - 1], W.epoch, W.timeout_ns, W.err_host, tcode(9, lr, __ffs(m) - 1));
}

cudaError_t launch_ns_wait(const NsWaitParams& W, cudaStream_t st) {
  void* args[] = {(void*)&W};
  return cudaLaunchKernel((const void*)k_ns_wait, dim3(1), dim3(kMaxLocal), args, 0, st);
}

cudaError_t launch_ns_x(const NsXParams& X, int layout, int max_rows, cudaStream_t st) {
  if (X.n_local <= 0) return cudaSuccess;
  const int gx = std::max(1, std::min((max_rows + 255) / 256, std::max(1, 148 * 8 / X.n_local)));
  void* args[] = {(void*)&X};
  cudaError_t e = cudaLaunchKernel(layout == 4 ? (const void*)k_ns_x<4> : (const void*)k_ns_x<3>,
                                   dim3(gx, X.n_local), dim3(256), args, 0, st);
  if (e != cudaSuccess) return e;
  bool remote = false;
  for (int l = 0; l < X.n_local; ++l) remote |= X.flag_dst[l] != nullptr;
  if (!remote) return cudaSuccess;
  return cudaLaunchKernel((const void*)k_ns_flag, dim3(1), dim3(kMaxLocal), args, 0, st);
}

// One CTA per local rank, one thread per destination rank: error agreement.
__global__ void k_status(const __grid_constant__ StatusParams S) {
  const int lr = blockIdx.x;
  const int me = S.first_rank + lr;
  const uint64_t ep = (uint64_t)S.epoch << 32;
  __shared__ int s_or;
  if (threadIdx.x == 0) s_or = 0;
  __syncthreads();
  // votes (same value in every CTA): R = 64 rows (latency regime; swept 32-512 at C3)
  // unless this process's pulses are so large that a CTA would run more than ~2 items
  uint32_t vote = 0;
  if (S.vote) {
    long rows = 0;
    uint64_t big = 0;
    for (int l = 0; l < S.n_local; ++l)
      for (int p = 0; p < S.P; ++p) {
        rows += max(S.ctrl->send_size[l][p], S.ctrl->recv_size[l][p]);
        big = max(big, (uint64_t)S.ctrl->send_size[l][p] * S.W * sizeof(float));
      }
    if (S.auto_tr && big >= S.ce_bytes) vote |= kVoteCE;
    int R = S.rows_fixed;
    if (!R) {
      R = 64;
      while (R < kMaxItemRows && rows / R > 2 * S.ctas) R *= 2;
    }
    vote |= (uint32_t)kVoteRows << (31 - __clz((unsigned)(R / kMinItemRows)));
  }
  const uint32_t mine = (uint32_t)S.ctrl->err[lr] | vote;
  for (int t = threadIdx.x; t < S.nranks; t += blockDim.x) {
    if (S.all_local) st_release_gpu(&S.all[t]->status[me], ep | mine);
    else st_release_sys(&S.all[t]->status[me], ep | mine);
  }
  for (int t = threadIdx.x; t < S.nranks; t += blockDim.x) {
    const uint32_t v = wait_epoch(&S.own[lr]->status[t], S.epoch, S.timeout_ns, S.err_host, tcode(8, lr, 0));
    if (v != 0xffffffffu && v != 0) atomicOr(&s_or, (int)v);
  }
  __syncthreads();
  if (threadIdx.x == 0) S.ctrl->agreed_err[lr] = s_or;
}

// ---------------------------------------------------- NCCL-baseline pulse kernels
template <int W>
__global__ void k_pack_x(const int32_t* __restrict__ map, int n, const float* __restrict__ x, float* __restrict__ out,
                         int has_shift, float s0, float s1, float s2) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const int idx = map[i];
    float v[4];
#pragma unroll
    for (int c = 0; c < W; ++c) v[c] = x[(size_t)idx * W + c];
    if (has_shift) { v[0] = __fadd_rn(v[0], s0); v[1] = __fadd_rn(v[1], s1); v[2] = __fadd_rn(v[2], s2); }
#pragma unroll
    for (int c = 0; c < W; ++c) out[(size_t)i * W + c] = v[c];
  }
}

template <int W>
__global__ void k_unpack_f(const int32_t* __restrict__ map, int n, const float* __restrict__ buf, float* __restrict__ f,
                           int accumulate, double* fs_dim) {
  double a0 = 0, a1 = 0, a2 = 0;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const int t = map[i];
    float v[4];
#pragma unroll
    for (int c = 0; c < W; ++c) v[c] = buf[(size_t)i * W + c];
#pragma unroll
    for (int c = 0; c < W; ++c) {
      float* d = f + (size_t)t * W + c;
      *d = accumulate ? __fadd_rn(*d, v[c]) : v[c];
    }
    a0 += v[0]; a1 += v[1]; a2 += v[2];
  }
  if (fs_dim) {
    a0 = warp_sum(a0); a1 = warp_sum(a1); a2 = warp_sum(a2);
    if ((threadIdx.x & 31) == 0) { atomicAdd(fs_dim, a0); atomicAdd(fs_dim + 1, a1); atomicAdd(fs_dim + 2, a2); }
  }
}

// --------------------------------------------------------------- latency floor
// One CTA per side; launched with 2 CTAs when both ranks live on this GPU
// (CTA 1 plays the responder: own/peer swapped).
__global__ void k_pingpong(uint64_t* own, uint64_t* peer, int iters, uint64_t base, int initiator, int relaxed,
                           uint64_t* rtt_ns, uint64_t timeout_ns, int* err_host) {
  if (threadIdx.x != 0) return;
  if (blockIdx.x == 1) {
    uint64_t* t = own;
    own = peer;
    peer = t;
    initiator = 0;
  }
  for (int i = 1; i <= iters; ++i) {
    const uint64_t v = base + (uint64_t)i;
    const uint64_t t0 = gtimer();
    if (initiator) {
      if (relaxed) st_relaxed_sys(peer, v); else st_release_sys(peer, v);
    }
    if (relaxed) {
      uint64_t t1 = 0;
      for (uint32_t it = 1; ld_relaxed_sys(own) < v; ++it) {
        if ((it & 1023u) == 0) {
          const uint64_t now = gtimer();
          if (t1 == 0) t1 = now;
          else if (now - t1 > timeout_ns) { report_timeout(err_host, tcode(9, initiator, 1)); return; }
        }
      }
    } else if (!wait_geq<true>(own, v, timeout_ns, err_host, tcode(9, initiator, 0))) {
      return;
    }
    if (initiator) {
      rtt_ns[i - 1] = gtimer() - t0;
    } else {
      if (relaxed) st_relaxed_sys(peer, v); else st_release_sys(peer, v);
    }
  }
}

// Bandwidth floor: 16-B vector copy src -> dst (dst may be a peer pointer:
// NVLink SM stores), 4 independent loads in flight per thread.
__global__ void __launch_bounds__(256) k_bw_copy(const int4* __restrict__ src, int4* __restrict__ dst, size_t n16) {
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n16; i += 4 * stride) {
    int4 v[4];
#pragma unroll
    for (int k = 0; k < 4; ++k)
      if (i + k * stride < n16) v[k] = __ldcg(src + i + k * stride);
#pragma unroll
    for (int k = 0; k < 4; ++k)
      if (i + k * stride < n16) dst[i + k * stride] = v[k];
  }
}

cudaError_t launch_bw_copy(const void* src, void* dst, size_t bytes, int grid, cudaStream_t st) {
  k_bw_copy<<<grid, 256, 0, st>>>((const int4*)src, (int4*)dst, bytes / 16);
  return cudaGetLastError();
}

// Packed host-buffer step (halo_step_host_packed): copies between the packed
// staging buffers and the per-rank x / f rows, one segment per blockIdx.y,
// 4-B words (rows are 12 B: 4-B aligned only), 4 loads in flight per thread.
__global__ void __launch_bounds__(256) k_seg_copy(const SegCopy* __restrict__ segs) {
  const SegCopy S = segs[blockIdx.y];
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < S.words; i += 4 * stride) {
    uint32_t v[4];
#pragma unroll
    for (int k = 0; k < 4; ++k)
      if (i + k * stride < S.words) v[k] = __ldcg(S.src + i + k * stride);
#pragma unroll
    for (int k = 0; k < 4; ++k)
      if (i + k * stride < S.words) S.dst[i + k * stride] = v[k];
  }
}

cudaError_t launch_seg_copy(const SegCopy* segs, int nseg, size_t max_words, cudaStream_t st) {
  if (nseg <= 0 || max_words == 0) return cudaSuccess;
  const unsigned gx = (unsigned)std::min<size_t>(64, (max_words + 1023) / 1024);
  k_seg_copy<<<dim3(gx, (unsigned)nseg), 256, 0, st>>>(segs);
  return cudaGetLastError();
}

// Empty kernel with the exchange kernels' PDL prologue (launch floor).
// remote != nullptr: threads [0, nwords) of the grid also store one 8-B word
// each there (a peer's scratch): the launch floor of a kernel that wrote to
// NVLink peer memory.
__global__ void k_empty(uint64_t* remote, uint32_t nwords) {
  pdl_launch_dependents();
  pdl_wait();
  const uint32_t g = blockIdx.x * blockDim.x + threadIdx.x;
  if (remote != nullptr && g < nwords) st_relaxed_sys(remote + g, 0ull);
}

// ------------------------------------------------------------- host launchers
// Cooperative launch (hardware-checked co-residency) is opt-in (HALO_COOP=1):
// it disables programmatic dependent launch, which hides ~4 us of launch gap per
// kernel.  Without it, co-residency holds because the grid never exceeds the
// occupancy-computed capacity and PDL dependents are only scheduled once every
// CTA of the primary grid is resident.
// Cooperative launch (hardware-checked co-residency): HALO_COOP=1, and by default
// under MPS (an active-thread percentage can leave fewer SMs to this context than the
// occupancy calculation assumes).
static int coop_enabled() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("HALO_COOP");
    if (e) v = e[0] == '1' ? 1 : 0;
    else v = (getenv("CUDA_MPS_ACTIVE_THREAD_PERCENTAGE") || getenv("CUDA_MPS_PIPE_DIRECTORY")) ? 1 : 0;
  }
  return v;
}

static int pdl_enabled() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("HALO_PDL");
    v = (e && e[0] == '0') ? 0 : 1;
  }
  return v;
}

// Exchange-kernel launch: cooperative (every CTA co-resident)
// unless HALO_COOP=0; `pdl` adds programmatic stream serialisation (the kernel
// is scheduled while its predecessor drains and blocks in griddepcontrol.wait).
cudaError_t launch_coop_kernel_ex(const void* fn, int grid, int block, void** args, cudaStream_t st, bool pdl,
                                  size_t smem, const cudaAccessPolicyWindow* win) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(block);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[3];
  int n = 0;
  if (win != nullptr && win->num_bytes > 0) {  // HALO_F_L2_PERSIST: the static plan stays in L2
    attr[n].id = cudaLaunchAttributeAccessPolicyWindow;
    attr[n].val.accessPolicyWindow = *win;
    ++n;
  }
  if (coop_enabled()) {
    attr[n].id = cudaLaunchAttributeCooperative;
    attr[n].val.cooperative = 1;
    ++n;
  }
  if (pdl && pdl_enabled()) {
    attr[n].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[n].val.programmaticStreamSerializationAllowed = 1;
    ++n;
  }
  cfg.attrs = attr;
  cfg.numAttrs = n;
  return cudaLaunchKernelExC(&cfg, fn, args);
}

cudaError_t launch_empty(int grid, cudaStream_t st, uint64_t* remote, uint32_t nwords) {
  void* args[] = {(void*)&remote, (void*)&nwords};
  static const int block = getenv("HALO_EMPTY_BLOCK") ? atoi(getenv("HALO_EMPTY_BLOCK")) : kThreads;  // grid-size study
  return launch_coop_kernel_ex((const void*)k_empty, grid, block, args, st, true, 0, nullptr);
}

cudaError_t launch_coop_kernel(const void* fn, int grid, int block, void** args, cudaStream_t st) {
  return launch_coop_kernel_ex(fn, grid, block, args, st, false, 0, nullptr);
}

static const void* x_paper_fn(int layout, bool tma) {
  if (tma) return layout == 4 ? (const void*)k_exchange_x<4, true> : (const void*)k_exchange_x<3, true>;
  return layout == 4 ? (const void*)k_exchange_x<4, false> : (const void*)k_exchange_x<3, false>;
}

cudaError_t launch_exchange_x(const ExParams& p, int layout, int grid, cudaStream_t st) {
  void* args[] = {(void*)&p};
  const void* fn = x_paper_fn(layout, (p.flags & HALO_F_TMA_STORE) != 0);
  return launch_coop_kernel(fn, grid, kThreads, args, st);
}

static const void* f_paper_fn(int layout, bool get) {
  if (get) return layout == 4 ? (const void*)k_exchange_f<4, true> : (const void*)k_exchange_f<3, true>;
  return layout == 4 ? (const void*)k_exchange_f<4, false> : (const void*)k_exchange_f<3, false>;
}

cudaError_t launch_exchange_f(const ExParams& p, int layout, int grid, cudaStream_t st) {
  void* args[] = {(void*)&p};
  const void* fn = f_paper_fn(layout, (p.flags & HALO_F_TMA_GET) != 0);
  return launch_coop_kernel(fn, grid, kThreads, args, st);
}

cudaError_t max_coresident(int layout, int* x_blocks, int* f_blocks) {
  int dev = 0, sms = 0, bx = 0, bf = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  if (e != cudaSuccess) return e;
  // the smaller of the two x variants (SM stores / TMA stores with their staging buffers)
  int bt = 0;
  e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bx, x_paper_fn(layout, false), kThreads, 0);
  if (e != cudaSuccess) return e;
  e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bt, x_paper_fn(layout, true), kThreads, 0);
  if (e != cudaSuccess) return e;
  bx = bx < bt ? bx : bt;
  e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bf, f_paper_fn(layout, false), kThreads, 0);
  if (e != cudaSuccess) return e;
  e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bt, f_paper_fn(layout, true), kThreads, 0);
  if (e != cudaSuccess) return e;
  bf = bf < bt ? bf : bt;
  *x_blocks = bx * sms;
  *f_blocks = bf * sms;
  return cudaSuccess;
}

cudaError_t launch_select(const SelParams& s, int n_local, cudaStream_t st) {
  void* args[] = {(void*)&s};
  const dim3 grid((unsigned)std::max(1, s.max_chunks), (unsigned)n_local);
  cudaError_t e = cudaLaunchKernel((const void*)k_select<false>, grid, dim3(1024), args, 0, st);
  if (e != cudaSuccess) return e;
  return cudaLaunchKernel((const void*)k_select<true>, grid, dim3(1024), args, 0, st);
}

cudaError_t launch_handshake(const HsParams& h, cudaStream_t st) {
  void* args[] = {(void*)&h};
  return launch_coop_kernel((const void*)k_handshake, h.n_local, 32, args, st);
}

cudaError_t launch_depmask(const RankDev* ranks, Ctrl* ctrl, int p, int map_stride, int n_local, cudaStream_t st) {
  k_depmask<<<n_local, 256, 0, st>>>(ranks, ctrl, p, map_stride);
  return cudaGetLastError();
}

cudaError_t launch_status(const StatusParams& s, cudaStream_t st) {
  void* args[] = {(void*)&s};
  return launch_coop_kernel((const void*)k_status, s.n_local, 64, args, st);
}

cudaError_t launch_pack_x(int layout, const int32_t* map, int n, const float* x, float* out, int has_shift,
                          const float* shift, cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  const int grid = (n + 255) / 256;
  if (layout == 4)
    k_pack_x<4><<<grid, 256, 0, st>>>(map, n, x, out, has_shift, shift[0], shift[1], shift[2]);
  else
    k_pack_x<3><<<grid, 256, 0, st>>>(map, n, x, out, has_shift, shift[0], shift[1], shift[2]);
  return cudaGetLastError();
}

cudaError_t launch_unpack_f(int layout, const int32_t* map, int n, const float* buf, float* f, int accumulate,
                            double* fs_dim, cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  const int grid = (n + 255) / 256;
  if (layout == 4)
    k_unpack_f<4><<<grid, 256, 0, st>>>(map, n, buf, f, accumulate, fs_dim);
  else
    k_unpack_f<3><<<grid, 256, 0, st>>>(map, n, buf, f, accumulate, fs_dim);
  return cudaGetLastError();
}

cudaError_t launch_pingpong(uint64_t* own, uint64_t* peer, int iters, uint64_t base, int initiator, int relaxed,
                            uint64_t* rtt_ns, uint64_t timeout_ns, int* err_host, cudaStream_t st) {
  k_pingpong<<<initiator == 2 ? 2 : 1, 32, 0, st>>>(own, peer, iters, base, initiator == 2 ? 1 : initiator, relaxed,
                                                    rtt_ns, timeout_ns, err_host);
  return cudaGetLastError();
}

}  // namespace halo
