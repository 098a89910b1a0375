// kernels_floor.cu — the measured floors of SURVEY §8(d) beyond the 8-B flag
// ping-pong (kernels.cu k_pingpong): the latency-vs-payload curve
// t(B) = t0 + B / BW_peer ("payload stores before the flag", B = 4 KB .. 64 MB)
// and the SM peer-store bandwidth to 1 or several concurrent peers.  Not on the
// hot path; they bound it.
#include <cuda_runtime.h>
#include <stdint.h>

#include "halo_internal.h"
#include "ptx.cuh"

namespace halo {

// Payload ping-pong between two ranks (each side one launch of G CTAs; both on
// this GPU: one launch of 2G CTAs, CTAs [G, 2G) play the responder).  Per
// iteration the initiator's CTAs each store their 16-B-vector slice of the B
// bytes into the peer's probe area, then (after the CTA barrier) one thread
// publishes it: fence.acq_rel.sys + a relaxed sys-scope add on the peer's
// counter — the paper's per-CTA completion + signal (Alg. 5).  The
// responder's CTAs wait until the counter reaches G * (iteration), send their
// slices back the same way.  CTA 0 of the initiator times each round trip.
// `cnt_base` = the value this side's counter holds before the call
// (`cnt_base_peer`: the responder half's, same-GPU mode).
__global__ void __launch_bounds__(256) k_payload_pingpong(const int4* __restrict__ src_own, int4* dst_peer,
                                                          const int4* __restrict__ src_peer_side, int4* dst_own,
                                                          uint64_t* cnt_own, uint64_t* cnt_peer, size_t n16, int G,
                                                          int iters, uint64_t cnt_base, uint64_t cnt_base_peer, int initiator, uint64_t* rtt_ns,
                                                          uint64_t timeout_ns, int* err_host) {
  int b = (int)blockIdx.x;
  const int4* src = src_own;
  int4* dst = dst_peer;
  uint64_t* own = cnt_own;
  uint64_t* peer = cnt_peer;
  if (b >= G) {  // same-GPU responder half: the peer's view
    b -= G;
    initiator = 0;
    src = src_peer_side;
    dst = dst_own;
    uint64_t* t = own;
    own = peer;
    peer = t;
    cnt_base = cnt_base_peer;
  }
  const size_t per = (n16 + G - 1) / G;
  const size_t lo = per * b, hi = lo + per < n16 ? lo + per : n16;
  __shared__ int s_fail;
  if (threadIdx.x == 0) s_fail = 0;
  __syncthreads();
  auto send = [&]() {
    for (size_t i = lo + threadIdx.x; i < hi; i += 4 * blockDim.x) {
      int4 v[4];
#pragma unroll
      for (int k = 0; k < 4; ++k)
        if (i + k * blockDim.x < hi) v[k] = __ldcg(src + i + k * blockDim.x);
#pragma unroll
      for (int k = 0; k < 4; ++k)
        if (i + k * blockDim.x < hi) dst[i + k * blockDim.x] = v[k];
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      fence_sys();  // this CTA's payload stores before its signal (cumulativity through the barrier)
      asm volatile("red.relaxed.sys.global.add.u64 [%0], 1;" ::"l"(peer) : "memory");
    }
  };
  auto wait = [&](uint64_t target) {
    if (threadIdx.x == 0 && !wait_geq<true>(own, target, timeout_ns, err_host, tcode(16, initiator, 0))) s_fail = 1;
    __syncthreads();
    return s_fail == 0;
  };
  for (int it = 1; it <= iters; ++it) {
    const uint64_t target = cnt_base + (uint64_t)G * (uint64_t)it;
    uint64_t t0 = 0;
    if (initiator) {
      if (b == 0 && threadIdx.x == 0) t0 = gtimer();
      send();
      if (!wait(target)) return;
      if (b == 0 && threadIdx.x == 0) rtt_ns[it - 1] = gtimer() - t0;
    } else {
      if (!wait(target)) return;
      send();
    }
  }
}

cudaError_t launch_payload_pingpong(const void* src_own, void* dst_peer, const void* src_peer_side, void* dst_own,
                                    uint64_t* cnt_own, uint64_t* cnt_peer, size_t bytes, int G, int iters,
                                    uint64_t cnt_base, uint64_t cnt_base_peer, int mode /* 0 responder, 1 initiator, 2 both */,
                                    uint64_t* rtt_ns, uint64_t timeout_ns, int* err_host, cudaStream_t st) {
  k_payload_pingpong<<<mode == 2 ? 2 * G : G, 256, 0, st>>>(
      (const int4*)src_own, (int4*)dst_peer, (const int4*)src_peer_side, (int4*)dst_own, cnt_own, cnt_peer, bytes / 16,
      G, iters, cnt_base, cnt_base_peer, mode == 0 ? 0 : 1, rtt_ns, timeout_ns, err_host);
  return cudaGetLastError();
}

// SM peer-store bandwidth to n concurrent peers: CTA b copies its share of
// `bytes` to peer (b mod n) — every peer receives `bytes` per launch.
struct MultiDst {
  int4* dst[kMaxRanks];
};
__global__ void __launch_bounds__(256) k_bw_multi(const int4* __restrict__ src, const __grid_constant__ MultiDst D,
                                                  int n, size_t n16) {
  const int peer = (int)blockIdx.x % n;
  const int G = (int)gridDim.x / n;  // CTAs per peer (grid = G * n)
  const int b = (int)blockIdx.x / n;
  int4* dst = D.dst[peer];
  const size_t stride = (size_t)G * blockDim.x;
  for (size_t i = (size_t)b * blockDim.x + threadIdx.x; i < n16; i += 4 * stride) {
    int4 v[4];
#pragma unroll
    for (int k = 0; k < 4; ++k)
      if (i + k * stride < n16) v[k] = __ldcg(src + i + k * stride);
#pragma unroll
    for (int k = 0; k < 4; ++k)
      if (i + k * stride < n16) dst[i + k * stride] = v[k];
  }
}

cudaError_t launch_bw_multi(const void* src, void* const* dst, int n, size_t bytes, int ctas_per_peer,
                            cudaStream_t st) {
  MultiDst D{};
  for (int i = 0; i < n && i < kMaxRanks; ++i) D.dst[i] = (int4*)dst[i];
  k_bw_multi<<<ctas_per_peer * n, 256, 0, st>>>((const int4*)src, D, n, bytes / 16);
  return cudaGetLastError();
}

}  // namespace halo
