// kernels_ce.cu — copy-engine path (HALO_F_CE_PATH) of the hot path.
//
// north_star: "A copy-engine path covers large contiguous pulses."  The data
// of a pulse crosses NVLink as ONE cudaMemcpyAsync (copy engine, no SM time)
// instead of SM peer stores; the SMs only gather/scatter in local HBM:
//
//   x, pulse p ascending (Alg. 3/4):
//     k_ce_pack     gather x[map_p] (+shift, R25) into a contiguous staging
//                   buffer — skipped when map_p is one contiguous run of rows
//                   and the pulse has no shift (then the CE reads x directly)
//     CE copy       staging (or x) -> receiver's x at remote_off_p
//     k_ce_sync     st.release.sys flag_x[p] = seq on the receiver, then
//                   acquire-wait the own flag_x[p] (the upper neighbour's copy
//                   has landed): pulse p+1 may forward these rows (R9, coarse)
//   f, pulse p descending (Alg. 6 + Alg. 5 DEP_MGMT):
//     CE copy       own halo slice f[atomOffset_p, +recv_p) (contiguous by
//                   construction, R12) -> x-sender's force buffer of pulse p;
//                   stream order after the unpacks of every q > p = DEP_MGMT
//     k_ce_sync     flag_f[p] on the x-sender, acquire-wait the own flag_f[p]
//     k_ce_unpack   f[map_p[i]] += fbuf_p[i] (one fp32 RNE add per entry, pulses
//                   descending: bit-exact vs the oracle, R15) + fp64 shift
//                   forces of a wrapping pulse (R13)
//
// Every kernel serves all local DD ranks of the process in one launch
// (blockIdx.y = local rank).  Sequence numbers are read from device memory
// (graph-capturable, R17).
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>

#include "halo_internal.h"
#include "ptx.cuh"

namespace halo {

// 4 units per thread per batch: all gathers of a batch in flight before the stores.
template <int W>
__global__ void __launch_bounds__(256) k_ce_pack(const CeEnt* __restrict__ ents) {
  const CeEnt& e = ents[blockIdx.y];
  if (!e.pack) return;
  const uint32_t n = (uint32_t)e.n * W;
  const float s[3] = {e.shift[0], e.shift[1], e.shift[2]};
  const uint32_t G = gridDim.x * blockDim.x;
  for (uint32_t base = blockIdx.x * blockDim.x + threadIdx.x; base < n; base += 4 * G) {
    float v[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const uint32_t u = base + k * G;
      if (u < n) {
        const uint32_t i = u / W;
        v[k] = __ldg(e.src + (size_t)__ldg(e.map + i) * W + (u - i * W));
      }
    }
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const uint32_t u = base + k * G;
      if (u >= n) continue;
      const int c = (int)(u % W);
      e.dst[u] = (e.has_shift && c < 3) ? __fadd_rn(v[k], s[c]) : v[k];  // coalesced
    }
  }
}

__device__ __forceinline__ double warp_sum_ce(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

template <int W>
__global__ void __launch_bounds__(256) k_ce_unpack(const CeEnt* __restrict__ ents, double* fshift, int accumulate) {
  const CeEnt& e = ents[blockIdx.y];
  const uint32_t n = (uint32_t)e.n;
  const bool fs = fshift != nullptr && e.has_shift;
  double a[3] = {0.0, 0.0, 0.0};
  const uint32_t G = gridDim.x * blockDim.x;
  for (uint32_t base = blockIdx.x * blockDim.x + threadIdx.x; base < n; base += 2 * G) {
    int t[2];
    float v[2][W], o[2][W];
#pragma unroll
    for (int k = 0; k < 2; ++k) {
      const uint32_t i = base + k * G;
      if (i >= n) continue;
      t[k] = __ldg(e.map + i);
#pragma unroll
      for (int c = 0; c < W; ++c) v[k][c] = __ldcg(e.src + (size_t)i * W + c);  // written by a peer's copy engine
    }
#pragma unroll
    for (int k = 0; k < 2; ++k) {
      if (base + k * G >= n) continue;
#pragma unroll
      for (int c = 0; c < W; ++c) o[k][c] = e.dst[(size_t)t[k] * W + c];
    }
#pragma unroll
    for (int k = 0; k < 2; ++k) {
      if (base + k * G >= n) continue;
#pragma unroll
      for (int c = 0; c < W; ++c)  // targets unique within a pulse
        e.dst[(size_t)t[k] * W + c] = accumulate ? __fadd_rn(o[k][c], v[k][c]) : v[k][c];
      if (fs) {
#pragma unroll
        for (int c = 0; c < 3; ++c) a[c] += (double)v[k][c];
      }
    }
  }
  if (!fs) return;  // uniform over the CTA
  __shared__ double s_red[3][8];
#pragma unroll
  for (int c = 0; c < 3; ++c) a[c] = warp_sum_ce(a[c]);
  if ((threadIdx.x & 31) == 0)
#pragma unroll
    for (int c = 0; c < 3; ++c) s_red[c][threadIdx.x >> 5] = a[c];
  __syncthreads();
  if (threadIdx.x < 3) {
    double t = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += s_red[threadIdx.x][w];
    atomicAdd(fshift + 9 * blockIdx.y + 3 * e.dim + threadIdx.x, t);
  }
}

// One thread per local rank: release the pulse flag on the peer (the copy
// engine's writes precede this kernel in stream order; the sys fence orders
// them before the flag for the peer's acquire), then acquire-wait the own flag.
__global__ void k_ce_sync(const __grid_constant__ CeSyncParams S) {
  const int l = threadIdx.x;
  uint64_t seq = 0;
  if (l < S.n_local) {
    seq = ld_relaxed_gpu(S.seq_slot) + 1;
    fence_sys();
    st_release_sys(S.dst[l], seq);
    wait_geq<true>(S.own[l], seq, S.timeout_ns, S.err_host, tcode(20 + S.kind, l, S.pulse));
  }
  __syncthreads();
  if (S.publish && threadIdx.x == 0) st_relaxed_gpu(S.seq_slot, seq);
}

cudaError_t launch_ce_pack(int layout, const CeEnt* ents, int n_local, int max_rows, cudaStream_t st) {
  if (max_rows <= 0) return cudaSuccess;
  const int bx = std::min((max_rows * layout + 255) / 256, 1184);
  dim3 grid(bx, n_local);
  if (layout == 4)
    k_ce_pack<4><<<grid, 256, 0, st>>>(ents);
  else
    k_ce_pack<3><<<grid, 256, 0, st>>>(ents);
  return cudaGetLastError();
}

cudaError_t launch_ce_unpack(int layout, const CeEnt* ents, int n_local, int max_rows, double* fshift, int accumulate,
                             cudaStream_t st) {
  if (max_rows <= 0) return cudaSuccess;
  const int bx = std::min((max_rows + 255) / 256, 1184);
  dim3 grid(bx, n_local);
  if (layout == 4)
    k_ce_unpack<4><<<grid, 256, 0, st>>>(ents, fshift, accumulate);
  else
    k_ce_unpack<3><<<grid, 256, 0, st>>>(ents, fshift, accumulate);
  return cudaGetLastError();
}

cudaError_t launch_ce_sync(const CeSyncParams& s, cudaStream_t st) {
  void* args[] = {(void*)&s};
  const int threads = (s.n_local + 31) / 32 * 32;
  return cudaLaunchKernel((const void*)k_ce_sync, dim3(1), dim3(threads), args, 0, st);
}

}  // namespace halo
