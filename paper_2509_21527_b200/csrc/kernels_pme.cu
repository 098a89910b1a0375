// kernels_pme.cu — PP <-> PME coordinate / force redistribution (SURVEY §8(f)
// f4; the paper's future work: "the communication of coordinates and
// forces to and from the PME tasks"), with the halo path's one-sided machinery.
//
// The PME task lives on the GPU of DD rank `pme_rank`; its coordinate and force
// buffers (pme_x, pme_f: the home rows of every DD rank concatenated in rank
// order, rank r at rows [off_r, off_r + n_home_r)) sit in that rank's scratch,
// which every process has peer-mapped.
//
//   k_pme_allgather  halo_pme_setup: every rank's n_home to every rank
//                    ((epoch << 32) | n, system-scope release; as k_status)
//   k_pme_x          every DD rank stores its home rows straight into pme_x over
//                    NVLink (peer stores, coalesced 16-B / 12-B rows); per rank a
//                    CTA completion counter, the last CTA releases
//                    pme_x_flag[rank] = seq on the PME rank (Alg. 5's scheme);
//                    on the PME process one CTA acquire-waits every rank's flag,
//                    so the launch completes when pme_x is complete
//   k_pme_f          the PME process releases pme_f_flag = seq to every rank
//                    (its force kernel precedes in stream order); every DD rank
//                    acquire-waits it, reads its slice of pme_f over NVLink and
//                    adds it into its home forces (one fp32 RNE add per
//                    component, or overwrite), then acks pme_ack[rank]; the PME
//                    process's launch completes when every slice was read
//
// Sequence numbers: 64-bit, in device memory (ctrl->seq_pme_x / seq_pme_f),
// read by every CTA at entry and advanced by the last CTA to finish (graph
// replays stay correct, R17).  Every wait is bounded (%globaltimer).
#include <cuda_runtime.h>
#include <stdint.h>
#include "halo_internal.h"
#include "ptx.cuh"

namespace halo {

__global__ void k_pme_allgather(const __grid_constant__ PmeParams M) {
  const int l = blockIdx.x;
  const int me = M.r[l].rank;
  const uint64_t ep = (uint64_t)M.epoch << 32;
  for (int t = threadIdx.x; t < M.nranks; t += blockDim.x)
    st_release_sys(&M.all_hdr[t]->pme_nh[me], ep | (uint32_t)M.r[l].n_home);
  for (int t = threadIdx.x; t < M.nranks; t += blockDim.x) {
    const uint32_t v = wait_epoch(&M.r[l].hdr->pme_nh[t], M.epoch, M.timeout_ns, M.err_host, tcode(17, l, 0));
    M.ctrl->pme_nh[l][t] = (int32_t)(v == 0xffffffffu ? 0 : v);
  }
}

// the CTA's share [b, e) of n rows when G CTAs split them
__device__ __forceinline__ void share(int n, int G, int g, int& b, int& e) {
  const int per = (n + G - 1) / G;
  b = min(n, g * per);
  e = min(n, b + per);
}

// last CTA of the launch publishes the sequence number (every CTA read it at entry)
__device__ __forceinline__ void pme_depart(uint32_t* done, uint64_t* seq_slot, uint64_t seq) {
  __syncthreads();
  if (threadIdx.x == 0) {
    const uint32_t total = gridDim.x * gridDim.y;
    if (atomicAdd(done, 1u) == total - 1) {
      *done = 0;
      st_relaxed_gpu(seq_slot, seq);
    }
  }
}

template <int W>
__global__ void __launch_bounds__(256) k_pme_x(const __grid_constant__ PmeParams M) {
  __shared__ uint64_t s_seq;
  if (threadIdx.x == 0) s_seq = ld_relaxed_gpu(&M.ctrl->seq_pme_x) + 1;
  __syncthreads();
  const uint64_t seq = s_seq;
  // row 0 = the PME CTA on the PME process (scheduled first: the CTAs that wait
  // for it can never starve it of a slot), rows after it = the local DD ranks
  const int l = (int)blockIdx.y - (M.hosts_pme ? 1 : 0);
  if (l >= 0) {
    const PmeRank& R = M.r[l];
    int b, e;
    share(R.n_home, gridDim.x, blockIdx.x, b, e);
    float* dst = M.pme_x + (size_t)R.off * W;
    if constexpr (W == 4) {
      const float4* s4 = reinterpret_cast<const float4*>(R.x);
      float4* d4 = reinterpret_cast<float4*>(dst);
      for (int i = b + threadIdx.x; i < e; i += blockDim.x) d4[i] = __ldg(s4 + i);
    } else {
      for (int i = 3 * b + threadIdx.x; i < 3 * e; i += blockDim.x) dst[i] = __ldg(R.x + i);
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      fence_sys();  // this CTA's peer stores before its completion increment
      if (atom_add_acqrel_gpu(&M.ctrl->cnt_pme[0][l], 1u) == gridDim.x - 1) {
        M.ctrl->cnt_pme[0][l] = 0;
        st_release_sys(&M.pme_hdr->pme_x_flag[R.rank], seq);
      }
    }
  } else if (blockIdx.x == 0) {
    // PME process: the launch completes when every rank's rows are in pme_x
    for (int t = threadIdx.x; t < M.nranks; t += blockDim.x)
      wait_geq<true>(&M.pme_hdr->pme_x_flag[t], seq, M.timeout_ns, M.err_host, tcode(18, t, 0), 0);
  }
  pme_depart(&M.ctrl->done_pme[0], &M.ctrl->seq_pme_x, seq);
}

template <int W>
__global__ void __launch_bounds__(256) k_pme_f(const __grid_constant__ PmeParams M) {
  __shared__ uint64_t s_seq;
  if (threadIdx.x == 0) s_seq = ld_relaxed_gpu(&M.ctrl->seq_pme_f) + 1;
  __syncthreads();
  const uint64_t seq = s_seq;
  const int l = (int)blockIdx.y - (M.hosts_pme ? 1 : 0);  // row 0: the PME CTA (as k_pme_x)
  if (l >= 0) {
    const PmeRank& R = M.r[l];
    if (threadIdx.x == 0)
      wait_geq<true>(&R.hdr->pme_f_flag, seq, M.timeout_ns, M.err_host, tcode(19, l, 0), 0);
    __syncthreads();
    int b, e;
    share(R.n_home, gridDim.x, blockIdx.x, b, e);
    const float* src = M.pme_f + (size_t)R.off * W;
    for (int i = W * b + threadIdx.x; i < W * e; i += blockDim.x) {
      const float v = __ldcg(src + i);  // written by the PME task on another GPU
      R.f[i] = M.accumulate ? __fadd_rn(R.f[i], v) : v;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      fence_sys();  // this CTA's reads of pme_f are complete before the ack
      if (atom_add_acqrel_gpu(&M.ctrl->cnt_pme[1][l], 1u) == gridDim.x - 1) {
        M.ctrl->cnt_pme[1][l] = 0;
        st_release_sys(&M.pme_hdr->pme_ack[R.rank], seq);
      }
    }
  } else if (blockIdx.x == 0) {
    // PME process: forces ready (its force kernel precedes this launch) -> every
    // rank; then wait until every slice was read (pme_f may be overwritten after)
    fence_sys();
    for (int t = threadIdx.x; t < M.nranks; t += blockDim.x) st_release_sys(&M.all_hdr[t]->pme_f_flag, seq);
    for (int t = threadIdx.x; t < M.nranks; t += blockDim.x)
      wait_geq<true>(&M.pme_hdr->pme_ack[t], seq, M.timeout_ns, M.err_host, tcode(18, t, 1), 0);
  }
  pme_depart(&M.ctrl->done_pme[1], &M.ctrl->seq_pme_f, seq);
}

cudaError_t launch_pme(const PmeParams& M, int which, int ctas_per_rank, cudaStream_t st) {
  void* args[] = {(void*)&M};
  if (which == 0)
    return cudaLaunchKernel((const void*)k_pme_allgather, dim3(M.n_local), dim3(64), args, 0, st);
  const dim3 grid(ctas_per_rank, M.n_local + (M.hosts_pme ? 1 : 0));
  const void* fn = which == 1 ? (M.layout == 4 ? (const void*)k_pme_x<4> : (const void*)k_pme_x<3>)
                              : (M.layout == 4 ? (const void*)k_pme_f<4> : (const void*)k_pme_f<3>);
  return cudaLaunchKernel(fn, grid, dim3(256), args, 0, st);
}

}  // namespace halo
