// kernels_ns.cu — NS-step kernels of libhalo: home-atom redistribution
// (halo_migrate).
//
// At a neighbour-search step (every nstlist steps) the domains are
// re-populated with the atoms inside their region before the send
// maps are rebuilt (halo_set_maps).  Per local rank, stream-ordered:
//
//   k_mig_count     wrap every home row into the box (R29), find its cell
//   k_mig_scan      (fp64 planes, R3/R4) and its stencil slot (R30); count per
//   k_mig_scatter   CTA, prefix, then write the rows grouped by destination — a
//                   stable compaction over contiguous CTA ranges, so every group
//                   stays in ascending gid — into the own staging-out area
//   k_mig_publish   per stencil rank: (offset, count) of its group into ITS
//                   header, count by system-scope release (the rows before it)
//   k_mig_wait      acquire every stencil rank's count for this rank; prefix ->
//                   where each received list goes in staging-in; capacity check
//   (k_status)      error bits agreed over all ranks before any row moves
//   k_mig_gather    copy the lists (NVLink peer loads from the sources'
//                   staging-out) into the own staging-in, concatenated
//   k_mig_merge     k-way merge by gid: a row's output index = its index in its
//                   list + the number of smaller gids in every other list
//                   (binary searches; gids are unique) -> x, gid, v rows
//   k_mig_ack       tell every source its rows were copied; wait for the same
//                   from every destination (staging-out may be reused after)
//
// Every wait is bounded (%globaltimer; timeout -> HALO_ERR_TIMEOUT).  On an
// agreed error nothing is gathered or merged (x, gid, v keep their rows) and the
// acks still flow, so no rank waits forever.
#include <cuda_runtime.h>
#include <stdint.h>
#include "halo_internal.h"
#include "ptx.cuh"

namespace halo {

constexpr int kPlaneStride = kMaxRanks + 1;

// Staging area rows (SoA, capacity rows each): x | v | gid.
__device__ __forceinline__ float* stage_x(char* base) { return reinterpret_cast<float*>(base); }
__device__ __forceinline__ float* stage_v(char* base, int cap, int W) {
  return reinterpret_cast<float*>(base) + (size_t)cap * W;
}
__device__ __forceinline__ int32_t* stage_gid(char* base, int cap, int W) {
  return reinterpret_cast<int32_t*>(reinterpret_cast<float*>(base) + 2 * (size_t)cap * W);
}

// R29: one periodic wrap in float32 (x >= L -> x - L; x < 0 -> x + L, RNE), then
// a result equal to L or to zero becomes +0.0.  Returns false if the row is
// still outside [0, L) (it moved more than a box length).
__device__ __forceinline__ bool wrap_into_box(float& x, float L) {
  if (x >= L) x = __fsub_rn(x, L);
  else if (x < 0.0f) x = __fadd_rn(x, L);
  if (x == L || x == 0.0f) x = 0.0f;
  return x >= 0.0f && x < L;
}

// The stencil slot of home row i of rank R (or -1: outside the stencil, R30),
// with its wrapped coordinates.
template <int W>
__device__ __forceinline__ int mig_slot(const MigParams& M, const MigRank& R, int i, float (&v)[4]) {
  const float* src = R.x + (size_t)i * W;
#pragma unroll
  for (int c = 0; c < W; ++c) v[c] = src[c];
  bool ok = true;
  int cell[3];
#pragma unroll
  for (int d = 0; d < 3; ++d) {
    ok &= wrap_into_box(v[d], M.box[d]);
    // c_d = the largest k in [0, grid-1] with b_d[k] <= float64(x_d) (R4: ties go up)
    const double xd = (double)v[d];
    const double* b = M.planes + d * kPlaneStride;
    int k = 0;
    for (int kk = 1; kk < M.grid[d]; ++kk)
      if (b[kk] <= xd) k = kk;
    cell[d] = k;
  }
  if (!ok) return -1;
  const int dest = (cell[0] * M.grid[1] + cell[1]) * M.grid[2] + cell[2];
  for (int k = 0; k < R.n_nb; ++k)
    if (R.nb_rank[k] == dest) return k;
  return -1;
}

// CTA g of rank l handles rows [g*per, (g+1)*per): contiguous ranges keep the
// per-group order stable across CTAs.
__device__ __forceinline__ void mig_range(int n, int g, int& b, int& e) {
  const int per = (n + kMigBlocks - 1) / kMigBlocks;
  b = min(n, g * per);
  e = min(n, b + per);
}

// pass 1 (grid kMigBlocks x n_local): group sizes per CTA; gid strictly ascending
template <int W>
__global__ void __launch_bounds__(256) k_mig_count(const __grid_constant__ MigParams M, MigCtrl* C) {
  const int l = blockIdx.y, g = blockIdx.x;
  const MigRank& R = M.r[l];
  __shared__ int s_cnt[kStencil];
  __shared__ int s_err;
  if (threadIdx.x < kStencil) s_cnt[threadIdx.x] = 0;
  if (threadIdx.x == 0) s_err = 0;
  __syncthreads();
  int b, e;
  mig_range(R.n_home, g, b, e);
  for (int i = b + threadIdx.x; i < e; i += blockDim.x) {
    float v[4];
    const int k = mig_slot<W>(M, R, i, v);
    if (k < 0) atomicOr(&s_err, kErrGeometry);
    else atomicAdd(&s_cnt[k], 1);
    if (i > 0 && R.gid[i] <= R.gid[i - 1]) atomicOr(&s_err, kErrMap);
  }
  __syncthreads();
  if (threadIdx.x < kStencil) C->blk[l][g][threadIdx.x] = s_cnt[threadIdx.x];
  if (threadIdx.x == 0 && s_err) atomicOr(&C->err[l], s_err);
}

// group bases and per-CTA offsets inside each group (one warp per rank, lane = group)
__global__ void k_mig_scan(const __grid_constant__ MigParams M, MigCtrl* C) {
  const int l = blockIdx.x, k = threadIdx.x;
  const MigRank& R = M.r[l];
  __shared__ int s_tot[kStencil];
  int acc = 0;
  if (k < R.n_nb)
    for (int g = 0; g < kMigBlocks; ++g) {
      const int c = C->blk[l][g][k];
      C->blk[l][g][k] = acc;
      acc += c;
    }
  if (k < kStencil) s_tot[k] = acc;
  __syncwarp();
  if (k < R.n_nb) {
    int base = 0;
    for (int j = 0; j < k; ++j) base += s_tot[j];
    C->out_off[l][k] = base;
    C->out_cnt[l][k] = acc;
  }
}

// pass 2 (grid kMigBlocks x n_local): stable scatter of the CTA's rows into the
// staging-out groups, 256 rows at a time (per group: warp ballot rank + warp
// prefix + running base)
template <int W>
__global__ void __launch_bounds__(256) k_mig_scatter(const __grid_constant__ MigParams M, const MigCtrl* C) {
  const int l = blockIdx.y, g = blockIdx.x;
  const MigRank& R = M.r[l];
  const int cap = M.capacity;
  __shared__ int s_run[kStencil];
  __shared__ int s_wcnt[8][kStencil];
  if (threadIdx.x < R.n_nb) s_run[threadIdx.x] = C->out_off[l][threadIdx.x] + C->blk[l][g][threadIdx.x];
  __syncthreads();
  int b, e;
  mig_range(R.n_home, g, b, e);
  float* sx = stage_x(R.stage_out);
  float* sv = stage_v(R.stage_out, cap, W);
  int32_t* sg = stage_gid(R.stage_out, cap, W);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t lt = (1u << lane) - 1u;
  for (int base = b; base < e; base += blockDim.x) {
    const int i = base + threadIdx.x;
    float v[4] = {0.f, 0.f, 0.f, 0.f};
    const int k = (i < e) ? mig_slot<W>(M, R, i, v) : -1;
    int in_warp = 0;
    for (int kk = 0; kk < R.n_nb; ++kk) {
      const uint32_t m = __ballot_sync(0xffffffffu, k == kk);
      if (lane == 0) s_wcnt[warp][kk] = __popc(m);
      if (k == kk) in_warp = __popc(m & lt);
    }
    __syncthreads();
    if (threadIdx.x < R.n_nb) {
      int acc = s_run[threadIdx.x];
      for (int w = 0; w < (int)(blockDim.x >> 5); ++w) {
        const int c = s_wcnt[w][threadIdx.x];
        s_wcnt[w][threadIdx.x] = acc;
        acc += c;
      }
      s_run[threadIdx.x] = acc;
    }
    __syncthreads();
    if (k >= 0) {
      const size_t pos = (size_t)s_wcnt[warp][k] + in_warp;
#pragma unroll
      for (int c = 0; c < W; ++c) sx[pos * W + c] = v[c];
      sg[pos] = R.gid[i];
      if (M.has_v) {
#pragma unroll
        for (int c = 0; c < W; ++c) sv[pos * W + c] = R.v[(size_t)i * W + c];
      }
    }
    __syncthreads();
  }
}

__global__ void k_mig_publish(const __grid_constant__ MigParams M, const MigCtrl* C) {
  const int l = blockIdx.x;
  const MigRank& R = M.r[l];
  const int k = threadIdx.x;
  if (k >= R.n_nb) return;
  const uint64_t ep = (uint64_t)M.epoch << 32;
  fence_sys();  // the staging rows of k_mig_classify before the counts
  st_relaxed_sys(&R.nb_hdr[k]->mig_off[R.rank], ep | (uint32_t)C->out_off[l][k]);
  st_release_sys(&R.nb_hdr[k]->mig_cnt[R.rank], ep | (uint32_t)C->out_cnt[l][k]);
}

__global__ void k_mig_wait(const __grid_constant__ MigParams M, MigCtrl* C) {
  const int l = blockIdx.x;
  const MigRank& R = M.r[l];
  const int k = threadIdx.x;
  __shared__ int s_err;
  if (k == 0) s_err = 0;
  __syncthreads();
  if (k < R.n_nb) {
    const int src = R.nb_rank[k];
    uint32_t cnt = wait_epoch(&R.hdr->mig_cnt[src], M.epoch, M.timeout_ns, M.err_host, tcode(15, l, k));
    uint32_t off = 0;
    if (cnt == 0xffffffffu) {
      cnt = 0;
      atomicOr(&s_err, kErrCapacity);  // timed out: the error word reports it
    } else {
      off = (uint32_t)ld_relaxed_sys(&R.hdr->mig_off[src]);  // ordered by the acquire above
    }
    C->in_cnt[l][k] = (int)cnt;
    C->in_src_off[l][k] = (int)off;
  }
  __syncthreads();
  if (k == 0) {
    long acc = 0;
    for (int j = 0; j < R.n_nb; ++j) {
      C->in_off[l][j] = (int)acc;
      acc += C->in_cnt[l][j];
    }
    if (acc > M.capacity) {
      s_err |= kErrCapacity;
      acc = 0;  // nothing is gathered or merged on this rank
      for (int j = 0; j < R.n_nb; ++j) C->in_cnt[l][j] = C->in_off[l][j] = 0;
    }
    C->in_off[l][R.n_nb] = (int)acc;
    C->err[l] |= s_err;
    M.ctrl->err[l] = C->err[l];  // agreed over all ranks (k_status) before any row moves
  }
}

// list of received row g: the k with in_off[k] <= g < in_off[k+1]
__device__ __forceinline__ int list_of(const int32_t* in_off, int n_nb, int g) {
  int k = 0;
  while (k + 1 < n_nb && in_off[k + 1] <= g) ++k;
  return k;
}

template <int W>
__global__ void __launch_bounds__(256) k_mig_gather(const __grid_constant__ MigParams M, const MigCtrl* C) {
  const int l = blockIdx.y;
  const MigRank& R = M.r[l];
  const int cap = M.capacity;
  if (M.ctrl->agreed_err[l] != 0) return;  // some rank failed: no row moves anywhere
  const int total = C->in_off[l][R.n_nb];
  float* dx = stage_x(R.stage_in);
  float* dv = stage_v(R.stage_in, cap, W);
  int32_t* dg = stage_gid(R.stage_in, cap, W);
  for (int g = blockIdx.x * blockDim.x + threadIdx.x; g < total; g += gridDim.x * blockDim.x) {
    const int k = list_of(C->in_off[l], R.n_nb, g);
    const size_t src = (size_t)C->in_src_off[l][k] + (size_t)(g - C->in_off[l][k]);
    char* sb = const_cast<char*>(R.nb_stage[k]);  // the source's staging-out (peer memory)
    const float* sx = stage_x(sb);
#pragma unroll
    for (int c = 0; c < W; ++c) dx[(size_t)g * W + c] = __ldcg(sx + src * W + c);
    dg[g] = __ldcg(stage_gid(sb, cap, W) + src);
    if (M.has_v) {
      const float* sv = stage_v(sb, cap, W);
#pragma unroll
      for (int c = 0; c < W; ++c) dv[(size_t)g * W + c] = __ldcg(sv + src * W + c);
    }
  }
}

// number of entries < key in the ascending array a[0, n)
__device__ __forceinline__ int lower_bound(const int32_t* a, int n, int32_t key) {
  int lo = 0, hi = n;
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (a[mid] < key) lo = mid + 1;
    else hi = mid;
  }
  return lo;
}

template <int W>
__global__ void __launch_bounds__(256) k_mig_merge(const __grid_constant__ MigParams M, const MigCtrl* C) {
  const int l = blockIdx.y;
  const MigRank& R = M.r[l];
  const int cap = M.capacity;
  if (M.ctrl->agreed_err[l] != 0) return;
  const int total = C->in_off[l][R.n_nb];
  const float* sx = stage_x(R.stage_in);
  const float* sv = stage_v(R.stage_in, cap, W);
  const int32_t* sg = stage_gid(R.stage_in, cap, W);
  for (int g = blockIdx.x * blockDim.x + threadIdx.x; g < total; g += gridDim.x * blockDim.x) {
    const int k = list_of(C->in_off[l], R.n_nb, g);
    const int32_t key = sg[g];
    int pos = g - C->in_off[l][k];
    for (int j = 0; j < R.n_nb; ++j)
      if (j != k) pos += lower_bound(sg + C->in_off[l][j], C->in_cnt[l][j], key);
#pragma unroll
    for (int c = 0; c < W; ++c) R.x[(size_t)pos * W + c] = sx[(size_t)g * W + c];
    R.gid[pos] = key;
    if (M.has_v) {
#pragma unroll
      for (int c = 0; c < W; ++c) R.v[(size_t)pos * W + c] = sv[(size_t)g * W + c];
    }
  }
}

// ack every source, then wait for every destination's ack
__global__ void k_mig_ack(const __grid_constant__ MigParams M, const MigCtrl* C) {
  const int l = blockIdx.x;
  const MigRank& R = M.r[l];
  const int k = threadIdx.x;
  const uint64_t ep = (uint64_t)M.epoch << 32;
  if (k < R.n_nb) {
    st_release_sys(&R.nb_hdr[k]->mig_ack[R.rank], ep);  // after k_mig_gather (stream order)
    wait_epoch(&R.hdr->mig_ack[R.nb_rank[k]], M.epoch, M.timeout_ns, M.err_host, tcode(16, l, k));
  }
}

// phase 0: classify, publish, wait (then the caller agrees the error bits);
// phase 1: gather, merge, ack.
cudaError_t launch_migrate(const MigParams& M, MigCtrl* C, int max_rows, int phase, cudaStream_t st) {
  const int L = M.n_local;
  const int W = M.layout;
  void* a2[] = {(void*)&M, (void*)&C};
  cudaError_t e;
  if (phase == 0) {
    const dim3 gb(kMigBlocks, L);
    e = cudaLaunchKernel(W == 4 ? (const void*)k_mig_count<4> : (const void*)k_mig_count<3>, gb, dim3(256), a2, 0, st);
    if (e != cudaSuccess) return e;
    if ((e = cudaLaunchKernel((const void*)k_mig_scan, dim3(L), dim3(32), a2, 0, st)) != cudaSuccess) return e;
    e = cudaLaunchKernel(W == 4 ? (const void*)k_mig_scatter<4> : (const void*)k_mig_scatter<3>, gb, dim3(256), a2, 0,
                         st);
    if (e != cudaSuccess) return e;
    if ((e = cudaLaunchKernel((const void*)k_mig_publish, dim3(L), dim3(32), a2, 0, st)) != cudaSuccess) return e;
    return cudaLaunchKernel((const void*)k_mig_wait, dim3(L), dim3(32), a2, 0, st);
  }
  const int gx = max_rows > 0 ? (max_rows + 255) / 256 : 1;
  const dim3 grid(gx < 1184 ? gx : 1184, L);
  if ((e = cudaLaunchKernel(W == 4 ? (const void*)k_mig_gather<4> : (const void*)k_mig_gather<3>, grid, dim3(256),
                            a2, 0, st)) != cudaSuccess)
    return e;
  if ((e = cudaLaunchKernel(W == 4 ? (const void*)k_mig_merge<4> : (const void*)k_mig_merge<3>, grid, dim3(256), a2,
                            0, st)) != cudaSuccess)
    return e;
  return cudaLaunchKernel((const void*)k_mig_ack, dim3(L), dim3(32), a2, 0, st);
}

// ------------------------------------------------------------ home assignment
// halo_assign_home: the home DD rank of every atom of a global coordinate array
// ("divides the simulation box into spatial regions (domains)"; R3/R4:
// c_d = the number of interior planes b_d[k] <= float64(x_d), ties go up; rank =
// (cx*np_y + cy)*np_z + cz), then a stable counting sort of the atom ids by
// rank.  Pass 1: rank per atom + per-rank counts (CTA histogram, one atomic per
// rank and CTA, also binned per atom segment); x outside [0, L_d) sets err.
// Pass 2: one CTA per (rank, segment) scans its segment in order and appends
// the rank's atom ids (warp ballot + CTA prefix) at the rank's offset plus the
// rank's count in the earlier segments, so every rank's ids come out ascending.
__global__ void __launch_bounds__(256) k_home_rank(const float* __restrict__ x, int n, int stride, AssignParams A,
                                                   int32_t* __restrict__ rank, int* __restrict__ counts,
                                                   int* __restrict__ seg, int seg_len, int* err) {
  __shared__ int s_cnt[kMaxRanks];
  const int nr = A.grid[0] * A.grid[1] * A.grid[2];
  for (int r = threadIdx.x; r < nr; r += blockDim.x) s_cnt[r] = 0;
  __syncthreads();
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) {
    int cell[3];
    bool ok = true;
#pragma unroll
    for (int d = 0; d < 3; ++d) {
      const double xd = (double)x[(size_t)i * stride + d];
      const double* b = A.planes + d * kPlaneStride;
      ok &= xd >= 0.0 && xd < b[A.grid[d]];  // also false for NaN
      int k = 0;
      for (int kk = 1; kk < A.grid[d]; ++kk)
        if (b[kk] <= xd) k = kk;
      cell[d] = k;
    }
    if (!ok) atomicOr(err, 1);
    const int r = (cell[0] * A.grid[1] + cell[1]) * A.grid[2] + cell[2];
    rank[i] = r;
    atomicAdd(&s_cnt[r], 1);
  }
  __syncthreads();
  // seg_len is a multiple of blockDim.x: the CTA lies in one segment
  const int sg = (int)(((size_t)blockIdx.x * blockDim.x) / seg_len);
  for (int r = threadIdx.x; r < nr; r += blockDim.x)
    if (s_cnt[r]) {
      atomicAdd(&counts[r], s_cnt[r]);
      atomicAdd(&seg[sg * nr + r], s_cnt[r]);
    }
}

__global__ void __launch_bounds__(1024) k_home_compact(const int32_t* __restrict__ rank, int n,
                                                       const int* __restrict__ counts, const int* __restrict__ seg,
                                                       int seg_len, int32_t* __restrict__ ids) {
  __shared__ int s_warp[32];
  __shared__ int s_base;
  const int r = blockIdx.x, sg = blockIdx.y, nr = gridDim.x;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  if (threadIdx.x == 0) {
    int b = 0;
    for (int q = 0; q < r; ++q) b += counts[q];
    for (int t = 0; t < sg; ++t) b += seg[t * nr + r];
    s_base = b;
  }
  __syncthreads();
  int base = s_base;
  const int lo = sg * seg_len, hi = min(n, lo + seg_len);
  for (int c0 = lo; c0 < hi; c0 += blockDim.x) {
    const int i = c0 + threadIdx.x;
    const bool mine = i < hi && rank[i] == r;
    const unsigned m = __ballot_sync(0xffffffffu, mine);
    if (lane == 0) s_warp[warp] = __popc(m);
    __syncthreads();
    int before = 0, tot = 0;
    for (int w = 0; w < nw; ++w) {
      const int c = s_warp[w];
      before += w < warp ? c : 0;
      tot += c;
    }
    if (mine) ids[base + before + __popc(m & ((1u << lane) - 1u))] = i;
    base += tot;
    __syncthreads();  // s_warp is rewritten by the next chunk
  }
}

cudaError_t launch_assign_home(const float* x, int n, int stride, const AssignParams& A, int32_t* rank, int* counts,
                               int* seg, int32_t* ids, int* err, cudaStream_t st) {
  const int nr = A.grid[0] * A.grid[1] * A.grid[2];
  cudaError_t e = cudaMemsetAsync(counts, 0, sizeof(int) * nr, st);
  if (e == cudaSuccess) e = cudaMemsetAsync(err, 0, sizeof(int), st);
  if (e == cudaSuccess) e = cudaMemsetAsync(seg, 0, sizeof(int) * kAssignSegs * nr, st);
  if (e != cudaSuccess || n == 0) return e;
  // segments of a whole number of pass-1 CTAs; at most kAssignSegs of them
  const int per = (n + kAssignSegs - 1) / kAssignSegs;
  const int seg_len = (per + 255) / 256 * 256;
  const int nseg = (n + seg_len - 1) / seg_len;
  k_home_rank<<<(n + 255) / 256, 256, 0, st>>>(x, n, stride, A, rank, counts, seg, seg_len, err);
  if ((e = cudaGetLastError()) != cudaSuccess) return e;
  k_home_compact<<<dim3(nr, nseg), 1024, 0, st>>>(rank, n, counts, seg, seg_len, ids);
  return cudaGetLastError();
}

}  // namespace halo
