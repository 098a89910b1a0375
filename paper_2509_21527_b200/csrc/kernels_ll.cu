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
// Items are processed in a static order in which every wait targets an
// earlier item, and the grid is launched cooperatively.
#include <cuda_runtime.h>
#include <stdint.h>

#include "halo_internal.h"
#include "ptx.cuh"

namespace halo {

__device__ __forceinline__ uint64_t ll_pack(float v, uint32_t tag) {
  return ((uint64_t)tag << 32) | (uint64_t)__float_as_uint(v);
}

// Poll one LL unit until it carries `tag`; bounded like every other wait.
__device__ __forceinline__ float ll_wait(const uint64_t* u, uint32_t tag, uint64_t timeout_ns, int* err_host,
                                         int code) {
  uint64_t v = ld_relaxed_sys(u);
  if ((uint32_t)(v >> 32) == tag) return __uint_as_float((uint32_t)v);
  uint64_t t0 = 0;
  for (uint32_t it = 1;; ++it) {
    v = ld_relaxed_sys(u);
    if ((uint32_t)(v >> 32) == tag) return __uint_as_float((uint32_t)v);
    if ((it & 1023u) == 0) {
      const uint64_t now = gtimer();
      if (t0 == 0) {
        t0 = now;
      } else if (now - t0 > timeout_ns) {
        report_timeout(err_host, code);
        return __uint_as_float((uint32_t)v);
      }
      if (*(volatile int*)err_host != 0) return __uint_as_float((uint32_t)v);
    }
  }
}

// ---------------------------------------------------------------- x (LL)
template <int W>
__global__ void __launch_bounds__(kThreads) k_exchange_x_ll(const __grid_constant__ ExParams P) {
  __shared__ uint64_t s_seq;
  Ctrl* ctrl = P.ctrl;
  if (threadIdx.x == 0) s_seq = ld_relaxed_gpu(&ctrl->seq_x) + 1;
  timer_start(P.flags, &ctrl->t_start_x);
  __syncthreads();
  const uint64_t seq = s_seq;
  const uint32_t tag = (uint32_t)seq;

  for (int it = blockIdx.x; it < P.n_items; it += gridDim.x) {
    const Item w = P.items[it];
    const RankDev& rd = P.ranks[w.lrank];
    const uint32_t u0 = w.begin * W, u1 = w.end * W;
    if (w.kind == kItemXRecv) {
      // this rank's halo rows of pulse p: LL units -> x rows [recv_off, +recv_size)
      const uint64_t* src = rd.xll + (size_t)w.pulse * P.ll_stride;
      float* dst = rd.x + (size_t)rd.recv_off[w.pulse] * W;
      for (uint32_t u = u0 + threadIdx.x; u < u1; u += blockDim.x)
        dst[u] = ll_wait(src + u, tag, P.timeout_ns, P.err_host, tcode(10, w.lrank, w.pulse));
      continue;
    }
    // SEND: gather through the map, shift (R25), tag, store into the receiver's LL buffer
    const PulseDev& pd = P.pulses[w.lrank * P.P + w.pulse];
    const int32_t* __restrict__ map = pd.map;
    const float* __restrict__ x = rd.x;
    uint64_t* dst = pd.xll_dst;
    const bool dep = (w.kind == kItemXDep);
    const bool sh = pd.has_shift != 0;
    for (uint32_t u = u0 + threadIdx.x; u < u1; u += blockDim.x) {
      const uint32_t i = u / W;
      const int c = (int)(u - i * W);
      const int idx = __ldg(map + i);
      float v;
      if (!dep) {
        v = __ldg(x + (size_t)idx * W + c);  // home row: never written during the kernel
      } else {
        // forwarded row: find the pulse it arrived in (Alg. 4 dependent part, R8/R9)
        int q = 0;
        while (q < P.P - 1 && (unsigned)(idx - rd.recv_off[q]) >= (unsigned)rd.recv_size[q]) ++q;
        if (q < P.p_lo) {
          v = __ldcg(x + (size_t)idx * W + c);  // arrived in an earlier launch (set_maps)
        } else {
          const uint64_t* src = rd.xll + (size_t)q * P.ll_stride + (size_t)(idx - rd.recv_off[q]) * W + c;
          v = ll_wait(src, tag, P.timeout_ns, P.err_host, tcode(11, w.lrank, q));
        }
      }
      if (sh && c < 3) v = __fadd_rn(v, pd.shift[c]);
      st_relaxed_sys(dst + u, ll_pack(v, tag));
    }
  }
  __syncthreads();
  finish_launch(P.flags, &ctrl->done_x, &ctrl->seq_x, seq, &ctrl->t_start_x, &ctrl->t_end_x, &ctrl->span_x);
}

// ---------------------------------------------------------------- f (LL)
__device__ __forceinline__ double warp_sum_d(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

template <int W>
__global__ void __launch_bounds__(kThreads) k_exchange_f_ll(const __grid_constant__ ExParams P) {
  __shared__ uint64_t s_seq;
  Ctrl* ctrl = P.ctrl;
  if (threadIdx.x == 0) s_seq = ld_relaxed_gpu(&ctrl->seq_f) + 1;
  timer_start(P.flags, &ctrl->t_start_f);
  __syncthreads();
  const uint64_t seq = s_seq;
  const uint32_t tag = (uint32_t)seq;

  for (int it = blockIdx.x; it < P.n_items; it += gridDim.x) {
    const Item w = P.items[it];
    const RankDev& rd = P.ranks[w.lrank];
    const int level = w.pulse;  // pulse whose slice these rows are, or kHomeLevel
    const bool push = level != kHomeLevel;
    uint64_t* pdst = nullptr;
    int poff = 0;
    if (push) {
      const PulseDev& pd = P.pulses[w.lrank * P.P + level];
      pdst = pd.fll_dst;
      poff = rd.recv_off[level];
    }
    const int wrap = (P.fshift != nullptr) ? rd.wrap_mask : 0;
    double acc[3][3] = {{0.0, 0.0, 0.0}, {0.0, 0.0, 0.0}, {0.0, 0.0, 0.0}};
    float* __restrict__ f = rd.f;
    const uint32_t u0 = w.begin * W, u1 = w.end * W;
    for (uint32_t u = u0 + threadIdx.x; u < u1; u += blockDim.x) {
      const uint32_t k = u / W;
      const int c = (int)(u - k * W);
      const int t = __ldg(rd.task_row + k);
      const int j0 = __ldg(rd.task_off + k), j1 = __ldg(rd.task_off + k + 1);
      float v = f[(size_t)t * W + c];
      for (int j = j0; j < j1; ++j) {  // contributions, pulses descending (R15)
        const uint32_t cc = __ldg(rd.contrib + j);
        const int q = (int)(cc >> 24);
        const uint32_t i = cc & 0xffffffu;
        const float val = ll_wait(rd.fll + (size_t)q * P.ll_stride + (size_t)i * W + c, tag, P.timeout_ns,
                                  P.err_host, tcode(12, w.lrank, q));
        v = P.accumulate ? __fadd_rn(v, val) : val;
        if (((wrap >> q) & 1) && c < 3) {
          const int d = rd.pulse_dim[q];
#pragma unroll
          for (int dd = 0; dd < 3; ++dd)
#pragma unroll
            for (int cc2 = 0; cc2 < 3; ++cc2)
              if (dd == d && cc2 == c) acc[dd][cc2] += (double)val;
        }
      }
      f[(size_t)t * W + c] = v;
      if (push) st_relaxed_sys(pdst + (size_t)(t - poff) * W + c, ll_pack(v, tag));
    }
    if (wrap) {  // shift forces (R13): warp-reduce, one fp64 atomic per (dim, comp) per warp
      double* fs = P.fshift + 9 * w.lrank;
      for (int d = 0; d < 3; ++d) {
        bool has = false;
        for (int q = 0; q < P.P; ++q) has |= ((wrap >> q) & 1) && rd.pulse_dim[q] == d;
        if (!has) continue;
#pragma unroll
        for (int c = 0; c < 3; ++c) {
          const double s = warp_sum_d(acc[d][c]);
          if ((threadIdx.x & 31) == 0 && s != 0.0) atomicAdd(fs + 3 * d + c, s);
        }
      }
    }
  }
  __syncthreads();
  finish_launch(P.flags, &ctrl->done_f, &ctrl->seq_f, seq, &ctrl->t_start_f, &ctrl->t_end_f, &ctrl->span_f);
}

// ------------------------------------------------------------- launchers
cudaError_t launch_coop_kernel(const void* fn, int grid, int block, void** args, cudaStream_t st);

cudaError_t launch_exchange_x_ll(const ExParams& p, int layout, int grid, cudaStream_t st) {
  void* args[] = {(void*)&p};
  const void* fn = layout == 4 ? (const void*)k_exchange_x_ll<4> : (const void*)k_exchange_x_ll<3>;
  return launch_coop_kernel(fn, grid, kThreads, args, st);
}

cudaError_t launch_exchange_f_ll(const ExParams& p, int layout, int grid, cudaStream_t st) {
  void* args[] = {(void*)&p};
  const void* fn = layout == 4 ? (const void*)k_exchange_f_ll<4> : (const void*)k_exchange_f_ll<3>;
  return launch_coop_kernel(fn, grid, kThreads, args, st);
}

cudaError_t max_coresident_ll(int layout, int* x_blocks, int* f_blocks) {
  int dev = 0, sms = 0, bx = 0, bf = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  if (e != cudaSuccess) return e;
  e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(
      &bx, layout == 4 ? (const void*)k_exchange_x_ll<4> : (const void*)k_exchange_x_ll<3>, kThreads, 0);
  if (e != cudaSuccess) return e;
  e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(
      &bf, layout == 4 ? (const void*)k_exchange_f_ll<4> : (const void*)k_exchange_f_ll<3>, kThreads, 0);
  if (e != cudaSuccess) return e;
  *x_blocks = bx * sms;
  *f_blocks = bf * sms;
  return cudaSuccess;
}

}  // namespace halo
