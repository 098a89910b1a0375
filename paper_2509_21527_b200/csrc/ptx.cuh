// ptx.cuh — device-side memory-ordering helpers, bounded waits and launch
// epilogue shared by the libhalo kernels.  Private to libhalo.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>
#include "halo_internal.h"

namespace halo {

// ----------------------------------------------------------------- PTX helpers
__device__ __forceinline__ uint64_t ld_acquire_sys(const uint64_t* p) {
  uint64_t v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ uint64_t ld_acquire_gpu(const uint64_t* p) {
  uint64_t v;
  asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ uint64_t ld_relaxed_gpu(const uint64_t* p) {
  uint64_t v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_sys(uint64_t* p, uint64_t v) {
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ void st_release_gpu(uint64_t* p, uint64_t v) {
  asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ void st_relaxed_gpu(uint64_t* p, uint64_t v) {
  asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ uint32_t atom_add_acqrel_gpu(uint32_t* p, uint32_t v) {
  uint32_t old;
  asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], %2;" : "=r"(old) : "l"(p), "r"(v) : "memory");
  return old;
}
__device__ __forceinline__ void red_add_release_sys(uint64_t* p, uint64_t v) {
  asm volatile("red.release.sys.global.add.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ void red_add_relaxed_sys(uint64_t* p, uint64_t v) {
  asm volatile("red.relaxed.sys.global.add.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ void fence_sys() { asm volatile("fence.acq_rel.sys;" ::: "memory"); }
__device__ __forceinline__ void fence_gpu() { asm volatile("fence.acq_rel.gpu;" ::: "memory"); }
__device__ __forceinline__ uint64_t gtimer() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

__device__ __forceinline__ void st_relaxed_sys(uint64_t* p, uint64_t v) {
  asm volatile("st.relaxed.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ uint64_t ld_relaxed_sys(const uint64_t* p) {
  uint64_t v;
  asm volatile("ld.relaxed.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

// Asynchronous global -> shared copies (LDGSTS): the next work item's block is
// fetched while the current one is processed.
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  const uint32_t s = (uint32_t)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(s), "l"(gmem) : "memory");
}
// 4-byte asynchronous global -> shared copy (cached in L1: .ca is the only mode
// for sizes below 16 B)
__device__ __forceinline__ void cp_async4(void* smem, const void* gmem) {
  const uint32_t s = (uint32_t)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(s), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }

// Block copy of `bytes` (multiple of 16) by the whole CTA, asynchronous.
__device__ __forceinline__ void cp_async_block(void* smem, const void* gmem, uint32_t bytes) {
  for (uint32_t o = threadIdx.x * 16u; o < bytes; o += blockDim.x * 16u)
    cp_async16(static_cast<char*>(smem) + o, static_cast<const char*>(gmem) + o);
  cp_async_commit();
}

// Bulk (TMA engine) global -> shared copy completing on an mbarrier: one
// elected thread moves a whole work-item block (cp.async.bulk; 16-B aligned,
// size a multiple of 16), every thread waits on the barrier's phase.
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
// Issue the copy (caller: one thread).  The barrier's current phase completes
// when `bytes` have landed.
__device__ __forceinline__ void bulk_load(void* smem, const void* gmem, uint32_t bytes, uint64_t* bar) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
               ::"r"(smem_u32(smem)), "l"(gmem), "r"(bytes), "r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)), "r"(phase) : "memory");
}

// Bulk (TMA engine) shared -> global store, bulk-group completion (the paper's
// warp-leader TMA put, Alg. 3).  The destination may be a peer GPU's
// memory (CUDA-IPC mapping over NVLink).  16-B aligned, size a multiple of 16.
__device__ __forceinline__ void bulk_store(void* gmem, const void* smem, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;"
               ::"l"(gmem), "r"(smem_u32(smem)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
// all but the newest N groups have finished READING shared memory (buffer reuse)
template <int N>
__device__ __forceinline__ void bulk_wait_read() { asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory"); }
// every group of this thread is complete: its writes are performed
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
// order async-proxy global writes with the generic proxy (the release that follows)
__device__ __forceinline__ void fence_proxy_async_global() { asm volatile("fence.proxy.async.global;" ::: "memory"); }

// Programmatic dependent launch (sm_90+): let the next kernel of the stream be
// scheduled now, and block until the previous kernel's memory is complete.
// Bulk L2 prefetch (no data returned; a hint, coherent with later loads): 16-B
// aligned address, size a multiple of 16.
__device__ __forceinline__ void prefetch_l2_bulk(const void* gmem, uint32_t bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(gmem), "r"(bytes) : "memory");
}
__device__ __forceinline__ void pdl_launch_dependents() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

// Report a timeout once: host-mapped word (system scope) + give up.
static __device__ __noinline__ void report_timeout(int* err_host, int code) {
  volatile int* e = err_host;
  if (*e == 0) *e = code;
  fence_sys();
}

// Bounded spin: returns false on timeout.  `kSys` selects the scope of the acquire.
// Polls with RELAXED loads (an ld.acquire compiles to LDG.STRONG + CCTL.IVALL, i.e.
// it invalidates the SM's whole L1 on every poll, which slows every co-resident
// CTA); once the value is seen, one acquire load of the same (monotonic) word
// establishes the synchronisation.  The timer and the host-mapped (PCIe) error
// word are only looked at every 1024 polls, never on the latency path.
template <bool kSys>
__device__ __forceinline__ bool wait_geq(const uint64_t* p, uint64_t v, uint64_t timeout_ns, int* err_host,
                                         int code, uint32_t poll_ns = 0) {
  if ((kSys ? ld_relaxed_sys(p) : ld_relaxed_gpu(p)) < v) {
    uint64_t t0 = 0;
    for (uint32_t it = 1;; ++it) {
      if (poll_ns && poll_ns != 0xffffffffu) __nanosleep(poll_ns);  // 0xffffffff: kPollTight
      if ((kSys ? ld_relaxed_sys(p) : ld_relaxed_gpu(p)) >= v) break;
      if ((it & 1023u) == 0) {
        const uint64_t now = gtimer();
        if (t0 == 0) {
          t0 = now;
        } else if (now - t0 > timeout_ns) {
          report_timeout(err_host, code);
          return false;
        }
        if (*(volatile int*)err_host != 0) return false;  // another wait already failed: drain
      }
    }
  }
  (void)(kSys ? ld_acquire_sys(p) : ld_acquire_gpu(p));
  return true;
}

// Wait until (*p >> 32) == epoch; returns the low 32 bits (or 0xffffffff on timeout).
__device__ __forceinline__ uint32_t wait_epoch(const uint64_t* p, uint32_t epoch, uint64_t timeout_ns,
                                               int* err_host, int code) {
  uint64_t t0 = 0;
  for (uint32_t it = 0;; ++it) {
    uint64_t v = ld_relaxed_sys(p);
    if ((uint32_t)(v >> 32) == epoch) {
      v = ld_acquire_sys(p);  // same word (only its writer changes it during this epoch)
      return (uint32_t)v;
    }
    if ((it & 1023u) == 1023u) {
      const uint64_t now = gtimer();
      if (t0 == 0) {
        t0 = now;
      } else if (now - t0 > timeout_ns) {
        report_timeout(err_host, code);
        return 0xffffffffu;
      }
      if (*(volatile int*)err_host != 0) return 0xffffffffu;
    }
  }
}

// timeout codes: kind << 16 | lrank << 8 | pulse
__device__ __forceinline__ int tcode(int kind, int lr, int p) { return (kind << 16) | (lr << 8) | p; }

// ------------------------------------------------------------- per-CTA timing
__device__ __forceinline__ void timer_start(unsigned flags, uint64_t* t_start) {
  if ((flags & HALO_F_TIMERS) && threadIdx.x == 0) atomicMin((unsigned long long*)t_start, gtimer());
}

// Kernel epilogue: the last CTA publishes the sequence number (graph-safe) and timer span.
__device__ __forceinline__ void finish_launch(unsigned flags, uint32_t* done, uint64_t* seq_slot, uint64_t seq,
                                              uint64_t* t_start, uint64_t* t_end, uint64_t* span) {
  if (threadIdx.x == 0) {
    if (flags & HALO_F_TIMERS) atomicMax((unsigned long long*)t_end, gtimer());
    uint32_t old = atom_add_acqrel_gpu(done, 1u);
    if (old == gridDim.x - 1) {
      *done = 0;
      if (flags & HALO_F_TIMERS) {
        *span = *t_end - *t_start;
        *t_start = ~0ull;
        *t_end = 0;
      }
      st_release_gpu(seq_slot, seq);
    }
  }
}

// Early-arrive variant of finish_launch (LL kernels).  Thread 0 increments the
// launch's arrival counter right after reading the sequence number (ordered by
// the preceding __syncthreads, which consumed the load), so the atomic's round
// trip overlaps the CTA's work.  The CTA that arrived last publishes the
// sequence number at its exit: by then every CTA of the launch has read it.
__device__ __forceinline__ uint32_t launch_arrive(uint32_t* done) {
  uint32_t old = 0;
  // relaxed: the sequence-number load it must follow was consumed before the
  // barrier that precedes this call; no fence (a MEMBAR drains behind pollers)
  if (threadIdx.x == 0)
    asm volatile("atom.relaxed.gpu.global.add.u32 %0, [%1], 1;" : "=r"(old) : "l"(done) : "memory");
  return old;
}

__device__ __forceinline__ void launch_depart(unsigned flags, uint32_t arrived, uint32_t* done, uint64_t* seq_slot,
                                              uint64_t seq, uint64_t* t_start, uint64_t* t_end, uint64_t* span) {
  if (threadIdx.x != 0) return;
  if (flags & HALO_F_TIMERS) atomicMax((unsigned long long*)t_end, gtimer());
  if (arrived == gridDim.x - 1) {
    *done = 0;
    st_relaxed_gpu(seq_slot, seq);
    if (flags & HALO_F_TIMERS) {
      // spans need every CTA's end stamp: only approximate here (the last arriver's exit)
      *span = gtimer() - *t_start;
      *t_start = ~0ull;
      *t_end = 0;
    }
  }
}

}  // namespace halo
