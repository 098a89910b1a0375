// kernels_plan.cu — GPU build of the LL protocol's per-epoch plan (set_maps, SURVEY
// §8(f) f2: "the map build ... and the gather plan on the device").
//
// The host version (runtime.cu build_ll_x / build_ll_f) walks every halo row of every
// local rank; at C3 that took milliseconds of host time per NS step plus the download
// of every map and the upload of the MB-sized item blocks.  Here the maps never leave
// the device: the host fills a small descriptor (PlanDev: per (local rank, pulse)
// relations and pointers), the kernels below count the work items, the host reads the
// counts (a few hundred bytes) and fixes the item offsets, and the kernels write the
// item blocks in place.  The blocks are the ones the host builds,
// except that a force item's shift-force buckets are the targets of every tree rooted
// at its rank (<= 2^P - 1 <= 7 for P <= 3, R13) instead of its own trees' targets.
//
//   x (Alg. 3/4, rows from their origin):
//     k_plan_org_home / k_plan_org_pulse(q): the origin of every row (a home row of a
//       rank of this group, or the LL unit in which it entered the group) and the
//       pulses whose +L shift it picked up since (R25), pulses in order;
//     k_plan_x<0/1/2>: the send entries of every (pulse, local rank) cut into items at
//       every change of dependency class and every R rows (chunked: last class changes,
//       counts, then write).
//   f (Alg. 5/6, trees):
//     k_plan_child: the inverse maps (row t of rank l is entry i of map q);
//     k_plan_roots: which rows root a tree and its class (a depth-first walk, children
//       in descending pulse order: R15), roots per class per CTA; k_plan_rank: their
//       prefix over the CTAs (a root's rank within its (class, local rank) is that
//       prefix + its rank in its CTA, row order);
//     k_plan_f: each root's 32-B record + node indices into its item, item records.
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>

#include "halo_internal.h"

namespace {
// The plan kernels run back to back on one stream, each a programmatic dependent of
// the previous one (plan_launch): its CTAs become resident while the previous grid
// drains, and griddepcontrol.wait holds them until that grid completed and its
// writes are visible (each kernel waits before touching memory, so the chain is
// transitive).  Saves the launch gap between the ~12 small kernels of an NS step.
__device__ __forceinline__ void plan_pdl() {
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}
// Checked build (-DHALO_BOUNDS_CHECK): item indices of the block writes and
// map entries are checked; a failure reports kErrKindBounds (local rank 0xfe = plan) and
// the write is skipped.
#ifdef HALO_BOUNDS_CHECK
__device__ __noinline__ bool plan_bc_fail(const halo::PlanDev* D, int code) {
  volatile int* e = D->err_host;
  if (*e == 0) *e = (halo::kErrKindBounds << 16) | (0xfe << 8) | code;
  __threadfence_system();
  return false;
}
#define PLAN_BC(cond, code) ((cond) ? true : plan_bc_fail(D, (code)))
#else
#define PLAN_BC(cond, code) true
#endif
template <typename... Args, typename... Actual>
cudaError_t plan_launch(void (*k)(Args...), dim3 grid, unsigned block, cudaStream_t st, Actual... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = dim3(block);
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, k, static_cast<Args>(args)...);
}
}  // namespace

namespace halo {

namespace {

constexpr int kPB = 256;  // threads per CTA of the scan kernels

__device__ __forceinline__ uint64_t org_pack(uint32_t row, uint32_t l, uint32_t kq, uint32_t mask, uint32_t cls) {
  return (uint64_t)row | ((uint64_t)l << 24) | ((uint64_t)kq << 32) | ((uint64_t)mask << 40) | ((uint64_t)cls << 48);
}
__device__ __forceinline__ uint32_t org_cls(uint64_t o) { return (uint32_t)(o >> 48) & 0xffu; }

// Inclusive max-scan over the CTA (kPB threads); every thread gets its prefix.
__device__ __forceinline__ int block_scan_max(int v, int* s_w) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, v, o);
    if (lane >= o) v = max(v, y);
  }
  if (lane == 31) s_w[w] = v;
  __syncthreads();
  int pre = -1;
  for (int k = 0; k < w; ++k) pre = max(pre, s_w[k]);
  __syncthreads();
  return max(v, pre);
}

// Per class c < nc: the number of threads t <= me with pred && cls == c (inclusive),
// returned for the caller's own class (pred or not; 0 <= cls < nc); totals of every
// class into s_tot.
__device__ __forceinline__ int block_count_class(bool pred, int cls, int nc, int (*s_w)[kPB / 32], int* s_tot) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  int mine = 0;
  for (int c = 0; c < nc; ++c) {
    const unsigned b = __ballot_sync(0xffffffffu, pred && cls == c);
    if (lane == 0) s_w[c][w] = __popc(b);
    if (cls == c) mine = __popc(b & (0xffffffffu >> (31 - lane)));
  }
  __syncthreads();
  int pre = 0;  // (every thread: an entry inside an item counts the starts before it too)
  for (int k = 0; k < w; ++k) pre += s_w[cls][k];
  if (threadIdx.x < nc) {
    int t = 0;
    for (int k = 0; k < kPB / 32; ++k) t += s_w[threadIdx.x][k];
    s_tot[threadIdx.x] = t;
  }
  __syncthreads();
  return pre + mine;
}

}  // namespace

// ------------------------------------------------------------------ x origins
__global__ void k_plan_org_home(const PlanDev* __restrict__ D) {
  plan_pdl();
  const int l = blockIdx.y;
  const int n = D->n_home[l];
  uint64_t* o = D->org + (size_t)l * D->cap;
  for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < n; t += gridDim.x * blockDim.x)
    o[t] = org_pack((uint32_t)t, (uint32_t)l, 0, 0, 0);
}

// The rows this rank received in pulse q: from a rank of this group, the origin of the
// sent row (+ this pulse's shift bit if the sender wrapped); from another group, the
// LL unit i of slot q (class q + 1).  Pulses in order (stream-ordered launches).
__global__ void k_plan_org_pulse(const PlanDev* __restrict__ D, int q) {
  plan_pdl();
  const int l = blockIdx.y;
  const PlanLQ& a = D->lq[l][q];
  uint64_t* o = D->org + (size_t)l * D->cap + a.atom_offset;
  const int s = a.snd_l;
  const int32_t* m = s >= 0 ? D->maps[s] + (size_t)q * D->map_stride : nullptr;
  const uint64_t sh = (s >= 0 && D->lq[s][q].wraps) ? ((uint64_t)(1u << q) << 40) : 0;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < a.recv_size; i += gridDim.x * blockDim.x)
    o[i] = s >= 0 ? (D->org[(size_t)s * D->cap + m[i]] | sh)
                  : org_pack((uint32_t)i, (uint32_t)l, 0x80u | (uint32_t)q, 0, (uint32_t)q + 1);
}

// ------------------------------------------------------------------ x items
// The send entries of (pulse p, local rank l), map order, cut into items at every change
// of dependency class and every R entries within a run of one class (the host's
// build_ll_x).  kPB entries per CTA (blockIdx.x = chunk, blockIdx.y = p * L + l); three
// passes so that no CTA walks a whole map:
//   A: the last class change in each chunk (xlast[pl][c]);
//   B: with the run start carried from the chunks before (max of their last changes),
//      the item starts per class (xcnt totals, xccnt per chunk) and the last start;
//   C: with every carry (run start, item start, items per class before the chunk), each
//      entry's XEnt and, by each item's last entry, its XRec, at item
//      xoff[class][p][l] + (index in class).
__device__ __forceinline__ int plan_x_cls(const uint64_t* org, const int32_t* m, int k) {
  return (int)org_cls(org[m[k]]);
}

template <int kPass>
__global__ void __launch_bounds__(kPB) k_plan_x(const PlanDev* __restrict__ D) {
  plan_pdl();
  const int pl = blockIdx.y, p = pl / D->L, l = pl % D->L, c = blockIdx.x;
  const PlanLQ& a = D->lq[l][p];
  const int n = a.send_size, R = D->R, nc = D->P + 1;
  const int k = c * kPB + threadIdx.x;
  if (c * kPB >= max(n, 1)) return;  // (uniform per CTA)
  const int32_t* m = D->maps[l] + (size_t)p * D->map_stride;
  const uint64_t* org = D->org + (size_t)l * D->cap;
  const size_t cb = (size_t)pl * D->xnch;  // this (p, l)'s chunk records
  __shared__ int s_w[kMaxP + 1][kPB / 32];
  __shared__ int s_mx[kPB / 32];
  __shared__ int s_tot[kMaxP + 1];
  __shared__ int s_carry[2 + kMaxP + 1];  // run start, item start, items per class before this chunk
  __shared__ uint8_t s_cls[kPB + 1];
  const bool valid = k < n;
  const uint64_t o = valid ? org[m[k]] : 0;
  const int cls = valid ? (int)org_cls(o) : 0;
  s_cls[threadIdx.x] = (uint8_t)cls;
  if (threadIdx.x == 0) s_cls[kPB] = (k + kPB < n) ? (uint8_t)plan_x_cls(org, m, k + kPB) : 0xffu;
  if (kPass > 0 && threadIdx.x < 32) {  // carries from the chunks before this one
    int rs = -1, is = -1;
    for (int j = threadIdx.x; j < c; j += 32) {
      rs = max(rs, D->xlast[cb + j]);
      if (kPass == 2) is = max(is, D->xlstart[cb + j]);
    }
#pragma unroll
    for (int o2 = 16; o2 > 0; o2 >>= 1) {
      rs = max(rs, __shfl_xor_sync(0xffffffffu, rs, o2));
      is = max(is, __shfl_xor_sync(0xffffffffu, is, o2));
    }
    if (threadIdx.x == 0) {
      s_carry[0] = rs;
      s_carry[1] = is;
    }
    if (kPass == 2)
      for (int cc = 0; cc < nc; ++cc) {
        int t = 0;
        for (int j = threadIdx.x; j < c; j += 32) t += D->xccnt[(cb + j) * (kMaxP + 1) + cc];
#pragma unroll
        for (int o2 = 16; o2 > 0; o2 >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o2);
        if (threadIdx.x == 0) s_carry[2 + cc] = t;
      }
  }
  __syncthreads();
  const int prev = threadIdx.x == 0 ? (k > 0 && valid ? plan_x_cls(org, m, k - 1) : -1) : (int)s_cls[threadIdx.x - 1];
  const bool change = valid && (k == 0 || cls != prev);
  if (kPass == 0) {
    const int lc = block_scan_max(change ? k : -1, s_mx);
    if (threadIdx.x == kPB - 1) D->xlast[cb + c] = lc;
    return;
  }
  const int runstart = max(block_scan_max(change ? k : -1, s_mx), s_carry[0]);
  const bool start = valid && (change || (k - runstart) % R == 0);
  if (kPass == 1) {
    const int ls = block_scan_max(start ? k : -1, s_mx);
    (void)block_count_class(start, cls, nc, s_w, s_tot);
    if (threadIdx.x == kPB - 1) D->xlstart[cb + c] = ls;
    if (threadIdx.x < nc) {
      D->xccnt[(cb + c) * (kMaxP + 1) + threadIdx.x] = s_tot[threadIdx.x];
      if (s_tot[threadIdx.x]) atomicAdd(&D->xcnt[((size_t)p * D->L + l) * nc + threadIdx.x], s_tot[threadIdx.x]);
    }
    return;
  }
  const int istart = max(block_scan_max(start ? k : -1, s_mx), s_carry[1]);
  const int idx = block_count_class(start, cls, nc, s_w, s_tot);  // inclusive count of my class's starts
  if (!valid) return;
  const int item = D->xoff[cls][p][l] + s_carry[2 + cls] + idx - 1;
  char* blk = D->xblk + (size_t)item * D->XB;
  const int e = k - istart;
  if (!PLAN_BC(item >= 0 && item < D->nx_send && e >= 0 && e < R, 20)) return;
  XEnt E;
  E.row = (uint32_t)(o & 0xffffffu);
  E.l = (uint8_t)((o >> 24) & 0xffu);
  E.kq = (uint8_t)((o >> 32) & 0xffu);
  E.mask = (uint8_t)(((o >> 40) & 0xffu) | (a.wraps ? 1u << p : 0u));
  E.pad = 0;
  reinterpret_cast<XEnt*>(blk + 128)[e] = E;
  // the item's last entry writes its record
  const int ncls = (int)s_cls[threadIdx.x + 1];
  const bool last = k + 1 == n || ncls != cls || (k + 1 - runstart) % R == 0;
  if (last) {
    XRec r;
    memset(&r, 0, sizeof r);
    r.kind = kItemXSend;
    r.pulse = (uint8_t)p;
    r.lrank = (uint16_t)l;
    r.n_units = (uint32_t)(e + 1) * D->W;
    r.begin = (uint32_t)istart;
    r.cls = (uint32_t)cls;
    r.dst_x = a.dst_x;    // a rank of this group, or a bulk pulse (the host set exactly one of the two)
    r.dst_ll = a.dst_ll;
    r.bulk = a.bulk;
    r.bulk_total = a.bulk ? (uint32_t)n : 0u;
    for (int q = 0; q < kMaxP; ++q) {
      r.shiftL[q] = D->shiftL[q];
      r.pdim[q] = D->pdim[q];
    }
    r.epoch = D->epoch;
    *reinterpret_cast<XRec*>(blk) = r;
  }
}

// ------------------------------------------------------------------ f trees
__global__ void k_plan_child(const PlanDev* __restrict__ D) {
  plan_pdl();
  const int l = blockIdx.y / D->P, q = blockIdx.y % D->P;
  const int n = D->lq[l][q].send_size;
  const int32_t* m = D->maps[l] + (size_t)q * D->map_stride;
  int32_t* c = D->child + (size_t)l * D->cap * D->P;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    if (PLAN_BC(m[i] >= 0 && m[i] < D->n_total[l], 21)) c[(size_t)m[i] * D->P + q] = i;
}

// Depth-first node list of the tree under row t of local rank l, children in
// descending pulse order (the oracle's accumulation order, R15) — the host's emit_tree.
// Returns the node count (<= 2^P <= kFastNodes); lowest = lowest pulse of its LL nodes.
__device__ int plan_tree(const PlanDev* __restrict__ D, int l, int t, TNode* v, int& lowest) {
  struct Fr {
    int l, t, me, q, depth;
  } st[kMaxP + 1];
  const int P = D->P;
  int n = 0, top = 0;
  v[n++] = TNode{(uint32_t)t | ((uint32_t)l << 24), 0, 0xff, 0, 0xff};
  st[top++] = Fr{l, t, 0, P - 1, 0};
  lowest = P;
  while (top > 0) {
    Fr& f = st[top - 1];
    if (f.q < 0) {
      --top;
      continue;
    }
    const int q = f.q--;
    const int i = D->child[((size_t)f.l * D->cap + f.t) * P + q];
    if (i < 0) continue;
    v[f.me].flags |= 1;  // has children: its folded value is stored
    const PlanLQ& a = D->lq[f.l][q];
    const int fl = f.l, fme = f.me, fd = f.depth;
    if (a.rcv_l >= 0) {
      const int me = n;
      v[n++] = TNode{(uint32_t)(a.remote_off + i) | ((uint32_t)a.rcv_l << 24), 0, (uint8_t)fme,
                     (uint8_t)((fd + 1) << 1), a.efs};
      st[top++] = Fr{a.rcv_l, a.remote_off + i, me, P - 1, fd + 1};
    } else {
      v[n++] = TNode{(uint32_t)i | ((uint32_t)fl << 24), (uint8_t)(0x80u | q), (uint8_t)fme,
                     (uint8_t)((fd + 1) << 1), a.efs};
      lowest = min(lowest, q);
    }
  }
  return n;
}

// Is row t of local rank l a root?  Home rows with images; halo rows whose x-sender is
// in another group (they push their value back there; push = that LL unit).
__device__ __forceinline__ bool plan_is_root(const PlanDev* __restrict__ D, int l, int t, uint64_t** push) {
  const int P = D->P;
  *push = nullptr;
  if (t < D->n_home[l]) {
    const int32_t* c = D->child + ((size_t)l * D->cap + t) * P;
    for (int q = 0; q < P; ++q)
      if (c[q] >= 0) return true;
    return false;
  }
  for (int q = 0; q < P; ++q) {
    const PlanLQ& a = D->lq[l][q];
    if (t >= a.atom_offset && t < a.atom_offset + a.recv_size) {
      if (a.snd_l >= 0) return false;
      *push = a.push + (size_t)(t - a.atom_offset) * D->W;
      return true;
    }
  }
  return false;
}

// The shift-force targets of a tree as a mask over its rank's table (bucket_fs[l]).
__device__ __forceinline__ uint8_t plan_fs_mask(const PlanDev* __restrict__ D, int l, const TNode* v, int nn) {
  uint32_t m = 0;
  for (int k = 0; k < nn; ++k)
    if (v[k].fs != 0xff)
      for (int j = 0; j < D->n_buckets[l]; ++j)
        if (D->bucket_fs[l][j] == v[k].fs) m |= 1u << j;
  return (uint8_t)m;
}

// One thread per row, kPB rows per CTA (blockIdx.x), blockIdx.y = local rank: is the row
// a root, its tree's class (rcls, 0xff = not a root), and the CTA's roots per class.
__global__ void __launch_bounds__(kPB) k_plan_roots(const PlanDev* __restrict__ D) {
  plan_pdl();
  const int l = blockIdx.y, nc = D->P + 1;
  const int t = blockIdx.x * kPB + threadIdx.x;
  __shared__ int s_w[kMaxP + 1][kPB / 32];
  __shared__ int s_tot[kMaxP + 1];
  uint8_t cls = 0xff, mask = 0;
  if (t < D->n_total[l]) {
    uint64_t* push;
    if (plan_is_root(D, l, t, &push)) {
      TNode v[kFastNodes];
      int lowest;
      const int nn = plan_tree(D, l, t, v, lowest);
      cls = (uint8_t)(D->P - lowest);
      mask = plan_fs_mask(D, l, v, nn);
    }
    D->rcls[(size_t)l * D->cap + t] = cls;
    D->rmask[(size_t)l * D->cap + t] = mask;
  }
  (void)block_count_class(cls != 0xff, cls != 0xff ? cls : 0, nc, s_w, s_tot);
  if (threadIdx.x < nc) D->bcnt[((size_t)l * D->nblk + blockIdx.x) * nc + threadIdx.x] = s_tot[threadIdx.x];
}

// One CTA per local rank, one warp per class: exclusive prefix of the per-CTA root
// counts (boff) and the totals (rcnt), 32 blocks per step (shuffle scan).
__global__ void k_plan_rank(const PlanDev* __restrict__ D) {
  plan_pdl();
  const int l = blockIdx.x, nc = D->P + 1, c = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (c >= nc) return;
  const int nb = D->nblk;
  int acc = 0;
  for (int b0 = 0; b0 < nb; b0 += 32) {
    const int b = b0 + lane;
    const size_t i = ((size_t)l * nb + b) * nc + c;
    const int v = b < nb ? D->bcnt[i] : 0;
    int incl = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += y;
    }
    if (b < nb) D->boff[i] = acc + incl - v;
    acc += __shfl_sync(0xffffffffu, incl, 31);
  }
  if (lane == 0) D->rcnt[l * nc + c] = acc;
}

// Every root writes its 32-B record and node indices into slot rank % RT of item
// foff[class][l] + rank / RT; slot 0 also writes the item's record.
// kMask: pass 1, the item's bucket mask = OR of its trees' masks (imask, zeroed before);
// otherwise pass 2: records with the item-local bucket numbers (the item's buckets are the
// set bits of its mask, in table order: what the host builder gives, R13).
template <bool kMask>
__global__ void __launch_bounds__(kPB) k_plan_f(const PlanDev* __restrict__ D) {
  plan_pdl();
  const int l = blockIdx.y, nc = D->P + 1;
  const int n = D->n_total[l], RT = D->RT;
  const int t = blockIdx.x * kPB + threadIdx.x;
  __shared__ int s_w[kMaxP + 1][kPB / 32];
  __shared__ int s_tot[kMaxP + 1];
  const uint8_t cls = t < n ? D->rcls[(size_t)l * D->cap + t] : (uint8_t)0xff;
  const int idx = block_count_class(cls != 0xff, cls != 0xff ? cls : 0, nc, s_w, s_tot);  // rank in the CTA
  if (kMask) {
    if (cls != 0xff) {
      const int rank = D->boff[((size_t)l * D->nblk + blockIdx.x) * nc + cls] + idx - 1;
      const uint32_t m = D->rmask[(size_t)l * D->cap + t];
      if (!PLAN_BC(D->foff[cls][l] + rank / RT < D->nf, 22)) return;
      if (m) atomicOr(&D->imask[D->foff[cls][l] + rank / RT], m);
    }
    return;
  }
  if (cls != 0xff) {
    uint64_t* push;
    (void)plan_is_root(D, l, t, &push);
    TNode v[kFastNodes];
    int lowest;
    const int nn = plan_tree(D, l, t, v, lowest);
    const int rank = D->boff[((size_t)l * D->nblk + blockIdx.x) * nc + cls] + idx - 1;
    const int item = D->foff[cls][l] + rank / RT, slot = rank % RT;
    if (!PLAN_BC(item >= 0 && item < D->nf && nn >= 1 && nn <= kFastNodes, 23)) return;
    char* blk = D->fblk + (size_t)item * D->FB;
    const uint32_t imask = D->imask[item];
    TRoot R;
    memset(&R, 0, sizeof R);
    R.push = push;
    R.par = 0xffffffffu;
    R.bucket = 0xffffffffu;
    R.nn = (uint8_t)nn;
    {  // postorder of the non-root nodes: close every open node at least as deep as the next
      int stk[kFastNodes], top = 0, e = 0;
      for (int k = 0; k <= nn; ++k) {
        const int dk = k < nn ? (v[k].flags >> 1) : 0;
        while (top > 0 && (v[stk[top - 1]].flags >> 1) >= dk) {
          const int c = stk[--top];
          if (c != 0) R.post |= (uint32_t)c << (4 * e++);
        }
        if (k < nn) stk[top++] = k;
      }
    }
    uint32_t* il = reinterpret_cast<uint32_t*>(blk + 128 + 32 * (size_t)RT) + 8 * slot;
    for (int k = 0; k < nn; ++k) {
      const TNode& x = v[k];
      const uint32_t sh = 4 * (uint32_t)k;
      uint32_t b = kFsNone;
      if (x.fs != 0xff)
        for (int j = 0; j < D->n_buckets[l]; ++j)
          if (D->bucket_fs[l][j] == x.fs) b = (uint32_t)__popc(imask & ((1u << j) - 1u));
      R.par = (R.par & ~(15u << sh)) | ((uint32_t)(x.parent == 0xff ? 15 : x.parent) << sh);
      R.bucket = (R.bucket & ~(15u << sh)) | (b << sh);
      R.q |= (uint32_t)(x.kq & 7) << sh;
      if (x.kq & 0x80u) R.llmask |= (uint8_t)(1u << k);
      if (x.flags & 1u) R.stmask |= (uint8_t)(1u << k);
      il[k] = x.il;
    }
    reinterpret_cast<TRoot*>(blk + 128)[slot] = R;
    if (slot == 0) {
      GRec g;
      memset(&g, 0, sizeof g);
      g.kind = kItemTree;
      g.level = cls;
      g.lrank = (uint16_t)l;
      g.n_roots = (uint32_t)min(RT, D->fcnt[cls][l] - rank);
      g.n_units = g.n_roots * D->W;
      g.n_buckets = (uint8_t)__popc(imask);
      for (int j = 0, k = 0; j < D->n_buckets[l]; ++j)
        if (imask >> j & 1u) g.bucket_fs[k++] = D->bucket_fs[l][j];
      g.epoch = D->epoch;
      *reinterpret_cast<GRec*>(blk) = g;
    }
  }
}

// ------------------------------------------------------------------ launchers
static unsigned plan_gx(int rows) { return (unsigned)std::max(1, std::min(64, (rows + 255) / 256)); }

cudaError_t launch_plan_count(const PlanDev* D, int L, int P, int max_rows, int max_send, cudaStream_t st) {
  const unsigned gx = plan_gx(max_rows);
  cudaError_t e = plan_launch(k_plan_org_home, dim3(gx, L), 256, st, D);
  for (int q = 0; q < P && e == cudaSuccess; ++q) e = plan_launch(k_plan_org_pulse, dim3(gx, L), 256, st, D, q);
  const unsigned xnch = (unsigned)((max_send + kPB - 1) / kPB);
  if (e == cudaSuccess) e = plan_launch(k_plan_x<0>, dim3(std::max(1u, xnch), P * L), kPB, st, D);
  if (e == cudaSuccess) e = plan_launch(k_plan_x<1>, dim3(std::max(1u, xnch), P * L), kPB, st, D);
  if (e == cudaSuccess) e = plan_launch(k_plan_child, dim3(gx, L * P), 256, st, D);
  const unsigned nblk = (unsigned)((max_rows + kPB - 1) / kPB);
  if (e == cudaSuccess) e = plan_launch(k_plan_roots, dim3(nblk, L), kPB, st, D);
  if (e == cudaSuccess) e = plan_launch(k_plan_rank, dim3(L), 32 * (P + 1), st, D);
  return e;
}

cudaError_t launch_plan_write(const PlanDev* D, int L, int P, int max_rows, int max_send, cudaStream_t st) {
  const unsigned xnch = (unsigned)((max_send + kPB - 1) / kPB);
  cudaError_t e = plan_launch(k_plan_x<2>, dim3(std::max(1u, xnch), P * L), kPB, st, D);
  const unsigned nblk = (unsigned)((max_rows + kPB - 1) / kPB);
  if (e == cudaSuccess) e = plan_launch(k_plan_f<true>, dim3(nblk, L), kPB, st, D);
  if (e == cudaSuccess) e = plan_launch(k_plan_f<false>, dim3(nblk, L), kPB, st, D);
  return e;
}

int plan_rows_per_cta() { return kPB; }

}  // namespace halo
