// runtime.cu — host side of libhalo: config validation, pulse plan, IPC peer
// table, set_maps driver, work-item tables, C ABI entry points.
//
// Citations: P:<n> = PAPER.md line, R<n> = DESIGN.md reading.
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstddef>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <string>
#include <thread>
#include <atomic>
#include <vector>

#include "halo_internal.h"

namespace halo {
cudaError_t launch_exchange_x(const ExParams& p, int layout, int grid, cudaStream_t st);
cudaError_t launch_exchange_f(const ExParams& p, int layout, int grid, cudaStream_t st);
cudaError_t max_coresident(int layout, int* x_blocks, int* f_blocks);
cudaError_t launch_migrate(const MigParams& M, MigCtrl* C, int max_rows, int phase, cudaStream_t st);
cudaError_t launch_pme(const PmeParams& M, int which, int ctas_per_rank, cudaStream_t st);
cudaError_t launch_select(const SelParams& s, int n_local, cudaStream_t st);
cudaError_t launch_handshake(const HsParams& h, cudaStream_t st);
cudaError_t launch_depmask(const RankDev* ranks, Ctrl* ctrl, int p, int map_stride, int n_local, cudaStream_t st);
cudaError_t launch_status(const StatusParams& s, cudaStream_t st);
cudaError_t launch_pack_x(int layout, const int32_t* map, int n, const float* x, float* out, int has_shift,
                          const float* shift, cudaStream_t st);
cudaError_t launch_unpack_f(int layout, const int32_t* map, int n, const float* buf, float* f, int accumulate,
                            double* fs_dim, cudaStream_t st);
cudaError_t launch_pingpong(uint64_t* own, uint64_t* peer, int iters, uint64_t base, int initiator, int relaxed,
                            uint64_t* rtt_ns, uint64_t timeout_ns, int* err_host, cudaStream_t st);
cudaError_t launch_exchange_ll(const ExParams& p, int mode, int layout, int grid, bool wide,
                               const cudaAccessPolicyWindow* win, cudaStream_t st, bool chk);
cudaError_t max_coresident_ll(int layout, bool wide, int* blocks, int local_sel);
int ll_ring(int mode, bool wide);
void ll_set_ring_f(int r);
void ll_set_x_variant(int v);
cudaError_t launch_empty(int grid, cudaStream_t st, uint64_t* remote, uint32_t nwords);
cudaError_t launch_ce_pack(int layout, const CeEnt* ents, int n_local, int max_rows, cudaStream_t st);
cudaError_t launch_ce_unpack(int layout, const CeEnt* ents, int n_local, int max_rows, double* fshift, int accumulate,
                             cudaStream_t st);
cudaError_t launch_ce_sync(const CeSyncParams& s, cudaStream_t st);
cudaError_t launch_bw_copy(const void* src, void* dst, size_t bytes, int grid, cudaStream_t st);
cudaError_t launch_seg_copy(const SegCopy* segs, int nseg, size_t max_words, cudaStream_t st);
cudaError_t launch_ns_x(const NsXParams& X, int layout, int max_rows, cudaStream_t st);
cudaError_t launch_zero_ll(uint64_t* const* base_dev, size_t units, int n, cudaStream_t st);
cudaError_t launch_ns_wait(const NsWaitParams& W, cudaStream_t st);
cudaError_t launch_plan_count(const PlanDev* D, int L, int P, int max_rows, int max_send, cudaStream_t st);
cudaError_t launch_plan_write(const PlanDev* D, int L, int P, int max_rows, int max_send, cudaStream_t st);
int plan_rows_per_cta();
uint32_t ll_xblk_bytes(int rows);
uint32_t ll_fblk_bytes(int rows);
cudaError_t launch_assign_home(const float* x, int n, int stride, const AssignParams& A, int32_t* rank, int* counts,
                               int* seg, int32_t* ids, int* err, cudaStream_t st);
// floors (kernels_floor.cu)
cudaError_t launch_payload_pingpong(const void* src_own, void* dst_peer, const void* src_peer_side, void* dst_own,
                                    uint64_t* cnt_own, uint64_t* cnt_peer, size_t bytes, int G, int iters,
                                    uint64_t cnt_base, uint64_t cnt_base_peer, int mode, uint64_t* rtt_ns,
                                    uint64_t timeout_ns, int* err_host, cudaStream_t st);
cudaError_t launch_bw_multi(const void* src, void* const* dst, int n, size_t bytes, int ctas_per_peer,
                            cudaStream_t st);
// NCCL send/recv baseline (nccl_baseline.cu)
bool nccl_available(std::string* why);
int nccl_version();
bool nccl_unique_id(void* out, std::string* why);
void* nccl_comm_init(const void* id, int nranks, int rank, std::string* why);
void nccl_comm_destroy(void* comm);
std::string nccl_sendrecv(void* comm, const float* sbuf, size_t sn, int speer, float* rbuf, size_t rn, int rpeer,
                          cudaStream_t st);
}  // namespace halo

using namespace halo;

namespace {

constexpr uint32_t kBlobMagic = 0x48414c4fu;  // "HALO"

struct BlobHdr {
  uint32_t magic;
  uint32_t version;
  int32_t proc;
  int32_t n_local;
  int32_t first_rank;
  int32_t device;
  int32_t layout;
  int32_t capacity;
  uint64_t pid;
};
struct BlobEntry {
  cudaIpcMemHandle_t hx;
  uint64_t offx;
  cudaIpcMemHandle_t hs;
  uint64_t offs;
  cudaIpcMemHandle_t hf;  // f: read by peers only with HALO_F_TMA_GET (receiver-driven get)
  uint64_t offf;
};

// cuMemGetAddressRange through the runtime's driver entry point (no -lcuda link,
// so the library loads on hosts without a driver).
typedef int (*PFN_memGetAddressRange)(unsigned long long* base, size_t* size, unsigned long long dptr);

PFN_memGetAddressRange get_addr_range_fn() {
  static PFN_memGetAddressRange fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuMemGetAddressRange", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = (PFN_memGetAddressRange)p;
  }
  return fn;
}

}  // namespace

struct halo_ctx {
  halo_config cfg{};
  int nranks = 0, n_local = 0, first_rank = 0, P = 0, W = 3;
  int pdim[kMaxP] = {0}, pk[kMaxP] = {0};
  size_t map_stride = 0, fbuf_stride = 0, ll_stride = 0, fsp_slots = 0, scratch_bytes = 0;
  size_t mig_off = 0;                // halo_migrate staging: [out | in] at this scratch offset
  size_t mig_stage = 0;              // bytes of one staging area (x | v | gid rows, capacity each)
  size_t probe_off = 0, probe_max = 0;  // halo_probe_reserve: [counter 256 B | send | recv] (probe_max each)
  uint64_t probe_cnt[kMaxLocal] = {0};  // value of each local rank's probe counter (all increments it has seen)
  int pme_rank = -1;                 // halo_pme_reserve: DD rank whose scratch holds pme_x | pme_f
  size_t pme_off = 0;                // their offset in that scratch (same layout on every rank)
  bool pme_ready = false;            // halo_pme_setup done for the current maps
  std::vector<int> pme_row_off;      // first pme row of every DD rank
  int pme_total = 0;
  bool ll = true;                   // LL protocol (default) vs the paper's flag protocol
  bool ce = false;                  // copy-engine path (HALO_F_CE_PATH; set_maps uses the paper kernels)
  std::string last_error;

  // registered local buffers
  std::vector<float*> x, f;
  std::vector<char*> scratch;
  // every rank's peer view (local pointers for this process's ranks)
  std::vector<float*> peer_x;
  std::vector<float*> peer_f;
  std::vector<char*> peer_scratch;
  std::vector<void*> opened;  // IPC bases to close
  bool peers_ready = false;

  // library-owned device memory
  Ctrl* ctrl = nullptr;
  char* plan = nullptr;
  size_t plan_bytes = 0;
  std::vector<char*> retired;       // plans replaced while a captured graph may reference them
  // GPU-built LL plan (kernels_plan.cu): block areas written by the kernels
  size_t gpu_xblk_bytes = 0, gpu_fblk_bytes = 0;
  int gpu_n_items_x = 0, gpu_n_items_f = 0;
  bool gpu_plan = true;             // HALO_PLAN_HOST=1: the host builder (reference; also P > 3)
  PlanDev* d_pl = nullptr;          // descriptor + scratch of the GPU plan build
  PlanDev* h_pl = nullptr;          // (pinned host copy)
  char* d_pl_scratch = nullptr;
  size_t pl_scratch_bytes = 0;
  int32_t* h_pl_cnt = nullptr;      // pinned: xcnt | rcnt read back after the counting pass
  XRec* h_recv = nullptr;           // pinned: the receive items' records
  size_t h_recv_cap = 0;
  RankDev* d_ranks = nullptr;
  PulseDev* d_pulses = nullptr;
  Item* d_items_x = nullptr;
  Item* d_items_f = nullptr;
  int n_items_x = 0, n_items_f = 0;
  int n_tail_f = 0;                 // LL: shift-force combine items at the end of the f list
  double* d_fshift_tmp = nullptr;  // halo_step_host
  char* h_small = nullptr;          // pinned 64 KiB: set_maps result read-backs and small uploads
  int32_t* d_selcnt = nullptr;      // set_maps select: rows per 1024-row chunk
  // halo_step_host_packed: packed staging in / out, segment tables (x unpack | f unpack | pack),
  // rebuilt once per NS epoch; side streams for the f upload and the halo-x download
  char* d_pk_in = nullptr;
  char* d_pk_out = nullptr;
  size_t pk_in_cap = 0, pk_out_cap = 0;
  SegCopy* d_segs = nullptr;
  uint32_t pk_epoch = 0;
  char* pk_out_dev = nullptr;       // the output block's device address the tables were built for
  size_t pk_max_words[3] = {0, 0, 0};
  cudaStream_t pk_h2d = nullptr, pk_d2h = nullptr;
  cudaEvent_t pk_ev[4] = {nullptr, nullptr, nullptr, nullptr};
  cudaStream_t pk_cap = nullptr;    // capture stream of the packed-step graph
  cudaGraphExec_t pk_exec = nullptr;
  uint32_t pk_g_epoch = 0;
  const void* pk_g_in = nullptr;
  const void* pk_g_out = nullptr;
  char* d_small = nullptr;          // set_maps argument staging
  MigRank* d_mig = nullptr;         // halo_migrate: per local rank tables
  MigCtrl* d_migctrl = nullptr;
  double* d_planes = nullptr;
  uint64_t* d_rtt = nullptr;
  char* d_assign = nullptr;         // halo_assign_home: rank per atom | counts | error word
  size_t assign_bytes = 0;
  int* err_host = nullptr;          // host-mapped error word
  int* err_dev = nullptr;
  std::vector<LocalBase> h_lbase;       // LL: per local rank base pointers (copied to shared memory by the kernels)
  LocalBase* d_lbase = nullptr;
  std::vector<char> h_xblk, h_fblk;     // item blocks [record | map slice] / [record | task records]
  char* h_pin = nullptr;                // pinned image of the plan (one DMA per upload)
  size_t h_pin_bytes = 0;
  char* d_xblk = nullptr;
  char* d_fblk = nullptr;
  std::vector<std::vector<std::vector<int32_t>>> h_maps;  // host copy of every local rank's maps [l][p]

  // copy-engine path (HALO_F_CE_PATH): per pulse, per local rank
  struct CeCopy {
    void* dst;
    const void* src;
    size_t bytes;
  };
  std::vector<CeEnt> h_ce_pack, h_ce_unpack;   // [P][n_local]
  std::vector<CeCopy> ce_copy_x, ce_copy_f;    // [P][n_local]
  // HALO_CE_PROFILE=1: CUDA events between the copy-engine path's operations (study of
  // where its time goes); the mean per operation is printed at halo_destroy
  struct CeProf {
    bool on = getenv("HALO_CE_PROFILE") != nullptr;
    std::vector<std::pair<cudaEvent_t, cudaEvent_t>> pend;  // (start, end) per op, in order
    std::vector<std::string> names, agg_names;
    std::vector<double> sum;
    std::vector<int> cnt;
  } ce_prof;
  std::vector<int> ce_pack_rows, ce_unpack_rows;  // [P]: largest entry needing the kernel (0 = no launch)
  CeEnt* d_ce = nullptr;                       // pack table then unpack table
  float* d_stage = nullptr;                    // contiguous send rows of every (pulse, local rank) that packs
  size_t ce_bytes = 0, stage_bytes = 0;


  // host plan
  std::vector<RankDev> h_ranks;
  std::vector<PulseDev> h_pulses;
  std::vector<Item> h_items_x, h_items_f;
  std::vector<int> n_home, n_total;
  std::vector<int> send_size, recv_size, atom_offset, remote_off, n_indep;  // [n_local*P]
  std::vector<unsigned> dep;
  bool maps_ready = false;
  bool x_done = false;
  uint32_t epoch = 0;
  uint64_t ping_base = 0;
  cudaAccessPolicyWindow l2win{};    // HALO_F_L2_PERSIST: the static plan (item blocks) persists in L2
  int max_x = 0, max_f = 0, max_xf = 0;        // co-resident CTAs of the exchange kernels (LL: narrow variants)
  int max_x128 = 0;                              // ... of the x kernel with 128-row items (two units per thread)
  // ... of the hop-group-local variants (used when all_local: their register budget differs)
  int max_x_loc = 0, max_f_loc = 0, max_xf_loc = 0, max_x128_loc = 0;
  bool all_local = false;           // LL plan: every pulse of every local rank stays in this hop group
  int max_x_w = 0, max_f_w = 0, max_xf_w = 0;  // LL: batched variants for large work items
  int grid_cap = 0;                 // HALO_CTAS_PER_SM x SMs (0 = occupancy limit only)
  int x_cap = 0;                    // HALO_X_CTAS_PER_SM x SMs: the x kernel only (leaves SM room for
                                    // the f kernel's CTAs to become resident early under PDL)
  bool wide() const { return ll && item_rows >= 256; }
  bool loc() const { return ll && all_local && max_f_loc > 0; }
  int cap_x() const {
    int c = wide() ? max_x_w : item_rows > 64 ? (loc() ? max_x128_loc : max_x128) : (loc() ? max_x_loc : max_x);
    if (grid_cap) c = std::min(c, grid_cap);
    return x_cap ? std::min(c, x_cap) : c;
  }
  int cap_f() const {
    const int c = wide() ? max_f_w : loc() ? max_f_loc : max_f;
    return grid_cap ? std::min(c, grid_cap) : c;
  }
  int cap_xf() const {
    const int c = wide() ? max_xf_w : loc() ? max_xf_loc : max_xf;
    return grid_cap ? std::min(c, grid_cap) : c;
  }
  int last_grid[2] = {0, 0};
  int item_rows = 64;
  int tree_rows = 64;               // LL: roots per small-tree f item (chosen per NS epoch, build_ll_f)
  int tree_rows_max = kMaxTreeRows; // ... at most (more roots than fit the co-resident grid at kTreeRowsOcc:
                                    // the bandwidth regime; two passes per thread)
  bool item_rows_fixed = false;     // HALO_ITEM_ROWS given: no adaptive choice
  uint32_t poll_ns = 0;
  uint32_t debug = 0;
  // LL sequence numbers mirrored on the host: launches take them by value until the
  // ctx is first used under stream capture (a replayed graph must read the device
  // counter, R17); every LL launch advances the device counter in any case
  uint64_t seq_host_x = 0, seq_host_f = 0;
  bool captured = false;
  bool auto_tr = false;             // HALO_F_AUTO_TRANSPORT: LL or copy engine chosen at every set_maps
  size_t auto_ce_bytes = (size_t)4 << 20;  // ... copy engine when some pulse sends >= this (HALO_AUTO_CE_BYTES)
  bool collapse = true;             // LL: the ranks of this process form one hop group (HALO_COLLAPSE=0 /
                                    // HALO_DIRECT_X=0: every rank its own group, the staged schedule)
  bool prefetch = false;            // LL x launch: L2 prefetch of the f item blocks and home x rows (HALO_PREFETCH=1;
                                    // measured slower at C3: 17.3 -> 18.1 us/step, the prefetches delay the x blocks)
  bool packed_blocking = false;      // halo_step_host_packed waits with cudaStreamSynchronize (HALO_PACKED_BLOCKING)
  int bulk_rows = kBulkRowsDefault;  // bulk x pulses from this many rows (HALO_BULK_ROWS; 0: never, the default), §6.9
  int recv_mult = 1;                // x receive items are recv_mult x item_rows rows (HALO_RECV_MULT; 2, 4 measured slower)
  // NCCL send/recv baseline (halo_nccl_*, HALO_F_NCCL_BASELINE): communicator + packed send rows
  void* nccl_comm = nullptr;
  float* d_nccl_send = nullptr;
  size_t nccl_send_bytes = 0;

  int cell(int r, int d) const {
    const int* g = cfg.grid;
    if (d == 2) return r % g[2];
    if (d == 1) return (r / g[2]) % g[1];
    return r / (g[1] * g[2]);
  }
  int rank_of(int cx, int cy, int cz) const { return (cx * cfg.grid[1] + cy) * cfg.grid[2] + cz; }
  bool is_local(int r) const { return r >= first_rank && r < first_rank + n_local; }
  int neighbour(int r, int d, int delta) const {
    int c[3] = {cell(r, 0), cell(r, 1), cell(r, 2)};
    c[d] = ((c[d] + delta) % cfg.grid[d] + cfg.grid[d]) % cfg.grid[d];
    return rank_of(c[0], c[1], c[2]);
  }
  // b_d[k] = float64(L_d) * k / grid[d]  (R3: multiply then divide, IEEE double)
  double plane(int d, int k) const { return (double)cfg.box[d] * (double)k / (double)cfg.grid[d]; }
  ScratchHdr* hdr_of(int r) const { return reinterpret_cast<ScratchHdr*>(peer_scratch[r]); }
  int32_t* maps_of_local(int l) const { return reinterpret_cast<int32_t*>(scratch[l] + kHdrBytes); }
  float* fbuf_of(int r) const {
    return reinterpret_cast<float*>(peer_scratch[r] + kHdrBytes + (size_t)P * map_stride * sizeof(int32_t));
  }
  uint64_t* xll_of(int r) const {
    return reinterpret_cast<uint64_t*>(peer_scratch[r] + kHdrBytes + (size_t)P * map_stride * sizeof(int32_t) +
                                       (size_t)P * fbuf_stride * sizeof(float));
  }
  uint64_t* fll_of(int r) const { return xll_of(r) + (size_t)P * ll_stride; }
  uint64_t* fsp_of(int r) const { return fll_of(r) + (size_t)P * ll_stride; }  // 6 units per slot
};

// --------------------------------------------------------------------- helpers
static halo_status fail(halo_ctx* c, halo_status s, const std::string& msg) {
  if (c) c->last_error = msg;
  return s;
}
static halo_status cuda_fail(halo_ctx* c, cudaError_t e, const char* where) {
  std::string m = std::string(where) + ": " + cudaGetErrorString(e);
  (void)cudaGetLastError();
  return fail(c, HALO_ERR_CUDA, m);
}
#define CK(call)                                                   \
  do {                                                             \
    cudaError_t e__ = (call);                                      \
    if (e__ != cudaSuccess) return cuda_fail(ctx, e__, #call);     \
  } while (0)

static size_t align_up(size_t v, size_t a) { return (v + a - 1) / a * a; }

// Scratch layout of one DD rank (halo_internal.h): header | maps | force
// buffers (paper protocol) | coordinate LL buffers | force LL buffers.
struct ScratchLayout {
  size_t map_stride, fbuf_stride, ll_stride, fsp_slots, mig_off, mig_stage, total;
};
static ScratchLayout scratch_layout(int P, int capacity, int layout) {
  ScratchLayout L;
  L.map_stride = align_up((size_t)capacity, 64);                // int32 per pulse slot
  L.fbuf_stride = align_up((size_t)capacity * layout, 64);      // fp32 per pulse slot
  L.ll_stride = align_up((size_t)capacity * layout, 32);        // u64 units per pulse slot
  L.fsp_slots = align_up(((size_t)capacity + kMinItemRows - 1) / kMinItemRows, 8);  // shift-force slots per pulse
  L.total = kHdrBytes + (size_t)P * L.map_stride * sizeof(int32_t) + (size_t)P * L.fbuf_stride * sizeof(float) +
            2 * (size_t)P * L.ll_stride * sizeof(uint64_t) + (size_t)P * L.fsp_slots * 6 * sizeof(uint64_t);
  // halo_migrate staging-out and staging-in: x | v | gid rows, capacity each
  L.mig_off = align_up(L.total, 256);
  // (at least 4 MiB each: with the LL areas before them they also give halo_floor_bandwidth
  // a peer-mapped area of >= 8 MiB at any capacity)
  L.mig_stage = std::max(align_up((size_t)capacity * (2 * layout + 1) * sizeof(float), 256), (size_t)4 << 20);
  L.total = L.mig_off + 2 * L.mig_stage;
  return L;
}

static halo_status check_err_word(halo_ctx* ctx) {
  if (ctx->err_host && *(volatile int*)ctx->err_host != 0) {
    char buf[128];
    int code = *(volatile int*)ctx->err_host;
    if ((code >> 16) == kErrKindBounds) {
      snprintf(buf, sizeof buf, "bounds check failed in the checked build (local rank %d, check %d)",
               (code >> 8) & 0xff, code & 0xff);
      return fail(ctx, HALO_ERR_STATE, buf);
    }
    if ((code >> 16) == kErrKindStalePlan)
      return fail(ctx, HALO_ERR_STATE, "a CUDA graph captured before the last halo_set_maps / halo_migrate was "
                                       "replayed (its plan is gone): re-capture after every NS step");
    snprintf(buf, sizeof buf, "device wait timed out (kind %d, local rank %d, pulse %d)", code >> 16,
             (code >> 8) & 0xff, code & 0xff);
    return fail(ctx, HALO_ERR_TIMEOUT, buf);
  }
  return HALO_OK;
}

static halo_status validate(const halo_config* c, std::string& why) {
  if (!c) { why = "cfg is NULL"; return HALO_ERR_ARG; }
  if (c->layout != 3 && c->layout != 4) { why = "layout must be 3 or 4"; return HALO_ERR_ARG; }
  if (c->capacity <= 0 || c->capacity >= (1 << 24)) { why = "capacity must be in (0, 2^24)"; return HALO_ERR_ARG; }
  if (c->nprocs < 1 || c->proc < 0 || c->proc >= c->nprocs) { why = "bad nprocs/proc"; return HALO_ERR_ARG; }
  long long nr = 1;
  int P = 0;
  for (int d = 0; d < 3; ++d) {
    if (c->grid[d] < 1) { why = "grid[d] must be >= 1"; return HALO_ERR_GEOMETRY; }
    nr *= c->grid[d];
    if ((c->grid[d] > 1) != (c->pulses[d] >= 1)) { why = "pulses[d] >= 1 iff grid[d] > 1"; return HALO_ERR_GEOMETRY; }
    if (c->pulses[d] > std::max(c->grid[d] - 1, 0)) { why = "pulses[d] must be <= grid[d]-1"; return HALO_ERR_GEOMETRY; }
    if (c->pulses[d] > 2) { why = "at most two pulses per dimension (P:143)"; return HALO_ERR_UNSUPPORTED; }
    if (!(c->box[d] > 0.0f) || !std::isfinite(c->box[d])) { why = "box lengths must be > 0"; return HALO_ERR_GEOMETRY; }
    if (c->grid[d] > 1 && (double)c->pulses[d] * ((double)c->box[d] / c->grid[d]) < (double)c->cutoff) {
      why = "not enough pulses: pulses[d]*L_d/grid[d] < rc";
      return HALO_ERR_GEOMETRY;
    }
    P += c->grid[d] > 1 ? c->pulses[d] : 0;
  }
  double minL = std::min(std::min((double)c->box[0], (double)c->box[1]), (double)c->box[2]);
  if (!((double)c->cutoff > 0.0 && (double)c->cutoff < minL / 2.0)) { why = "need 0 < rc < min(L)/2"; return HALO_ERR_GEOMETRY; }
  if (nr > kMaxRanks) { why = "too many ranks for this build (HALO_MAX_RANKS)"; return HALO_ERR_UNSUPPORTED; }
  if (nr % c->nprocs != 0) { why = "nranks must be a multiple of nprocs"; return HALO_ERR_ARG; }
  if (nr / c->nprocs > kMaxLocal) { why = "too many ranks per process (HALO_MAX_LOCAL)"; return HALO_ERR_UNSUPPORTED; }
  if (P > kMaxP) { why = "too many pulses"; return HALO_ERR_UNSUPPORTED; }
  if ((c->flags & HALO_F_AUTO_TRANSPORT) &&
      (c->flags & (HALO_F_PAPER_FLAGS | HALO_F_CE_PATH | HALO_F_TMA_STORE | HALO_F_TMA_GET))) {
    why = "HALO_F_AUTO_TRANSPORT chooses between the LL protocol and the copy engine itself";
    return HALO_ERR_UNSUPPORTED;
  }
  if ((c->flags & (HALO_F_TMA_STORE | HALO_F_TMA_GET)) &&
      (!(c->flags & HALO_F_PAPER_FLAGS) || (c->flags & HALO_F_CE_PATH))) {
    why = "HALO_F_TMA_STORE / HALO_F_TMA_GET are variants of the paper protocol (HALO_F_PAPER_FLAGS, no HALO_F_CE_PATH)";
    return HALO_ERR_UNSUPPORTED;
  }
  return HALO_OK;
}

// ------------------------------------------------------------------- C ABI
extern "C" {

const char* halo_strerror(halo_status s) {
  switch (s) {
    case HALO_OK: return "ok";
    case HALO_ERR_ARG: return "invalid argument";
    case HALO_ERR_GEOMETRY: return "invalid geometry";
    case HALO_ERR_CAPACITY: return "capacity exceeded";
    case HALO_ERR_STATE: return "call out of order";
    case HALO_ERR_CUDA: return "CUDA error";
    case HALO_ERR_PEER: return "peer/IPC error";
    case HALO_ERR_TIMEOUT: return "device wait timed out";
    case HALO_ERR_UNSUPPORTED: return "unsupported";
  }
  return "unknown status";
}

const char* halo_last_error(const halo_ctx* ctx) { return ctx ? ctx->last_error.c_str() : ""; }

halo_status halo_init(const halo_config* cfg, halo_ctx** out) {
  if (!out) return HALO_ERR_ARG;
  *out = nullptr;
  std::string why;
  halo_status s = validate(cfg, why);
  if (s != HALO_OK) return s;
  halo_ctx* ctx = new halo_ctx();
  ctx->cfg = *cfg;
  if (ctx->cfg.timeout_s <= 0) ctx->cfg.timeout_s = 10.0;
  ctx->W = cfg->layout;
  ctx->nranks = cfg->grid[0] * cfg->grid[1] * cfg->grid[2];
  ctx->n_local = ctx->nranks / cfg->nprocs;
  ctx->first_rank = cfg->proc * ctx->n_local;
  const int order[3] = {2, 1, 0};  // z -> y -> x
  for (int i = 0; i < 3; ++i) {
    const int d = order[i];
    if (cfg->grid[d] > 1)
      for (int k = 0; k < cfg->pulses[d]; ++k) {
        ctx->pdim[ctx->P] = d;
        ctx->pk[ctx->P] = k;
        ctx->P++;
      }
  }
  {
    const ScratchLayout SL = scratch_layout(ctx->P, cfg->capacity, cfg->layout);
    ctx->map_stride = SL.map_stride;
    ctx->fbuf_stride = SL.fbuf_stride;
    ctx->ll_stride = SL.ll_stride;
    ctx->fsp_slots = SL.fsp_slots;
    ctx->mig_off = SL.mig_off;
    ctx->mig_stage = SL.mig_stage;
    ctx->scratch_bytes = SL.total;
  }
  ctx->ce = (cfg->flags & HALO_F_CE_PATH) != 0;
  ctx->ll = !(cfg->flags & HALO_F_PAPER_FLAGS) && !ctx->ce;
  ctx->auto_tr = (cfg->flags & HALO_F_AUTO_TRANSPORT) != 0;
  ctx->x.assign(ctx->n_local, nullptr);
  ctx->f.assign(ctx->n_local, nullptr);
  ctx->scratch.assign(ctx->n_local, nullptr);
  ctx->peer_x.assign(ctx->nranks, nullptr);
  ctx->peer_f.assign(ctx->nranks, nullptr);
  ctx->peer_scratch.assign(ctx->nranks, nullptr);
  if (const char* e = getenv("HALO_ITEM_ROWS")) {
    ctx->item_rows = std::min(kMaxItemRows, std::max(kMinItemRows, atoi(e)));
    ctx->item_rows_fixed = true;
  }
  if (const char* e = getenv("HALO_POLL_NS")) ctx->poll_ns = atoi(e) < 0 ? kPollTight : (uint32_t)atoi(e);
  if (const char* e = getenv("HALO_DIRECT_X")) ctx->collapse = atoi(e) != 0;
  if (const char* e = getenv("HALO_COLLAPSE")) ctx->collapse = atoi(e) != 0;
  if (const char* e = getenv("HALO_PACKED_BLOCKING")) ctx->packed_blocking = atoi(e) != 0;
  if (const char* e = getenv("HALO_BULK_ROWS")) ctx->bulk_rows = std::max(0, atoi(e));
  if (const char* e = getenv("HALO_RECV_MULT")) ctx->recv_mult = std::min(16, std::max(1, atoi(e)));
  if (const char* e = getenv("HALO_PREFETCH")) ctx->prefetch = atoi(e) != 0;
  if (const char* e = getenv("HALO_PLAN_HOST")) ctx->gpu_plan = atoi(e) == 0;
  if (const char* e = getenv("HALO_TIMEOUT_S")) ctx->cfg.timeout_s = std::max(0.001, atof(e));  // sanitizer runs
  ll_set_x_variant(getenv("HALO_X_VARIANT") ? atoi(getenv("HALO_X_VARIANT")) : 0);
  ll_set_ring_f(getenv("HALO_RING_F") ? atoi(getenv("HALO_RING_F")) : 0);
  if (const char* e = getenv("HALO_TREE_ROWS_MAX")) ctx->tree_rows_max = std::min(kMaxTreeRows, std::max(8, atoi(e)));
  if (const char* e = getenv("HALO_DEBUG")) ctx->debug = (uint32_t)std::max(0, atoi(e));

  cudaError_t e = cudaSetDevice(cfg->device);
  if (e == cudaSuccess) e = cudaMalloc(&ctx->ctrl, sizeof(Ctrl));
  if (e == cudaSuccess) e = cudaMemset(ctx->ctrl, 0, sizeof(Ctrl));
  if (e == cudaSuccess) {
    uint64_t init[4] = {~0ull, 0, ~0ull, 0};
    e = cudaMemcpy(&ctx->ctrl->t_start_x, init, sizeof init, cudaMemcpyHostToDevice);
  }
  if (e == cudaSuccess && getenv("HALO_SEQ_BASE")) {  // test hook: start the sequence numbers near a tag wrap
    const uint64_t b[2] = {strtoull(getenv("HALO_SEQ_BASE"), nullptr, 0), strtoull(getenv("HALO_SEQ_BASE"), nullptr, 0)};
    e = cudaMemcpy(&ctx->ctrl->seq_x, b, sizeof b, cudaMemcpyHostToDevice);
  }
  if (e == cudaSuccess) e = cudaHostAlloc(&ctx->err_host, 64, cudaHostAllocMapped);
  if (e == cudaSuccess) { memset(ctx->err_host, 0, 64); e = cudaHostGetDevicePointer(&ctx->err_dev, ctx->err_host, 0); }
  if (e == cudaSuccess) e = cudaMalloc(&ctx->d_fshift_tmp, sizeof(double) * 9 * ctx->n_local);
  if (e == cudaSuccess) e = cudaMalloc(&ctx->d_small, 64 * 1024);
  if (e == cudaSuccess) e = cudaMallocHost(&ctx->h_small, 64 * 1024);
  if (e == cudaSuccess)
    e = cudaMalloc(&ctx->d_selcnt, sizeof(int32_t) * ctx->n_local * ((cfg->capacity + 1023) / 1024 + 1));
  if (e == cudaSuccess) e = cudaMalloc(&ctx->d_mig, sizeof(MigRank) * ctx->n_local);
  if (e == cudaSuccess) e = cudaMalloc(&ctx->d_migctrl, sizeof(MigCtrl));
  if (e == cudaSuccess) e = cudaMalloc(&ctx->d_planes, sizeof(double) * 3 * (kMaxRanks + 1));
  if (e == cudaSuccess) {
    // LL occupancy always (HALO_F_AUTO_TRANSPORT can switch a ctx to LL); the paper
    // protocol's kernels for the paper / copy-engine paths
    int b[4] = {0, 0, 0, 0}, bl[4] = {0, 0, 0, 0}, bw[4] = {0, 0, 0, 0};
    e = max_coresident_ll(cfg->layout, false, b, 0);
    if (e == cudaSuccess) e = max_coresident_ll(cfg->layout, false, bl, 1);
    if (e == cudaSuccess) e = max_coresident_ll(cfg->layout, true, bw, -1);
    ctx->max_x = b[0]; ctx->max_f = b[1]; ctx->max_xf = b[2]; ctx->max_x128 = b[3];
    ctx->max_x_loc = bl[0]; ctx->max_f_loc = bl[1]; ctx->max_xf_loc = bl[2]; ctx->max_x128_loc = bl[3];
    ctx->max_x_w = bw[0]; ctx->max_f_w = bw[1]; ctx->max_xf_w = bw[2];
    if (e == cudaSuccess && !ctx->ll) e = max_coresident(cfg->layout, &ctx->max_x, &ctx->max_f);
  }
  if (e == cudaSuccess) {
    // HALO_CTAS_PER_SM: cap the exchange grids (fewer, longer-lived CTAs; leaves SM
    // slots to a concurrently running compute kernel, Alg. 2)
    int sms = 0;
    if (const char* v = getenv("HALO_CTAS_PER_SM"))
      if (atoi(v) > 0 && cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, cfg->device) == cudaSuccess)
        ctx->grid_cap = atoi(v) * sms;
    if (const char* v = getenv("HALO_X_CTAS_PER_SM"))
      if (atoi(v) > 0 && cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, cfg->device) == cudaSuccess)
        ctx->x_cap = atoi(v) * sms;
  }
  if (e != cudaSuccess) {
    // keep ctx to carry the message? The ABI returns NULL on error; print once.
    fprintf(stderr, "halo_init: %s\n", cudaGetErrorString(e));
    (void)cudaGetLastError();
    halo_destroy(ctx);
    return HALO_ERR_CUDA;
  }
  *out = ctx;
  return HALO_OK;
}

halo_status halo_query_config(const halo_config* cfg, int* first_rank, int* n_local, int* npulse, int* dims,
                              size_t* scratch_bytes) {
  std::string why;
  halo_status s = validate(cfg, why);
  if (s != HALO_OK) return s;
  const int nr = cfg->grid[0] * cfg->grid[1] * cfg->grid[2];
  const int nl = nr / cfg->nprocs;
  int P = 0;
  const int order[3] = {2, 1, 0};
  for (int i = 0; i < 3; ++i)
    if (cfg->grid[order[i]] > 1)
      for (int k = 0; k < cfg->pulses[order[i]]; ++k) {
        if (dims) dims[P] = order[i];
        ++P;
      }
  if (first_rank) *first_rank = cfg->proc * nl;
  if (n_local) *n_local = nl;
  if (npulse) *npulse = P;
  if (scratch_bytes) *scratch_bytes = scratch_layout(P, cfg->capacity, cfg->layout).total;
  return HALO_OK;
}

halo_status halo_local_ranks(const halo_ctx* ctx, int* first_rank, int* n_local) {
  if (!ctx) return HALO_ERR_ARG;
  if (first_rank) *first_rank = ctx->first_rank;
  if (n_local) *n_local = ctx->n_local;
  return HALO_OK;
}

halo_status halo_pulse_order(const halo_ctx* ctx, int* npulse, int* dims) {
  if (!ctx || !npulse) return HALO_ERR_ARG;
  *npulse = ctx->P;
  if (dims)
    for (int p = 0; p < ctx->P; ++p) dims[p] = ctx->pdim[p];
  return HALO_OK;
}

halo_status halo_scratch_bytes(const halo_ctx* ctx, size_t* bytes) {
  if (!ctx || !bytes) return HALO_ERR_ARG;
  *bytes = ctx->scratch_bytes;
  return HALO_OK;
}

halo_status halo_register_buffers(halo_ctx* ctx, int local, void* x, void* f, void* scratch) {
  if (!ctx) return HALO_ERR_ARG;
  if (local < 0 || local >= ctx->n_local) return fail(ctx, HALO_ERR_ARG, "local rank out of range");
  if (!x || !f || !scratch) return fail(ctx, HALO_ERR_ARG, "NULL buffer");
  if (((uintptr_t)x | (uintptr_t)f) & 15) return fail(ctx, HALO_ERR_ARG, "x and f must be 16-B aligned");
  if ((uintptr_t)scratch & 255) return fail(ctx, HALO_ERR_ARG, "scratch must be 256-B aligned");
  CK(cudaSetDevice(ctx->cfg.device));
  CK(cudaMemset(scratch, 0, ctx->scratch_bytes));
  CK(cudaDeviceSynchronize());
  ctx->x[local] = (float*)x;
  ctx->f[local] = (float*)f;
  ctx->scratch[local] = (char*)scratch;
  const int r = ctx->first_rank + local;
  ctx->peer_x[r] = (float*)x;
  ctx->peer_f[r] = (float*)f;
  ctx->peer_scratch[r] = (char*)scratch;
  ctx->maps_ready = false;
  bool all = true;
  for (int l = 0; l < ctx->n_local; ++l) all &= ctx->scratch[l] != nullptr;
  if (all && ctx->cfg.nprocs == 1) ctx->peers_ready = true;
  return HALO_OK;
}

halo_status halo_ipc_export(halo_ctx* ctx, void* blob, size_t* len) {
  if (!ctx || !len) return HALO_ERR_ARG;
  const size_t need = sizeof(BlobHdr) + (size_t)ctx->n_local * sizeof(BlobEntry);
  if (!blob) { *len = need; return HALO_OK; }
  if (*len < need) return fail(ctx, HALO_ERR_ARG, "blob too small");
  for (int l = 0; l < ctx->n_local; ++l)
    if (!ctx->x[l]) return fail(ctx, HALO_ERR_STATE, "register all local buffers before export");
  PFN_memGetAddressRange range = get_addr_range_fn();
  if (!range) return fail(ctx, HALO_ERR_CUDA, "cuMemGetAddressRange entry point unavailable");
  CK(cudaSetDevice(ctx->cfg.device));
  BlobHdr h{};
  h.magic = kBlobMagic;
  h.version = HALO_ABI_VERSION;
  h.proc = ctx->cfg.proc;
  h.n_local = ctx->n_local;
  h.first_rank = ctx->first_rank;
  h.device = ctx->cfg.device;
  h.layout = ctx->cfg.layout;
  h.capacity = ctx->cfg.capacity;
  h.pid = 0;
  memcpy(blob, &h, sizeof h);
  BlobEntry* ents = reinterpret_cast<BlobEntry*>((char*)blob + sizeof h);
  for (int l = 0; l < ctx->n_local; ++l) {
    BlobEntry be{};
    unsigned long long base = 0;
    size_t sz = 0;
    if (range(&base, &sz, (unsigned long long)(uintptr_t)ctx->x[l]) != 0)
      return fail(ctx, HALO_ERR_PEER, "cuMemGetAddressRange(x) failed");
    CK(cudaIpcGetMemHandle(&be.hx, (void*)(uintptr_t)base));
    be.offx = (uintptr_t)ctx->x[l] - base;
    if (range(&base, &sz, (unsigned long long)(uintptr_t)ctx->scratch[l]) != 0)
      return fail(ctx, HALO_ERR_PEER, "cuMemGetAddressRange(scratch) failed");
    CK(cudaIpcGetMemHandle(&be.hs, (void*)(uintptr_t)base));
    be.offs = (uintptr_t)ctx->scratch[l] - base;
    if (range(&base, &sz, (unsigned long long)(uintptr_t)ctx->f[l]) != 0)
      return fail(ctx, HALO_ERR_PEER, "cuMemGetAddressRange(f) failed");
    CK(cudaIpcGetMemHandle(&be.hf, (void*)(uintptr_t)base));
    be.offf = (uintptr_t)ctx->f[l] - base;
    memcpy(&ents[l], &be, sizeof be);
  }
  *len = need;
  return HALO_OK;
}

halo_status halo_ipc_import(halo_ctx* ctx, const void* blobs, size_t len_each) {
  if (!ctx || !blobs) return HALO_ERR_ARG;
  const size_t need = sizeof(BlobHdr) + (size_t)ctx->n_local * sizeof(BlobEntry);
  if (len_each < need) return fail(ctx, HALO_ERR_ARG, "blob length too small");
  CK(cudaSetDevice(ctx->cfg.device));
  std::map<std::string, char*> opened;
  for (int pr = 0; pr < ctx->cfg.nprocs; ++pr) {
    const char* b = (const char*)blobs + (size_t)pr * len_each;
    BlobHdr h;
    memcpy(&h, b, sizeof h);
    if (h.magic != kBlobMagic || h.version != HALO_ABI_VERSION || h.proc != pr || h.n_local != ctx->n_local ||
        h.layout != ctx->cfg.layout || h.capacity != ctx->cfg.capacity)
      return fail(ctx, HALO_ERR_PEER, "inconsistent peer blob (proc " + std::to_string(pr) + ")");
    if (pr == ctx->cfg.proc) continue;
    const BlobEntry* ents = reinterpret_cast<const BlobEntry*>(b + sizeof h);
    for (int l = 0; l < h.n_local; ++l) {
      BlobEntry be;
      memcpy(&be, &ents[l], sizeof be);
      char* bases[3] = {nullptr, nullptr, nullptr};
      const cudaIpcMemHandle_t* hs[3] = {&be.hx, &be.hs, &be.hf};
      for (int k = 0; k < 3; ++k) {
        std::string key((const char*)hs[k], sizeof(cudaIpcMemHandle_t));
        auto it = opened.find(key);
        if (it != opened.end()) { bases[k] = it->second; continue; }
        void* ptr = nullptr;
        cudaError_t e = cudaIpcOpenMemHandle(&ptr, *hs[k], cudaIpcMemLazyEnablePeerAccess);
        if (e != cudaSuccess) {
          (void)cudaGetLastError();
          return fail(ctx, HALO_ERR_PEER, std::string("cudaIpcOpenMemHandle: ") + cudaGetErrorString(e));
        }
        opened[key] = (char*)ptr;
        ctx->opened.push_back(ptr);
        bases[k] = (char*)ptr;
      }
      const int r = h.first_rank + l;
      ctx->peer_x[r] = reinterpret_cast<float*>(bases[0] + be.offx);
      ctx->peer_scratch[r] = bases[1] + be.offs;
      ctx->peer_f[r] = reinterpret_cast<float*>(bases[2] + be.offf);
    }
  }
  for (int r = 0; r < ctx->nranks; ++r)
    if (!ctx->peer_x[r] || !ctx->peer_scratch[r]) return fail(ctx, HALO_ERR_PEER, "missing peer buffers");
  ctx->peers_ready = true;
  ctx->maps_ready = false;
  return HALO_OK;
}

}  // extern "C"

// ---------------------------------------------------------- plan construction
static void fill_rank_dev(halo_ctx* ctx) {
  ctx->h_ranks.resize(ctx->n_local);
  for (int l = 0; l < ctx->n_local; ++l) {
    RankDev& rd = ctx->h_ranks[l];
    rd.x = ctx->x[l];
    rd.f = ctx->f[l];
    rd.hdr = reinterpret_cast<ScratchHdr*>(ctx->scratch[l]);
    rd.maps = ctx->maps_of_local(l);
    rd.fbuf = ctx->fbuf_of(ctx->first_rank + l);
    rd.n_home = ctx->n_home[l];
    rd.n_total = ctx->n_total[l];
    rd.rank = ctx->first_rank + l;
  }
}

static void fill_pulse_dev(halo_ctx* ctx, int l, int p) {
  PulseDev& pd = ctx->h_pulses[l * ctx->P + p];
  memset(&pd, 0, sizeof pd);
  const int r = ctx->first_rank + l;
  const int d = ctx->pdim[p];
  const int lower = ctx->neighbour(r, d, -1);  // coordinates go to the lower neighbour (R1)
  const int upper = ctx->neighbour(r, d, +1);
  const int W = ctx->W;
  const int i = l * ctx->P + p;
  pd.map = ctx->maps_of_local(l) + (size_t)p * ctx->map_stride;
  pd.x_dst = ctx->peer_x[lower] + (size_t)ctx->remote_off[i] * W;
  pd.flag_x_dst = &ctx->hdr_of(lower)->flag_x[p];
  pd.fbuf_dst = ctx->fbuf_of(upper) + (size_t)p * ctx->fbuf_stride;
  pd.flag_f_dst = &ctx->hdr_of(upper)->flag_f[p];
  pd.fbuf_own = ctx->fbuf_of(r) + (size_t)p * ctx->fbuf_stride;
  pd.has_shift = ctx->cell(r, d) == 0;  // the wrapping sender adds +L_d (R1, R25)
  pd.shift[0] = pd.shift[1] = pd.shift[2] = 0.0f;
  if (pd.has_shift) pd.shift[d] = ctx->cfg.box[d];
  pd.dim = d;
  pd.send_size = ctx->send_size[i];
  pd.n_indep = ctx->n_indep[i];
  pd.atom_offset = ctx->atom_offset[i];
  pd.recv_size = ctx->recv_size[i];
  pd.dep_x = ctx->dep[i];
  uint32_t fdep = 0, chain = 0;
  for (int q = p + 1; q < ctx->P; ++q) {
    if (ctx->dep[l * ctx->P + q] & (1u << p)) fdep |= 1u << q;
    if (ctx->send_size[l * ctx->P + q] > 0) chain |= 1u << q;
  }
  pd.fdep = fdep;
  pd.chain = chain;
  pd.xll_dst = ctx->xll_of(lower) + (size_t)p * ctx->ll_stride;
  pd.fll_dst = ctx->fll_of(upper) + (size_t)p * ctx->ll_stride;
  pd.f_src = ctx->peer_f[lower] + (size_t)ctx->remote_off[i] * W;
  pd.consumed_dst = &ctx->hdr_of(lower)->consumed[p];
}

static void add_items(std::vector<Item>& v, int l, int p, uint8_t kind, int b, int e, int rows) {
  for (int s = b; s < e; s += rows) {
    Item it;
    it.lrank = (uint16_t)l;
    it.pulse = (uint8_t)p;
    it.kind = kind;
    it.begin = (uint32_t)s;
    it.end = (uint32_t)std::min(e, s + rows);
    v.push_back(it);
  }
}

// x items: independent chunks of every pulse first, then dependent chunks in
// pulse order (deadlock-free static schedule).
static void build_x_items(halo_ctx* ctx, int p_lo, int p_hi) {
  auto& v = ctx->h_items_x;
  v.clear();
  const int R = ctx->item_rows;
  for (int p = p_lo; p < p_hi; ++p)
    for (int l = 0; l < ctx->n_local; ++l) {
      const int i = l * ctx->P + p;
      add_items(v, l, p, kItemXIndep, 0, ctx->n_indep[i], R);
    }
  for (int p = p_lo; p < p_hi; ++p)
    for (int l = 0; l < ctx->n_local; ++l) {
      const int i = l * ctx->P + p;
      add_items(v, l, p, kItemXDep, ctx->n_indep[i], ctx->send_size[i], R);
    }
  for (int l = 0; l < ctx->n_local; ++l)
    for (int p = 0; p < ctx->P; ++p) ctx->h_pulses[l * ctx->P + p].n_items_x = 0;
  for (const Item& it : v) ctx->h_pulses[it.lrank * ctx->P + it.pulse].n_items_x++;
}

// f items: level by level from the last pulse down: push(p) then unpack(p).
static void build_f_items(halo_ctx* ctx) {
  auto& v = ctx->h_items_f;
  v.clear();
  const int R = ctx->item_rows;
  for (int p = ctx->P - 1; p >= 0; --p) {
    for (int l = 0; l < ctx->n_local; ++l) add_items(v, l, p, kItemPush, 0, ctx->recv_size[l * ctx->P + p], R);
    for (int l = 0; l < ctx->n_local; ++l) add_items(v, l, p, kItemUnpack, 0, ctx->send_size[l * ctx->P + p], R);
  }
  for (int l = 0; l < ctx->n_local; ++l)
    for (int p = 0; p < ctx->P; ++p) {
      PulseDev& pd = ctx->h_pulses[l * ctx->P + p];
      pd.n_items_push = pd.n_items_unpack = 0;
    }
  for (const Item& it : v) {
    PulseDev& pd = ctx->h_pulses[it.lrank * ctx->P + it.pulse];
    if (it.kind == kItemPush) pd.n_items_push++; else pd.n_items_unpack++;
  }
}

// Host loops of the NS-step plan build over many independent items: split over a
// few threads (the item blocks are MBs at C3/C4; the NS step is host-bound).
template <class F>
static void parallel_for(size_t n, F&& body) {
  const size_t T = n < 512 ? 1 : std::min<size_t>(8, std::max(1u, std::thread::hardware_concurrency()));
  if (T == 1) {
    for (size_t k = 0; k < n; ++k) body(k);
    return;
  }
  std::vector<std::thread> th;
  for (size_t t = 0; t < T; ++t)
    th.emplace_back([&, t] {
      for (size_t k = n * t / T; k < n * (t + 1) / T; ++k) body(k);
    });
  for (auto& x : th) x.join();
}

// ------------------------------------------------------------- LL plan (hop groups)
// The DD ranks of this process share one GPU: they form one hop group (DESIGN.md
// §6.1; HALO_COLLAPSE=0: every rank its own group).  A pulse between two ranks of
// the group moves no data through the LL areas: the plan below resolves it.
static bool same_group(const halo_ctx* ctx, int r1, int r2) {
  return ctx->collapse && ctx->is_local(r1) && ctx->is_local(r2);
}

// A bulk x pulse: the last pulse (no later pulse forwards its rows)
// from another hop group, rows >= bulk_rows.  The x-sender stores the rows straight
// into the receiver's x and counts them in its header; the receiver waits for the
// count instead of polling LL units: each byte crosses NVLink once, untagged.  Both
// ends decide on the same number (the sender's send_size is the receiver's recv_size).
static bool bulk_pulse(const halo_ctx* ctx, int p, int rows) {
  return ctx->bulk_rows > 0 && p == ctx->P - 1 && rows >= ctx->bulk_rows;
}

static void fill_lbase(halo_ctx* ctx) {
  const int L = ctx->n_local, P = ctx->P;
  ctx->h_lbase.assign(std::max(1, L), LocalBase{});
  for (int l = 0; l < L; ++l) {
    LocalBase& b = ctx->h_lbase[l];
    const int r = ctx->first_rank + l;
    b.x = ctx->x[l];
    b.f = ctx->f[l];
    b.xll = ctx->xll_of(r);
    b.fll = ctx->fll_of(r);
    for (int q = 0; q < kMaxP; ++q) b.recv_off[q] = q < P ? ctx->atom_offset[l * P + q] : 0;
    b.n_home = ctx->n_home[l];
  }
}

// Origin of every row of every local rank, pulses < p_hi (the rows a send of
// pulse < p_hi can read): a home row, or the LL unit in which the row entered
// the group, plus the pulses whose shift it picked up since (R25).  cls = 0 for
// a home origin, q+1 for an LL unit of pulse q (x dependency class).
struct XOrig {
  uint32_t row;
  uint8_t l, kq, mask, cls;
};
static void resolve_origins(const halo_ctx* ctx, int p_hi, std::vector<std::vector<XOrig>>& org) {
  const int L = ctx->n_local, P = ctx->P;
  org.assign(L, {});
  for (int l = 0; l < L; ++l) {
    org[l].resize(ctx->n_total[l]);
    for (int t = 0; t < ctx->n_home[l]; ++t) org[l][t] = XOrig{(uint32_t)t, (uint8_t)l, 0, 0, 0};
  }
  for (int q = 0; q < p_hi; ++q)
    for (int l = 0; l < L; ++l) {
      const int r = ctx->first_rank + l, i0 = ctx->atom_offset[l * P + q], n = ctx->recv_size[l * P + q];
      const int s = ctx->neighbour(r, ctx->pdim[q], +1);  // the x-sender of this rank's pulse-q rows
      if (same_group(ctx, r, s)) {
        const int sl = s - ctx->first_rank;
        const auto& m = ctx->h_maps[sl][q];
        const bool wraps = ctx->cell(s, ctx->pdim[q]) == 0;
        for (int i = 0; i < n; ++i) {
          XOrig o = org[sl][m[i]];
          if (wraps) o.mask |= (uint8_t)(1u << q);
          org[l][i0 + i] = o;
        }
      } else {
        for (int i = 0; i < n; ++i) org[l][i0 + i] = XOrig{(uint32_t)i, (uint8_t)l, (uint8_t)(0x80u | q), 0, (uint8_t)(q + 1)};
      }
    }
}

// x items of pulses [p_lo, p_hi): the sends of every local rank (entries = the
// origins of the rows it sends, split into runs of one dependency class), sorted
// by class (a wait targets a lower class only: deadlock-free static order), then
// the receive items of the rows that come from another group.
static void build_ll_x(halo_ctx* ctx, int p_lo, int p_hi) {
  const int L = ctx->n_local, P = ctx->P, W = ctx->W, R = ctx->item_rows;
  std::vector<std::vector<XOrig>> org;
  resolve_origins(ctx, p_hi, org);
  struct XI {
    XRec rec;
    std::vector<XEnt> ent;
  };
  std::vector<XI> items;
  for (int p = p_lo; p < p_hi; ++p)
    for (int l = 0; l < L; ++l) {
      const int r = ctx->first_rank + l, d = ctx->pdim[p];
      const auto& m = ctx->h_maps[l][p];
      const int n = (int)m.size();
      const int rcv = ctx->neighbour(r, d, -1);  // coordinates go to the lower neighbour (R1)
      const bool wraps = ctx->cell(r, d) == 0;   // the wrapping sender adds +L_d (R25)
      const bool local = same_group(ctx, r, rcv);
      const bool bulk = !local && bulk_pulse(ctx, p, n);
      for (int b = 0; b < n;) {
        const uint8_t cls = org[l][m[b]].cls;
        int e = b;
        while (e < n && e - b < R && org[l][m[e]].cls == cls) ++e;
        XI it;
        memset(&it.rec, 0, sizeof it.rec);
        XRec& x = it.rec;
        x.kind = kItemXSend;
        x.pulse = (uint8_t)p;
        x.lrank = (uint16_t)l;
        x.n_units = (uint32_t)(e - b) * W;
        x.begin = (uint32_t)b;
        x.cls = cls;
        x.epoch = ctx->epoch;
        if (local) {
          x.dst_x = ctx->x[rcv - ctx->first_rank] + (size_t)ctx->remote_off[l * P + p] * W;
        } else if (bulk) {
          x.dst_x = ctx->peer_x[rcv] + (size_t)ctx->remote_off[l * P + p] * W;
          x.bulk = &ctx->hdr_of(rcv)->bulk_x[p];
          x.bulk_total = (uint32_t)n;
        } else {
          x.dst_ll = ctx->xll_of(rcv) + (size_t)p * ctx->ll_stride;
        }
        for (int q = 0; q < P; ++q) {
          x.shiftL[q] = ctx->cfg.box[ctx->pdim[q]];
          x.pdim[q] = (uint8_t)ctx->pdim[q];
        }
        it.ent.resize(e - b);
        for (int k = b; k < e; ++k) {
          const XOrig& o = org[l][m[k]];
          it.ent[k - b] = XEnt{o.row, o.l, o.kq, (uint8_t)(o.mask | (wraps ? 1u << p : 0u)), 0};
        }
        items.push_back(std::move(it));
        b = e;
      }
    }
  std::stable_sort(items.begin(), items.end(), [](const XI& a, const XI& b) { return a.rec.cls < b.rec.cls; });
  // receives: this rank's rows of a pulse whose sender is in another group
  for (int p = p_lo; p < p_hi; ++p)
    for (int l = 0; l < L; ++l) {
      const int r = ctx->first_rank + l;
      if (same_group(ctx, r, ctx->neighbour(r, ctx->pdim[p], +1))) continue;
      const int n = ctx->recv_size[l * P + p];
      if (bulk_pulse(ctx, p, n)) {  // one wait item for the whole pulse
        XI it;
        memset(&it.rec, 0, sizeof it.rec);
        it.rec.kind = kItemXWait;
        it.rec.pulse = (uint8_t)p;
        it.rec.lrank = (uint16_t)l;
        it.rec.n_units = (uint32_t)n;  // rows
        it.rec.cls = 0xff;
        it.rec.epoch = ctx->epoch;
        it.rec.bulk = &ctx->hdr_of(r)->bulk_x[p];
        items.push_back(std::move(it));
        continue;
      }
      const int RR = std::min(kMaxItemRows, ctx->recv_mult * R);
      for (int b = 0; b < n; b += RR) {
        const int e = std::min(n, b + RR);
        XI it;
        memset(&it.rec, 0, sizeof it.rec);
        XRec& x = it.rec;
        x.kind = kItemXRecv;
        x.pulse = (uint8_t)p;
        x.lrank = (uint16_t)l;
        x.n_units = (uint32_t)(e - b) * W;
        x.begin = (uint32_t)b;
        x.cls = 0xff;
        x.epoch = ctx->epoch;
        x.ll = ctx->xll_of(r) + (size_t)p * ctx->ll_stride + (size_t)b * W;
        x.xdst = ctx->x[l] + (size_t)(ctx->atom_offset[l * P + p] + b) * W;
        items.push_back(std::move(it));
      }
    }
  const size_t XB = ll_xblk_bytes(R);
  ctx->h_items_x.assign(items.size(), Item{});
  ctx->h_xblk.assign(items.size() * XB, 0);
  for (size_t k = 0; k < items.size(); ++k) {
    Item& w = ctx->h_items_x[k];
    w.lrank = items[k].rec.lrank;
    w.pulse = items[k].rec.pulse;
    w.kind = items[k].rec.kind;
  }
  parallel_for(items.size(), [&](size_t k) {
    memcpy(&ctx->h_xblk[k * XB], &items[k].rec, sizeof(XRec));
    if (!items[k].ent.empty()) memcpy(&ctx->h_xblk[k * XB + 128], items[k].ent.data(), sizeof(XEnt) * items[k].ent.size());
  });
}

// Node list of the tree under row t of local rank l, depth first, children in
// descending pulse order (the oracle's accumulation order, R15).  `fs` of the
// edge into a node: 3 * (parent's local rank) + dim when the parent's rank
// wrapped in the edge's pulse (R13), else 0xff.  Appends to `v` (a per-thread
// arena: no allocation per tree).
static void emit_tree(const halo_ctx* ctx, const std::vector<std::vector<int32_t>>& child, int l, int t, int depth,
                      int parent, uint8_t fs, std::vector<TNode>& v, size_t base, int& lowest_ll) {
  const int P = ctx->P, r = ctx->first_rank + l;
  const size_t me = v.size();
  v.push_back(TNode{(uint32_t)t | ((uint32_t)l << 24), 0, (uint8_t)(parent < 0 ? 0xff : parent),
                    (uint8_t)(depth << 1), fs});
  for (int q = P - 1; q >= 0; --q) {
    const int i = child[l][(size_t)t * P + q];
    if (i < 0) continue;
    v[me].flags |= 1;  // has children: its folded value is stored
    const int d = ctx->pdim[q];
    const uint8_t efs = ctx->cell(r, d) == 0 ? (uint8_t)(3 * l + d) : (uint8_t)0xff;
    const int rcv = ctx->neighbour(r, d, -1);
    if (same_group(ctx, r, rcv)) {
      emit_tree(ctx, child, rcv - ctx->first_rank, ctx->remote_off[l * P + q] + i, depth + 1, (int)(me - base), efs,
                v, base, lowest_ll);
    } else {
      v.push_back(TNode{(uint32_t)i | ((uint32_t)l << 24), (uint8_t)(0x80u | q), (uint8_t)(me - base),
                        (uint8_t)((depth + 1) << 1), efs});
      lowest_ll = std::min(lowest_ll, q);
    }
  }
}

struct PhaseTimer {
  bool on = getenv("HALO_PROFILE") != nullptr;
  std::chrono::steady_clock::time_point t = std::chrono::steady_clock::now();
  std::string acc;
  void lap(const char* name) {
    if (!on) return;
    const auto now = std::chrono::steady_clock::now();
    char buf[96];
    snprintf(buf, sizeof buf, " %s=%.0f", name, std::chrono::duration<double, std::micro>(now - t).count());
    acc += buf;
    t = now;
  }
  void print(int rank) const {
    if (on) fprintf(stderr, "[halo_profile rank %d set_maps us]%s\n", rank, acc.c_str());
  }
};

// Distinct shift-force targets of one tree or one item (<= kMaxBuckets + 1 kept).
struct FsSet {
  uint8_t v[kMaxBuckets + 1];
  int n = 0;
  bool add(uint8_t x) {  // false once more than kMaxBuckets distinct targets were seen
    for (int k = 0; k < n; ++k)
      if (v[k] == x) return true;
    if (n <= kMaxBuckets) v[n++] = x;
    return n <= kMaxBuckets;
  }
  int find(uint8_t x) const {
    for (int k = 0; k < n; ++k)
      if (v[k] == x) return k;
    return -1;
  }
};

// f items: the trees of this group.  A row's children are its images (one per
// pulse whose map sends it); children in this group are nodes of the same tree,
// children in another group are LL nodes (the value they push back).  Roots: home
// rows with children, and halo rows whose x-sender is in another group (they push
// their value back there).  Dependency class of a tree = P - (lowest pulse of its
// LL nodes), 0 without: a pushed value comes from a tree whose LL nodes all have
// higher pulses, i.e. a lower class.  NS-step host work: no allocation per tree
// (per-thread node arenas, fixed-size shift-force sets and postorder stacks).
static halo_status build_ll_f(halo_ctx* ctx, PhaseTimer* prof = nullptr) {
  const int L = ctx->n_local, P = ctx->P, W = ctx->W;
  // child[l][t*P + q] = i: row t of rank l is entry i of map_q (one per pulse at most)
  std::vector<std::vector<int32_t>> child(L);
  parallel_for((size_t)L, [&](size_t l) {
    child[l].assign((size_t)ctx->n_total[l] * P, -1);
    for (int q = 0; q < P; ++q) {
      const auto& m = ctx->h_maps[l][q];
      for (size_t i = 0; i < m.size(); ++i) child[l][(size_t)m[i] * P + q] = (int32_t)i;
    }
  });
  if (prof) prof->lap("f:child");
  struct Tree {
    int l, t;
    uint8_t cls;
    bool small;
    bool direct;  // more than kMaxBuckets shift-force targets: its edges add directly
    uint16_t nn;
    const TNode* nodes;
    uint64_t* push;
    FsSet fs;
  };
  std::vector<Tree> roots;
  {
    size_t nr = 0;
    for (int l = 0; l < L; ++l) nr += ctx->n_total[l];
    roots.reserve(nr);
  }
  for (int l = 0; l < L; ++l) {
    const int r = ctx->first_rank + l;
    const int32_t* cl = child[l].data();
    for (int t = 0; t < ctx->n_home[l]; ++t) {
      bool any = false;
      for (int q = 0; q < P && !any; ++q) any = cl[(size_t)t * P + q] >= 0;
      if (any) roots.push_back(Tree{l, t, 0, true, false, 0, nullptr, nullptr, {}});
    }
    for (int q = 0; q < P; ++q) {
      const int s = ctx->neighbour(r, ctx->pdim[q], +1);
      if (same_group(ctx, r, s)) continue;
      const int i0 = ctx->atom_offset[l * P + q];
      uint64_t* base = ctx->fll_of(s) + (size_t)q * ctx->ll_stride;
      for (int i = 0; i < ctx->recv_size[l * P + q]; ++i)
        roots.push_back(Tree{l, i0 + i, 0, true, false, 0, nullptr, base + (size_t)i * W, {}});
    }
  }
  if (prof) prof->lap("f:roots");
  // depth-first node lists (children pulses descending, R15) into per-thread arenas
  const size_t NR = roots.size();
  const size_t T = NR < 4096 ? 1 : std::min<size_t>(8, std::max(1u, std::thread::hardware_concurrency()));
  std::vector<std::vector<TNode>> arena(T);
  auto emit_range = [&](size_t th) {
    const size_t k0 = NR * th / T, k1 = NR * (th + 1) / T;
    auto& v = arena[th];
    v.reserve((k1 - k0) * 3 + 16);
    std::vector<size_t> begin(k1 - k0);
    for (size_t k = k0; k < k1; ++k) {
      int lowest_ll = P;
      begin[k - k0] = v.size();
      emit_tree(ctx, child, roots[k].l, roots[k].t, 0, -1, 0xff, v, v.size(), lowest_ll);
      Tree& R = roots[k];
      R.cls = (uint8_t)(P - lowest_ll);
      R.nn = (uint16_t)(v.size() - begin[k - k0]);
      R.small = R.nn <= kFastNodes;
      for (size_t m = begin[k - k0]; m < v.size(); ++m)
        if (v[m].fs != 0xff && !R.fs.add(v[m].fs)) R.direct = true;
    }
    for (size_t k = k0; k < k1; ++k) roots[k].nodes = v.data() + begin[k - k0];  // the arena no longer grows
  };
  if (T == 1) {
    emit_range(0);
  } else {
    std::vector<std::thread> th;
    for (size_t t = 0; t < T; ++t) th.emplace_back(emit_range, t);
    for (auto& x : th) x.join();
  }
  if (prof) prof->lap("f:emit");
  // items: roots ordered by class, rank, small/large, in row order
  std::vector<uint32_t> order(NR);
  for (size_t k = 0; k < NR; ++k) order[k] = (uint32_t)k;
  std::stable_sort(order.begin(), order.end(), [&](uint32_t a, uint32_t b) {
    const Tree &x = roots[a], &y = roots[b];
    if (x.cls != y.cls) return x.cls < y.cls;
    if (x.l != y.l) return x.l < y.l;
    return x.small > y.small;
  });
  struct FI {
    size_t b, e;  // range of `order`
    bool small;
    int nodes;
    FsSet fs;     // bucket targets
  };
  auto form = [&](int RT, std::vector<FI>& fis) {
    fis.clear();
    const int RG = std::max(1, RT / 8);                      // large trees per item
    const int NG = (int)((ll_fblk_bytes(RT) - 128 - 16 * RG) / 8);  // their node capacity
    for (size_t k = 0; k < NR;) {
      const Tree& t0 = roots[order[k]];
      FI f{k, k, t0.small, 0, {}};
      while (f.e < NR) {
        const Tree& t = roots[order[f.e]];
        if (t.cls != t0.cls || t.l != t0.l || t.small != t0.small) break;
        if ((int)(f.e - f.b) >= (f.small ? RT : RG)) break;
        if (!f.small && f.nodes + (int)t.nn > NG && f.e > f.b) break;
        if (!t.direct) {  // (a tree with more targets than buckets adds its edges directly)
          FsSet u = f.fs;
          bool ok = true;
          for (int j = 0; j < t.fs.n && ok; ++j) ok = u.add(t.fs.v[j]);
          if (!ok && f.e > f.b) break;
          f.fs = u;
        }
        f.nodes += (int)t.nn;
        ++f.e;
      }
      fis.push_back(f);
      k = fis.back().e;
    }
  };
  // roots per item: the smallest size whose items all fit the co-resident grid
  // (one item per CTA, one pass of 3 components per root), else kTreeRowsOcc
  std::vector<FI> fis;
  int RT = 32;
  for (;; RT = std::min(kTreeRowsOcc, RT + 16)) {
    form(RT, fis);
    if ((int)fis.size() <= ctx->cap_f() || RT == kTreeRowsOcc) break;
  }
  if (const char* e = getenv("HALO_TREE_ROWS")) {
    RT = std::min(kTreeRowsOcc, std::max(8, atoi(e)));
    form(RT, fis);
  }
  if (prof) prof->lap("f:form");
  const int RG = std::max(1, RT / 8);
  for (const FI& f : fis)
    if (!f.small && (int)(128 + 16 * RG + 8 * f.nodes) > (int)ll_fblk_bytes(RT))
      return fail(ctx, HALO_ERR_UNSUPPORTED, "a force tree exceeds the node capacity of a work item");
  ctx->tree_rows = RT;
  const size_t FB = ll_fblk_bytes(RT);
  const size_t nt = fis.size();
  ctx->h_items_f.assign(nt, Item{});
  ctx->h_fblk.assign(nt * FB, 0);
  parallel_for(nt, [&](size_t k) {
    const FI& f = fis[k];
    char* blk = &ctx->h_fblk[k * FB];
    GRec g;
    memset(&g, 0, sizeof g);
    g.kind = f.small ? kItemTree : kItemTreeG;
    g.level = roots[order[f.b]].cls;
    g.lrank = (uint16_t)roots[order[f.b]].l;
    g.n_roots = (uint32_t)(f.e - f.b);
    g.n_units = g.n_roots * W;
    g.n_nodes = (uint32_t)f.nodes;
    g.n_buckets = (uint8_t)f.fs.n;
    g.epoch = ctx->epoch;
    for (int b = 0; b < f.fs.n; ++b) g.bucket_fs[b] = f.fs.v[b];
    memcpy(blk, &g, sizeof g);
    auto bucket_of = [&](const TNode& x, bool direct) -> uint8_t {
      if (x.fs == 0xff) return kFsNone;
      return direct ? kFsDirect : (uint8_t)f.fs.find(x.fs);
    };
    if (f.small) {
      TRoot* rr = reinterpret_cast<TRoot*>(blk + 128);
      uint32_t* il = reinterpret_cast<uint32_t*>(blk + 128 + 32 * (size_t)RT);
      for (size_t j = f.b; j < f.e; ++j) {
        const Tree& tr = roots[order[j]];
        const TNode* v = tr.nodes;
        const int nn = tr.nn;
        TRoot R;
        memset(&R, 0, sizeof R);
        R.push = tr.push;
        R.par = 0xffffffffu;
        R.bucket = 0xffffffffu;
        R.nn = (uint8_t)nn;
        // postorder of the non-root nodes (a node after all its descendants, siblings in
        // preorder = descending pulse order): close every open node at least as deep as
        // the next node in preorder
        {
          int stk[kFastNodes], top = 0, e = 0;
          for (int m = 0; m <= nn; ++m) {
            const int dm = m < nn ? (v[m].flags >> 1) : 0;
            while (top > 0 && (v[stk[top - 1]].flags >> 1) >= dm) {
              const int c = stk[--top];
              if (c != 0) R.post |= (uint32_t)c << (4 * e++);
            }
            if (m < nn) stk[top++] = m;
          }
        }
        for (int m = 0; m < nn; ++m) {
          const TNode& x = v[m];
          const uint32_t sh = 4 * (uint32_t)m;
          R.par = (R.par & ~(15u << sh)) | ((uint32_t)(x.parent == 0xff ? 15 : x.parent) << sh);
          R.bucket = (R.bucket & ~(15u << sh)) | ((uint32_t)bucket_of(x, false) << sh);
          R.q |= (uint32_t)(x.kq & 7) << sh;
          if (x.kq & 0x80u) R.llmask |= (uint8_t)(1u << m);
          if (x.flags & 1u) R.stmask |= (uint8_t)(1u << m);
          il[8 * (j - f.b) + m] = x.il;
        }
        rr[j - f.b] = R;
      }
    } else {
      TRootG* rr = reinterpret_cast<TRootG*>(blk + 128);
      TNode* nn = reinterpret_cast<TNode*>(blk + 128 + 16 * (size_t)RG);
      uint32_t at = 0;
      for (size_t j = f.b; j < f.e; ++j) {
        const Tree& tr = roots[order[j]];
        rr[j - f.b] = TRootG{tr.push, at, tr.nn, 0};
        for (int m = 0; m < tr.nn; ++m) {
          TNode x = tr.nodes[m];
          x.kq = (uint8_t)((x.kq & 0x87u) | (bucket_of(x, tr.direct) << 3));
          nn[at + m] = x;
        }
        at += tr.nn;
      }
    }
    Item& w = ctx->h_items_f[k];
    w.lrank = g.lrank;
    w.pulse = g.level;
    w.kind = g.kind;
  });
  ctx->n_tail_f = 0;
  if (prof) prof->lap("f:blocks");
  return HALO_OK;
}

// Shift-force targets of every force tree rooted at local rank l (R13): the edges of
// the rank-level tree (a row of rank r received in pulse qlast can be sent in any later
// pulse q; a wrapping sender's edges add into fshift[r][d_q]; same-group receivers
// continue the tree).  At most 2^P - 1 edges, i.e. <= kMaxBuckets for P <= 3.
static halo_status upload_plan(halo_ctx* ctx, cudaStream_t st = nullptr);
static halo_status pull_maps(halo_ctx* ctx, int p, cudaStream_t st);

static bool rank_tree_fs(const halo_ctx* ctx, int r, int qlast, FsSet& fs) {
  for (int q = qlast + 1; q < ctx->P; ++q) {
    const int d = ctx->pdim[q];
    if (ctx->cell(r, d) == 0 && !fs.add((uint8_t)(3 * (r - ctx->first_rank) + d))) return false;
    const int rcv = ctx->neighbour(r, d, -1);
    if (same_group(ctx, r, rcv) && !rank_tree_fs(ctx, rcv, q, fs)) return false;
  }
  return true;
}

// HALO_PLAN_CHECK=1 (debug): the host builder's plan of the same maps vs the GPU-built
// blocks, field by field (the shift-force bucket numbering differs by design); the
// first mismatches go to stderr and fail set_maps.
static halo_status plan_check(halo_ctx* ctx, cudaStream_t st) {
  const int P = ctx->P;
  const int nx = ctx->gpu_n_items_x, nf = ctx->gpu_n_items_f;
  const uint32_t XB = ll_xblk_bytes(ctx->item_rows), FB = ll_fblk_bytes(ctx->tree_rows);
  std::vector<char> gx((size_t)nx * XB), gf((size_t)nf * FB);
  CK(cudaStreamSynchronize(st));
  CK(cudaMemcpy(gx.data(), ctx->d_xblk, gx.size(), cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(gf.data(), ctx->d_fblk, gf.size(), cudaMemcpyDeviceToHost));
  for (int p = 0; p < P; ++p) {
    halo_status s = pull_maps(ctx, p, st);
    if (s != HALO_OK) return s;
  }
  const int RT = ctx->tree_rows;
  build_ll_x(ctx, 0, P);
  halo_status s = build_ll_f(ctx);
  if (s != HALO_OK) return s;
  int bad = 0;
  auto report = [&](const char* what, int item, int k, long a, long b) {
    if (bad++ < 12) fprintf(stderr, "[plan_check] %s item %d k %d: gpu %ld host %ld\n", what, item, k, a, b);
  };
  if ((int)ctx->h_items_x.size() != nx) report("n_items_x", -1, -1, nx, (long)ctx->h_items_x.size());
  for (int i = 0; i < std::min(nx, (int)ctx->h_items_x.size()); ++i) {
    const XRec& g = *reinterpret_cast<const XRec*>(&gx[(size_t)i * XB]);
    const XRec& h = *reinterpret_cast<const XRec*>(&ctx->h_xblk[(size_t)i * XB]);
    if (memcmp(&g, &h, sizeof(XRec)) != 0) {
      report("XRec kind", i, 0, g.kind, h.kind);
      report("XRec pulse/lrank", i, 0, g.pulse * 1000 + g.lrank, h.pulse * 1000 + h.lrank);
      report("XRec n_units/begin", i, 0, (long)g.n_units * 100000 + g.begin, (long)h.n_units * 100000 + h.begin);
      report("XRec cls/epoch", i, 0, (long)g.cls * 100000 + g.epoch, (long)h.cls * 100000 + h.epoch);
      report("XRec dst", i, 0, (long)(uintptr_t)g.dst_x ^ (long)(uintptr_t)g.dst_ll, (long)(uintptr_t)h.dst_x ^ (long)(uintptr_t)h.dst_ll);
      continue;
    }
    for (uint32_t e = 0; e < h.n_units / ctx->W && h.kind == kItemXSend; ++e) {
      const XEnt& a = reinterpret_cast<const XEnt*>(&gx[(size_t)i * XB + 128])[e];
      const XEnt& b = reinterpret_cast<const XEnt*>(&ctx->h_xblk[(size_t)i * XB + 128])[e];
      if (memcmp(&a, &b, sizeof(XEnt)) != 0) report("XEnt row|l|kq|mask", i, (int)e,
          ((long)a.row << 24) | (a.l << 16) | (a.kq << 8) | a.mask, ((long)b.row << 24) | (b.l << 16) | (b.kq << 8) | b.mask);
    }
  }
  if ((int)ctx->h_items_f.size() != nf) report("n_items_f", -1, -1, nf, (long)ctx->h_items_f.size());
  if (ctx->tree_rows != RT) report("tree_rows", -1, -1, RT, ctx->tree_rows);
  for (int i = 0; i < std::min(nf, (int)ctx->h_items_f.size()) && ctx->tree_rows == RT; ++i) {
    const GRec& g = *reinterpret_cast<const GRec*>(&gf[(size_t)i * FB]);
    const GRec& h = *reinterpret_cast<const GRec*>(&ctx->h_fblk[(size_t)i * FB]);
    if (g.kind != h.kind || g.level != h.level || g.lrank != h.lrank || g.n_roots != h.n_roots || g.n_units != h.n_units ||
        g.epoch != h.epoch) {
      report("GRec kind/level/lrank", i, 0, g.kind * 10000 + g.level * 1000 + g.lrank, h.kind * 10000 + h.level * 1000 + h.lrank);
      report("GRec n_roots/n_units", i, 0, (long)g.n_roots * 100000 + g.n_units, (long)h.n_roots * 100000 + h.n_units);
      continue;
    }
    for (uint32_t j = 0; j < h.n_roots; ++j) {
      const TRoot& a = reinterpret_cast<const TRoot*>(&gf[(size_t)i * FB + 128])[j];
      const TRoot& b = reinterpret_cast<const TRoot*>(&ctx->h_fblk[(size_t)i * FB + 128])[j];
      if (a.push != b.push || a.par != b.par || a.q != b.q || a.nn != b.nn || a.llmask != b.llmask ||
          a.stmask != b.stmask || a.post != b.post)
        report("TRoot nn|par|post", i, (int)j, ((long)a.nn << 40) ^ ((long)a.par << 8) ^ a.post,
               ((long)b.nn << 40) ^ ((long)b.par << 8) ^ b.post);
      const uint32_t* ia = reinterpret_cast<const uint32_t*>(&gf[(size_t)i * FB + 128 + 32 * (size_t)RT]) + 8 * j;
      const uint32_t* ib = reinterpret_cast<const uint32_t*>(&ctx->h_fblk[(size_t)i * FB + 128 + 32 * (size_t)RT]) + 8 * j;
      for (int k = 0; k < b.nn; ++k)
        if (ia[k] != ib[k]) report("TRoot il", i, (int)j * 8 + k, ia[k], ib[k]);
    }
  }
  ctx->h_items_x.clear();
  ctx->h_items_f.clear();
  ctx->h_xblk.clear();
  ctx->h_fblk.clear();
  fprintf(stderr, "[plan_check] rank %d: %d mismatches (x items %d, f items %d)\n", ctx->first_rank, bad, nx, nf);
  return bad ? fail(ctx, HALO_ERR_STATE, "GPU plan != host plan (HALO_PLAN_CHECK)") : HALO_OK;
}

static halo_status build_ll_plan_gpu(halo_ctx* ctx, cudaStream_t st, PhaseTimer* prof) {
  const int L = ctx->n_local, P = ctx->P, W = ctx->W, R = ctx->item_rows;
  const size_t cap = (size_t)ctx->cfg.capacity;
  if (!ctx->d_pl) {
    CK(cudaMalloc(&ctx->d_pl, sizeof(PlanDev)));
    CK(cudaMallocHost(&ctx->h_pl, sizeof(PlanDev)));
    CK(cudaMallocHost(&ctx->h_pl_cnt, sizeof(int32_t) * (kMaxP + 1) * (kMaxP + 1) * kMaxLocal));
  }
  int max_rows = 1, max_send = 1;
  for (int l = 0; l < L; ++l) max_rows = std::max(max_rows, ctx->n_total[l]);
  for (int i = 0; i < L * P; ++i) max_send = std::max(max_send, ctx->send_size[i]);
  const int nblk = (max_rows + plan_rows_per_cta() - 1) / plan_rows_per_cta();
  const int xnch = (max_send + plan_rows_per_cta() - 1) / plan_rows_per_cta();
  const size_t sxc = align_up(sizeof(int32_t) * (size_t)P * L * xnch * (2 + kMaxP + 1), 256);
  const size_t so = align_up(sizeof(uint64_t) * L * cap, 256), sc = align_up(sizeof(int32_t) * L * cap * P, 256),
               sr = align_up(2 * L * cap, 256), sk = align_up(2 * sizeof(int32_t) * L * nblk * (P + 1), 256),
               si = align_up(sizeof(uint32_t) * (L * cap / 8 + (size_t)(kMaxP + 1) * L + 1), 256),
               sx = align_up(sizeof(int32_t) * (P * L + L) * (P + 1), 256);
  const size_t sbytes = so + sc + sr + sk + sx + si + sxc;
  if (sbytes > ctx->pl_scratch_bytes) {
    if (ctx->d_pl_scratch) CK(cudaFree(ctx->d_pl_scratch));
    ctx->d_pl_scratch = nullptr;
    CK(cudaMalloc(&ctx->d_pl_scratch, sbytes));
    ctx->pl_scratch_bytes = sbytes;
  }
  PlanDev& H = *ctx->h_pl;
  memset(&H, 0, sizeof H);
  H.err_host = ctx->err_dev;
  H.L = L;
  H.P = P;
  H.W = W;
  H.R = R;
  H.cap = (int)cap;
  H.map_stride = (int)ctx->map_stride;
  H.epoch = ctx->epoch;
  H.XB = ll_xblk_bytes(R);
  for (int q = 0; q < P; ++q) {
    H.shiftL[q] = ctx->cfg.box[ctx->pdim[q]];
    H.pdim[q] = (uint8_t)ctx->pdim[q];
  }
  H.nblk = nblk;
  for (int l = 0; l < L; ++l) {
    const int r = ctx->first_rank + l;
    H.n_home[l] = ctx->n_home[l];
    H.n_total[l] = ctx->n_total[l];
    H.maps[l] = ctx->maps_of_local(l);
    FsSet fs;
    if (!rank_tree_fs(ctx, r, -1, fs)) return HALO_ERR_UNSUPPORTED;  // host builder
    H.n_buckets[l] = (uint8_t)fs.n;
    for (int b = 0; b < fs.n; ++b) H.bucket_fs[l][b] = fs.v[b];
    for (int q = 0; q < P; ++q) {
      const int i = l * P + q, d = ctx->pdim[q];
      const int rcv = ctx->neighbour(r, d, -1), snd = ctx->neighbour(r, d, +1);  // coordinates go down (R1)
      PlanLQ& a = H.lq[l][q];
      a.rcv_l = same_group(ctx, r, rcv) ? rcv - ctx->first_rank : -1;
      a.snd_l = same_group(ctx, r, snd) ? snd - ctx->first_rank : -1;
      const bool bulk = a.rcv_l < 0 && bulk_pulse(ctx, q, ctx->send_size[i]);
      a.dst_x = a.rcv_l >= 0 ? ctx->x[a.rcv_l] + (size_t)ctx->remote_off[i] * W
                : bulk     ? ctx->peer_x[rcv] + (size_t)ctx->remote_off[i] * W
                           : nullptr;
      a.dst_ll = a.rcv_l >= 0 || bulk ? nullptr : ctx->xll_of(rcv) + (size_t)q * ctx->ll_stride;
      a.bulk = bulk ? &ctx->hdr_of(rcv)->bulk_x[q] : nullptr;
      a.push = a.snd_l >= 0 ? nullptr : ctx->fll_of(snd) + (size_t)q * ctx->ll_stride;
      a.remote_off = ctx->remote_off[i];
      a.atom_offset = ctx->atom_offset[i];
      a.send_size = ctx->send_size[i];
      a.recv_size = ctx->recv_size[i];
      a.wraps = ctx->cell(r, d) == 0;  // the wrapping sender adds +L_d (R25)
      a.efs = a.wraps ? (uint8_t)(3 * l + d) : (uint8_t)0xff;
    }
  }
  char* sp = ctx->d_pl_scratch;
  H.org = reinterpret_cast<uint64_t*>(sp);
  H.child = reinterpret_cast<int32_t*>(sp + so);
  H.rcls = reinterpret_cast<uint8_t*>(sp + so + sc);
  H.rmask = H.rcls + (size_t)L * cap;
  H.imask = reinterpret_cast<uint32_t*>(sp + so + sc + sr + sk + sx);
  H.xnch = xnch;
  H.xlast = reinterpret_cast<int32_t*>(sp + so + sc + sr + sk + sx + si);
  H.xlstart = H.xlast + (size_t)P * L * xnch;
  H.xccnt = H.xlstart + (size_t)P * L * xnch;
  H.bcnt = reinterpret_cast<int32_t*>(sp + so + sc + sr);
  H.boff = H.bcnt + (size_t)L * nblk * (P + 1);
  H.xcnt = reinterpret_cast<int32_t*>(sp + so + sc + sr + sk);
  H.rcnt = H.xcnt + (size_t)P * L * (P + 1);
  CK(cudaMemcpyAsync(ctx->d_pl, &H, sizeof(PlanDev), cudaMemcpyHostToDevice, st));
  CK(cudaMemsetAsync(H.child, 0xff, sizeof(int32_t) * L * cap * P, st));
  CK(cudaMemsetAsync(H.xcnt, 0, sizeof(int32_t) * (size_t)P * L * (P + 1), st));
  CK(launch_plan_count(ctx->d_pl, L, P, max_rows, max_send, st));
  const size_t ncnt = (size_t)(P * L + L) * (P + 1);
  CK(cudaMemcpyAsync(ctx->h_pl_cnt, H.xcnt, sizeof(int32_t) * ncnt, cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  if (prof) prof->lap("plan:count");
  const int32_t* xc = ctx->h_pl_cnt;
  const int32_t* rc = ctx->h_pl_cnt + (size_t)P * L * (P + 1);
  // x items: class-major (a wait only targets a lower class: deadlock-free static
  // order), then pulse, then local rank; the receives last
  int nx = 0;
  for (int c = 0; c <= P; ++c)
    for (int p = 0; p < P; ++p)
      for (int l = 0; l < L; ++l) {
        H.xoff[c][p][l] = nx;
        nx += xc[((size_t)p * L + l) * (P + 1) + c];
      }
  std::vector<XRec> recv;
  for (int p = 0; p < P; ++p)
    for (int l = 0; l < L; ++l) {
      const int r = ctx->first_rank + l;
      if (same_group(ctx, r, ctx->neighbour(r, ctx->pdim[p], +1))) continue;
      const int n = ctx->recv_size[l * P + p];
      if (bulk_pulse(ctx, p, n)) {  // one wait item for the whole pulse (build_ll_x)
        XRec x;
        memset(&x, 0, sizeof x);
        x.kind = kItemXWait;
        x.pulse = (uint8_t)p;
        x.lrank = (uint16_t)l;
        x.n_units = (uint32_t)n;
        x.cls = 0xff;
        x.epoch = ctx->epoch;
        x.bulk = &ctx->hdr_of(r)->bulk_x[p];
        recv.push_back(x);
        continue;
      }
      const int RR = std::min(kMaxItemRows, ctx->recv_mult * R);
      for (int b = 0; b < n; b += RR) {
        XRec x;
        memset(&x, 0, sizeof x);
        x.kind = kItemXRecv;
        x.pulse = (uint8_t)p;
        x.lrank = (uint16_t)l;
        x.n_units = (uint32_t)(std::min(n, b + RR) - b) * W;
        x.begin = (uint32_t)b;
        x.cls = 0xff;
        x.ll = ctx->xll_of(r) + (size_t)p * ctx->ll_stride + (size_t)b * W;
        x.xdst = ctx->x[l] + (size_t)(ctx->atom_offset[l * P + p] + b) * W;
        x.epoch = ctx->epoch;
        recv.push_back(x);
      }
    }
  const int n_send = nx;
  nx += (int)recv.size();
  // f items: roots per item (RT) the smallest size whose items all fit the co-resident
  // grid (one item per CTA), else kTreeRowsOcc; class-major, then local rank
  auto f_items = [&](int RT) {
    int n = 0;
    for (int c = 0; c <= P; ++c)
      for (int l = 0; l < L; ++l) n += (rc[l * (P + 1) + c] + RT - 1) / RT;
    return n;
  };
  int RT = 32;
  while (f_items(RT) > ctx->cap_f() && RT < kTreeRowsOcc) RT = std::min(kTreeRowsOcc, RT + 16);
  // bandwidth regime (wide variants: two item blocks in flight, so the shared memory the
  // co-resident grid was computed for holds kMaxTreeRows): fewer, larger items, two
  // passes of kTreeRowsOcc roots per thread
  const int rt_max = ctx->wide() ? ctx->tree_rows_max : kTreeRowsOcc;
  while (f_items(RT) > ctx->cap_f() && RT < rt_max) RT = std::min(rt_max, RT + 17);
  if (const char* e = getenv("HALO_TREE_ROWS")) RT = std::min(rt_max, std::max(8, atoi(e)));
  int nf = 0;
  for (int c = 0; c <= P; ++c)
    for (int l = 0; l < L; ++l) {
      H.foff[c][l] = nf;
      H.fcnt[c][l] = rc[l * (P + 1) + c];
      nf += (H.fcnt[c][l] + RT - 1) / RT;
    }
  ctx->tree_rows = RT;
  H.RT = RT;
  H.FB = ll_fblk_bytes(RT);
  ctx->h_items_x.clear();
  ctx->h_items_f.clear();
  ctx->h_xblk.clear();
  ctx->h_fblk.clear();
  ctx->gpu_n_items_x = nx;
  ctx->gpu_n_items_f = nf;
  ctx->gpu_xblk_bytes = std::max<size_t>(1, (size_t)nx * H.XB);
  ctx->gpu_fblk_bytes = std::max<size_t>(1, (size_t)nf * H.FB);
  fill_rank_dev(ctx);
  halo_status s = upload_plan(ctx, st);
  if (s != HALO_OK) return s;
  H.xblk = ctx->d_xblk;
  H.fblk = ctx->d_fblk;
  H.nx_send = n_send;
  H.nf = nf;
  H.err_host = ctx->err_dev;
#ifdef HALO_BOUNDS_CHECK
  if (getenv("HALO_BC_ITEMS")) H.nx_send = H.nf = 1;  // self-test: the plan-write checks must fire
#endif
  CK(cudaMemcpyAsync(ctx->d_pl, &H, sizeof(PlanDev), cudaMemcpyHostToDevice, st));
  if (!recv.empty()) {  // the receive items' records (no entries): straight from pinned memory
    if (ctx->h_recv_cap < recv.size()) {
      if (ctx->h_recv) CK(cudaFreeHost(ctx->h_recv));
      ctx->h_recv = nullptr;
      CK(cudaMallocHost(&ctx->h_recv, sizeof(XRec) * recv.size()));
      ctx->h_recv_cap = recv.size();
    }
    memcpy(ctx->h_recv, recv.data(), sizeof(XRec) * recv.size());
    CK(cudaMemcpy2DAsync(ctx->d_xblk + (size_t)n_send * H.XB, H.XB, ctx->h_recv, sizeof(XRec), sizeof(XRec),
                         recv.size(), cudaMemcpyHostToDevice, st));
  }
  CK(cudaMemsetAsync(H.imask, 0, sizeof(uint32_t) * nf, st));
  CK(launch_plan_write(ctx->d_pl, L, P, max_rows, max_send, st));
  ctx->n_tail_f = 0;
  if (prof) prof->lap("plan:write");
  if (getenv("HALO_PLAN_CHECK")) return plan_check(ctx, st);
  return HALO_OK;
}

// Plan layout: RankDev | PulseDev | x items | f items | LocalBase | x item blocks | f
// item blocks.  Host-built plans (h_xblk / h_fblk) go up in one DMA from a pinned
// image; a GPU-built plan (gpu_xblk_bytes > 0, kernels_plan.cu) uploads only the head
// and leaves the block areas to the kernels.
// st != null: the DMA is enqueued on st (the pinned image must then stay untouched until
// st passes it); null: synchronous.
static halo_status upload_plan(halo_ctx* ctx, cudaStream_t st) {
  const size_t a = 256;
  const bool gpu = ctx->gpu_xblk_bytes > 0;
  const size_t nr = align_up(sizeof(RankDev) * ctx->n_local, a);
  const size_t np = align_up(sizeof(PulseDev) * std::max(1, ctx->n_local * ctx->P), a);
  const size_t nx = align_up(sizeof(Item) * std::max<size_t>(1, ctx->h_items_x.size()), a);
  const size_t nf = align_up(sizeof(Item) * std::max<size_t>(1, ctx->h_items_f.size()), a);
  const size_t nlb = align_up(sizeof(LocalBase) * std::max<size_t>(1, ctx->h_lbase.size()), a);
  const size_t nxr = align_up(std::max<size_t>(1, gpu ? ctx->gpu_xblk_bytes : ctx->h_xblk.size()), a);
  const size_t ngr = align_up(std::max<size_t>(1, gpu ? ctx->gpu_fblk_bytes : ctx->h_fblk.size()), a);
  const size_t need = nr + np + nx + nf + nlb + nxr + ngr;
  if (need > ctx->plan_bytes) {  // 25% headroom: NS steps rarely grow the plan again
    if (ctx->plan && ctx->captured) {
      // a captured graph may still reference the old plan: keep it mapped, with every
      // record's epoch zeroed (a replay then refuses every item, HALO_ERR_STATE)
      CK(cudaMemset(ctx->plan, 0, ctx->plan_bytes));
      ctx->retired.push_back(ctx->plan);
    } else if (ctx->plan) {
      CK(cudaFree(ctx->plan));
    }
    ctx->plan = nullptr;
    CK(cudaMalloc(&ctx->plan, need + need / 4));
    ctx->plan_bytes = need + need / 4;
  }
  const size_t img_need = gpu ? nr + np + nx + nf + nlb : need;
  if (img_need > ctx->h_pin_bytes) {
    if (ctx->h_pin) CK(cudaFreeHost(ctx->h_pin));
    ctx->h_pin = nullptr;
    CK(cudaMallocHost(&ctx->h_pin, img_need + img_need / 4));
    ctx->h_pin_bytes = img_need + img_need / 4;
  }
  ctx->d_ranks = reinterpret_cast<RankDev*>(ctx->plan);
  ctx->d_pulses = reinterpret_cast<PulseDev*>(ctx->plan + nr);
  ctx->d_items_x = reinterpret_cast<Item*>(ctx->plan + nr + np);
  ctx->d_items_f = reinterpret_cast<Item*>(ctx->plan + nr + np + nx);
  ctx->d_lbase = reinterpret_cast<LocalBase*>(ctx->plan + nr + np + nx + nf);
  ctx->d_xblk = ctx->plan + nr + np + nx + nf + nlb;
  ctx->d_fblk = ctx->plan + nr + np + nx + nf + nlb + nxr;
  // the plan image in pinned memory, then one synchronous DMA (pageable copies of
  // the MB-sized item blocks cost ms at the NS step)
  char* img = ctx->h_pin;
  auto put = [&](char* dev, const void* src, size_t n) {
    if (n) memcpy(img + (dev - ctx->plan), src, n);
  };
  put(reinterpret_cast<char*>(ctx->d_ranks), ctx->h_ranks.data(), sizeof(RankDev) * ctx->n_local);
  if (ctx->P)
    put(reinterpret_cast<char*>(ctx->d_pulses), ctx->h_pulses.data(), sizeof(PulseDev) * ctx->n_local * ctx->P);
  put(reinterpret_cast<char*>(ctx->d_items_x), ctx->h_items_x.data(), sizeof(Item) * ctx->h_items_x.size());
  put(reinterpret_cast<char*>(ctx->d_items_f), ctx->h_items_f.data(), sizeof(Item) * ctx->h_items_f.size());
  put(reinterpret_cast<char*>(ctx->d_lbase), ctx->h_lbase.data(), sizeof(LocalBase) * ctx->h_lbase.size());
  size_t used = (size_t)(reinterpret_cast<char*>(ctx->d_lbase) - ctx->plan) + sizeof(LocalBase) * ctx->h_lbase.size();
  if (!gpu) {
    put(ctx->d_xblk, ctx->h_xblk.data(), ctx->h_xblk.size());
    put(ctx->d_fblk, ctx->h_fblk.data(), ctx->h_fblk.size());
    if (!ctx->h_fblk.empty()) used = (size_t)(ctx->d_fblk - ctx->plan) + ctx->h_fblk.size();
    else if (!ctx->h_xblk.empty()) used = (size_t)(ctx->d_xblk - ctx->plan) + ctx->h_xblk.size();
  }
  if (st) CK(cudaMemcpyAsync(ctx->plan, img, used, cudaMemcpyHostToDevice, st));
  else CK(cudaMemcpy(ctx->plan, img, used, cudaMemcpyHostToDevice));
  ctx->n_items_x = gpu ? ctx->gpu_n_items_x : (int)ctx->h_items_x.size();
  ctx->n_items_f = gpu ? ctx->gpu_n_items_f : (int)ctx->h_items_f.size();
  return HALO_OK;
}

// Sequence number of the next LL launch on `st`: by value (host mirror) unless the
// ctx has ever been captured into a graph (then 0: the kernel reads the device
// counter, which every LL launch advances).
static uint64_t next_seq(halo_ctx* ctx, cudaStream_t st, uint64_t* host, bool* capturing = nullptr) {
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  bool cap = false;
  if (cudaStreamIsCapturing(st, &cs) != cudaSuccess) {
    (void)cudaGetLastError();
    cap = true;
  }
  if (cs != cudaStreamCaptureStatusNone) cap = true;
  if (cap) ctx->captured = true;
  if (capturing) *capturing = cap;
  *host = ll_seq_next(*host);
  return ctx->captured ? 0 : *host;
}

static ExParams make_params(halo_ctx* ctx, const Item* items, int n_items, int p_lo, int p_hi) {
  ExParams P{};
  P.ranks = ctx->d_ranks;
  P.pulses = ctx->d_pulses;
  P.items = items;
  P.n_items = n_items;
  P.n_local = ctx->n_local;
  P.P = ctx->P;
  P.p_lo = p_lo;
  P.p_hi = p_hi;
  P.ctrl = ctx->ctrl;
  P.err_host = ctx->err_dev;
  P.timeout_ns = (uint64_t)(ctx->cfg.timeout_s * 1e9);
  P.flags = ctx->cfg.flags;
  P.fshift = nullptr;
  P.accumulate = 1;
  P.poll_ns = ctx->poll_ns;
  P.debug = ctx->debug;
  P.fsp_slots = (uint32_t)ctx->fsp_slots;
  P.ll_stride = ctx->ll_stride;
  P.xblk = ctx->d_xblk;
  P.fblk = ctx->d_fblk;
  P.item_rows = ctx->item_rows;
  P.tree_rows = ctx->tree_rows;
  P.ring = ll_ring(0, ctx->wide());  // (the f and fused launches set theirs)
  P.delay_rank = ctx->P ? ctx->neighbour(0, ctx->pdim[0], +1) : -1;
  P.lbase = ctx->d_lbase;
  P.plan_epoch = ctx->epoch;
  P.all_local = ctx->all_local ? 1 : 0;
  P.cap_rows = ctx->cfg.capacity;
#ifdef HALO_BOUNDS_CHECK
  // self-test of the checked build: pretend the buffers hold this many rows (the checks must fire)
  if (const char* e = getenv("HALO_BC_CAP")) P.cap_rows = std::max(1, atoi(e));
#endif
  return P;
}

static int grid_for(int n_items, int n_local, int max_blocks) {
  int g = std::min(n_items, max_blocks);
  return std::max(std::max(g, n_local), 1);
}

// Pull the set_maps results of every local rank back to the host.
// ctx->h_small (pinned 64 KiB) regions: set_maps result read-back (and the seq read-back
// after it) | reset upload | LL-area table | planes
constexpr size_t kPinResults = 0, kPinReset = 16384, kPinLLTab = 20480, kPinPlanes = 24576;
static_assert(offsetof(Ctrl, agreed_err) + sizeof(int32_t) * kMaxLocal - offsetof(Ctrl, send_size) <= kPinReset,
              "pinned result region");

static halo_status pull_ctrl(halo_ctx* ctx, cudaStream_t st, int32_t* agreed = nullptr) {
  const int L = ctx->n_local, P = ctx->P;
  // the set_maps result arrays are contiguous in Ctrl (through agreed_err): one copy
  // into pinned memory, one synchronisation
  static_assert(offsetof(Ctrl, n_indep) > offsetof(Ctrl, send_size) && offsetof(Ctrl, n_total) > offsetof(Ctrl, dep) &&
                    offsetof(Ctrl, agreed_err) > offsetof(Ctrl, n_total),
                "set_maps result block layout");
  const size_t lo = offsetof(Ctrl, send_size), hi = offsetof(Ctrl, agreed_err) + sizeof(ctx->ctrl->agreed_err);
  char* hb = ctx->h_small + kPinResults;  // pinned; viewed as a Ctrl shifted by lo
  const Ctrl& h = *reinterpret_cast<const Ctrl*>(hb - lo);
  cudaError_t e = cudaMemcpyAsync(hb, reinterpret_cast<const char*>(ctx->ctrl) + lo, hi - lo, cudaMemcpyDeviceToHost, st);
  if (e == cudaSuccess) e = cudaStreamSynchronize(st);
  if (e != cudaSuccess) return cuda_fail(ctx, e, "pull_ctrl");
  for (int l = 0; l < L; ++l) {
    for (int p = 0; p < P; ++p) {
      const int i = l * P + p;
      ctx->send_size[i] = h.send_size[l][p];
      ctx->recv_size[i] = h.recv_size[l][p];
      ctx->atom_offset[i] = h.atom_offset[l][p];
      ctx->remote_off[i] = h.remote_off[l][p];
      ctx->n_indep[i] = h.n_indep[l][p];
      ctx->dep[i] = h.dep[l][p];
    }
    ctx->n_total[l] = h.n_total[l];
    if (agreed) agreed[l] = h.agreed_err[l];
  }
  return HALO_OK;
}

// Host copy of pulse p's maps of every local rank (sizes final after the handshake).
static halo_status pull_maps(halo_ctx* ctx, int p, cudaStream_t st) {
  for (int l = 0; l < ctx->n_local; ++l) {
    const int n = ctx->send_size[l * ctx->P + p];
    auto& m = ctx->h_maps[l][p];
    m.resize(n);
    if (n)
      CK(cudaMemcpyAsync(m.data(), ctx->maps_of_local(l) + (size_t)p * ctx->map_stride, sizeof(int32_t) * n,
                         cudaMemcpyDeviceToHost, st));
  }
  CK(cudaStreamSynchronize(st));
  return HALO_OK;
}

// Copy-engine plan (HALO_F_CE_PATH, kernels_ce.cu): per (pulse, local rank) the
// x gather entry (skipped for a contiguous unshifted map: the CE reads x
// directly), the x copy to the receiver, the force-slice copy to the x-sender
// (contiguous by construction, R12) and the scatter-add entry.
static halo_status build_ce(halo_ctx* ctx) {
  const int L = ctx->n_local, P = ctx->P, W = ctx->W;
  ctx->h_ce_pack.assign((size_t)P * L, CeEnt{});
  ctx->h_ce_unpack.assign((size_t)P * L, CeEnt{});
  ctx->ce_copy_x.assign((size_t)P * L, halo_ctx::CeCopy{nullptr, nullptr, 0});
  ctx->ce_copy_f.assign((size_t)P * L, halo_ctx::CeCopy{nullptr, nullptr, 0});
  ctx->ce_pack_rows.assign(P, 0);
  ctx->ce_unpack_rows.assign(P, 0);
  size_t stage_rows = 0;
  for (int p = 0; p < P; ++p)
    for (int l = 0; l < L; ++l) stage_rows += ctx->send_size[l * P + p];
  const size_t need_stage = std::max<size_t>(stage_rows * W * sizeof(float), 256);
  if (need_stage > ctx->stage_bytes) {
    if (ctx->d_stage) CK(cudaFree(ctx->d_stage));
    ctx->d_stage = nullptr;
    CK(cudaMalloc(&ctx->d_stage, need_stage));
    ctx->stage_bytes = need_stage;
  }
  float* stage = ctx->d_stage;
  for (int p = 0; p < P; ++p)
    for (int l = 0; l < L; ++l) {
      const int i = l * P + p, k = p * L + l;
      const PulseDev& pd = ctx->h_pulses[i];
      const auto& m = ctx->h_maps[l][p];
      const int n = (int)m.size();
      bool contiguous = n > 0;
      for (int j = 1; contiguous && j < n; ++j) contiguous = m[j] == m[0] + j;
      CeEnt& e = ctx->h_ce_pack[k];
      e.map = pd.map;
      e.src = ctx->x[l];
      e.dst = stage;
      e.n = n;
      e.pack = (n > 0 && (pd.has_shift || !contiguous)) ? 1 : 0;
      e.has_shift = pd.has_shift;
      e.dim = pd.dim;
      for (int c = 0; c < 3; ++c) e.shift[c] = pd.shift[c];
      if (e.pack) ctx->ce_pack_rows[p] = std::max(ctx->ce_pack_rows[p], n);
      ctx->ce_copy_x[k] = {pd.x_dst, e.pack ? (const void*)stage : (const void*)(ctx->x[l] + (size_t)(n ? m[0] : 0) * W),
                           (size_t)n * W * sizeof(float)};
      stage += (size_t)n * W;
      CeEnt& u = ctx->h_ce_unpack[k];
      u = e;
      u.src = pd.fbuf_own;
      u.dst = ctx->f[l];
      u.pack = 0;
      ctx->ce_unpack_rows[p] = std::max(ctx->ce_unpack_rows[p], n);
      // force slice of pulse p (this rank's receive range) -> the x-sender's force buffer
      ctx->ce_copy_f[k] = {pd.fbuf_dst, ctx->f[l] + (size_t)pd.atom_offset * W, (size_t)pd.recv_size * W * sizeof(float)};
    }
  const size_t need = 2 * sizeof(CeEnt) * std::max<size_t>(1, (size_t)P * L);
  if (need > ctx->ce_bytes) {
    if (ctx->d_ce) CK(cudaFree(ctx->d_ce));
    ctx->d_ce = nullptr;
    CK(cudaMalloc(&ctx->d_ce, need));
    ctx->ce_bytes = need;
  }
  if (P) {
    CK(cudaMemcpy(ctx->d_ce, ctx->h_ce_pack.data(), sizeof(CeEnt) * P * L, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(ctx->d_ce + (size_t)P * L, ctx->h_ce_unpack.data(), sizeof(CeEnt) * P * L, cudaMemcpyHostToDevice));
  }
  return HALO_OK;
}

static CeSyncParams ce_sync_params(halo_ctx* ctx, int kind, int p, bool publish) {
  CeSyncParams S{};
  S.seq_slot = kind == 0 ? &ctx->ctrl->seq_x : &ctx->ctrl->seq_f;
  for (int l = 0; l < ctx->n_local; ++l) {
    const PulseDev& pd = ctx->h_pulses[l * ctx->P + p];
    ScratchHdr* own = ctx->hdr_of(ctx->first_rank + l);
    S.dst[l] = kind == 0 ? pd.flag_x_dst : pd.flag_f_dst;
    S.own[l] = kind == 0 ? &own->flag_x[p] : &own->flag_f[p];
  }
  S.n_local = ctx->n_local;
  S.publish = publish ? 1 : 0;
  S.kind = kind;
  S.pulse = p;
  S.err_host = ctx->err_dev;
  S.timeout_ns = (uint64_t)(ctx->cfg.timeout_s * 1e9);
  return S;
}

// HALO_CE_PROFILE: one timed event pair around an operation of the CE path.
struct CeMark {
  halo_ctx* ctx;
  cudaStream_t st;
  cudaEvent_t a = nullptr;
  const char* name;
  CeMark(halo_ctx* c, cudaStream_t s, const char* n) : ctx(c), st(s), name(n) {
    if (!ctx->ce_prof.on) return;
    (void)cudaEventCreate(&a);
    (void)cudaEventRecord(a, st);
  }
  ~CeMark() {
    if (!ctx->ce_prof.on) return;
    cudaEvent_t b = nullptr;
    (void)cudaEventCreate(&b);
    (void)cudaEventRecord(b, st);
    ctx->ce_prof.pend.push_back({a, b});
    ctx->ce_prof.names.push_back(name);
  }
};
static void ce_prof_collect(halo_ctx* ctx) {
  auto& P = ctx->ce_prof;
  if (!P.on || P.pend.empty()) return;
  (void)cudaDeviceSynchronize();
  for (size_t i = 0; i < P.pend.size(); ++i) {
    float ms = 0.f;
    (void)cudaEventElapsedTime(&ms, P.pend[i].first, P.pend[i].second);
    (void)cudaEventDestroy(P.pend[i].first);
    (void)cudaEventDestroy(P.pend[i].second);
    size_t k = 0;
    while (k < P.agg_names.size() && P.agg_names[k] != P.names[i]) ++k;
    if (k == P.agg_names.size()) {
      P.agg_names.push_back(P.names[i]);
      P.sum.push_back(0.0);
      P.cnt.push_back(0);
    }
    P.sum[k] += ms * 1e3;
    P.cnt[k] += 1;
  }
  P.pend.clear();
  P.names.clear();
}

// x over the copy engine: per pulse ascending, gather -> CE copy -> flag + wait.
static halo_status ce_exchange_x(halo_ctx* ctx, cudaStream_t st) {
  const int L = ctx->n_local, P = ctx->P;
  for (int p = 0; p < P; ++p) {
    {
      CeMark m(ctx, st, "x pack");
      CK(launch_ce_pack(ctx->W, ctx->d_ce + (size_t)p * L, L, ctx->ce_pack_rows[p], st));
    }
    {
      CeMark m(ctx, st, "x copy");
      for (int l = 0; l < L; ++l) {
        const halo_ctx::CeCopy& c = ctx->ce_copy_x[(size_t)p * L + l];
        if (c.bytes) CK(cudaMemcpyAsync(c.dst, c.src, c.bytes, cudaMemcpyDefault, st));
      }
    }
    CeMark m(ctx, st, "x sync");
    CK(launch_ce_sync(ce_sync_params(ctx, 0, p, p == P - 1), st));
  }
  return HALO_OK;
}

// f over the copy engine: per pulse descending, CE copy of the halo slice ->
// flag + wait -> ordered scatter-add (+ shift forces).
static halo_status ce_exchange_f(halo_ctx* ctx, double* fshift, int accumulate, cudaStream_t st) {
  const int L = ctx->n_local, P = ctx->P;
  for (int p = P - 1; p >= 0; --p) {
    {
      CeMark m(ctx, st, "f copy");
      for (int l = 0; l < L; ++l) {
        const halo_ctx::CeCopy& c = ctx->ce_copy_f[(size_t)p * L + l];
        if (c.bytes) CK(cudaMemcpyAsync(c.dst, c.src, c.bytes, cudaMemcpyDefault, st));
      }
    }
    {
      CeMark m(ctx, st, "f sync");
      CK(launch_ce_sync(ce_sync_params(ctx, 1, p, p == 0), st));
    }
    CeMark m(ctx, st, "f unpack");
    CK(launch_ce_unpack(ctx->W, ctx->d_ce + (size_t)P * L + (size_t)p * L, L, ctx->ce_unpack_rows[p], fshift,
                        accumulate, st));
  }
  if (ctx->ce_prof.on && ctx->ce_prof.pend.size() > 4096) ce_prof_collect(ctx);
  return HALO_OK;
}

// Shared driver of halo_set_maps / halo_set_maps_explicit.
// HALO_PROFILE=1: host wall time of the set_maps phases on stderr (NS-step cost study).

static halo_status set_maps_impl(halo_ctx* ctx, const int* n_home, const int* send_sizes, const int* const* maps,
                                 cudaStream_t st) {
  if (!ctx->peers_ready) return fail(ctx, HALO_ERR_STATE, "register buffers and import peers first");
  CK(cudaSetDevice(ctx->cfg.device));
  // exchanges queued on any stream of this device read the plan rewritten below
  CK(cudaDeviceSynchronize());
  halo_status s = check_err_word(ctx);
  if (s != HALO_OK) return s;
  PhaseTimer prof;
  ctx->pme_ready = false;  // the home counts change: halo_pme_setup again
  const int L = ctx->n_local, P = ctx->P, W = ctx->W;
  if (ctx->auto_tr) {  // the per-pulse exchanges below run the LL kernels; the vote decides the epoch's transport
    ctx->ll = true;
    ctx->ce = false;
  }
  ctx->maps_ready = false;
  ctx->x_done = false;
  ctx->epoch++;
  ctx->n_home.assign(n_home, n_home + L);
  ctx->n_total = ctx->n_home;
  ctx->send_size.assign(L * P, 0);
  ctx->recv_size.assign(L * P, 0);
  ctx->atom_offset.assign(L * P, 0);
  ctx->remote_off.assign(L * P, 0);
  ctx->n_indep.assign(L * P, 0);
  ctx->dep.assign(L * P, 0u);
  ctx->h_pulses.assign(std::max(1, L * P), PulseDev{});
  ctx->h_maps.assign(L, std::vector<std::vector<int32_t>>(P));
  int local_err = 0;
  for (int l = 0; l < L; ++l)
    if (n_home[l] < 0 || n_home[l] > ctx->cfg.capacity) local_err |= kErrCapacity;

  // reset device-side set_maps state
  {
    int32_t zero[kMaxLocal * kMaxP] = {0};
    int32_t nt[kMaxLocal] = {0}, errs[kMaxLocal] = {0};
    for (int l = 0; l < L; ++l) {
      nt[l] = std::min(std::max(n_home[l], 0), ctx->cfg.capacity);
      errs[l] = local_err;
    }
    (void)zero;
    // the result block [send_size .. n_total) zeroed, then n_total and err from pinned
    // memory (stream-ordered before the first select: no synchronisation)
    CK(cudaMemsetAsync(ctx->ctrl->send_size, 0, offsetof(Ctrl, n_total) - offsetof(Ctrl, send_size), st));
    static_assert(offsetof(Ctrl, err) == offsetof(Ctrl, n_total) + sizeof(int32_t) * kMaxLocal, "n_total | err");
    char* pin = ctx->h_small + kPinReset;
    memcpy(pin, nt, sizeof nt);
    memcpy(pin + sizeof nt, errs, sizeof errs);
    CK(cudaMemcpyAsync(ctx->ctrl->n_total, pin, sizeof nt + sizeof errs, cudaMemcpyHostToDevice, st));
    for (int l = 0; l < L; ++l) ctx->n_total[l] = nt[l];
  }
  ctx->n_home.assign(ctx->n_total.begin(), ctx->n_total.end());
  // LL areas zeroed every NS epoch (ll_seq_next): no peer writes them before the
  // pulse-0 handshake below, which this stream reaches only after the memset
  if (ctx->ll || ctx->auto_tr) {
    uint64_t** tab = reinterpret_cast<uint64_t**>(ctx->h_small + kPinLLTab);  // pinned
    for (int l = 0; l < L; ++l) tab[l] = ctx->xll_of(ctx->first_rank + l);
    CK(cudaMemcpyAsync(ctx->d_small + 16384, tab, sizeof(uint64_t*) * L, cudaMemcpyHostToDevice, st));
    CK(launch_zero_ll(reinterpret_cast<uint64_t* const*>(ctx->d_small + 16384), 2 * (size_t)P * ctx->ll_stride, L, st));
    for (int l = 0; l < L && ctx->bulk_rows > 0; ++l)  // bulk x counters (0 between launches; reset after an aborted one)
      CK(cudaMemsetAsync(ctx->hdr_of(ctx->first_rank + l)->bulk_x, 0, sizeof(ScratchHdr::bulk_x), st));
  }
  fill_rank_dev(ctx);
  // ranks/pulse tables are needed by the select/depmask kernels already
  ctx->h_items_x.clear();
  ctx->h_items_f.clear();
  ctx->h_fblk.clear();  // the last epoch's force blocks: not re-uploaded with every pulse's x plan
  ctx->h_xblk.clear();
  ctx->gpu_xblk_bytes = ctx->gpu_fblk_bytes = 0;
  if ((s = upload_plan(ctx, st)) != HALO_OK) return s;  // (the next upload follows a synchronisation)

  const uint64_t timeout_ns = (uint64_t)(ctx->cfg.timeout_s * 1e9);
  // static planes of the GPU map builder (R2, R3): b_d[c_d] of every dim, and b_d[c_d + 1]
  char* sm = ctx->d_small;
  if (!maps) {
    std::vector<double> blo(3 * L), bhi(3 * L);
    for (int l = 0; l < L; ++l)
      for (int dd = 0; dd < 3; ++dd) {
        blo[3 * l + dd] = ctx->plane(dd, ctx->cell(ctx->first_rank + l, dd));
        bhi[3 * l + dd] = ctx->plane(dd, ctx->cell(ctx->first_rank + l, dd) + 1);
      }
    double* pin = reinterpret_cast<double*>(ctx->h_small + kPinPlanes);  // pinned: [blo | bhi], 4 KiB each
    memcpy(pin, blo.data(), sizeof(double) * 3 * L);
    memcpy(pin + 512, bhi.data(), sizeof(double) * 3 * L);
    CK(cudaMemcpyAsync(sm + 4096, pin, sizeof(double) * 3 * L, cudaMemcpyHostToDevice, st));
    CK(cudaMemcpyAsync(sm + 8192, pin + 512, sizeof(double) * 3 * L, cudaMemcpyHostToDevice, st));
  }
  // Per pulse, all stream-ordered on the device (no host round trip): select (fp64
  // predicate + compaction) -> handshake (sizes / offsets with the neighbours) ->
  // dependency masks -> the pulse's coordinate exchange (pulse p+1 selects among
  // and forwards these rows).  The explicit-map test entry validates on the host.
  for (int p = 0; p < P; ++p) {
    const int d = ctx->pdim[p], k = ctx->pk[p];
    if (maps) {
      // explicit maps (test entry): validate on the host and upload
      int errs_now = 0;
      for (int l = 0; l < L; ++l) {
        const int i = l * P + p;
        const int n = send_sizes[i];
        const int* m = maps[i];
        bool ok = n >= 0 && n <= ctx->cfg.capacity && (n == 0 || m != nullptr);
        for (int j = 0; ok && j < n; ++j) ok = m[j] >= 0 && m[j] < ctx->n_total[l] && (j == 0 || m[j] > m[j - 1]);
        if (!ok) { errs_now |= kErrMap; continue; }
        if (n) CK(cudaMemcpyAsync(ctx->maps_of_local(l) + (size_t)p * ctx->map_stride, m, sizeof(int) * n,
                                  cudaMemcpyHostToDevice, st));
        int32_t nn = n;
        CK(cudaMemcpyAsync(&ctx->ctrl->send_size[l][p], &nn, sizeof nn, cudaMemcpyHostToDevice, st));
        CK(cudaStreamSynchronize(st));
      }
      if (errs_now) {
        for (int l = 0; l < L; ++l) {
          int32_t e = errs_now;
          CK(cudaMemcpyAsync(&ctx->ctrl->err[l], &e, sizeof e, cudaMemcpyHostToDevice, st));
          CK(cudaStreamSynchronize(st));
        }
      }
    } else {
      SelParams S{};
      S.ranks = ctx->d_ranks;
      S.ctrl = ctx->ctrl;
      S.p = p;
      S.dim = d;
      S.rc = (double)ctx->cfg.cutoff;
      S.cand = nullptr;  // from the device-side handshake results
      S.kfirst = k == 0;
      S.b_lo = reinterpret_cast<const double*>(sm + 4096);  // [n_local][3]: b_d[c_d]
      const bool check = (p == 0) && !(ctx->cfg.flags & HALO_F_NO_HOME_CHECK);
      S.home_lo = check ? reinterpret_cast<const double*>(sm + 4096) : nullptr;
      S.home_hi = check ? reinterpret_cast<const double*>(sm + 8192) : nullptr;
      S.b_up = (ctx->cfg.flags & HALO_F_ROUNDED_ZONES) ? reinterpret_cast<const double*>(sm + 8192) : nullptr;
      S.rc2 = S.rc * S.rc;
      S.decomposed_mask = (ctx->cfg.grid[0] > 1) | ((ctx->cfg.grid[1] > 1) << 1) | ((ctx->cfg.grid[2] > 1) << 2);
      S.map_stride = (int)ctx->map_stride;
      S.layout = W;
      S.epoch = ctx->epoch;
      S.err_host = ctx->err_dev;
      S.timeout_ns = timeout_ns;
      S.max_chunks = (ctx->cfg.capacity + 1023) / 1024;
      S.sel_cnt = ctx->d_selcnt;
      for (int l = 0; l < L; ++l) {
        const int r = ctx->first_rank + l;
        for (int q = 0; q < p; ++q)
          if (!ctx->is_local(ctx->neighbour(r, ctx->pdim[q], +1))) S.wait_mask[l] |= 1u << q;
      }
      CK(launch_select(S, L, st));
    }
    // handshake with the neighbours (device flags)
    HsParams H{};
    H.ctrl = ctx->ctrl;
    H.p = p;
    H.epoch = ctx->epoch;
    H.capacity = ctx->cfg.capacity;
    H.n_local = L;
    H.err_host = ctx->err_dev;
    H.timeout_ns = timeout_ns;
    for (int l = 0; l < L; ++l) {
      const int r = ctx->first_rank + l;
      H.own[l] = ctx->hdr_of(r);
      H.size_dst[l] = &ctx->hdr_of(ctx->neighbour(r, d, -1))->meta_size[p];
      H.off_dst[l] = &ctx->hdr_of(ctx->neighbour(r, d, +1))->meta_off[p];
      if (!ctx->is_local(ctx->neighbour(r, d, -1))) H.sys_mask |= 1u << l;
      if (!ctx->is_local(ctx->neighbour(r, d, +1))) H.sys_mask |= 1u << (16 + l);
    }
    CK(launch_handshake(H, st));  // (dependency masks: in k_ns_x below)
    if (maps) {  // the next pulse's host validation needs n_total
      if ((s = pull_ctrl(ctx, st)) != HALO_OK) return s;
      if ((s = check_err_word(ctx)) != HALO_OK) return s;
    }
    // this pulse's coordinates now: pulse p+1 selects among and forwards them
    NsXParams NX{};
    NX.ranks = ctx->d_ranks;
    NX.ctrl = ctx->ctrl;
    NX.p = p;
    NX.dim = d;
    NX.map_stride = (int)ctx->map_stride;
    NX.n_local = L;
    NX.epoch = ctx->epoch;
    for (int l = 0; l < L; ++l) {
      const int r = ctx->first_rank + l, lower = ctx->neighbour(r, d, -1);  // coordinates go down (R1)
      NX.dst_x[l] = ctx->peer_x[lower];
      NX.flag_dst[l] = ctx->is_local(lower) ? nullptr : &ctx->hdr_of(lower)->ns_x[p];
      NX.has_shift[l] = ctx->cell(r, d) == 0;  // the wrapping sender adds +L_d (R25)
      NX.shift[l] = ctx->cfg.box[d];
      for (int q = 0; q < p; ++q)
        if (!ctx->is_local(ctx->neighbour(r, ctx->pdim[q], +1))) NX.wait_mask[l] |= 1u << q;
    }
    NX.err_host = ctx->err_dev;
    NX.timeout_ns = timeout_ns;
    NX.cap = ctx->cfg.capacity;
#ifdef HALO_BOUNDS_CHECK
    if (const char* e = getenv("HALO_BC_NS")) NX.cap = std::max(1, atoi(e));  // self-test: the NS checks must fire
#endif
    CK(launch_ns_x(NX, W, ctx->cfg.capacity, st));
    prof.lap("pulse");
  }
  {  // rows from other processes: in x before set_maps returns (the caller may read them)
    NsWaitParams NW{};
    NW.n_local = L;
    NW.epoch = ctx->epoch;
    NW.err_host = ctx->err_dev;
    NW.timeout_ns = timeout_ns;
    bool any = false;
    for (int l = 0; l < L; ++l) {
      const int r = ctx->first_rank + l;
      NW.own[l] = ctx->hdr_of(r);
      for (int q = 0; q < P; ++q)
        if (!ctx->is_local(ctx->neighbour(r, ctx->pdim[q], +1))) NW.mask[l] |= 1u << q;
      any |= NW.mask[l] != 0;
    }
    if (any) CK(launch_ns_wait(NW, st));
  }
  // error agreement + votes over all ranks, then ONE read-back of every result
  StatusParams SP{};
  SP.ctrl = ctx->ctrl;
  SP.epoch = ctx->epoch;
  SP.nranks = ctx->nranks;
  SP.n_local = L;
  SP.first_rank = ctx->first_rank;
  for (int l = 0; l < L; ++l) SP.own[l] = ctx->hdr_of(ctx->first_rank + l);
  for (int r = 0; r < ctx->nranks; ++r) SP.all[r] = ctx->hdr_of(r);
  SP.all_local = ctx->nranks == ctx->n_local;
  SP.err_host = ctx->err_dev;
  SP.timeout_ns = timeout_ns;
  SP.vote = 1;
  SP.P = P;
  SP.W = W;
  SP.auto_tr = ctx->auto_tr ? 1 : 0;
  SP.ce_bytes = ctx->auto_ce_bytes;
  if (const char* e = getenv("HALO_AUTO_CE_BYTES")) SP.ce_bytes = (uint64_t)std::max(0LL, atoll(e));  // per NS step
  SP.rows_fixed = ctx->item_rows_fixed ? ctx->item_rows : 0;
  // the CTA budget the item size is voted for: the same number in every process (the f grid
  // of the larger-occupancy variant: the hop-group-local one's 4 CTAs per SM, not the 3 of the
  // variant with LL paths, HALO_F_MIN_BLOCKS — C3 keeps R = 64 rows on 1 GPU)
  SP.ctas = std::max(1, std::min(ctx->max_x, std::max(ctx->max_f, ctx->max_f_loc)));
  CK(launch_status(SP, st));
  int32_t agreed[kMaxLocal];
  if ((s = pull_ctrl(ctx, st, agreed)) != HALO_OK) return s;
  if ((s = check_err_word(ctx)) != HALO_OK) return s;
  prof.lap("sizes");
  int any = 0;
  for (int l = 0; l < L; ++l) any |= agreed[l];
  if (any & kErrCapacity) return fail(ctx, HALO_ERR_CAPACITY, "n_home + received rows exceed capacity on some rank");
  if (any & kErrGeometry) return fail(ctx, HALO_ERR_GEOMETRY, "a home atom lies outside its rank's cell");
  if (any & kErrMap) return fail(ctx, HALO_ERR_ARG, "invalid explicit map on some rank");
  if (ctx->auto_tr && (any & kVoteCE)) {
    ctx->ll = false;
    ctx->ce = true;
  }
  {  // the largest work-item size any rank voted for
    const uint32_t rv = ((uint32_t)any & kVoteRowsMask) / (uint32_t)kVoteRows;
    if (rv == 0) return fail(ctx, HALO_ERR_STATE, "work-item size vote missing");
    ctx->item_rows = kMinItemRows << (31 - __builtin_clz(rv));
  }
  prof.lap("status");
  // final plan: all pulses
  for (int l = 0; l < L; ++l)
    for (int p = 0; p < P; ++p) fill_pulse_dev(ctx, l, p);
  bool gpu_built = false;
  ctx->gpu_xblk_bytes = ctx->gpu_fblk_bytes = 0;
  ctx->all_local = ctx->ll && !getenv("HALO_NO_LOCAL_VARIANT");
  for (int l = 0; l < L && ctx->all_local; ++l)
    for (int q = 0; q < P; ++q) {
      const int r = ctx->first_rank + l;
      if (!same_group(ctx, r, ctx->neighbour(r, ctx->pdim[q], -1)) || !same_group(ctx, r, ctx->neighbour(r, ctx->pdim[q], +1)))
        ctx->all_local = false;
    }
  if (ctx->ll) {
    fill_lbase(ctx);
    if (ctx->gpu_plan && P <= 3) {  // the plan built on the device from the device-resident maps
      s = build_ll_plan_gpu(ctx, st, &prof);
      if (s == HALO_OK) gpu_built = true;
      else if (s != HALO_ERR_UNSUPPORTED) return s;
      else ctx->gpu_xblk_bytes = ctx->gpu_fblk_bytes = 0;
    }
  }
  if (!gpu_built) {  // host builders: every map on the host
    for (int p = 0; p < P; ++p)
      if ((s = pull_maps(ctx, p, st)) != HALO_OK) return s;
    prof.lap("pull maps");
    if (ctx->ll) {
      build_ll_x(ctx, 0, P);
      prof.lap("x plan");
      if ((s = build_ll_f(ctx, &prof)) != HALO_OK) return s;
      prof.lap("f plan");
    } else {
      ctx->h_xblk.clear();
      ctx->h_fblk.clear();
      build_x_items(ctx, 0, P);
      build_f_items(ctx);
    }
    fill_rank_dev(ctx);
    if ((s = upload_plan(ctx)) != HALO_OK) return s;
    prof.lap("upload");
  }
  if (ctx->ce && (s = build_ce(ctx)) != HALO_OK) return s;
  ctx->l2win = cudaAccessPolicyWindow{};
  if ((ctx->cfg.flags & HALO_F_L2_PERSIST) && ctx->ll) {
    // the item blocks (records, map slices, task records) are re-read every step
    // and change only here: keep them in the persisting L2 carve-out
    int dev = ctx->cfg.device, max_win = 0, max_persist = 0;
    CK(cudaDeviceGetAttribute(&max_win, cudaDevAttrMaxAccessPolicyWindowSize, dev));
    CK(cudaDeviceGetAttribute(&max_persist, cudaDevAttrMaxPersistingL2CacheSize, dev));
    const size_t bytes = std::min(ctx->plan_bytes, (size_t)std::min(max_win, max_persist));
    size_t cur = 0;
    CK(cudaDeviceGetLimit(&cur, cudaLimitPersistingL2CacheSize));
    if (cur < bytes) CK(cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, bytes));
    ctx->l2win.base_ptr = ctx->plan;
    ctx->l2win.num_bytes = bytes;
    ctx->l2win.hitRatio = 1.0f;
    ctx->l2win.hitProp = cudaAccessPropertyPersisting;
    ctx->l2win.missProp = cudaAccessPropertyStreaming;
  }
  // the LL launches take their sequence numbers by value from a host mirror: resync it
  // with the device counters (the paper / copy-engine launches advance those too)
  uint64_t* seqs = reinterpret_cast<uint64_t*>(ctx->h_small);  // pinned; seq_x | seq_f adjacent
  static_assert(offsetof(Ctrl, seq_f) == offsetof(Ctrl, seq_x) + sizeof(uint64_t), "seq_x | seq_f");
  CK(cudaMemcpyAsync(seqs, &ctx->ctrl->seq_x, 2 * sizeof(uint64_t), cudaMemcpyDeviceToHost, st));
  // the fused launch's per-rank halo counters count from here (the per-pulse x
  // launches above counted too)
  CK(cudaMemsetAsync(&ctx->ctrl->xf_cnt, 0, sizeof(uint32_t), st));
  if (ctx->bulk_rows > 0) CK(cudaMemsetAsync(ctx->ctrl->bulk_rows, 0, sizeof(Ctrl::bulk_rows), st));
  CK(cudaStreamSynchronize(st));
  ctx->seq_host_x = seqs[0];
  ctx->seq_host_f = seqs[1];
  prof.lap("plan");
  prof.print(ctx->first_rank);
  if (prof.on)
    fprintf(stderr, "[halo_profile rank %d] items x %d f %d, grid caps x %d f %d xf %d (local variants: %d), R %d RT %d\n",
            ctx->first_rank, ctx->gpu_n_items_x ? ctx->gpu_n_items_x : (int)ctx->h_items_x.size(),
            ctx->gpu_n_items_f ? ctx->gpu_n_items_f : (int)ctx->h_items_f.size(), ctx->cap_x(), ctx->cap_f(),
            ctx->cap_xf(), ctx->loc() ? 1 : 0, ctx->item_rows, ctx->tree_rows);
  ctx->maps_ready = true;
  ctx->x_done = true;  // set_maps exchanged every pulse's coordinates
  return HALO_OK;
}

extern "C" {

halo_status halo_set_maps(halo_ctx* ctx, const int* n_home, void* stream) {
  if (!ctx || !n_home) return HALO_ERR_ARG;
  return set_maps_impl(ctx, n_home, nullptr, nullptr, (cudaStream_t)stream);
}

halo_status halo_set_maps_explicit(halo_ctx* ctx, const int* n_home, const int* send_sizes, const int* const* maps,
                                   void* stream) {
  if (!ctx || !n_home || (ctx->P > 0 && (!send_sizes || !maps))) return HALO_ERR_ARG;
  return set_maps_impl(ctx, n_home, send_sizes, maps, (cudaStream_t)stream);
}

// NS-step redistribution (kernels_ns.cu).
halo_status halo_migrate(halo_ctx* ctx, const int* n_home_in, int32_t* const* gid, float* const* v, int* n_home_out,
                         void* stream) {
  if (!ctx || !n_home_in || !gid || !n_home_out) return HALO_ERR_ARG;
  if (!ctx->peers_ready) return fail(ctx, HALO_ERR_STATE, "register buffers and import peers first");
  const int L = ctx->n_local, W = ctx->W;
  const bool has_v = v != nullptr;
  for (int l = 0; l < L; ++l) {
    if (!gid[l] || (has_v && !v[l])) return fail(ctx, HALO_ERR_ARG, "NULL gid / v array");
    if (n_home_in[l] < 0 || n_home_in[l] > ctx->cfg.capacity) return fail(ctx, HALO_ERR_ARG, "n_home out of range");
  }
  CK(cudaSetDevice(ctx->cfg.device));
  halo_status s = check_err_word(ctx);
  if (s != HALO_OK) return s;
  cudaStream_t st = (cudaStream_t)stream;
  ctx->maps_ready = false;
  ctx->x_done = false;
  ctx->pme_ready = false;
  ctx->epoch++;
  // the home rows move: a graph captured with the current plan must not run it again
  if (ctx->captured && ctx->plan) CK(cudaMemsetAsync(ctx->plan, 0, ctx->plan_bytes, st));
  // stencil of every local rank: the distinct ranks of cells c + delta (R30)
  std::vector<MigRank> mr(L);
  for (int l = 0; l < L; ++l) {
    MigRank& R = mr[l];
    memset(&R, 0, sizeof R);
    const int r = ctx->first_rank + l;
    R.x = ctx->x[l];
    R.gid = gid[l];
    R.v = has_v ? v[l] : nullptr;
    R.stage_out = ctx->scratch[l] + ctx->mig_off;
    R.stage_in = ctx->scratch[l] + ctx->mig_off + ctx->mig_stage;
    R.hdr = ctx->hdr_of(r);
    R.rank = r;
    R.n_home = n_home_in[l];
    const int* g = ctx->cfg.grid;
    for (int dx = -1; dx <= 1; ++dx)
      for (int dy = -1; dy <= 1; ++dy)
        for (int dz = -1; dz <= 1; ++dz) {
          const int cx = ((ctx->cell(r, 0) + dx) % g[0] + g[0]) % g[0];
          const int cy = ((ctx->cell(r, 1) + dy) % g[1] + g[1]) % g[1];
          const int cz = ((ctx->cell(r, 2) + dz) % g[2] + g[2]) % g[2];
          const int nb = ctx->rank_of(cx, cy, cz);
          bool seen = false;
          for (int k = 0; k < R.n_nb; ++k) seen |= R.nb_rank[k] == nb;
          if (seen) continue;
          R.nb_rank[R.n_nb] = nb;
          R.nb_hdr[R.n_nb] = ctx->hdr_of(nb);
          R.nb_stage[R.n_nb] = ctx->peer_scratch[nb] + ctx->mig_off;
          R.n_nb++;
        }
  }
  double planes[3 * (kMaxRanks + 1)] = {0};
  for (int d = 0; d < 3; ++d)
    for (int k = 0; k <= ctx->cfg.grid[d]; ++k) planes[d * (kMaxRanks + 1) + k] = ctx->plane(d, k);
  CK(cudaMemcpyAsync(ctx->d_mig, mr.data(), sizeof(MigRank) * L, cudaMemcpyHostToDevice, st));
  CK(cudaMemcpyAsync(ctx->d_planes, planes, sizeof planes, cudaMemcpyHostToDevice, st));
  CK(cudaMemsetAsync(ctx->d_migctrl, 0, sizeof(MigCtrl), st));
  MigParams M{};
  M.r = ctx->d_mig;
  M.ctrl = ctx->ctrl;
  M.planes = ctx->d_planes;
  for (int d = 0; d < 3; ++d) {
    M.grid[d] = ctx->cfg.grid[d];
    M.box[d] = ctx->cfg.box[d];
  }
  M.n_local = L;
  M.layout = W;
  M.has_v = has_v ? 1 : 0;
  M.capacity = ctx->cfg.capacity;
  M.epoch = ctx->epoch;
  M.err_host = ctx->err_dev;
  M.timeout_ns = (uint64_t)(ctx->cfg.timeout_s * 1e9);
  CK(launch_migrate(M, ctx->d_migctrl, ctx->cfg.capacity, 0, st));
  // error agreement over all ranks (as set_maps), before any row moves
  StatusParams SP{};
  SP.ctrl = ctx->ctrl;
  SP.epoch = ctx->epoch;
  SP.nranks = ctx->nranks;
  SP.n_local = L;
  SP.first_rank = ctx->first_rank;
  for (int l = 0; l < L; ++l) SP.own[l] = ctx->hdr_of(ctx->first_rank + l);
  for (int r = 0; r < ctx->nranks; ++r) SP.all[r] = ctx->hdr_of(r);
  SP.all_local = ctx->nranks == ctx->n_local;
  SP.err_host = ctx->err_dev;
  SP.timeout_ns = M.timeout_ns;
  CK(launch_status(SP, st));
  CK(launch_migrate(M, ctx->d_migctrl, ctx->cfg.capacity, 1, st));
  int32_t agreed[kMaxLocal];
  int32_t in_off[kMaxLocal][kStencil + 1];  // (MigCtrl is large: copy only the row counts)
  CK(cudaMemcpyAsync(agreed, ctx->ctrl->agreed_err, sizeof agreed, cudaMemcpyDeviceToHost, st));
  CK(cudaMemcpyAsync(in_off, ctx->d_migctrl->in_off, sizeof in_off, cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  if ((s = check_err_word(ctx)) != HALO_OK) return s;
  int any = 0;
  for (int l = 0; l < L; ++l) any |= agreed[l];
  if (any & kErrGeometry)
    return fail(ctx, HALO_ERR_GEOMETRY, "an atom moved more than one cell (or a box length) since the last NS step");
  if (any & kErrCapacity) return fail(ctx, HALO_ERR_CAPACITY, "a rank would hold more home rows than capacity");
  if (any & kErrMap) return fail(ctx, HALO_ERR_ARG, "gid rows are not strictly ascending on some rank");
  for (int l = 0; l < L; ++l) n_home_out[l] = in_off[l][mr[l].n_nb];
  return HALO_OK;
}

// ------------------------------------------------------------ floor probe area
halo_status halo_probe_reserve(halo_ctx* ctx, size_t max_bytes) {
  if (!ctx || max_bytes < 16) return HALO_ERR_ARG;
  if (ctx->probe_max) return fail(ctx, HALO_ERR_STATE, "probe area already reserved");
  if (ctx->pme_rank >= 0) return fail(ctx, HALO_ERR_STATE, "halo_probe_reserve must precede halo_pme_reserve");
  for (int l = 0; l < ctx->n_local; ++l)
    if (ctx->scratch[l]) return fail(ctx, HALO_ERR_STATE, "halo_probe_reserve must precede halo_register_buffers");
  ctx->probe_max = align_up(max_bytes, 4096);
  ctx->probe_off = align_up(ctx->scratch_bytes, 4096);
  ctx->scratch_bytes = ctx->probe_off + 4096 + 2 * ctx->probe_max;
  return HALO_OK;
}

// ------------------------------------------------------------ home assignment
halo_status halo_assign_home(halo_ctx* ctx, const float* x, int n_atoms, int stride, int32_t* ids, int* counts,
                             void* stream) {
  if (!ctx || n_atoms < 0 || (n_atoms > 0 && (!x || !ids)) || stride < 3 || !counts) return HALO_ERR_ARG;
  if ((uintptr_t)x & 3) return fail(ctx, HALO_ERR_ARG, "x must be 4-B aligned");
  CK(cudaSetDevice(ctx->cfg.device));
  cudaStream_t st = (cudaStream_t)stream;
  const size_t need = align_up(sizeof(int32_t) * std::max(n_atoms, 1), 256) + sizeof(int) * (kMaxRanks + 64 + kAssignSegs * kMaxRanks);
  if (need > ctx->assign_bytes) {
    if (ctx->d_assign) CK(cudaFree(ctx->d_assign));
    CK(cudaMalloc(&ctx->d_assign, need));
    ctx->assign_bytes = need;
  }
  int32_t* rank = reinterpret_cast<int32_t*>(ctx->d_assign);
  int* cnt = reinterpret_cast<int*>(ctx->d_assign + align_up(sizeof(int32_t) * std::max(n_atoms, 1), 256));
  int* err = cnt + kMaxRanks;
  int* seg = cnt + kMaxRanks + 64;  // [kAssignSegs][nranks] per-segment counts
  double planes[3 * (kMaxRanks + 1)] = {0};
  for (int d = 0; d < 3; ++d)
    for (int k = 0; k <= ctx->cfg.grid[d]; ++k) planes[d * (kMaxRanks + 1) + k] = ctx->plane(d, k);
  CK(cudaMemcpyAsync(ctx->d_planes, planes, sizeof planes, cudaMemcpyHostToDevice, st));
  AssignParams A{};
  A.planes = ctx->d_planes;
  for (int d = 0; d < 3; ++d) A.grid[d] = ctx->cfg.grid[d];
  CK(launch_assign_home(x, n_atoms, stride, A, rank, cnt, seg, ids, err, st));
  int h[kMaxRanks + 1] = {0};
  CK(cudaMemcpyAsync(h, cnt, sizeof(int) * (kMaxRanks + 1), cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  for (int r = 0; r < ctx->nranks; ++r) counts[r] = h[r];
  if (h[kMaxRanks]) return fail(ctx, HALO_ERR_GEOMETRY, "a coordinate lies outside [0, L_d) (or is NaN)");
  return HALO_OK;
}

// ------------------------------------------------------------ PP <-> PME (f4)
halo_status halo_pme_reserve(halo_ctx* ctx, int pme_rank) {
  if (!ctx || pme_rank < 0 || pme_rank >= ctx->nranks) return HALO_ERR_ARG;
  if (ctx->pme_rank >= 0) return fail(ctx, HALO_ERR_STATE, "PME already reserved");
  for (int l = 0; l < ctx->n_local; ++l)
    if (ctx->scratch[l]) return fail(ctx, HALO_ERR_STATE, "halo_pme_reserve must precede halo_register_buffers");
  ctx->pme_rank = pme_rank;
  ctx->pme_off = align_up(ctx->scratch_bytes, 256);
  const size_t area = align_up((size_t)ctx->nranks * ctx->cfg.capacity * ctx->W * sizeof(float), 256);
  // only the process hosting pme_rank grows its scratch (the others map it)
  if (pme_rank >= ctx->first_rank && pme_rank < ctx->first_rank + ctx->n_local) ctx->scratch_bytes = ctx->pme_off + 2 * area;
  return HALO_OK;
}

static PmeParams pme_params(halo_ctx* ctx) {
  PmeParams M{};
  const size_t area = align_up((size_t)ctx->nranks * ctx->cfg.capacity * ctx->W * sizeof(float), 256);
  char* base = ctx->peer_scratch[ctx->pme_rank] + ctx->pme_off;
  M.pme_x = reinterpret_cast<float*>(base);
  M.pme_f = reinterpret_cast<float*>(base + area);
  M.pme_hdr = ctx->hdr_of(ctx->pme_rank);
  for (int r = 0; r < ctx->nranks; ++r) M.all_hdr[r] = ctx->hdr_of(r);
  for (int l = 0; l < ctx->n_local; ++l) {
    const int r = ctx->first_rank + l;
    M.r[l].x = ctx->x[l];
    M.r[l].f = ctx->f[l];
    M.r[l].hdr = ctx->hdr_of(r);
    M.r[l].n_home = ctx->n_home.empty() ? 0 : ctx->n_home[l];
    M.r[l].off = ctx->pme_row_off.empty() ? 0 : ctx->pme_row_off[r];
    M.r[l].rank = r;
  }
  M.ctrl = ctx->ctrl;
  M.n_local = ctx->n_local;
  M.nranks = ctx->nranks;
  M.layout = ctx->W;
  M.hosts_pme = ctx->pme_rank >= ctx->first_rank && ctx->pme_rank < ctx->first_rank + ctx->n_local;
  M.accumulate = 1;
  M.epoch = ctx->epoch;
  M.err_host = ctx->err_dev;
  M.timeout_ns = (uint64_t)(ctx->cfg.timeout_s * 1e9);
  return M;
}

static int pme_ctas(halo_ctx* ctx) {
  int mx = 0;
  for (int l = 0; l < ctx->n_local; ++l) mx = std::max(mx, ctx->n_home[l]);
  // ~512 rows per CTA (bandwidth regime needs the whole GPU); any grid size is safe:
  // the PME CTA is row 0 of the grid, resident before every CTA that waits on it
  return std::min(2048, std::max(1, (mx + 511) / 512));
}

halo_status halo_pme_setup(halo_ctx* ctx, void* stream, int* n_total) {
  if (!ctx) return HALO_ERR_ARG;
  if (ctx->pme_rank < 0) return fail(ctx, HALO_ERR_STATE, "halo_pme_reserve first");
  if (!ctx->maps_ready) return fail(ctx, HALO_ERR_STATE, "halo_pme_setup after halo_set_maps");
  CK(cudaSetDevice(ctx->cfg.device));
  halo_status s = check_err_word(ctx);
  if (s != HALO_OK) return s;
  cudaStream_t st = (cudaStream_t)stream;
  ctx->epoch++;
  ctx->pme_ready = false;
  PmeParams M = pme_params(ctx);
  CK(launch_pme(M, 0, 1, st));
  std::vector<int32_t> nh(ctx->nranks);
  CK(cudaMemcpyAsync(nh.data(), ctx->ctrl->pme_nh[0], sizeof(int32_t) * ctx->nranks, cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  if ((s = check_err_word(ctx)) != HALO_OK) return s;
  ctx->pme_row_off.assign(ctx->nranks + 1, 0);
  for (int r = 0; r < ctx->nranks; ++r) ctx->pme_row_off[r + 1] = ctx->pme_row_off[r] + nh[r];
  ctx->pme_total = ctx->pme_row_off[ctx->nranks];
  if (n_total) *n_total = ctx->pme_total;
  ctx->pme_ready = true;
  return HALO_OK;
}

halo_status halo_pme_buffers(const halo_ctx* ctx, float** pme_x, float** pme_f, int* row_off) {
  if (!ctx || !pme_x || !pme_f) return HALO_ERR_ARG;
  if (ctx->pme_rank < 0 || !ctx->peers_ready) return HALO_ERR_STATE;
  const bool hosts = ctx->pme_rank >= ctx->first_rank && ctx->pme_rank < ctx->first_rank + ctx->n_local;
  const size_t area = align_up((size_t)ctx->nranks * ctx->cfg.capacity * ctx->W * sizeof(float), 256);
  char* base = hosts ? ctx->peer_scratch[ctx->pme_rank] + ctx->pme_off : nullptr;
  *pme_x = hosts ? reinterpret_cast<float*>(base) : nullptr;
  *pme_f = hosts ? reinterpret_cast<float*>(base + area) : nullptr;
  if (row_off && ctx->pme_ready)
    for (int r = 0; r <= ctx->nranks; ++r) row_off[r] = ctx->pme_row_off[r];
  return HALO_OK;
}

halo_status halo_pme_send_x(halo_ctx* ctx, void* stream) {
  if (!ctx) return HALO_ERR_ARG;
  if (!ctx->pme_ready || !ctx->maps_ready) return fail(ctx, HALO_ERR_STATE, "halo_pme_setup after every halo_set_maps");
  halo_status s = check_err_word(ctx);
  if (s != HALO_OK) return s;
  CK(launch_pme(pme_params(ctx), 1, pme_ctas(ctx), (cudaStream_t)stream));
  return HALO_OK;
}

halo_status halo_pme_recv_f(halo_ctx* ctx, int accumulate, void* stream) {
  if (!ctx) return HALO_ERR_ARG;
  if (!ctx->pme_ready || !ctx->maps_ready) return fail(ctx, HALO_ERR_STATE, "halo_pme_setup after every halo_set_maps");
  halo_status s = check_err_word(ctx);
  if (s != HALO_OK) return s;
  PmeParams M = pme_params(ctx);
  M.accumulate = accumulate ? 1 : 0;
  CK(launch_pme(M, 2, pme_ctas(ctx), (cudaStream_t)stream));
  return HALO_OK;
}

halo_status halo_transport(const halo_ctx* ctx, int* transport) {
  if (!ctx || !transport) return HALO_ERR_ARG;
  *transport = ctx->ce ? 2 : (ctx->ll ? 0 : 1);
  return HALO_OK;
}

halo_status halo_get_layout(const halo_ctx* ctx, int local, int* n_home, int* n_total, int* npulse, int* recv_off,
                            int* recv_size, int* send_size, int* remote_off, unsigned* dep_mask) {
  if (!ctx || local < 0 || local >= ctx->n_local) return HALO_ERR_ARG;
  if (!ctx->maps_ready) return HALO_ERR_STATE;
  if (n_home) *n_home = ctx->n_home[local];
  if (n_total) *n_total = ctx->n_total[local];
  if (npulse) *npulse = ctx->P;
  for (int p = 0; p < ctx->P; ++p) {
    const int i = local * ctx->P + p;
    if (recv_off) recv_off[p] = ctx->atom_offset[i];
    if (recv_size) recv_size[p] = ctx->recv_size[i];
    if (send_size) send_size[p] = ctx->send_size[i];
    if (remote_off) remote_off[p] = ctx->remote_off[i];
    if (dep_mask) dep_mask[p] = ctx->dep[i];
  }
  return HALO_OK;
}

halo_status halo_get_map(const halo_ctx* ctx, int local, int pulse, int* host_out, int cap) {
  if (!ctx || local < 0 || local >= ctx->n_local || pulse < 0 || pulse >= ctx->P || (!host_out && cap > 0))
    return HALO_ERR_ARG;
  if (!ctx->maps_ready) return HALO_ERR_STATE;
  const int n = ctx->send_size[local * ctx->P + pulse];
  if (cap < n) return HALO_ERR_ARG;
  if (n == 0) return HALO_OK;
  cudaError_t e = cudaMemcpy(host_out, ctx->maps_of_local(local) + (size_t)pulse * ctx->map_stride, sizeof(int) * n,
                             cudaMemcpyDeviceToHost);
  if (e != cudaSuccess) {
    (void)cudaGetLastError();
    return HALO_ERR_CUDA;
  }
  return HALO_OK;
}

// ------------------------------------------------ NCCL send/recv baseline (G2)
halo_status halo_nccl_unique_id(void* id, size_t* len) {
  if (!len) return HALO_ERR_ARG;
  if (!id) { *len = 128; return HALO_OK; }
  if (*len < 128) return HALO_ERR_ARG;
  std::string why;
  if (!nccl_unique_id(id, &why)) {
    fprintf(stderr, "halo_nccl_unique_id: %s\n", why.c_str());
    return HALO_ERR_UNSUPPORTED;
  }
  *len = 128;
  return HALO_OK;
}

halo_status halo_nccl_init(halo_ctx* ctx, const void* id, size_t len) {
  if (!ctx || !id || len < 128) return HALO_ERR_ARG;
  if (ctx->n_local != 1) return fail(ctx, HALO_ERR_UNSUPPORTED, "the NCCL baseline runs one DD rank per process");
  if (ctx->nccl_comm) return fail(ctx, HALO_ERR_STATE, "NCCL communicator already initialised");
  CK(cudaSetDevice(ctx->cfg.device));
  std::string why;
  ctx->nccl_comm = nccl_comm_init(id, ctx->cfg.nprocs, ctx->cfg.proc, &why);
  if (!ctx->nccl_comm) return fail(ctx, HALO_ERR_PEER, why);
  return HALO_OK;
}

halo_status halo_nccl_version(int* version) {
  if (!version) return HALO_ERR_ARG;
  *version = nccl_version();
  return HALO_OK;
}

// x: per pulse ascending, pack kernel -> one NCCL group (send to the lower
// neighbour, receive the upper one's rows into the halo range).
halo_status halo_nccl_exchange_x(halo_ctx* ctx, void* stream) {
  if (!ctx) return HALO_ERR_ARG;
  if (!ctx->nccl_comm) return fail(ctx, HALO_ERR_STATE, "halo_nccl_init first");
  if (!ctx->maps_ready) return fail(ctx, HALO_ERR_STATE, "exchange before set_maps");
  cudaStream_t st = (cudaStream_t)stream;
  const int W = ctx->W, P = ctx->P, r = ctx->first_rank;
  size_t rows = 0;
  for (int p = 0; p < P; ++p) rows += ctx->send_size[p];
  if (rows * W * sizeof(float) > ctx->nccl_send_bytes) {  // NS-step sizes; first call of the epoch only
    CK(cudaDeviceSynchronize());
    if (ctx->d_nccl_send) CK(cudaFree(ctx->d_nccl_send));
    ctx->nccl_send_bytes = std::max<size_t>(rows * W * sizeof(float) * 5 / 4, 256);
    CK(cudaMalloc(&ctx->d_nccl_send, ctx->nccl_send_bytes));
  }
  ctx->x_done = true;
  float* sbuf = ctx->d_nccl_send;
  for (int p = 0; p < P; ++p) {
    const PulseDev& pd = ctx->h_pulses[p];
    const int ns = ctx->send_size[p], nr = ctx->recv_size[p];
    if (ns) CK(launch_pack_x(W, pd.map, ns, ctx->x[0], sbuf, pd.has_shift, pd.shift, st));
    const std::string e = nccl_sendrecv(ctx->nccl_comm, sbuf, (size_t)ns * W, ctx->neighbour(r, ctx->pdim[p], -1),
                                        ctx->x[0] + (size_t)ctx->atom_offset[p] * W, (size_t)nr * W,
                                        ctx->neighbour(r, ctx->pdim[p], +1), st);
    if (!e.empty()) return fail(ctx, HALO_ERR_PEER, e);
    sbuf += (size_t)ns * W;
  }
  return HALO_OK;
}

// f: per pulse descending, one NCCL group (the halo slice back to the x-sender,
// this rank's returned slice from its x-receiver) -> ordered scatter-add kernel.
halo_status halo_nccl_exchange_f(halo_ctx* ctx, double* fshift, int accumulate, void* stream) {
  if (!ctx) return HALO_ERR_ARG;
  if (!ctx->nccl_comm) return fail(ctx, HALO_ERR_STATE, "halo_nccl_init first");
  if (!ctx->maps_ready || !ctx->x_done) return fail(ctx, HALO_ERR_STATE, "exchange_f before set_maps/exchange_x");
  if (!accumulate && ctx->P != 1) return fail(ctx, HALO_ERR_UNSUPPORTED, "accumulate=0 needs exactly one pulse (R14)");
  cudaStream_t st = (cudaStream_t)stream;
  const int W = ctx->W, P = ctx->P, r = ctx->first_rank;
  for (int p = P - 1; p >= 0; --p) {
    const PulseDev& pd = ctx->h_pulses[p];
    const int ns = ctx->send_size[p], nr = ctx->recv_size[p];
    float* rbuf = ctx->fbuf_of(r) + (size_t)p * ctx->fbuf_stride;
    const std::string e = nccl_sendrecv(ctx->nccl_comm, ctx->f[0] + (size_t)ctx->atom_offset[p] * W, (size_t)nr * W,
                                        ctx->neighbour(r, ctx->pdim[p], +1), rbuf, (size_t)ns * W,
                                        ctx->neighbour(r, ctx->pdim[p], -1), st);
    if (!e.empty()) return fail(ctx, HALO_ERR_PEER, e);
    double* fs = (fshift && pd.has_shift) ? fshift + 3 * pd.dim : nullptr;
    if (ns) CK(launch_unpack_f(W, pd.map, ns, rbuf, ctx->f[0], accumulate ? 1 : 0, fs, st));
  }
  return HALO_OK;
}

halo_status halo_exchange_x(halo_ctx* ctx, void* stream) {
  if (!ctx) return HALO_ERR_ARG;
  if (!ctx->maps_ready) return fail(ctx, HALO_ERR_STATE, "exchange_x before set_maps");
  halo_status s = check_err_word(ctx);
  if (s != HALO_OK) return s;
  ctx->x_done = true;
  if (ctx->P == 0) return HALO_OK;
  if (ctx->cfg.flags & HALO_F_NCCL_BASELINE) return halo_nccl_exchange_x(ctx, stream);
  if (ctx->ce) return ce_exchange_x(ctx, (cudaStream_t)stream);
  ExParams X = make_params(ctx, ctx->d_items_x, ctx->n_items_x, 0, ctx->P);
  const int grid = grid_for(ctx->n_items_x, ctx->n_local, ctx->cap_x());
  ctx->last_grid[0] = grid;
  if (ctx->ll) {
    bool cap = false;
    X.seq = next_seq(ctx, (cudaStream_t)stream, &ctx->seq_host_x, &cap);
    X.n_items_x = ctx->n_items_x;
    if (ctx->prefetch) {  // the f launch's item blocks and the home x rows (L2 prefetch)
      X.pf_f = ctx->d_fblk;
      X.pf_f_bytes = (uint64_t)ctx->n_items_f * ll_fblk_bytes(ctx->tree_rows);
      X.pf_x = 1;
    }
    CK(launch_exchange_ll(X, 0, ctx->W, grid, ctx->wide(), &ctx->l2win, (cudaStream_t)stream, cap));
  }
  if (!ctx->ll)
    CK(launch_exchange_x(X, ctx->W, grid, (cudaStream_t)stream));
  return HALO_OK;
}

halo_status halo_exchange_f(halo_ctx* ctx, double* fshift, int accumulate, void* stream) {
  if (!ctx) return HALO_ERR_ARG;
  if (!ctx->maps_ready || !ctx->x_done) return fail(ctx, HALO_ERR_STATE, "exchange_f before set_maps/exchange_x");
  if (!accumulate && ctx->P != 1) return fail(ctx, HALO_ERR_UNSUPPORTED, "accumulate=0 needs exactly one pulse (R14)");
  halo_status s = check_err_word(ctx);
  if (s != HALO_OK) return s;
  if (ctx->P == 0) return HALO_OK;
  if (ctx->cfg.flags & HALO_F_NCCL_BASELINE) return halo_nccl_exchange_f(ctx, fshift, accumulate, stream);
  if (ctx->ce) return ce_exchange_f(ctx, fshift, accumulate ? 1 : 0, (cudaStream_t)stream);
  ExParams F = make_params(ctx, ctx->d_items_f, ctx->n_items_f, 0, ctx->P);
  F.fshift = fshift;
  F.accumulate = accumulate ? 1 : 0;
  int grid = grid_for(ctx->n_items_f, ctx->n_local, ctx->cap_f());
  if (ctx->ll) {  // dedicated CTAs for the combines
    F.n_tail = ctx->n_tail_f;
    grid = std::min(ctx->n_items_f - ctx->n_tail_f, ctx->cap_f() - ctx->n_tail_f) + ctx->n_tail_f;
    grid = std::max(grid, 1);
  }
  ctx->last_grid[1] = grid;
  if (ctx->ll) {
    bool cap = false;
    F.ring = ll_ring(1, ctx->wide());
    F.seq_f = next_seq(ctx, (cudaStream_t)stream, &ctx->seq_host_f, &cap);
    CK(launch_exchange_ll(F, 1, ctx->W, grid, ctx->wide(), &ctx->l2win, (cudaStream_t)stream, cap));
  }
  if (!ctx->ll)
    CK(launch_exchange_f(F, ctx->W, grid, (cudaStream_t)stream));
  return HALO_OK;
}

halo_status halo_exchange_xf(halo_ctx* ctx, double* fshift, int accumulate, void* stream) {
  if (!ctx) return HALO_ERR_ARG;
  if (!ctx->maps_ready) return fail(ctx, HALO_ERR_STATE, "exchange_xf before set_maps");
  if (!accumulate && ctx->P != 1) return fail(ctx, HALO_ERR_UNSUPPORTED, "accumulate=0 needs exactly one pulse (R14)");
  if (!ctx->ll) return fail(ctx, HALO_ERR_UNSUPPORTED, "the fused x+f launch exists for the LL protocol only");
  halo_status s = check_err_word(ctx);
  if (s != HALO_OK) return s;
  ctx->x_done = true;
  if (ctx->P == 0) return HALO_OK;
  // one item list: every x item, then the gather items, then the combines (tail)
  ExParams X = make_params(ctx, ctx->d_items_x, ctx->n_items_x + ctx->n_items_f, 0, ctx->P);
  X.n_items_x = ctx->n_items_x;
  X.n_tail = ctx->n_tail_f;
  X.fshift = fshift;
  X.accumulate = accumulate ? 1 : 0;
  int grid = std::min(X.n_items - X.n_tail, ctx->cap_xf() - X.n_tail) + X.n_tail;
  grid = std::max(grid, 1);
  ctx->last_grid[0] = grid;
  bool cap = false;
  X.ring = ll_ring(2, ctx->wide());
  X.seq = next_seq(ctx, (cudaStream_t)stream, &ctx->seq_host_x, &cap);
  X.seq_f = next_seq(ctx, (cudaStream_t)stream, &ctx->seq_host_f);
  CK(launch_exchange_ll(X, 2, ctx->W, grid, ctx->wide(), &ctx->l2win, (cudaStream_t)stream, cap));
  return HALO_OK;
}

halo_status halo_step_host(halo_ctx* ctx, const float* const* x_home, const float* const* f_all,
                           float* const* x_halo_out, float* const* f_home_out, double* fshift_host, void* stream) {
  if (!ctx || !x_home || !f_all) return HALO_ERR_ARG;
  if (!ctx->maps_ready) return fail(ctx, HALO_ERR_STATE, "step before set_maps");
  cudaStream_t st = (cudaStream_t)stream;
  const int W = ctx->W;
  for (int l = 0; l < ctx->n_local; ++l) {
    CK(cudaMemcpyAsync(ctx->x[l], x_home[l], sizeof(float) * W * ctx->n_home[l], cudaMemcpyHostToDevice, st));
    CK(cudaMemcpyAsync(ctx->f[l], f_all[l], sizeof(float) * W * ctx->n_total[l], cudaMemcpyHostToDevice, st));
  }
  halo_status s = halo_exchange_x(ctx, stream);
  if (s != HALO_OK) return s;
  // halo x leaves before exchange_f: a neighbour's next exchange_x may only
  // overwrite these rows after our exchange_f has pushed (R17)
  if (x_halo_out)
    for (int l = 0; l < ctx->n_local; ++l)
      if (x_halo_out[l] && ctx->n_total[l] > ctx->n_home[l])
        CK(cudaMemcpyAsync(x_halo_out[l], ctx->x[l] + (size_t)W * ctx->n_home[l],
                           sizeof(float) * W * (ctx->n_total[l] - ctx->n_home[l]), cudaMemcpyDeviceToHost, st));
  CK(cudaMemsetAsync(ctx->d_fshift_tmp, 0, sizeof(double) * 9 * ctx->n_local, st));
  s = halo_exchange_f(ctx, ctx->d_fshift_tmp, 1, stream);
  if (s != HALO_OK) return s;
  if (f_home_out)
    for (int l = 0; l < ctx->n_local; ++l)
      if (f_home_out[l])
        CK(cudaMemcpyAsync(f_home_out[l], ctx->f[l], sizeof(float) * W * ctx->n_home[l], cudaMemcpyDeviceToHost, st));
  if (fshift_host)
    CK(cudaMemcpyAsync(fshift_host, ctx->d_fshift_tmp, sizeof(double) * 9 * ctx->n_local, cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  return check_err_word(ctx);
}

// Packed host layout (halo_step_host_packed): in = [x home rows of local ranks 0..L-1 |
// f rows [0, n_total) of local ranks 0..L-1]; out = [x halo rows of every local rank |
// f home rows of every local rank | fshift, n_local*9 doubles, at an 8-B aligned offset].
static void packed_sizes(const halo_ctx* ctx, size_t* in_b, size_t* out_b, size_t* fs_off) {
  size_t xh = 0, fa = 0, xo = 0, fo = 0;
  for (int l = 0; l < ctx->n_local; ++l) {
    xh += ctx->n_home[l];
    fa += ctx->n_total[l];
    xo += ctx->n_total[l] - ctx->n_home[l];
    fo += ctx->n_home[l];
  }
  const size_t rb = sizeof(float) * ctx->W;
  *in_b = (xh + fa) * rb;
  *fs_off = align_up((xo + fo) * rb, 8);
  *out_b = *fs_off + sizeof(double) * 9 * ctx->n_local;
}

static halo_status packed_prepare(halo_ctx* ctx, char* out_dev) {
  size_t in_b, out_b, fs_off;
  packed_sizes(ctx, &in_b, &out_b, &fs_off);
  const int L = ctx->n_local;
  if (in_b > ctx->pk_in_cap) {
    if (ctx->d_pk_in) CK(cudaFree(ctx->d_pk_in));
    ctx->d_pk_in = nullptr;
    CK(cudaMalloc(&ctx->d_pk_in, in_b + in_b / 4));
    ctx->pk_in_cap = in_b + in_b / 4;
  }
  if (out_b > ctx->pk_out_cap) {
    if (ctx->d_pk_out) CK(cudaFree(ctx->d_pk_out));
    ctx->d_pk_out = nullptr;
    CK(cudaMalloc(&ctx->d_pk_out, out_b + out_b / 4));
    ctx->pk_out_cap = out_b + out_b / 4;
  }
  if (!ctx->d_segs) CK(cudaMalloc(&ctx->d_segs, sizeof(SegCopy) * (4 * kMaxLocal + 1)));
  if (!ctx->pk_h2d) {
    CK(cudaStreamCreateWithFlags(&ctx->pk_h2d, cudaStreamNonBlocking));
    CK(cudaStreamCreateWithFlags(&ctx->pk_d2h, cudaStreamNonBlocking));
    for (auto& e : ctx->pk_ev) CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  }
  // segment tables: [0, L) x home in; [L, 2L) f in; [2L, 4L+1) out (x halo, f home, fshift)
  std::vector<SegCopy> sg(4 * L + 1);
  const size_t W = ctx->W;
  size_t o = 0;
  for (auto& m : ctx->pk_max_words) m = 0;
  auto words = [](size_t b) { return b / 4; };
  for (int l = 0; l < L; ++l) {
    sg[l] = SegCopy{reinterpret_cast<const uint32_t*>(ctx->d_pk_in + o), reinterpret_cast<uint32_t*>(ctx->x[l]),
                    W * ctx->n_home[l]};
    o += 4 * W * ctx->n_home[l];
    ctx->pk_max_words[0] = std::max(ctx->pk_max_words[0], sg[l].words);
  }
  for (int l = 0; l < L; ++l) {
    sg[L + l] = SegCopy{reinterpret_cast<const uint32_t*>(ctx->d_pk_in + o), reinterpret_cast<uint32_t*>(ctx->f[l]),
                        W * ctx->n_total[l]};
    o += 4 * W * ctx->n_total[l];
    ctx->pk_max_words[1] = std::max(ctx->pk_max_words[1], sg[L + l].words);
  }
  o = 0;
  for (int l = 0; l < L; ++l) {
    const size_t nh = ctx->n_total[l] - ctx->n_home[l];
    sg[2 * L + l] = SegCopy{reinterpret_cast<const uint32_t*>(ctx->x[l] + W * ctx->n_home[l]),
                            reinterpret_cast<uint32_t*>(ctx->d_pk_out + o), W * nh};
    o += 4 * W * nh;
  }
  // the forces and fshift: straight into the caller's (mapped, pinned) host block when
  // it is device-accessible (no download after the last kernel), else into staging
  char* fo = out_dev ? out_dev : ctx->d_pk_out;
  for (int l = 0; l < L; ++l) {
    sg[3 * L + l] = SegCopy{reinterpret_cast<const uint32_t*>(ctx->f[l]), reinterpret_cast<uint32_t*>(fo + o),
                            W * ctx->n_home[l]};
    o += 4 * W * ctx->n_home[l];
  }
  sg[4 * L] = SegCopy{reinterpret_cast<const uint32_t*>(ctx->d_fshift_tmp),
                      reinterpret_cast<uint32_t*>(fo + fs_off), words(sizeof(double) * 9 * L)};
  for (int k = 2 * L; k <= 4 * L; ++k) ctx->pk_max_words[2] = std::max(ctx->pk_max_words[2], sg[k].words);
  CK(cudaMemcpy(ctx->d_segs, sg.data(), sizeof(SegCopy) * sg.size(), cudaMemcpyHostToDevice));
  ctx->pk_epoch = ctx->epoch;
  ctx->pk_out_dev = out_dev;
  return HALO_OK;
}

halo_status halo_packed_sizes(const halo_ctx* ctx, size_t* in_bytes, size_t* out_bytes) {
  if (!ctx || !in_bytes || !out_bytes) return HALO_ERR_ARG;
  if (!ctx->maps_ready) return HALO_ERR_STATE;
  size_t fs_off;
  packed_sizes(ctx, in_bytes, out_bytes, &fs_off);
  return HALO_OK;
}

// The packed step's operations, enqueued on st (eager, or under capture: packed_graph).
static halo_status packed_enqueue(halo_ctx* ctx, const void* in_host, void* out_host, char* out_dev, cudaStream_t st) {
  halo_status s;
  const int L = ctx->n_local;
  size_t in_b, out_b, fs_off;
  packed_sizes(ctx, &in_b, &out_b, &fs_off);
  size_t bx = 0, bxo = 0;
  for (int l = 0; l < L; ++l) {
    bx += sizeof(float) * ctx->W * ctx->n_home[l];
    bxo += sizeof(float) * ctx->W * (ctx->n_total[l] - ctx->n_home[l]);
  }
  const char* in = static_cast<const char*>(in_host);
  char* out = static_cast<char*>(out_host);
  // x home rows first; the forces follow on a side stream (PCIe H2D) while x is exchanged
  CK(cudaMemcpyAsync(ctx->d_pk_in, in, bx, cudaMemcpyHostToDevice, st));
  CK(cudaEventRecord(ctx->pk_ev[0], st));
  CK(cudaStreamWaitEvent(ctx->pk_h2d, ctx->pk_ev[0], 0));
  CK(cudaMemcpyAsync(ctx->d_pk_in + bx, in + bx, in_b - bx, cudaMemcpyHostToDevice, ctx->pk_h2d));
  CK(cudaEventRecord(ctx->pk_ev[1], ctx->pk_h2d));
  CK(launch_seg_copy(ctx->d_segs, L, ctx->pk_max_words[0], st));
  if ((s = halo_exchange_x(ctx, st)) != HALO_OK) return s;
  // halo x rows -> staging (before exchange_f: a neighbour's next exchange_x may only
  // overwrite them after our exchange_f, R17), downloaded on a side stream (PCIe D2H)
  CK(launch_seg_copy(ctx->d_segs + 2 * L, L, ctx->pk_max_words[2], st));
  CK(cudaEventRecord(ctx->pk_ev[2], st));
  if (out) {
    CK(cudaStreamWaitEvent(ctx->pk_d2h, ctx->pk_ev[2], 0));
    CK(cudaMemcpyAsync(out, ctx->d_pk_out, bxo, cudaMemcpyDeviceToHost, ctx->pk_d2h));
    CK(cudaEventRecord(ctx->pk_ev[3], ctx->pk_d2h));
  }
  CK(cudaStreamWaitEvent(st, ctx->pk_ev[1], 0));
  CK(launch_seg_copy(ctx->d_segs + L, L, ctx->pk_max_words[1], st));
  CK(cudaMemsetAsync(ctx->d_fshift_tmp, 0, sizeof(double) * 9 * L, st));
  if ((s = halo_exchange_f(ctx, ctx->d_fshift_tmp, 1, st)) != HALO_OK) return s;
  if (out) {
    CK(launch_seg_copy(ctx->d_segs + 3 * L, L + 1, ctx->pk_max_words[2], st));
    if (!out_dev) CK(cudaMemcpyAsync(out + bxo, ctx->d_pk_out + bxo, out_b - bxo, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamWaitEvent(st, ctx->pk_ev[3], 0));
  }
  return HALO_OK;
}

halo_status halo_step_host_packed(halo_ctx* ctx, const void* in_host, void* out_host, void* stream) {
  if (!ctx || !in_host) return HALO_ERR_ARG;
  if (!ctx->maps_ready) return fail(ctx, HALO_ERR_STATE, "step before set_maps");
  halo_status s;
  // a device-accessible (mapped pinned) output block takes the forces directly
  char* out_dev = nullptr;
  if (out_host && getenv("HALO_PACKED_DIRECT")) {  // measured slower than staging + one copy (C3: 184 vs 130 us)
    cudaPointerAttributes pa{};
    if (cudaPointerGetAttributes(&pa, out_host) == cudaSuccess && pa.type == cudaMemoryTypeHost && pa.devicePointer)
      out_dev = static_cast<char*>(pa.devicePointer);
    (void)cudaGetLastError();
  }
  if (ctx->pk_epoch != ctx->epoch || !ctx->d_segs || ctx->pk_out_dev != out_dev)
    if ((s = packed_prepare(ctx, out_dev)) != HALO_OK) return s;
  cudaStream_t st = (cudaStream_t)stream;
  if (getenv("HALO_PACKED_GRAPH") && atoi(getenv("HALO_PACKED_GRAPH")) == 0) {
    if ((s = packed_enqueue(ctx, in_host, out_host, out_dev, st)) != HALO_OK) return s;
  } else {
    // the whole step (2 uploads, 4 copy kernels, 2 exchanges, 2 downloads on 3 streams) as
    // ONE CUDA graph per (NS epoch, host blocks): one launch instead of ~14 API calls
    if (!ctx->pk_exec || ctx->pk_g_epoch != ctx->epoch || ctx->pk_g_in != in_host || ctx->pk_g_out != out_host) {
      if (ctx->pk_exec) CK(cudaGraphExecDestroy(ctx->pk_exec));
      ctx->pk_exec = nullptr;
      if (!ctx->pk_cap) CK(cudaStreamCreateWithFlags(&ctx->pk_cap, cudaStreamNonBlocking));
      const bool was = ctx->captured;
      const uint64_t sx = ctx->seq_host_x, sf = ctx->seq_host_f;
      CK(cudaStreamBeginCapture(ctx->pk_cap, cudaStreamCaptureModeThreadLocal));
      const halo_status se = packed_enqueue(ctx, in_host, out_host, out_dev, ctx->pk_cap);
      cudaGraph_t g = nullptr;
      const cudaError_t ee = cudaStreamEndCapture(ctx->pk_cap, &g);
      ctx->captured = was;  // the capture launched nothing: the eager launches keep their by-value numbers
      ctx->seq_host_x = sx;
      ctx->seq_host_f = sf;
      if (se != HALO_OK) {
        if (g) (void)cudaGraphDestroy(g);
        return se;
      }
      if (ee != cudaSuccess) return cuda_fail(ctx, ee, "packed step capture");
      CK(cudaGraphInstantiate(&ctx->pk_exec, g, 0));
      CK(cudaGraphDestroy(g));
      ctx->pk_g_epoch = ctx->epoch;
      ctx->pk_g_in = in_host;
      ctx->pk_g_out = out_host;
    }
    CK(cudaGraphLaunch(ctx->pk_exec, st));
    // the replay advanced the device sequence counters by one x and one f launch
    if (ctx->ll) {
      ctx->seq_host_x = ll_seq_next(ctx->seq_host_x);
      ctx->seq_host_f = ll_seq_next(ctx->seq_host_f);
    }
  }
  // the caller's results are in out_host when this returns: poll the stream instead of a
  // blocking synchronise (whose yield / wake-up latency lands in every step of a
  // latency-bound host loop); HALO_PACKED_BLOCKING=1 restores cudaStreamSynchronize
  if (ctx->packed_blocking) {
    CK(cudaStreamSynchronize(st));
  } else {
    cudaError_t q;
    while ((q = cudaStreamQuery(st)) == cudaErrorNotReady) {
    }
    CK(q);
  }
  return check_err_word(ctx);
}

halo_status halo_pack_x_pulse(halo_ctx* ctx, int local, int pulse, float* sendbuf, void* stream) {
  if (!ctx || local < 0 || local >= ctx->n_local || pulse < 0 || pulse >= ctx->P || !sendbuf) return HALO_ERR_ARG;
  if (!ctx->maps_ready) return fail(ctx, HALO_ERR_STATE, "pack before set_maps");
  const PulseDev& pd = ctx->h_pulses[local * ctx->P + pulse];
  CK(launch_pack_x(ctx->W, pd.map, pd.send_size, ctx->x[local], sendbuf, pd.has_shift, pd.shift, (cudaStream_t)stream));
  return HALO_OK;
}

halo_status halo_unpack_f_pulse(halo_ctx* ctx, int local, int pulse, const float* recvbuf, double* fshift,
                                int accumulate, void* stream) {
  if (!ctx || local < 0 || local >= ctx->n_local || pulse < 0 || pulse >= ctx->P || !recvbuf) return HALO_ERR_ARG;
  if (!ctx->maps_ready) return fail(ctx, HALO_ERR_STATE, "unpack before set_maps");
  const PulseDev& pd = ctx->h_pulses[local * ctx->P + pulse];
  double* fs = (fshift && pd.has_shift) ? fshift + 9 * local + 3 * pd.dim : nullptr;
  CK(launch_unpack_f(ctx->W, pd.map, pd.send_size, recvbuf, ctx->f[local], accumulate, fs, (cudaStream_t)stream));
  return HALO_OK;
}

halo_status halo_get_timers(halo_ctx* ctx, uint64_t* x_ns, uint64_t* f_ns) {
  if (!ctx) return HALO_ERR_ARG;
  uint64_t v[2];
  CK(cudaSetDevice(ctx->cfg.device));
  CK(cudaDeviceSynchronize());
  CK(cudaMemcpy(v, &ctx->ctrl->span_x, sizeof v, cudaMemcpyDeviceToHost));
  if (ctx->ll) {  // exact spans from the per-CTA trace: max(exit) - min(start)
    for (int which = 0; which < 2; ++which) {
      const int m = std::min(ctx->last_grid[which], kTraceCTAs);
      if (m <= 0) continue;
      std::vector<uint64_t> t(kTraceW * (size_t)m);
      CK(cudaMemcpy(t.data(), &ctx->ctrl->trace[which][0][0], sizeof(uint64_t) * kTraceW * m, cudaMemcpyDeviceToHost));
      uint64_t lo = ~0ull, hi = 0;
      for (int i = 0; i < m; ++i) {
        lo = std::min(lo, t[kTraceW * i]);
        hi = std::max(hi, t[kTraceW * i + 3]);
      }
      // (with programmatic dependent launch the stamps of consecutive launches can
      // interleave; keep the last arriver's span when the trace is inconsistent)
      if (hi > lo) v[which] = hi - lo;
    }
  }
  if (x_ns) *x_ns = v[0];
  if (f_ns) *f_ns = v[1];
  return HALO_OK;
}

halo_status halo_get_notify_counts(halo_ctx* ctx, int which, uint32_t* out, int cap) {
  if (!ctx || which < 0 || which > 1 || !out || cap < ctx->n_local * ctx->P) return HALO_ERR_ARG;
  CK(cudaSetDevice(ctx->cfg.device));
  CK(cudaDeviceSynchronize());
  uint32_t v[kMaxLocal][kMaxP];
  CK(cudaMemcpy(v, &ctx->ctrl->notify[which][0][0], sizeof v, cudaMemcpyDeviceToHost));
  for (int l = 0; l < ctx->n_local; ++l)
    for (int p = 0; p < ctx->P; ++p) out[l * ctx->P + p] = v[l][p];
  return HALO_OK;
}

halo_status halo_get_trace(halo_ctx* ctx, int which, uint64_t* out, int cap, int* n) {
  if (!ctx || which < 0 || which > 1 || !out || !n) return HALO_ERR_ARG;
  const int m = std::min(std::min(ctx->last_grid[which], kTraceCTAs), cap / kTraceW);
  *n = m;
  if (m <= 0) return HALO_OK;
  CK(cudaSetDevice(ctx->cfg.device));
  CK(cudaDeviceSynchronize());
  CK(cudaMemcpy(out, &ctx->ctrl->trace[which][0][0], sizeof(uint64_t) * kTraceW * m, cudaMemcpyDeviceToHost));
  return HALO_OK;
}

halo_status halo_floor_pingpong(halo_ctx* ctx, int peer_rank, int iters, int relaxed, double* one_way_us) {
  if (!ctx || peer_rank < 0 || peer_rank >= ctx->nranks || iters <= 0) return HALO_ERR_ARG;
  if (!ctx->peers_ready) return fail(ctx, HALO_ERR_STATE, "import peers first");
  const int me = ctx->first_rank;
  if (peer_rank == me) return fail(ctx, HALO_ERR_ARG, "ping-pong peer must differ from local rank 0");
  // both ranks on this GPU: one launch plays both sides (2 CTAs); else the
  // initiator is the process that hosts the lower of the two ranks
  const bool local = peer_rank >= ctx->first_rank && peer_rank < ctx->first_rank + ctx->n_local;
  CK(cudaSetDevice(ctx->cfg.device));
  const bool initiator = local || me < peer_rank;
  if (ctx->d_rtt == nullptr || iters > 1 << 16) {
    if (ctx->d_rtt) CK(cudaFree(ctx->d_rtt));
    CK(cudaMalloc(&ctx->d_rtt, sizeof(uint64_t) * std::max(iters, 1 << 16)));
  }
  cudaStream_t st;
  CK(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
  uint64_t* own = &ctx->hdr_of(me)->ping;
  uint64_t* peer = &ctx->hdr_of(peer_rank)->ping;
  CK(launch_pingpong(own, peer, iters, ctx->ping_base, local ? 2 : (initiator ? 1 : 0), relaxed ? 1 : 0, ctx->d_rtt,
                     (uint64_t)(ctx->cfg.timeout_s * 1e9), ctx->err_dev, st));
  CK(cudaStreamSynchronize(st));
  CK(cudaStreamDestroy(st));
  ctx->ping_base += (uint64_t)iters;
  halo_status s = check_err_word(ctx);
  if (s != HALO_OK) return s;
  if (one_way_us) {
    *one_way_us = 0.0;
    if (initiator) {
      std::vector<uint64_t> v(iters);
      CK(cudaMemcpy(v.data(), ctx->d_rtt, sizeof(uint64_t) * iters, cudaMemcpyDeviceToHost));
      std::sort(v.begin(), v.end());
      *one_way_us = (double)v[iters / 2] / 2.0 / 1000.0;
    }
  }
  return HALO_OK;
}

static halo_status floor_launch_impl(halo_ctx* ctx, int iters, int graph, uint64_t* remote, uint32_t nwords,
                                     double* us_per_launch) {
  if (!ctx || iters <= 0 || !us_per_launch) return HALO_ERR_ARG;
  CK(cudaSetDevice(ctx->cfg.device));
  cudaStream_t st;
  CK(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  const int grid = std::max(1, std::min(ctx->max_x, 512));
  float ms = 0.f;
  if (!graph) {
    for (int i = 0; i < 10; ++i) CK(launch_empty(grid, st, remote, nwords));
    CK(cudaEventRecord(e0, st));
    for (int i = 0; i < iters; ++i) CK(launch_empty(grid, st, remote, nwords));
    CK(cudaEventRecord(e1, st));
    CK(cudaEventSynchronize(e1));
    CK(cudaEventElapsedTime(&ms, e0, e1));
  } else {
    cudaGraph_t g;
    cudaGraphExec_t ge;
    CK(cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal));
    for (int i = 0; i < iters; ++i) CK(launch_empty(grid, st, remote, nwords));
    CK(cudaStreamEndCapture(st, &g));
    CK(cudaGraphInstantiate(&ge, g, 0));
    CK(cudaGraphLaunch(ge, st));
    CK(cudaStreamSynchronize(st));
    CK(cudaEventRecord(e0, st));
    CK(cudaGraphLaunch(ge, st));
    CK(cudaEventRecord(e1, st));
    CK(cudaEventSynchronize(e1));
    CK(cudaEventElapsedTime(&ms, e0, e1));
    CK(cudaGraphExecDestroy(ge));
    CK(cudaGraphDestroy(g));
  }
  *us_per_launch = 1e3 * (double)ms / iters;
  CK(cudaEventDestroy(e0));
  CK(cudaEventDestroy(e1));
  CK(cudaStreamDestroy(st));
  return HALO_OK;
}

halo_status halo_floor_empty_pair(halo_ctx* ctx, void* stream) {
  if (!ctx) return HALO_ERR_ARG;
  if (!ctx->maps_ready) return fail(ctx, HALO_ERR_STATE, "floor before set_maps");
  // the step's two launches with no work: the grids of the current x and f launches,
  // the same programmatic-dependent-launch attributes, empty bodies
  int gx = grid_for(ctx->n_items_x, ctx->n_local, ctx->cap_x());
  int gf = grid_for(ctx->n_items_f, ctx->n_local, ctx->cap_f());
  // grid-size study (HALO_EMPTY_GX / HALO_EMPTY_GF): what the CTA count alone costs
  if (const char* e = getenv("HALO_EMPTY_GX")) gx = std::max(1, atoi(e));
  if (const char* e = getenv("HALO_EMPTY_GF")) gf = std::max(1, atoi(e));
  CK(launch_empty(gx, (cudaStream_t)stream, nullptr, 0));
  CK(launch_empty(gf, (cudaStream_t)stream, nullptr, 0));
  return HALO_OK;
}

halo_status halo_floor_launch(halo_ctx* ctx, int iters, int graph, double* us_per_launch) {
  return floor_launch_impl(ctx, iters, graph, nullptr, 0, us_per_launch);
}

halo_status halo_floor_launch_remote(halo_ctx* ctx, int peer_rank, int words, int iters, int graph,
                                     double* us_per_launch) {
  if (!ctx || peer_rank < 0 || peer_rank >= ctx->nranks || words < 0) return HALO_ERR_ARG;
  if (!ctx->peers_ready) return fail(ctx, HALO_ERR_STATE, "import peers first");
  const int grid = std::max(1, std::min(ctx->max_x, 512));
  const size_t area = 2 * (size_t)ctx->P * ctx->ll_stride;  // u64 words of the peer's LL receive areas
  if ((size_t)words > std::min(area, (size_t)grid * kThreads)) return fail(ctx, HALO_ERR_ARG, "too many words");
  // the peer's LL receive areas: the caller keeps the peer idle (no exchange in flight)
  return floor_launch_impl(ctx, iters, graph, ctx->xll_of(peer_rank), (uint32_t)words, us_per_launch);
}

halo_status halo_floor_bandwidth(halo_ctx* ctx, int peer_rank, size_t bytes, int mode, int iters, double* gbs) {
  if (!ctx || peer_rank < 0 || peer_rank >= ctx->nranks || iters <= 0 || !gbs || (mode != 0 && mode != 1))
    return HALO_ERR_ARG;
  if (!ctx->peers_ready) return fail(ctx, HALO_ERR_STATE, "import peers first");
  // the peer's scratch from its coordinate LL receive area to the end (LL areas,
  // shift-force slots, migration staging: >= 8 MiB, scratch_layout)
  const size_t xll_off = kHdrBytes + (size_t)ctx->P * ctx->map_stride * sizeof(int32_t) +
                         (size_t)ctx->P * ctx->fbuf_stride * sizeof(float);
  // (the base layout every rank shares; a PME rank's scratch is longer, halo_pme_reserve)
  const size_t area = scratch_layout(ctx->P, ctx->cfg.capacity, ctx->W).total - xll_off;
  bytes = bytes / 16 * 16;
  if (bytes == 0 || bytes > area) return fail(ctx, HALO_ERR_ARG, "bytes must be in [16, probe area]");
  CK(cudaSetDevice(ctx->cfg.device));
  const int me = ctx->first_rank;
  char* src = reinterpret_cast<char*>(ctx->xll_of(me));
  char* dst = reinterpret_cast<char*>(ctx->xll_of(peer_rank));
  cudaStream_t st;
  CK(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  int sms = 148, dev = ctx->cfg.device;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  auto one = [&]() -> cudaError_t {
    return mode == 0 ? launch_bw_copy(src, dst, bytes, 8 * sms, st) : cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDefault, st);
  };
  for (int i = 0; i < 3; ++i) CK(one());
  CK(cudaEventRecord(e0, st));
  for (int i = 0; i < iters; ++i) CK(one());
  CK(cudaEventRecord(e1, st));
  CK(cudaEventSynchronize(e1));
  float ms = 0.f;
  CK(cudaEventElapsedTime(&ms, e0, e1));
  *gbs = (double)bytes * iters / (1e-3 * (double)ms) / 1e9;
  CK(cudaEventDestroy(e0));
  CK(cudaEventDestroy(e1));
  CK(cudaStreamDestroy(st));
  return HALO_OK;
}

// t(B): one-way latency of a B-byte payload + its signal, half the median round trip.
halo_status halo_floor_payload(halo_ctx* ctx, int peer_rank, size_t bytes, int iters, int ctas, double* one_way_us) {
  if (!ctx || peer_rank < 0 || peer_rank >= ctx->nranks || iters <= 0 || ctas <= 0) return HALO_ERR_ARG;
  if (!ctx->peers_ready) return fail(ctx, HALO_ERR_STATE, "import peers first");
  if (!ctx->probe_max) return fail(ctx, HALO_ERR_STATE, "halo_probe_reserve first");
  bytes = bytes / 16 * 16;
  if (bytes == 0 || bytes > ctx->probe_max) return fail(ctx, HALO_ERR_ARG, "bytes must be in [16, reserved probe bytes]");
  const int me = ctx->first_rank;
  if (peer_rank == me) return fail(ctx, HALO_ERR_ARG, "peer must differ from local rank 0");
  const bool local = peer_rank >= ctx->first_rank && peer_rank < ctx->first_rank + ctx->n_local;
  const bool initiator = local || me < peer_rank;
  const int G = (int)std::min<size_t>((size_t)ctas, std::max<size_t>(1, (bytes + 16383) / 16384));
  if (local && 2 * G > std::max(2, ctx->max_x)) return fail(ctx, HALO_ERR_ARG, "too many CTAs for a same-GPU probe");
  CK(cudaSetDevice(ctx->cfg.device));
  if (ctx->d_rtt == nullptr || iters > 1 << 16) {
    if (ctx->d_rtt) CK(cudaFree(ctx->d_rtt));
    CK(cudaMalloc(&ctx->d_rtt, sizeof(uint64_t) * std::max(iters, 1 << 16)));
  }
  auto area = [&](int r) { return ctx->peer_scratch[r] + ctx->probe_off; };
  uint64_t* cnt_own = reinterpret_cast<uint64_t*>(area(me));
  uint64_t* cnt_peer = reinterpret_cast<uint64_t*>(area(peer_rank));
  const int lp = peer_rank - ctx->first_rank;
  cudaStream_t st;
  CK(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
  CK(launch_payload_pingpong(area(me) + 4096, area(peer_rank) + 4096 + ctx->probe_max,
                             local ? area(peer_rank) + 4096 : nullptr, area(me) + 4096 + ctx->probe_max, cnt_own,
                             cnt_peer, bytes, G, iters, ctx->probe_cnt[0], local ? ctx->probe_cnt[lp] : 0,
                             local ? 2 : (initiator ? 1 : 0), ctx->d_rtt, (uint64_t)(ctx->cfg.timeout_s * 1e9),
                             ctx->err_dev, st));
  CK(cudaStreamSynchronize(st));
  CK(cudaStreamDestroy(st));
  ctx->probe_cnt[0] += (uint64_t)G * iters;
  if (local) ctx->probe_cnt[lp] += (uint64_t)G * iters;
  halo_status s = check_err_word(ctx);
  if (s != HALO_OK) return s;
  if (one_way_us) {
    *one_way_us = 0.0;
    if (initiator) {
      std::vector<uint64_t> v(iters);
      CK(cudaMemcpy(v.data(), ctx->d_rtt, sizeof(uint64_t) * iters, cudaMemcpyDeviceToHost));
      std::sort(v.begin(), v.end());
      *one_way_us = (double)v[iters / 2] / 2.0 / 1000.0;
    }
  }
  return HALO_OK;
}

// SM peer-store (mode 0) or copy-engine (mode 1) bandwidth from local rank 0 to
// n concurrent peers (bytes each, back-to-back launches); *gbs = total GB/s out.
halo_status halo_floor_bandwidth_multi(halo_ctx* ctx, const int* peers, int n, size_t bytes, int mode, int iters,
                                       double* gbs) {
  if (!ctx || !peers || n <= 0 || n > kMaxRanks || iters <= 0 || !gbs || (mode != 0 && mode != 1)) return HALO_ERR_ARG;
  if (!ctx->peers_ready) return fail(ctx, HALO_ERR_STATE, "import peers first");
  if (!ctx->probe_max) return fail(ctx, HALO_ERR_STATE, "halo_probe_reserve first");
  bytes = bytes / 16 * 16;
  if (bytes == 0 || bytes > ctx->probe_max) return fail(ctx, HALO_ERR_ARG, "bytes must be in [16, reserved probe bytes]");
  void* dst[kMaxRanks];
  for (int i = 0; i < n; ++i) {
    if (peers[i] < 0 || peers[i] >= ctx->nranks || peers[i] == ctx->first_rank) return HALO_ERR_ARG;
    dst[i] = ctx->peer_scratch[peers[i]] + ctx->probe_off + 4096 + ctx->probe_max;
  }
  const char* src = ctx->scratch[0] + ctx->probe_off + 4096;
  CK(cudaSetDevice(ctx->cfg.device));
  int sms = 148;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, ctx->cfg.device));
  std::vector<cudaStream_t> ss(mode == 1 ? n : 1);
  for (auto& s : ss) CK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  std::vector<cudaEvent_t> ej(ss.size());
  for (auto& e : ej) CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  auto one = [&]() -> cudaError_t {
    if (mode == 0) return launch_bw_multi(src, dst, n, bytes, std::max(1, 8 * sms / n), ss[0]);
    for (int i = 0; i < n; ++i) {
      cudaError_t e = cudaMemcpyAsync(dst[i], src, bytes, cudaMemcpyDefault, ss[i]);
      if (e != cudaSuccess) return e;
    }
    return cudaSuccess;
  };
  for (int i = 0; i < 3; ++i) CK(one());
  // start: every stream past the warm-up; end: every stream's copies done
  CK(cudaEventRecord(e0, ss[0]));
  for (size_t i = 1; i < ss.size(); ++i) CK(cudaStreamWaitEvent(ss[i], e0, 0));
  for (int i = 0; i < iters; ++i) CK(one());
  for (size_t i = 1; i < ss.size(); ++i) {
    CK(cudaEventRecord(ej[i], ss[i]));
    CK(cudaStreamWaitEvent(ss[0], ej[i], 0));
  }
  CK(cudaEventRecord(e1, ss[0]));
  CK(cudaEventSynchronize(e1));
  float ms = 0.f;
  CK(cudaEventElapsedTime(&ms, e0, e1));
  *gbs = (double)bytes * n * iters / (1e-3 * (double)ms) / 1e9;
  CK(cudaEventDestroy(e0));
  CK(cudaEventDestroy(e1));
  for (auto& e : ej) CK(cudaEventDestroy(e));
  for (auto& s : ss) CK(cudaStreamDestroy(s));
  return HALO_OK;
}

halo_status halo_sync(halo_ctx* ctx) {
  if (!ctx) return HALO_ERR_ARG;
  CK(cudaSetDevice(ctx->cfg.device));
  CK(cudaDeviceSynchronize());
  return check_err_word(ctx);
}

halo_status halo_destroy(halo_ctx* ctx) {
  if (ctx && ctx->ce_prof.on) {
    ce_prof_collect(ctx);
    for (size_t j = 0; j < ctx->ce_prof.sum.size(); ++j)
      if (ctx->ce_prof.cnt[j])
        fprintf(stderr, "[halo_ce_profile rank %d] %-9s %8.2f us (n=%d)\n", ctx->first_rank, ctx->ce_prof.agg_names[j].c_str(),
                ctx->ce_prof.sum[j] / ctx->ce_prof.cnt[j], ctx->ce_prof.cnt[j]);
  }
  if (!ctx) return HALO_OK;
  (void)cudaSetDevice(ctx->cfg.device);
  (void)cudaDeviceSynchronize();
  for (void* p : ctx->opened) (void)cudaIpcCloseMemHandle(p);
  if (ctx->plan) (void)cudaFree(ctx->plan);
  for (char* r : ctx->retired) (void)cudaFree(r);
  if (ctx->ctrl) (void)cudaFree(ctx->ctrl);
  if (ctx->d_fshift_tmp) (void)cudaFree(ctx->d_fshift_tmp);
  if (ctx->d_pk_in) (void)cudaFree(ctx->d_pk_in);
  if (ctx->d_pk_out) (void)cudaFree(ctx->d_pk_out);
  if (ctx->d_segs) (void)cudaFree(ctx->d_segs);
  if (ctx->h_small) (void)cudaFreeHost(ctx->h_small);
  if (ctx->d_selcnt) (void)cudaFree(ctx->d_selcnt);
  if (ctx->d_pl) (void)cudaFree(ctx->d_pl);
  if (ctx->h_pl) (void)cudaFreeHost(ctx->h_pl);
  if (ctx->h_pl_cnt) (void)cudaFreeHost(ctx->h_pl_cnt);
  if (ctx->d_pl_scratch) (void)cudaFree(ctx->d_pl_scratch);
  if (ctx->h_recv) (void)cudaFreeHost(ctx->h_recv);
  for (auto e : ctx->pk_ev)
    if (e) (void)cudaEventDestroy(e);
  if (ctx->pk_exec) (void)cudaGraphExecDestroy(ctx->pk_exec);
  if (ctx->pk_cap) (void)cudaStreamDestroy(ctx->pk_cap);
  if (ctx->pk_h2d) (void)cudaStreamDestroy(ctx->pk_h2d);
  if (ctx->pk_d2h) (void)cudaStreamDestroy(ctx->pk_d2h);
  if (ctx->d_small) (void)cudaFree(ctx->d_small);
  if (ctx->h_pin) (void)cudaFreeHost(ctx->h_pin);
  if (ctx->d_mig) (void)cudaFree(ctx->d_mig);
  if (ctx->d_migctrl) (void)cudaFree(ctx->d_migctrl);
  if (ctx->d_planes) (void)cudaFree(ctx->d_planes);
  if (ctx->d_rtt) (void)cudaFree(ctx->d_rtt);
  if (ctx->d_assign) (void)cudaFree(ctx->d_assign);
  if (ctx->d_ce) (void)cudaFree(ctx->d_ce);
  if (ctx->d_stage) (void)cudaFree(ctx->d_stage);
  if (ctx->d_nccl_send) (void)cudaFree(ctx->d_nccl_send);
  if (ctx->nccl_comm) nccl_comm_destroy(ctx->nccl_comm);
  if (ctx->err_host) (void)cudaFreeHost(ctx->err_host);
  (void)cudaGetLastError();
  delete ctx;
  return HALO_OK;
}

}  // extern "C"
