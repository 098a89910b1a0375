// halo_internal.h — device-visible plan structures and PTX memory-ordering
// helpers of libhalo.  Private to libhalo (not part of the C ABI).
//
// Data layout in HBM:
//   x, f      caller-owned, capacity rows x layout floats per DD rank
//   scratch   caller-owned per DD rank, peer-mapped (CUDA IPC):
//               [0, 8192)                ScratchHdr: flags written by peers
//               [4096, ...)              P index maps (int32, capacity each)
//               [..., ...)               P force receive buffers, flag protocol (capacity rows each)
//               [..., ...)               P coordinate LL receive buffers (capacity*layout u64 units)
//               [..., ...)               P force LL receive buffers (capacity*layout u64 units)
//               [..., ...)               P shift-force slot areas (ceil(capacity/32) slots of 6 u64 units)
//             An LL unit is {fp32 value (low word), 32-bit sequence tag (high word)}
//             written with one 8-byte store: single-copy atomic, so a reader that
//             sees the current tag sees the value (no fence, no flag).
//   ctrl      library-owned per process: sequence numbers, completion
//             counters, local "unpacked" flags, set_maps results
//   plan      library-owned per process: RankDev[], PulseDev[], work items
#pragma once
#include <stdint.h>
#include "../../include/halo.h"

namespace halo {

constexpr int kMaxP = HALO_MAX_PULSES;
constexpr int kMaxLocal = HALO_MAX_LOCAL;
constexpr int kMaxRanks = HALO_MAX_RANKS;
constexpr int kAssignSegs = 64;  // atom segments of halo_assign_home's compaction (one CTA per rank and segment)
constexpr int kThreads = 256;          // threads per CTA of the exchange kernels
constexpr int kHdrBytes = 8192;
constexpr int kTraceCTAs = 2048;       // per-CTA timestamps kept for HALO_F_TIMERS
constexpr int kTraceW = 16;            // ... words per CTA: 4 stamps + (tag, end) of its first 6 items
constexpr int kMinItemRows = 32;       // smallest work item (sizes the shift-force slot area)
constexpr int kMaxItemRows = 512;      // largest work item (x items carry their map slice in shared memory)
constexpr int kBulkRowsDefault = 0;  // bulk x pulses from HALO_BULK_ROWS rows; 0: off (measured slower)
constexpr int kMaxTreeRows = 170;      // largest small-tree item (2 passes of 85 roots x 3 components)
constexpr int kTreeRowsOcc = 85;       // tree item size the occupancy (co-resident grid) is computed for
constexpr int kRing = 4;                 // LL kernels: item blocks in flight per CTA (narrow variants)
// LL sequence numbers: the tag of a launch is the low 32 bits of its sequence number;
// values whose tag would be 0 are skipped (a never-written unit is zero), and every
// set_maps zeroes the LL areas, so a unit carries this launch's tag only if this
// launch wrote it (within an NS epoch of < 2^32 launches).
__host__ __device__ __forceinline__ uint64_t ll_seq_next(uint64_t s) {
  ++s;
  return (uint32_t)s == 0 ? s + 1 : s;
}
constexpr int kErrKindStalePlan = 31;        // error-word kind: a replayed graph met a plan of another NS epoch
constexpr int kErrKindBounds = 30;           // error-word kind: a bounds check of the checked build (HALO_BOUNDS_CHECK) failed
constexpr uint32_t kPollTight = 0xffffffffu;  // ExParams.poll_ns: tight polling only, no backoff (HALO_POLL_NS=-1)

// Written by PEERS (system scope).  Each array on its own 128-B lines.
struct __align__(128) ScratchHdr {
  uint64_t flag_x[8];      // flag_x[p] = seq: the x-sender (upper neighbour) finished pulse p
  uint64_t pad0[8];
  uint64_t flag_f[8];      // flag_f[p] = seq: the x-receiver (lower neighbour) pushed slice p
  uint64_t pad1[8];
  uint64_t meta_size[8];   // set_maps: (epoch << 32) | send_size of the upper neighbour
  uint64_t pad2[8];
  uint64_t meta_off[8];    // set_maps: (epoch << 32) | atomOffset granted by the lower neighbour
  uint64_t pad3[8];
  uint64_t ping;           // floor ping-pong flag
  uint64_t pad4[15];
  uint64_t status[kMaxRanks];  // set_maps error agreement: (epoch << 32) | err, per source rank
  uint64_t consumed[8];    // HALO_F_TMA_GET: consumed[p] = seq: the x-sender has read (got) slice p
  // halo_migrate, indexed by the SOURCE / DESTINATION global rank, (epoch << 32) | value:
  uint64_t mig_cnt[kMaxRanks];  // rows source s sends here (release: its staging rows are written)
  uint64_t mig_off[kMaxRanks];  // where they start in source s's staging-out area
  uint64_t mig_ack[kMaxRanks];  // destination t has copied what this rank sent it
  // PP <-> PME (kernels_pme.cu); pme_x_flag / pme_ack live on the PME rank:
  uint64_t pme_nh[kMaxRanks];      // (epoch << 32) | n_home of rank t (halo_pme_setup all-gather)
  uint64_t pme_x_flag[kMaxRanks];  // seq: rank t's home rows are in pme_x
  uint64_t pme_ack[kMaxRanks];     // seq: rank t has read its slice of pme_f
  uint64_t pme_f_flag;             // seq: pme_f holds this step's PME forces (written by the PME rank)
  uint64_t pad5[15];
  uint64_t ns_x[8];        // set_maps: (epoch << 32) | 1: the x-sender's NS-step rows of pulse p landed
  uint64_t pad6[8];
  // bulk x pulses: rows of pulse p the x-sender has stored into this
  // rank's x (one release add per launch, by the item that completed the pulse); the
  // receive's wait item subtracts recv_size once it saw them all: 0 between launches
  uint64_t bulk_x[8];
  uint64_t pad7[8];
};
static_assert(sizeof(ScratchHdr) <= kHdrBytes, "ScratchHdr too large");

// Library-owned control block (device memory, one per process).
struct Ctrl {
  uint64_t seq_x;                       // last completed exchange_x sequence number
  uint64_t seq_f;                       // last completed exchange_f sequence number
  uint32_t done_x, done_f;              // CTAs finished in the current launch
  uint64_t t_start_x, t_end_x, t_start_f, t_end_f;  // globaltimer spans (HALO_F_TIMERS)
  uint64_t span_x, span_f;
  uint32_t cnt_x[kMaxLocal][kMaxP];       // per-pulse CTA completion counters (Alg. 5 blockCompletionCounter)
  uint32_t cnt_push[kMaxLocal][kMaxP];
  uint32_t cnt_unpack[kMaxLocal][kMaxP];
  uint64_t unpacked[kMaxLocal][kMaxP];    // local flag: pulse p scatter-added (gpu scope)
  // set_maps results (read back by the host)
  int32_t send_size[kMaxLocal][kMaxP];
  int32_t n_indep[kMaxLocal][kMaxP];
  int32_t recv_size[kMaxLocal][kMaxP];
  int32_t atom_offset[kMaxLocal][kMaxP];
  int32_t remote_off[kMaxLocal][kMaxP];
  uint32_t dep[kMaxLocal][kMaxP];
  int32_t n_total[kMaxLocal];
  int32_t err[kMaxLocal];                 // set_maps error bits (kErr*)
  int32_t agreed_err[kMaxLocal];          // OR over all ranks after the status exchange
  // HALO_F_TIMERS: per-CTA %globaltimer stamps of the last x (0) / f (1) launch:
  // [start, plan record loaded, items done, exit, item0 tag, item0 end, ..., item5 tag, item5 end]
  // tag = kind << 16 | lrank << 8 | pulse (level)
  uint64_t trace[2][kTraceCTAs][kTraceW];
  // HALO_DEBUG & kCountNotify (pin G4): system-scope flag stores per (x/f, local rank, pulse), cumulative
  uint32_t notify[2][kMaxLocal][kMaxP];
  // PP <-> PME (kernels_pme.cu)
  uint64_t seq_pme_x, seq_pme_f;
  uint32_t done_pme[2];
  uint32_t cnt_pme[2][kMaxLocal];
  int32_t pme_nh[kMaxLocal][kMaxRanks];   // halo_pme_setup: n_home of every rank, seen by local rank l
  // fused x+f launch: x items finished in the current launch (acq_rel increments; the
  // last one resets it and releases xf_done = the launch's x sequence number, which
  // the tree items acquire: the non-bonded kernel's slot, Alg. 2).  Own 128-B lines.
  uint32_t xf_cnt;
  uint32_t pad_xf0[31];
  uint32_t bulk_rows[kMaxLocal][kMaxP];  // rows of bulk pulse (l, p) stored in the current launch (gpu scope)
  uint64_t xf_done;
  uint64_t pad_xf1[15];
};

enum : int32_t { kErrCapacity = 1, kErrGeometry = 2, kErrMap = 4,
                 kVoteCE = 256,     // not errors: votes ORed by the status exchange (HALO_F_AUTO_TRANSPORT,
                 kVoteRows = 4096,  // work-item size one-hot: kVoteRows << log2(R / kMinItemRows))
                 kVoteRowsMask = 31 * 4096};

// ---------------------------------------------------------------- halo_migrate
// (csrc/kernels_ns.cu).  The stencil of a rank = the distinct
// ranks of the cells c + delta, delta in {-1,0,1}^3 (periodic): the only ranks a
// home atom may move to between NS steps (R30), and, symmetrically, the only
// ranks it can receive atoms from.  Staging area rows are SoA: x (layout
// floats), v (layout floats), gid (int32), capacity rows each.
constexpr int kStencil = 27;
constexpr int kMigBlocks = 64;     // classify CTAs per rank (contiguous row ranges, stable order)
struct MigRank {
  float* x;                   // own x (rows re-written in place by the merge)
  int32_t* gid;               // own gid array (caller's)
  float* v;                   // payload rows or nullptr
  char* stage_out;            // own staging-out (grouped by destination, ascending gid per group)
  char* stage_in;             // own staging-in (the lists received, concatenated)
  ScratchHdr* hdr;            // own header
  ScratchHdr* nb_hdr[kStencil];      // headers of the stencil ranks
  const char* nb_stage[kStencil];    // their staging-out areas (peer pointers)
  int nb_rank[kStencil];
  int n_nb;                   // distinct stencil ranks (self included)
  int rank;
  int n_home;
  int pad;
};
struct MigParams {
  const MigRank* r;           // n_local entries (device)
  Ctrl* ctrl;
  const double* planes;       // planes[d*(kMaxRanks+1) + k] = float64(L_d)*k/grid[d], k = 0..grid[d] (R3)
  int grid[3];
  float box[3];
  int n_local;
  int layout;
  int has_v;
  int capacity;
  uint32_t epoch;
  int* err_host;
  uint64_t timeout_ns;
};
// halo_assign_home (kernels_ns.cu)
struct AssignParams {
  const double* planes;  // as MigParams::planes
  int grid[3];
};
// per local rank results of the migration kernels
struct MigCtrl {
  int32_t out_cnt[kMaxLocal][kStencil];   // rows this rank sends to stencil rank k (self included)
  int32_t out_off[kMaxLocal][kStencil];
  int32_t in_cnt[kMaxLocal][kStencil];    // rows received from stencil rank k
  int32_t in_src_off[kMaxLocal][kStencil];  // ... starting there in its staging-out
  int32_t in_off[kMaxLocal][kStencil + 1];  // prefix of in_cnt: list k is rows [in_off[k], in_off[k+1]) of staging-in
  int32_t err[kMaxLocal];
  // classify split over kMigBlocks CTAs per rank (contiguous row ranges): per-CTA
  // group counts, then their exclusive prefix within each group
  int32_t blk[kMaxLocal][kMigBlocks][kStencil];
};

// HALO_DEBUG bits: protocol mutations for the dependency-safety tests (G3);
// never set in production.
enum : uint32_t { kMutateXNoWait = 16u, kMutateFNoWait = 32u, kCountNotify = 64u, kFenceAfterPeerStores = 128u,
                   kLocalSink = 256u,  // timing experiment: peer stores go to own memory, receivers do not wait
                   // G3 (ii): paper protocol, the a4/a5 pulse flags without release semantics (no
                   // per-CTA fence, relaxed counter, relaxed flag store)
                   kMutateRelaxedFlags = 512u,
                   // G3 (iv): paper protocol, the paper-literal firstDependentPulse (x0 -> y0
                   // only): a dependent item waits only for pulse p-1, not its whole dependency set (R9)
                   kMutatePaperQ9 = 1024u,
                   // slow producer (not a mutation; widens races for the G3 tests): the pulse-0
                   // x send items of ONE rank (the one sending to DD rank 0) sleep ~20 us before their
                   // data stores, so rank 0's z0 rows arrive after everything else
                   kDelayPulse0 = 2048u,
                   // fshift partials accumulated in fp32 (shows the 1e-12 * sum|terms| bound catches it)
                   kMutateFshiftF32 = 4096u,
                   // timing experiment: per-CTA stamps inside the first tree item (trace slots 10-13)
                   kTraceDetail = 8192u};

struct RankDev {
  float* x;                 // own x (capacity rows)
  float* f;                 // own f
  ScratchHdr* hdr;          // own scratch header
  int32_t* maps;            // own maps region (P slots of map_stride ints)
  float* fbuf;              // own force receive buffers (P slots of fbuf_stride floats)
  int n_home;
  int n_total;
  int rank;                 // global DD rank
  int pad;
};

struct PulseDev {
  const int32_t* map;       // own map of this pulse (send_size entries, ascending)
  float* x_dst;             // receiver's x + remote_off rows (peer pointer)
  uint64_t* flag_x_dst;     // &receiver.hdr->flag_x[p]
  float* fbuf_dst;          // x-sender's force receive buffer of pulse p (peer pointer)
  uint64_t* flag_f_dst;     // &x-sender.hdr->flag_f[p]
  const float* fbuf_own;    // own force receive buffer of pulse p
  float shift[3];           // +L_d on the dim axis when has_shift (R25)
  int has_shift;
  int dim;
  int send_size;
  int n_indep;              // entries < n_home (Alg. 4 depOffset = n_home, R8)
  int atom_offset;          // own receive range of pulse p
  int recv_size;
  uint32_t dep_x;           // pulses q < p whose receive range map_p reads (R9)
  uint32_t fdep;            // pulses q > p whose maps read slice p: push(p) waits unpacked[q]
  uint32_t chain;           // pulses q > p with send_size > 0 (deterministic unpack order)
  uint64_t* xll_dst;        // receiver's coordinate LL buffer of pulse p (peer pointer), LL protocol
  uint64_t* fll_dst;        // x-sender's force LL buffer of pulse p (peer pointer), LL protocol
  const float* f_src;       // HALO_F_TMA_GET: the x-receiver's f at its remote_off rows (peer pointer)
  uint64_t* consumed_dst;   // HALO_F_TMA_GET: &x-receiver.hdr->consumed[p]
  int n_items_x;
  int n_items_push;
  int n_items_unpack;
  int pad;
};

enum : uint8_t { kItemXIndep = 0, kItemXDep = 1, kItemPush = 2, kItemUnpack = 3, kItemXRecv = 4, kItemGather = 5,
                 kItemFshift = 6, kItemXSend = 7, kItemTree = 8, kItemTreeG = 9, kItemXWait = 10 };
constexpr uint8_t kHomeLevel = 0xff;   // Item.pulse of gather items over home rows

struct Item {
  uint16_t lrank;
  uint8_t pulse;
  uint8_t kind;
  uint32_t begin;
  uint32_t end;
};

// LL protocol work records.  Ranks of this process that share a GPU form one
// HOP GROUP: a pulse between two ranks of a group is not a
// transport hop, so the plan resolves it on the host at the NS step — every halo
// row an item writes names its ORIGIN (a home row, or the LL unit in which it
// crossed from another group) plus the periodic shifts of the pulses it went
// through, and the force halo of a group is a set of TREES (a row, the images it
// was sent as, their images, ...) each folded by one thread in the oracle's
// order.  Only pulses between groups move LL units and wait for their tags.
// Each item's block starts with one 128-B record followed by its entries (x),
// or its roots and nodes (f); blocks are fixed-size and bulk-loaded into a ring
// of shared-memory slots.
struct LocalBase {          // per local rank, copied to shared memory at kernel start
  float* x;                 // own x
  float* f;                 // own f
  uint64_t* xll;            // own coordinate LL area (slot q at + q*ll_stride)
  uint64_t* fll;            // own force LL area
  int32_t recv_off[kMaxP];  // own receive ranges (rows)
  int32_t n_home;           // home rows (the x launch's L2 prefetch)
  int32_t pad;
};
static_assert(sizeof(LocalBase) == 64, "LocalBase");

// x entry (8 B): the origin of one halo row an item writes.
//   row   origin row in x of local rank l (kind X), or the unit row i of l's
//         coordinate LL slot q (kind LL: the row crossed from another group there)
//   kq    bit 7: LL origin, bits 0-2: q
//   mask  pulses whose +L shift the row picked up after its origin, ascending
//         (R25: one fp32 add of the shift vector per such pulse)
struct XEnt {
  uint32_t row;
  uint8_t l, kq, mask, pad;
};
static_assert(sizeof(XEnt) == 8, "XEnt");

struct __align__(128) XRec {
  uint8_t kind;             // kItemXSend / kItemXRecv / kItemXWait
  uint8_t pulse;
  uint16_t lrank;
  uint32_t n_units;         // rows * layout
  uint32_t begin;           // send: first send index (destination row remote_off + begin + e)
  uint32_t cls;             // dependency class (plan order; trace only)
  float* dst_x;             // send to a rank of this group, or a bulk pulse: its x at row remote_off (direct store)
  uint64_t* dst_ll;         // send to another group: the receiver's coordinate LL slot p
  float shiftL[kMaxP];      // L_{d_q}: the shift of pulse q (applied iff the entry's mask has q)
  uint8_t pdim[kMaxP];      // d_q
  uint8_t pad0[2];
  uint64_t* ll;             // recv: own LL slot p + begin*W
  float* xdst;              // recv: own x + (recv_off_p + begin)*W
  uint32_t epoch;           // NS epoch of the plan (a graph captured before a later set_maps is refused)
  uint32_t pad2;
  uint64_t* bulk;           // bulk pulse: send: &receiver.hdr->bulk_x[p] (release-add the item's rows);
                            // wait (n_units = recv_size rows): &own hdr->bulk_x[p]
  uint32_t bulk_total;      // bulk send: rows of the whole pulse (the item completing them releases them all)
  uint8_t pad1[128 - 100];
};
static_assert(sizeof(XRec) == 128, "XRec must be one 128-B line");

// f trees.  value(node) = f[node] + sum over children, pulses descending (R15);
// a node is a row of f of local rank l (kind F) or the LL unit in which a child
// in another group pushed its value (kind LL: unit row i of l's force LL slot q).
// F nodes with children store their value.  A root with its parent in another
// group pushes its value to `push` (the parent's force LL slot) — Alg. 5 DEP_MGMT
// across groups.  Every edge (parent, child) lies in the tree of its parent, so
// the shift force of the edge (R13: the parent's rank wrapped in the edge's pulse)
// is added there, into one of the item's buckets (targets 3 * local rank + dim).
//
// Small trees (<= kFastNodes nodes: every tree when P <= 3) — kItemTree blocks:
// [GRec | TRoot x rows | node rows (8 x u32: row | l << 24, depth-first, children
// in descending pulse order) x rows]; the tree's shape lives in the root record
// as 4-bit fields, so a thread folds its tree in registers.
struct TRoot {
  uint64_t* push;           // or null
  uint32_t par;             // nibble k: index of node k's parent (0xf: none / the root)
  uint32_t bucket;          // nibble k: the item's shift-force bucket of the edge into node k (kFsNone: none)
  uint32_t q;               // nibble k: pulse of node k when it is an LL node
  uint8_t nn;               // nodes
  uint8_t llmask;           // bit k: node k is an LL node
  uint8_t stmask;           // bit k: node k (F, with children) stores its folded value
  uint8_t pad0;
  uint32_t post;            // nibble e: the e-th non-root node in postorder (nn - 1 of them)
  uint32_t pad1;
};
static_assert(sizeof(TRoot) == 32, "TRoot");
// Larger trees — kItemTreeG blocks: [GRec | TRootG x rows/8 | TNode x (rest)].
struct TRootG {
  uint64_t* push;
  uint32_t node_begin;
  uint16_t n_nodes;
  uint16_t pad;
};
static_assert(sizeof(TRootG) == 16, "TRootG");
struct TNode {
  uint32_t il;              // idx | l << 24 (F: row; LL: unit row i; rows < 2^24)
  uint8_t kq;               // bit 7: LL node, bits 0-2: its pulse q, bits 3-6: the item's shift-force
                            // bucket of the edge from the parent (kFsNone: none, kFsDirect: use fs)
  uint8_t parent;           // index of the parent node in the tree (0xff: the root)
  uint8_t flags;            // bit 0: store the folded value; bits 1-7: depth
  uint8_t fs;               // shift-force target of that edge (3 * parent's local rank + dim), or 0xff
};
static_assert(sizeof(TNode) == 8, "TNode");
constexpr int kMaxDepth = kMaxP + 1;
constexpr int kFastNodes = 8;
constexpr int kMaxBuckets = 8;     // distinct shift-force targets per f item (reduced in shared memory)
constexpr uint8_t kFsNone = 15, kFsDirect = 14;
constexpr uint32_t kMaxRows = 1u << 24;

struct __align__(128) GRec {
  uint8_t kind;             // kItemTree / kItemTreeG
  uint8_t level;            // dependency class
  uint16_t lrank;
  uint32_t n_units;         // roots * layout
  uint32_t n_roots, n_nodes;
  uint8_t n_buckets;        // shift-force buckets of this item's edges
  uint8_t bucket_fs[kMaxBuckets];  // their targets (3 * local rank + dim)
  uint8_t pad0[3];
  uint32_t epoch;           // NS epoch of the plan (as XRec.epoch)
  uint8_t pad[128 - 16 - 1 - kMaxBuckets - 3 - 4];
};
static_assert(sizeof(GRec) == 128, "GRec must be one 128-B line");

struct ExParams {
  const RankDev* ranks;
  const PulseDev* pulses;   // [n_local * P]
  const Item* items;
  int n_items;
  int n_tail;               // LL f: trailing items that get one dedicated CTA each (shift-force combines)
  int n_local;
  int P;
  int p_lo, p_hi;           // pulse range of this launch (set_maps runs one pulse at a time)
  Ctrl* ctrl;
  int* err_host;            // host-mapped error word (timeout)
  uint64_t timeout_ns;
  unsigned flags;
  double* fshift;           // [n_local][3][3] or nullptr
  int accumulate;
  uint32_t poll_ns;         // __nanosleep between flag polls (0 = tight, then backoff; kPollTight = tight only)
  uint64_t ll_stride;       // u64 units per pulse slot of the LL receive buffers
  uint32_t debug;           // HALO_DEBUG experiment bits (0 in production)
  uint32_t fsp_slots;       // shift-force slots per pulse in each rank's scratch
  uint64_t seq;             // LL: this launch's sequence number by value (eager launches; 0 = read
                            // ctrl->seq_x/f + 1 in the kernel: graph-captured launches, R17)
  const char* xblk;         // LL x item blocks: [XRec | map slice, item_rows int32], 128 + 4*item_rows B each
  const char* fblk;         // LL f item blocks: [GRec | task records, item_rows x 32 B], 128 + 32*item_rows B each
  int item_rows;            // LL: x entries per item (x block = 128 + 8 * item_rows B)
  int tree_rows;            // LL: roots per small-tree item (f block = 128 + 64 * tree_rows B)
  int n_items_x;            // fused launch: items [0, n_items_x) are x items, then the f items
  int ring;                 // LL: item-block ring slots per CTA
  uint64_t seq_f;           // fused launch: the f sequence number by value (0 = read ctrl->seq_f + 1)
  int delay_rank;           // HALO_DEBUG kDelayPulse0: the DD rank whose pulse-0 sends are slowed
  const LocalBase* lbase;   // LL: [n_local] (copied to shared memory by every CTA)
  // x launch: L2 prefetch (before griddepcontrol.wait) of the f kernel's item blocks and
  // of the home x rows the sends read, spread over the CTAs (0 bytes = off, HALO_PREFETCH=0)
  const char* pf_f;
  uint64_t pf_f_bytes;
  int pf_x;                 // 1: prefetch every local rank's home x rows
  uint32_t plan_epoch;      // LL: the NS epoch whose item blocks this launch expects (records carry theirs)
  int all_local;            // LL: every pulse of every local rank stays in this hop group (no LL units)
  int cap_rows;             // rows of every x / f buffer (the checked build's bounds)
};

// GPU plan build of the LL protocol (set_maps, P <= 3: every force tree has <= 8
// nodes): the x send items and the force trees are built by kernels_plan.cu from the
// device-resident maps; the host only fills this descriptor (per (local rank, pulse)
// relations, pointers, and after the counting pass the item offsets).
struct PlanLQ {
  float* dst_x;             // send of (l, q) to a rank of this group: its x + remote_off rows
  uint64_t* dst_ll;         // ... to another group: the receiver's coordinate LL slot q
  uint64_t* push;           // rows of (l, q) whose x-sender is in another group: its force LL slot q
  uint64_t* bulk;           // bulk pulse: &receiver.hdr->bulk_x[q] (dst_x is then its x)
  int32_t rcv_l;            // the receiver's (lower neighbour) local index if in this group, else -1
  int32_t snd_l;            // the sender's (upper neighbour) local index if in this group, else -1
  int32_t remote_off;       // where the receiver put this rank's pulse-q rows
  int32_t atom_offset;      // own receive range of pulse q
  int32_t send_size, recv_size;
  uint8_t wraps;            // this rank adds +L_{d_q} in pulse q (R1, R25)
  uint8_t efs;              // 3 * l + d_q if wraps, else 0xff (shift-force target of its edges, R13)
  uint8_t pad[6];
};
struct PlanDev {
  int L, P, W, R, RT, cap, map_stride;
  uint32_t epoch;
  uint32_t XB, FB;          // item block sizes
  PlanLQ lq[kMaxLocal][kMaxP];
  int32_t n_home[kMaxLocal], n_total[kMaxLocal];
  const int32_t* maps[kMaxLocal];
  uint8_t bucket_fs[kMaxLocal][kMaxBuckets];  // shift-force targets of every tree rooted at rank l
  uint8_t n_buckets[kMaxLocal];
  float shiftL[kMaxP];
  uint8_t pdim[kMaxP];
  uint8_t pad0[2];
  // device scratch ([L][cap] rows)
  uint64_t* org;            // x origin of every row: row | l << 24 | kq << 32 | mask << 40 | cls << 48
  int32_t* child;           // [L][cap][P]: entry of row t in map q, or -1
  uint8_t* rcls;            // tree class of a root row, 0xff = not a root
  uint8_t* rmask;           // its shift-force targets, a mask over bucket_fs[l]
  uint32_t* imask;          // per f item: OR of its trees' masks (the item's buckets)
  int32_t* bcnt;            // [L][nblk][P + 1] roots per class in each CTA's rows (k_plan_roots)
  int32_t* boff;            // ... their exclusive prefix over the CTAs of a rank (k_plan_rank)
  int nblk;                 // CTAs per local rank of the per-row kernels
  int32_t* xcnt;            // [P][L][P + 1] send items per class (counting pass, zeroed before)
  int32_t* xlast;           // [P*L][xnch]: last class change in each kPB-entry chunk of a map (or -1)
  int32_t* xlstart;         // ... last item start in the chunk
  int32_t* xccnt;           // [P*L][xnch][kMaxP + 1]: item starts per class in the chunk
  int xnch;                 // chunks per map
  int32_t* rcnt;            // [L][P + 1] roots per class
  // second pass (after the counts): item offsets and the block areas
  int32_t xoff[kMaxP + 1][kMaxP][kMaxLocal];  // first x item of (class, pulse, local rank)
  int32_t foff[kMaxP + 1][kMaxLocal];         // first f item of (class, local rank)
  int32_t fcnt[kMaxP + 1][kMaxLocal];         // roots of (class, local rank)
  char* xblk;
  char* fblk;
  int nx_send, nf;          // send items / f items (the checked build's bounds of the block writes)
  int* err_host;            // host-mapped error word (the checked build reports failed checks there)
};

// halo_step_host_packed: one contiguous copy between a packed staging buffer and
// one local rank's rows (4-B words).
struct SegCopy {
  const uint32_t* src;
  uint32_t* dst;
  size_t words;
};

// Copy-engine path (HALO_F_CE_PATH, kernels_ce.cu): one entry per (pulse, local rank).
struct CeEnt {
  const int32_t* map;       // map_p (send_size entries)
  const float* src;         // pack: own x; unpack: own force receive buffer of pulse p
  float* dst;               // pack: staging rows; unpack: own f
  int n;                    // send_size_p
  int pack;                 // pack: 1 iff a gather is needed (map not one contiguous run, or shifted)
  int has_shift;
  int dim;
  float shift[3];
  int pad;
};

struct CeSyncParams {
  uint64_t* seq_slot;       // &ctrl->seq_x or &ctrl->seq_f
  uint64_t* dst[kMaxLocal]; // flag on the peer this local rank's copy went to
  const uint64_t* own[kMaxLocal];  // own flag of the pulse
  int n_local;
  int publish;              // last sync of the exchange: store seq into seq_slot
  int kind;                 // 0 = x, 1 = f (timeout code)
  int pulse;
  int* err_host;
  uint64_t timeout_ns;
};

struct SelParams {
  const RankDev* ranks;
  Ctrl* ctrl;
  int p;                    // pulse index
  int dim;
  double rc;
  const int32_t* cand;      // [n_local][2] candidate row range
  const double* b_lo;       // [n_local][3] lower planes b_d[c_d] (the pulse's dim is used)
  const double* home_lo;    // [n_local][3] (home check; nullptr = skip)
  const double* home_hi;    // [n_local][3]
  const double* b_up;       // [n_local][3] upper planes b_d[c_d+1]: rounded zones (R31); nullptr = slab
  int kfirst;               // 1: the dim's first pulse (candidates [0, n_total)); 0: the rows received
                            // in pulse p-1 (cand == nullptr: both from the device-side handshake results)
  uint32_t epoch;
  uint32_t wait_mask[kMaxLocal];   // pulses q < p whose x-sender is in another process: wait ns_x[q]
  int* err_host;
  uint64_t timeout_ns;
  int32_t* sel_cnt;         // [n_local][max_chunks] selected rows per 1024-row chunk (count pass)
  int max_chunks;           // chunks per local rank (>= candidates / 1024)
  double rc2;               // float64(rc)^2 (R31)
  int decomposed_mask;      // bit d set iff grid[d] > 1
  int map_stride;
  int layout;
};

// set_maps: the coordinate exchange of one pulse (k_ns_x), driven by the device-side
// sizes and offsets of the handshake (no host round trip per pulse).
struct NsXParams {
  const RankDev* ranks;
  Ctrl* ctrl;
  int p;
  int dim;
  int map_stride;
  int n_local;
  uint32_t epoch;
  float* dst_x[kMaxLocal];         // the receiver's x (peer pointer; rows at remote_off)
  uint64_t* flag_dst[kMaxLocal];   // the receiver's ns_x[p] when it is in another process, else null
  float shift[kMaxLocal];          // +L_d when the sender wraps (R1, R25), applied iff has_shift
  int has_shift[kMaxLocal];
  uint32_t wait_mask[kMaxLocal];   // pulses q < p whose x-sender is in another process (forwarded rows)
  int* err_host;
  uint64_t timeout_ns;
  int cap;                         // rows of every x buffer (the checked build's bounds)
};

struct NsWaitParams {
  int n_local;
  uint32_t epoch;
  ScratchHdr* own[kMaxLocal];
  uint32_t mask[kMaxLocal];        // pulses whose x-sender is in another process
  int* err_host;
  uint64_t timeout_ns;
};

struct HsParams {
  Ctrl* ctrl;
  int p;
  uint32_t epoch;
  int capacity;
  int n_local;
  ScratchHdr* own[kMaxLocal];
  uint64_t* size_dst[kMaxLocal];   // &lower.hdr->meta_size[p]
  uint64_t* off_dst[kMaxLocal];    // &upper.hdr->meta_off[p]
  int* err_host;
  uint64_t timeout_ns;
  uint32_t sys_mask;               // bit l: size_dst[l] in another process; bit 16+l: off_dst[l] (else gpu-scope release)
};

struct StatusParams {
  Ctrl* ctrl;
  uint32_t epoch;
  int nranks;
  int n_local;
  int first_rank;
  ScratchHdr* own[kMaxLocal];
  ScratchHdr* all[kMaxRanks];       // every rank's scratch header (local or peer-mapped)
  int* err_host;
  uint64_t timeout_ns;
  // votes that ride on the exchange (computed on the device from this process's
  // handshake results, identically in every CTA): the copy engine if some pulse sends
  // >= ce_bytes (auto_tr), and the work-item size (kVoteRows << log2(R / 32))
  int vote;                        // 0: no votes (halo_migrate, PME setup: errors only)
  int P, W, auto_tr, rows_fixed;   // rows_fixed: R given (HALO_ITEM_ROWS), else 0
  int64_t ctas;                    // co-resident CTAs the item size is chosen for
  uint64_t ce_bytes;
  int all_local;                   // every rank in this process: gpu-scope releases suffice
};

// PP <-> PME redistribution (halo_pme_*, kernels_pme.cu)
struct PmeRank {
  const float* x;           // own x (home rows sent)
  float* f;                 // own f (home rows receive the PME forces)
  ScratchHdr* hdr;          // own header
  int n_home;
  int off;                  // first row of this rank in pme_x / pme_f
  int rank;
  int pad;
};
struct PmeParams {
  PmeRank r[kMaxLocal];
  ScratchHdr* all_hdr[kMaxRanks];
  ScratchHdr* pme_hdr;      // the PME rank's header (peer)
  float* pme_x;             // the PME rank's coordinate / force buffers (peer)
  float* pme_f;
  Ctrl* ctrl;
  int n_local, nranks, layout, hosts_pme, accumulate;
  uint32_t epoch;
  int* err_host;
  uint64_t timeout_ns;
};

}  // namespace halo
