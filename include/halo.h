/*
 * halo.h — C ABI of libhalo.so: the per-step eighth-shell (neutral-territory)
 * domain-decomposition halo exchange of arXiv 2509.21527, B200-native.
 *
 * Citations: P:<n> = line n of the paper text; R<n> = a reading of
 * the paper recorded in DESIGN.md ("Readings").
 *
 * Model (Alg. 1):
 *   - A periodic rectangular box L[3] is split into grid[0] x grid[1] x grid[2]
 *     cells ("DD ranks"), rank = (cx*np_y + cy)*np_z + cz (R5).
 *   - Each DD rank owns a coordinate array x and a force array f of `capacity`
 *     rows.  Rows [0, n_home) are its home atoms; halo rows received in the
 *     coordinate halo are appended contiguously after them, pulses in global
 *     order z -> y -> x (R12).
 *   - A row is `layout` floats: 3 (12-byte float3, GROMACS rvec) or 4 (16-byte
 *     float4; x: w copied, never shifted; f: w accumulated like x,y,z) (R25).
 *   - One PROCESS drives one GPU and hosts a contiguous block of DD ranks
 *     ("local ranks"): ranks [proc*R/nprocs, (proc+1)*R/nprocs), R = nranks.
 *     With nprocs == nranks this is the paper's one-rank-per-GPU setup; with
 *     nprocs < nranks several DD ranks share one GPU and are executed by the
 *     same kernel launch (never as separate spinning launches).
 *
 * Conventions for every call:
 *   - Returns halo_status; HALO_OK == 0.  No C++ exception crosses the ABI.
 *   - On error the ctx keeps a message readable with halo_last_error().
 *   - `stream` is a cudaStream_t passed as void* (NULL = legacy default stream).
 *   - Device pointers are plain CUDA device pointers (e.g. torch data_ptr()).
 *   - A ctx is not thread-safe; use one ctx per process.
 *   - COLLECTIVE calls must be made by every process, the same number of
 *     times, in the same order (they synchronise through device-side flags).
 */
#ifndef HALO_H_
#define HALO_H_

#include <stddef.h>
#include <stdint.h>

#if defined(__GNUC__)
#define HALO_API __attribute__((visibility("default")))
#else
#define HALO_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

#define HALO_ABI_VERSION 1
#define HALO_MAX_PULSES 6     /* up to two pulses per dimension */
#define HALO_MAX_RANKS 64     /* DD ranks per job supported by this build */
#define HALO_MAX_LOCAL 64     /* DD ranks per process */

typedef struct halo_ctx halo_ctx; /* opaque */

typedef enum {
  HALO_OK = 0,
  HALO_ERR_ARG = 1,         /* bad argument (NULL, out of range, misaligned) */
  HALO_ERR_GEOMETRY = 2,    /* invalid grid/box/cutoff/pulses, or a home atom outside its cell */
  HALO_ERR_CAPACITY = 3,    /* n_home + sum(recv) > capacity on some rank (agreed by all ranks) */
  HALO_ERR_STATE = 4,       /* call out of order (e.g. exchange before set_maps) */
  HALO_ERR_CUDA = 5,        /* a CUDA runtime error; text in halo_last_error() */
  HALO_ERR_PEER = 6,        /* IPC import failed or a peer blob is inconsistent */
  HALO_ERR_TIMEOUT = 7,     /* a device-side wait exceeded the timeout (protocol bug or dead peer) */
  HALO_ERR_UNSUPPORTED = 8  /* valid request this build does not support */
} halo_status;

/* Flags (halo_config.flags). */
#define HALO_F_DETERMINISTIC  0u        /* the default (no bit): forces added in the oracle's fixed order
                                           (pulses descending, one fp32 RNE add per image), bit-exact (R15) */
#define HALO_F_ATOMIC_UNPACK  (1u << 0) /* unordered f unpack (paper's atomicAdd); default is the
                                           deterministic pulse-descending order (bit-exact vs oracle, R15) */
#define HALO_F_NO_HOME_CHECK  (1u << 1) /* skip the "home atoms lie in their cell" check in halo_set_maps */
#define HALO_F_GPU_FENCE      (1u << 2) /* per-CTA gpu-scope release + sys-scope release by the last CTA
                                           only (the paper's P:425-427 scheme); default: per-CTA sys fence */
#define HALO_F_TIMERS         (1u << 3) /* record %globaltimer spans of each exchange kernel */
#define HALO_F_PAPER_FLAGS    (1u << 4) /* the paper's per-pulse signalling (Alg. 5: per-CTA completion counter,
                                           one release flag per pulse, receiver acquire-wait; force slices
                                           pushed then scatter-added).  Default: the LL protocol (every 8-B
                                           store carries a 32-bit sequence tag; row-level forwarding; the
                                           force halo is a deterministic gather) */
#define HALO_F_CE_PATH        (1u << 5) /* copy-engine path (north_star: "a copy-engine path covers large
                                           contiguous pulses"): per pulse, a local gather kernel packs the send
                                           rows (skipped when the map is one contiguous unshifted run), ONE
                                           cudaMemcpyAsync moves them over NVLink, a one-thread-per-rank kernel
                                           releases the pulse flag on the peer and acquire-waits its own; forces:
                                           CE copy of the contiguous halo slice, flag, ordered scatter-add.
                                           ~3 launches + L copies per pulse; bit-exact like the default.
                                           Takes precedence over HALO_F_PAPER_FLAGS (set_maps uses its kernels). */
#define HALO_F_L2_PERSIST     (1u << 6) /* LL protocol: keep the static plan (work-item blocks: records, map
                                           slices, gather task records; rebuilt only by set_maps) in the
                                           persisting L2 carve-out (access-policy window on the exchange
                                           launches; raises cudaLimitPersistingL2CacheSize device-wide to the
                                           plan size if lower).  Coordinates and forces are never persisted. */
#define HALO_F_TMA_STORE      (1u << 7) /* with HALO_F_PAPER_FLAGS only: the x put as the paper's warp-leader TMA
                                           store (Alg. 3): each warp packs a 32-row chunk into
                                           shared memory, one cp.async.bulk store writes it into the receiver's
                                           x over NVLink.  HALO_ERR_UNSUPPORTED with the LL or copy-engine path. */
#define HALO_F_TMA_GET        (1u << 8) /* with HALO_F_PAPER_FLAGS only: the force halo as the paper's receiver-
                                           driven get (Alg. 6): the x-receiver only signals
                                           that its halo slice p is final; the x-sender acquire-waits, bulk-loads
                                           (TMA) each chunk of the slice from the peer's f into shared memory and
                                           scatter-adds it (same order, same bits as the push).  The reader then
                                           acks each slice (one flag per pulse), and an exchange_f launch
                                           completes only after its slices were read, so f may be overwritten
                                           once the stream passes exchange_f (DESIGN R28).  f is peer-mapped. */
#define HALO_F_ROUNDED_ZONES  (1u << 9) /* halo_set_maps: GROMACS-style rounded zones (SURVEY f2 variant, R31):
                                           a row beyond this rank's upper face in another dim is sent only if
                                           its float64 distance to the receiver's cell, dd^2 + sum (x_d' -
                                           b_d'[c_d'+1])^2 over the dims it lies beyond, is < rc^2; default: the
                                           slab criterion (box-shaped zones, R2).  Fewer halo rows in 2D/3D. */
#define HALO_F_AUTO_TRANSPORT (1u << 10) /* pick the transport per NS epoch by pulse size — the LL
                                           protocol (latency regime) unless some rank's pulse sends at least
                                           HALO_AUTO_CE_BYTES (env, default 4 MiB: the measured LL / copy-engine
                                           crossover on B200), then the copy-engine path.  Decided
                                           collectively in halo_set_maps (all ranks agree); results identical.
                                           Not combinable with PAPER_FLAGS / CE_PATH / TMA_*.  */
#define HALO_F_NCCL_BASELINE  (1u << 11) /* halo_exchange_x / halo_exchange_f run the NCCL send/recv schedule
                                           (halo_nccl_exchange_x / _f; needs halo_nccl_init): the BASELINE the
                                           fused kernels are measured against, not a
                                           product transport.  set_maps still builds the maps on the GPU. */

typedef struct {
  int grid[3];        /* cells per dim (np_x, np_y, np_z), each >= 1 */
  float box[3];       /* box lengths L_x, L_y, L_z in nm (rectangular) */
  float cutoff;       /* communication cutoff rc in nm: 0 < rc < min(L)/2 */
  int pulses[3];      /* pulses per dim: >= 1 iff grid[d] > 1, <= grid[d]-1, pulses*L/grid >= rc */
  int layout;         /* 3 or 4 floats per row of x and f */
  int capacity;       /* rows of every registered x and f array (home + halo) */
  int device;         /* CUDA device ordinal this process uses */
  unsigned flags;     /* HALO_F_* */
  int nprocs;         /* processes (GPUs) in the job; nranks % nprocs == 0 */
  int proc;           /* this process, 0 <= proc < nprocs */
  double timeout_s;   /* bound of every device-side wait; <= 0 selects 10 s */
} halo_config;

/* Validate `cfg` and create a context (PulseData/CommContext).
 * Geometry is validated before any CUDA call: an invalid config returns
 * HALO_ERR_GEOMETRY/HALO_ERR_ARG without touching the GPU.  Then selects
 * cfg->device and allocates the library-owned control block.
 * *out receives the ctx (NULL on error; use halo_strerror). */
HALO_API halo_status halo_init(const halo_config* cfg, halo_ctx** out);

/* Host-only query (no CUDA call, usable before choosing a device): validates
 * `cfg` like halo_init and returns the DD ranks this process would host
 * ([*first_rank, *first_rank + *n_local)), the pulse count and order (dims[p]
 * in 0/1/2 = x/y/z, z -> y -> x; dims sized HALO_MAX_PULSES or NULL)
 * and halo_scratch_bytes().  Any output pointer may be NULL. */
HALO_API halo_status halo_query_config(const halo_config* cfg, int* first_rank, int* n_local, int* npulse,
                                       int* dims, size_t* scratch_bytes);

/* DD ranks hosted by this process: [*first_rank, *first_rank + *n_local). */
HALO_API halo_status halo_local_ranks(const halo_ctx* ctx, int* first_rank, int* n_local);

/* Total pulses (sum of cfg.pulses) and the global pulse order: dims[p] = 0/1/2
 * (x/y/z), in z -> y -> x order.  dims may be NULL. */
HALO_API halo_status halo_pulse_order(const halo_ctx* ctx, int* npulse, int* dims);

/* Bytes of the caller-owned `scratch` device buffer each local rank needs
 * (flags, handshake slots, index maps, force receive buffers; 256-B aligned). */
HALO_API halo_status halo_scratch_bytes(const halo_ctx* ctx, size_t* bytes);

/* Register the device buffers of local rank `local` (0 <= local < n_local):
 * x, f: capacity*layout floats, 16-B aligned; scratch: halo_scratch_bytes().
 * Caller-owned; they must stay allocated at fixed addresses until halo_destroy
 * because peer processes map them (P:436-439 symmetric/registered buffers).
 * Zero-fills scratch (stream-ordered on the legacy stream, synchronised). */
HALO_API halo_status halo_register_buffers(halo_ctx* ctx, int local, void* x, void* f, void* scratch);

/* CUDA-IPC export of this process's registered x and scratch buffers (replaces
 * nvshmem_ptr / symmetric allocation).  blob == NULL: *len = size needed.
 * The caller all-gathers the blobs (e.g. torch.distributed all_gather_object). */
HALO_API halo_status halo_ipc_export(halo_ctx* ctx, void* blob, size_t* len);

/* Import the nprocs blobs (rank order, each len_each bytes, own blob included
 * and skipped) and open the peer mappings.  Not needed when nprocs == 1. */
HALO_API halo_status halo_ipc_import(halo_ctx* ctx, const void* blobs, size_t len_each);

/* COLLECTIVE.  Neighbour-search step (every nstlist steps): build every
 * pulse's send index map from x[0:n_home) of each local rank (n_home[local]),
 * agree sizes/offsets with the neighbours through device flags, and exchange
 * the coordinates pulse by pulse (forwarding needs the earlier pulses' rows).
 * Selection (R2, R3): float64(x_d) - b_d[c_d] < float64(rc), strict, over the
 * candidate rows (k = 0: all rows present before the dim's first pulse; k > 0:
 * rows received in pulse (d, k-1)), ascending row order (R11).  Host-synchronises
 * (device-wide first: exchanges still running on any stream of this device finish
 * before the plan they read is rewritten).  Errors are agreed by all ranks (every
 * rank returns the same status). */
HALO_API halo_status halo_set_maps(halo_ctx* ctx, const int* n_home, void* stream);

/* COLLECTIVE test entry: like halo_set_maps but with caller-given maps.
 * send_sizes[local*npulse + p]; maps[local*npulse + p] = host int32 array of
 * send_sizes[...] ascending local row indices.  Coordinates are exchanged as
 * in halo_set_maps. */
HALO_API halo_status halo_set_maps_explicit(halo_ctx* ctx, const int* n_home, const int* send_sizes,
                                   const int* const* maps, void* stream);

/* Initial domain assignment (the DD "divides the simulation box into
 * spatial regions (domains)"; readings R3/R4): for the n_atoms rows of a GLOBAL
 * coordinate array x (DEVICE float32, row i at x + i*stride, stride >= 3 floats,
 * every x_d in [0, L_d)), the home rank of row i is (cx*np_y + cy)*np_z + cz with
 * c_d = the number of interior planes float64(L_d)*k/grid[d], k = 1..grid[d]-1,
 * that are <= float64(x_d) (a coordinate on a plane goes to the upper cell).
 *   ids     (DEVICE int32[n_atoms], out) the atom ids grouped by home rank,
 *           rank 0 first, ascending within each rank (a stable counting sort)
 *   counts  (host int[nranks], out) atoms per rank: rank r's ids start at
 *           counts[0] + ... + counts[r-1].
 * Needs no peers (any process, before or after registration).  HALO_ERR_GEOMETRY
 * if some coordinate lies outside [0, L_d) or is NaN (counts and ids are still
 * written).  Host-synchronises on `stream`. */
HALO_API halo_status halo_assign_home(halo_ctx* ctx, const float* x, int n_atoms, int stride, int32_t* ids,
                                      int* counts, void* stream);

/* COLLECTIVE, NS step: home-atom redistribution before
 * halo_set_maps.  Between NS steps atoms move (the decomposition is
 * rebuilt every nstlist steps); the domains own the atoms inside their region
 * (P:139-141), so every home atom is re-homed first.
 *   n_home_in[l]   home rows of local rank l in x (and gid, v) before the call
 *   gid[l]         DEVICE int32[capacity]: global atom ids of those rows, strictly
 *                  ascending (the order halo_set_maps' maps refer to, R11)
 *   v[l]           DEVICE float[capacity*layout] rows carried along unchanged
 *                  (velocities, ...); v == NULL or v[l] == NULL: no payload
 *   n_home_out[l]  (host, out) home rows after the call.
 * Each row is wrapped into the box in float32 (R29: x >= L_d -> x - L_d,
 * x < 0 -> x + L_d, a result of L_d or -0.0 -> +0.0; the w of float4 rows is
 * copied), assigned to the rank whose cell holds it (R3/R4) and moved there
 * (peer stores + loads over NVLink through the scratch staging area); afterwards
 * rank r holds exactly the atoms of its cell in x/gid/v[0:n_home_out), ascending
 * gid, bit-exact copies.  An atom may move at most one cell per dimension between
 * NS steps (R30); otherwise HALO_ERR_GEOMETRY.  HALO_ERR_CAPACITY when a rank
 * would hold more than `capacity` rows.  Errors are agreed by all ranks.  Halo
 * rows of x and the maps are invalid afterwards: call halo_set_maps next.
 * Host-synchronises on `stream`. */
HALO_API halo_status halo_migrate(halo_ctx* ctx, const int* n_home_in, int32_t* const* gid, float* const* v,
                                  int* n_home_out, void* stream);

/* ---- PP <-> PME coordinate / force redistribution ----
 * The PME task runs on the GPU of DD rank `pme_rank`.  Its buffers pme_x / pme_f
 * (rows of `layout` floats) hold the home rows of every DD rank concatenated in
 * rank order — rank r at rows [row_off[r], row_off[r+1]) — and live in that
 * rank's scratch (peer-mapped like the rest).  Per MD step:
 *   halo_pme_send_x  (after the integration)  every rank's x[0:n_home) -> pme_x
 *   ... the caller's PME kernel on the PME GPU reads pme_x, writes pme_f ...
 *   halo_pme_recv_f  (after the PME kernel)    pme_f slices -> every rank's f[0:n_home)
 * Same one-sided machinery as the halo: peer stores / loads over NVLink, one
 * system-scope release flag per rank and direction, acks, 64-bit sequence numbers
 * in device memory (graph-capturable), bounded waits. */

/* Before halo_register_buffers, on every process with the same pme_rank: grows
 * the scratch of the process hosting pme_rank by 2 * nranks * capacity rows
 * (query halo_scratch_bytes after this call). */
HALO_API halo_status halo_pme_reserve(halo_ctx* ctx, int pme_rank);

/* COLLECTIVE, after every halo_set_maps (the home counts changed): all-gathers
 * n_home over device flags and fixes row_off.  *n_total (optional) = sum of n_home.
 * Host-synchronises on `stream`. */
HALO_API halo_status halo_pme_setup(halo_ctx* ctx, void* stream, int* n_total);

/* Device pointers of pme_x / pme_f on the process hosting pme_rank (NULL
 * elsewhere); row_off (optional, host, nranks+1 ints) after halo_pme_setup. */
HALO_API halo_status halo_pme_buffers(const halo_ctx* ctx, float** pme_x, float** pme_f, int* row_off);

/* COLLECTIVE, asynchronous: every local rank stores x[0:n_home) into pme_x over
 * NVLink and releases its flag on the PME rank; the PME process's launch
 * completes when pme_x is complete (rows are bit-exact copies). */
HALO_API halo_status halo_pme_send_x(halo_ctx* ctx, void* stream);

/* COLLECTIVE, asynchronous: the PME process releases "pme_f ready" (its stream
 * has run the PME force kernel); every local rank acquire-waits, then
 * f[i] = f[i] + pme_f[row_off[r] + i] for its home rows (fp32 RNE per component;
 * accumulate = 0 overwrites) and acks; the PME process's launch completes when
 * every slice was read (pme_f may then be overwritten). */
HALO_API halo_status halo_pme_recv_f(halo_ctx* ctx, int accumulate, void* stream);

/* The transport the last halo_set_maps chose (HALO_F_AUTO_TRANSPORT, or fixed by the flags):
 * 0 = LL protocol, 1 = paper protocol, 2 = copy engine. */
HALO_API halo_status halo_transport(const halo_ctx* ctx, int* transport);

/* Layout of local rank `local` after set_maps (host arrays sized npulse; any may be NULL):
 * recv_off[p] = atomOffset, recv_size[p], send_size[p], remote_off[p] = where
 * this rank's pulse-p rows land on its receiver, dep_mask[p] = bit q set iff
 * map_p reads rows received in pulse q (the wait set of Alg. 4, R9). */
HALO_API halo_status halo_get_layout(const halo_ctx* ctx, int local, int* n_home, int* n_total, int* npulse,
                            int* recv_off, int* recv_size, int* send_size, int* remote_off,
                            unsigned* dep_mask);

/* Copy map of (local, pulse) to host (cap ints available); for parity tests. */
HALO_API halo_status halo_get_map(const halo_ctx* ctx, int local, int pulse, int* host_out, int cap);

/* COLLECTIVE, asynchronous, HOT PATH (Alg. 3 FusedPackCommX, Alg. 4, Alg. 5):
 * one kernel launch on `stream` that, for every local rank and pulse, gathers
 * x rows through the map, adds the periodic shift (float32 add of the full
 * 3-vector on the wrapping rank, R25) and writes them to the receiver over
 * NVLink peer stores; dependent rows are forwarded once the rows they come from
 * have arrived (R8/R9).  Default (LL protocol): every 8-B store carries the
 * step's sequence tag, a receiver on another GPU copies its tagged units into x,
 * a receiver on this GPU gets its rows stored directly, and forwarding waits per
 * row; HALO_F_PAPER_FLAGS: the paper's per-pulse scheme — rows straight into the
 * receiver's x at its atomOffset, one system-scope release flag per pulse
 * (P:427), acquire-waits on exactly the pulses a dependent chunk reads.
 * When `stream` has executed it, rows [n_home, n_total) hold this step's halo.
 * CUDA-graph capturable (the sequence number lives in device memory).  A captured
 * launch holds the plan of the NS epoch it was captured in: re-capture after every
 * halo_set_maps / halo_migrate (a graph replayed across them reads a stale or freed plan).
 * Precondition (R17): steps alternate exchange_x / exchange_f on all ranks. */
HALO_API halo_status halo_exchange_x(halo_ctx* ctx, void* stream);

/* COLLECTIVE, asynchronous, HOT PATH (Alg. 6 FusedCommUnpackF, Alg. 5 DEP_MGMT):
 * one kernel launch: each halo slice row is pushed back to the rank that sent it
 * once every later pulse that forwarded it has delivered its force (P:412,
 * P:421), and the received forces are added into f through the maps (pulses
 * descending, one float32 add per entry: bit-exact vs the oracle, R15).  Default
 * (LL protocol): a deterministic gather per target row with row-level DEP_MGMT;
 * HALO_F_PAPER_FLAGS: per-pulse push + flag + scatter-add (HALO_F_ATOMIC_UNPACK:
 * the paper's unordered atomics; HALO_F_TMA_GET: the receiver-driven TMA get).  fshift (device, [n_local][3][3] float64,
 * may be NULL) is ADDED the received force sums of the pulses this rank
 * shifted (R13).  accumulate = 0 overwrites and is only supported with a single
 * pulse in total (R14), else HALO_ERR_UNSUPPORTED.  Halo rows of f keep their
 * values.  CUDA-graph capturable. */
HALO_API halo_status halo_exchange_f(halo_ctx* ctx, double* fshift, int accumulate, void* stream);

/* COLLECTIVE, asynchronous: exchange_x and exchange_f of one step in ONE launch
 * (LL protocol only, "a single kernel for x+f when no compute
 * sits between them" — the paper's one-launch-per-exchange design, taken
 * one step further for a step with no non-bonded work between the halves).
 * Results are identical to halo_exchange_x followed by halo_exchange_f with the
 * same arguments (bit-exact).  Ordering inside the launch: the gather items of a
 * local rank start only once every x item that completes that rank's halo rows
 * has finished in this launch — the place of the non-bonded kernel of Alg. 2,
 * so f may be written by nothing between the halves: the forces in
 * f when the launch starts are the ones exchanged.  HALO_ERR_UNSUPPORTED for
 * the paper / copy-engine transports.  CUDA-graph capturable. */
HALO_API halo_status halo_exchange_xf(halo_ctx* ctx, double* fshift, int accumulate, void* stream);

/* ---- NCCL send/recv baseline (pin G2) ----
 * The paper's serialized schedule (Fig. 1) on the maps of
 * the last halo_set_maps: per pulse ascending a pack kernel (gather + shift) and
 * one ncclGroupStart / ncclSend (to the lower neighbour) / ncclRecv (the upper
 * neighbour's rows straight into this rank's halo range) / ncclGroupEnd; forces
 * per pulse descending: one group sending the halo slice back to the x-sender and
 * receiving this rank's slice, then the ordered scatter-add kernel (+ fp64 shift
 * forces).  All on `stream`: eager or captured in a CUDA graph.  Results are
 * bit-identical to the fused path.  One DD rank per process (nprocs == nranks,
 * NCCL rank = DD rank); NCCL is the libnccl.so.2 the process already loaded
 * (torch's), else dlopen("libnccl.so.2") / $HALO_NCCL_LIB. */

/* ncclGetUniqueId: id == NULL -> *len = 128; else writes the id (caller broadcasts it). */
HALO_API halo_status halo_nccl_unique_id(void* id, size_t* len);
/* COLLECTIVE over all processes: ncclCommInitRank(nprocs, id, proc). */
HALO_API halo_status halo_nccl_init(halo_ctx* ctx, const void* id, size_t len);
/* ncclGetVersion of the resolved library (0 if none). */
HALO_API halo_status halo_nccl_version(int* version);
/* COLLECTIVE, asynchronous: the baseline x halo (P pack kernels + P NCCL groups). */
HALO_API halo_status halo_nccl_exchange_x(halo_ctx* ctx, void* stream);
/* COLLECTIVE, asynchronous: the baseline force halo (P NCCL groups + P unpack kernels);
 * fshift / accumulate as halo_exchange_f. */
HALO_API halo_status halo_nccl_exchange_f(halo_ctx* ctx, double* fshift, int accumulate, void* stream);

/* COLLECTIVE end-to-end step through host buffers (the e2e measurement path):
 * per local rank copies x_home[l] (n_home*layout floats, pinned host) and
 * f_all[l] (n_total*layout floats) to the device, runs exchange_x and
 * exchange_f, copies the halo x rows to x_halo_out[l] ((n_total-n_home)*layout
 * floats), the home f rows to f_home_out[l] and fshift (n_local*9 doubles) to
 * fshift_host; any output may be NULL.  Enqueued on `stream`; synchronises it. */
HALO_API halo_status halo_step_host(halo_ctx* ctx, const float* const* x_home, const float* const* f_all,
                           float* const* x_halo_out, float* const* f_home_out, double* fshift_host,
                           void* stream);

/* Host block sizes of halo_step_host_packed for the current maps (bytes).
 * HALO_ERR_STATE before set_maps. */
HALO_API halo_status halo_packed_sizes(const halo_ctx* ctx, size_t* in_bytes, size_t* out_bytes);

/* COLLECTIVE end-to-end step through ONE host block in and ONE out (the e2e
 * measurement path; same computation as halo_step_host, bit-identical).
 *   in  (in_bytes, pinned host, caller-owned, read): the x home rows of local
 *       ranks 0..L-1 concatenated (n_home*layout floats each), then the f rows
 *       [0, n_total) of local ranks 0..L-1 (the step's non-bonded forces);
 *   out (out_bytes, pinned host, caller-owned, written; NULL = no outputs): the
 *       halo x rows [n_home, n_total) of every local rank, then the home f rows
 *       of every local rank, then at the next 8-B aligned offset the shift
 *       forces, n_local*9 doubles ([local][dim][component], zeroed each step).
 * Two uploads (x home, then the forces on a library-owned side stream while x
 * is exchanged), two downloads (halo x on a side stream while f is exchanged,
 * then the forces and fshift); packing to and from the per-rank rows is done
 * by a copy kernel.  The whole sequence is captured once per (NS epoch, in,
 * out) into a library-owned CUDA graph and replayed on `stream`
 * (HALO_PACKED_GRAPH=0: enqueued eagerly).  HALO_PACKED_DIRECT=1: the last copy
 * kernel writes the forces straight into `out` when it is device-accessible
 * pinned memory (measured slower).  Synchronises `stream`.  Not itself
 * graph-capturable by the caller. */
HALO_API halo_status halo_step_host_packed(halo_ctx* ctx, const void* in, void* out, void* stream);

/* Baseline building blocks (the NCCL send/recv schedule of P:178-181 / Fig. 1
 * drives these from the host; not on the fused path):
 * pack pulse p of local rank into sendbuf (send_size*layout floats, shift applied);
 * unpack a received force slice (send_size*layout floats) into f (+ fshift). */
HALO_API halo_status halo_pack_x_pulse(halo_ctx* ctx, int local, int pulse, float* sendbuf, void* stream);
HALO_API halo_status halo_unpack_f_pulse(halo_ctx* ctx, int local, int pulse, const float* recvbuf,
                                double* fshift, int accumulate, void* stream);

/* Device-side kernel spans (HALO_F_TIMERS): last exchange_x and exchange_f
 * durations in ns (max end - min start over the CTAs), read after halo_sync. */
HALO_API halo_status halo_get_timers(halo_ctx* ctx, uint64_t* x_ns, uint64_t* f_ns);

/* Per-CTA device timestamps of the last exchange_x (which = 0) or exchange_f
 * (which = 1) launch, HALO_F_TIMERS only (the paper's %globaltimer
 * instrumentation): out[8*i .. 8*i+7] = CTA i's [start, plan record
 * loaded, items done, exit, item0 tag, item0 end, item1 tag, item1 end] in ns,
 * tag = kind << 16 | local rank << 8 | pulse; *n = CTAs recorded (<= cap/8).
 * LL protocol kernels only.  Synchronises. */
HALO_API halo_status halo_get_trace(halo_ctx* ctx, int which, uint64_t* out, int cap, int* n);

/* Debug (pin G4, "emitting system-scope operations only from the
 * last block"): with HALO_DEBUG=64 in the environment at halo_init, the paper
 * protocol (HALO_F_PAPER_FLAGS) counts its system-scope flag stores; out[l*P + p]
 * = cumulative count for local rank l, pulse p of the x (which = 0) or force
 * (which = 1) exchange since init (set_maps' per-pulse x launches included).
 * cap >= n_local * npulse.  Synchronises. */
HALO_API halo_status halo_get_notify_counts(halo_ctx* ctx, int which, uint32_t* out, int cap);

/* Floors (measurement): ping-pong `iters` round trips of a
 * 64-bit flag between this process's local rank 0 and DD rank `peer_rank`
 * (COLLECTIVE between the two processes only; other processes must not call;
 * a peer hosted by this process is served by a second CTA of the same launch:
 * the same-GPU floor).
 * relaxed = 0: st.release.sys / ld.acquire.sys (the paper's signal);
 * relaxed = 1: st.relaxed.sys / ld.relaxed.sys (the LL protocol's unit).
 * *one_way_us = median round trip / 2 (initiator; 0 on the responder). */
HALO_API halo_status halo_floor_pingpong(halo_ctx* ctx, int peer_rank, int iters, int relaxed, double* one_way_us);

/* Launch floor (SURVEY 8(d) floor iii): mean device time per launch of an
 * empty kernel launched back to back the way the exchange kernels are
 * (regular launch + programmatic dependent launch), `iters` launches between
 * two events on an internal stream; graph = 1 captures them in a CUDA graph and
 * times its replay.  Synchronises. */
/* Launch floor of one step: enqueues on `stream` two EMPTY kernels with the grids
 * and launch attributes of the current exchange_x / exchange_f launches (PDL), so a
 * caller can time the step's fixed cost (launch, grid drain, hand-off) with the
 * same events, flush and reset as the real step.  HALO_ERR_STATE before set_maps. */
HALO_API halo_status halo_floor_empty_pair(halo_ctx* ctx, void* stream);

HALO_API halo_status halo_floor_launch(halo_ctx* ctx, int iters, int graph, double* us_per_launch);

/* Launch floor of a kernel that wrote to (NVLink) peer memory: as
 * halo_floor_launch, but `words` threads of each launch also store one 8-B word
 * each into DD rank `peer_rank`'s LL receive area (words <= that area and <=
 * grid threads).  The difference to halo_floor_launch is the completion cost of
 * a kernel with remote writes.  One-sided: the peer's process must be idle (no
 * exchange in flight); synchronises. */
HALO_API halo_status halo_floor_launch_remote(halo_ctx* ctx, int peer_rank, int words, int iters, int graph,
                                              double* us_per_launch);

/* Bandwidth floor (SURVEY 8(d) floor ii): one-directional GB/s of `iters`
 * back-to-back transfers of `bytes` (multiple of 16, at most the LL receive
 * area of a rank's scratch) from this process's local rank 0 into DD rank
 * `peer_rank`'s scratch LL receive area.  mode 0 = SM stores (16-B vectors from
 * 8 CTAs per SM, the hot path's transport), mode 1 = copy engine
 * (cudaMemcpyAsync, the HALO_F_CE_PATH transport).  One-sided: the peer's
 * process must be idle (no exchange in flight; the caller barriers before and
 * after), its LL areas are overwritten with data whose tags never match a
 * live sequence number.  Synchronises. */
HALO_API halo_status halo_floor_bandwidth(halo_ctx* ctx, int peer_rank, size_t bytes, int mode, int iters,
                                          double* gbs);

/* Floor-probe area (SURVEY 8(d) floors i/ii at payloads up to 64 MB): before
 * halo_register_buffers and halo_pme_reserve, on every process with the same
 * max_bytes, grows every rank's scratch by 4 KiB + 2 * max_bytes (a counter, a
 * send area, a receive area; query halo_scratch_bytes after this call).
 * HALO_ERR_STATE when called late or twice. */
HALO_API halo_status halo_probe_reserve(halo_ctx* ctx, size_t max_bytes);

/* Latency-vs-payload floor t(B) (SURVEY 8(d) floor i: "payload stores before
 * the flag"): a ping-pong between this process's local rank 0 and `peer_rank`
 * in which each leg stores `bytes` (multiple of 16, <= the reserved probe bytes)
 * from the sender's probe send area into the receiver's probe receive area from
 * min(ctas, ceil(bytes / 16 KiB)) CTAs, each CTA then signalling its slice with
 * fence.acq_rel.sys + a system-scope add on the receiver's probe counter (the
 * paper's per-CTA completion + signal, Alg. 5); the receiver's CTAs
 * wait for all slices, then answer.  *one_way_us = median round trip / 2 of
 * `iters` round trips (0 on the responder).  COLLECTIVE between the two
 * processes (both call it with the same arguments; the lower rank initiates;
 * both ranks on this GPU: one launch plays both sides).  Synchronises. */
HALO_API halo_status halo_floor_payload(halo_ctx* ctx, int peer_rank, size_t bytes, int iters, int ctas,
                                        double* one_way_us);

/* Bandwidth floor to several concurrent peers (SURVEY 8(d) floor ii "one pair,
 * and 3 concurrent peers"): `iters` back-to-back transfers of `bytes` from local
 * rank 0's probe send area into the probe receive area of each of the n ranks
 * in peers[] at once.  mode 0 = SM 16-B stores (8 CTAs per SM split over the
 * peers), mode 1 = one cudaMemcpyAsync stream per peer.  *gbs = total bytes out
 * / elapsed (GB/s).  One-sided; the peers must be idle.  Synchronises. */
HALO_API halo_status halo_floor_bandwidth_multi(halo_ctx* ctx, const int* peers, int n, size_t bytes, int mode,
                                                int iters, double* gbs);

/* Host-block until all work this ctx enqueued is done; surfaces device error
 * words (HALO_ERR_TIMEOUT) and CUDA errors. */
HALO_API halo_status halo_sync(halo_ctx* ctx);

HALO_API const char* halo_strerror(halo_status s);
HALO_API const char* halo_last_error(const halo_ctx* ctx);

/* Close peer mappings and free library-owned memory.  Callers barrier across
 * processes before freeing the registered buffers. */
HALO_API halo_status halo_destroy(halo_ctx* ctx);

#ifdef __cplusplus
}
#endif
#endif /* HALO_H_ */
