// nccl_baseline.cu — the NCCL send/recv schedule of the halo exchange: the
// BASELINE the fused kernels are measured against, not the product.
//
// The paper's serialized pulses (Fig. 1; §3: "the MPI
// formulation ... relies on distinct pack/unpack kernels per pulse"): per pulse
// p ascending, a pack kernel gathers x[map_p] (+ shift) into a contiguous send
// buffer, and one NCCL group sends it to the lower neighbour while receiving the
// upper neighbour's rows straight into this rank's halo range [atomOffset_p,
// +recvSize_p) (contiguous by construction, R12); forces run p descending: one
// NCCL group sends the halo slice f[atomOffset_p, +recvSize_p) back to the upper
// neighbour (the x-sender) and receives this rank's returned slice into a
// buffer, then the ordered scatter-add kernel adds it through map_p (+ fp64
// shift forces).  Same maps as the fused path, so results are bit-identical
// (pin G2).  Everything is enqueued on the caller's stream: eager or captured
// into a CUDA graph.
//
// NCCL is resolved at run time (dlopen of the libnccl.so.2 the process already
// has — torch's, 2.28.9 — with RTLD_NOLOAD first), so libhalo loads on hosts
// without NCCL and never mixes two NCCL builds in one process.
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <stdint.h>

#include <cstring>
#include <string>

#include "halo_internal.h"

namespace halo {

// The few NCCL entry points used (ABI of nccl.h, stable since 2.0).
typedef struct ncclComm* ncclComm_t;
typedef int ncclResult_t;  // ncclSuccess = 0
constexpr int kNcclIdBytes = 128;
typedef struct {
  char internal[kNcclIdBytes];
} ncclUniqueId;
constexpr int kNcclFloat32 = 7;

struct NcclApi {
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  ncclResult_t (*Send)(const void*, size_t, int, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Recv)(void*, size_t, int, int, ncclComm_t, cudaStream_t) = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
  ncclResult_t (*GetVersion)(int*) = nullptr;
  bool ok = false;
  std::string why;
};

static NcclApi& nccl_api() {
  static NcclApi a;
  static bool tried = false;
  if (tried) return a;
  tried = true;
  void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);  // the one torch loaded
  if (!h) {
    const char* p = getenv("HALO_NCCL_LIB");
    h = dlopen(p ? p : "libnccl.so.2", RTLD_NOW | RTLD_LOCAL);
  }
  if (!h) {
    a.why = std::string("dlopen(libnccl.so.2): ") + dlerror();
    return a;
  }
  auto sym = [&](const char* n) { return dlsym(h, n); };
  a.GetUniqueId = (decltype(a.GetUniqueId))sym("ncclGetUniqueId");
  a.CommInitRank = (decltype(a.CommInitRank))sym("ncclCommInitRank");
  a.CommDestroy = (decltype(a.CommDestroy))sym("ncclCommDestroy");
  a.GroupStart = (decltype(a.GroupStart))sym("ncclGroupStart");
  a.GroupEnd = (decltype(a.GroupEnd))sym("ncclGroupEnd");
  a.Send = (decltype(a.Send))sym("ncclSend");
  a.Recv = (decltype(a.Recv))sym("ncclRecv");
  a.GetErrorString = (decltype(a.GetErrorString))sym("ncclGetErrorString");
  a.GetVersion = (decltype(a.GetVersion))sym("ncclGetVersion");
  a.ok = a.GetUniqueId && a.CommInitRank && a.CommDestroy && a.GroupStart && a.GroupEnd && a.Send && a.Recv &&
         a.GetErrorString;
  if (!a.ok) a.why = "libnccl.so.2 lacks a required symbol";
  return a;
}

bool nccl_available(std::string* why) {
  NcclApi& a = nccl_api();
  if (!a.ok && why) *why = a.why;
  return a.ok;
}

int nccl_version() {
  NcclApi& a = nccl_api();
  int v = 0;
  if (a.ok && a.GetVersion) a.GetVersion(&v);
  return v;
}

bool nccl_unique_id(void* out, std::string* why) {
  NcclApi& a = nccl_api();
  if (!a.ok) {
    if (why) *why = a.why;
    return false;
  }
  ncclUniqueId id;
  const ncclResult_t r = a.GetUniqueId(&id);
  if (r != 0) {
    if (why) *why = std::string("ncclGetUniqueId: ") + a.GetErrorString(r);
    return false;
  }
  memcpy(out, &id, kNcclIdBytes);
  return true;
}

void* nccl_comm_init(const void* id, int nranks, int rank, std::string* why) {
  NcclApi& a = nccl_api();
  if (!a.ok) {
    if (why) *why = a.why;
    return nullptr;
  }
  ncclUniqueId u;
  memcpy(&u, id, kNcclIdBytes);
  ncclComm_t c = nullptr;
  const ncclResult_t r = a.CommInitRank(&c, nranks, u, rank);
  if (r != 0) {
    if (why) *why = std::string("ncclCommInitRank: ") + a.GetErrorString(r);
    return nullptr;
  }
  return c;
}

void nccl_comm_destroy(void* comm) {
  NcclApi& a = nccl_api();
  if (a.ok && comm) a.CommDestroy((ncclComm_t)comm);
}

// One pulse's grouped send/recv (either may be empty).  Returns an error string or "".
std::string nccl_sendrecv(void* comm, const float* sbuf, size_t sn, int speer, float* rbuf, size_t rn, int rpeer,
                          cudaStream_t st) {
  NcclApi& a = nccl_api();
  if (!sn && !rn) return "";
  ncclResult_t r = a.GroupStart();
  if (r == 0 && sn) r = a.Send(sbuf, sn, kNcclFloat32, speer, (ncclComm_t)comm, st);
  if (r == 0 && rn) r = a.Recv(rbuf, rn, kNcclFloat32, rpeer, (ncclComm_t)comm, st);
  const ncclResult_t r2 = a.GroupEnd();
  if (r == 0) r = r2;
  return r == 0 ? std::string() : std::string("NCCL send/recv: ") + a.GetErrorString(r);
}

}  // namespace halo
