// NCCL communicator entry points of the C ABI (swb_comm_*): what a C / C++
// host needs to run the z-slab sharded path without
// Python -- communicator bootstrap from a ncclUniqueId, the one-plane halo
// Send/Recv of the basis and the fixed-order f64 all-reduce of the K x K /
// S x K partials.  The reference has no communication layer at all (it is a
// single-process numpy package); these replace what sharded.py does with
// torch.distributed.
//
// NCCL is loaded at run time (dlopen of libnccl.so.2, reusing the copy the
// process already has, e.g. PyTorch's): the library itself links no NCCL, so
// it still loads on a host without one; the comm calls then return
// SWB_COMM_ERROR with the reason in swb_comm_last_error().
#include <dlfcn.h>
#include <nccl.h>

#include <atomic>
#include <cstdio>
#include <cstring>
#include <mutex>

#include "swb_common.cuh"

namespace {

struct NcclApi {
  ncclResult_t (*GetUniqueId)(ncclUniqueId*);
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int);
  ncclResult_t (*CommDestroy)(ncclComm_t);
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t, cudaStream_t);
  ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t);
  ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t);
  ncclResult_t (*GroupStart)();
  ncclResult_t (*GroupEnd)();
  const char* (*GetErrorString)(ncclResult_t);
  ncclResult_t (*GetVersion)(int*);
  bool ok = false;
};

std::mutex g_mu;
NcclApi g_api;
char g_err[256] = "";

void set_err(const char* what, const char* detail) {
  std::snprintf(g_err, sizeof(g_err), "%s: %s", what, detail ? detail : "");
}

const NcclApi* api() {
  std::lock_guard<std::mutex> lock(g_mu);
  if (g_api.ok) return &g_api;
  const char* names[] = {"libnccl.so.2", "libnccl.so"};
  void* h = nullptr;
  for (const char* n : names)
    if ((h = dlopen(n, RTLD_NOW | RTLD_NOLOAD))) break;   // the process's copy (e.g. PyTorch's)
  if (!h)
    for (const char* n : names)
      if ((h = dlopen(n, RTLD_NOW | RTLD_GLOBAL))) break;
  if (!h) {
    set_err("dlopen libnccl.so.2", dlerror());
    return nullptr;
  }
#define SWB_SYM(field, sym)                                             \
  g_api.field = reinterpret_cast<decltype(g_api.field)>(dlsym(h, sym)); \
  if (!g_api.field) {                                                   \
    set_err("dlsym", sym);                                              \
    return nullptr;                                                     \
  }
  SWB_SYM(GetUniqueId, "ncclGetUniqueId")
  SWB_SYM(CommInitRank, "ncclCommInitRank")
  SWB_SYM(CommDestroy, "ncclCommDestroy")
  SWB_SYM(AllReduce, "ncclAllReduce")
  SWB_SYM(Send, "ncclSend")
  SWB_SYM(Recv, "ncclRecv")
  SWB_SYM(GroupStart, "ncclGroupStart")
  SWB_SYM(GroupEnd, "ncclGroupEnd")
  SWB_SYM(GetErrorString, "ncclGetErrorString")
  SWB_SYM(GetVersion, "ncclGetVersion")
#undef SWB_SYM
  g_api.ok = true;
  return &g_api;
}

int nccl_status(const NcclApi* a, ncclResult_t r, const char* what) {
  if (r == ncclSuccess) return SWB_OK;
  set_err(what, a->GetErrorString(r));
  return SWB_COMM_ERROR;
}

}  // namespace

struct swb_comm {
  ncclComm_t nccl;
  int nranks, rank;
};

extern "C" const char* swb_comm_last_error(void) { return g_err; }

extern "C" int swb_comm_nccl_version(int* version) {
  const NcclApi* a = api();
  if (!a) return SWB_COMM_ERROR;
  if (!version) return SWB_INVALID_PARAM;
  return nccl_status(a, a->GetVersion(version), "ncclGetVersion");
}

extern "C" int swb_comm_unique_id(uint8_t* id_out) {
  static_assert(sizeof(ncclUniqueId) == SWB_COMM_ID_BYTES, "ncclUniqueId size");
  if (!id_out) return SWB_INVALID_PARAM;
  const NcclApi* a = api();
  if (!a) return SWB_COMM_ERROR;
  ncclUniqueId id;
  int rc = nccl_status(a, a->GetUniqueId(&id), "ncclGetUniqueId");
  if (rc) return rc;
  std::memcpy(id_out, &id, sizeof(id));
  return SWB_OK;
}

extern "C" int swb_comm_init(const uint8_t* id, int nranks, int rank, swb_comm** out) {
  if (!id || !out || nranks < 1 || rank < 0 || rank >= nranks) return SWB_INVALID_PARAM;
  *out = nullptr;
  const NcclApi* a = api();
  if (!a) return SWB_COMM_ERROR;
  ncclUniqueId uid;
  std::memcpy(&uid, id, sizeof(uid));
  ncclComm_t c = nullptr;
  int rc = nccl_status(a, a->CommInitRank(&c, nranks, uid, rank), "ncclCommInitRank");
  if (rc) return rc;
  *out = new swb_comm{c, nranks, rank};
  return SWB_OK;
}

extern "C" int swb_comm_destroy(swb_comm* comm) {
  if (!comm) return SWB_OK;
  const NcclApi* a = api();
  int rc = a ? nccl_status(a, a->CommDestroy(comm->nccl), "ncclCommDestroy") : SWB_COMM_ERROR;
  delete comm;
  return rc;
}

extern "C" int swb_comm_rank(const swb_comm* comm, int* rank, int* nranks) {
  if (!comm) return SWB_INVALID_PARAM;
  if (rank) *rank = comm->rank;
  if (nranks) *nranks = comm->nranks;
  return SWB_OK;
}

extern "C" int swb_comm_allreduce_f64(swb_comm* comm, const double* send, double* recv, int64_t count, void* stream) {
  if (!comm || count < 0 || (count > 0 && (!send || !recv))) return SWB_INVALID_PARAM;
  if (count == 0) return SWB_OK;
  const NcclApi* a = api();
  if (!a) return SWB_COMM_ERROR;
  return nccl_status(a, a->AllReduce(send, recv, size_t(count), ncclFloat64, ncclSum, comm->nccl, swb_stream(stream)),
                     "ncclAllReduce");
}

extern "C" int swb_comm_halo_exchange(swb_comm* comm, double* V, int64_t ldv, int64_t unit_rows, int64_t own_rows,
                                      int has_lo, int has_hi, void* stream) {
  if (!comm || !V || ldv <= 0 || unit_rows <= 0 || own_rows < unit_rows) return SWB_INVALID_PARAM;
  if ((has_lo && comm->rank == 0) || (has_hi && comm->rank == comm->nranks - 1)) return SWB_INVALID_PARAM;
  if (!has_lo && !has_hi) return SWB_OK;
  const NcclApi* a = api();
  if (!a) return SWB_COMM_ERROR;
  cudaStream_t st = swb_stream(stream);
  const size_t unit = size_t(unit_rows) * size_t(ldv);          // one xy-plane of rows, contiguous
  double* own = V + (has_lo ? unit : 0);                         // first owned row
  int rc = nccl_status(a, a->GroupStart(), "ncclGroupStart");
  if (rc) return rc;
  if (has_lo) {
    a->Send(own, unit, ncclFloat64, comm->rank - 1, comm->nccl, st);
    a->Recv(V, unit, ncclFloat64, comm->rank - 1, comm->nccl, st);
  }
  if (has_hi) {
    a->Send(own + size_t(own_rows - unit_rows) * size_t(ldv), unit, ncclFloat64, comm->rank + 1, comm->nccl, st);
    a->Recv(own + size_t(own_rows) * size_t(ldv), unit, ncclFloat64, comm->rank + 1, comm->nccl, st);
  }
  return nccl_status(a, a->GroupEnd(), "ncclGroupEnd (halo Send/Recv)");
}
