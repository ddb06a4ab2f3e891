// NCCL behind the C-ABI (SURVEY.md 8(b) pmp_nccl_*): the sequence driver's
// only two collectives -- replicating the base SPAI P1 (one broadcast, or the
// grouped all-gather of a column-sharded build) and gathering the
// per-system scalars -- over NVLink / NVSwitch.
//
// libnccl.so.2 is opened at run time (dlopen) rather than linked: the
// library then loads on hosts without NCCL (the CPU build / test container),
// and inside a PyTorch process it binds to the NCCL torch already mapped
// (same soname, same ABI).  Only the types come from <nccl.h>.
#include <dlfcn.h>
#include <nccl.h>
#include <string.h>

#include <cuda_runtime.h>

#include "../../include/pmorb200.h"

namespace pmp {
void set_error(const char* fmt, ...);
}

namespace {

struct NcclApi {
  void* h = nullptr;
  ncclResult_t (*getUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*commInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*commDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*bcast)(const void*, void*, size_t, ncclDataType_t, int, ncclComm_t,
                        cudaStream_t) = nullptr;
  ncclResult_t (*allReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*groupStart)() = nullptr;
  ncclResult_t (*groupEnd)() = nullptr;
  const char* (*errStr)(ncclResult_t) = nullptr;
};

NcclApi g_api;

bool load_nccl() {
  if (g_api.h) return true;
  void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
  if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
  if (!h) {
    pmp::set_error("pmp_nccl: cannot load libnccl.so.2 (%s)", dlerror());
    return false;
  }
#define PMP_SYM(field, name)                                               \
  g_api.field = reinterpret_cast<decltype(g_api.field)>(dlsym(h, name));   \
  if (!g_api.field) {                                                      \
    pmp::set_error("pmp_nccl: symbol %s missing from libnccl", name);      \
    return false;                                                          \
  }
  PMP_SYM(getUniqueId, "ncclGetUniqueId")
  PMP_SYM(commInitRank, "ncclCommInitRank")
  PMP_SYM(commDestroy, "ncclCommDestroy")
  PMP_SYM(bcast, "ncclBroadcast")
  PMP_SYM(allReduce, "ncclAllReduce")
  PMP_SYM(groupStart, "ncclGroupStart")
  PMP_SYM(groupEnd, "ncclGroupEnd")
  PMP_SYM(errStr, "ncclGetErrorString")
#undef PMP_SYM
  g_api.h = h;
  return true;
}

int nccl_status(ncclResult_t r, const char* where) {
  if (r == ncclSuccess) return PMP_OK;
  pmp::set_error("%s: %s", where, g_api.errStr ? g_api.errStr(r) : "nccl error");
  return PMP_ERR_CUDA;
}

}  // namespace

extern "C" {

int pmp_nccl_available(void) { return load_nccl() ? 1 : 0; }

int pmp_nccl_unique_id(unsigned char* out128) {
  if (!out128) {
    pmp::set_error("pmp_nccl_unique_id: null output");
    return PMP_ERR_ARG;
  }
  if (!load_nccl()) return PMP_ERR_CUDA;
  ncclUniqueId id;
  const int rc = nccl_status(g_api.getUniqueId(&id), "ncclGetUniqueId");
  if (rc) return rc;
  static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId is 128 bytes");
  memcpy(out128, &id, sizeof(id));
  return PMP_OK;
}

int pmp_nccl_init(int rank, int world, const unsigned char* id128, void** comm) {
  if (!id128 || !comm || world < 1 || rank < 0 || rank >= world) {
    pmp::set_error("pmp_nccl_init: bad arguments (rank %d, world %d)", rank, world);
    return PMP_ERR_ARG;
  }
  if (!load_nccl()) return PMP_ERR_CUDA;
  ncclUniqueId id;
  memcpy(&id, id128, sizeof(id));
  ncclComm_t c = nullptr;
  const int rc = nccl_status(g_api.commInitRank(&c, world, id, rank), "ncclCommInitRank");
  if (rc) return rc;
  *comm = c;
  return PMP_OK;
}

int pmp_nccl_destroy(void* comm) {
  if (!comm) return PMP_OK;
  if (!load_nccl()) return PMP_ERR_CUDA;
  return nccl_status(g_api.commDestroy((ncclComm_t)comm), "ncclCommDestroy");
}

int pmp_nccl_bcast(void* buf, size_t bytes, int root, void* comm, void* stream) {
  if (!comm || (!buf && bytes)) {
    pmp::set_error("pmp_nccl_bcast: bad arguments");
    return PMP_ERR_ARG;
  }
  if (!bytes) return PMP_OK;
  return nccl_status(g_api.bcast(buf, buf, bytes, ncclUint8, root, (ncclComm_t)comm,
                                 (cudaStream_t)stream),
                     "ncclBroadcast");
}

// Variable-size all-gather in place: rank r's segment [displ[r], displ[r] +
// count[r]) bytes of buf is replicated on every rank -- one broadcast per
// rank inside one NCCL group (the column-sharded base-SPAI build).
int pmp_nccl_allgatherv(void* buf, const size_t* h_counts, const size_t* h_displs, int world,
                        void* comm, void* stream) {
  if (!comm || !buf || !h_counts || !h_displs || world < 1) {
    pmp::set_error("pmp_nccl_allgatherv: bad arguments");
    return PMP_ERR_ARG;
  }
  int rc = nccl_status(g_api.groupStart(), "ncclGroupStart");
  if (rc) return rc;
  for (int r = 0; r < world && !rc; ++r) {
    if (!h_counts[r]) continue;
    char* seg = static_cast<char*>(buf) + h_displs[r];
    rc = nccl_status(g_api.bcast(seg, seg, h_counts[r], ncclUint8, r, (ncclComm_t)comm,
                                 (cudaStream_t)stream),
                     "ncclBroadcast (allgatherv)");
  }
  const int rc2 = nccl_status(g_api.groupEnd(), "ncclGroupEnd");
  return rc ? rc : rc2;
}

int pmp_nccl_allreduce_f64(double* buf, size_t count, void* comm, void* stream) {
  if (!comm || (!buf && count)) {
    pmp::set_error("pmp_nccl_allreduce_f64: bad arguments");
    return PMP_ERR_ARG;
  }
  if (!count) return PMP_OK;
  return nccl_status(g_api.allReduce(buf, buf, count, ncclFloat64, ncclSum, (ncclComm_t)comm,
                                     (cudaStream_t)stream),
                     "ncclAllReduce");
}

}  // extern "C"
