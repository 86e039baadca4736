// ZeRO chunk-group collectives behind the C ABI (SURVEY §8(b) cs_comm_*,
// cs_allgather, cs_reduce_scatter_avg) for callers that do not run
// torch.distributed.  The protocol is the reference's
// (`/root/reference/pkg/src/chunkstar/parallel.py:196-264`): all-gather of a
// group's p chunks into a p×cap buffer before its first FWD / BWD / RE_FWD
// access (:196-223), reduce-scatter(avg) of the group's gradients once every
// member is HOLD_AFTER_BWD (:241-264); slot k of a group buffer is rank k's
// chunk, NCCL's rank order, so no reordering copy exists.
//
// NCCL is loaded at first use with dlopen (RTLD_NOLOAD first, so a process
// that already has torch's libnccl.so.2 reuses that copy; $CS_NCCL_LIB
// overrides the name).  The library has no link-time NCCL dependency and the
// other entry points work without it.
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>

#include <cstdlib>
#include <cstring>
#include <mutex>

#include "cs_internal.h"

namespace {

struct Nccl {
  ncclResult_t (*get_unique_id)(ncclUniqueId*);
  ncclResult_t (*comm_init_rank)(ncclComm_t*, int, ncclUniqueId, int);
  ncclResult_t (*comm_destroy)(ncclComm_t);
  ncclResult_t (*all_gather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t,
                             cudaStream_t);
  ncclResult_t (*reduce_scatter)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t,
                                 ncclComm_t, cudaStream_t);
  ncclResult_t (*all_reduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t,
                             ncclComm_t, cudaStream_t);
  const char* (*error_string)(ncclResult_t);
  ncclResult_t (*get_version)(int*);
  ncclResult_t (*get_async_error)(ncclComm_t, ncclResult_t*);
  ncclResult_t (*comm_abort)(ncclComm_t);
  bool ok = false;
};

Nccl g_nccl;
std::once_flag g_once;

void load_nccl() {
  const char* env = std::getenv("CS_NCCL_LIB");
  const char* name = env && *env ? env : "libnccl.so.2";
  void* h = dlopen(name, RTLD_NOW | RTLD_NOLOAD);
  if (!h) h = dlopen(name, RTLD_NOW | RTLD_GLOBAL);
  if (!h) {
    cs::set_error("cs_comm: dlopen(%s) failed: %s", name, dlerror());
    return;
  }
#define CS_SYM(field, sym)                                                  \
  *reinterpret_cast<void**>(&g_nccl.field) = dlsym(h, sym);                 \
  if (!g_nccl.field) {                                                      \
    cs::set_error("cs_comm: %s lacks %s", name, sym);                       \
    return;                                                                 \
  }
  CS_SYM(get_unique_id, "ncclGetUniqueId")
  CS_SYM(comm_init_rank, "ncclCommInitRank")
  CS_SYM(comm_destroy, "ncclCommDestroy")
  CS_SYM(all_gather, "ncclAllGather")
  CS_SYM(reduce_scatter, "ncclReduceScatter")
  CS_SYM(all_reduce, "ncclAllReduce")
  CS_SYM(error_string, "ncclGetErrorString")
  CS_SYM(get_version, "ncclGetVersion")
  CS_SYM(get_async_error, "ncclCommGetAsyncError")
  CS_SYM(comm_abort, "ncclCommAbort")
#undef CS_SYM
  int v = 0;
  if (g_nccl.get_version(&v) != ncclSuccess || v < 21000) {  // ncclAvg: NCCL >= 2.10
    cs::set_error("cs_comm: NCCL %d is older than 2.10 (no ncclAvg)", v);
    return;
  }
  g_nccl.ok = true;
}

bool nccl_ready() {
  std::call_once(g_once, load_nccl);
  return g_nccl.ok;
}

int nccl_rc(ncclResult_t r, const char* who) {
  if (r == ncclSuccess) return 0;
  cs::set_error("%s: %s", who, g_nccl.error_string(r));
  return static_cast<int>(r);
}

bool nccl_type(int dtype, ncclDataType_t* t) {
  switch (dtype) {
    case CS_FP16: *t = ncclFloat16; return true;
    case CS_BF16: *t = ncclBfloat16; return true;
    case CS_FP32: *t = ncclFloat32; return true;
    default: return false;
  }
}

}  // namespace

extern "C" int cs_comm_version(void) {
  if (!nccl_ready()) return CS_EUNAVAIL;
  int v = 0;
  g_nccl.get_version(&v);
  return v;
}

extern "C" int cs_comm_unique_id(void* id_out) {
  if (!id_out) {
    cs::set_error("cs_comm_unique_id: null id_out");
    return CS_EINVAL;
  }
  if (!nccl_ready()) return CS_EUNAVAIL;
  static_assert(sizeof(ncclUniqueId) == CS_COMM_ID_BYTES, "ncclUniqueId size");
  ncclUniqueId id;
  if (int rc = nccl_rc(g_nccl.get_unique_id(&id), "cs_comm_unique_id")) return rc;
  std::memcpy(id_out, &id, sizeof(id));
  return 0;
}

extern "C" int cs_comm_init(const void* id, int nranks, int rank, void** comm) {
  if (!id || !comm || nranks <= 0 || rank < 0 || rank >= nranks) {
    cs::set_error("cs_comm_init: invalid argument (rank %d of %d)", rank, nranks);
    return CS_EINVAL;
  }
  if (!nccl_ready()) return CS_EUNAVAIL;
  ncclUniqueId uid;
  std::memcpy(&uid, id, sizeof(uid));
  ncclComm_t c = nullptr;
  if (int rc = nccl_rc(g_nccl.comm_init_rank(&c, nranks, uid, rank), "cs_comm_init")) return rc;
  *comm = c;
  return 0;
}

extern "C" int cs_comm_destroy(void* comm) {
  if (!comm) return 0;
  if (!nccl_ready()) return CS_EUNAVAIL;
  return nccl_rc(g_nccl.comm_destroy(static_cast<ncclComm_t>(comm)), "cs_comm_destroy");
}

extern "C" int cs_allgather(void* group_buf, const void* local, int64_t count, int dtype,
                            void* comm, void* stream) {
  ncclDataType_t t;
  if (!group_buf || !local || !comm || count < 0 || !nccl_type(dtype, &t)) {
    cs::set_error("cs_allgather: invalid argument");
    return CS_EINVAL;
  }
  if (!nccl_ready()) return CS_EUNAVAIL;
  if (count == 0) return 0;
  // in place when local is slot `rank` of group_buf (the executor's layout)
  return nccl_rc(g_nccl.all_gather(local, group_buf, (size_t)count, t,
                                   static_cast<ncclComm_t>(comm),
                                   static_cast<cudaStream_t>(stream)),
                 "cs_allgather");
}

extern "C" int cs_reduce_scatter_avg(void* local, const void* group_buf, int64_t count,
                                     int dtype, void* comm, void* stream) {
  ncclDataType_t t;
  if (!local || !group_buf || !comm || count < 0 || !nccl_type(dtype, &t)) {
    cs::set_error("cs_reduce_scatter_avg: invalid argument");
    return CS_EINVAL;
  }
  if (!nccl_ready()) return CS_EUNAVAIL;
  if (count == 0) return 0;
  return nccl_rc(g_nccl.reduce_scatter(group_buf, local, (size_t)count, t, ncclAvg,
                                       static_cast<ncclComm_t>(comm),
                                       static_cast<cudaStream_t>(stream)),
                 "cs_reduce_scatter_avg");
}

extern "C" int cs_allreduce(void* buf, int64_t count, int dtype, int avg, void* comm,
                            void* stream) {
  ncclDataType_t t;
  if (!buf || !comm || count < 0 || !nccl_type(dtype, &t)) {
    cs::set_error("cs_allreduce: invalid argument");
    return CS_EINVAL;
  }
  if (!nccl_ready()) return CS_EUNAVAIL;
  if (count == 0) return 0;
  return nccl_rc(g_nccl.all_reduce(buf, buf, (size_t)count, t, avg ? ncclAvg : ncclSum,
                                   static_cast<ncclComm_t>(comm),
                                   static_cast<cudaStream_t>(stream)),
                 "cs_allreduce");
}

// Failure detection: a collective that fails after it was
// enqueued (a peer died, a network / NVLink error) is reported by NCCL only
// through the communicator's asynchronous error; the stream it runs on may
// never complete.  The host polls this (native_comm.py does at every issue
// and while it waits) and aborts the communicator on error, which unblocks
// the kernels stuck on it.  Returns 0 while healthy, CS_EINPROGRESS while a
// nonblocking init / abort is pending, else the ncclResult_t.
extern "C" int cs_comm_check(void* comm) {
  if (!comm) {
    cs::set_error("cs_comm_check: null communicator");
    return CS_EINVAL;
  }
  if (!nccl_ready()) return CS_EUNAVAIL;
  ncclResult_t async_err = ncclSuccess;
  if (int rc = nccl_rc(g_nccl.get_async_error(static_cast<ncclComm_t>(comm), &async_err),
                       "cs_comm_check"))
    return rc;
  if (async_err == ncclInProgress) return CS_EINPROGRESS;
  return nccl_rc(async_err, "cs_comm_check (asynchronous NCCL error)");
}

// Abort: tear the communicator down without waiting for outstanding
// collectives (ncclCommAbort); the handle is invalid afterwards.
extern "C" int cs_comm_abort(void* comm) {
  if (!comm) return 0;
  if (!nccl_ready()) return CS_EUNAVAIL;
  return nccl_rc(g_nccl.comm_abort(static_cast<ncclComm_t>(comm)), "cs_comm_abort");
}
