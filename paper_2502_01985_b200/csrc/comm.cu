// NCCL communicator for sharded sessions.
//
// With a communicator attached (fl_*_set_comm), a session's run() executes
// partial -> ncclAllReduce(red, sum) -> update per iteration on its own
// stream, and captures those iterations in CUDA graphs exactly like the
// single-GPU path: the per-iteration exchange is one all-reduce of the
// session's fp64 reduce buffer over NVLink / NVSwitch, with no host round
// trip between iterations.
//
// NCCL is resolved at run time (dlopen), so the library has no link-time
// NCCL dependency and shares the copy torch has already loaded
// ("libnccl.so.2" is looked up among the loaded objects first; FL_NCCL_LIB
// names another file).
#include <dlfcn.h>
#include <nccl.h>

#include <cstring>

#include "internal.h"

struct fl_comm {
  void* lib = nullptr;
  ncclComm_t comm = nullptr;
  int nranks = 1, rank = 0, device = 0;
  ncclResult_t (*all_reduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                             cudaStream_t) = nullptr;
  ncclResult_t (*destroy)(ncclComm_t) = nullptr;
  const char* (*err_str)(ncclResult_t) = nullptr;
};

namespace flb {

static void* nccl_open() {
  if (const char* p = getenv("FL_NCCL_LIB")) return dlopen(p, RTLD_NOW | RTLD_GLOBAL);
  void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
  if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
  if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
  return h;
}

int comm_allreduce(fl_comm* c, double* buf, size_t n, cudaStream_t st) {
  const ncclResult_t r = c->all_reduce(buf, buf, n, ncclFloat64, ncclSum, c->comm, st);
  if (r != ncclSuccess) {
    set_error("ncclAllReduce failed: %s", c->err_str ? c->err_str(r) : "?");
    return FL_ERR_CUDA;
  }
  return FL_OK;
}

}  // namespace flb

using namespace flb;

extern "C" {

int fl_comm_unique_id(uint8_t* out, int32_t len) {
  if (!out || len < (int32_t)sizeof(ncclUniqueId)) {
    set_error("fl_comm_unique_id: need a %zu-byte buffer", sizeof(ncclUniqueId));
    return FL_ERR_ARG;
  }
  void* lib = nccl_open();
  if (!lib) {
    set_error("NCCL library not found (%s)", dlerror());
    return FL_ERR_CUDA;
  }
  auto get_id = (ncclResult_t(*)(ncclUniqueId*))dlsym(lib, "ncclGetUniqueId");
  if (!get_id) {
    set_error("ncclGetUniqueId not found");
    return FL_ERR_CUDA;
  }
  ncclUniqueId id;
  if (get_id(&id) != ncclSuccess) {
    set_error("ncclGetUniqueId failed");
    return FL_ERR_CUDA;
  }
  std::memcpy(out, &id, sizeof(id));
  return FL_OK;
}

int fl_comm_init(const uint8_t* id_bytes, int32_t len, int32_t nranks, int32_t rank,
                 int32_t device, fl_comm** out) {
  if (!id_bytes || len < (int32_t)sizeof(ncclUniqueId) || nranks < 1 || rank < 0 ||
      rank >= nranks || !out) {
    set_error("fl_comm_init: bad arguments");
    return FL_ERR_ARG;
  }
  FL_CUDA(cudaSetDevice(device));
  auto* c = new fl_comm();
  std::unique_ptr<fl_comm> guard(c);
  c->lib = nccl_open();
  if (!c->lib) {
    set_error("NCCL library not found (%s)", dlerror());
    return FL_ERR_CUDA;
  }
  auto init = (ncclResult_t(*)(ncclComm_t*, int, ncclUniqueId, int))dlsym(c->lib, "ncclCommInitRank");
  c->all_reduce = (decltype(c->all_reduce))dlsym(c->lib, "ncclAllReduce");
  c->destroy = (decltype(c->destroy))dlsym(c->lib, "ncclCommDestroy");
  c->err_str = (decltype(c->err_str))dlsym(c->lib, "ncclGetErrorString");
  if (!init || !c->all_reduce || !c->destroy) {
    set_error("NCCL symbols not found");
    return FL_ERR_CUDA;
  }
  ncclUniqueId id;
  std::memcpy(&id, id_bytes, sizeof(id));
  const ncclResult_t r = init(&c->comm, nranks, id, rank);
  if (r != ncclSuccess) {
    set_error("ncclCommInitRank failed: %s", c->err_str ? c->err_str(r) : "?");
    return FL_ERR_CUDA;
  }
  c->nranks = nranks;
  c->rank = rank;
  c->device = device;
  *out = guard.release();
  return FL_OK;
}

/* in-place sum of n doubles over the communicator's ranks (stream-ordered) */
int fl_comm_allreduce(fl_comm* c, double* buf, int64_t n, void* stream) {
  if (!c || !buf || n < 0) return FL_ERR_ARG;
  FL_CUDA(cudaSetDevice(c->device));
  return comm_allreduce(c, buf, (size_t)n, (cudaStream_t)stream);
}

int fl_comm_destroy(fl_comm* c) {
  if (!c) return FL_OK;
  if (c->comm && c->destroy) c->destroy(c->comm);
  delete c;
  return FL_OK;
}

}  // extern "C"
