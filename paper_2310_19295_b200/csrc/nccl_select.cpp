// The multi-GPU candidate selection exchange in libroam: every
// rank evaluates its shard of candidate ids (rm_eval_select_key leaves the
// rank's first strict minimum as one packed int64 key on the device), then
// ONE 8-byte ncclAllReduce(MIN) over NVLink gives every rank the global first
// strict minimum -- the (peak, candidate id) lexicographic minimum, i.e. the
// planner's "first strict minimum in candidate order" (planner.py:209-216,
// tests/oracles.py:46-56), because the key is (peak << id_bits) | id.
//
// NCCL is loaded with dlopen on first use (the soname libnccl.so.2: the copy
// already mapped into the process -- torch's -- when there is one), so
// libroam itself links no NCCL and a host without it only fails these calls.
#include <dlfcn.h>
#include <nccl.h>

#include <cstring>
#include <mutex>

#include "roam.h"
#include "roam_internal.h"

using namespace roam;

namespace {

struct NcclApi {
  bool ok = false;
  ncclResult_t (*get_unique_id)(ncclUniqueId*) = nullptr;
  ncclResult_t (*comm_init_rank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*comm_destroy)(ncclComm_t) = nullptr;
  ncclResult_t (*all_reduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                             cudaStream_t) = nullptr;
  const char* (*get_error_string)(ncclResult_t) = nullptr;
};

NcclApi& nccl() {
  static NcclApi api;
  static std::once_flag once;
  std::call_once(once, [] {
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) return;
    api.get_unique_id = reinterpret_cast<decltype(api.get_unique_id)>(dlsym(h, "ncclGetUniqueId"));
    api.comm_init_rank = reinterpret_cast<decltype(api.comm_init_rank)>(dlsym(h, "ncclCommInitRank"));
    api.comm_destroy = reinterpret_cast<decltype(api.comm_destroy)>(dlsym(h, "ncclCommDestroy"));
    api.all_reduce = reinterpret_cast<decltype(api.all_reduce)>(dlsym(h, "ncclAllReduce"));
    api.get_error_string = reinterpret_cast<decltype(api.get_error_string)>(dlsym(h, "ncclGetErrorString"));
    api.ok = api.get_unique_id && api.comm_init_rank && api.comm_destroy && api.all_reduce;
  });
  return api;
}

int nccl_fail(ncclResult_t r, const char* what) {
  const NcclApi& api = nccl();
  std::string msg = std::string(what) + " failed: ";
  msg += api.get_error_string ? api.get_error_string(r) : "NCCL error";
  return fail(RM_ERR_CUDA, msg);
}

}  // namespace

extern "C" int rm_nccl_unique_id(uint8_t* id, int64_t id_bytes) {
  if (!id || id_bytes < (int64_t)sizeof(ncclUniqueId))
    return fail(RM_ERR_INVALID_ARG, "rm_nccl_unique_id needs a buffer of RM_NCCL_ID_BYTES");
  NcclApi& api = nccl();
  if (!api.ok) return fail(RM_ERR_NO_DEVICE, "NCCL (libnccl.so.2) not available");
  ncclUniqueId uid;
  const ncclResult_t r = api.get_unique_id(&uid);
  if (r != ncclSuccess) return nccl_fail(r, "ncclGetUniqueId");
  std::memcpy(id, &uid, sizeof(uid));
  return RM_OK;
}

extern "C" int rm_nccl_comm_init(int32_t nranks, const uint8_t* id, int32_t rank, void** comm) {
  if (!comm || !id || nranks < 1 || rank < 0 || rank >= nranks)
    return fail(RM_ERR_INVALID_ARG, "bad rm_nccl_comm_init arguments");
  NcclApi& api = nccl();
  if (!api.ok) return fail(RM_ERR_NO_DEVICE, "NCCL (libnccl.so.2) not available");
  ncclUniqueId uid;
  std::memcpy(&uid, id, sizeof(uid));
  ncclComm_t c = nullptr;
  const ncclResult_t r = api.comm_init_rank(&c, nranks, uid, rank);
  if (r != ncclSuccess) return nccl_fail(r, "ncclCommInitRank");
  *comm = c;
  return RM_OK;
}

extern "C" int rm_nccl_comm_destroy(void* comm) {
  if (!comm) return RM_OK;
  NcclApi& api = nccl();
  if (!api.ok) return fail(RM_ERR_NO_DEVICE, "NCCL (libnccl.so.2) not available");
  const ncclResult_t r = api.comm_destroy(static_cast<ncclComm_t>(comm));
  if (r != ncclSuccess) return nccl_fail(r, "ncclCommDestroy");
  return RM_OK;
}

extern "C" int rm_nccl_select_key(void* comm, int64_t* key_dev, void* stream) {
  if (!comm || !key_dev) return fail(RM_ERR_INVALID_ARG, "bad rm_nccl_select_key arguments");
  NcclApi& api = nccl();
  if (!api.ok) return fail(RM_ERR_NO_DEVICE, "NCCL (libnccl.so.2) not available");
  const ncclResult_t r = api.all_reduce(key_dev, key_dev, 1, ncclInt64, ncclMin, static_cast<ncclComm_t>(comm),
                                        static_cast<cudaStream_t>(stream));
  if (r != ncclSuccess) return nccl_fail(r, "ncclAllReduce(MIN)");
  return RM_OK;
}
