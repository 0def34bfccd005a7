#include "comm.hpp"

#include <dlfcn.h>
#include <nccl.h>

#include <cstring>
#include <mutex>
#include <string>

#include "errors.hpp"

namespace sdb {

namespace {

struct NcclApi {
    ncclResult_t (*get_unique_id)(ncclUniqueId *) = nullptr;
    ncclResult_t (*comm_init_rank)(ncclComm_t *, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*all_reduce)(const void *, void *, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                               cudaStream_t) = nullptr;
    ncclResult_t (*comm_destroy)(ncclComm_t) = nullptr;
    const char *(*error_string)(ncclResult_t) = nullptr;
};

const NcclApi &nccl() {
    static NcclApi api;
    static std::string error;
    static std::once_flag once;
    std::call_once(once, [] {
        void *h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
        if (!h) {
            error = std::string("NCCL not available: ") + dlerror();
            return;
        }
        api.get_unique_id = reinterpret_cast<decltype(api.get_unique_id)>(dlsym(h, "ncclGetUniqueId"));
        api.comm_init_rank = reinterpret_cast<decltype(api.comm_init_rank)>(dlsym(h, "ncclCommInitRank"));
        api.all_reduce = reinterpret_cast<decltype(api.all_reduce)>(dlsym(h, "ncclAllReduce"));
        api.comm_destroy = reinterpret_cast<decltype(api.comm_destroy)>(dlsym(h, "ncclCommDestroy"));
        api.error_string = reinterpret_cast<decltype(api.error_string)>(dlsym(h, "ncclGetErrorString"));
        if (!api.get_unique_id || !api.comm_init_rank || !api.all_reduce || !api.comm_destroy)
            error = "NCCL library lacks the needed symbols";
    });
    if (!error.empty()) throw DeviceFailure(error);
    return api;
}

void check_nccl(ncclResult_t r, const char *what) {
    if (r == ncclSuccess) return;
    const char *msg = nccl().error_string ? nccl().error_string(r) : "unknown";
    throw DeviceFailure(std::string(what) + ": " + msg);
}

}  // namespace

void comm_unique_id(unsigned char *out) {
    ncclUniqueId id;
    check_nccl(nccl().get_unique_id(&id), "ncclGetUniqueId");
    std::memcpy(out, id.internal, kCommIdBytes);
}

void *comm_create(const unsigned char *id, int rank, int world, int device) {
    if (world < 1 || rank < 0 || rank >= world) throw InvalidArgument("comm_create: rank outside [0, world)");
    if (cudaSetDevice(device) != cudaSuccess) throw DeviceFailure("comm_create: cudaSetDevice failed");
    ncclUniqueId uid;
    std::memcpy(uid.internal, id, kCommIdBytes);
    ncclComm_t comm = nullptr;
    check_nccl(nccl().comm_init_rank(&comm, world, uid, rank), "ncclCommInitRank");
    return comm;
}

void comm_destroy(void *comm) {
    if (comm) nccl().comm_destroy(static_cast<ncclComm_t>(comm));
}

void comm_allreduce_min_u64(void *comm, unsigned long long *buf, size_t n, cudaStream_t stream) {
    check_nccl(nccl().all_reduce(buf, buf, n, ncclUint64, ncclMin, static_cast<ncclComm_t>(comm), stream),
               "ncclAllReduce");
}

}  // namespace sdb
