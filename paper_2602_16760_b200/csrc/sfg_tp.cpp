// Tensor parallelism (SURVEY.md §8e, configs[3]: the 12B shape at TP=2):
// the NCCL group (IPC-handle exchange for the megakernel's peer-memory inbox,
// sfg_engine.cpp) and the NCCL all-reduce of the row-parallel projections'
// partial outputs on the per-GEMM (prompt) path.  The decode step's
// layer-stack kernel exchanges its O/down partials over peer memory instead.
//
// NCCL is bound at run time (dlopen of the libnccl.so.2 already in the
// process — torch's — or the system one), so libsfg.so does not pin a second
// NCCL next to torch's.  Only the five entry points below are used.
#include <dlfcn.h>
#include <nccl.h>

#include <cstring>
#include <mutex>

#include "sfg_engine.h"

namespace sfg {
namespace {

struct NcclApi {
    ncclResult_t (*get_unique_id)(ncclUniqueId*) = nullptr;
    ncclResult_t (*comm_init_rank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*all_reduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                               cudaStream_t) = nullptr;
    ncclResult_t (*comm_destroy)(ncclComm_t) = nullptr;
    ncclResult_t (*all_gather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
    const char* (*error_string)(ncclResult_t) = nullptr;
};

const NcclApi& nccl() {
    static NcclApi api;
    static std::once_flag once;
    std::call_once(once, [] {
        void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
        if (!h) return;
        api.get_unique_id = reinterpret_cast<decltype(api.get_unique_id)>(dlsym(h, "ncclGetUniqueId"));
        api.comm_init_rank = reinterpret_cast<decltype(api.comm_init_rank)>(dlsym(h, "ncclCommInitRank"));
        api.all_reduce = reinterpret_cast<decltype(api.all_reduce)>(dlsym(h, "ncclAllReduce"));
        api.comm_destroy = reinterpret_cast<decltype(api.comm_destroy)>(dlsym(h, "ncclCommDestroy"));
        api.all_gather = reinterpret_cast<decltype(api.all_gather)>(dlsym(h, "ncclAllGather"));
        api.error_string = reinterpret_cast<decltype(api.error_string)>(dlsym(h, "ncclGetErrorString"));
    });
    if (!api.get_unique_id || !api.comm_init_rank || !api.all_reduce || !api.comm_destroy)
        throw Error(Kind::config, "tensor parallelism needs NCCL (libnccl.so.2 not found)");
    return api;
}

void check(ncclResult_t r, const char* what) {
    if (r != ncclSuccess) {
        const char* msg = nccl().error_string ? nccl().error_string(r) : "?";
        throw Error(Kind::internal, std::string("NCCL ") + what + ": " + msg);
    }
}

}  // namespace

void tp_unique_id(uint8_t* out, size_t n) {
    static_assert(sizeof(ncclUniqueId) == NCCL_UNIQUE_ID_BYTES, "ncclUniqueId layout");
    if (n < sizeof(ncclUniqueId)) throw Error(Kind::input, "unique id buffer too small");
    ncclUniqueId id;
    check(nccl().get_unique_id(&id), "GetUniqueId");
    std::memcpy(out, &id, sizeof(id));
}

void* tp_comm_init(int size, int rank, const uint8_t* uid) {
    ncclUniqueId id;
    std::memcpy(&id, uid, sizeof(id));
    ncclComm_t comm = nullptr;
    check(nccl().comm_init_rank(&comm, size, id, rank), "CommInitRank");
    return comm;
}

void tp_comm_destroy(void* comm) {
    if (comm) nccl().comm_destroy(static_cast<ncclComm_t>(comm));
}

// Every rank's `n` bytes (device) -> [size][n] on every rank.
void tp_allgather_bytes(void* comm, const void* src, void* dst, size_t n, cudaStream_t s) {
    check(nccl().all_gather(src, dst, n, ncclUint8, static_cast<ncclComm_t>(comm), s), "AllGather");
}

// In-place fp32 sum over the tensor-parallel ranks.  With two ranks every
// element is a + b (commutative), so the result is deterministic and
// identical on both ranks.
void tp_allreduce_sum(void* comm, float* buf, size_t n, cudaStream_t s) {
    check(nccl().all_reduce(buf, buf, n, ncclFloat32, ncclSum, static_cast<ncclComm_t>(comm), s), "AllReduce");
}

}  // namespace sfg
