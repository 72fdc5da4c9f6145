// comm.cpp -- the one collective of the path (SURVEY.md 8(b) mtk_comm_init /
// mtk_allgather, 8(e)): shadow models shard across GPUs with no gradient
// exchange, and after querying, every rank's posterior features are
// all-gathered over NCCL (NVLink / NVSwitch on one box) so the attack model
// trains on all shadows.  The reference has no multi-process code at all
// (SURVEY.md section 0); this stands in for the per-rank feature exchange
// north_star names.
//
// NCCL is resolved at run time (dlopen "libnccl.so.2"): inside a process
// that already loaded torch, the already-loaded NCCL is reused (RTLD_NOLOAD),
// so a Python driver and this library share one NCCL; a plain C++ caller gets
// the system library.  No link-time NCCL dependency, no second copy.
#include <dlfcn.h>
#include <nccl.h>

#include <cstring>
#include <memory>
#include <mutex>
#include <string>

#include "internal.h"

struct mtk_comm {
    ncclComm_t comm = nullptr;
    int nranks = 0, rank = 0, device = 0;
};

namespace mtk {
namespace {

struct Nccl {
    void* h = nullptr;
    ncclResult_t (*get_unique_id)(ncclUniqueId*) = nullptr;
    ncclResult_t (*comm_init_rank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*comm_destroy)(ncclComm_t) = nullptr;
    ncclResult_t (*all_gather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
    const char* (*error_string)(ncclResult_t) = nullptr;
    ncclResult_t (*get_version)(int*) = nullptr;
};

const Nccl& nccl() {
    static Nccl n;
    static std::once_flag once;
    static std::string err;
    std::call_once(once, [] {
        void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);  // torch's, when loaded
        if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
        if (!h) {
            err = std::string("NCCL not found: ") + dlerror();
            return;
        }
        n.h = h;
        n.get_unique_id = reinterpret_cast<decltype(n.get_unique_id)>(dlsym(h, "ncclGetUniqueId"));
        n.comm_init_rank = reinterpret_cast<decltype(n.comm_init_rank)>(dlsym(h, "ncclCommInitRank"));
        n.comm_destroy = reinterpret_cast<decltype(n.comm_destroy)>(dlsym(h, "ncclCommDestroy"));
        n.all_gather = reinterpret_cast<decltype(n.all_gather)>(dlsym(h, "ncclAllGather"));
        n.error_string = reinterpret_cast<decltype(n.error_string)>(dlsym(h, "ncclGetErrorString"));
        n.get_version = reinterpret_cast<decltype(n.get_version)>(dlsym(h, "ncclGetVersion"));
        if (!n.get_unique_id || !n.comm_init_rank || !n.comm_destroy || !n.all_gather || !n.error_string) {
            err = "NCCL: missing symbols in libnccl.so.2";
            n.h = nullptr;
        }
    });
    if (!n.h) fail(MTK_ERROR, err);
    return n;
}

void nccl_check(ncclResult_t r, const char* what) {
    if (r != ncclSuccess) fail(MTK_ERROR, std::string(what) + ": " + nccl().error_string(r));
}

}  // namespace
}  // namespace mtk

using namespace mtk;

extern "C" {

int mtk_comm_unique_id(void* out128) {
    return guard([&] {
        need(out128 != nullptr, MTK_VALUE_ERROR, "comm_unique_id: null out");
        ncclUniqueId id;
        nccl_check(nccl().get_unique_id(&id), "ncclGetUniqueId");
        std::memcpy(out128, &id, sizeof(id));
    });
}

int mtk_comm_init(int nranks, int rank, const void* nccl_id, mtk_comm** out) {
    return guard([&] {
        need(nccl_id && out, MTK_VALUE_ERROR, "comm_init: null argument");
        need(nranks >= 1 && rank >= 0 && rank < nranks, MTK_CONFIG_ERROR, "comm_init: rank outside [0, nranks)");
        *out = nullptr;
        std::unique_ptr<mtk_comm> c(new mtk_comm());
        c->nranks = nranks;
        c->rank = rank;
        c->device = current_device();
        ncclUniqueId id;
        std::memcpy(&id, nccl_id, sizeof(id));
        nccl_check(nccl().comm_init_rank(&c->comm, nranks, id, rank), "ncclCommInitRank");
        *out = c.release();
    });
}

int mtk_comm_destroy(mtk_comm* c) {
    return guard([&] {
        if (!c) return;
        DeviceScope ds(c->device);
        if (c->comm) nccl_check(nccl().comm_destroy(c->comm), "ncclCommDestroy");
        delete c;
    });
}

int mtk_comm_info(mtk_comm* c, int* nranks, int* rank, int* device, int* nccl_version) {
    return guard([&] {
        need(c != nullptr, MTK_VALUE_ERROR, "comm_info: null comm");
        if (nranks) *nranks = c->nranks;
        if (rank) *rank = c->rank;
        if (device) *device = c->device;
        if (nccl_version) {
            *nccl_version = 0;
            if (nccl().get_version) nccl_check(nccl().get_version(nccl_version), "ncclGetVersion");
        }
    });
}

// recv[r * bytes_per_rank, (r + 1) * bytes_per_rank) = rank r's send buffer,
// stream-ordered on the context's stream (asynchronous).
int mtk_allgather(mtk_comm* c, mtk_ctx* ctx, const void* send, void* recv, size_t bytes_per_rank) {
    return guard_on(ctx, [&] {
        need(c && ctx && recv && (send || bytes_per_rank == 0), MTK_VALUE_ERROR, "allgather: null argument");
        need(c->device == ctx->device, MTK_CONFIG_ERROR, "allgather: comm and ctx are on different devices");
        if (bytes_per_rank == 0) return;
        nccl_check(nccl().all_gather(send, recv, bytes_per_rank, ncclUint8, c->comm, ctx->stream), "ncclAllGather");
    });
}

}  // extern "C"
