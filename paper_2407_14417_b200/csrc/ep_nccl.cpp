// ep_nccl.cpp -- the expert-parallel exchange of the C ABI (SURVEY.md §8b:
// "EP adds moe_ep_dispatch / moe_ep_combine taking an ncclComm_t").
//
// Per layer (ep.py): dispatch = all-gather of every rank's
// token rows (bf16), combine = reduce-scatter of the fp32 expert shares, so
// each rank receives the summed share of its own tokens.  NCCL is loaded at
// run time (dlopen): the NCCL already in the process (torch's bundled
// libnccl.so.2) is reused, else the bundled copy, else the system one, so
// this library never pins a second NCCL next to torch's.
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>

#include <cstdlib>
#include <cstring>
#include <mutex>
#include <stdexcept>
#include <string>

#include "moe_b200.h"

namespace {

struct NcclApi {
    ncclResult_t (*get_unique_id)(ncclUniqueId*) = nullptr;
    ncclResult_t (*comm_init_rank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*comm_destroy)(ncclComm_t) = nullptr;
    ncclResult_t (*all_gather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*reduce_scatter)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                                   cudaStream_t) = nullptr;
    const char* (*error_string)(ncclResult_t) = nullptr;
    std::string path;
};

const NcclApi& nccl() {
    static NcclApi api;
    static std::once_flag once;
    std::call_once(once, [] {
        const char* env = std::getenv("MOE_NCCL_LIB");
        const char* cands[] = {env, "libnccl.so.2",
                               "/opt/prime-rl/.venv/lib/python3.12/site-packages/nvidia/nccl/lib/libnccl.so.2",
                               "/usr/lib/x86_64-linux-gnu/libnccl.so.2"};
        void* h = nullptr;
        // an NCCL already loaded in the process (torch's) first
        h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
        if (h) api.path = "libnccl.so.2 (already loaded)";
        for (const char* c : cands) {
            if (h) break;
            if (c && (h = dlopen(c, RTLD_NOW | RTLD_LOCAL))) api.path = c;
        }
        if (!h) return;
        api.get_unique_id = reinterpret_cast<decltype(api.get_unique_id)>(dlsym(h, "ncclGetUniqueId"));
        api.comm_init_rank = reinterpret_cast<decltype(api.comm_init_rank)>(dlsym(h, "ncclCommInitRank"));
        api.comm_destroy = reinterpret_cast<decltype(api.comm_destroy)>(dlsym(h, "ncclCommDestroy"));
        api.all_gather = reinterpret_cast<decltype(api.all_gather)>(dlsym(h, "ncclAllGather"));
        api.reduce_scatter = reinterpret_cast<decltype(api.reduce_scatter)>(dlsym(h, "ncclReduceScatter"));
        api.error_string = reinterpret_cast<decltype(api.error_string)>(dlsym(h, "ncclGetErrorString"));
    });
    if (!api.get_unique_id || !api.comm_init_rank || !api.all_gather || !api.reduce_scatter)
        throw std::runtime_error("NCCL not available (set MOE_NCCL_LIB to libnccl.so.2)");
    return api;
}

void nck(ncclResult_t r, const char* what) {
    if (r != ncclSuccess)
        throw std::runtime_error(std::string(what) + ": " + (nccl().error_string ? nccl().error_string(r) : "NCCL error"));
}

thread_local std::string g_ep_err;

template <class F>
int ep_guard(F&& f) {
    try {
        f();
        return MOE_OK;
    } catch (const std::invalid_argument& e) {
        g_ep_err = e.what();
        return MOE_ERR_USAGE;
    } catch (const std::exception& e) {
        g_ep_err = e.what();
        return MOE_ERR_INTERNAL;
    }
}

void usage(bool bad, const char* msg) {
    if (bad) throw std::invalid_argument(msg);
}

}  // namespace

struct moe_ep_comm {
    ncclComm_t comm = nullptr;
    int world = 0, rank = 0;
    bool owned = false;
};

extern "C" {

const char* moe_ep_last_error(void) { return g_ep_err.c_str(); }

int moe_ep_unique_id(char id[MOE_EP_ID_BYTES]) {
    return ep_guard([&] {
        usage(id == nullptr, "null argument");
        static_assert(sizeof(ncclUniqueId) <= MOE_EP_ID_BYTES, "id buffer");
        ncclUniqueId u;
        nck(nccl().get_unique_id(&u), "ncclGetUniqueId");
        std::memcpy(id, &u, sizeof u);
    });
}

int moe_ep_comm_init(const char id[MOE_EP_ID_BYTES], int world, int rank, int device, moe_ep_comm** out) {
    return ep_guard([&] {
        usage(id == nullptr || out == nullptr, "null argument");
        usage(world < 1 || rank < 0 || rank >= world, "bad world / rank");
        if (cudaSetDevice(device) != cudaSuccess) throw std::runtime_error("cudaSetDevice");
        ncclUniqueId u;
        std::memcpy(&u, id, sizeof u);
        auto* c = new moe_ep_comm;
        c->world = world;
        c->rank = rank;
        c->owned = true;
        const ncclResult_t r = nccl().comm_init_rank(&c->comm, world, u, rank);
        if (r != ncclSuccess) {
            delete c;
            nck(r, "ncclCommInitRank");
        }
        *out = c;
    });
}

int moe_ep_comm_wrap(void* nccl_comm, int world, int rank, moe_ep_comm** out) {
    return ep_guard([&] {
        usage(nccl_comm == nullptr || out == nullptr, "null argument");
        usage(world < 1 || rank < 0 || rank >= world, "bad world / rank");
        *out = new moe_ep_comm{static_cast<ncclComm_t>(nccl_comm), world, rank, false};
    });
}

void moe_ep_comm_destroy(moe_ep_comm* c) {
    if (c == nullptr) return;
    if (c->owned && c->comm) nccl().comm_destroy(c->comm);
    delete c;
}

int moe_ep_dispatch(moe_ep_comm* c, const void* x_local, int T_local, int d, void* x_all, void* stream) {
    return ep_guard([&] {
        usage(c == nullptr || x_local == nullptr || x_all == nullptr, "null argument");
        usage(T_local < 0 || d <= 0, "bad shape");
        // bf16 rows move as raw 16-bit words (no arithmetic)
        nck(nccl().all_gather(x_local, x_all, static_cast<size_t>(T_local) * d, ncclBfloat16,
                              c->comm, static_cast<cudaStream_t>(stream)),
            "ncclAllGather");
    });
}

int moe_ep_combine(moe_ep_comm* c, const float* part, int T_local, int d, float* mine, void* stream) {
    return ep_guard([&] {
        usage(c == nullptr || part == nullptr || mine == nullptr, "null argument");
        usage(T_local < 0 || d <= 0, "bad shape");
        nck(nccl().reduce_scatter(part, mine, static_cast<size_t>(T_local) * d, ncclFloat32, ncclSum, c->comm,
                                  static_cast<cudaStream_t>(stream)),
            "ncclReduceScatter");
    });
}

}  // extern "C"
