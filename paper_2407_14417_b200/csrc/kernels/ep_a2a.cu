// ep_a2a.cu -- expert-parallel all-to-all of routed rows over peer memory
// (NVLink P2P / CUDA IPC), the sharded engine's exchange (SURVEY.md §8e,
// DESIGN.md §6).  Every rank owns the experts of slots s with s*G/E == rank
// in every layer; tokens stay on their rank.  Per layer:
//
//   dispatch   each routed entry (t, j) of this rank's T tokens goes to the
//              owner of its expert: the normalised token row is stored
//              straight into the owner's rows[rank][t*k+j], the expert id into
//              meta[rank][t*k+j] (-1 in every other rank's copy of the slot),
//              then one system-scope release flag per peer.  Only routed
//              rows move (G*T*k rows per layer over all ranks, not G*T*d).
//   wait       the G row flags of this layer
//   (the owner's experts run on the received entries: meta -> counting sort
//    with the not-mine entries under a dummy expert E, then the GEMV or the
//    tcgen05 GEMM with k = 1 -- the product kernels)
//   return     each computed entry's fp32 output row goes straight into its
//              source rank's ret[t*k+j], then one release flag per peer
//   wait       the G return flags
//   combine    out[t] = bf16(x[t] + sum_j w[t,j] * ret[t*k+j]), fp32 fma
//              chain in j order (moek_combine with the identity inverse).
//
// Epochs: a device word per rank (`epoch`), bumped by L at the end of each
// step; layer l of the step waits for flags >= epoch + l + 1, so a captured
// graph replays with fresh epochs.  A rank cannot run more than one layer
// ahead of a peer (it waits for that peer's returns every layer), and a peer
// reads its rows / meta before it returns, so one buffer per direction is
// enough.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>

#include "common.cuh"
#include "launch.h"

namespace moek {
namespace epa {

constexpr int kMaxRanks = 8;

struct Peers {
    char* base[kMaxRanks];
};

struct Layout {
    size_t rows, meta, ret, flags, ticket, total;
};

__host__ __device__ inline size_t al(size_t v) { return (v + 255) / 256 * 256; }

// C = capacity (entries) per source rank = T_max * k
__host__ __device__ inline Layout layout(int G, int C, int d) {
    Layout l;
    l.rows = 0;
    l.meta = al(static_cast<size_t>(G) * C * d * 2);
    l.ret = l.meta + al(static_cast<size_t>(G) * C * 4);
    l.flags = l.ret + al(static_cast<size_t>(C) * d * 4);
    l.ticket = l.flags + al(2 * kMaxRanks * 4);
    l.total = l.ticket + 256;
    return l;
}

MOE_DEVI void st_release_sys(uint32_t* p, uint32_t v) {
    asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
MOE_DEVI uint32_t ld_acquire_sys(const uint32_t* p) {
    uint32_t v;
    asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

MOE_DEVI int owner_of(int slot, int E, int G) { return slot * G / E; }

// The last block to finish releases flag `which`[rank] = epoch on every peer.
MOE_DEVI void release_all(const Peers& pe, int G, const Layout& L, int which, int rank, uint32_t epoch,
                          unsigned int* ticket) {
    __shared__ bool last;
    __threadfence_system();  // this block's peer stores, system-wide
    __syncthreads();
    if (threadIdx.x == 0) last = atomicAdd(ticket, 1u) == gridDim.x - 1;
    __syncthreads();
    if (!last) return;
    __threadfence_system();
    if (static_cast<int>(threadIdx.x) < G) {
        uint32_t* f = reinterpret_cast<uint32_t*>(pe.base[threadIdx.x] + L.flags) + which * kMaxRanks + rank;
        st_release_sys(f, epoch);
    }
    if (threadIdx.x == 0) *ticket = 0;
}

// rows of this rank's T tokens -> owners; meta for every (peer, entry < C)
__global__ void dispatch_kernel(const uint16_t* __restrict__ xn, const int32_t* __restrict__ idx, int T, int k,
                                int E, int d, int C, int rank, int G, Peers pe, const uint32_t* epoch_base,
                                int layer) {
    const Layout L = layout(G, C, d);
    const int n = T * k, chunks = d / 8;
    const long long total = static_cast<long long>(n) * chunks;
    for (long long i = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x; i < total;
         i += static_cast<long long>(gridDim.x) * blockDim.x) {
        const int e = static_cast<int>(i / chunks), c = static_cast<int>(i - static_cast<long long>(e) * chunks);
        const int o = owner_of(idx[e], E, G);
        const uint4 v = reinterpret_cast<const uint4*>(xn + static_cast<size_t>(e / k) * d)[c];
        reinterpret_cast<uint4*>(pe.base[o] + L.rows + (static_cast<size_t>(rank) * C + e) * d * 2)[c] = v;
    }
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < G * C; i += gridDim.x * blockDim.x) {
        const int p = i / C, e = i - p * C;
        const int ex = e < n ? idx[e] : -1;
        reinterpret_cast<int32_t*>(pe.base[p] + L.meta)[static_cast<size_t>(rank) * C + e] =
            ex >= 0 && owner_of(ex, E, G) == p ? ex : -1;
    }
    release_all(pe, G, L, 0, rank, *epoch_base + layer + 1, reinterpret_cast<unsigned int*>(pe.base[rank] + L.ticket));
}

MOE_DEVI unsigned long long gtime() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}

// Spins until every peer's flag reaches this layer's epoch.  A peer that
// never arrives (a rank died, a mismatched step count) traps after 20 s
// instead of hanging the device.
__global__ void wait_kernel(const uint32_t* flags, int G, const uint32_t* epoch_base, int layer) {
    const uint32_t want = *epoch_base + layer + 1;
    if (static_cast<int>(threadIdx.x) < G) {
        const unsigned long long t0 = gtime();
        while (ld_acquire_sys(flags + threadIdx.x) < want)
            if (gtime() - t0 > 20000000000ull) {
                printf("ep wait timeout: layer %d flag[%d]=%u want %u\n", layer, threadIdx.x, flags[threadIdx.x], want);
                __trap();
            }
    }
    __syncthreads();
}

// meta (-1: not mine) -> the counting-sort key: this rank's entries keep
// their expert, the rest go to the dummy expert E (sorted after every real one)
__global__ void meta_keys_kernel(const int32_t* __restrict__ meta, int n, int E, int32_t* __restrict__ keys) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        const int m = meta[i];
        keys[i] = m < 0 ? E : m;
    }
}

// computed slot q (perm[q] = entry position p = src*C + e) -> src's ret[e]
__global__ void return_kernel(const float* __restrict__ y, const int32_t* __restrict__ perm,
                              const int32_t* __restrict__ offsets, int E, int d, int C, int rank, int G, Peers pe,
                              const uint32_t* epoch_base, int layer) {
    const Layout L = layout(G, C, d);
    const int nvalid = offsets[E];
    const int chunks = d / 4;
    const long long total = static_cast<long long>(nvalid) * chunks;
    for (long long i = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x; i < total;
         i += static_cast<long long>(gridDim.x) * blockDim.x) {
        const int q = static_cast<int>(i / chunks), c = static_cast<int>(i - static_cast<long long>(q) * chunks);
        const int p = perm[q], src = p / C, e = p - src * C;
        const float4 v = reinterpret_cast<const float4*>(y + static_cast<size_t>(q) * d)[c];
        reinterpret_cast<float4*>(pe.base[src] + L.ret + static_cast<size_t>(e) * d * 4)[c] = v;
    }
    release_all(pe, G, L, 1, rank, *epoch_base + layer + 1, reinterpret_cast<unsigned int*>(pe.base[rank] + L.ticket));
}

// received rows in slot order (q < offsets[E]: row perm[q]) -> dense rows
// for the GEMV path (its workspace is sized by rows actually servable)
__global__ void gather_kernel(const uint16_t* __restrict__ rows, const int32_t* __restrict__ perm,
                              const int32_t* __restrict__ offsets, int E, int d, uint16_t* __restrict__ dense) {
    const int nvalid = offsets[E], chunks = d / 8;
    const long long total = static_cast<long long>(nvalid) * chunks;
    for (long long i = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x; i < total;
         i += static_cast<long long>(gridDim.x) * blockDim.x) {
        const int q = static_cast<int>(i / chunks), c = static_cast<int>(i - static_cast<long long>(q) * chunks);
        reinterpret_cast<uint4*>(dense + static_cast<size_t>(q) * d)[c] =
            reinterpret_cast<const uint4*>(rows + static_cast<size_t>(perm[q]) * d)[c];
    }
}

__global__ void bump_epoch_kernel(uint32_t* epoch_base, int L) {
    if (threadIdx.x == 0) *epoch_base += static_cast<uint32_t>(L);
}

}  // namespace epa
}  // namespace moek

namespace {

moek::epa::Peers peers_of(const void* const* bases, int G) {
    moek::epa::Peers p{};
    for (int i = 0; i < G; ++i) p.base[i] = static_cast<char*>(const_cast<void*>(bases[i]));
    return p;
}

unsigned grid_for(long long work) {
    return static_cast<unsigned>(std::max<long long>(1, std::min<long long>((work + 255) / 256, 592)));
}

}  // namespace

size_t moek_ep_a2a_bytes(int G, int C, int d) { return moek::epa::layout(G, C, d).total; }
size_t moek_ep_a2a_offset(int G, int C, int d, int which) {
    const moek::epa::Layout L = moek::epa::layout(G, C, d);
    switch (which) {
        case 0: return L.rows;
        case 1: return L.meta;
        case 2: return L.ret;
        case 3: return L.flags;
        default: return L.ticket;
    }
}

cudaError_t moek_ep_a2a_dispatch(const void* xn, const int32_t* idx, int T, int k, int E, int d, int C, int rank,
                                 int G, const void* const* bases, const uint32_t* epoch_base, int layer,
                                 cudaStream_t stream) {
    if (G < 1 || G > moek::epa::kMaxRanks || d % 8 != 0 || T * k > C || E < G) return cudaErrorInvalidValue;
    moek::epa::dispatch_kernel<<<grid_for(std::max<long long>(static_cast<long long>(T) * k * (d / 8), G * C)), 256, 0,
                                 stream>>>(static_cast<const uint16_t*>(xn), idx, T, k, E, d, C, rank, G,
                                           peers_of(bases, G), epoch_base, layer);
    return cudaGetLastError();
}

cudaError_t moek_ep_a2a_wait(const void* my_base, int which, int G, int C, int d, const uint32_t* epoch_base,
                             int layer, cudaStream_t stream) {
    const moek::epa::Layout L = moek::epa::layout(G, C, d);
    moek::epa::wait_kernel<<<1, 32, 0, stream>>>(
        reinterpret_cast<const uint32_t*>(static_cast<const char*>(my_base) + L.flags) + which * moek::epa::kMaxRanks, G,
        epoch_base, layer);
    return cudaGetLastError();
}

cudaError_t moek_ep_a2a_keys(const int32_t* meta, int n, int E, int32_t* keys, cudaStream_t stream) {
    moek::epa::meta_keys_kernel<<<grid_for(n), 256, 0, stream>>>(meta, n, E, keys);
    return cudaGetLastError();
}

cudaError_t moek_ep_a2a_return(const float* y, const int32_t* perm, const int32_t* offsets, int E, int d, int C,
                               int rank, int G, const void* const* bases, const uint32_t* epoch_base, int layer,
                               cudaStream_t stream) {
    if (G < 1 || G > moek::epa::kMaxRanks || d % 4 != 0) return cudaErrorInvalidValue;
    moek::epa::return_kernel<<<grid_for(static_cast<long long>(G) * C * (d / 4)), 256, 0, stream>>>(
        y, perm, offsets, E, d, C, rank, G, peers_of(bases, G), epoch_base, layer);
    return cudaGetLastError();
}

cudaError_t moek_ep_a2a_gather(const void* rows, const int32_t* perm, const int32_t* offsets, int E, int d,
                               int max_rows, void* dense, cudaStream_t stream) {
    moek::epa::gather_kernel<<<grid_for(static_cast<long long>(max_rows) * (d / 8)), 256, 0, stream>>>(
        static_cast<const uint16_t*>(rows), perm, offsets, E, d, static_cast<uint16_t*>(dense));
    return cudaGetLastError();
}

cudaError_t moek_ep_a2a_bump(uint32_t* epoch_base, int L, cudaStream_t stream) {
    moek::epa::bump_epoch_kernel<<<1, 32, 0, stream>>>(epoch_base, L);
    return cudaGetLastError();
}

// Loads this unit's kernels now (cudaFuncGetAttributes).  Under lazy module
// loading (CUDA 12 default) a kernel's first launch may wait for the device
// to idle; the expert-parallel step has kernels that spin on a peer's flags,
// so every kernel it can launch must be resident before the first step.
cudaError_t moek_preload_ep() {
    cudaFuncAttributes fa;
    MOE_CUDA_OK_PRELOAD(cudaFuncGetAttributes(&fa, moek::epa::dispatch_kernel));
    MOE_CUDA_OK_PRELOAD(cudaFuncGetAttributes(&fa, moek::epa::wait_kernel));
    MOE_CUDA_OK_PRELOAD(cudaFuncGetAttributes(&fa, moek::epa::meta_keys_kernel));
    MOE_CUDA_OK_PRELOAD(cudaFuncGetAttributes(&fa, moek::epa::return_kernel));
    MOE_CUDA_OK_PRELOAD(cudaFuncGetAttributes(&fa, moek::epa::gather_kernel));
    MOE_CUDA_OK_PRELOAD(cudaFuncGetAttributes(&fa, moek::epa::bump_epoch_kernel));
    return cudaSuccess;
}
