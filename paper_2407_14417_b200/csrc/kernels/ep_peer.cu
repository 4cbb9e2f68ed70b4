// ep_peer.cu -- the expert-parallel exchange fused into the kernels that
// produce it, over peer memory (NVLink P2P / CUDA IPC), instead of NCCL
// collectives.
//
// Every rank owns one exchange buffer (moe_ep_peer_bytes):
//   [xg    G*T_local rows x d bf16]  every rank's token rows (the gather)
//   [recv  G x T_local x d fp32]     every rank's share of this rank's tokens
//   [flags 2 x 8 u32]                epoch stamps: rows / shares arrived from rank src
//   [ticket u32]                     last-block election of the pushing kernels
// and holds the base pointers of all G buffers (its own included):
//   push_rows    its rows -> slot `rank` of every peer's xg, then releases
//                flags[0][rank] on every peer (one fence.sys after the last block)
//   wait_rows    spins until flags[0][*] == epoch
//   push_shares  the combine of its experts' outputs (moe_combine_partial's
//                arithmetic) written straight into the owner's recv[rank],
//                then flags[1][rank] on every owner
//   reduce       out = bf16(x + sum over src of recv[src]) in src order, after
//                flags[1][*] == epoch -- deterministic
#include <cuda_runtime.h>

#include "common.cuh"
#include "launch.h"

namespace moek {
namespace ep {

constexpr int kMaxPeers = 8;

struct Peers {
    char* base[kMaxPeers];
};

struct Layout {
    size_t xg, recv, flags, ticket, total;
};

__host__ __device__ inline size_t al(size_t v) { return (v + 255) / 256 * 256; }

__host__ __device__ inline Layout layout(int G, int T_local, int d) {
    Layout l;
    l.xg = 0;
    l.recv = al(static_cast<size_t>(G) * T_local * d * 2);
    l.flags = l.recv + al(static_cast<size_t>(G) * T_local * d * 4);
    l.ticket = l.flags + al(2 * kMaxPeers * 4);
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

// The last block to finish releases flag `which`[rank] on every peer.
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
        uint32_t* f = reinterpret_cast<uint32_t*>(pe.base[threadIdx.x] + L.flags) + which * kMaxPeers + rank;
        st_release_sys(f, epoch);
    }
    if (threadIdx.x == 0) *ticket = 0;
}

MOE_DEVI void wait_all(const uint32_t* flags, int G, uint32_t epoch) {
    if (static_cast<int>(threadIdx.x) < G)
        while (ld_acquire_sys(flags + threadIdx.x) < epoch) {
        }
    __syncthreads();
}

__global__ void push_rows_kernel(const uint16_t* __restrict__ x, int T_local, int d, int rank, int G, Peers pe,
                                 uint32_t epoch) {
    const Layout L = layout(G, T_local, d);
    const long long n16 = static_cast<long long>(T_local) * d / 8;  // 16-byte chunks of this rank's rows
    for (int p = 0; p < G; ++p) {
        uint4* dst = reinterpret_cast<uint4*>(pe.base[p] + L.xg + static_cast<size_t>(rank) * T_local * d * 2);
        for (long long i = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x; i < n16;
             i += static_cast<long long>(gridDim.x) * blockDim.x)
            dst[i] = reinterpret_cast<const uint4*>(x)[i];
    }
    release_all(pe, G, L, 0, rank, epoch, reinterpret_cast<unsigned int*>(pe.base[rank] + L.ticket));
}

__global__ void wait_kernel(const uint32_t* flags, int G, uint32_t epoch) { wait_all(flags, G, epoch); }

// token t of the gathered batch (owner t / T_local): this rank's share over
// its experts (bit idx of mask), fp32 fma chain in j order
__global__ void push_shares_kernel(const float* __restrict__ y, const int32_t* __restrict__ inv,
                                   const float* __restrict__ w, const int32_t* __restrict__ idx,
                                   unsigned long long mask, int T_local, int d, int k, int rank, int G, Peers pe,
                                   uint32_t epoch) {
    const Layout L = layout(G, T_local, d);
    const int groups = d / 4, T = G * T_local;
    for (long long gid = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
         gid < static_cast<long long>(T) * groups; gid += static_cast<long long>(gridDim.x) * blockDim.x) {
        const int t = static_cast<int>(gid / groups), c = static_cast<int>(gid - static_cast<long long>(t) * groups) * 4;
        float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
        for (int j = 0; j < k; ++j) {
            if (!((mask >> idx[t * k + j]) & 1ull)) continue;
            const float wj = w[t * k + j];
            const float4 v = *reinterpret_cast<const float4*>(y + static_cast<size_t>(inv[t * k + j]) * d + c);
            acc.x = __fmaf_rn(wj, v.x, acc.x);
            acc.y = __fmaf_rn(wj, v.y, acc.y);
            acc.z = __fmaf_rn(wj, v.z, acc.z);
            acc.w = __fmaf_rn(wj, v.w, acc.w);
        }
        const int owner = t / T_local, tl = t - owner * T_local;
        float* dst = reinterpret_cast<float*>(pe.base[owner] + L.recv) + (static_cast<size_t>(rank) * T_local + tl) * d + c;
        *reinterpret_cast<float4*>(dst) = acc;
    }
    release_all(pe, G, L, 1, rank, epoch, reinterpret_cast<unsigned int*>(pe.base[rank] + L.ticket));
}

__global__ void reduce_kernel(const uint16_t* __restrict__ x, int T_local, int d, int rank, int G, Peers pe,
                              uint32_t epoch, uint16_t* __restrict__ out) {
    const Layout L = layout(G, T_local, d);
    wait_all(reinterpret_cast<const uint32_t*>(pe.base[rank] + L.flags) + kMaxPeers, G, epoch);
    const float* recv = reinterpret_cast<const float*>(pe.base[rank] + L.recv);
    const long long n = static_cast<long long>(T_local) * d;
    for (long long i = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
         i += static_cast<long long>(gridDim.x) * blockDim.x) {
        float s = 0.0f;
        for (int src = 0; src < G; ++src) s = __fadd_rn(s, __ldcv(recv + static_cast<size_t>(src) * n + i));
        out[i] = f2bf(__fadd_rn(bf2f(x[i]), s));
    }
}

}  // namespace ep
}  // namespace moek

namespace {

moek::ep::Peers peers_of(const void* const* bases, int G) {
    moek::ep::Peers p{};
    for (int i = 0; i < G; ++i) p.base[i] = static_cast<char*>(const_cast<void*>(bases[i]));
    return p;
}

unsigned grid_for(long long work) {
    return static_cast<unsigned>(std::max<long long>(1, std::min<long long>((work + 255) / 256, 296)));
}

}  // namespace

size_t moek_ep_peer_bytes(int G, int T_local, int d) { return moek::ep::layout(G, T_local, d).total; }

cudaError_t moek_ep_push_rows(const void* x_local, int T_local, int d, int rank, int G, const void* const* bases,
                              uint32_t epoch, cudaStream_t stream) {
    if (G < 1 || G > moek::ep::kMaxPeers || d % 8 != 0) return cudaErrorInvalidValue;
    moek::ep::push_rows_kernel<<<grid_for(static_cast<long long>(T_local) * d / 8), 256, 0, stream>>>(
        static_cast<const uint16_t*>(x_local), T_local, d, rank, G, peers_of(bases, G), epoch);
    return cudaGetLastError();
}

cudaError_t moek_ep_wait_rows(const void* my_base, int G, int T_local, int d, uint32_t epoch, cudaStream_t stream) {
    const moek::ep::Layout L = moek::ep::layout(G, T_local, d);
    moek::ep::wait_kernel<<<1, 32, 0, stream>>>(
        reinterpret_cast<const uint32_t*>(static_cast<const char*>(my_base) + L.flags), G, epoch);
    return cudaGetLastError();
}

cudaError_t moek_ep_push_shares(const float* y, const int32_t* inv, const float* w, const int32_t* idx,
                                uint64_t mask, int T_local, int d, int k, int rank, int G, const void* const* bases,
                                uint32_t epoch, cudaStream_t stream) {
    if (G < 1 || G > moek::ep::kMaxPeers || d % 4 != 0) return cudaErrorInvalidValue;
    moek::ep::push_shares_kernel<<<grid_for(static_cast<long long>(G) * T_local * (d / 4)), 256, 0, stream>>>(
        y, inv, w, idx, mask, T_local, d, k, rank, G, peers_of(bases, G), epoch);
    return cudaGetLastError();
}

cudaError_t moek_ep_reduce(const void* x_local, int T_local, int d, int rank, int G, const void* const* bases,
                           uint32_t epoch, void* out, cudaStream_t stream) {
    if (G < 1 || G > moek::ep::kMaxPeers) return cudaErrorInvalidValue;
    moek::ep::reduce_kernel<<<grid_for(static_cast<long long>(T_local) * d), 256, 0, stream>>>(
        static_cast<const uint16_t*>(x_local), T_local, d, rank, G, peers_of(bases, G), epoch,
        static_cast<uint16_t*>(out));
    return cudaGetLastError();
}
