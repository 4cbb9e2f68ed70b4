// ring_bench.cu -- isolates the costs of the GEMV data path on B200.
//   mode 0: bulk-copy ring only (wait, release, refill)
//   mode 1: + int4 decode + HMMA per 128-K group (B fragments in registers)
//   mode 2: + B fragments loaded from global (L1-resident 8 KB row)
//   mode 3: LDG.128 streaming, no smem (reference)
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o ring_bench ring_bench.cu
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <vector>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e)); return 1; } } while (0)

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    asm volatile("{\n\t.reg .pred p;\nWAIT_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t@!p bra WAIT_%=;\n}" ::"r"(smem_u32(bar)), "r"(parity) : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
__device__ __forceinline__ uint32_t and_or(uint32_t a, uint32_t m, uint32_t o) {
    uint32_t d; asm("lop3.b32 %0, %1, %2, %3, 0xEA;" : "=r"(d) : "r"(a), "r"(m), "r"(o)); return d;
}
__device__ __forceinline__ void mma_bf16(float (&c)[4], uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3, uint32_t b0, uint32_t b1) {
    asm volatile("mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                 : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3]) : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}
__device__ __forceinline__ void decode_u(uint32_t w, uint32_t& p01, uint32_t& p23, uint32_t& p45, uint32_t& p67) {
    p01 = and_or(w, 0x000F000Fu, 0x43004300u);
    p23 = and_or(w >> 4, 0x000F000Fu, 0x43004300u);
    p45 = and_or(w >> 8, 0x000F000Fu, 0x43004300u);
    p67 = and_or(w >> 12, 0x000F000Fu, 0x43004300u);
}

template <int WARPS, int STAGES, int ITEM>
__global__ void __launch_bounds__(WARPS * 32, 1) ring_kernel(const uint8_t* __restrict__ src, long long n_items,
                                                             const uint16_t* __restrict__ bglob, int mode, float* out) {
    extern __shared__ __align__(128) uint8_t smem[];
    __shared__ __align__(8) uint64_t bars[WARPS][STAGES];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    uint8_t* ring = smem + static_cast<size_t>(warp) * STAGES * ITEM;
    if (lane == 0) {
        for (int s = 0; s < STAGES; ++s) mbar_init(&bars[warp][s], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    const long long W = static_cast<long long>(gridDim.x) * WARPS;
    const long long wid = static_cast<long long>(blockIdx.x) * WARPS + warp;
    const long long i0 = wid * n_items / W, i1 = (wid + 1) * n_items / W;
    long long issued = i0;
    for (int s = 0; s < STAGES && issued < i1; ++s, ++issued)
        if (lane == 0) { mbar_expect_tx(&bars[warp][s], ITEM); bulk_g2s(ring + s * ITEM, src + issued * ITEM, ITEM, &bars[warp][s]); }
    uint32_t phase = 0;
    int stage = 0;
    float acc[4] = {0.f, 0.f, 0.f, 0.f};
    uint4 b[4];
    for (int c = 0; c < 4; ++c) b[c] = make_uint4(0x3f803f80u, 0x3f803f80u, 0x3f803f80u, 0x3f803f80u);
    const int t = lane & 3;
    for (long long i = i0; i < i1; ++i) {
        mbar_wait(&bars[warp][stage], (phase >> stage) & 1u);
        phase ^= 1u << stage;
        const uint8_t* sp = ring + stage * ITEM;
        if (mode >= 1) {
            for (int g = 0; g < ITEM / 1024; ++g) {
                if (mode == 2)
                    for (int c = 0; c < 4; ++c) b[c] = *reinterpret_cast<const uint4*>(bglob + g * 128 + t * 32 + c * 8);
                const uint4 wl = *reinterpret_cast<const uint4*>(sp + g * 1024 + lane * 16);
                const uint4 wh = *reinterpret_cast<const uint4*>(sp + g * 1024 + 512 + lane * 16);
                const uint32_t lo[4] = {wl.x, wl.y, wl.z, wl.w};
                const uint32_t hi[4] = {wh.x, wh.y, wh.z, wh.w};
                float cg[4] = {0.f, 0.f, 0.f, 0.f}, ch[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    uint32_t r0, r2, r0b, r2b, s0, s2, s0b, s2b;
                    decode_u(lo[q], r0, r2, r0b, r2b);
                    decode_u(hi[q], s0, s2, s0b, s2b);
                    mma_bf16(cg, r0, s0, r2, s2, b[q].x, b[q].y);
                    mma_bf16(ch, r0b, s0b, r2b, s2b, b[q].z, b[q].w);
                }
                for (int r = 0; r < 4; ++r) acc[r] += cg[r] + ch[r];
            }
        } else {
            acc[0] += reinterpret_cast<const float*>(sp)[lane];
        }
        fence_proxy_async();
        __syncwarp();
        if (issued < i1) {
            if (lane == 0) { mbar_expect_tx(&bars[warp][stage], ITEM); bulk_g2s(ring + stage * ITEM, src + issued * ITEM, ITEM, &bars[warp][stage]); }
            ++issued;
        }
        stage = stage + 1 == STAGES ? 0 : stage + 1;
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc[0] + acc[1] + acc[2] + acc[3];
}

__global__ void ldg_kernel(const uint4* __restrict__ src, long long n16, float* out) {
    float acc = 0.f;
    const long long stride = static_cast<long long>(gridDim.x) * blockDim.x;
    for (long long i = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x; i < n16; i += stride * 4) {
        uint4 v[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const long long j = i + u * stride;
            if (j < n16) asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v[u].x), "=r"(v[u].y), "=r"(v[u].z), "=r"(v[u].w) : "l"(src + j));
            else v[u] = make_uint4(0, 0, 0, 0);
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) acc += __uint_as_float(v[u].x ^ v[u].w);
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

template <int WARPS, int STAGES, int ITEM>
int run(const uint8_t* d, long long bytes, const uint16_t* bg, float* out, int mode, int sms) {
    const long long n_items = bytes / ITEM;
    const size_t smem = static_cast<size_t>(WARPS) * STAGES * ITEM;
    CK(cudaFuncSetAttribute(ring_kernel<WARPS, STAGES, ITEM>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
    cudaEvent_t a, b;
    cudaEventCreate(&a); cudaEventCreate(&b);
    for (int w = 0; w < 2; ++w) ring_kernel<WARPS, STAGES, ITEM><<<sms, WARPS * 32, smem>>>(d, n_items, bg, mode, out);
    cudaEventRecord(a);
    const int reps = 5;
    for (int r = 0; r < reps; ++r) ring_kernel<WARPS, STAGES, ITEM><<<sms, WARPS * 32, smem>>>(d, n_items, bg, mode, out);
    cudaEventRecord(b);
    CK(cudaEventSynchronize(b));
    float ms = 0; cudaEventElapsedTime(&ms, a, b);
    printf("ring warps=%2d stages=%d item=%5d mode=%d : %7.1f GB/s\n", WARPS, STAGES, ITEM, mode, bytes * reps / (ms * 1e-3) / 1e9);
    return 0;
}

int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const long long bytes = 4LL << 30;  // 4 GiB >> L2
    uint8_t* d; uint16_t* bg; float* out;
    CK(cudaMalloc(&d, bytes));
    CK(cudaMemset(d, 0x11, bytes));
    CK(cudaMalloc(&bg, 1 << 20));
    CK(cudaMemset(bg, 0, 1 << 20));
    CK(cudaMalloc(&out, sms * 4096 * 4));
    {
        cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
        ldg_kernel<<<sms * 8, 256>>>(reinterpret_cast<const uint4*>(d), bytes / 16, out);
        cudaEventRecord(a);
        for (int r = 0; r < 5; ++r) ldg_kernel<<<sms * 8, 256>>>(reinterpret_cast<const uint4*>(d), bytes / 16, out);
        cudaEventRecord(b); cudaEventSynchronize(b);
        float ms; cudaEventElapsedTime(&ms, a, b);
        printf("ldg stream                           : %7.1f GB/s\n", bytes * 5 / (ms * 1e-3) / 1e9);
    }
    for (int mode = 0; mode < 3; ++mode) {
        run<8, 3, 8192>(d, bytes, bg, out, mode, sms);
        run<12, 2, 8192>(d, bytes, bg, out, mode, sms);
        run<16, 2, 6144>(d, bytes, bg, out, mode, sms);
        run<8, 6, 4096>(d, bytes, bg, out, mode, sms);
        run<4, 6, 8192>(d, bytes, bg, out, mode, sms);
        run<24, 2, 4096>(d, bytes, bg, out, mode, sms);
        run<16, 3, 4096>(d, bytes, bg, out, mode, sms);
    }
    return 0;
}
