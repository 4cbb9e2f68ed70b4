// misc.cu -- K5 combine, the int4-g128 quantiser, synthetic tensor generators.
#include <algorithm>

#include "common.cuh"
#include "launch.h"

namespace moek {

// K5: out[t, c] = bf16(res[t, c] + sum_j w[t,j] * y[inv[t*k+j], c]); fp32 fma
// chain in j order (oracle orc_combine).  One thread per 4 columns.
__global__ void combine_kernel(const float* __restrict__ y, const int32_t* __restrict__ inv,
                               const float* __restrict__ w, const uint16_t* __restrict__ res,
                               int T, int d, int k, uint16_t* __restrict__ out) {
    const int groups = d / 4;
    const long long gid = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (gid >= static_cast<long long>(T) * groups) return;
    const int t = static_cast<int>(gid / groups), c = static_cast<int>(gid - static_cast<long long>(t) * groups) * 4;
    float acc[4] = {0.f, 0.f, 0.f, 0.f};
    if (res) {
        const uint2 r = *reinterpret_cast<const uint2*>(res + static_cast<size_t>(t) * d + c);
        acc[0] = bf16_lo(r.x);
        acc[1] = bf16_hi(r.x);
        acc[2] = bf16_lo(r.y);
        acc[3] = bf16_hi(r.y);
    }
    for (int j = 0; j < k; ++j) {
        const float wj = w[t * k + j];
        const float4 v = *reinterpret_cast<const float4*>(y + static_cast<size_t>(inv[t * k + j]) * d + c);
        acc[0] = __fmaf_rn(wj, v.x, acc[0]);
        acc[1] = __fmaf_rn(wj, v.y, acc[1]);
        acc[2] = __fmaf_rn(wj, v.z, acc[2]);
        acc[3] = __fmaf_rn(wj, v.w, acc[3]);
    }
    uint2 o;
    o.x = static_cast<uint32_t>(f2bf(acc[0])) | (static_cast<uint32_t>(f2bf(acc[1])) << 16);
    o.y = static_cast<uint32_t>(f2bf(acc[2])) | (static_cast<uint32_t>(f2bf(acc[3])) << 16);
    *reinterpret_cast<uint2*>(out + static_cast<size_t>(t) * d + c) = o;
}

// Expert-parallel combine: this rank's share of every token's output,
// part[t, c] = sum over j with expert idx[t,j] in `mask` of w[t,j] * y[inv[t*k+j], c]
// (fp32 fma chain in j order from 0); the ranks' shares are summed by a
// reduce-scatter and added to the residual by residual_add_kernel.
__global__ void combine_partial_kernel(const float* __restrict__ y, const int32_t* __restrict__ inv,
                                       const float* __restrict__ w, const int32_t* __restrict__ idx,
                                       unsigned long long mask, int T, int d, int k, float* __restrict__ out) {
    const int groups = d / 4;
    const long long gid = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (gid >= static_cast<long long>(T) * groups) return;
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
    *reinterpret_cast<float4*>(out + static_cast<size_t>(t) * d + c) = acc;
}

// out = bf16(res + part), one rounding
__global__ void residual_add_kernel(const uint16_t* __restrict__ res, const float* __restrict__ part, long long n,
                                    uint16_t* __restrict__ out) {
    for (long long i = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
         i += static_cast<long long>(gridDim.x) * blockDim.x)
        out[i] = f2bf(__fadd_rn(bf2f(res[i]), part[i]));
}

// int4-g128 RTN quantiser (oracle orc_quantize_g128): one warp per
// (row, 128-group); lane l owns elements 4l..4l+3.
__global__ void quantize_kernel(const uint16_t* __restrict__ w, int rows, int cols,
                                uint32_t* __restrict__ q, uint16_t* __restrict__ s) {
    const int groups = cols / 128;
    const long long wid = (static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (wid >= static_cast<long long>(rows) * groups) return;
    const int r = static_cast<int>(wid / groups), g = static_cast<int>(wid - static_cast<long long>(r) * groups);
    const uint16_t* src = w + static_cast<size_t>(r) * cols + g * 128 + lane * 4;
    const uint2 raw = *reinterpret_cast<const uint2*>(src);
    const float v[4] = {bf16_lo(raw.x), bf16_hi(raw.x), bf16_lo(raw.y), bf16_hi(raw.y)};
    float amax = fmaxf(fmaxf(fabsf(v[0]), fabsf(v[1])), fmaxf(fabsf(v[2]), fabsf(v[3])));
#pragma unroll
    for (int off = 16; off >= 1; off >>= 1) amax = fmaxf(amax, __shfl_xor_sync(0xffffffffu, amax, off));
    const uint16_t sb = amax == 0.0f ? f2bf(1.0f) : f2bf(__fdiv_rn(amax, 7.0f));
    const float sf = bf2f(sb);
    // element e = lane*4 + i lies in word (lane*4+i)/8 = lane/2, j = (lane&1)*4 + i
    uint32_t part = 0;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        float qv = rintf(__fdiv_rn(v[i], sf));
        qv = fminf(7.0f, fmaxf(-8.0f, qv));
        const uint32_t u = static_cast<uint32_t>(static_cast<int>(qv) + 8);
        const int j = (lane & 1) * 4 + i;
        part |= u << (4 * (j >> 1) + 16 * (j & 1));
    }
    const uint32_t word = part | __shfl_xor_sync(0xffffffffu, part, 1);
    if ((lane & 1) == 0) q[static_cast<size_t>(r) * (cols / 8) + g * 16 + lane / 2] = word;
    if (lane == 0) s[static_cast<size_t>(r) * groups + g] = sb;
}

// ---- fragment-block storage layout (oracle orc_pack_*_blocks) -------------
MOE_DEVI int inv_perm_pos(int p) {  // pi^-1
    const int t = p >> 5, r = p & 31;
    return (r >> 2) * 16 + ((r >> 1) & 1) * 8 + t * 2 + (r & 1);
}

// bf16 block (16 rows x 128 K) in UMMA core-matrix order (oracle
// bf16_block_index): [K half][row half][8-K column][row][8 values].
MOE_DEVI size_t bf16_block_pos(int row, int c, int G) {
    const int kin = c & 127, rr = row & 15;
    return (static_cast<size_t>(row >> 4) * G + (c >> 7)) * 2048 +
           static_cast<size_t>((kin >> 6) * 1024 + (rr >> 3) * 512 + ((kin & 63) >> 3) * 64 + (rr & 7) * 8 + (kin & 7));
}

__global__ void pack_bf16_blocks_kernel(const uint16_t* __restrict__ w, int rows, int cols,
                                        uint16_t* __restrict__ out) {
    const long long n = static_cast<long long>(rows) * cols;
    const int G = cols / 128;
    for (long long o = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x; o < n;
         o += static_cast<long long>(gridDim.x) * blockDim.x) {
        const int row = static_cast<int>(o / cols), c = static_cast<int>(o - static_cast<long long>(row) * cols);
        out[bf16_block_pos(row, c, G)] = w[o];
    }
}

// Inverse of pack_bf16_blocks_kernel, walked in storage order (coalesced
// reads; each 8-value core-matrix row is one contiguous 16-byte write).
__global__ void unpack_bf16_blocks_kernel(const uint16_t* __restrict__ in, int rows, int cols,
                                          uint16_t* __restrict__ w) {
    const long long n = static_cast<long long>(rows) * cols;
    const int G = cols / 128;
    for (long long p = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x; p < n;
         p += static_cast<long long>(gridDim.x) * blockDim.x) {
        const int e = static_cast<int>(p & 7), r8 = static_cast<int>((p >> 3) & 7), cc = static_cast<int>((p >> 6) & 7);
        const int cr = static_cast<int>((p >> 9) & 1), h = static_cast<int>((p >> 10) & 1);
        const long long blk = p >> 11;
        const int rt = static_cast<int>(blk / G), g = static_cast<int>(blk - static_cast<long long>(rt) * G);
        const int row = rt * 16 + cr * 8 + r8, c = g * 128 + h * 64 + cc * 8 + e;
        w[static_cast<size_t>(row) * cols + c] = in[p];
    }
}

// int4-g128 RTN quantiser writing the block layout: one warp per (row,
// 128-group).  Same arithmetic as orc_quantize_g128.
__global__ void quantize_blocks_kernel(const uint16_t* __restrict__ w, int rows, int cols,
                                       uint32_t* __restrict__ qb, uint16_t* __restrict__ sb) {
    const int G = cols / 128;
    const long long wid = (static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (wid >= static_cast<long long>(rows) * G) return;
    const int row = static_cast<int>(wid / G), g = static_cast<int>(wid - static_cast<long long>(row) * G);
    const uint16_t* src = w + static_cast<size_t>(row) * cols + g * 128;
    const uint2 raw = *reinterpret_cast<const uint2*>(src + lane * 4);
    float amax = fmaxf(fmaxf(fabsf(bf16_lo(raw.x)), fabsf(bf16_hi(raw.x))),
                       fmaxf(fabsf(bf16_lo(raw.y)), fabsf(bf16_hi(raw.y))));
#pragma unroll
    for (int off = 16; off >= 1; off >>= 1) amax = fmaxf(amax, __shfl_xor_sync(0xffffffffu, amax, off));
    const uint16_t s16 = amax == 0.0f ? f2bf(1.0f) : f2bf(__fdiv_rn(amax, 7.0f));
    const float sf = bf2f(s16);
    const int rt = row >> 4, rr = row & 15, gr = rr & 7, half = rr >> 3;
    const size_t blk = static_cast<size_t>(rt) * G + g;
    if (lane < 16) {
        const int tb = lane >> 2, q = lane & 3;  // lane-block t, word q
        uint32_t word = 0;
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            const int k = inv_perm_pos(tb * 32 + q * 8 + j);
            float qv = rintf(__fdiv_rn(bf2f(src[k]), sf));
            qv = fminf(7.0f, fmaxf(-8.0f, qv));
            word |= static_cast<uint32_t>(static_cast<int>(qv) + 8) << (4 * (j >> 1) + 16 * (j & 1));
        }
        qb[blk * 256 + static_cast<size_t>((half * 32 + gr * 4 + tb) * 4 + q)] = word;
    }
    if (lane == 0) sb[blk * 16 + gr * 2 + half] = s16;
}

MOE_DEVI uint64_t mix64(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}

// r(seed, uid, i) = mix64(mix64(seed ^ uid*C) + (i+1)*golden)  (orc_rand64)
__global__ void synth_weight_kernel(uint64_t key, long long n, float scale, uint16_t* __restrict__ out) {
    const long long stride = static_cast<long long>(gridDim.x) * blockDim.x * 8;
    for (long long i0 = (static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x) * 8; i0 < n; i0 += stride) {
        if (i0 + 8 <= n) {
            uint32_t pk[4];
#pragma unroll
            for (int j = 0; j < 8; j += 2) {
                const int8_t a = static_cast<int8_t>(mix64(key + static_cast<uint64_t>(i0 + j + 1) * 0x9E3779B97F4A7C15ULL) >> 56);
                const int8_t b = static_cast<int8_t>(mix64(key + static_cast<uint64_t>(i0 + j + 2) * 0x9E3779B97F4A7C15ULL) >> 56);
                pk[j / 2] = static_cast<uint32_t>(f2bf(static_cast<float>(a) * scale)) |
                            (static_cast<uint32_t>(f2bf(static_cast<float>(b) * scale)) << 16);
            }
            *reinterpret_cast<uint4*>(out + i0) = make_uint4(pk[0], pk[1], pk[2], pk[3]);
        } else {
            for (long long i = i0; i < n; ++i) {
                const int8_t a = static_cast<int8_t>(mix64(key + static_cast<uint64_t>(i + 1) * 0x9E3779B97F4A7C15ULL) >> 56);
                out[i] = f2bf(static_cast<float>(a) * scale);
            }
        }
    }
}

__global__ void synth_input_kernel(uint64_t key, long long n, uint16_t* __restrict__ out) {
    const long long i = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const uint64_t r = mix64(key + static_cast<uint64_t>(i + 1) * 0x9E3779B97F4A7C15ULL);
    const int kq = static_cast<int>((r >> 32) % 129u) - 64;
    out[i] = f2bf(static_cast<float>(kq) / 64.0f);
}

uint64_t synth_key(uint64_t seed, uint64_t uid) {
    uint64_t z = seed ^ (uid * 0xD1B54A32D192ED03ULL);
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}

}  // namespace moek

cudaError_t moek_combine(const float* y, const int32_t* inv, const float* w, const void* res, int T,
                         int d, int k, void* out, cudaStream_t stream) {
    const long long n = static_cast<long long>(T) * (d / 4);
    if (n == 0) return cudaSuccess;
    const int threads = 256;
    moek::combine_kernel<<<static_cast<unsigned>((n + threads - 1) / threads), threads, 0, stream>>>(
        y, inv, w, static_cast<const uint16_t*>(res), T, d, k, static_cast<uint16_t*>(out));
    return cudaGetLastError();
}

cudaError_t moek_combine_partial(const float* y, const int32_t* inv, const float* w, const int32_t* idx,
                                 unsigned long long mask, int T, int d, int k, float* out, cudaStream_t stream) {
    const long long n = static_cast<long long>(T) * (d / 4);
    if (n == 0) return cudaSuccess;
    moek::combine_partial_kernel<<<static_cast<unsigned>((n + 255) / 256), 256, 0, stream>>>(y, inv, w, idx, mask, T, d,
                                                                                           k, out);
    return cudaGetLastError();
}

cudaError_t moek_residual_add(const void* res, const float* part, long long n, void* out, cudaStream_t stream) {
    if (n == 0) return cudaSuccess;
    const long long blocks = std::min<long long>((n + 255) / 256, 4096);
    moek::residual_add_kernel<<<static_cast<unsigned>(blocks), 256, 0, stream>>>(
        static_cast<const uint16_t*>(res), part, n, static_cast<uint16_t*>(out));
    return cudaGetLastError();
}

cudaError_t moek_quantize(const void* w, int rows, int cols, uint32_t* q, void* s, cudaStream_t stream) {
    const long long warps = static_cast<long long>(rows) * (cols / 128);
    if (warps == 0) return cudaSuccess;
    const int threads = 256;
    moek::quantize_kernel<<<static_cast<unsigned>((warps * 32 + threads - 1) / threads), threads, 0, stream>>>(
        static_cast<const uint16_t*>(w), rows, cols, q, static_cast<uint16_t*>(s));
    return cudaGetLastError();
}

cudaError_t moek_pack_bf16_blocks(const void* w, int rows, int cols, void* out, cudaStream_t stream) {
    const long long n = static_cast<long long>(rows) * cols;
    if (n == 0) return cudaSuccess;
    long long blocks = (n + 255) / 256;
    if (blocks > 148 * 64) blocks = 148 * 64;
    moek::pack_bf16_blocks_kernel<<<static_cast<unsigned>(blocks), 256, 0, stream>>>(
        static_cast<const uint16_t*>(w), rows, cols, static_cast<uint16_t*>(out));
    return cudaGetLastError();
}

cudaError_t moek_unpack_bf16_blocks(const void* in, int rows, int cols, void* w, cudaStream_t stream) {
    const long long n = static_cast<long long>(rows) * cols;
    if (n == 0) return cudaSuccess;
    long long blocks = (n + 255) / 256;
    if (blocks > 148 * 64) blocks = 148 * 64;
    moek::unpack_bf16_blocks_kernel<<<static_cast<unsigned>(blocks), 256, 0, stream>>>(
        static_cast<const uint16_t*>(in), rows, cols, static_cast<uint16_t*>(w));
    return cudaGetLastError();
}

cudaError_t moek_quantize_blocks(const void* w, int rows, int cols, uint32_t* qb, void* sb, cudaStream_t stream) {
    const long long warps = static_cast<long long>(rows) * (cols / 128);
    if (warps == 0) return cudaSuccess;
    const int threads = 256;
    moek::quantize_blocks_kernel<<<static_cast<unsigned>((warps * 32 + threads - 1) / threads), threads, 0, stream>>>(
        static_cast<const uint16_t*>(w), rows, cols, qb, static_cast<uint16_t*>(sb));
    return cudaGetLastError();
}

cudaError_t moek_synth_weight(uint64_t seed, uint64_t uid, long long n, int shift, void* out,
                              cudaStream_t stream) {
    if (n <= 0) return cudaSuccess;
    const float scale = ldexpf(1.0f, -shift);
    long long blocks = (n / 8 + 255) / 256 + 1;
    if (blocks > 148 * 64) blocks = 148 * 64;
    moek::synth_weight_kernel<<<static_cast<unsigned>(blocks), 256, 0, stream>>>(
        moek::synth_key(seed, uid), n, scale, static_cast<uint16_t*>(out));
    return cudaGetLastError();
}

cudaError_t moek_synth_input(uint64_t seed, uint64_t uid, long long n, void* out, cudaStream_t stream) {
    if (n <= 0) return cudaSuccess;
    moek::synth_input_kernel<<<static_cast<unsigned>((n + 255) / 256), 256, 0, stream>>>(
        moek::synth_key(seed, uid), n, static_cast<uint16_t*>(out));
    return cudaGetLastError();
}

// Loads this unit's kernels now (cudaFuncGetAttributes).  Under lazy module
// loading (CUDA 12 default) a kernel's first launch may wait for the device
// to idle; the expert-parallel step has kernels that spin on a peer's flags,
// so every kernel it can launch must be resident before the first step.
cudaError_t moek_preload_misc() {
    cudaFuncAttributes fa;
    MOE_CUDA_OK_PRELOAD(cudaFuncGetAttributes(&fa, moek::combine_kernel));
    MOE_CUDA_OK_PRELOAD(cudaFuncGetAttributes(&fa, moek::combine_partial_kernel));
    MOE_CUDA_OK_PRELOAD(cudaFuncGetAttributes(&fa, moek::residual_add_kernel));
    return cudaSuccess;
}
