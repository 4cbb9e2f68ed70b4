// common.cuh -- shared device helpers for the sm_100a MoE kernels.
#pragma once

#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <utility>

#include "moe_b200.h"

#define MOE_DEVI __device__ __forceinline__

namespace moek {

constexpr int kWarp = 32;
constexpr int kMaxExperts = MOE_MAX_EXPERTS;

MOE_DEVI float bf2f(uint16_t b) { return __uint_as_float(static_cast<uint32_t>(b) << 16); }
MOE_DEVI float bf16_lo(uint32_t v) { return __uint_as_float(v << 16); }
MOE_DEVI float bf16_hi(uint32_t v) { return __uint_as_float(v & 0xffff0000u); }

// round-to-nearest-even fp32 -> bf16 (same definition as the oracle's f2bf)
MOE_DEVI uint16_t f2bf(float f) {
    uint32_t u = __float_as_uint(f);
    if ((u & 0x7fffffffu) > 0x7f800000u) return 0x7fc0;
    u += 0x7fffu + ((u >> 16) & 1u);
    return static_cast<uint16_t>(u >> 16);
}

// 128-bit streaming load for weights: read exactly once per step, so bypass
// L1 allocation (the read-only, evict-first path).
MOE_DEVI uint4 ld_stream(const void* p) {
    uint4 r;
    asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
                 : "l"(p));
    return r;
}

MOE_DEVI uint16_t ld_nc_u16(const void* p) {
    uint16_t r;
    asm volatile("ld.global.nc.u16 %0, [%1];" : "=h"(r) : "l"(p));
    return r;
}

// acc += bf16 * bf16 with fp32 accumulate: one FHFMA.BF16 on sm_100a (PTX
// fma.rn.f32.bf16).  The product of two bf16 values is exact in fp32, so this
// is an fp32 FMA with bf16 operands -- no unpacking instructions.
MOE_DEVI float fma_lo(uint32_t w, uint32_t x, float acc) {
    uint16_t a, ah, b, bh;
    asm("mov.b32 {%0,%1}, %2;" : "=h"(a), "=h"(ah) : "r"(w));
    asm("mov.b32 {%0,%1}, %2;" : "=h"(b), "=h"(bh) : "r"(x));
    asm("fma.rn.f32.bf16 %0, %1, %2, %0;" : "+f"(acc) : "h"(a), "h"(b));
    return acc;
}
MOE_DEVI float fma_hi(uint32_t w, uint32_t x, float acc) {
    uint16_t a, al, b, bl;
    asm("mov.b32 {%0,%1}, %2;" : "=h"(al), "=h"(a) : "r"(w));
    asm("mov.b32 {%0,%1}, %2;" : "=h"(bl), "=h"(b) : "r"(x));
    asm("fma.rn.f32.bf16 %0, %1, %2, %0;" : "+f"(acc) : "h"(a), "h"(b));
    return acc;
}

// bf16x2 FMA, one rounding per half.
MOE_DEVI uint32_t hfma2_bf16(uint32_t a, uint32_t b, uint32_t c) {
    uint32_t d;
    asm("fma.rn.bf16x2 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(c));
    return d;
}

// (a & mask) | orv in one LOP3
MOE_DEVI uint32_t and_or(uint32_t a, uint32_t mask, uint32_t orv) {
    uint32_t d;
    asm("lop3.b32 %0, %1, %2, %3, 0xEA;" : "=r"(d) : "r"(a), "r"(mask), "r"(orv));
    return d;
}

// ---- int4-g128 word decode -------------------------------------------------
// A packed word holds elements j = 0..7 of 8 consecutive K positions, element
// j at bit 4*(j/2) + 16*(j%2), biased u = q + 8.  OR-ing a nibble into the
// low mantissa bits of bf16 128.0 (0x4300) gives the exact bf16 value 128 + u
// (bf16 has 7 mantissa bits, so every pair is first shifted down to bits
// 0-3 / 16-19).  Result: four bf16x2 pairs (128+u0, 128+u1) ... (128+u6,
// 128+u7) for 3 SHF + 4 LOP3.  The kernels accumulate sum((128+u) x) with
// FHFMA and remove the bias once per 32-element chunk:
//   sum(q x) = sum((128+u) x) - 136 * sum(x)
// with sum(x) precomputed per token and chunk, then apply the group scale:
// y += s * sum(q x), i.e. the exact dequant value q*s.
MOE_DEVI void decode_u8(uint32_t w, uint32_t& p01, uint32_t& p23, uint32_t& p45, uint32_t& p67) {
    p01 = and_or(w, 0x000F000Fu, 0x43004300u);
    p23 = and_or(w >> 4, 0x000F000Fu, 0x43004300u);
    p45 = and_or(w >> 8, 0x000F000Fu, 0x43004300u);
    p67 = and_or(w >> 12, 0x000F000Fu, 0x43004300u);
}
constexpr float kInt4Bias = 136.0f;  // 128 (magic) + 8 (storage bias)

// Programmatic dependent launch (PDL): every kernel of a layer is launched
// with programmatic stream serialization.  A kernel may read outputs of
// kernels two or more launches back before pdl_wait() (each kernel triggers
// its dependents only after its own pdl_wait(), so those are complete), and
// must call pdl_wait() before reading its immediate predecessor's output.
MOE_DEVI void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
MOE_DEVI void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

// fp16-operand range guard.  Both int4 paths multiply
// against fp16 copies of bf16 activations (x, h) and tcgen05 dequantises int4
// to fp16 q*s.  bf16 values above 65504 become inf in fp16; a 128-element
// activation group whose largest magnitude is below 2^-14 keeps few or no
// bits (the GEMV copies; single tiny elements in a normal group are
// negligible and not flagged); scales outside [2^-14, 8188] make q*s
// inexact or infinite.  The kernels that make
// those fp16 values set a bit in one process-wide word of mapped pinned host
// memory (zero cost unless it happens); the engine raises on it at its next
// sync (moe_numerics_status).  Each translation unit holds its own pointer
// (no -rdc), bound by its moek_numerics_bind_* function.
enum { MOE_NUM_F16_ACT = 1u, MOE_NUM_F16_SCALE = 2u };
static __device__ unsigned int* g_numerics = nullptr;
MOE_DEVI void numerics_flag(unsigned int bit) {
    unsigned int* p = g_numerics;
    if (p != nullptr) atomicOr(p, bit);
}
// a bf16 value whose fp16 copy is not finite (every bf16 > 65504 is >= 65536)
MOE_DEVI bool f16_overflow(float v) { return fabsf(v) > 65504.0f; }
// int4 scale (bf16 bits) whose fp16 q*s, |q| <= 8, is not exact: zero is
// fine, else 2^-14 <= |s| (fp16 normal) and 8|s| <= 65504 (|s| <= 8176 in bf16)
MOE_DEVI bool f16_scale_bad(uint16_t sb) {
    const uint32_t a = sb & 0x7fffu;
    return a != 0 && (a < 0x3880u || a > 0x45ffu);
}
#define MOE_NUMERICS_BINDER(name)                                                         \
    cudaError_t moek_numerics_bind_##name(unsigned int* p) {                              \
        return cudaMemcpyToSymbol(moek::g_numerics, &p, sizeof(p));                       \
    }

// One 16-byte chunk of the K-permuted activation copies of a 128-element
// group g (natural order in xg, any address space): chunk c*4+t holds, for
// kk in {2c, 2c+1}, hi in {0,1}, e in {0,1}, the element kk*16 + hi*8 + t*2 + e:
//   bf16 copy (perm_k):   word (kk%2)*2 + hi
//   fp16 copy (perm_k16): word hi*2 + kk%2      (fp16 exact for 2^-17 <= |x| <= 65504)
// Also returns this chunk's partial sums over k%16 < 8 (hi = 0) and >= 8
// (hi = 1) for the int4 bias term (summed in element order kk, e).
template <class T>
MOE_DEVI void permute_chunk(const T* xg, int chunk, uint4& cb, uint4& ch, float& s_lo, float& s_hi, float& amax) {
    const int c = chunk >> 2, t = chunk & 3;
    uint32_t wb[4], wh[4];
    s_lo = 0.0f;
    s_hi = 0.0f;
    amax = 0.0f;
#pragma unroll
    for (int kq = 0; kq < 2; ++kq) {
#pragma unroll
        for (int hi = 0; hi < 2; ++hi) {
            const int n = (2 * c + kq) * 16 + hi * 8 + t * 2;
            const uint16_t v0 = static_cast<uint16_t>(xg[n]), v1 = static_cast<uint16_t>(xg[n + 1]);
            const float f0 = bf2f(v0), f1 = bf2f(v1);
            wb[kq * 2 + hi] = static_cast<uint32_t>(v0) | (static_cast<uint32_t>(v1) << 16);
            wh[hi * 2 + kq] = static_cast<uint32_t>(__half_as_ushort(__float2half_rn(f0))) |
                              (static_cast<uint32_t>(__half_as_ushort(__float2half_rn(f1))) << 16);
            if (hi) s_hi += f0 + f1; else s_lo += f0 + f1;
            if (f16_overflow(f0) || f16_overflow(f1)) numerics_flag(MOE_NUM_F16_ACT);
            amax = fmaxf(amax, fmaxf(fabsf(f0), fabsf(f1)));
        }
    }
    cb = make_uint4(wb[0], wb[1], wb[2], wb[3]);
    ch = make_uint4(wh[0], wh[1], wh[2], wh[3]);
}

// The int4 bias term of an activation group, 1032*S_lo + 72*S_hi, rounded
// explicitly (no FMA contraction): every kernel that makes it -- route,
// permute_rows, finalize_h, the fused step -- must produce the same bits.
MOE_DEVI float int4_bias_term(float s_lo, float s_hi) {
    return __fadd_rn(__fmul_rn(1032.0f, s_lo), __fmul_rn(72.0f, s_hi));
}

// The 16 chunk maxima of a 128-element group (lanes xor 8..1 of a half
// warp; every lane of the warp must call): a nonzero group entirely below
// the fp16 normal range (2^-14) keeps few or no bits in its fp16 copy.
MOE_DEVI void numerics_group_check(float amax, bool leader) {
#pragma unroll
    for (int off = 8; off >= 1; off >>= 1) amax = fmaxf(amax, __shfl_xor_sync(0xffffffffu, amax, off));
    if (leader && amax > 0.0f && amax < 6.103515625e-05f) numerics_flag(MOE_NUM_F16_ACT);
}

// Debug layer trace (moe_debug_layer_trace): per kernel id, the earliest
// entry and post-PDL-wait globaltimer stamps (atomicMin) and the latest warp
// end (atomicMax).  One copy per translation unit (no -rdc); null = off.
static __device__ unsigned long long* g_layer_trace = nullptr;
// Kernels read the pointer once (ltr = g_layer_trace at entry) and pass it:
// a load per call would stall every traced point on an L2 round trip.
MOE_DEVI void ltrace(unsigned long long* tr, int id, int phase) {
    if (tr == nullptr || (threadIdx.x & 31) != 0) return;
    if (phase < 2 && threadIdx.x != 0) return;
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    if (phase < 2)
        atomicMin(tr + id * 3 + phase, t);
    else
        atomicMax(tr + id * 3 + 2, t);
}

MOE_DEVI float warp_sum(float v) {
#pragma unroll
    for (int off = 16; off >= 1; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
    return v;
}

MOE_DEVI float silu_f(float g) { return g / (1.0f + expf(-g)); }

#define MOE_CUDA_OK_PRELOAD(expr)                           \
    do {                                                    \
        cudaError_t err__ = (expr);                         \
        if (err__ != cudaSuccess) return err__;             \
    } while (0)

#define MOE_CUDA_OK(expr)                                   \
    do {                                                    \
        cudaError_t err__ = (expr);                         \
        if (err__ != cudaSuccess) return err__;             \
    } while (0)

// Host: launch with programmatic stream serialization (PDL edge to the
// previous kernel in the stream; captured as a programmatic graph edge).
template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t stream,
                              Args&&... args) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = stream;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
}

}  // namespace moek
