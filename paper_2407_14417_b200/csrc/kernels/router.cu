// router.cu -- K1 top-k softmax gate and K2 expert-major permutation.
//
// Replaces the reference's uniform router stand-in (gating.cpp:43-51) with
// the real MixtralTopKRouter semantics (HF modeling_mixtral.py:109-116).
// Bit-exactness contract:
//   logit(t,e): lane l of a warp owns elements k = c*256 + l*8 + j and
//   accumulates fmaf(x[k], w[k], acc) with c outer, j inner; the 32 lane sums
//   are folded by an xor butterfly (16, 8, 4, 2, 1).  oracle/moe_oracle.cpp
//   orc_gate_topk restates exactly this order, so indices AND logits match
//   bit for bit.  Top-k selects on logits (ties -> lower index); weights are
//   softmax over the selected logits (tolerance-checked: expf differs by ulps
//   between CUDA and libm).
#include "common.cuh"
#include "launch.h"

namespace moek {

constexpr int kRouteThreads = 256;

struct RouteArgs {
    const uint16_t* x;
    const uint16_t* wg;
    int T, d, E, k;
    int32_t* idx;
    float* w;
    float* logits;
    // fused K2 (optional: counts == nullptr -> no permutation)
    int32_t* counts;
    int32_t* offsets;
    int32_t* perm;
    int32_t* inv_perm;
    unsigned int* ticket;  // zero-initialised; reset by the last CTA
};

// One logit in the pinned order.  x_s is the token row staged in smem.
MOE_DEVI float router_dot(const uint16_t* __restrict__ x_s, const uint16_t* __restrict__ we, int d,
                          int lane) {
    float acc = 0.0f;
    for (int c = 0; c * 256 < d; ++c) {
        const int k0 = c * 256 + lane * 8;
        if (k0 + 8 <= d) {
            const uint4 wv = *reinterpret_cast<const uint4*>(we + k0);
            const uint4 xv = *reinterpret_cast<const uint4*>(x_s + k0);
            const uint32_t ww[4] = {wv.x, wv.y, wv.z, wv.w};
            const uint32_t xx[4] = {xv.x, xv.y, xv.z, xv.w};
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                acc = __fmaf_rn(bf16_lo(xx[q]), bf16_lo(ww[q]), acc);
                acc = __fmaf_rn(bf16_hi(xx[q]), bf16_hi(ww[q]), acc);
            }
        } else {
            for (int j = 0; j < 8 && k0 + j < d; ++j)
                acc = __fmaf_rn(bf2f(x_s[k0 + j]), bf2f(we[k0 + j]), acc);
        }
    }
#pragma unroll
    for (int off = 16; off >= 1; off >>= 1) acc = __fadd_rn(acc, __shfl_xor_sync(0xffffffffu, acc, off));
    return acc;
}

// Stable counting sort of n = T*k items by expert, one CTA, no atomics:
// thread i owns the contiguous item range [i*per, (i+1)*per), and for every
// expert a block-wide exclusive scan of the per-thread counts gives each
// thread its write position, so ties keep ascending (t, j) order.
MOE_DEVI void block_permute(const int32_t* idx, int n, int E, int32_t* counts,
                            int32_t* offsets, int32_t* perm, int32_t* inv_perm, int* s_warp) {
    const int tid = threadIdx.x, nth = blockDim.x;
    const int lane = tid & 31, wid = tid >> 5, nwarps = nth >> 5;
    const int per = (n + nth - 1) / nth;
    const int i0 = min(n, tid * per), i1 = min(n, i0 + per);
    int base = 0;
    if (tid == 0) offsets[0] = 0;
    for (int e = 0; e < E; ++e) {
        int c = 0;
        for (int i = i0; i < i1; ++i) c += idx[i] == e;
        // inclusive warp scan
        int incl = c;
#pragma unroll
        for (int off = 1; off < 32; off <<= 1) {
            const int v = __shfl_up_sync(0xffffffffu, incl, off);
            if (lane >= off) incl += v;
        }
        if (lane == 31) s_warp[wid] = incl;
        __syncthreads();
        int warp_base = 0, total = 0;
        for (int w = 0; w < nwarps; ++w) {
            const int v = s_warp[w];
            if (w < wid) warp_base += v;
            total += v;
        }
        int pos = base + warp_base + incl - c;
        for (int i = i0; i < i1; ++i)
            if (idx[i] == e) {
                perm[pos] = i;
                inv_perm[i] = pos;
                ++pos;
            }
        if (tid == 0) {
            counts[e] = total;
            offsets[e + 1] = base + total;
        }
        base += total;
        __syncthreads();
    }
}

__global__ void __launch_bounds__(kRouteThreads) route_kernel(RouteArgs a) {
    extern __shared__ __align__(16) uint8_t smem[];
    uint16_t* x_s = reinterpret_cast<uint16_t*>(smem);
    float* lg_s = reinterpret_cast<float*>(smem + ((a.d * 2 + 15) / 16) * 16);
    __shared__ int s_warp[kRouteThreads / 32];
    __shared__ bool s_last;

    const int t = blockIdx.x;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    pdl_wait();     // x is the previous layer's output
    pdl_trigger();
    const uint16_t* xt = a.x + static_cast<size_t>(t) * a.d;
    for (int i = threadIdx.x * 8; i < a.d; i += blockDim.x * 8) {
        if (i + 8 <= a.d)
            *reinterpret_cast<uint4*>(x_s + i) = *reinterpret_cast<const uint4*>(xt + i);
        else
            for (int j = i; j < a.d; ++j) x_s[j] = xt[j];
    }
    __syncthreads();
    for (int e = wid; e < a.E; e += blockDim.x / 32) {
        const float v = router_dot(x_s, a.wg + static_cast<size_t>(e) * a.d, a.d, lane);
        if (lane == 0) lg_s[e] = v;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        if (a.logits)
            for (int e = 0; e < a.E; ++e) a.logits[static_cast<size_t>(t) * a.E + e] = lg_s[e];
        uint64_t taken = 0;
        float sel[MOE_MAX_TOPK];
        for (int j = 0; j < a.k; ++j) {
            int best = -1;
            for (int e = 0; e < a.E; ++e)
                if (!((taken >> e) & 1ull) && (best < 0 || lg_s[e] > lg_s[best])) best = e;
            taken |= 1ull << best;
            a.idx[static_cast<size_t>(t) * a.k + j] = best;
            sel[j] = lg_s[best];
        }
        float ex[MOE_MAX_TOPK], sum = 0.0f;
        for (int j = 0; j < a.k; ++j) {
            ex[j] = expf(sel[j] - sel[0]);
            sum += ex[j];
        }
        for (int j = 0; j < a.k; ++j) a.w[static_cast<size_t>(t) * a.k + j] = ex[j] / sum;
    }
    if (a.counts == nullptr) return;
    // Fused K2: the last CTA to finish permutes all tokens.
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) s_last = atomicAdd(a.ticket, 1u) == gridDim.x - 1;
    __syncthreads();
    if (!s_last) return;
    __threadfence();
    block_permute(a.idx, a.T * a.k, a.E, a.counts, a.offsets, a.perm, a.inv_perm, s_warp);
    if (threadIdx.x == 0) *a.ticket = 0;
}

__global__ void __launch_bounds__(512) permute_kernel(const int32_t* idx, int n, int E,
                                                      int32_t* counts, int32_t* offsets,
                                                      int32_t* perm, int32_t* inv_perm) {
    __shared__ int s_warp[16];
    block_permute(idx, n, E, counts, offsets, perm, inv_perm, s_warp);
}

}  // namespace moek

// ---------------------------------------------------------------------------
// launchers (called by capi.cu / engine.cu)
cudaError_t moek_route(const void* x, const void* wg, int T, int d, int E, int k, int32_t* idx,
                       float* w, float* logits, int32_t* counts, int32_t* offsets, int32_t* perm,
                       int32_t* inv_perm, unsigned int* ticket, cudaStream_t stream) {
    moek::RouteArgs a{static_cast<const uint16_t*>(x), static_cast<const uint16_t*>(wg), T, d, E, k,
                      idx, w, logits, counts, offsets, perm, inv_perm, ticket};
    const size_t smem = ((static_cast<size_t>(d) * 2 + 15) / 16) * 16 + static_cast<size_t>(E) * 4;
    if (smem > 48 * 1024) {
        cudaError_t e = cudaFuncSetAttribute(moek::route_kernel,
                                             cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             static_cast<int>(smem));
        if (e != cudaSuccess) return e;
    }
    return moek::launch_pdl(moek::route_kernel, dim3(T), dim3(moek::kRouteThreads), smem, stream, a);
}

cudaError_t moek_permute(const int32_t* idx, int T, int E, int k, int32_t* counts, int32_t* offsets,
                         int32_t* perm, int32_t* inv_perm, cudaStream_t stream) {
    moek::permute_kernel<<<1, 512, 0, stream>>>(idx, T * k, E, counts, offsets, perm, inv_perm);
    return cudaGetLastError();
}
