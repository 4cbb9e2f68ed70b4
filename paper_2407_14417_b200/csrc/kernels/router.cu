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
#include "route_common.cuh"

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
    // fused K-permuted activation copies for the expert GEMV (optional)
    uint16_t* xperm;
    uint16_t* xperm16;
    float* xsum;
    int xstride;
    float norm_eps;        // > 0: unit-weight RMSNorm of x before routing / experts (oracle orc_rmsnorm)
    uint16_t* xnat;        // optional: the (normalised) token rows in natural order [T][d]
};

// K-permuted position (must match gemv.cu perm_k / perm_k16)
MOE_DEVI int rperm_k(int n) {
    const int kin = n & 127, kk = kin >> 4;
    return (n & ~127) + ((kk >> 1) * 4 + ((kin & 7) >> 1)) * 8 + ((kk & 1) * 2 + ((kin >> 3) & 1)) * 2 + (kin & 1);
}
MOE_DEVI int rperm_k16(int n) {
    const int kin = n & 127, kk = kin >> 4;
    return (n & ~127) + ((kk >> 1) * 4 + ((kin & 7) >> 1)) * 8 + (((kin >> 3) & 1) * 2 + (kk & 1)) * 2 + (kin & 1);
}

// Stable counting sort of n = T*k items by expert, one CTA, no global
// atomics: per 256-item chunk every warp ballots each expert (rank inside
// the warp = popc of the lower lanes), a per-chunk warp prefix in shared
// memory orders the warps, and a running per-expert base orders the chunks
// -- so ties keep ascending (t, j) order.  Two passes: counts, positions.
MOE_DEVI void block_permute(const int32_t* idx, int n, int E, int32_t* counts, int32_t* offsets, int32_t* perm,
                            int32_t* inv_perm) {
    __shared__ int s_cnt[kRouteThreads / 32][MOE_MAX_EXPERTS];
    __shared__ int s_off[MOE_MAX_EXPERTS + 1];
    __shared__ int s_run[MOE_MAX_EXPERTS];
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5, nw = blockDim.x >> 5;
    const unsigned lt = (1u << lane) - 1u;
    if (tid < E) {
        s_off[tid] = 0;
        s_run[tid] = 0;
    }
    __syncthreads();
    // pass 1: per-expert totals
    for (int c0 = 0; c0 < n; c0 += blockDim.x) {
        const int i = c0 + tid;
        const int ei = i < n ? idx[i] : -1;
        for (int e = 0; e < E; ++e) {
            const unsigned m = __ballot_sync(0xffffffffu, ei == e);
            if (lane == 0 && m) atomicAdd(&s_off[e], __popc(m));
        }
    }
    __syncthreads();
    if (tid == 0) {
        int acc = 0;
        for (int e = 0; e < E; ++e) {
            const int c = s_off[e];
            counts[e] = c;
            s_off[e] = acc;
            offsets[e] = acc;
            acc += c;
        }
        s_off[E] = acc;
        offsets[E] = acc;
    }
    __syncthreads();
    // pass 2: stable positions
    for (int c0 = 0; c0 < n; c0 += blockDim.x) {
        const int i = c0 + tid;
        const int ei = i < n ? idx[i] : -1;
        int rank = 0;
        for (int e = 0; e < E; ++e) {
            const unsigned m = __ballot_sync(0xffffffffu, ei == e);
            if (lane == 0) s_cnt[wid][e] = __popc(m);
            if (ei == e) rank = __popc(m & lt);
        }
        __syncthreads();
        if (i < n) {
            int pos = s_off[ei] + s_run[ei] + rank;
            for (int w = 0; w < wid; ++w) pos += s_cnt[w][ei];
            perm[pos] = i;
            inv_perm[i] = pos;
        }
        __syncthreads();
        if (tid < E)
            for (int w = 0; w < nw; ++w) s_run[tid] += s_cnt[w][tid];
        __syncthreads();
    }
}

__global__ void __launch_bounds__(kRouteThreads) route_kernel(RouteArgs a) {
    extern __shared__ __align__(16) uint8_t smem[];
    uint16_t* x_s = reinterpret_cast<uint16_t*>(smem);
    float* lg_s = reinterpret_cast<float*>(smem + ((a.d * 2 + 15) / 16) * 16);
    __shared__ int s_idx[MOE_MAX_TOPK];
    __shared__ bool s_last;

    const int t = blockIdx.x;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    unsigned long long* const ltr = g_layer_trace;
    ltrace(ltr, 0, 0);
    // The router weights do not depend on the previous layer: this warp's
    // first expert row goes into registers before the PDL wait.
    uint4 wpre[kPreChunks];
    if (wid < a.E) preload_w(wpre, a.wg + static_cast<size_t>(wid) * a.d, a.d, lane);
    pdl_wait();     // x is the previous layer's output
    pdl_trigger();
    ltrace(ltr, 0, 1);
    const uint16_t* xt = a.x + static_cast<size_t>(t) * a.d;
    for (int i = threadIdx.x * 8; i < a.d; i += blockDim.x * 8) {
        if (i + 8 <= a.d)
            *reinterpret_cast<uint4*>(x_s + i) = *reinterpret_cast<const uint4*>(xt + i);
        else
            for (int j = i; j < a.d; ++j) x_s[j] = xt[j];
    }
    __syncthreads();
    if (a.norm_eps > 0.0f) {
        // pinned order: thread i's fmaf chain over x[c*256+i]^2, then the
        // pairwise tree over 256 partials (orc_rmsnorm)
        float acc = 0.0f;
        for (int c = 0; c * 256 + static_cast<int>(threadIdx.x) < a.d; ++c) {
            const float v = bf2f(x_s[c * 256 + threadIdx.x]);
            acc = __fmaf_rn(v, v, acc);
        }
        lg_s[MOE_MAX_EXPERTS + threadIdx.x] = acc;
        __syncthreads();
        for (int s2 = 128; s2 >= 32; s2 >>= 1) {
            if (static_cast<int>(threadIdx.x) < s2)
                lg_s[MOE_MAX_EXPERTS + threadIdx.x] =
                    __fadd_rn(lg_s[MOE_MAX_EXPERTS + threadIdx.x], lg_s[MOE_MAX_EXPERTS + threadIdx.x + s2]);
            __syncthreads();
        }
        if (wid == 0) {  // the same pairwise steps 16..1 as warp shuffles
            float v = lg_s[MOE_MAX_EXPERTS + lane];
#pragma unroll
            for (int s2 = 16; s2 >= 1; s2 >>= 1) v = __fadd_rn(v, __shfl_down_sync(0xffffffffu, v, s2));
            if (lane == 0) lg_s[MOE_MAX_EXPERTS] = v;
        }
        __syncthreads();
        const float rstd = __fdiv_rn(1.0f, __fsqrt_rn(__fadd_rn(__fdiv_rn(lg_s[MOE_MAX_EXPERTS],
                                                                            static_cast<float>(a.d)), a.norm_eps)));
        // x * rstd, 8 elements (one 16-byte chunk) per thread and step
        for (int i = threadIdx.x * 8; i < a.d; i += blockDim.x * 8) {
            if (i + 8 <= a.d) {
                uint4 v = *reinterpret_cast<const uint4*>(x_s + i);
                uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
                for (int q = 0; q < 4; ++q)
                    w[q] = static_cast<uint32_t>(f2bf(__fmul_rn(bf16_lo(w[q]), rstd))) |
                           (static_cast<uint32_t>(f2bf(__fmul_rn(bf16_hi(w[q]), rstd))) << 16);
                *reinterpret_cast<uint4*>(x_s + i) = make_uint4(w[0], w[1], w[2], w[3]);
            } else {
                for (int j = i; j < a.d; ++j) x_s[j] = f2bf(__fmul_rn(bf2f(x_s[j]), rstd));
            }
        }
        __syncthreads();
    }
    ltrace(ltr, 1, 0);
    if (a.xnat != nullptr)
        for (int i = threadIdx.x * 8; i + 8 <= a.d; i += blockDim.x * 8)
            *reinterpret_cast<uint4*>(a.xnat + static_cast<size_t>(t) * a.d + i) = *reinterpret_cast<const uint4*>(x_s + i);
    for (int e = wid; e < a.E; e += blockDim.x / 32) {
        if (e != wid) preload_w(wpre, a.wg + static_cast<size_t>(e) * a.d, a.d, lane);
        const float v = router_dot(x_s, wpre, a.wg + static_cast<size_t>(e) * a.d, a.d, lane);
        if (lane == 0) lg_s[e] = v;
    }
    __syncthreads();
    ltrace(ltr, 1, 1);
    if (a.logits && threadIdx.x < a.E) a.logits[static_cast<size_t>(t) * a.E + threadIdx.x] = lg_s[threadIdx.x];
    if (wid == 0) warp_topk(lg_s, a.E, a.k, lane, a.idx + static_cast<size_t>(t) * a.k, a.w + static_cast<size_t>(t) * a.k, s_idx);
    // K-permuted bf16 / fp16 copies of this token row + int4 bias terms
    // (same definition as gemv.cu permute_rows_kernel): a 128-K group is 16
    // chunks of 16 bytes, so each warp half assembles one group per pass
    if (a.xperm != nullptr) {
        const int G = a.d / 128;
        // warps 1.. (warp 0 is on the top-k / permutation critical path)
        const int nw = blockDim.x / 32 - 1;
        for (int g0 = (wid - 1) * 2; wid > 0 && g0 < G; g0 += nw * 2) {
            const int g = g0 + (lane >> 4), c = lane & 15;
            uint4 cb = make_uint4(0, 0, 0, 0), ch = cb;
            float s_lo = 0.0f, s_hi = 0.0f, amax = 0.0f;
            if (g < G) permute_chunk(x_s + g * 128, c, cb, ch, s_lo, s_hi, amax);
            numerics_group_check(amax, c == 0);
#pragma unroll
            for (int off = 8; off >= 1; off >>= 1) {
                s_lo += __shfl_xor_sync(0xffffffffu, s_lo, off);
                s_hi += __shfl_xor_sync(0xffffffffu, s_hi, off);
            }
            if (g < G) {
                reinterpret_cast<uint4*>(a.xperm + static_cast<size_t>(t) * a.d + g * 128)[c] = cb;
                reinterpret_cast<uint4*>(a.xperm16 + static_cast<size_t>(t) * a.d + g * 128)[c] = ch;
                if (c == 0) a.xsum[static_cast<size_t>(t) * a.xstride + g] = int4_bias_term(s_lo, s_hi);
            }
        }
    }
    if (a.counts == nullptr) {
        ltrace(ltr, 0, 2);
        return;
    }
    if (gridDim.x == 1) {
        // single token: warp 0 permutes straight from its top-k (shared memory)
        if (wid == 0) {
            __syncwarp();
            ltrace(ltr, 1, 2);
            warp_permute(s_idx, a.k, a.E, a.counts, a.offsets, a.perm, a.inv_perm, lane);
        }
        ltrace(ltr, 0, 2);
        return;
    }
    // Fused K2: the last CTA to finish permutes all tokens.
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) s_last = atomicAdd(a.ticket, 1u) == gridDim.x - 1;
    __syncthreads();
    if (!s_last) {
        ltrace(ltr, 0, 2);
        return;
    }
    __threadfence();
    block_permute(a.idx, a.T * a.k, a.E, a.counts, a.offsets, a.perm, a.inv_perm);
    if (threadIdx.x == 0) *a.ticket = 0;
    ltrace(ltr, 0, 2);
}

__global__ void __launch_bounds__(kRouteThreads) permute_kernel(const int32_t* idx, int n, int E,
                                                                int32_t* counts, int32_t* offsets,
                                                                int32_t* perm, int32_t* inv_perm) {
    block_permute(idx, n, E, counts, offsets, perm, inv_perm);
}

}  // namespace moek

// ---------------------------------------------------------------------------
// launchers (called by capi.cu / engine.cu)
cudaError_t moek_route(const void* x, const void* wg, int T, int d, int E, int k, int32_t* idx,
                       float* w, float* logits, int32_t* counts, int32_t* offsets, int32_t* perm,
                       int32_t* inv_perm, unsigned int* ticket, cudaStream_t stream, void* xperm, void* xperm16,
                       float* xsum, int xstride, float norm_eps, void* xnat) {
    moek::RouteArgs a{static_cast<const uint16_t*>(x), static_cast<const uint16_t*>(wg), T, d, E, k,
                      idx, w, logits, counts, offsets, perm, inv_perm, ticket,
                      static_cast<uint16_t*>(xperm), static_cast<uint16_t*>(xperm16), xsum, xstride, norm_eps,
                      static_cast<uint16_t*>(xnat)};
    // x row + logits [MOE_MAX_EXPERTS] + RMSNorm partials [kRouteThreads]
    const size_t smem = ((static_cast<size_t>(d) * 2 + 15) / 16) * 16 + (MOE_MAX_EXPERTS + moek::kRouteThreads) * 4;
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
    moek::permute_kernel<<<1, moek::kRouteThreads, 0, stream>>>(idx, T * k, E, counts, offsets, perm, inv_perm);
    return cudaGetLastError();
}

cudaError_t moek_debug_layer_trace_router(void* host_ptr, cudaStream_t stream) {
    return cudaMemcpyToSymbolAsync(moek::g_layer_trace, host_ptr, sizeof(void*), 0, cudaMemcpyHostToDevice, stream);
}

MOE_NUMERICS_BINDER(router)

// Loads this unit's kernels now (cudaFuncGetAttributes).  Under lazy module
// loading (CUDA 12 default) a kernel's first launch may wait for the device
// to idle; the expert-parallel step has kernels that spin on a peer's flags,
// so every kernel it can launch must be resident before the first step.
cudaError_t moek_preload_router() {
    cudaFuncAttributes fa;
    MOE_CUDA_OK_PRELOAD(cudaFuncGetAttributes(&fa, moek::route_kernel));
    MOE_CUDA_OK_PRELOAD(cudaFuncGetAttributes(&fa, moek::permute_kernel));
    return cudaSuccess;
}
