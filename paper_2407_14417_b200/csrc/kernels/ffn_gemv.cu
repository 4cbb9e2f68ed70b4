// ffn_gemv.cu -- K3 (int4-g128) and K4 (bf16) SwiGLU expert FFN, decode-batch
// GEMV path.  Replaces the constant compute latency of the reference's
// MoE-layer stand-in (simulator.cpp:31-32, :107) with the real expert math
// of HF MixtralExperts (modeling_mixtral.py:90-95): y = Wd (silu(Wg x) * Wu x).
//
// Layout per expert:
//   bf16: w_gate_up [2f, d] row-major (rows [0,f) gate, [f,2f) up), w_down [d, f]
//   int4: q words [rows, K/8] (8 elements per uint32, element j at bit
//         4*(j/2)+16*(j%2), biased by 8) + bf16 scales [rows, K/128]
//
// Work decomposition: the (expert, token-tile) segments of the permutation
// are enumerated on the device from `offsets`, every segment contributes f
// (gate/up row pairs) or d (down rows) warp items, and the concatenated item
// range is split evenly over a persistent grid (148 x occupancy CTAs).  Each
// warp streams one row (pair) with 128-bit L1-bypassing loads, lanes striding
// 16-byte chunks so every warp load is one fully used 512-byte transaction.
// Activations (x tile, or h tile for the down projection) are staged once per
// segment in shared memory.
//
// Arithmetic: bf16 weights -> FHFMA.BF16 (fp32 += bf16*bf16).  int4 weights
// -> LOP3 magic-number decode + one bf16x2 FMA per pair gives q exactly, the
// 32-element chunk dot sum(q*x) accumulates in fp32 with FHFMA, then one FFMA
// applies the group scale: sum_chunk(q*s*x) with the exact dequant value q*s.
#include "common.cuh"
#include "launch.h"

namespace moek {

constexpr int kFfnThreads = 256;
constexpr int kFfnWarps = kFfnThreads / 32;
constexpr int kChunksPerStep = 4;   // 128-bit loads in flight per lane per row

struct FfnArgs {
    const uint16_t* x;        // [T, d]
    const int32_t* perm;      // [T*k]
    const int32_t* offsets;   // [E+1]
    int T, k, E, d, f;
    uint64_t active_mask;     // experts computed by this launch
    uint16_t* h;              // [T*k, f]
    float* y;                 // [T*k, d]
    moe_expert_weights ex[MOE_MAX_EXPERTS];
};

// seg[e] = index of the first (e, tile) segment of expert e; seg[E] = total.
template <int MT>
MOE_DEVI int build_segments(const FfnArgs& a, int* seg) {
    if (threadIdx.x == 0) {
        int acc = 0;
        for (int e = 0; e < a.E; ++e) {
            seg[e] = acc;
            const int m = ((a.active_mask >> e) & 1ull) ? a.offsets[e + 1] - a.offsets[e] : 0;
            acc += (m + MT - 1) / MT;
        }
        seg[a.E] = acc;
    }
    __syncthreads();
    return seg[a.E];
}

MOE_DEVI int expert_of_segment(const int* seg, int E, int s) {
    int e = 0;
    while (e + 1 < E && seg[e + 1] <= s) ++e;
    return e;
}

// ---- one gate/up row pair --------------------------------------------------
template <int MT>
MOE_DEVI void rowpair_int4(const moe_expert_weights& W, int n, int d, int f, const uint16_t* xs,
                           const float* xsum, int lane, float (&ag)[MT], float (&au)[MT]) {
    const int wpr = d / 8;                     // uint32 words per row
    const uint4* qg = reinterpret_cast<const uint4*>(static_cast<const uint32_t*>(W.w_gate_up) + static_cast<size_t>(n) * wpr);
    const uint4* qu = reinterpret_cast<const uint4*>(static_cast<const uint32_t*>(W.w_gate_up) + static_cast<size_t>(n + f) * wpr);
    const uint16_t* sg = static_cast<const uint16_t*>(W.s_gate_up) + static_cast<size_t>(n) * (d / 128);
    const uint16_t* su = static_cast<const uint16_t*>(W.s_gate_up) + static_cast<size_t>(n + f) * (d / 128);
    const int nch = d / 32;                    // 16-byte chunks (32 elements)
#pragma unroll
    for (int m = 0; m < MT; ++m) ag[m] = au[m] = 0.0f;
    for (int c0 = lane; c0 < nch; c0 += 32 * kChunksPerStep) {
        uint4 vg[kChunksPerStep], vu[kChunksPerStep];
        uint16_t sgv[kChunksPerStep], suv[kChunksPerStep];
#pragma unroll
        for (int i = 0; i < kChunksPerStep; ++i) {
            const int c = c0 + 32 * i;
            if (c < nch) {
                vg[i] = ld_stream(qg + c);
                vu[i] = ld_stream(qu + c);
                sgv[i] = ld_nc_u16(sg + c / 4);
                suv[i] = ld_nc_u16(su + c / 4);
            }
        }
#pragma unroll
        for (int i = 0; i < kChunksPerStep; ++i) {
            const int c = c0 + 32 * i;
            if (c >= nch) break;
            float cg[MT], cu[MT];
#pragma unroll
            for (int m = 0; m < MT; ++m) cg[m] = cu[m] = 0.0f;
            const uint32_t gw[4] = {vg[i].x, vg[i].y, vg[i].z, vg[i].w};
            const uint32_t uw[4] = {vu[i].x, vu[i].y, vu[i].z, vu[i].w};
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                uint32_t g0, g1, g2, g3, u0, u1, u2, u3;
                decode_u8(gw[q], g0, g1, g2, g3);
                decode_u8(uw[q], u0, u1, u2, u3);
#pragma unroll
                for (int m = 0; m < MT; ++m) {
                    const uint4 xv = *reinterpret_cast<const uint4*>(xs + static_cast<size_t>(m) * d + c * 32 + q * 8);
                    cg[m] = fma_hi(g0, xv.x, fma_lo(g0, xv.x, cg[m]));
                    cg[m] = fma_hi(g1, xv.y, fma_lo(g1, xv.y, cg[m]));
                    cg[m] = fma_hi(g2, xv.z, fma_lo(g2, xv.z, cg[m]));
                    cg[m] = fma_hi(g3, xv.w, fma_lo(g3, xv.w, cg[m]));
                    cu[m] = fma_hi(u0, xv.x, fma_lo(u0, xv.x, cu[m]));
                    cu[m] = fma_hi(u1, xv.y, fma_lo(u1, xv.y, cu[m]));
                    cu[m] = fma_hi(u2, xv.z, fma_lo(u2, xv.z, cu[m]));
                    cu[m] = fma_hi(u3, xv.w, fma_lo(u3, xv.w, cu[m]));
                }
            }
            const float sgf = bf2f(sgv[i]), suf = bf2f(suv[i]);
#pragma unroll
            for (int m = 0; m < MT; ++m) {
                const float xc = xsum[m * nch + c];
                ag[m] = __fmaf_rn(sgf, __fmaf_rn(-kInt4Bias, xc, cg[m]), ag[m]);
                au[m] = __fmaf_rn(suf, __fmaf_rn(-kInt4Bias, xc, cu[m]), au[m]);
            }
        }
    }
}

template <int MT>
MOE_DEVI void rowpair_bf16(const moe_expert_weights& W, int n, int d, int f, const uint16_t* xs,
                           int lane, float (&ag)[MT], float (&au)[MT]) {
    const uint4* wg = reinterpret_cast<const uint4*>(static_cast<const uint16_t*>(W.w_gate_up) + static_cast<size_t>(n) * d);
    const uint4* wu = reinterpret_cast<const uint4*>(static_cast<const uint16_t*>(W.w_gate_up) + static_cast<size_t>(n + f) * d);
    const int nch = d / 8;                     // 16-byte chunks (8 elements)
#pragma unroll
    for (int m = 0; m < MT; ++m) ag[m] = au[m] = 0.0f;
    for (int c0 = lane; c0 < nch; c0 += 32 * kChunksPerStep) {
        uint4 vg[kChunksPerStep], vu[kChunksPerStep];
#pragma unroll
        for (int i = 0; i < kChunksPerStep; ++i) {
            const int c = c0 + 32 * i;
            if (c < nch) {
                vg[i] = ld_stream(wg + c);
                vu[i] = ld_stream(wu + c);
            }
        }
#pragma unroll
        for (int i = 0; i < kChunksPerStep; ++i) {
            const int c = c0 + 32 * i;
            if (c >= nch) break;
#pragma unroll
            for (int m = 0; m < MT; ++m) {
                const uint4 xv = *reinterpret_cast<const uint4*>(xs + static_cast<size_t>(m) * d + c * 8);
                float g = ag[m], u = au[m];
                g = fma_hi(vg[i].x, xv.x, fma_lo(vg[i].x, xv.x, g));
                g = fma_hi(vg[i].y, xv.y, fma_lo(vg[i].y, xv.y, g));
                g = fma_hi(vg[i].z, xv.z, fma_lo(vg[i].z, xv.z, g));
                g = fma_hi(vg[i].w, xv.w, fma_lo(vg[i].w, xv.w, g));
                u = fma_hi(vu[i].x, xv.x, fma_lo(vu[i].x, xv.x, u));
                u = fma_hi(vu[i].y, xv.y, fma_lo(vu[i].y, xv.y, u));
                u = fma_hi(vu[i].z, xv.z, fma_lo(vu[i].z, xv.z, u));
                u = fma_hi(vu[i].w, xv.w, fma_lo(vu[i].w, xv.w, u));
                ag[m] = g;
                au[m] = u;
            }
        }
    }
}

// ---- one down-projection row ------------------------------------------------
template <int MT>
MOE_DEVI void row_down_int4(const moe_expert_weights& W, int j, int f, const uint16_t* hs,
                            const float* hsum, int lane, float (&acc)[MT]) {
    const uint4* q = reinterpret_cast<const uint4*>(static_cast<const uint32_t*>(W.w_down) + static_cast<size_t>(j) * (f / 8));
    const uint16_t* s = static_cast<const uint16_t*>(W.s_down) + static_cast<size_t>(j) * (f / 128);
    const int nch = f / 32;
#pragma unroll
    for (int m = 0; m < MT; ++m) acc[m] = 0.0f;
    for (int c0 = lane; c0 < nch; c0 += 32 * kChunksPerStep) {
        uint4 v[kChunksPerStep];
        uint16_t sv[kChunksPerStep];
#pragma unroll
        for (int i = 0; i < kChunksPerStep; ++i) {
            const int c = c0 + 32 * i;
            if (c < nch) {
                v[i] = ld_stream(q + c);
                sv[i] = ld_nc_u16(s + c / 4);
            }
        }
#pragma unroll
        for (int i = 0; i < kChunksPerStep; ++i) {
            const int c = c0 + 32 * i;
            if (c >= nch) break;
            float cc[MT];
#pragma unroll
            for (int m = 0; m < MT; ++m) cc[m] = 0.0f;
            const uint32_t ww[4] = {v[i].x, v[i].y, v[i].z, v[i].w};
#pragma unroll
            for (int qq = 0; qq < 4; ++qq) {
                uint32_t p0, p1, p2, p3;
                decode_u8(ww[qq], p0, p1, p2, p3);
#pragma unroll
                for (int m = 0; m < MT; ++m) {
                    const uint4 hv = *reinterpret_cast<const uint4*>(hs + static_cast<size_t>(m) * f + c * 32 + qq * 8);
                    cc[m] = fma_hi(p0, hv.x, fma_lo(p0, hv.x, cc[m]));
                    cc[m] = fma_hi(p1, hv.y, fma_lo(p1, hv.y, cc[m]));
                    cc[m] = fma_hi(p2, hv.z, fma_lo(p2, hv.z, cc[m]));
                    cc[m] = fma_hi(p3, hv.w, fma_lo(p3, hv.w, cc[m]));
                }
            }
            const float sf = bf2f(sv[i]);
#pragma unroll
            for (int m = 0; m < MT; ++m)
                acc[m] = __fmaf_rn(sf, __fmaf_rn(-kInt4Bias, hsum[m * nch + c], cc[m]), acc[m]);
        }
    }
}

template <int MT>
MOE_DEVI void row_down_bf16(const moe_expert_weights& W, int j, int f, const uint16_t* hs, int lane,
                            float (&acc)[MT]) {
    const uint4* w = reinterpret_cast<const uint4*>(static_cast<const uint16_t*>(W.w_down) + static_cast<size_t>(j) * f);
    const int nch = f / 8;
#pragma unroll
    for (int m = 0; m < MT; ++m) acc[m] = 0.0f;
    for (int c0 = lane; c0 < nch; c0 += 32 * kChunksPerStep * 2) {
        uint4 v[kChunksPerStep * 2];
#pragma unroll
        for (int i = 0; i < kChunksPerStep * 2; ++i) {
            const int c = c0 + 32 * i;
            if (c < nch) v[i] = ld_stream(w + c);
        }
#pragma unroll
        for (int i = 0; i < kChunksPerStep * 2; ++i) {
            const int c = c0 + 32 * i;
            if (c >= nch) break;
#pragma unroll
            for (int m = 0; m < MT; ++m) {
                const uint4 hv = *reinterpret_cast<const uint4*>(hs + static_cast<size_t>(m) * f + c * 8);
                float a = acc[m];
                a = fma_hi(v[i].x, hv.x, fma_lo(v[i].x, hv.x, a));
                a = fma_hi(v[i].y, hv.y, fma_lo(v[i].y, hv.y, a));
                a = fma_hi(v[i].z, hv.z, fma_lo(v[i].z, hv.z, a));
                a = fma_hi(v[i].w, hv.w, fma_lo(v[i].w, hv.w, a));
                acc[m] = a;
            }
        }
    }
}

// Per-token, per-32-element chunk sums of a staged activation tile (the
// int4 bias correction, see decode_u8).  Fixed summation order.
MOE_DEVI void chunk_sums(const uint16_t* tile, float* sums, int rows, int K) {
    const int nch = K / 32;
    for (int i = threadIdx.x; i < rows * nch; i += blockDim.x) {
        const uint4* p = reinterpret_cast<const uint4*>(tile + static_cast<size_t>(i) * 32);
        float acc = 0.0f;
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const uint4 v = p[q];
            acc += bf16_lo(v.x) + bf16_hi(v.x);
            acc += bf16_lo(v.y) + bf16_hi(v.y);
            acc += bf16_lo(v.z) + bf16_hi(v.z);
            acc += bf16_lo(v.w) + bf16_hi(v.w);
        }
        sums[i] = acc;
    }
}

// ---- kernels ----------------------------------------------------------------
template <int MT>
__global__ void __launch_bounds__(kFfnThreads) ffn_gateup_kernel(const __grid_constant__ FfnArgs a) {
    extern __shared__ __align__(16) uint8_t smem[];
    uint16_t* xs = reinterpret_cast<uint16_t*>(smem);                              // [MT][d]
    float* xsum = reinterpret_cast<float*>(smem + static_cast<size_t>(MT) * a.d * 2);  // [MT][d/32]
    __shared__ int seg[MOE_MAX_EXPERTS + 1];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int nseg = build_segments<MT>(a, seg);
    const long long total = static_cast<long long>(nseg) * a.f;
    const long long r_begin = total * blockIdx.x / gridDim.x;
    const long long r_end = total * (blockIdx.x + 1) / gridDim.x;
    const int cpr = a.d / 8;  // 16-byte chunks per x row
    for (long long r = r_begin; r < r_end;) {
        const int s = static_cast<int>(r / a.f);
        const long long piece_end = min(r_end, static_cast<long long>(s + 1) * a.f);
        const int e = expert_of_segment(seg, a.E, s);
        const int row0 = a.offsets[e] + (s - seg[e]) * MT;
        const int mcount = min(MT, a.offsets[e + 1] - row0);
        __syncthreads();
        for (int i = threadIdx.x; i < MT * cpr; i += blockDim.x) {
            const int m = i / cpr, c = i - m * cpr;
            uint4 v = make_uint4(0, 0, 0, 0);
            if (m < mcount) {
                const int t = a.perm[row0 + m] / a.k;
                v = *reinterpret_cast<const uint4*>(a.x + static_cast<size_t>(t) * a.d + c * 8);
            }
            reinterpret_cast<uint4*>(xs)[i] = v;
        }
        __syncthreads();
        const moe_expert_weights& W = a.ex[e];
        if (W.precision == MOE_P4) {
            chunk_sums(xs, xsum, MT, a.d);
            __syncthreads();
        }
        const int n_base = static_cast<int>(r - static_cast<long long>(s) * a.f);
        const int cnt = static_cast<int>(piece_end - r);
        for (int i = warp; i < cnt; i += kFfnWarps) {
            const int n = n_base + i;
            float ag[MT], au[MT];
            if (W.precision == MOE_P4)
                rowpair_int4<MT>(W, n, a.d, a.f, xs, xsum, lane, ag, au);
            else
                rowpair_bf16<MT>(W, n, a.d, a.f, xs, lane, ag, au);
#pragma unroll
            for (int m = 0; m < MT; ++m) {
                const float g = warp_sum(ag[m]);
                const float u = warp_sum(au[m]);
                if (lane == 0 && m < mcount)
                    a.h[static_cast<size_t>(row0 + m) * a.f + n] = f2bf(silu_f(g) * u);
            }
        }
        r = piece_end;
    }
}

template <int MT>
__global__ void __launch_bounds__(kFfnThreads) ffn_down_kernel(const __grid_constant__ FfnArgs a) {
    extern __shared__ __align__(16) uint8_t smem[];
    uint16_t* hs = reinterpret_cast<uint16_t*>(smem);                              // [MT][f]
    float* hsum = reinterpret_cast<float*>(smem + static_cast<size_t>(MT) * a.f * 2);  // [MT][f/32]
    __shared__ int seg[MOE_MAX_EXPERTS + 1];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int nseg = build_segments<MT>(a, seg);
    const long long total = static_cast<long long>(nseg) * a.d;
    const long long r_begin = total * blockIdx.x / gridDim.x;
    const long long r_end = total * (blockIdx.x + 1) / gridDim.x;
    const int cpr = a.f / 8;
    for (long long r = r_begin; r < r_end;) {
        const int s = static_cast<int>(r / a.d);
        const long long piece_end = min(r_end, static_cast<long long>(s + 1) * a.d);
        const int e = expert_of_segment(seg, a.E, s);
        const int row0 = a.offsets[e] + (s - seg[e]) * MT;
        const int mcount = min(MT, a.offsets[e + 1] - row0);
        __syncthreads();
        for (int i = threadIdx.x; i < MT * cpr; i += blockDim.x) {
            const int m = i / cpr, c = i - m * cpr;
            uint4 v = make_uint4(0, 0, 0, 0);
            if (m < mcount) v = *reinterpret_cast<const uint4*>(a.h + static_cast<size_t>(row0 + m) * a.f + c * 8);
            reinterpret_cast<uint4*>(hs)[i] = v;
        }
        __syncthreads();
        const moe_expert_weights& W = a.ex[e];
        if (W.precision == MOE_P4) {
            chunk_sums(hs, hsum, MT, a.f);
            __syncthreads();
        }
        const int j_base = static_cast<int>(r - static_cast<long long>(s) * a.d);
        const int cnt = static_cast<int>(piece_end - r);
        for (int i = warp; i < cnt; i += kFfnWarps) {
            const int j = j_base + i;
            float acc[MT];
            if (W.precision == MOE_P4)
                row_down_int4<MT>(W, j, a.f, hs, hsum, lane, acc);
            else
                row_down_bf16<MT>(W, j, a.f, hs, lane, acc);
#pragma unroll
            for (int m = 0; m < MT; ++m) {
                const float v = warp_sum(acc[m]);
                if (lane == 0 && m < mcount) a.y[static_cast<size_t>(row0 + m) * a.d + j] = v;
            }
        }
        r = piece_end;
    }
}

template <int MT>
cudaError_t launch_ffn(const FfnArgs& a, cudaStream_t stream) {
    // Launch geometry is a pure function of (d, f): cache it so the hot path
    // issues no attribute/occupancy queries (and stays graph-capturable).
    static int cached_d = -1, cached_f = -1, grid_gu = 0, grid_dn = 0;
    const size_t smem_gu = static_cast<size_t>(MT) * a.d * 2 + static_cast<size_t>(MT) * (a.d / 32) * 4;
    const size_t smem_dn = static_cast<size_t>(MT) * a.f * 2 + static_cast<size_t>(MT) * (a.f / 32) * 4;
    if (cached_d != a.d || cached_f != a.f) {
        MOE_CUDA_OK(cudaFuncSetAttribute(ffn_gateup_kernel<MT>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem_gu)));
        MOE_CUDA_OK(cudaFuncSetAttribute(ffn_down_kernel<MT>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem_dn)));
        int dev = 0, sms = 0, occ_gu = 0, occ_dn = 0;
        MOE_CUDA_OK(cudaGetDevice(&dev));
        MOE_CUDA_OK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
        MOE_CUDA_OK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ_gu, ffn_gateup_kernel<MT>, kFfnThreads, smem_gu));
        MOE_CUDA_OK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ_dn, ffn_down_kernel<MT>, kFfnThreads, smem_dn));
        grid_gu = sms * (occ_gu > 0 ? occ_gu : 1);
        grid_dn = sms * (occ_dn > 0 ? occ_dn : 1);
        cached_d = a.d;
        cached_f = a.f;
    }
    ffn_gateup_kernel<MT><<<grid_gu, kFfnThreads, smem_gu, stream>>>(a);
    MOE_CUDA_OK(cudaGetLastError());
    ffn_down_kernel<MT><<<grid_dn, kFfnThreads, smem_dn, stream>>>(a);
    return cudaGetLastError();
}

}  // namespace moek

cudaError_t moek_ffn_gemv(const void* x, const int32_t* perm, const int32_t* offsets, int T, int k,
                          const moe_expert_weights* experts, int E, int d, int f, void* h_ws,
                          float* y_perm, uint64_t active_mask, cudaStream_t stream) {
    moek::FfnArgs a{};
    a.active_mask = active_mask;
    a.x = static_cast<const uint16_t*>(x);
    a.perm = perm;
    a.offsets = offsets;
    a.T = T;
    a.k = k;
    a.E = E;
    a.d = d;
    a.f = f;
    a.h = static_cast<uint16_t*>(h_ws);
    a.y = y_perm;
    for (int e = 0; e < E; ++e) a.ex[e] = experts[e];
    if (T <= 1) return moek::launch_ffn<1>(a, stream);
    if (T <= 2) return moek::launch_ffn<2>(a, stream);
    return moek::launch_ffn<4>(a, stream);
}
