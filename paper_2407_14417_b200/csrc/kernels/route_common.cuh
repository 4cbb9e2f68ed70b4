// route_common.cuh -- the router's per-token device functions, shared by
// the route kernel (router.cu) and the fused decode-step kernel (gemv.cu),
// so both compute bit-identical logits, top-k and permutations
// (oracle orc_gate_topk / orc_permute).
#pragma once

#include "common.cuh"

namespace moek {

// One logit in the pinned order.  x_s is the token row staged in smem.
constexpr int kPreChunks = 16;  // router-weight chunks (256 elements each) held in registers

// One logit in the pinned order.  x_s is the token row staged in smem; the
// first kPreChunks chunks of this lane's weights come preloaded in wpre
// (issued before the PDL wait), the rest are loaded 8 chunks at a time.
MOE_DEVI float router_dot(const uint16_t* __restrict__ x_s, const uint4 (&wpre)[kPreChunks],
                          const uint16_t* __restrict__ we, int d, int lane) {
    float acc = 0.0f;
    const int nfull = d / 256;  // chunks where every lane has 8 elements
    auto fma8 = [&](const uint4& wv, int c) {
        const uint4 xv = *reinterpret_cast<const uint4*>(x_s + c * 256 + lane * 8);
        const uint32_t ww[4] = {wv.x, wv.y, wv.z, wv.w};
        const uint32_t xx[4] = {xv.x, xv.y, xv.z, xv.w};
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            acc = __fmaf_rn(bf16_lo(xx[q]), bf16_lo(ww[q]), acc);
            acc = __fmaf_rn(bf16_hi(xx[q]), bf16_hi(ww[q]), acc);
        }
    };
#pragma unroll
    for (int c = 0; c < kPreChunks; ++c)
        if (c < nfull) fma8(wpre[c], c);
    for (int c0 = kPreChunks; c0 < nfull; c0 += 8) {
        uint4 wv[8];
#pragma unroll
        for (int u = 0; u < 8; ++u)
            if (c0 + u < nfull) wv[u] = __ldg(reinterpret_cast<const uint4*>(we + (c0 + u) * 256 + lane * 8));
#pragma unroll
        for (int u = 0; u < 8; ++u)
            if (c0 + u < nfull) fma8(wv[u], c0 + u);
    }
    {
        const int k0 = nfull * 256 + lane * 8;  // ragged tail chunk
        for (int j = 0; j < 8 && k0 + j < d; ++j) acc = __fmaf_rn(bf2f(x_s[k0 + j]), bf2f(we[k0 + j]), acc);
    }
#pragma unroll
    for (int off = 16; off >= 1; off >>= 1) acc = __fadd_rn(acc, __shfl_xor_sync(0xffffffffu, acc, off));
    return acc;
}

MOE_DEVI void preload_w(uint4 (&wpre)[kPreChunks], const uint16_t* __restrict__ we, int d, int lane) {
    const int nfull = d / 256;
#pragma unroll
    for (int c = 0; c < kPreChunks; ++c)
        if (c < nfull) wpre[c] = __ldg(reinterpret_cast<const uint4*>(we + c * 256 + lane * 8));
}

// The same stable counting sort for n <= 32 items by one warp, no block
// barriers: lane i holds item i's expert; its position is the count of
// items with a smaller expert, plus those with the same expert and a lower
// index.
MOE_DEVI void warp_permute(const int32_t* idx, int n, int E, int32_t* counts, int32_t* offsets, int32_t* perm,
                           int32_t* inv_perm, int lane) {
    const int ei = lane < n ? idx[lane] : 0x7fffffff;
    int pos = 0;
    for (int j = 0; j < n; ++j) {
        const int ej = __shfl_sync(0xffffffffu, ei, j);
        pos += (ej < ei) || (ej == ei && j < lane);
    }
    if (lane < n) {
        perm[pos] = lane;
        inv_perm[lane] = pos;
    }
    // counts / offsets: lane e (and e+32) counts its expert
    for (int e = lane; e < E; e += 32) {
        int c = 0, below = 0;
        for (int j = 0; j < n; ++j) {
            const int ej = idx[j];
            c += ej == e;
            below += ej < e;
        }
        counts[e] = c;
        offsets[e] = below;
        if (e == E - 1) offsets[E] = n;
    }
}

// Top-k on logits by one warp, in registers: lane e holds logits e and
// e+32; k rounds of a butterfly argmax (ties -> lower index) give the
// selection in descending-logit order; weights = softmax over the selected
// logits (sequential j order, as the oracle).
MOE_DEVI void warp_topk(const float* lg, int E, int k, int lane, int32_t* idx_out, float* w_out, int* s_idx) {
    float v0 = lane < E ? lg[lane] : 0.0f, v1 = lane + 32 < E ? lg[lane + 32] : 0.0f;
    bool ok0 = lane < E, ok1 = lane + 32 < E;
    float sel[MOE_MAX_TOPK];
    int sid[MOE_MAX_TOPK];
#pragma unroll
    for (int j = 0; j < MOE_MAX_TOPK; ++j) {
        sel[j] = 0.0f;
        sid[j] = 0;
        if (j < k) {
            bool has;
            float bv;
            int bi;
            if (ok1 && (!ok0 || v1 > v0)) {
                has = true; bv = v1; bi = lane + 32;
            } else {
                has = ok0; bv = v0; bi = lane;
            }
#pragma unroll
            for (int off = 16; off >= 1; off >>= 1) {
                const float ov = __shfl_xor_sync(0xffffffffu, bv, off);
                const int oi = __shfl_xor_sync(0xffffffffu, bi, off);
                const bool oh = __shfl_xor_sync(0xffffffffu, has ? 1 : 0, off) != 0;
                if (oh && (!has || ov > bv || (ov == bv && oi < bi))) {
                    bv = ov;
                    bi = oi;
                    has = true;
                }
            }
            sel[j] = bv;
            sid[j] = bi;
            if (bi == lane) ok0 = false;
            if (bi == lane + 32) ok1 = false;
        }
    }
    // softmax over the selected logits: lane j < k takes sel[j]; the sum is
    // accumulated in j order (as the oracle) from the lanes' exponentials
    float mine = 0.0f;
    int mid = 0;
#pragma unroll
    for (int j = 0; j < MOE_MAX_TOPK; ++j)
        if (j == lane) {
            mine = sel[j];
            mid = sid[j];
        }
    const float ex = lane < k ? expf(mine - sel[0]) : 0.0f;
    float sum = 0.0f;
    for (int j = 0; j < k; ++j) sum += __shfl_sync(0xffffffffu, ex, j);
    if (lane < k) {
        idx_out[lane] = mid;
        w_out[lane] = ex / sum;
        s_idx[lane] = mid;
    }
}


}  // namespace moek
