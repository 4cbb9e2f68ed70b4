// gemv.cu -- K3/K4 expert-FFN GEMV for decode batches (<= 8 tokens per
// expert segment): int4-g128 and bf16 experts, mixed in one launch.
//
// Replaces the constant compute latency of the reference's MoE-layer
// stand-in (simulator.cpp:31-32, :107) with the expert math of HF
// MixtralExperts (modeling_mixtral.py:90-95).
//
// Data path (B200):
//   HBM --cp.async.bulk (TMA bulk copy, mbarrier complete_tx)--> per-warp
//   shared-memory ring (3 stages x 8.25 KB) --LDS.128--> mma.m16n8k16 A
//   fragments.  Each warp owns a contiguous range of equal-byte work items
//   and keeps its next items in flight while computing the current one, so
//   the bytes in flight per SM (up to 8 warps x 3 x 8 KB) do not depend on
//   register pressure.
// Weights are stored as 16-row x 128-K "fragment blocks" (oracle
// orc_pack_*_blocks): a work item (16-row tile, K-part) is one contiguous
// span of blocks (one bulk copy), and a lane's 16-byte smem read is exactly
// its A fragment.  int4 fragments are decoded in registers (LOP3 magic
// number -> bf16 128+u, one bf16x2 FMA -> q exactly); the tensor core does
// the multiply-accumulate in fp32 and the group scale is applied after each
// 128-K group, y += s * sum(q*x) -- the exact dequant values q*s.  B
// fragments (x or h) come from a K-permuted copy (xperm / hperm) with the
// same 128-bit pattern.  Up to 8 tokens of an expert share each weight byte.
//
// Split-K bookkeeping: a warp accumulates consecutive K-parts of a row tile
// in registers ("run") and adds one fp32 partial into a zero-initialised
// slot per run; per-tile counters count finished items, and the warp that
// completes a tile reduces its K-part slots in fixed order (deterministic),
// re-zeroes them, and runs the fused epilogue: SwiGLU + bf16 h (gate/up
// pass) or routing-weighted combine + residual (down pass).
#include "common.cuh"
#include "launch.h"

namespace moek {

constexpr int kWarps = 12;
constexpr int kThreads = kWarps * 32;
constexpr int kStages = 2;
constexpr int kStageBytes = 8192 + 256;  // 8 KB of weights + int4 scales
constexpr int kTile = 8;                 // tokens per segment tile (MMA n)
constexpr int kMaxSegs = 128;

struct GemvArgs {
    const int32_t* offsets;   // [E+1]
    const int32_t* perm;      // [T*k]: slot -> t*k + j
    int T, k, E;
    int kshift;               // log2(k)
    int rows, K;              // matrix rows / columns of this pass
    int down;                 // 0 gate/up pass, 1 down pass
    int gk4, gk16;            // 128-K groups per item (int4, bf16)
    const uint16_t* bperm;    // B operand, K-permuted: [T][K] (gate/up) or [T*k][K] (down)
    const float* bsum;        // per-(B row, 128-group) sums of B: [rows of B][K/128]
    float* part;              // zeroed partial slots [KPmax][T*k][rows]
    unsigned int* counters;   // zeroed arrival counters
    unsigned int* gcounters;  // zeroed per-(segment, h group) counters (gate/up)
    uint16_t* hperm;          // gate/up epilogue output [T*k][f] (K-permuted)
    float* hsum16;            // gate/up epilogue: sums of 16 h rows [T*k][f/16]
    float* hsum;              // gate/up epilogue: sums of 128 h rows [T*k][f/128]
    int f;
    const float* wts;         // down epilogue: routing weights [T*k]
    const int32_t* inv;       // [T*k]
    const uint16_t* resid;    // [T][d] or null
    uint16_t* out;            // [T][d]; null -> write y per slot
    float* y;                 // [T*k][d]
    uint64_t active_mask;
    moe_expert_weights ex[MOE_MAX_EXPERTS];
};

struct SegTable {
    int n;
    int items_per_rt;         // sum over segments of KP (down-pass tile total)
    int e[kMaxSegs];
    int tile[kMaxSegs];
    int kp[kMaxSegs];
    int gk[kMaxSegs];
    long long pre[kMaxSegs + 1];
};

// ---- PTX wrappers: mbarrier + bulk async copy ------------------------------
MOE_DEVI uint32_t smem_u32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }
MOE_DEVI void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
MOE_DEVI void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}
MOE_DEVI void mbar_wait(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra WAIT_%=;\n}" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}
MOE_DEVI void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}
MOE_DEVI void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
// Release-only arrival: orders this warp's partial stores (after __syncwarp)
// before the counter update without the L1 invalidation a full gpu-scope
// fence costs; only the completing warp pays the acquire fence.
MOE_DEVI unsigned int atom_add_release(unsigned int* p, unsigned int v) {
    unsigned int old;
    asm volatile("atom.release.gpu.global.add.u32 %0, [%1], %2;" : "=r"(old) : "l"(p), "r"(v) : "memory");
    return old;
}
MOE_DEVI void fence_mbar_init() { asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }

MOE_DEVI void mma_bf16(float (&c)[4], uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3, uint32_t b0,
                       uint32_t b1) {
    asm volatile(
        "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
        "{%0,%1,%2,%3};"
        : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
        : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}

// Optional per-warp phase trace (moe_debug_gemv_trace): globaltimer stamps
// [entry, after pdl_wait, first item ready, loop end] + item / run / epilogue
// counts, 8 x u64 per warp.  Null (the default) costs one branch per warp.
__device__ unsigned long long* g_gemv_trace = nullptr;
MOE_DEVI unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}

MOE_DEVI uint4 lds128(const uint8_t* p) { return *reinterpret_cast<const uint4*>(p); }
MOE_DEVI uint4 ldb(const uint16_t* p) { return *reinterpret_cast<const uint4*>(p); }

// B fragments of one 128-K group: 4 x 16 B of this lane's token row
MOE_DEVI void load_b(uint4 (&b)[4], const uint16_t* bp, bool valid) {
#pragma unroll
    for (int c = 0; c < 4; ++c) b[c] = valid ? ldb(bp + c * 8) : make_uint4(0, 0, 0, 0);
}

// biased bf16 pairs (128+u) from a packed word (3 SHF + 4 LOP3, no FMA):
// pairs for MMA kk=2q (p01 reg0, p23 reg2) and kk=2q+1 (p45, p67)
MOE_DEVI void decode_u(uint32_t w, uint32_t& p01, uint32_t& p23, uint32_t& p45, uint32_t& p67) {
    p01 = and_or(w, 0x000F000Fu, 0x43004300u);
    p23 = and_or(w >> 4, 0x000F000Fu, 0x43004300u);
    p45 = and_or(w >> 8, 0x000F000Fu, 0x43004300u);
    p67 = and_or(w >> 12, 0x000F000Fu, 0x43004300u);
}

// One int4 item (gk 128-K groups).  The MMA sees the biased values 128+u
// (exact in bf16); per group sum(q x) = sum((128+u) x) - 136 sum(x), with
// sum(x) of the column's activation group (scol0: column 2t, scol1: 2t+1),
// then y += s * sum(q x) (two independent HMMA chains per group).
MOE_DEVI void item_int4(const uint8_t* stage, int gk, const uint16_t* bp, bool bvalid, const float* scol0,
                        const float* scol1, int g0, int lane, float (&acc)[4]) {
    const int t = lane & 3;
    const uint8_t* sc = stage + gk * 1024;
    float sv0[8], sv1[8];
#pragma unroll
    for (int g = 0; g < 8; ++g) {
        sv0[g] = (scol0 && g < gk) ? __ldg(scol0 + g0 + g) : 0.0f;
        sv1[g] = (scol1 && g < gk) ? __ldg(scol1 + g0 + g) : 0.0f;
    }
    uint4 ba[4], bb[4];
    load_b(ba, bp + t * 32, bvalid);
#pragma unroll
    for (int g = 0; g < 8; g += 2) {
        if (g >= gk) break;
        // ping-pong B buffers (no register copies): ba = group g, bb = g+1
        if (g + 1 < gk) load_b(bb, bp + (g + 1) * 128 + t * 32, bvalid);
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const int gg = g + h;
            if (gg >= gk) break;
            const uint4(&b)[4] = h == 0 ? ba : bb;
            const uint32_t s2 = *reinterpret_cast<const uint32_t*>(sc + gg * 32 + (lane >> 2) * 4);
            const float S0 = sv0[gg], S1 = sv1[gg];
            const uint4 wl = lds128(stage + gg * 1024 + lane * 16);
            const uint4 wh = lds128(stage + gg * 1024 + 512 + lane * 16);
            const uint32_t lo[4] = {wl.x, wl.y, wl.z, wl.w};
            const uint32_t hi[4] = {wh.x, wh.y, wh.z, wh.w};
            float cg[4] = {0.f, 0.f, 0.f, 0.f}, ch[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                uint32_t r0, r2, r0b, r2b, s0, sq2, s0b, s2b;
                decode_u(lo[q], r0, r2, r0b, r2b);   // row gr
                decode_u(hi[q], s0, sq2, s0b, s2b);  // row gr+8
                mma_bf16(cg, r0, s0, r2, sq2, b[q].x, b[q].y);
                mma_bf16(ch, r0b, s0b, r2b, s2b, b[q].z, b[q].w);
            }
            const float s_lo = bf16_lo(s2), s_hi = bf16_hi(s2);
            acc[0] = __fmaf_rn(s_lo, __fmaf_rn(-kInt4Bias, S0, cg[0] + ch[0]), acc[0]);
            acc[1] = __fmaf_rn(s_lo, __fmaf_rn(-kInt4Bias, S1, cg[1] + ch[1]), acc[1]);
            acc[2] = __fmaf_rn(s_hi, __fmaf_rn(-kInt4Bias, S0, cg[2] + ch[2]), acc[2]);
            acc[3] = __fmaf_rn(s_hi, __fmaf_rn(-kInt4Bias, S1, cg[3] + ch[3]), acc[3]);
            if (h == 0 && g + 2 < gk) load_b(ba, bp + (g + 2) * 128 + t * 32, bvalid);
        }
    }
}

MOE_DEVI void item_bf16(const uint8_t* stage, int gk, const uint16_t* bp, bool bvalid, int lane, float (&acc)[4]) {
    const int t = lane & 3;
    float c1[4] = {0.f, 0.f, 0.f, 0.f};  // second chain (odd kk)
    uint4 ba[4], bb[4];
    load_b(ba, bp + t * 32, bvalid);
    for (int g = 0; g < gk; g += 2) {
        if (g + 1 < gk) load_b(bb, bp + (g + 1) * 128 + t * 32, bvalid);
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const int gg = g + h;
            if (gg >= gk) break;
            const uint4(&b)[4] = h == 0 ? ba : bb;
#pragma unroll
            for (int c = 0; c < 4; ++c) {
                // part c = row gr words for kk = 2c, 2c+1; part 4+c = row gr+8
                const uint4 lo = lds128(stage + gg * 4096 + c * 512 + lane * 16);
                const uint4 hi = lds128(stage + gg * 4096 + (4 + c) * 512 + lane * 16);
                mma_bf16(acc, lo.x, hi.x, lo.y, hi.y, b[c].x, b[c].y);
                mma_bf16(c1, lo.z, hi.z, lo.w, hi.w, b[c].z, b[c].w);
            }
            if (h == 0 && g + 2 < gk) load_b(ba, bp + (g + 2) * 128 + t * 32, bvalid);
        }
    }
#pragma unroll
    for (int r = 0; r < 4; ++r) acc[r] += c1[r];
}

// token of a permutation slot (perm[slot] = t*k + j); k is a power of two in
// every config we run, so this is a shift (division otherwise)
MOE_DEVI int tok_of_slot(const GemvArgs& a, int slot) {
    return a.kshift >= 0 ? a.perm[slot] >> a.kshift : a.perm[slot] / a.k;
}

// K-permuted position of natural index n (orc_perm_k)
MOE_DEVI int perm_k(int n) {
    const int kin = n & 127;
    return (n & ~127) + ((kin & 7) >> 1) * 32 + (kin >> 4) * 4 + ((kin >> 3) & 1) * 2 + (kin & 1);
}

MOE_DEVI void build_segs(const GemvArgs& a, SegTable& st, int* cnt) {
    // expert token counts read in parallel (one L2 round trip), then a short
    // serial pass over <= 64 experts in shared memory
    if (threadIdx.x < a.E)
        cnt[threadIdx.x] = ((a.active_mask >> threadIdx.x) & 1ull)
                               ? a.offsets[threadIdx.x + 1] - a.offsets[threadIdx.x]
                               : 0;
    __syncthreads();
    if (threadIdx.x == 0) {
        const int RT = a.rows / 16, G = a.K / 128;
        int n = 0, items_rt = 0;
        long long acc = 0;
        for (int e = 0; e < a.E; ++e) {
            const int m = cnt[e];
            if (m == 0) continue;
            const int gk = a.ex[e].precision == MOE_P4 ? a.gk4 : a.gk16;
            const int kp = G / gk;
            for (int t = 0; t * kTile < m && n < kMaxSegs; ++t) {
                st.e[n] = e;
                st.tile[n] = t;
                st.kp[n] = kp;
                st.gk[n] = gk;
                st.pre[n] = acc;
                acc += static_cast<long long>(RT) * kp;
                items_rt += kp;
                ++n;
            }
        }
        st.pre[n] = acc;
        st.n = n;
        st.items_per_rt = items_rt;
    }
    __syncthreads();
}

// reduce + re-zero the K-part slots of (row, slot)
MOE_DEVI float take_partial(const GemvArgs& a, int kp_count, int row, int slot) {
    const int nslots = a.T * a.k;
    const size_t stride = static_cast<size_t>(nslots) * a.rows;
    float* base = a.part + static_cast<size_t>(slot) * a.rows + row;
    float v = 0.0f;
    for (int kp = 0; kp < kp_count; kp += 8) {
        float x[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) x[u] = kp + u < kp_count ? __ldcg(base + (kp + u) * stride) : 0.0f;
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            if (x[u] != 0.0f) {
                v += x[u];
                __stcg(base + (kp + u) * stride, 0.0f);
            }
        }
    }
    return v;
}

MOE_DEVI int seg_of_slot(const GemvArgs& a, const SegTable& st, int slot) {
    for (int s = 0; s < st.n; ++s) {
        const int e = st.e[s];
        const int lo = a.offsets[e] + st.tile[s] * kTile;
        if (slot >= lo && slot < min(lo + kTile, a.offsets[e + 1])) return s;
    }
    return -1;
}

// SwiGLU for the 16 rows of pair tile prt and every token of segment s, plus
// the activation-group sums the int4 down pass needs: sum of the 16 rounded
// h values (fixed xor-butterfly order), and -- by the last of the 8 pair
// tiles of a 128-row group -- their fixed-order total.
MOE_DEVI void epilogue_gateup(const GemvArgs& a, const SegTable& st, int s, int prt, int lane) {
    const int e = st.e[s];
    const int slot0 = a.offsets[e] + st.tile[s] * kTile;
    const int m_cnt = min(kTile, a.offsets[e + 1] - slot0);
    const int f16 = a.f / 16, f128 = a.f / 128;
    for (int i0 = 0; i0 < m_cnt * 16; i0 += 32) {
        const int i = i0 + lane;
        const int m = i >> 4, n = prt * 16 + (i & 15), slot = slot0 + m;
        float hv = 0.0f;
        if (i < m_cnt * 16) {
            const float g = take_partial(a, st.kp[s], n, slot);
            const float u = take_partial(a, st.kp[s], a.f + n, slot);
            const uint16_t hb = f2bf(silu_f(g) * u);
            a.hperm[static_cast<size_t>(slot) * a.f + perm_k(n)] = hb;
            hv = bf2f(hb);
        }
        // sum over the 16 rows held by each half-warp
#pragma unroll
        for (int off = 8; off >= 1; off >>= 1) hv += __shfl_xor_sync(0xffffffffu, hv, off);
        if ((lane & 15) == 0 && i < m_cnt * 16) __stcg(a.hsum16 + static_cast<size_t>(slot) * f16 + prt, hv);
    }
    __syncwarp();
    int last = 0;
    if (lane == 0) {
        unsigned int* ctr = a.gcounters + static_cast<size_t>(s) * f128 + prt / 8;
        if (atom_add_release(ctr, 1u) + 1 == 8u) {
            *ctr = 0;
            last = 1;
        }
    }
    last = __shfl_sync(0xffffffffu, last, 0);
    if (last) {
        const int g = prt / 8;
        for (int m = lane; m < m_cnt; m += 32) {
            const float* p = a.hsum16 + static_cast<size_t>(slot0 + m) * f16 + g * 8;
            float v = 0.0f;
#pragma unroll
            for (int r = 0; r < 8; ++r) v += __ldcg(p + r);
            a.hsum[static_cast<size_t>(slot0 + m) * f128 + g] = v;
        }
    }
}

MOE_DEVI void epilogue_down(const GemvArgs& a, const SegTable& st, int rt, int lane) {
    const int d = a.rows;
    if (a.out == nullptr) {
        for (int i = lane; i < a.T * a.k * 16; i += 32) {
            const int slot = i >> 4, j = rt * 16 + (i & 15);
            const int s = seg_of_slot(a, st, slot);
            if (s >= 0) a.y[static_cast<size_t>(slot) * d + j] = take_partial(a, st.kp[s], j, slot);
        }
        return;
    }
    for (int i = lane; i < a.T * 16; i += 32) {
        const int t = i >> 4, j = rt * 16 + (i & 15);
        float accv = a.resid ? bf2f(a.resid[static_cast<size_t>(t) * d + j]) : 0.0f;
        for (int jj = 0; jj < a.k; ++jj) {
            const int slot = a.inv[t * a.k + jj];
            const int s = seg_of_slot(a, st, slot);
            const float yv = s < 0 ? 0.0f : take_partial(a, st.kp[s], j, slot);
            accv = __fmaf_rn(a.wts[t * a.k + jj], yv, accv);
        }
        a.out[static_cast<size_t>(t) * d + j] = f2bf(accv);
    }
}

struct ItemIt {
    int s, rt, kp;
};

MOE_DEVI void advance(ItemIt& it, const SegTable& st, int RT) {
    if (++it.kp == st.kp[it.s]) {
        it.kp = 0;
        if (++it.rt == RT) {
            it.rt = 0;
            ++it.s;
        }
    }
}

MOE_DEVI ItemIt locate(long long i, const SegTable& st) {
    ItemIt it{0, 0, 0};
    while (st.pre[it.s + 1] <= i) ++it.s;
    const long long local = i - st.pre[it.s];
    it.rt = static_cast<int>(local / st.kp[it.s]);
    it.kp = static_cast<int>(local - static_cast<long long>(it.rt) * st.kp[it.s]);
    return it;
}

// issue the bulk copies of one item into a ring stage (lane 0 only)
MOE_DEVI void issue_item(const GemvArgs& a, const SegTable& st, const ItemIt& it, uint8_t* stage, uint64_t* bar) {
    const moe_expert_weights& W = a.ex[st.e[it.s]];
    const int G = a.K / 128, gk = st.gk[it.s];
    const size_t blk = static_cast<size_t>(it.rt) * G + static_cast<size_t>(it.kp) * gk;
    const uint8_t* w = static_cast<const uint8_t*>(a.down ? W.w_down : W.w_gate_up);
    if (W.precision == MOE_P4) {
        const uint8_t* sc = static_cast<const uint8_t*>(a.down ? W.s_down : W.s_gate_up);
        mbar_expect_tx(bar, gk * 1024 + gk * 32);
        bulk_g2s(stage, w + blk * 1024, gk * 1024, bar);
        bulk_g2s(stage + gk * 1024, sc + blk * 32, gk * 32, bar);
    } else {
        mbar_expect_tx(bar, gk * 4096);
        bulk_g2s(stage, w + blk * 4096, gk * 4096, bar);
    }
}

__global__ void __launch_bounds__(kThreads, 1) gemv_kernel(const __grid_constant__ GemvArgs a) {
    extern __shared__ __align__(128) uint8_t smem[];
    __shared__ SegTable st;
    __shared__ __align__(8) uint64_t bars[kWarps][kStages];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    uint8_t* ring = smem + static_cast<size_t>(warp) * kStages * kStageBytes;
    if (lane == 0) {
        for (int s = 0; s < kStages; ++s) mbar_init(&bars[warp][s], 1);
        fence_mbar_init();
    }
    __shared__ int cnt[MOE_MAX_EXPERTS];
    // Routing (offsets) comes from the route kernel two launches back, so the
    // segment table and the first weight bulk copies are issued before the
    // PDL wait -- weight streaming overlaps the predecessor's tail.
    const unsigned long long t_entry = gtimer();
    build_segs(a, st, cnt);  // contains __syncthreads
    const int N = static_cast<int>(st.pre[st.n]);
    const int W = static_cast<int>(gridDim.x) * kWarps;
    const int wid = static_cast<int>(blockIdx.x) * kWarps + warp;
    // equal contiguous ranges: q items each, the first r warps one more
    const int q = N / W, r = N - q * W;
    const long long i0 = static_cast<long long>(wid) * q + min(wid, r);
    const long long i1 = i0 + q + (wid < r ? 1 : 0);
    const int RT = a.rows / 16;
    const int nslots = a.T * a.k;
    const int gr = lane >> 2, t = lane & 3;

    // prologue: fill the ring (weights only: independent of the predecessor)
    ItemIt issue_it{0, 0, 0};
    long long issued = i0;
    if (i0 < i1) {
        issue_it = locate(i0, st);
        for (int s = 0; s < kStages && issued < i1; ++s, ++issued) {
            if (lane == 0) issue_item(a, st, issue_it, ring + s * kStageBytes, &bars[warp][s]);
            advance(issue_it, st, RT);
        }
    }
    pdl_wait();     // B operand / counters / partials of the predecessor
    pdl_trigger();
    if (i0 >= i1) return;
    const unsigned long long t_wait = gtimer();
    unsigned long long t_first = 0;
    int n_runs = 0, n_epi = 0;

    ItemIt it = locate(i0, st);
    long long i = i0;
    uint32_t phase_bits = 0;  // per-stage parity
    int stage = 0;
    while (i < i1) {
        const int s = it.s, rt = it.rt;
        const int e = st.e[s];
        const int prec = a.ex[e].precision;
        const int gk = st.gk[s];
        const int kp0 = it.kp;
        const int slot0 = a.offsets[e] + st.tile[s] * kTile;
        const int m_cnt = min(kTile, a.offsets[e + 1] - slot0);
        const bool bvalid = gr < m_cnt;
        int brow = 0;
        if (bvalid) brow = a.down ? slot0 + gr : tok_of_slot(a, slot0 + gr);
        const uint16_t* brow_p = a.bperm + static_cast<size_t>(brow) * a.K;
        // activation-group sums of this lane's two C columns (int4 bias)
        const int G = a.K / 128;
        const float* scol[2] = {nullptr, nullptr};
#pragma unroll
        for (int c = 0; c < 2; ++c) {
            const int n = 2 * t + c;
            if (n < m_cnt) {
                const int rb = a.down ? slot0 + n : tok_of_slot(a, slot0 + n);
                scol[c] = a.bsum + static_cast<size_t>(rb) * G;
            }
        }
        float acc[4] = {0.f, 0.f, 0.f, 0.f};
        int run_len = 0;
        // one run: consecutive K-parts of (s, rt) within this warp's range
        while (i < i1 && it.s == s && it.rt == rt) {
            mbar_wait(&bars[warp][stage], (phase_bits >> stage) & 1u);
            if (t_first == 0) t_first = gtimer();
            phase_bits ^= 1u << stage;
            const uint8_t* sp = ring + stage * kStageBytes;
            const uint16_t* bp = brow_p + static_cast<size_t>(it.kp) * gk * 128;
            if (prec == MOE_P4)
                item_int4(sp, gk, bp, bvalid, scol[0], scol[1], it.kp * gk, lane, acc);
            else
                item_bf16(sp, gk, bp, bvalid, lane, acc);
            // release the stage and refill it with the item kStages ahead
            fence_proxy_async();
            __syncwarp();
            if (issued < i1) {
                if (lane == 0) issue_item(a, st, issue_it, ring + stage * kStageBytes, &bars[warp][stage]);
                advance(issue_it, st, RT);
                ++issued;
            }
            stage = stage + 1 == kStages ? 0 : stage + 1;
            advance(it, st, RT);
            ++i;
            ++run_len;
        }
        // flush the run into its (zeroed) K-part slot: columns 2t, 2t+1
        const int row = rt * 16 + gr;
#pragma unroll
        for (int c = 0; c < 2; ++c) {
            const int m = 2 * t + c;
            if (m < m_cnt) {
                float* p = a.part + (static_cast<size_t>(kp0) * nslots + slot0 + m) * a.rows;
                __stcg(p + row, acc[c]);
                __stcg(p + row + 8, acc[2 + c]);
            }
        }
        __syncwarp();
        int last = 0;
        if (lane == 0) {
            unsigned int* ctr;
            unsigned int total;
            if (!a.down) {
                const int ftiles = a.f / 16;
                ctr = a.counters + static_cast<size_t>(s) * ftiles + (rt >= ftiles ? rt - ftiles : rt);
                total = 2u * static_cast<unsigned>(st.kp[s]);
            } else {
                ctr = a.counters + rt;
                total = static_cast<unsigned>(st.items_per_rt);
            }
            // The completing warp reads the partials with L2-coherent ld.cg
            // after observing the final count (no L1-invalidating acquire
            // fence: every value it reads was written by other SMs to L2).
            if (atom_add_release(ctr, static_cast<unsigned>(run_len)) + run_len == total) {
                *ctr = 0;
                last = 1;
            }
        }
        last = __shfl_sync(0xffffffffu, last, 0);
        ++n_runs;
        if (last) {
            ++n_epi;
            if (!a.down)
                epilogue_gateup(a, st, s, rt >= a.f / 16 ? rt - a.f / 16 : rt, lane);
            else
                epilogue_down(a, st, rt, lane);
        }
    }
    unsigned long long* tr = g_gemv_trace;
    if (tr != nullptr && lane == 0) {
        tr += (static_cast<size_t>(a.down) * gridDim.x * kWarps + static_cast<size_t>(wid)) * 8;
        tr[0] = t_entry;
        tr[1] = t_wait;
        tr[2] = t_first;
        tr[3] = gtimer();
        tr[4] = static_cast<unsigned long long>(i1 - i0);
        tr[5] = static_cast<unsigned long long>(n_runs);
        tr[6] = static_cast<unsigned long long>(n_epi);
        tr[7] = static_cast<unsigned long long>(blockIdx.x);
    }
}

// x (natural, [rows][K]) -> K-permuted copy + per-128-group sums (fixed
// xor-butterfly order).  One warp per (row, group); lane owns 4 elements.
__global__ void permute_rows_kernel(const uint16_t* __restrict__ x, int rows, int K, uint16_t* __restrict__ xp,
                                    float* __restrict__ xsum) {
    const int G = K / 128;
    const long long wid = (static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    pdl_wait();     // x is the previous layer's output
    pdl_trigger();
    if (wid >= static_cast<long long>(rows) * G) return;
    const long long r = wid / G;
    const int g = static_cast<int>(wid - r * G);
    const uint16_t* src = x + r * K + g * 128 + lane * 4;
    uint16_t* dst = xp + r * K + g * 128;
    float s = 0.0f;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
        const uint16_t v = src[j];
        dst[perm_k(lane * 4 + j)] = v;
        s += bf2f(v);
    }
#pragma unroll
    for (int off = 16; off >= 1; off >>= 1) s += __shfl_xor_sync(0xffffffffu, s, off);
    if (lane == 0) xsum[r * G + g] = s;
}

int host_pick_gk(int G, int maxgk) {
    for (int g = maxgk; g > 1; g >>= 1)
        if (G % g == 0) return g;
    return 1;
}

cudaError_t launch_pass(GemvArgs& a, cudaStream_t stream) {
    static int grid = 0;
    const size_t smem = static_cast<size_t>(kWarps) * kStages * kStageBytes;
    if (grid == 0) {
        MOE_CUDA_OK(cudaFuncSetAttribute(gemv_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
        int dev = 0, sms = 0;
        MOE_CUDA_OK(cudaGetDevice(&dev));
        MOE_CUDA_OK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
        grid = sms;
    }
    const int G = a.K / 128;
    a.gk4 = host_pick_gk(G, 8);
    a.gk16 = host_pick_gk(G, 2);
    return launch_pdl(gemv_kernel, dim3(grid), dim3(kThreads), smem, stream, a);
}

}  // namespace moek

namespace {

size_t align256(size_t v) { return (v + 255) / 256 * 256; }

struct WsSizes {
    size_t xperm, xsum, hperm, hsum16, hsum, part, counters, gcounters;
};

WsSizes ws_sizes(int T, int k, int d, int f) {
    const size_t slots = static_cast<size_t>(T) * k;
    WsSizes w;
    w.xperm = static_cast<size_t>(T) * d * 2;
    w.xsum = static_cast<size_t>(T) * (d / 128) * 4;
    w.hperm = slots * f * 2;
    w.hsum16 = slots * (f / 16) * 4;
    w.hsum = slots * (f / 128) * 4;
    // K-parts per pass <= number of 128-K groups
    const size_t gu = static_cast<size_t>(d / 128) * slots * 2 * f;
    const size_t dn = static_cast<size_t>(f / 128) * slots * d;
    w.part = (gu > dn ? gu : dn) * 4;
    const size_t cgu = static_cast<size_t>(moek::kMaxSegs) * (f / 16);
    const size_t cdn = static_cast<size_t>(d) / 16;
    w.counters = (cgu > cdn ? cgu : cdn) * 4;
    w.gcounters = static_cast<size_t>(moek::kMaxSegs) * (f / 128) * 4;
    return w;
}

}  // namespace

cudaError_t moek_debug_gemv_trace(void* buf) {
    return cudaMemcpyToSymbol(moek::g_gemv_trace, &buf, sizeof(buf));
}

size_t moek_gemv_workspace_bytes(int T, int k, int d, int f) {
    const WsSizes w = ws_sizes(T, k, d, f);
    return align256(w.xperm) + align256(w.xsum) + align256(w.hperm) + align256(w.hsum16) + align256(w.hsum) +
           align256(w.part) + align256(w.counters) + align256(w.gcounters);
}

GemvWorkspace moek_gemv_workspace_view(void* base, int T, int k, int d, int f) {
    const WsSizes w = ws_sizes(T, k, d, f);
    char* p = static_cast<char*>(base);
    GemvWorkspace ws{};
    ws.xperm = p;
    p += align256(w.xperm);
    ws.xsum = reinterpret_cast<float*>(p);
    p += align256(w.xsum);
    ws.hperm = p;
    p += align256(w.hperm);
    ws.hsum16 = reinterpret_cast<float*>(p);
    p += align256(w.hsum16);
    ws.hsum = reinterpret_cast<float*>(p);
    p += align256(w.hsum);
    ws.part = reinterpret_cast<float*>(p);
    p += align256(w.part);
    ws.counters = reinterpret_cast<unsigned int*>(p);
    p += align256(w.counters);
    ws.gcounters = reinterpret_cast<unsigned int*>(p);
    return ws;
}

cudaError_t moek_permute_rows(const void* x, int rows, int K, void* xperm, float* xsum, cudaStream_t stream) {
    const long long warps = static_cast<long long>(rows) * (K / 128);
    if (warps == 0) return cudaSuccess;
    return moek::launch_pdl(moek::permute_rows_kernel, dim3(static_cast<unsigned>((warps * 32 + 255) / 256)), dim3(256),
                            0, stream, static_cast<const uint16_t*>(x), rows, K, static_cast<uint16_t*>(xperm), xsum);
}

cudaError_t moek_ffn_mma(const GemvWorkspace& ws, const void* x, const int32_t* perm, const int32_t* offsets,
                         const int32_t* inv, const float* wts, const void* resid, int T, int k,
                         const moe_expert_weights* experts, int E, int d, int f, uint64_t active_mask, void* out,
                         float* y, bool xperm_ready, cudaStream_t stream) {
    if (!xperm_ready) MOE_CUDA_OK(moek_permute_rows(x, T, d, ws.xperm, ws.xsum, stream));
    moek::GemvArgs a{};
    a.offsets = offsets;
    a.perm = perm;
    a.T = T;
    a.k = k;
    a.kshift = (k & (k - 1)) == 0 ? __builtin_ctz(static_cast<unsigned>(k)) : -1;
    a.E = E;
    a.active_mask = active_mask;
    for (int e = 0; e < E; ++e) a.ex[e] = experts[e];
    a.part = ws.part;
    a.counters = ws.counters;
    a.gcounters = ws.gcounters;
    a.f = f;
    // gate/up pass: [2f, d] x xperm -> hperm (fused SwiGLU + h group sums)
    a.rows = 2 * f;
    a.K = d;
    a.down = 0;
    a.bperm = static_cast<const uint16_t*>(ws.xperm);
    a.bsum = ws.xsum;
    a.hperm = static_cast<uint16_t*>(ws.hperm);
    a.hsum16 = ws.hsum16;
    a.hsum = ws.hsum;
    MOE_CUDA_OK(moek::launch_pass(a, stream));
    // down pass: [d, f] x hperm -> combine (or per-slot y)
    a.rows = d;
    a.K = f;
    a.down = 1;
    a.bperm = static_cast<const uint16_t*>(ws.hperm);
    a.bsum = ws.hsum;
    a.wts = wts;
    a.inv = inv;
    a.resid = static_cast<const uint16_t*>(resid);
    a.out = static_cast<uint16_t*>(out);
    a.y = y;
    return moek::launch_pass(a, stream);
}
