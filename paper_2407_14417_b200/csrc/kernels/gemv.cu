// gemv.cu -- K3/K4 expert-FFN GEMV for decode batches (<= 8 tokens per
// expert): int4-g128 and bf16 experts, mixed in one launch.
//
// Replaces the constant compute latency of the reference's MoE-layer
// stand-in (simulator.cpp:31-32, :107) with the expert math of HF
// MixtralExperts (modeling_mixtral.py:90-95).
//
// Weights live in HBM as 16-row x 128-K "fragment blocks" (oracle
// orc_pack_*_blocks): one 128-bit load per lane per 512-byte block part gives
// each lane exactly its mma.m16n8k16 A fragments, so every warp load is one
// fully used 512-byte transaction.  int4 fragments are decoded in registers
// (LOP3 magic-number -> bf16 128+u, one bf16x2 FMA -> q exactly); the tensor
// core does the multiply-accumulate (fp32), the per-group scale is applied
// after each 128-K group: y += s * sum(q*x), i.e. exact dequant values q*s.
// Activations are read in the same K permutation (xperm / hperm) so the B
// fragments are 128-bit loads too; up to 8 tokens of an expert share every
// weight byte (the n=8 MMA columns).
//
// Work decomposition: items = (segment, 16-row tile, K-part) with K-parts of
// equal bytes (int4: 8 groups, bf16: 2 groups).  The item space is cut into
// equal contiguous ranges, one per warp of a persistent grid; a warp
// accumulates consecutive K-parts of a row tile in registers ("runs") and
// writes one fp32 partial per run.  Per-tile arrival counters elect the last
// warp, which reduces the runs in fixed K order (deterministic) and runs the
// fused epilogue: SwiGLU + bf16 rounding of h (gate/up pass) or the
// routing-weighted combine + residual (down pass).
#include "common.cuh"
#include "launch.h"

namespace moek {

constexpr int kGemvThreads = 256;
constexpr int kGemvWarps = kGemvThreads / 32;
constexpr int kTile = 8;      // tokens per segment tile (MMA n)
constexpr int kMaxSegs = 256;

struct GemvArgs {
    const int32_t* offsets;   // [E+1]
    const int32_t* perm;      // [T*k]: slot -> t*k + j
    int T, k, E;
    int rows, K;              // matrix rows / columns
    int down;                 // 0 gate/up pass, 1 down pass
    int gk4, gk16;            // groups per K-part (int4, bf16)
    const uint16_t* bperm;    // B operand, K-permuted: [T][K] (gate/up) or [T*k][K] (down)
    float* part;              // partial sums [kp_stride][T*k][rows]
    int kp_stride;
    unsigned int* counters;   // arrival counters (zeroed; reset by the last arriver)
    // gate/up epilogue
    uint16_t* hperm;          // [T*k][f] K-permuted h
    int f;
    // down epilogue
    const float* wts;         // [T*k] routing weights
    const int32_t* inv;       // [T*k]
    const uint16_t* resid;    // [T][d] or null
    uint16_t* out;            // [T][d]; null -> write y
    float* y;                 // [T*k][d] (when out == null)
    uint64_t active_mask;
    moe_expert_weights ex[MOE_MAX_EXPERTS];
};

struct SegTable {
    int n;
    int e[kMaxSegs];
    int tile[kMaxSegs];
    int kp[kMaxSegs];
    long long pre[kMaxSegs + 1];
};

MOE_DEVI int ktile_groups(const GemvArgs& a, int prec) { return prec == MOE_P4 ? a.gk4 : a.gk16; }

// Segments = (expert, tile of <= 8 tokens) of the active experts, in expert
// order; items per segment = (rows/16) * KP.
MOE_DEVI void build_segs(const GemvArgs& a, SegTable& st) {
    if (threadIdx.x == 0) {
        const int RT = a.rows / 16, G = a.K / 128;
        int n = 0;
        long long acc = 0;
        for (int e = 0; e < a.E; ++e) {
            if (!((a.active_mask >> e) & 1ull)) continue;
            const int m = a.offsets[e + 1] - a.offsets[e];
            const int kp = G / ktile_groups(a, a.ex[e].precision);
            for (int t = 0; t * kTile < m && n < kMaxSegs; ++t) {
                st.e[n] = e;
                st.tile[n] = t;
                st.kp[n] = kp;
                st.pre[n] = acc;
                acc += static_cast<long long>(RT) * kp;
                ++n;
            }
        }
        st.pre[n] = acc;
        st.n = n;
    }
    __syncthreads();
}

MOE_DEVI long long ceil_div(long long a, long long b) { return (a + b - 1) / b; }

// Number of runs covering item range [lo, hi) when N items are cut into W
// equal ranges start(w) = floor(w*N/W).
MOE_DEVI int runs_in(long long lo, long long hi, long long N, long long W) {
    return 1 + static_cast<int>(ceil_div(hi * W, N) - ceil_div((lo + 1) * W, N));
}

MOE_DEVI bool is_run_start(long long i, long long lo, long long N, long long W) {
    if (i == lo) return true;
    const long long w = ceil_div(i * W, N);
    return w < W && (w * N) / W == i;
}

MOE_DEVI uint4 ld_b(const uint16_t* p) { return *reinterpret_cast<const uint4*>(p); }

MOE_DEVI void mma_bf16(float (&c)[4], uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3, uint32_t b0,
                       uint32_t b1) {
    asm volatile(
        "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
        "{%0,%1,%2,%3};"
        : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
        : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}

// exact q (bf16x2) from a packed word: four pairs for MMAs kk=2q (p01, p23)
// and kk=2q+1 (p45, p67)
MOE_DEVI void decode_q(uint32_t w, uint32_t& p01, uint32_t& p23, uint32_t& p45, uint32_t& p67) {
    constexpr uint32_t one2 = 0x3F803F80u, m136 = 0xC308C308u;
    p01 = hfma2_bf16(and_or(w, 0x000F000Fu, 0x43004300u), one2, m136);
    p23 = hfma2_bf16(and_or(w >> 4, 0x000F000Fu, 0x43004300u), one2, m136);
    p45 = hfma2_bf16(and_or(w >> 8, 0x000F000Fu, 0x43004300u), one2, m136);
    p67 = hfma2_bf16(and_or(w >> 12, 0x000F000Fu, 0x43004300u), one2, m136);
}

// One int4 item: GK groups of a 16-row tile, C += sum_g s_g * (A_g . B_g).
template <int GKMAX>
MOE_DEVI void item_int4(const uint8_t* wblk, const uint16_t* sblk, int gk, const uint16_t* bp, bool bvalid,
                        int lane, float (&acc)[4]) {
    uint4 wq[GKMAX][2];
    uint32_t sc[GKMAX];
#pragma unroll
    for (int g = 0; g < GKMAX; ++g) {
        if (g < gk) {
            wq[g][0] = ld_stream(wblk + static_cast<size_t>(g) * 1024 + lane * 16);
            wq[g][1] = ld_stream(wblk + static_cast<size_t>(g) * 1024 + 512 + lane * 16);
            sc[g] = __ldg(reinterpret_cast<const uint32_t*>(sblk + static_cast<size_t>(g) * 16) + (lane >> 2));
        }
    }
    const int t = lane & 3;
#pragma unroll
    for (int g = 0; g < GKMAX; ++g) {
        if (g >= gk) break;
        uint4 b[4];
#pragma unroll
        for (int c = 0; c < 4; ++c)
            b[c] = bvalid ? ld_b(bp + static_cast<size_t>(g) * 128 + t * 32 + c * 8) : make_uint4(0, 0, 0, 0);
        float cg[4] = {0.f, 0.f, 0.f, 0.f};
        const uint32_t lo[4] = {wq[g][0].x, wq[g][0].y, wq[g][0].z, wq[g][0].w};
        const uint32_t hi[4] = {wq[g][1].x, wq[g][1].y, wq[g][1].z, wq[g][1].w};
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            uint32_t r0, r2, r0b, r2b, s0, s2, s0b, s2b;
            decode_q(lo[q], r0, r2, r0b, r2b);   // row gr
            decode_q(hi[q], s0, s2, s0b, s2b);   // row gr+8
            mma_bf16(cg, r0, s0, r2, s2, b[q].x, b[q].y);
            mma_bf16(cg, r0b, s0b, r2b, s2b, b[q].z, b[q].w);
        }
        const float s_lo = bf16_lo(sc[g]), s_hi = bf16_hi(sc[g]);
        acc[0] = __fmaf_rn(s_lo, cg[0], acc[0]);
        acc[1] = __fmaf_rn(s_lo, cg[1], acc[1]);
        acc[2] = __fmaf_rn(s_hi, cg[2], acc[2]);
        acc[3] = __fmaf_rn(s_hi, cg[3], acc[3]);
    }
}

// One bf16 item: GK groups, A fragments straight from memory.
template <int GKMAX>
MOE_DEVI void item_bf16(const uint8_t* wblk, int gk, const uint16_t* bp, bool bvalid, int lane,
                        float (&acc)[4]) {
    uint4 wv[GKMAX][8];
#pragma unroll
    for (int g = 0; g < GKMAX; ++g)
        if (g < gk)
#pragma unroll
            for (int p = 0; p < 8; ++p) wv[g][p] = ld_stream(wblk + static_cast<size_t>(g) * 4096 + p * 512 + lane * 16);
    const int t = lane & 3;
#pragma unroll
    for (int g = 0; g < GKMAX; ++g) {
        if (g >= gk) break;
#pragma unroll
        for (int c = 0; c < 4; ++c) {
            const uint4 b = bvalid ? ld_b(bp + static_cast<size_t>(g) * 128 + t * 32 + c * 8) : make_uint4(0, 0, 0, 0);
            // part c = row gr words for kk=2c,2c+1; part 4+c = row gr+8
            mma_bf16(acc, wv[g][c].x, wv[g][4 + c].x, wv[g][c].y, wv[g][4 + c].y, b.x, b.y);
            mma_bf16(acc, wv[g][c].z, wv[g][4 + c].z, wv[g][c].w, wv[g][4 + c].w, b.z, b.w);
        }
    }
}

// K-permuted position of natural index n (orc_perm_k)
MOE_DEVI int perm_k(int n) {
    const int kin = n & 127;
    return (n & ~127) + ((kin & 7) >> 1) * 32 + (kin >> 4) * 4 + ((kin >> 3) & 1) * 2 + (kin & 1);
}

// reduce the fp32 partial runs of (segment s, row) for one slot
MOE_DEVI float reduce_runs(const GemvArgs& a, const SegTable& st, int s, int rt, int row, int slot,
                           long long N, long long W) {
    const int KP = st.kp[s];
    const long long lo = st.pre[s] + static_cast<long long>(rt) * KP;
    const int nslots = a.T * a.k;
    float v = 0.0f;
    for (int kp = 0; kp < KP; ++kp)
        if (is_run_start(lo + kp, lo, N, W))
            v += __ldcg(a.part + (static_cast<size_t>(kp) * nslots + slot) * a.rows + row);
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

// gate/up epilogue for pair tile prt of segment s: h = bf16(silu(g) * u)
MOE_DEVI void epilogue_gateup(const GemvArgs& a, const SegTable& st, int s, int prt, long long N, long long W,
                              int lane) {
    const int e = st.e[s];
    const int slot0 = a.offsets[e] + st.tile[s] * kTile;
    const int m_cnt = min(kTile, a.offsets[e + 1] - slot0);
    const int ftiles = a.f / 16;
    for (int i = lane; i < m_cnt * 16; i += 32) {
        const int m = i >> 4, rr = i & 15;
        const int n = prt * 16 + rr, slot = slot0 + m;
        const float g = reduce_runs(a, st, s, prt, n, slot, N, W);
        const float u = reduce_runs(a, st, s, prt + ftiles, a.f + n, slot, N, W);
        a.hperm[static_cast<size_t>(slot) * a.f + perm_k(n)] = f2bf(silu_f(g) * u);
    }
}

// down epilogue for row tile rt: y per slot (reduced runs), then combine
MOE_DEVI void epilogue_down(const GemvArgs& a, const SegTable& st, int rt, long long N, long long W, int lane) {
    const int d = a.rows;
    if (a.out == nullptr) {
        const int nslots = a.T * a.k;
        for (int i = lane; i < nslots * 16; i += 32) {
            const int slot = i >> 4, j = rt * 16 + (i & 15);
            const int s = seg_of_slot(a, st, slot);
            if (s < 0) continue;
            a.y[static_cast<size_t>(slot) * d + j] = reduce_runs(a, st, s, rt, j, slot, N, W);
        }
        return;
    }
    for (int i = lane; i < a.T * 16; i += 32) {
        const int t = i >> 4, j = rt * 16 + (i & 15);
        float accv = a.resid ? bf2f(a.resid[static_cast<size_t>(t) * d + j]) : 0.0f;
        for (int jj = 0; jj < a.k; ++jj) {
            const int slot = a.inv[t * a.k + jj];
            const int s = seg_of_slot(a, st, slot);
            const float yv = s < 0 ? 0.0f : reduce_runs(a, st, s, rt, j, slot, N, W);
            accv = __fmaf_rn(a.wts[t * a.k + jj], yv, accv);
        }
        a.out[static_cast<size_t>(t) * d + j] = f2bf(accv);
    }
}

template <int GK4, int GK16>
__global__ void __launch_bounds__(kGemvThreads) gemv_kernel(const __grid_constant__ GemvArgs a) {
    __shared__ SegTable st;
    build_segs(a, st);
    const int lane = threadIdx.x & 31;
    const long long W = static_cast<long long>(gridDim.x) * kGemvWarps;
    const long long wid = static_cast<long long>(blockIdx.x) * kGemvWarps + (threadIdx.x >> 5);
    const long long N = st.pre[st.n];
    if (N == 0) return;
    long long i = wid * N / W;
    const long long i_end = (wid + 1) * N / W;
    if (i >= i_end) return;
    const int nslots = a.T * a.k;
    const int gr = lane >> 2, t = lane & 3;
    const int G = a.K / 128;
    const int RT = a.rows / 16;
    int s = 0;
    while (st.pre[s + 1] <= i) ++s;

    while (i < i_end) {
        const int e = st.e[s];
        const moe_expert_weights& Wt = a.ex[e];
        const int prec = Wt.precision;
        const int KP = st.kp[s];
        const int gk = G / KP;
        const long long local = i - st.pre[s];
        const int rt = static_cast<int>(local / KP);
        int kp = static_cast<int>(local - static_cast<long long>(rt) * KP);
        const int kp0 = kp;
        const int slot0 = a.offsets[e] + st.tile[s] * kTile;
        const int m_cnt = min(kTile, a.offsets[e + 1] - slot0);
        // B row for this lane's MMA column gr
        const bool bvalid = gr < m_cnt;
        int brow = 0;
        if (bvalid) brow = a.down ? slot0 + gr : a.perm[slot0 + gr] / a.k;
        const uint16_t* brow_p = a.bperm + static_cast<size_t>(brow) * a.K;
        const uint8_t* wbase = static_cast<const uint8_t*>(a.down ? Wt.w_down : Wt.w_gate_up);
        const uint16_t* sbase = static_cast<const uint16_t*>(a.down ? Wt.s_down : Wt.s_gate_up);
        float acc[4] = {0.f, 0.f, 0.f, 0.f};
        for (; kp < KP && i < i_end; ++kp, ++i) {
            const size_t blk = static_cast<size_t>(rt) * G + static_cast<size_t>(kp) * gk;
            const uint16_t* bp = brow_p + static_cast<size_t>(kp) * gk * 128;
            if (prec == MOE_P4)
                item_int4<GK4>(wbase + blk * 1024, sbase + blk * 16, gk, bp, bvalid, lane, acc);
            else
                item_bf16<GK16>(wbase + blk * 4096, gk, bp, bvalid, lane, acc);
        }
        // flush the run: C columns 2t, 2t+1 = tokens of the tile; rows gr, gr+8
        const int row = rt * 16 + gr;
#pragma unroll
        for (int c = 0; c < 2; ++c) {
            const int m = 2 * t + c;
            if (m < m_cnt) {
                float* p = a.part + (static_cast<size_t>(kp0) * nslots + slot0 + m) * a.rows;
                p[row] = acc[c];
                p[row + 8] = acc[2 + c];
            }
        }
        __threadfence();
        __syncwarp();
        // arrival
        int last = 0;
        if (lane == 0) {
            if (!a.down) {
                const int ftiles = a.f / 16;
                const int prt = rt % ftiles;
                const long long lo_g = st.pre[s] + static_cast<long long>(prt) * KP;
                const long long lo_u = st.pre[s] + static_cast<long long>(prt + ftiles) * KP;
                const int need = runs_in(lo_g, lo_g + KP, N, W) + runs_in(lo_u, lo_u + KP, N, W);
                unsigned int* ctr = a.counters + static_cast<size_t>(s) * ftiles + prt;
                if (atomicAdd(ctr, 1u) + 1 == static_cast<unsigned>(need)) {
                    *ctr = 0;
                    last = 1;
                }
            } else {
                int need = 0;
                for (int ss = 0; ss < st.n; ++ss) {
                    const long long lo = st.pre[ss] + static_cast<long long>(rt) * st.kp[ss];
                    need += runs_in(lo, lo + st.kp[ss], N, W);
                }
                unsigned int* ctr = a.counters + rt;
                if (atomicAdd(ctr, 1u) + 1 == static_cast<unsigned>(need)) {
                    *ctr = 0;
                    last = 1;
                }
            }
        }
        last = __shfl_sync(0xffffffffu, last, 0);
        if (last) {
            __threadfence();
            if (!a.down)
                epilogue_gateup(a, st, s, rt % (a.f / 16), N, W, lane);
            else
                epilogue_down(a, st, rt, N, W, lane);
        }
        if (i < i_end && i >= st.pre[s + 1]) ++s;
        (void)RT;
    }
}

// x (natural, [T][K]) -> xperm (K-permuted per 128-group), one thread per
// 8 elements of output
__global__ void permute_rows_kernel(const uint16_t* __restrict__ x, int rows, int K, uint16_t* __restrict__ xp) {
    const long long n = static_cast<long long>(rows) * K;
    for (long long o = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x; o < n;
         o += static_cast<long long>(gridDim.x) * blockDim.x) {
        const long long r = o / K;
        const int c = static_cast<int>(o - r * K);
        xp[r * K + perm_k(c)] = x[o];
    }
}

template <int GK4, int GK16>
cudaError_t launch_gemv(const GemvArgs& a, cudaStream_t stream) {
    static int grid = 0;
    if (grid == 0) {
        int dev = 0, sms = 0, occ = 0;
        MOE_CUDA_OK(cudaGetDevice(&dev));
        MOE_CUDA_OK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
        MOE_CUDA_OK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, gemv_kernel<GK4, GK16>, kGemvThreads, 0));
        grid = sms * (occ > 0 ? occ : 1);
    }
    gemv_kernel<GK4, GK16><<<grid, kGemvThreads, 0, stream>>>(a);
    return cudaGetLastError();
}

int pick_gk(int G, int maxgk) {
    for (int g = maxgk; g > 1; g >>= 1)
        if (G % g == 0) return g;
    return 1;
}

cudaError_t launch_pass(GemvArgs& a, cudaStream_t stream) {
    const int G = a.K / 128;
    a.gk4 = pick_gk(G, 4);
    a.gk16 = pick_gk(G, 2);
    if (a.gk4 == 4) return launch_gemv<4, 2>(a, stream);
    return launch_gemv<2, 2>(a, stream);
}

}  // namespace moek

size_t moek_gemv_partial_floats(int T, int k, int d, int f) {
    // K-parts per matrix are at most G/1 for bf16 with gk16 = 1; size for the
    // worst case (gk16 >= 1 -> KP <= G).
    const size_t slots = static_cast<size_t>(T) * k;
    const size_t gu = static_cast<size_t>(d / 128) * slots * 2 * f;
    const size_t dn = static_cast<size_t>(f / 128) * slots * d;
    return gu > dn ? gu : dn;
}

size_t moek_gemv_counter_count(int T, int E, int d, int f) {
    const size_t segs = static_cast<size_t>(E) * ((T + moek::kTile - 1) / moek::kTile);
    const size_t gu = segs * (f / 16);
    const size_t dn = static_cast<size_t>(d) / 16;
    return gu > dn ? gu : dn;
}

cudaError_t moek_permute_rows(const void* x, int rows, int K, void* xperm, cudaStream_t stream) {
    const long long n = static_cast<long long>(rows) * K;
    if (n == 0) return cudaSuccess;
    long long blocks = (n + 255) / 256;
    if (blocks > 148 * 16) blocks = 148 * 16;
    moek::permute_rows_kernel<<<static_cast<unsigned>(blocks), 256, 0, stream>>>(
        static_cast<const uint16_t*>(x), rows, K, static_cast<uint16_t*>(xperm));
    return cudaGetLastError();
}

cudaError_t moek_ffn_mma(const GemvWorkspace& ws, const void* x, const int32_t* perm, const int32_t* offsets,
                         const int32_t* inv, const float* wts, const void* resid, int T, int k,
                         const moe_expert_weights* experts, int E, int d, int f, uint64_t active_mask, void* out,
                         float* y, bool xperm_ready, cudaStream_t stream) {
    if (!xperm_ready) MOE_CUDA_OK(moek_permute_rows(x, T, d, ws.xperm, stream));
    moek::GemvArgs a{};
    a.offsets = offsets;
    a.perm = perm;
    a.T = T;
    a.k = k;
    a.E = E;
    a.active_mask = active_mask;
    for (int e = 0; e < E; ++e) a.ex[e] = experts[e];
    a.part = ws.part;
    a.counters = ws.counters;
    a.f = f;
    // gate/up pass: [2f, d] x xperm -> hperm
    a.rows = 2 * f;
    a.K = d;
    a.down = 0;
    a.bperm = static_cast<const uint16_t*>(ws.xperm);
    a.hperm = static_cast<uint16_t*>(ws.hperm);
    MOE_CUDA_OK(moek::launch_pass(a, stream));
    // down pass: [d, f] x hperm -> combine (or y)
    a.rows = d;
    a.K = f;
    a.down = 1;
    a.bperm = static_cast<const uint16_t*>(ws.hperm);
    a.wts = wts;
    a.inv = inv;
    a.resid = static_cast<const uint16_t*>(resid);
    a.out = static_cast<uint16_t*>(out);
    a.y = y;
    return moek::launch_pass(a, stream);
}
