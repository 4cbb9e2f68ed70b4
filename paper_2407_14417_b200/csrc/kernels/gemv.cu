// gemv.cu -- K3/K4 expert-FFN GEMV for decode batches (<= 8 tokens per
// expert segment): int4-g128 and bf16 experts, mixed in one launch.
//
// Replaces the constant compute latency of the reference's MoE-layer
// stand-in (simulator.cpp:31-32, :107) with the expert math of HF
// MixtralExperts (modeling_mixtral.py:90-95).
//
// Per layer (all launches PDL-chained on one stream, one CUDA graph):
//   permute_rows   x -> K-permuted bf16/fp16 copies + int4 bias terms
//   stream<0>      gate/up rows of every selected expert x x  -> fp32 partials
//   finalize_h     partials -> SwiGLU -> h (bf16 + fp16 copies + bias terms)
//   stream<1>      down rows x h -> fp32 partials
//   finalize_out   partials -> routing-weighted combine + residual -> out
//
// stream: HBM --cp.async.bulk (TMA bulk copy, mbarrier complete_tx)--> a
// per-warp shared-memory ring --LDS.128--> mma.m16n8k16 fragments.  A work
// item = (16-row tile, K-part of GK 128-K groups) of one expert segment: one
// bulk copy of its weight blocks (+ one of its int4 scales) plus one per
// token row of the matching activation slice (+ its int4 bias terms), all
// completing on the stage's mbarrier, kStages items ahead of use.  The warp
// never waits on anything but its ring: no global loads, no atomics, no
// epilogue -- each item ends in plain stores of its fp32 partial (one slot
// per K-part, so the finalize sums in a fixed order: bit-reproducible under
// any schedule).  Items are statically partitioned into contiguous warp
// ranges, except a tail pool handed out in small chunks from a global
// counter so the warps that run fast absorb the imbalance.
//
// Weights are stored as 16-row x 128-K "fragment blocks" (oracle
// orc_pack_*_blocks): a lane's 16-byte smem read is exactly one A operand
// (bf16) or the 8 nibble pairs of one row half (int4).  int4 is decoded in
// registers with the fp16 magic number (0x6400 | nibble -> 1024+u or
// 1024+16u: 4 LOP3 + 1 SHF per 8 weights) and multiplied on the tensor core
// against an fp16 copy of the activations (exact for 2^-17 <= |x| <= 65504);
// the per-128-K-group scale is applied after the group's integer-exact dot,
// y += s * sum(q*x) -- the exact dequant values q*s.
#include <algorithm>
#include <cstdio>
#include <cstdlib>

#include "common.cuh"
#include "launch.h"
#include "route_common.cuh"

namespace moek {

constexpr int kStages = 2;
constexpr int kTile = 8;                 // tokens per segment tile (MMA n)
constexpr int kMaxSegs = 64;             // (active expert, 8-token tile) segments per launch
constexpr int kBRowPad = 64;             // activation row stride in a stage = GK*256 + 64: conflict-free LDS.128

// Stream-kernel configurations.  Stage layout: [weights <= W][int4 scales
// <= W/32][activation rows <= B][bias terms 8 x 32 B].
//   Batch : 8 warps, 8 KB weight items; activation area for up to 8 token
//           rows (GK shrinks with the rows: m * (GK*256+64) <= B).
//   Decode: 8 warps, 8 KB weight items; T == 1 (one token row per segment,
//           <= 2 segments, rows of K <= 14336): the rows are resident per CTA.
template <int WARPS, int W, int B, bool RES = false>
struct StreamCfg {
    static constexpr bool kRes = RES;     // activations resident per CTA (T == 1), not per item
    static constexpr int kResBytes = RES ? 2 * (14336 * 2 + 512 * 4) : 0;  // 2 segments x (row of K <= 14336 + bias)
    static constexpr int kWarps = WARPS;
    static constexpr int kThreads = WARPS * 32;
    static constexpr int kW = W;
    static constexpr int kS = W / 32;
    static constexpr int kBBytes = B;
    static constexpr int kStageW = 0;
    static constexpr int kStageS = W;
    static constexpr int kStageB = W + W / 32;
    static constexpr int kStageX = kStageB + B;
    static constexpr int kStageBytes = (kStageX + kTile * 32 + 127) / 128 * 128;
    static constexpr int kGk4 = W / 1024;   // max 128-K groups per int4 item
    static constexpr int kGk16 = W / 4096;  // max 128-K groups per bf16 item
};
using CfgBatch = StreamCfg<8, 8192, 4608>;
// batch-1 decode: each segment's single activation row (and its int4 bias
// terms) is loaded once per launch into shared memory; items carry only weights
#ifndef MOE_DECODE_ITEM
#define MOE_DECODE_ITEM 8192  // bytes of weights per batch-1 item (A/B: 4096)
#endif
using CfgDecode = StreamCfg<8, MOE_DECODE_ITEM, 0, true>;
constexpr int kChunk = 2;                // items per dynamic tail chunk
constexpr int kSmallPool = 5000;         // pools up to this many items are handed out one item per grab
constexpr int kMaxSlots = 512;           // permutation slots staged in smem by build_segs

struct StreamArgs {
    const int32_t* offsets;   // [E+1]
    const int32_t* perm;      // [T*k]: slot -> t*k + j
    int T, k, E;
    int kshift;               // log2(k) (-1: not a power of two)
    int p;                    // 0: gate/up rows against x, 1: down rows against h
    int rows, K;              // this pass's matrix shape
    const uint16_t* b16;      // B operand for bf16 experts, K-permuted (perm_k): [rows of B][K]
    const uint16_t* b16h;     // fp16 copy for int4 experts (perm_k16)
    const float* bsum;        // int4 bias term per (B row, 128-group), row stride bstride
    int bstride;
    float* part;              // [K/128][T*k][rows]: one fp32 partial per (K-part, slot, row)
    int* kpslot;              // [T*k]: K-parts written for the slot (0: expert not in this launch)
    unsigned int* sched;      // tail-pool counter (reset by the finalize kernel)
    int wait_first;           // 1: the predecessor produced the routing -> PDL wait before reading it
    int dbg;                  // experiments (MOE_GEMV_DBG): bit0 skip activation copies, bit1 skip scale copies
    uint64_t active_mask;
    moe_expert_weights ex[MOE_MAX_EXPERTS];
};

struct SegTable {
    int n, N;
    int e[kMaxSegs];
    int slot0[kMaxSegs];       // first permutation slot of the segment
    int mcnt[kMaxSegs];        // tokens in the segment (<= kTile)
    int kp[kMaxSegs];          // K-parts per row tile
    int gk[kMaxSegs];          // 128-K groups per item
    int wbytes[kMaxSegs];      // bytes of weights per item
    int sbytes[kMaxSegs];      // bytes of int4 scales per item (0: bf16)
    int brow[kMaxSegs][kTile]; // B row of MMA column c (clamped to mcnt-1)
    const uint8_t* wptr[kMaxSegs];
    const uint8_t* sptr[kMaxSegs];
    int pre[kMaxSegs + 1];     // item prefix over segments
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
// bulk copy with an L2 cache-policy hint (evict_first for streamed weights,
// so the partials / activations the finalize kernels re-read stay in L2)
MOE_DEVI void bulk_g2s_hint(void* dst, const void* src, uint32_t bytes, uint64_t* bar, uint64_t pol) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(pol)
        : "memory");
}
MOE_DEVI uint64_t policy_evict_first() {
    uint64_t pol;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    return pol;
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
MOE_DEVI void mma_f16(float (&c)[4], uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3, uint32_t b0,
                      uint32_t b1) {
    asm volatile(
        "mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
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

// One int4 group (16 rows x 128 K, 1024 B at gp + 32 B scales at sc); bp:
// this lane's activation chunks of the group (4 x 16 B at stride 64).
// Nibbles (0,16)/(8,24) of a word hold the K positions with k%16 < 8 ("lo"),
// nibbles (4,20)/(12,28) those with k%16 >= 8 ("hi").  The fp16 magic
// numbers read them as exact values of the same unit: 0x6400 | nibble =
// 1024 + u (lo) and 0x5400 | nibble<<4 = 64 + u (hi, ulp 1/16), u = q + 8,
// so one MMA chain accumulates both and per group
//   sum(q x) = c - (1032 S_lo + 72 S_hi)
// with the bias term precomputed per activation group (B0: column 2t, B1:
// 2t+1) and loaded as the chain's start value.  Then y += s * sum(q x): the
// exact dequant values q*s.  Chunk q of the fp16 activation copy holds the
// K positions of (lo0, lo1, hi0, hi1).
// fp16 magic-number decode of one packed word (4 LOP3 + 1 SHF):
//   lo0: nibbles (0,16) -> 1024+u      hi0: nibbles (4,20) -> 64+u
//   lo1: nibbles (8,24)                hi1: nibbles (12,28)
MOE_DEVI void decode_lohi(uint32_t w, uint32_t& lo0, uint32_t& hi0, uint32_t& lo1, uint32_t& hi1) {
    lo0 = and_or(w, 0x000F000Fu, 0x64006400u);
    hi0 = and_or(w, 0x00F000F0u, 0x54005400u);
    const uint32_t w8 = w >> 8;
    lo1 = and_or(w8, 0x000F000Fu, 0x64006400u);
    hi1 = and_or(w8, 0x00F000F0u, 0x54005400u);
}

MOE_DEVI void group_int4(const uint8_t* gp, const uint8_t* sc, const uint8_t* bp, float B0, float B1, int lane,
                         float (&acc)[4]) {
    const uint32_t s2 = *reinterpret_cast<const uint32_t*>(sc + (lane >> 2) * 4);
    const uint4 wl = lds128(gp + lane * 16);
    const uint4 wh = lds128(gp + 512 + lane * 16);
    const uint32_t lo[4] = {wl.x, wl.y, wl.z, wl.w};
    const uint32_t hi[4] = {wh.x, wh.y, wh.z, wh.w};
    float c[4] = {-B0, -B1, -B0, -B1};
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        const uint4 b = lds128(bp + q * 64);
        uint32_t a_l0, a_h0, a_l1, a_h1, c_l0, c_h0, c_l1, c_h1;
        decode_lohi(lo[q], a_l0, a_h0, a_l1, a_h1);  // row gr
        decode_lohi(hi[q], c_l0, c_h0, c_l1, c_h1);  // row gr+8
        mma_f16(c, a_l0, c_l0, a_l1, c_l1, b.x, b.y);
        mma_f16(c, a_h0, c_h0, a_h1, c_h1, b.z, b.w);
    }
    const float s_lo = bf16_lo(s2), s_hi = bf16_hi(s2);
    acc[0] = __fmaf_rn(s_lo, c[0], acc[0]);
    acc[1] = __fmaf_rn(s_lo, c[1], acc[1]);
    acc[2] = __fmaf_rn(s_hi, c[2], acc[2]);
    acc[3] = __fmaf_rn(s_hi, c[3], acc[3]);
}

// One bf16 group (16 rows x 128 K, 4096 B): part kk (512 B) holds every
// lane's {a0, a1, a2, a3} of MMA kk, so one LDS.128 is one A operand; even
// kk accumulate into acc, odd kk into the second chain c1.  Chunk c of the
// bf16 activation copy holds (kk=2c: k<8, k>=8; kk=2c+1: k<8, k>=8).
// ldmatrix.x4: the four 8x8 core matrices whose row addresses lanes 0-7,
// 8-15, 16-23, 24-31 supply -> one mma.m16n8k16 A fragment {a0, a1, a2, a3}
MOE_DEVI uint4 ldsm_x4(const uint8_t* p) {
    uint4 v;
    asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                 : "r"(static_cast<uint32_t>(__cvta_generic_to_shared(p))));
    return v;
}

// bf16 block in core-matrix order: K slice kk (16 wide) of the
// 16-row block is the core matrices (row half q&1, 8-K column 2*(kk%4) +
// (q>>1)) of K half kk/4; lane l supplies row l&7 of matrix q = l>>3.
MOE_DEVI void group_bf16(const uint8_t* gp, const uint8_t* bp, int lane, float (&acc)[4], float (&c1)[4]) {
    const int q = lane >> 3;
    const uint8_t* lp = gp + (q & 1) * 1024 + (q >> 1) * 128 + (lane & 7) * 16;
#pragma unroll
    for (int c = 0; c < 4; ++c) {
        const uint4 b = lds128(bp + c * 64);
        const int k0 = 2 * c, k1 = 2 * c + 1;  // K slices of this step
        const uint4 e = ldsm_x4(lp + (k0 >> 2) * 2048 + (k0 & 3) * 256);
        const uint4 o = ldsm_x4(lp + (k1 >> 2) * 2048 + (k1 & 3) * 256);
        mma_bf16(acc, e.x, e.y, e.z, e.w, b.x, b.y);
        mma_bf16(c1, o.x, o.y, o.z, o.w, b.z, b.w);
    }
}

// Activation layouts inside a 128-K group (kin = kk*16 + hi*8 + t*2 + e):
// 16-byte chunk (kk/2)*4 + t belongs to lane t, so the 4 lanes of a row read
// 64 contiguous bytes per LDS.128 (conflict-free); inside the chunk
//   bf16 copy (perm_k):   word (kk%2)*2 + hi
//   fp16 copy (perm_k16): word hi*2 + kk%2
MOE_DEVI int perm_k(int n) {
    const int kin = n & 127, kk = kin >> 4;
    return (n & ~127) + ((kk >> 1) * 4 + ((kin & 7) >> 1)) * 8 + ((kk & 1) * 2 + ((kin >> 3) & 1)) * 2 + (kin & 1);
}
MOE_DEVI int perm_k16(int n) {
    const int kin = n & 127, kk = kin >> 4;
    return (n & ~127) + ((kk >> 1) * 4 + ((kin & 7) >> 1)) * 8 + (((kin >> 3) & 1) * 2 + (kk & 1)) * 2 + (kin & 1);
}

// 128-K groups per item: the largest power of two <= cap dividing G, where
// cap keeps m activation rows of the item inside the stage.
template <class C>
MOE_DEVI int pick_gk(int G, int prec, int m) {
    int cap = prec == MOE_P4 ? C::kGk4 : C::kGk16;
    while (!C::kRes && cap > 1 && m * (cap * 256 + kBRowPad) > C::kBBytes) cap >>= 1;  // resident rows: no cap
    while (cap > 1 && G % cap) cap >>= 1;
    return cap;
}

// Segment table (one segment per (active expert, 8-token tile)), built
// redundantly by every CTA from the routing; CTA 0 also publishes each
// slot's K-part count for the finalize kernel.
template <class C>
MOE_DEVI void build_segs(const StreamArgs& a, SegTable& st, int* cnt, int* sperm) {
    // offsets and perm in one round trip
    const int nslots = a.T * a.k;
    int o0 = 0, o1 = 0;
    if (threadIdx.x < a.E) {
        o0 = a.offsets[threadIdx.x];
        o1 = a.offsets[threadIdx.x + 1];
    }
    if (a.p == 0)
        for (int i = threadIdx.x; i < nslots && i < kMaxSlots; i += blockDim.x) sperm[i] = a.perm[i];
    if (threadIdx.x < a.E) {
        cnt[threadIdx.x] = ((a.active_mask >> threadIdx.x) & 1ull) ? o1 - o0 : 0;
        cnt[MOE_MAX_EXPERTS + threadIdx.x] = o0;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        const int RT = a.rows / 16, G = a.K / 128;
        int n = 0, acc = 0;
        for (int e = 0; e < a.E; ++e) {
            const int m = cnt[e];
            if (m == 0) continue;
            const moe_expert_weights& W = a.ex[e];
            for (int t = 0; t * kTile < m && n < kMaxSegs; ++t) {
                const int mc = min(kTile, m - t * kTile);
                const int gk = pick_gk<C>(G, W.precision, mc);
                st.e[n] = e;
                st.slot0[n] = cnt[MOE_MAX_EXPERTS + e] + t * kTile;
                st.mcnt[n] = mc;
                st.kp[n] = G / gk;
                st.gk[n] = gk;
                st.wptr[n] = static_cast<const uint8_t*>(a.p == 0 ? W.w_gate_up : W.w_down);
                st.sptr[n] = static_cast<const uint8_t*>(a.p == 0 ? W.s_gate_up : W.s_down);
                st.wbytes[n] = W.precision == MOE_P4 ? gk * 1024 : gk * 4096;
                st.sbytes[n] = W.precision == MOE_P4 ? gk * 32 : 0;
                st.pre[n] = acc;
                acc += RT * (G / gk);
                ++n;
            }
        }
        st.pre[n] = acc;
        st.n = n;
        st.N = acc;
    }
    __syncthreads();
    for (int i = threadIdx.x; i < st.n * kTile; i += blockDim.x) {
        const int s = i / kTile, c = i - s * kTile;
        const int slot = st.slot0[s] + min(c, st.mcnt[s] - 1);
        const int pv = slot < kMaxSlots ? sperm[slot] : a.perm[slot];
        st.brow[s][c] = a.p == 1 ? slot : (a.kshift >= 0 ? pv >> a.kshift : pv / a.k);
    }
    if (blockIdx.x == 0) {
        for (int slot = threadIdx.x; slot < a.T * a.k; slot += blockDim.x) {
            int kp = 0;
            for (int s = 0; s < st.n; ++s)
                if (slot >= st.slot0[s] && slot < st.slot0[s] + st.mcnt[s]) kp = st.kp[s];
            a.kpslot[slot] = kp;
        }
    }
    __syncthreads();
}

struct Item {
    int s, rt, kp;
};

MOE_DEVI Item item_at(const SegTable& st, int i) {
    Item it;
    it.s = 0;
    while (st.pre[it.s + 1] <= i) ++it.s;
    const int local = i - st.pre[it.s];
    it.rt = local / st.kp[it.s];
    it.kp = local - it.rt * st.kp[it.s];
    return it;
}

// Issue the weight half of an item (expect_tx covers the whole item).
template <class C>
MOE_DEVI void issue_weights(const StreamArgs& a, const SegTable& st, const Item& it, uint8_t* stage, uint64_t* bar,
                            uint64_t pol) {
    const int s = it.s, wb = st.wbytes[s], sb = st.sbytes[s], m = st.mcnt[s];
    const int acts = (C::kRes || (a.dbg & 1)) ? 0 : m * st.gk[s] * 256 + (sb ? m * 32 : 0);
    const int scl = (a.dbg & 2) ? 0 : sb;
    mbar_expect_tx(bar, wb + scl + acts);
    const size_t blk = static_cast<size_t>(it.rt) * (a.K / 128) + static_cast<size_t>(it.kp) * st.gk[s];
    bulk_g2s_hint(stage + C::kStageW, st.wptr[s] + blk * (sb ? 1024 : 4096), wb, bar, pol);
    if (scl) bulk_g2s_hint(stage + C::kStageS, st.sptr[s] + blk * 32, sb, bar, pol);
}

// Issue the activation half: the item's K slice of every token row of the
// segment (fp16 copy for int4, bf16 for bf16) and, for int4, the 32-byte
// bias-term chunk holding the item's groups.
template <class C>
MOE_DEVI void issue_acts(const StreamArgs& a, const SegTable& st, const Item& it, uint8_t* stage, uint64_t* bar) {
    if (C::kRes || (a.dbg & 1)) return;
    const int s = it.s, m = st.mcnt[s], gk = st.gk[s];
    const int rowb = gk * 256;
    const size_t k0 = static_cast<size_t>(it.kp) * gk * 128;
    if (st.sbytes[s]) {
        const int g8 = (it.kp * gk) & ~7;
        for (int r = 0; r < m; ++r) {
            const int br = st.brow[s][r];
            bulk_g2s(stage + C::kStageB + r * (rowb + kBRowPad), a.b16h + static_cast<size_t>(br) * a.K + k0, rowb, bar);
            bulk_g2s(stage + C::kStageX + r * 32, a.bsum + static_cast<size_t>(br) * a.bstride + g8, 32, bar);
        }
    } else {
        for (int r = 0; r < m; ++r)
            bulk_g2s(stage + C::kStageB + r * (rowb + kBRowPad), a.b16 + static_cast<size_t>(st.brow[s][r]) * a.K + k0,
                     rowb, bar);
    }
}

// Item sequence of one warp: its static range, then tail-pool chunks grabbed
// one chunk ahead by lane 0 (the atomic's result is consumed a chunk later).
// The issue side walks it with an incremental (segment, row tile, K-part)
// cursor -- a search only at chunk jumps -- and hands each stage's item to
// the compute side in registers.
struct Sched {
    unsigned int* ctr;
    int N, ns;
    int cur, end;          // current static range / chunk [cur, end)
    int dyn;               // in the tail pool
    unsigned int pend;     // lane 0: pre-grabbed chunk start
    int lane;
    int RT;
    Item it;               // item of index cur-1 (valid once started)
    int started;
    int chunk;             // items per pool grab

    MOE_DEVI void grab_ahead() {
        if (lane == 0) pend = atomicAdd(ctr, static_cast<unsigned>(chunk));
    }
    MOE_DEVI void step(const SegTable& st) {
        if (++it.kp == st.kp[it.s]) {
            it.kp = 0;
            if (++it.rt == RT) {
                it.rt = 0;
                ++it.s;
            }
        }
    }
    MOE_DEVI bool next(const SegTable& st, Item& out) {
        bool jump = !started;
        while (cur >= end) {
            if (!dyn) {
                dyn = 1;
                grab_ahead();
            }
            const int start = ns + static_cast<int>(__shfl_sync(0xffffffffu, pend, 0));
            if (start >= N) return false;
            jump = jump || start != cur;
            cur = start;
            end = min(start + chunk, N);
            grab_ahead();
        }
        if (jump)
            it = item_at(st, cur);
        else
            step(st);
        started = 1;
        ++cur;
        out = it;
        return true;
    }
};

// bp: this lane's activation chunks of the item's first group (groups at
// stride 256 B); x0 / x1: the int4 bias terms of columns 2t / 2t+1 for the
// item's first group.
template <class C>
MOE_DEVI void compute_item(const SegTable& st, const Item& it, const uint8_t* sp, const uint8_t* bp, const float* x0,
                           const float* x1, int lane, float (&acc)[4]) {
    const int gk = st.gk[it.s];
    if (st.sbytes[it.s]) {
        if (C::kGk4 >= 8 && gk == 8) {
#pragma unroll
            for (int g = 0; g < 8; ++g)
                group_int4(sp + C::kStageW + g * 1024, sp + C::kStageS + g * 32, bp + g * 256, x0[g], x1[g], lane, acc);
        } else {
            for (int g = 0; g < gk; ++g)
                group_int4(sp + C::kStageW + g * 1024, sp + C::kStageS + g * 32, bp + g * 256, x0[g], x1[g], lane, acc);
        }
    } else {
        float c1[4] = {0.f, 0.f, 0.f, 0.f};
        group_bf16(sp + C::kStageW, bp, lane, acc, c1);
        if (C::kGk16 >= 2 && gk == 2) group_bf16(sp + C::kStageW + 4096, bp + 256, lane, acc, c1);
#pragma unroll
        for (int r = 0; r < 4; ++r) acc[r] += c1[r];
    }
}

template <class C>
__global__ void __launch_bounds__(C::kThreads, 1) stream_kernel(const __grid_constant__ StreamArgs a) {
    constexpr int kWarps = C::kWarps;
    constexpr int kStageBytes = C::kStageBytes;
    static_assert(kStages == 2, "the per-stage item registers are written for two stages");
    extern __shared__ __align__(128) uint8_t smem[];
    __shared__ SegTable st;
    __shared__ __align__(8) uint64_t bars[kWarps][kStages];
    __shared__ int cnt[2 * MOE_MAX_EXPERTS];
    __shared__ int sperm[kMaxSlots];
    __shared__ __align__(8) uint64_t res_bar;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (lane == 0) {
        for (int s = 0; s < kStages; ++s) mbar_init(&bars[warp][s], 1);
        if (C::kRes && warp == 0) mbar_init(&res_bar, 1);
        fence_mbar_init();
    }
    const unsigned long long t_entry = gtimer();
    unsigned long long* const ltr = g_layer_trace;
    ltrace(ltr, 2 + 2 * a.p, 0);
    // When the routing comes from two or more launches back, the segment
    // table and the first items' weight copies go out before the PDL wait;
    // their activation copies (the predecessor's output) after it.
    // resident activation rows (T == 1 configuration)
    uint8_t* res = smem + static_cast<size_t>(kWarps) * kStages * kStageBytes;
    float* resx = reinterpret_cast<float*>(res + 2 * a.K * 2);
    auto res_pass0 = [&]() {
        // gate/up pass: the one token's row in both formats + its bias terms,
        // issued as soon as the predecessor is complete (before the table)
        if (C::kRes && a.p == 0 && threadIdx.x == 0) {
            mbar_expect_tx(&res_bar, 2 * a.K * 2 + a.bstride * 4);
            bulk_g2s(res, a.b16, a.K * 2, &res_bar);
            bulk_g2s(res + a.K * 2, a.b16h, a.K * 2, &res_bar);
            bulk_g2s(resx, a.bsum, a.bstride * 4, &res_bar);
        }
    };
    if (a.wait_first) {
        pdl_wait();
        if (C::kRes) __syncthreads();  // res_bar initialised
        res_pass0();
    }
    build_segs<C>(a, st, cnt, sperm);  // contains __syncthreads
    const uint64_t pol = policy_evict_first();
    const int W = static_cast<int>(gridDim.x) * kWarps;
    const int wid = static_cast<int>(blockIdx.x) * kWarps + warp;
    const int gr = lane >> 2, t = lane & 3;
    const int nslots = a.T * a.k;
    uint8_t* ring = smem + static_cast<size_t>(warp) * kStages * kStageBytes;

    // static part: contiguous equal ranges over the first ~7/8 of the items
    const int N = st.N;
    // single-item grabs while the pool is small enough for one counter's
    // atomic throughput (int4-heavy launches: a shorter tail); pairs above
    const int pool = min(N / 8, W * kChunk * 2);
    const int chunk = pool <= kSmallPool ? 1 : kChunk;
    const int ns = N - pool;
    const int qs = ns / W, rs = ns - qs * W;
    Sched sc;
    sc.ctr = a.sched;
    sc.N = N;
    sc.ns = ns;
    sc.cur = wid * qs + min(wid, rs);
    sc.end = sc.cur + qs + (wid < rs ? 1 : 0);
    sc.dyn = 0;
    sc.pend = 0;
    sc.lane = lane;
    sc.RT = a.rows / 16;
    sc.started = 0;
    sc.it = Item{0, 0, 0};
    sc.chunk = chunk;

    Item it0{0, 0, 0}, it1{0, 0, 0};
    int npro = 0;
    if (sc.next(st, it0)) {
        if (lane == 0) issue_weights<C>(a, st, it0, ring, &bars[warp][0], pol);
        npro = 1;
        if (sc.next(st, it1)) {
            if (lane == 0) issue_weights<C>(a, st, it1, ring + kStageBytes, &bars[warp][1], pol);
            npro = 2;
        }
    }
    if (!a.wait_first) {
        pdl_wait();  // activations of the predecessor
        res_pass0();
    }
    pdl_trigger();
    ltrace(ltr, 2 + 2 * a.p, 1);
    if (C::kRes && a.p == 1) {
        // resident activations, down pass: segment s's slot row (its expert's
        // format) at res + s*K*2, its bias terms at resx + s*bstride
        if (threadIdx.x == 0) {
            uint32_t bytes = 0;
            for (int s = 0; s < st.n; ++s) bytes += a.K * 2 + (st.sbytes[s] ? a.bstride * 4 : 0);
            mbar_expect_tx(&res_bar, bytes);
            for (int s = 0; s < st.n; ++s) {
                const int br = st.brow[s][0];
                const bool p4 = st.sbytes[s] != 0;
                bulk_g2s(res + s * a.K * 2, (p4 ? a.b16h : a.b16) + static_cast<size_t>(br) * a.K, a.K * 2, &res_bar);
                if (p4) bulk_g2s(resx + s * a.bstride, a.bsum + static_cast<size_t>(br) * a.bstride, a.bstride * 4, &res_bar);
            }
        }
    }
    // the prologue items' activation halves (per-item configuration)
    if (!C::kRes && lane == 0) {
        if (npro > 0) issue_acts<C>(a, st, it0, ring, &bars[warp][0]);
        if (npro > 1) issue_acts<C>(a, st, it1, ring + kStageBytes, &bars[warp][1]);
    }
    if (C::kRes) mbar_wait(&res_bar, 0);
    const unsigned long long t_wait = gtimer();
    int issued = npro, computed = 0;
    uint32_t phase_bits = 0;

    while (computed < issued) {
        const int stage = computed & 1;
        const Item it = stage ? it1 : it0;
        mbar_wait(&bars[warp][stage], (phase_bits >> stage) & 1u);
        phase_bits ^= 1u << stage;
        uint8_t* sp = ring + stage * kStageBytes;
        float acc[4] = {0.f, 0.f, 0.f, 0.f};
        {
            const int gk = st.gk[it.s];
            const uint8_t* bp;
            const float *x0, *x1;
            if (C::kRes) {
                const bool p4 = st.sbytes[it.s] != 0;
                const int row = a.p == 0 ? (p4 ? 1 : 0) : it.s;  // pass 0: format slot; pass 1: segment
                bp = res + row * a.K * 2 + it.kp * gk * 256 + t * 16;
                x0 = x1 = resx + (a.p == 0 ? 0 : it.s * a.bstride) + it.kp * gk;
            } else {
                const int m_cnt = st.mcnt[it.s];
                bp = sp + C::kStageB + min(gr, m_cnt - 1) * (gk * 256 + kBRowPad) + t * 16;
                const int g0 = (it.kp * gk) & 7;
                x0 = reinterpret_cast<const float*>(sp + C::kStageX + min(2 * t, m_cnt - 1) * 32) + g0;
                x1 = reinterpret_cast<const float*>(sp + C::kStageX + min(2 * t + 1, m_cnt - 1) * 32) + g0;
            }
            compute_item<C>(st, it, sp, bp, x0, x1, lane, acc);
        }
        ++computed;
        // release the stage and refill it with the next item of the sequence
        fence_proxy_async();
        __syncwarp();
        Item nit;
        if (sc.next(st, nit)) {
            if (lane == 0) {
                issue_weights<C>(a, st, nit, sp, &bars[warp][stage], pol);
                issue_acts<C>(a, st, nit, sp, &bars[warp][stage]);
            }
            if (stage) it1 = nit; else it0 = nit;
            ++issued;
        }
        // this item's fp32 partial: columns 2t, 2t+1 of rows gr, gr+8
        const int m_cnt = st.mcnt[it.s];
        float* pp = a.part + (static_cast<size_t>(it.kp) * nslots + st.slot0[it.s] + 2 * t) * a.rows + it.rt * 16 + gr;
        if (2 * t < m_cnt) {
            __stcg(pp, acc[0]);
            __stcg(pp + 8, acc[2]);
        }
        if (2 * t + 1 < m_cnt) {
            __stcg(pp + a.rows, acc[1]);
            __stcg(pp + a.rows + 8, acc[3]);
        }
    }
    ltrace(ltr, 2 + 2 * a.p, 2);
    unsigned long long* tr = g_gemv_trace;
    if (tr != nullptr && lane == 0) {
        tr += (static_cast<size_t>(a.p) * W + static_cast<size_t>(wid)) * 8;
        tr[0] = t_entry;
        tr[1] = t_wait;
        tr[2] = t_wait;
        tr[3] = gtimer();
        tr[4] = static_cast<unsigned long long>(computed);
        tr[5] = 0;
        tr[6] = 0;
        tr[7] = 0;
    }
}

// Fixed-order reduction of the K-part partials of 4 consecutive rows of one
// slot: thread (q, kg) of a (quads x kGroups) block sums K-parts kg, kg+kG,
// ... with up to 8 loads in flight, then the kG partial sums are added in kg
// order through shared memory -- deterministic for a given KP.
constexpr int kKG = 8;  // K-part groups per quad (threads per 4 output rows)

MOE_DEVI float4 sum_kparts(const float* p, size_t kstride, int KP, int kg) {
    float4 acc[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) acc[u] = make_float4(0.f, 0.f, 0.f, 0.f);
    for (int kp0 = kg; kp0 < KP; kp0 += 8 * kKG) {
        float4 v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u)
            v[u] = kp0 + u * kKG < KP ? __ldcg(reinterpret_cast<const float4*>(p + (kp0 + u * kKG) * kstride))
                                      : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            acc[u].x += v[u].x; acc[u].y += v[u].y; acc[u].z += v[u].z; acc[u].w += v[u].w;
        }
    }
#pragma unroll
    for (int u = 1; u < 8; ++u) {
        acc[0].x += acc[u].x; acc[0].y += acc[u].y; acc[0].z += acc[u].z; acc[0].w += acc[u].w;
    }
    return acc[0];
}

// SwiGLU finalize: one block per (slot, 128-row group g of h).  64 quads
// (gate rows g*128.., up rows f+g*128..) x 4 K-part groups; h is rounded to
// bf16 and stored as bf16 (perm_k) and its exact fp16 copy (perm_k16), plus
// the group's int4 bias term 1032*S_lo + 72*S_hi.
constexpr int kFinHThreads = 64 * kKG;
constexpr int kFinOQuads = 8;   // 32 outputs per block: T=1 spreads d=4096 over 128 blocks
constexpr int kFinOThreads = kFinOQuads * kKG;
// SwiGLU tail of one (slot, 128-row group g of h) unit, warp 0 (lanes 0-31):
// red[kg][q] holds the K-part-group sums of gate rows g*128+4q.. (q < 32) and
// up rows (q >= 32); h rounded to bf16 goes out as the K-permuted bf16 copy,
// its exact fp16 copy and the group's int4 bias term.  Shared by
// finalize_h_kernel and the fused decode-step kernel (identical arithmetic).
// gv / uv: this lane's 4 summed gate rows g*128+4*lane.. and up rows.
MOE_DEVI void swiglu_store(const float (&gv)[4], const float (&uv)[4], uint16_t* hs, int slot, int g, int f,
                           uint16_t* __restrict__ hperm, uint16_t* __restrict__ hperm16, float* __restrict__ hsum,
                           int hstride, int lane) {
#pragma unroll
    for (int j = 0; j < 4; ++j) hs[lane * 4 + j] = f2bf(silu_f(gv[j]) * uv[j]);
    __syncwarp();
    uint4 cb = make_uint4(0, 0, 0, 0), ch = cb;
    float s_lo = 0.0f, s_hi = 0.0f, amax = 0.0f;
    if (lane < 16) permute_chunk(hs, lane, cb, ch, s_lo, s_hi, amax);
    numerics_group_check(amax, lane == 0);
    const size_t o = static_cast<size_t>(slot) * f + g * 128;
    if (lane < 16) {
        reinterpret_cast<uint4*>(hperm + o)[lane] = cb;
        reinterpret_cast<uint4*>(hperm16 + o)[lane] = ch;
    }
#pragma unroll
    for (int off = 8; off >= 1; off >>= 1) {
        s_lo += __shfl_xor_sync(0xffffffffu, s_lo, off);
        s_hi += __shfl_xor_sync(0xffffffffu, s_hi, off);
    }
    if (lane == 0) hsum[static_cast<size_t>(slot) * hstride + g] = int4_bias_term(s_lo, s_hi);
    __syncwarp();
}

MOE_DEVI void swiglu_unit(const float4 (&red)[kKG][64], uint16_t* hs, int slot, int g, int f, uint16_t* __restrict__ hperm,
                          uint16_t* __restrict__ hperm16, float* __restrict__ hsum, int hstride, int lane) {
    float gv[4], uv[4];
    {
        float4 a = red[0][lane], b = red[0][32 + lane];
#pragma unroll
        for (int k2 = 1; k2 < kKG; ++k2) {
            const float4 c = red[k2][lane], e = red[k2][32 + lane];
            a.x += c.x; a.y += c.y; a.z += c.z; a.w += c.w;
            b.x += e.x; b.y += e.y; b.z += e.z; b.w += e.w;
        }
        gv[0] = a.x; gv[1] = a.y; gv[2] = a.z; gv[3] = a.w;
        uv[0] = b.x; uv[1] = b.y; uv[2] = b.z; uv[3] = b.w;
    }
    swiglu_store(gv, uv, hs, slot, g, f, hperm, hperm16, hsum, hstride, lane);
}

__global__ void __launch_bounds__(kFinHThreads) finalize_h_kernel(
    const float* __restrict__ part, const int* __restrict__ kpslot, int nslots, int f, uint16_t* __restrict__ hperm,
    uint16_t* __restrict__ hperm16, float* __restrict__ hsum, int hstride, unsigned int* sched) {
    __shared__ float4 red[kKG][64];
    __shared__ uint16_t hs[128];
    const int G = f / 128;
    const int slot = blockIdx.x / G, g = blockIdx.x - slot * G;
    unsigned long long* const ltr = g_layer_trace;
    ltrace(ltr, 3, 0);
    // Trigger first: the down-pass stream kernel only reads the routing
    // before its own PDL wait, so its CTAs may start (and prefetch weights)
    // as the gate/up stream's CTAs drain.
    pdl_trigger();
    pdl_wait();
    ltrace(ltr, 3, 1);
    if (blockIdx.x == 0 && threadIdx.x == 0) *sched = 0;  // the stream kernel is complete
    const int KP = kpslot[slot];
    if (KP == 0) return;
    const size_t rows = static_cast<size_t>(2) * f;
    const int q = threadIdx.x & 63, kg = threadIdx.x >> 6;
    const int row = (q < 32 ? g * 128 + q * 4 : f + g * 128 + (q - 32) * 4);
    red[kg][q] = sum_kparts(part + static_cast<size_t>(slot) * rows + row, static_cast<size_t>(nslots) * rows, KP, kg);
    __syncthreads();
    if (threadIdx.x >= 32) return;
    swiglu_unit(red, hs, slot, g, f, hperm, hperm16, hsum, hstride, threadIdx.x);
    ltrace(ltr, 3, 2);
}

// Output finalize: one block per (token t, 128 output rows) -- or, with
// out == null, per (slot, 128 rows) writing y itself for the slots of this
// launch's experts.  y[slot][j] = fixed-order sum of the slot's pass-1
// partials; out[t][j] = bf16(resid[t][j] + sum_jj w[t,jj] * y[inv[t,jj]][j])
// (fp32 fma chain in jj order).
__global__ void __launch_bounds__(kFinOThreads) finalize_out_kernel(
    const float* __restrict__ part, const int* __restrict__ kpslot, int T, int k, int d,
    const int32_t* __restrict__ inv, const float* __restrict__ wts, const uint16_t* __restrict__ resid,
    uint16_t* __restrict__ out, float* __restrict__ y, unsigned int* sched) {
    __shared__ float4 red[kKG][kFinOQuads];
    const int nslots = T * k;
    const int nb = d / (kFinOQuads * 4);
    const int r = blockIdx.x / nb, j0 = (blockIdx.x - r * nb) * (kFinOQuads * 4);
    unsigned long long* const ltr = g_layer_trace;
    ltrace(ltr, 5, 0);
    pdl_trigger();  // the next layer's route kernel preloads router weights before its wait
    pdl_wait();
    ltrace(ltr, 5, 1);
    if (blockIdx.x == 0 && threadIdx.x == 0) *sched = 0;
    const size_t kstride = static_cast<size_t>(nslots) * d;
    const int q = threadIdx.x % kFinOQuads, kg = threadIdx.x / kFinOQuads;
    const int j = j0 + q * 4;
    if (out == nullptr) {
        const int KP = kpslot[r];
        if (KP == 0) return;
        red[kg][q] = sum_kparts(part + static_cast<size_t>(r) * d + j, kstride, KP, kg);
        __syncthreads();
        if (kg != 0) return;
        float4 a = red[0][q];
#pragma unroll
        for (int k2 = 1; k2 < kKG; ++k2) {
            const float4 c = red[k2][q];
            a.x += c.x; a.y += c.y; a.z += c.z; a.w += c.w;
        }
        *reinterpret_cast<float4*>(y + static_cast<size_t>(r) * d + j) = a;
        return;
    }
    const int t = r;
    float acc[4];
    if (kg == 0) {
#pragma unroll
        for (int u = 0; u < 4; ++u) acc[u] = resid ? bf2f(resid[static_cast<size_t>(t) * d + j + u]) : 0.0f;
    }
    for (int jj = 0; jj < k; ++jj) {
        const int slot = inv[t * k + jj];
        const int KP = kpslot[slot];
        red[kg][q] = KP ? sum_kparts(part + static_cast<size_t>(slot) * d + j, kstride, KP, kg)
                        : make_float4(0.f, 0.f, 0.f, 0.f);
        __syncthreads();
        if (kg == 0) {
            float4 a = red[0][q];
#pragma unroll
            for (int k2 = 1; k2 < kKG; ++k2) {
                const float4 c = red[k2][q];
                a.x += c.x; a.y += c.y; a.z += c.z; a.w += c.w;
            }
            const float w = wts[t * k + jj];
            acc[0] = __fmaf_rn(w, a.x, acc[0]);
            acc[1] = __fmaf_rn(w, a.y, acc[1]);
            acc[2] = __fmaf_rn(w, a.z, acc[2]);
            acc[3] = __fmaf_rn(w, a.w, acc[3]);
        }
        __syncthreads();
    }
    if (kg == 0) {
#pragma unroll
        for (int u = 0; u < 4; ++u) out[static_cast<size_t>(t) * d + j + u] = f2bf(acc[u]);
    }
    ltrace(ltr, 5, 2);
}

// x (natural, [rows][K]) -> K-permuted bf16 + fp16 copies and, per 128-K
// group, the int4 bias term 1032*S_lo + 72*S_hi (S_lo: elements with
// k%16 < 8, S_hi: the rest; fixed xor-butterfly order).  One warp per
// (row, group); lane owns 4 elements.
__global__ void permute_rows_kernel(const uint16_t* __restrict__ x, int rows, int K, uint16_t* __restrict__ xp,
                                    uint16_t* __restrict__ xp16, float* __restrict__ xsum, int xstride) {
    // one half-warp per (row, 128-K group): 16 chunks of 16 bytes
    const int G = K / 128;
    const long long hw = (static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x) >> 4;
    const int c = threadIdx.x & 15;
    unsigned long long* const ltr = g_layer_trace;
    ltrace(ltr, 1, 0);
    pdl_wait();     // x is the previous layer's output
    pdl_trigger();
    ltrace(ltr, 1, 1);
    const bool ok = hw < static_cast<long long>(rows) * G;
    const long long r = ok ? hw / G : 0;
    const int g = ok ? static_cast<int>(hw - r * G) : 0;
    uint4 cb = make_uint4(0, 0, 0, 0), ch = cb;
    float s_lo = 0.0f, s_hi = 0.0f, amax = 0.0f;
    if (ok) permute_chunk(x + r * K + g * 128, c, cb, ch, s_lo, s_hi, amax);
    numerics_group_check(amax, ok && c == 0);
#pragma unroll
    for (int off = 8; off >= 1; off >>= 1) {
        s_lo += __shfl_xor_sync(0xffffffffu, s_lo, off);
        s_hi += __shfl_xor_sync(0xffffffffu, s_hi, off);
    }
    if (!ok) return;
    reinterpret_cast<uint4*>(xp + r * K + g * 128)[c] = cb;
    reinterpret_cast<uint4*>(xp16 + r * K + g * 128)[c] = ch;
    if (c == 0) xsum[r * xstride + g] = int4_bias_term(s_lo, s_hi);
}

__host__ __device__ inline int group_stride(int K) { return (K / 128 + 7) / 8 * 8; }

// ===========================================================================
// Fused batch-1 decode step: the whole L-layer stack in ONE persistent launch
// (one CTA per SM, cooperative), replacing 5 launches per layer.  Per layer:
//   R  every CTA routes the token itself (RMSNorm, logits, top-k, permutation
//      -- route_common.cuh, bit-identical to route_kernel) straight into its
//      resident activation rows, and builds both passes' segment tables;
//   G  gate/up items (the streaming GEMV's items, rings, scheduler); once a
//      warp has issued its last gate/up item its ring runs on into the down
//      pass's weights, which do not depend on h;
//   |  grid barrier
//   H  SwiGLU finalize, (slot, 128-group) units spread over the CTAs;
//   |  grid barrier
//   D  h rows -> resident rows; down items (weights mostly already landed);
//   |  grid barrier
//   O  combine + residual, 32-output blocks spread over the CTAs -> x(l+1);
//   |  grid barrier (not after the last layer)
// The partial layouts, item decomposition, K-part sums and combine order are
// those of the per-layer kernels, so the output is bit-identical to them.
// What it removes per layer: 4 launch / PDL boundaries, the route kernel's
// own round trips and the stream kernels' prologues (≈ 9 of ≈ 18 µs of
// non-streaming time per int4 layer, profiles/README.md r02).
using DecodeArgs = MoeDecodeArgs;

// Debug (moe_debug_fused_trace): per layer and CTA, globaltimer stamps of the
// phase boundaries [L][gridDim][kFusedStamps]; null (default) = off.
constexpr int kFusedStamps = 18;  // 0-9 phase boundaries, 10-14 inside routing
__device__ unsigned long long* g_fused_trace = nullptr;
// The trace pointer is read once per kernel (ftr): a per-stamp load of the
// global would put an L2 round trip in front of every phase.  Stamps are SM
// cycles (clock64: a register read; %globaltimer reads cost ~0.5 us each).
// Stamps are warp-uniform (every lane reads the clock, lane 0 stores, then
// __syncwarp): a lane-0-only branch would leave the warp diverged into the
// next shuffle and slow it down -- the trace must not change what it measures.
MOE_DEVI void fstamp_lane0(unsigned long long* tr, int l, int i) {
    if (tr == nullptr) return;
    const unsigned long long c = clock64();
    if ((threadIdx.x & 31) == 0) tr[(static_cast<size_t>(l) * gridDim.x + blockIdx.x) * kFusedStamps + i] = c;
    __syncwarp();
}
MOE_DEVI void fstamp(unsigned long long* tr, int l, int i) {
    if (tr == nullptr || threadIdx.x >= 32) return;
    fstamp_lane0(tr, l, i);
}

MOE_DEVI unsigned int ld_acquire_gpu(const unsigned int* p) {
    unsigned int v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
MOE_DEVI void st_release_gpu(unsigned int* p, unsigned int v) {
    asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
MOE_DEVI void fence_proxy_async_global() { asm volatile("fence.proxy.async.global;" ::: "memory"); }

// Grid barrier over all CTAs (co-resident: cooperative launch) on one
// monotonic 64-bit arrival counter: a CTA's arrival number tells it its
// round r, and it proceeds once the counter reaches (r + 1) * gridDim.x.
// One release fetch-add per CTA, acquire polling, no reset step.  mode 1:
// a full fence + relaxed add instead of the release add (A/B).
MOE_DEVI void grid_barrier(unsigned long long* ctr, int mode) {
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned long long old;
        if (mode == 1) {
            __threadfence();
            asm volatile("atom.add.relaxed.gpu.global.u64 %0, [%1], 1;" : "=l"(old) : "l"(ctr) : "memory");
        } else {
            asm volatile("atom.add.release.gpu.global.u64 %0, [%1], 1;" : "=l"(old) : "l"(ctr) : "memory");
        }
        const unsigned long long target = (old / gridDim.x + 1) * gridDim.x;
        unsigned long long v;
        do {
            asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(ctr) : "memory");
        } while (v < target);
    }
    __syncthreads();
}

// Segment table of one pass for a batch-1 step: one segment per selected
// expert (mcnt = 1), in expert order -- build_segs' table for T = 1.
template <class C>
MOE_DEVI void build_segs_t1(SegTable& st, const moe_expert_weights* ex, const int32_t* offsets, int E, int p,
                            int rows, int K) {
    const int RT = rows / 16, G = K / 128;
    int n = 0, acc = 0;
    for (int e = 0; e < E; ++e) {
        if (offsets[e + 1] == offsets[e]) continue;
        const moe_expert_weights& W = ex[e];
        const int gk = pick_gk<C>(G, W.precision, 1);
        st.e[n] = e;
        st.slot0[n] = offsets[e];
        st.mcnt[n] = 1;
        st.kp[n] = G / gk;
        st.gk[n] = gk;
        st.wptr[n] = static_cast<const uint8_t*>(p == 0 ? W.w_gate_up : W.w_down);
        st.sptr[n] = static_cast<const uint8_t*>(p == 0 ? W.s_gate_up : W.s_down);
        st.wbytes[n] = W.precision == MOE_P4 ? gk * 1024 : gk * 4096;
        st.sbytes[n] = W.precision == MOE_P4 ? gk * 32 : 0;
        st.pre[n] = acc;
        for (int c = 0; c < kTile; ++c) st.brow[n][c] = p == 0 ? 0 : offsets[e];
        acc += RT * (G / gk);
        ++n;
    }
    st.pre[n] = acc;
    st.n = n;
    st.N = acc;
}

// The weight half of an item of a pass with reduction length K (issue_weights
// without the activation bytes: resident rows).
MOE_DEVI void issue_item_w(const SegTable& st, int K, const Item& it, uint8_t* stage, uint64_t* bar, uint64_t pol,
                           int stage_s_off) {
    const int s = it.s, wb = st.wbytes[s], sb = st.sbytes[s];
    mbar_expect_tx(bar, wb + sb);
    const size_t blk = static_cast<size_t>(it.rt) * (K / 128) + static_cast<size_t>(it.kp) * st.gk[s];
    bulk_g2s_hint(stage, st.wptr[s] + blk * (sb ? 1024 : 4096), wb, bar, pol);
    if (sb) bulk_g2s_hint(stage + stage_s_off, st.sptr[s] + blk * 32, sb, bar, pol);
}

MOE_DEVI void sched_init(Sched& sc, unsigned int* ctr, int N, int W, int wid, int lane, int RT) {
    const int pool = min(N / 8, W * kChunk * 2);
    sc.chunk = pool <= kSmallPool ? 1 : kChunk;
    sc.ctr = ctr;
    sc.N = N;
    sc.ns = N - pool;
    const int qs = sc.ns / W, rs = sc.ns - qs * W;
    sc.cur = wid * qs + min(wid, rs);
    sc.end = sc.cur + qs + (wid < rs ? 1 : 0);
    sc.dyn = 0;
    sc.pend = 0;
    sc.lane = lane;
    sc.RT = RT;
    sc.started = 0;
    sc.it = Item{0, 0, 0};
}

// Batch-1 routing tail of the fused step, one warp, no serial single-thread
// code and one barrier fewer: top-k on the E logits in registers (REDUX max
// of order-preserving keys, lowest index among ties -- route_kernel's
// warp_topk semantics), softmax over the selected logits in j order, the
// T = 1 permutation (slots in expert order), and both passes' segment tables
// (build_segs_t1's) filled by lanes 0..k-1 (gate/up) and 16..16+k-1 (down).
MOE_DEVI uint32_t order_key(float v) {
    const uint32_t u = __float_as_uint(v == 0.0f ? 0.0f : v);  // -0 ties with +0 (float compare)
    return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}
template <class C>
MOE_DEVI void route_tail_t1(const float* lg, const moe_expert_weights* ex, int E, int k, int d, int f, int lane,
                            int32_t* topi, float* wts, int32_t* inv, SegTable& st0, SegTable& st1) {
    const bool h0 = lane < E, h1 = lane + 32 < E;
    const float v0 = h0 ? lg[lane] : 0.0f, v1 = h1 ? lg[lane + 32] : 0.0f;
    uint32_t k0 = h0 ? order_key(v0) : 0u, k1 = h1 ? order_key(v1) : 0u;
    bool a0 = h0, a1 = h1;
    int sel[2] = {0, 0};
    float sv[2] = {0.0f, 0.0f};
#pragma unroll
    for (int j = 0; j < 2; ++j) {
        if (j >= k) break;
        const uint32_t m = __reduce_max_sync(0xffffffffu, max(a0 ? k0 : 0u, a1 ? k1 : 0u));
        const uint32_t b0 = __ballot_sync(0xffffffffu, a0 && k0 == m);
        const uint32_t b1 = __ballot_sync(0xffffffffu, a1 && k1 == m);
        const int w = b0 ? __ffs(b0) - 1 : 32 + __ffs(b1) - 1;  // lowest index among the maxima
        sel[j] = w;
        sv[j] = __shfl_sync(0xffffffffu, w < 32 ? v0 : v1, w & 31);
        if (w == lane) a0 = false;
        if (w == lane + 32) a1 = false;
    }
    // softmax over the selected logits, sum in j order (warp_topk / the oracle)
    float ex_[2] = {0.0f, 0.0f}, sum = 0.0f;
#pragma unroll
    for (int j = 0; j < 2; ++j)
        if (j < k) {
            ex_[j] = expf(sv[j] - sv[0]);
            sum += ex_[j];
        }
    // T = 1: slot of selection j = its rank among the selected experts
    int pos[2] = {0, 0};
#pragma unroll
    for (int j = 0; j < 2; ++j)
#pragma unroll
        for (int i = 0; i < 2; ++i)
            if (j < k && i < k && sel[i] < sel[j]) ++pos[j];
    if (lane < k) {
        const int j = lane;
        topi[j] = sel[j == 0 ? 0 : 1];
        wts[j] = ex_[j == 0 ? 0 : 1] / sum;
        inv[j] = pos[j == 0 ? 0 : 1];
    }
    // segment s = the selected expert of rank s
    const int p = lane >> 4, s = lane & 15;
    SegTable& st = p ? st1 : st0;
    const int rows = p ? d : 2 * f, K = p ? f : d;
    const int RT = rows / 16, G = K / 128;
    int e = 0;
#pragma unroll
    for (int j = 0; j < 2; ++j)
        if (j < k && pos[j] == s) e = sel[j];
    int items = 0, gk = 1;
    if (s < k && p < 2) {
        const moe_expert_weights& W = ex[e];
        gk = pick_gk<C>(G, W.precision, 1);
        items = RT * (G / gk);
    }
    // prefix over the (<= 2) segments of this pass
    const int prev = __shfl_up_sync(0xffffffffu, items, 1);
    const int pre = s == 0 ? 0 : prev;
    if (s < k && p < 2) {
        const moe_expert_weights& W = ex[e];
        st.e[s] = e;
        st.slot0[s] = s;
        st.mcnt[s] = 1;
        st.kp[s] = G / gk;
        st.gk[s] = gk;
        st.wptr[s] = static_cast<const uint8_t*>(p == 0 ? W.w_gate_up : W.w_down);
        st.sptr[s] = static_cast<const uint8_t*>(p == 0 ? W.s_gate_up : W.s_down);
        st.wbytes[s] = W.precision == MOE_P4 ? gk * 1024 : gk * 4096;
        st.sbytes[s] = W.precision == MOE_P4 ? gk * 32 : 0;
        st.pre[s] = pre;
#pragma unroll
        for (int c = 0; c < kTile; ++c) st.brow[s][c] = p == 0 ? 0 : s;
        if (s == k - 1) {
            st.pre[k] = pre + items;
            st.n = k;
            st.N = pre + items;
        }
    }
}

template <class C>
__global__ void __launch_bounds__(C::kThreads, 1) decode_step_kernel(const __grid_constant__ DecodeArgs a) {
    constexpr int kWarps = C::kWarps;
    constexpr int kStageBytes = C::kStageBytes;
    extern __shared__ __align__(128) uint8_t smem[];
    __shared__ SegTable st[2];
    __shared__ __align__(8) uint64_t bars[kWarps][kStages];
    __shared__ __align__(8) uint64_t res_bar;
    __shared__ __align__(16) moe_expert_weights s_ex[MOE_MAX_EXPERTS];
    __shared__ float lg_s[MOE_MAX_EXPERTS + C::kThreads];
    __shared__ int32_t s_idx[MOE_MAX_TOPK], s_counts[MOE_MAX_EXPERTS], s_offsets[MOE_MAX_EXPERTS + 1];
    __shared__ int32_t s_perm[MOE_MAX_TOPK], s_inv[MOE_MAX_TOPK], s_topi[MOE_MAX_TOPK];
    __shared__ float s_w[MOE_MAX_TOPK];
    __shared__ uint16_t hs[2][128];
    __shared__ float4 redo[MOE_MAX_TOPK][kKG][kFinOQuads];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, tid = threadIdx.x;
    const int d = a.d, f = a.f, E = a.E, k = a.k;
    unsigned long long* const ftr = g_fused_trace;
    if (lane == 0) {
        for (int s2 = 0; s2 < kStages; ++s2) mbar_init(&bars[warp][s2], 1);
        if (warp == 0) mbar_init(&res_bar, 1);
        fence_mbar_init();
    }
    __syncthreads();
    const uint64_t pol = policy_evict_first();
    const int W = static_cast<int>(gridDim.x) * kWarps;
    const int wid = static_cast<int>(blockIdx.x) * kWarps + warp;
    const int gr = lane >> 2, t4 = lane & 3;
    uint8_t* ring = smem + static_cast<size_t>(warp) * kStages * kStageBytes;
    uint8_t* res = smem + static_cast<size_t>(kWarps) * kStages * kStageBytes;
    uint16_t* xs = reinterpret_cast<uint16_t*>(smem);  // phase R scratch: raw row, then normalised row (rings idle)
    uint16_t* xn = xs + d;
    const int bs0 = group_stride(d), bs1 = group_stride(f);
    uint32_t phase_bits = 0, res_phase = 0;
    // router weights of the layer about to route, in registers: layer 0's
    // here, layer l+1's before layer l's last barrier (its L2 prefetch went
    // out at the start of layer l's gate/up phase)
    uint4 wpre[kPreChunks];
    if (warp < E) preload_w(wpre, a.wg + static_cast<size_t>(warp) * d, d, lane);

    for (int l = 0; l < a.L; ++l) {
        const uint16_t* xl = l == 0 ? a.x_in : ((l - 1) & 1 ? a.xbuf1 : a.xbuf0);
        uint16_t* yl = l == a.L - 1 ? a.x_out : (l & 1 ? a.xbuf1 : a.xbuf0);
        const uint16_t* wgl = a.wg + static_cast<size_t>(l) * E * d;
        fstamp(ftr, l, 0);
        // ---- R: route the token (every CTA, identical results) --------------
        for (int i = tid; i < E * static_cast<int>(sizeof(moe_expert_weights) / 8); i += blockDim.x)
            reinterpret_cast<uint2*>(s_ex)[i] =
                reinterpret_cast<const uint2*>(a.experts + static_cast<size_t>(l) * E)[i];
        for (int i = tid * 8; i < d; i += blockDim.x * 8)
            *reinterpret_cast<uint4*>(xs + i) = __ldcg(reinterpret_cast<const uint4*>(xl + i));
        __syncthreads();
        fstamp(ftr, l, 10);
        const uint16_t* xr = xs;
        if (a.norm_eps > 0.0f) {
            float acc = 0.0f;  // route_kernel's pinned order
            for (int c = 0; c * 256 + tid < d; ++c) {
                const float v = bf2f(xs[c * 256 + tid]);
                acc = __fmaf_rn(v, v, acc);
            }
            lg_s[MOE_MAX_EXPERTS + tid] = acc;
            __syncthreads();
            for (int s2 = 128; s2 >= 32; s2 >>= 1) {
                if (tid < s2) lg_s[MOE_MAX_EXPERTS + tid] = __fadd_rn(lg_s[MOE_MAX_EXPERTS + tid], lg_s[MOE_MAX_EXPERTS + tid + s2]);
                __syncthreads();
            }
            if (warp == 0) {
                float v = lg_s[MOE_MAX_EXPERTS + lane];
#pragma unroll
                for (int s2 = 16; s2 >= 1; s2 >>= 1) v = __fadd_rn(v, __shfl_down_sync(0xffffffffu, v, s2));
                if (lane == 0) lg_s[MOE_MAX_EXPERTS] = v;
            }
            __syncthreads();
            const float rstd = __fdiv_rn(1.0f, __fsqrt_rn(__fadd_rn(__fdiv_rn(lg_s[MOE_MAX_EXPERTS], static_cast<float>(d)),
                                                                    a.norm_eps)));
            fstamp(ftr, l, 11);
            for (int i = tid * 8; i < d; i += blockDim.x * 8) {
                uint4 v = *reinterpret_cast<const uint4*>(xs + i);
                uint32_t w4[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
                for (int q = 0; q < 4; ++q)
                    w4[q] = static_cast<uint32_t>(f2bf(__fmul_rn(bf16_lo(w4[q]), rstd))) |
                            (static_cast<uint32_t>(f2bf(__fmul_rn(bf16_hi(w4[q]), rstd))) << 16);
                *reinterpret_cast<uint4*>(xn + i) = make_uint4(w4[0], w4[1], w4[2], w4[3]);
            }
            __syncthreads();
            fstamp(ftr, l, 12);
            xr = xn;
        }
        for (int e = warp; e < E; e += kWarps) {
            if (e != warp) preload_w(wpre, wgl + static_cast<size_t>(e) * d, d, lane);
            const float v = router_dot(xr, wpre, wgl + static_cast<size_t>(e) * d, d, lane);
            if (lane == 0) lg_s[e] = v;
        }
        __syncthreads();
        fstamp(ftr, l, 13);
        if (warp == 0) {
            route_tail_t1<C>(lg_s, s_ex, E, k, d, f, lane, s_topi, s_w, s_inv, st[0], st[1]);
            __syncwarp();
            if (blockIdx.x == 0 && lane < k) {
                a.idx[static_cast<size_t>(l) * a.idx_stride + lane] = s_topi[lane];
                a.wts[static_cast<size_t>(l) * a.idx_stride + lane] = s_w[lane];
            }
            fstamp(ftr, l, 15);
        } else {
            // resident activation rows of the gate/up pass: K-permuted bf16
            // (res), fp16 (res + 2d) and the int4 bias terms (res + 4d)
            uint16_t* rb = reinterpret_cast<uint16_t*>(res);
            uint16_t* rh = rb + d;
            float* rx = reinterpret_cast<float*>(res + 4 * d);
            const int G = d / 128, nw = kWarps - 1;
            for (int g0 = (warp - 1) * 2; g0 < G; g0 += nw * 2) {
                const int g = g0 + (lane >> 4), c = lane & 15;
                uint4 cb = make_uint4(0, 0, 0, 0), ch = cb;
                float s_lo = 0.0f, s_hi = 0.0f, amax = 0.0f;
                if (g < G) permute_chunk(xr + g * 128, c, cb, ch, s_lo, s_hi, amax);
                numerics_group_check(amax, c == 0);
#pragma unroll
                for (int off = 8; off >= 1; off >>= 1) {
                    s_lo += __shfl_xor_sync(0xffffffffu, s_lo, off);
                    s_hi += __shfl_xor_sync(0xffffffffu, s_hi, off);
                }
                if (g < G) {
                    reinterpret_cast<uint4*>(rb + g * 128)[c] = cb;
                    reinterpret_cast<uint4*>(rh + g * 128)[c] = ch;
                    if (c == 0) rx[g] = int4_bias_term(s_lo, s_hi);
                }
            }
            if (warp == 1) fstamp_lane0(ftr, l, 16);
        }
        fence_proxy_async();  // scratch (generic) writes before the rings' bulk copies
        __syncthreads();
        fstamp(ftr, l, 14);
        fstamp(ftr, l, 1);

        if (l + 1 < a.L && blockIdx.x < 4 && tid == 0) {  // next layer's router weights -> L2
            const uint32_t chunk = static_cast<uint32_t>(E) * d * 2 / 4;
            if (chunk % 16 == 0)
                asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(wgl + static_cast<size_t>(E) * d +
                                                                            static_cast<size_t>(blockIdx.x) * chunk / 2),
                             "r"(chunk)
                             : "memory");
        }
        // ---- G: gate/up items, the ring running on into the down weights ------
        Sched sc[2];
        sched_init(sc[0], a.sched + 2 * l, st[0].N, W, wid, lane, (2 * f) / 16);
        sched_init(sc[1], a.sched + 2 * l + 1, st[1].N, W, wid, lane, d / 16);
        int np = 0;  // pass of the next item to issue
        auto next_item = [&](Item& it, int& pass) -> bool {
            if (np == 0) {
                if (sc[0].next(st[0], it)) {
                    pass = 0;
                    return true;
                }
                np = 1;
            }
            if (sc[1].next(st[1], it)) {
                pass = 1;
                return true;
            }
            return false;
        };
        // the two stages' items live in registers (static indices only: a
        // dynamically indexed array would go to local memory)
        static_assert(kStages == 2, "two ring stages");
        Item it0{0, 0, 0}, it1{0, 0, 0};
        int ps0 = 0, ps1 = 0;
        int issued = 0, computed = 0;
        if (next_item(it0, ps0)) {
            if (lane == 0) issue_item_w(st[ps0], ps0 ? f : d, it0, ring, &bars[warp][0], pol, C::kStageS);
            ++issued;
            if (next_item(it1, ps1)) {
                if (lane == 0) issue_item_w(st[ps1], ps1 ? f : d, it1, ring + kStageBytes, &bars[warp][1], pol, C::kStageS);
                ++issued;
            }
        }
        for (int pass = 0; pass < 2; ++pass) {
            if (pass == 1) {
                // ---- H: SwiGLU finalize over (slot, 128-group) units -------------
                fence_proxy_async();  // resident rows read (generic) before phase D's bulk copies
                fstamp(ftr, l, 2);
                grid_barrier(a.bar, a.bar_mode);
                fstamp(ftr, l, 3);
                const int Gf = f / 128;
                const size_t rows2 = static_cast<size_t>(2) * f;
                // up to two (slot, group) units per CTA at once: every K-part
                // load issued before any sum is used; the K-part-group sums go
                // to the (now free) resident area, warps 0 and 1 finish one unit each
                typedef float4 RedT[kKG][64];
                RedT* redu = reinterpret_cast<RedT*>(res);
                for (int u0 = blockIdx.x; u0 < k * Gf; u0 += 2 * gridDim.x) {
                    float4 v[2][2];
#pragma unroll
                    for (int j = 0; j < 2; ++j) {
                        const int u = u0 + j * gridDim.x;
                        const int slot = u / Gf, g = u - slot * Gf;
#pragma unroll
                        for (int h2 = 0; h2 < 2; ++h2) {
                            const int q = tid & 63, kg = (tid >> 6) + h2 * 4;
                            const int row = (q < 32 ? g * 128 + q * 4 : f + g * 128 + (q - 32) * 4);
                            v[j][h2] = u < k * Gf ? sum_kparts(a.part0 + static_cast<size_t>(slot) * rows2 + row,
                                                               static_cast<size_t>(k) * rows2, st[0].kp[slot], kg)
                                                  : make_float4(0.f, 0.f, 0.f, 0.f);
                        }
                    }
#pragma unroll
                    for (int j = 0; j < 2; ++j)
#pragma unroll
                        for (int h2 = 0; h2 < 2; ++h2) redu[j][(tid >> 6) + h2 * 4][tid & 63] = v[j][h2];
                    __syncthreads();
                    if (warp < 2) {
                        const int u = u0 + warp * gridDim.x;
                        if (u < k * Gf) {
                            const int slot = u / Gf, g = u - slot * Gf;
                            swiglu_unit(redu[warp], hs[warp], slot, g, f, a.hperm, a.hperm16, a.hsum, bs1, lane);
                        }
                    }
                    __syncthreads();
                }
                fence_proxy_async();  // generic scratch writes to the resident area before phase D's bulk copies
                fstamp(ftr, l, 4);
                grid_barrier(a.bar, a.bar_mode);
                fstamp(ftr, l, 5);
                // ---- D: h rows into the resident area (slot s's row in its format)
                if (tid == 0) {
                    fence_proxy_async_global();
                    uint32_t bytes = 0;
                    for (int s2 = 0; s2 < st[1].n; ++s2) bytes += f * 2 + (st[1].sbytes[s2] ? bs1 * 4 : 0);
                    mbar_expect_tx(&res_bar, bytes);
                    float* rx1 = reinterpret_cast<float*>(res + 2 * f * 2);
                    for (int s2 = 0; s2 < st[1].n; ++s2) {
                        const bool p4 = st[1].sbytes[s2] != 0;
                        const int slot = st[1].slot0[s2];
                        bulk_g2s(res + s2 * f * 2, (p4 ? a.hperm16 : a.hperm) + static_cast<size_t>(slot) * f, f * 2,
                                 &res_bar);
                        if (p4) bulk_g2s(rx1 + s2 * bs1, a.hsum + static_cast<size_t>(slot) * bs1, bs1 * 4, &res_bar);
                    }
                }
                mbar_wait(&res_bar, res_phase);
                res_phase ^= 1u;
                fstamp(ftr, l, 6);
            }
            const int K = pass ? f : d, rows = pass ? d : 2 * f;
            float* part = pass ? a.part1 : a.part0;
            const float* resx = reinterpret_cast<const float*>(res + 2 * K * 2);
            while (computed < issued) {
                const int stage = computed & 1;
                if ((stage ? ps1 : ps0) != pass) break;  // the next item belongs to the down pass
                const Item it = stage ? it1 : it0;
                mbar_wait(&bars[warp][stage], (phase_bits >> stage) & 1u);
                phase_bits ^= 1u << stage;
                uint8_t* sp = ring + stage * kStageBytes;
                float acc[4] = {0.f, 0.f, 0.f, 0.f};
                {
                    const SegTable& T = st[pass];
                    const int gk = T.gk[it.s];
                    const bool p4 = T.sbytes[it.s] != 0;
                    const int row = pass == 0 ? (p4 ? 1 : 0) : it.s;
                    const uint8_t* bp = res + row * K * 2 + it.kp * gk * 256 + t4 * 16;
                    const float* x0 = resx + (pass == 0 ? 0 : it.s * bs1) + it.kp * gk;
                    compute_item<C>(T, it, sp, bp, x0, x0, lane, acc);
                }
                ++computed;
                fence_proxy_async();
                __syncwarp();
                Item nit;
                int npass;
                if (next_item(nit, npass)) {
                    if (lane == 0)
                        issue_item_w(st[npass], npass ? f : d, nit, sp, &bars[warp][stage], pol, C::kStageS);
                    if (stage) {
                        it1 = nit;
                        ps1 = npass;
                    } else {
                        it0 = nit;
                        ps0 = npass;
                    }
                    ++issued;
                }
                const SegTable& T = st[pass];
                float* pp = part + (static_cast<size_t>(it.kp) * k + T.slot0[it.s] + 2 * t4) * rows + it.rt * 16 + gr;
                if (t4 == 0) {  // one token: column 0
                    __stcg(pp, acc[0]);
                    __stcg(pp + 8, acc[2]);
                }
            }
        }
        // ---- O: combine + residual -> x(l+1) ---------------------------------
        fstamp(ftr, l, 7);
        grid_barrier(a.bar, a.bar_mode);
        fstamp(ftr, l, 8);
        if (blockIdx.x == 0 && tid < 2) a.sched[2 * l + tid] = 0;  // this layer's pools, for the next step
        {
            const int nb = d / (kFinOQuads * 4);
            const size_t kstride = static_cast<size_t>(k) * d;
            for (int b = blockIdx.x; b < nb; b += gridDim.x) {
                // threads [jj*64, jj*64+64) sum slot inv[jj]'s K-parts (all
                // loads in flight together); the combine then runs in jj order
                const int j0 = b * (kFinOQuads * 4);
                const int jj = tid / kFinOThreads, r = tid % kFinOThreads;
                const int q = r % kFinOQuads, kg = r / kFinOQuads;
                const int j = j0 + q * 4;
                if (jj < k) {
                    const int slot = s_inv[jj];
                    redo[jj][kg][q] = sum_kparts(a.part1 + static_cast<size_t>(slot) * d + j, kstride, st[1].kp[slot], kg);
                }
                __syncthreads();
                if (tid < kFinOQuads) {
                    float acc[4];
#pragma unroll
                    for (int u = 0; u < 4; ++u) acc[u] = bf2f(xl[j + u]);
                    for (int jx = 0; jx < k; ++jx) {
                        float4 s4 = redo[jx][0][q];
#pragma unroll
                        for (int k2 = 1; k2 < kKG; ++k2) {
                            const float4 c = redo[jx][k2][q];
                            s4.x += c.x; s4.y += c.y; s4.z += c.z; s4.w += c.w;
                        }
                        const float w = s_w[jx];
                        acc[0] = __fmaf_rn(w, s4.x, acc[0]);
                        acc[1] = __fmaf_rn(w, s4.y, acc[1]);
                        acc[2] = __fmaf_rn(w, s4.z, acc[2]);
                        acc[3] = __fmaf_rn(w, s4.w, acc[3]);
                    }
#pragma unroll
                    for (int u = 0; u < 4; ++u) yl[j + u] = f2bf(acc[u]);
                }
                __syncthreads();
            }
        }
        fstamp(ftr, l, 9);
        if (l + 1 < a.L) {
            if (warp < E) preload_w(wpre, wgl + static_cast<size_t>(E) * d + static_cast<size_t>(warp) * d, d, lane);
            grid_barrier(a.bar, a.bar_mode);
        }
    }
}

// ===========================================================================
// Dataflow batch-1 decode step (decode_flow_kernel): the whole L-layer stack
// in one cooperative launch like decode_step_kernel, with its intra-layer
// grid barriers replaced by data readiness, so HBM streams through the
// gate/up -> SwiGLU -> down hand-off without a gap:
//   * items of both passes are dealt round-robin (item i -> warp i mod W,
//     warps numbered SM-fastest) in h-chunk order: the gate/up items of h
//     chunk c (8 SwiGLU units of 128 h rows) precede those of chunk c+1, and
//     a warp runs straight from its last gate/up item into its down items;
//     each lane decodes one of the warp's next 32 items, so the per-item cost
//     is two shuffles;
//   * streaming warps only store their fp32 partials: no counters, no
//     fences.  The partial buffers hold a sentinel (0xffffffff, a NaN no
//     arithmetic produces) wherever no partial is pending;
//   * a ninth "finisher" warp per CTA owns the SwiGLU units and 16-row output
//     tiles of index = blockIdx mod gridDim.  It polls a unit's last partial,
//     then loads them all; once none is the sentinel it runs the SwiGLU
//     (h rows -> global), puts the sentinel back and release-increments the
//     unit's h-chunk counter.  It polls every h-chunk counter and bulk-copies
//     each complete chunk into the CTA's resident h rows (one mbarrier per
//     chunk, which the down items wait on), and finishes its output tiles the
//     same way (combine + residual -> x(l+1), then the layer's x-ready counter);
//   * a layer starts by loading x(l) until none of it is the 0xffff sentinel
//     (3 rotating row buffers; see ld_relaxed_u4 below).
// Sums, SwiGLU and combine are the K-part orders of finalize_h /
// finalize_out (sum_kparts, swiglu_store), so the output is bit-identical to
// the per-layer kernels.  Counters live per layer in a.flow_ctl; the last
// CTA to finish zeroes them for the next step.
constexpr int kFlowStage = CfgDecode::kW + CfgDecode::kW / 32;  // ring stage: one item + its int4 scales
constexpr int kFlowMaxChunks = 16;                    // 1024-row h chunks per slot (f <= 16384)
constexpr uint32_t kFlowSentinel = 0xffffffffu;       // "no partial here" (memset 0xff)

struct FlowTab {
    const uint8_t* w[2][2];   // [pass][slot] fragment blocks of the slot's expert
    const uint8_t* sc[2][2];  // int4 scales
    int gk[2][2];             // 128-K groups per item
    int kp[2][2];             // K-parts per row tile
    int p4[2];                // slot's expert is int4
    int U[2];                 // gate/up items per SwiGLU unit: 16 row tiles x kp[0][s]
    int N0, N1;               // items per pass
    int stride0, stride1;     // items per full chunk
};

struct FItem {
    int pass, s, rt, kp, c;
};

MOE_DEVI FItem flow_item(const FlowTab& T, int i, int Gf, int f16, int RT1) {
    FItem it;
    if (i < T.N0) {  // chunk c, slot s, unit u of the chunk, tile t16 (8 gate, 8 up), K-part
        const int c = i / T.stride0;
        int r = i - c * T.stride0;
        const int nu = min(8, Gf - 8 * c);
        const int s = r < nu * T.U[0] ? 0 : 1;
        if (s) r -= nu * T.U[0];
        const int u = r / T.U[s];
        const int r2 = r - u * T.U[s];
        const int kp = T.kp[0][s];
        const int t16 = r2 / kp;
        const int g = 8 * c + u;
        it.pass = 0;
        it.s = s;
        it.kp = r2 - t16 * kp;
        it.c = c;
        it.rt = t16 < 8 ? g * 8 + t16 : f16 + g * 8 + (t16 - 8);
    } else {  // chunk c, slot s, output tile rt, K-part of the chunk
        const int j = i - T.N0;
        const int c = j / T.stride1;
        int r = j - c * T.stride1;
        const int nu = min(8, Gf - 8 * c);
        const int nk0 = nu / T.gk[1][0];
        const int s = r < nk0 * RT1 ? 0 : 1;
        if (s) r -= nk0 * RT1;
        const int nk = s ? nu / T.gk[1][1] : nk0;
        const int rt = r / nk;
        it.pass = 1;
        it.s = s;
        it.rt = rt;
        it.c = c;
        it.kp = (8 * c) / T.gk[1][s] + (r - rt * nk);
    }
    return it;
}
// packed: w0 = rt | kp << 16, w1 = pass | s << 1 | c << 2 (w1 < 0: no item)
MOE_DEVI void flow_pack(const FItem& it, int& w0, int& w1) {
    w0 = it.rt | (it.kp << 16);
    w1 = it.pass | (it.s << 1) | (it.c << 2);
}
MOE_DEVI FItem flow_unpack(int w0, int w1) {
    FItem it;
    it.rt = w0 & 0xffff;
    it.kp = w0 >> 16;
    it.pass = w1 & 1;
    it.s = (w1 >> 1) & 1;
    it.c = w1 >> 2;
    return it;
}

template <class C>
MOE_DEVI void flow_issue(const FlowTab& T, const FItem& it, int K, uint8_t* stage, uint64_t* bar, uint64_t pol) {
    const int gk = T.gk[it.pass][it.s];
    const bool p4 = T.p4[it.s] != 0;
    const int wb = p4 ? gk * 1024 : gk * 4096, sb = p4 ? gk * 32 : 0;
    mbar_expect_tx(bar, wb + sb);
    const size_t blk = static_cast<size_t>(it.rt) * (K / 128) + static_cast<size_t>(it.kp) * gk;
    bulk_g2s_hint(stage, T.w[it.pass][it.s] + blk * (p4 ? 1024 : 4096), wb, bar, pol);
    if (p4) bulk_g2s_hint(stage + C::kStageS, T.sc[it.pass][it.s] + blk * 32, sb, bar, pol);
}

// compute_item's arithmetic for one resident token row
template <class C>
MOE_DEVI void flow_compute(const uint8_t* sp, const uint8_t* bp, const float* x0, int gk, bool p4, int lane,
                           float (&acc)[4]) {
    if (p4) {
        if (gk == 8) {
#pragma unroll
            for (int g = 0; g < 8; ++g)
                group_int4(sp + g * 1024, sp + C::kStageS + g * 32, bp + g * 256, x0[g], x0[g], lane, acc);
        } else {
            for (int g = 0; g < gk; ++g)
                group_int4(sp + g * 1024, sp + C::kStageS + g * 32, bp + g * 256, x0[g], x0[g], lane, acc);
        }
    } else {
        float c1[4] = {0.f, 0.f, 0.f, 0.f};
        group_bf16(sp, bp, lane, acc, c1);
        if (gk == 2) group_bf16(sp + 4096, bp + 256, lane, acc, c1);
#pragma unroll
        for (int r = 0; r < 4; ++r) acc[r] += c1[r];
    }
}

// Layer-output rows of the dataflow step (x(1) .. x(L-1)) rotate through 3
// buffers holding 0xffff (a bf16 NaN f2bf never produces) wherever a row
// element is not yet written.  A layer starts by loading x(l) itself until no
// element is the sentinel -- one L2 round trip instead of a counter acquire
// followed by the row load.  Layer m's finisher resets its own tiles of
// buffer (m+1)%3 (x(m-1): every CTA finished reading it, since x(m) is
// complete) before its first x(m+1) store, with a release fence between; the
// readers' acquire fence after the load closes the pair.  The last CTA out
// resets all three for the next launch.
MOE_DEVI uint4 ld_relaxed_u4(const void* p) {
    uint4 v;
    asm volatile("ld.relaxed.gpu.global.v4.u32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                 : "l"(p)
                 : "memory");
    return v;
}
MOE_DEVI bool has_x_sentinel(const uint4& v) {
    return (__vcmpeq2(v.x, 0xffffffffu) | __vcmpeq2(v.y, 0xffffffffu) | __vcmpeq2(v.z, 0xffffffffu) |
            __vcmpeq2(v.w, 0xffffffffu)) != 0u;
}
MOE_DEVI uint16_t* flow_xbuf(const MoeDecodeArgs& a, int i) { return i == 0 ? a.xbuf0 : i == 1 ? a.xbuf1 : a.xbuf2; }

MOE_DEVI void red_release_gpu(unsigned int* p, unsigned int v) {
    asm volatile("red.release.gpu.global.add.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
MOE_DEVI uint32_t ld_relaxed_u32(const void* p) {
    uint32_t v;
    asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
MOE_DEVI float4 ld_relaxed_f4(const float* p) {
    float4 v;
    asm volatile("ld.relaxed.gpu.global.v4.f32 {%0,%1,%2,%3}, [%4];"
                 : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
                 : "l"(p)
                 : "memory");
    return v;
}
MOE_DEVI void st_relaxed_f32(float* p, float v) {
    asm volatile("st.relaxed.gpu.global.f32 [%0], %1;" ::"l"(p), "f"(v) : "memory");
}
MOE_DEVI void st_sentinel4(float* p) {
    const float s = __uint_as_float(kFlowSentinel);
    asm volatile("st.relaxed.gpu.global.v4.f32 [%0], {%1,%1,%1,%1};" ::"l"(p), "f"(s) : "memory");
}
MOE_DEVI bool has_sentinel(const float4& v) {
    return __float_as_uint(v.x) == kFlowSentinel || __float_as_uint(v.y) == kFlowSentinel ||
           __float_as_uint(v.z) == kFlowSentinel || __float_as_uint(v.w) == kFlowSentinel;
}

// sum_kparts without its loop (KP <= 8 * kKG): the same additions in the
// same order -- acc_u = 0 + v(kg + u*kKG) (0 past KP), then acc_0 + acc_1 +
// ... + acc_7 -- with every load issued up front; *miss set if a loaded
// partial is still the sentinel.
MOE_DEVI float4 sum_kparts_r(const float* p, size_t kstride, int KP, int kg, bool* miss) {
    float4 v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u)
        v[u] = kg + u * kKG < KP ? ld_relaxed_f4(p + (kg + u * kKG) * kstride) : make_float4(0.f, 0.f, 0.f, 0.f);
    bool m = false;
#pragma unroll
    for (int u = 0; u < 8; ++u) m |= has_sentinel(v[u]);
    *miss = *miss || m;
    float4 acc = make_float4(0.f + v[0].x, 0.f + v[0].y, 0.f + v[0].z, 0.f + v[0].w);
#pragma unroll
    for (int u = 1; u < 8; ++u) {
        acc.x += 0.f + v[u].x; acc.y += 0.f + v[u].y; acc.z += 0.f + v[u].z; acc.w += 0.f + v[u].w;
    }
    return acc;
}

// The same for 8 * kKG < KP <= 16 * kKG: sum_kparts' two passes,
// acc_u = (0 + v(kg + u*kKG)) + v(kg + 64 + u*kKG) (0 past KP).
MOE_DEVI float4 sum_kparts_r2(const float* p, size_t kstride, int KP, int kg, bool* miss) {
    float4 acc;
    bool m = false;
#pragma unroll
    for (int u = 0; u < 8; ++u) {
        const float4 v = kg + u * kKG < KP ? ld_relaxed_f4(p + (kg + u * kKG) * kstride) : make_float4(0.f, 0.f, 0.f, 0.f);
        const float4 w = kg + 8 * kKG + u * kKG < KP ? ld_relaxed_f4(p + (kg + 8 * kKG + u * kKG) * kstride)
                                                      : make_float4(0.f, 0.f, 0.f, 0.f);
        m |= has_sentinel(v) || has_sentinel(w);
        float4 e = make_float4(0.f + v.x, 0.f + v.y, 0.f + v.z, 0.f + v.w);
        if (kg + 8 * kKG < KP) {
            e.x += w.x; e.y += w.y; e.z += w.z; e.w += w.w;
        }
        if (u == 0) {
            acc = e;
        } else {
            acc.x += e.x; acc.y += e.y; acc.z += e.z; acc.w += e.w;
        }
    }
    *miss = *miss || m;
    return acc;
}

MOE_DEVI float4 sum_kparts_any(const float* p, size_t kstride, int KP, int kg, bool* miss) {
    return KP > 8 * kKG ? sum_kparts_r2(p, kstride, KP, kg, miss) : sum_kparts_r(p, kstride, KP, kg, miss);
}

// sum over kg of sum_kparts(p, kstride, KP, kg), added in kg order: the
// finalize kernels' K-part reduction of 4 rows, for one lane.  KP <= 16
// keeps every partial in registers (all loads in flight at once).
MOE_DEVI float4 kpart_total(const float* p, size_t kstride, int KP, bool* miss) {
    if (KP <= 16) {
        float4 v[16];
#pragma unroll
        for (int i = 0; i < 16; ++i)
            v[i] = i < KP ? ld_relaxed_f4(p + i * kstride) : make_float4(0.f, 0.f, 0.f, 0.f);
        bool m = false;
#pragma unroll
        for (int i = 0; i < 16; ++i) m |= has_sentinel(v[i]);
        *miss = *miss || m;
        float4 tot = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
        for (int kg = 0; kg < kKG; ++kg) {
            const float4 z = make_float4(0.f, 0.f, 0.f, 0.f);
            const float4 x0 = v[kg], x1 = v[kg + kKG];
            float4 acc = make_float4(0.f + x0.x, 0.f + x0.y, 0.f + x0.z, 0.f + x0.w);
            acc.x += 0.f + x1.x; acc.y += 0.f + x1.y; acc.z += 0.f + x1.z; acc.w += 0.f + x1.w;
#pragma unroll
            for (int u = 2; u < 8; ++u) {  // K-parts >= 16: zero
                acc.x += 0.f + z.x; acc.y += 0.f + z.y; acc.z += 0.f + z.z; acc.w += 0.f + z.w;
            }
            if (kg == 0) {
                tot = acc;
            } else {
                tot.x += acc.x; tot.y += acc.y; tot.z += acc.z; tot.w += acc.w;
            }
        }
        return tot;
    }
    float4 tot = sum_kparts_any(p, kstride, KP, 0, miss);
#pragma unroll
    for (int kg = 1; kg < kKG; ++kg) {
        const float4 c = sum_kparts_any(p, kstride, KP, kg, miss);
        tot.x += c.x; tot.y += c.y; tot.z += c.z; tot.w += c.w;
    }
    return tot;
}

// Batch-1 routing tail (route_tail_t1's selection, weights and permutation)
// filling the flow table.
template <class C>
MOE_DEVI void route_tail_flow(const float* lg, const moe_expert_weights* ex, int E, int k, int d, int f, int lane,
                              int32_t* topi, float* wts, int32_t* inv, FlowTab& T) {
    const bool h0 = lane < E, h1 = lane + 32 < E;
    const float v0 = h0 ? lg[lane] : 0.0f, v1 = h1 ? lg[lane + 32] : 0.0f;
    const uint32_t k0 = h0 ? order_key(v0) : 0u, k1 = h1 ? order_key(v1) : 0u;
    bool a0 = h0, a1 = h1;
    int sel[2] = {0, 0};
    float sv[2] = {0.0f, 0.0f};
#pragma unroll
    for (int j = 0; j < 2; ++j) {
        if (j >= k) break;
        const uint32_t m = __reduce_max_sync(0xffffffffu, max(a0 ? k0 : 0u, a1 ? k1 : 0u));
        const uint32_t b0 = __ballot_sync(0xffffffffu, a0 && k0 == m);
        const uint32_t b1 = __ballot_sync(0xffffffffu, a1 && k1 == m);
        const int w = b0 ? __ffs(b0) - 1 : 32 + __ffs(b1) - 1;
        sel[j] = w;
        sv[j] = __shfl_sync(0xffffffffu, w < 32 ? v0 : v1, w & 31);
        if (w == lane) a0 = false;
        if (w == lane + 32) a1 = false;
    }
    float ex_[2] = {0.0f, 0.0f}, sum = 0.0f;
#pragma unroll
    for (int j = 0; j < 2; ++j)
        if (j < k) {
            ex_[j] = expf(sv[j] - sv[0]);
            sum += ex_[j];
        }
    int pos[2] = {0, 0};
#pragma unroll
    for (int j = 0; j < 2; ++j)
#pragma unroll
        for (int i = 0; i < 2; ++i)
            if (j < k && i < k && sel[i] < sel[j]) ++pos[j];
    if (lane < k) {
        const int j = lane;
        topi[j] = sel[j == 0 ? 0 : 1];
        wts[j] = ex_[j == 0 ? 0 : 1] / sum;
        inv[j] = pos[j == 0 ? 0 : 1];
    }
    // lanes (p, s) = (0|1, 0|1) at 0, 1, 16, 17: pass p of slot s
    const int p = lane >> 4, s = lane & 15;
    if (p < 2 && s < 2) {
        const int K = p ? f : d, G = K / 128;
        if (s < k) {
            int e = 0;
#pragma unroll
            for (int j = 0; j < 2; ++j)
                if (j < k && pos[j] == s) e = sel[j];
            const moe_expert_weights& W = ex[e];
            // pick_gk<C>(G, precision, 1) for resident rows without its loop: the largest
            // power of two <= cap dividing G is min(cap, lowest set bit of G)
            const int cap = W.precision == MOE_P4 ? C::kGk4 : C::kGk16;
            const int gk = min(cap, G & -G);
            T.w[p][s] = static_cast<const uint8_t*>(p == 0 ? W.w_gate_up : W.w_down);
            T.sc[p][s] = static_cast<const uint8_t*>(p == 0 ? W.s_gate_up : W.s_down);
            T.gk[p][s] = gk;
            T.kp[p][s] = G >> (__ffs(gk) - 1);
            if (p == 0) T.p4[s] = W.precision == MOE_P4 ? 1 : 0;
        } else {
            T.w[p][s] = nullptr;
            T.sc[p][s] = nullptr;
            T.gk[p][s] = 1;
            T.kp[p][s] = 0;
            if (p == 0) T.p4[s] = 0;
        }
    }
    __syncwarp();
    if (lane == 0) {
        const int Gf = f / 128, RT1 = d / 16;
        T.U[0] = 16 * T.kp[0][0];
        T.U[1] = 16 * T.kp[0][1];
        T.stride0 = 8 * (T.U[0] + T.U[1]);
        T.N0 = Gf * (T.U[0] + T.U[1]);
        const int nk = (8 >> (__ffs(T.gk[1][0]) - 1)) + (k > 1 ? 8 >> (__ffs(T.gk[1][1]) - 1) : 0);
        T.stride1 = RT1 * nk;
        T.N1 = RT1 * (T.kp[1][0] + T.kp[1][1]);
    }
}

// per-layer counter block: [k*nC h chunks][finishers done][dynamic items], padded
__host__ __device__ inline int flow_layer_words(int k, int d, int f) {
    (void)d;
    const int nC = (f / 128 + 7) / 8;
    return (k * nC + 2 + 31) / 32 * 32;
}

// The finisher warp of one layer: this CTA's SwiGLU units and output tiles
// and every h chunk, as they become ready.
template <class C>
MOE_DEVI void flow_finisher(const DecodeArgs& a, const FlowTab& T, int l, unsigned int* ctl, uint8_t* hres,
                            float* hbias, uint64_t (*hbar)[kFlowMaxChunks], uint16_t* hs, const int32_t* s_inv,
                            const float* s_w, const uint16_t* xl, uint16_t* yl, int lane,
                            unsigned long long* ftr) {
    const int d = a.d, f = a.f, k = a.k, Gf = f / 128, nC = (Gf + 7) / 8, RT1 = d / 16;
    const int grid = static_cast<int>(gridDim.x), b = static_cast<int>(blockIdx.x);
    const int bs1 = group_stride(f);
    unsigned int* hcnt = ctl;
    unsigned int* xdone = hcnt + k * nC;
    const int nU = b < k * Gf ? (k * Gf - b + grid - 1) / grid : 0;  // <= 32 (moek_decode_flow_supported)
    const int nCh = k * nC;                                             // <= 32
    const int nR = b < RT1 ? (RT1 - b + grid - 1) / grid : 0;           // <= 32
    const size_t rows2 = static_cast<size_t>(2) * f, kstride0 = static_cast<size_t>(k) * rows2;
    const size_t kstride1 = static_cast<size_t>(k) * d;
    // this layer's partial buffers (two per pass, by layer parity: a buffer's sentinel
    // resets, issued after this finisher's releases, only have to land before layer l + 2)
    float* const P0 = a.part0 + static_cast<size_t>(l & 1) * a.part0_stride;
    float* const P1 = a.part1 + static_cast<size_t>(l & 1) * a.part1_stride;
    uint32_t reset_tiles = 0;
    {  // this CTA's tiles of the row buffer x(l+2) will use, back to the sentinel (it holds x(l-1), read by now)
        uint16_t* xr = flow_xbuf(a, (l + 1) % 3);
        for (int i = lane; i < nR * 2; i += 32)
            __stcg(reinterpret_cast<uint4*>(xr + (b + (i >> 1) * grid) * 16) + (i & 1),
                   make_uint4(0xffffffffu, 0xffffffffu, 0xffffffffu, 0xffffffffu));
        __threadfence();  // release: these resets and the previous layer's partial resets before any x(l+1) store
        __syncwarp();
    }
    uint32_t pu = nU >= 32 ? 0xffffffffu : (1u << nU) - 1u;
    uint32_t pc = nCh >= 32 ? 0xffffffffu : (1u << nCh) - 1u;
    uint32_t pr = nR >= 32 ? 0xffffffffu : (1u << nR) - 1u;
    while (pu | pc | pr) {
        bool progress = false;
        // chunk counters: relaxed loads issued first, in flight with the unit loads
        // (an acquire load would hold every later load of the round behind it)
        unsigned int cval = 0;
        if ((pc >> lane) & 1u) cval = ld_relaxed_u32(hcnt + lane);
        // ---- SwiGLU units: the unit's last partial first, then all of them
        if (pu) {
            bool w = false;
            if ((pu >> lane) & 1u) {
                const int u = b + lane * grid, s = u / Gf, g = u - s * Gf;
                const float* wp = P0 + (static_cast<size_t>(T.kp[0][s] - 1) * k + s) * rows2 + f + g * 128 + 7 * 16;
                // the last two chunks' units gate the end of the layer: polled with their full loads
                w = g / 8 >= nC - 2 || ld_relaxed_u32(wp) != kFlowSentinel;
            }
            uint32_t wm = __ballot_sync(0xffffffffu, w);
            while (wm) {
                const int i = __ffs(wm) - 1;
                wm &= wm - 1;
                const int u = b + i * grid, s = u / Gf, g = u - s * Gf, KP = T.kp[0][s];
                float* pg = P0 + static_cast<size_t>(s) * rows2 + g * 128 + lane * 4;
                bool miss = false;
                const float4 gs = kpart_total(pg, kstride0, KP, &miss);
                const float4 us = kpart_total(pg + f, kstride0, KP, &miss);
                if (__any_sync(0xffffffffu, miss)) continue;
                fstamp_lane0(ftr, l, 13);  // (last written wins: the CTA's last unit) data complete
                const float gv[4] = {gs.x, gs.y, gs.z, gs.w}, uv[4] = {us.x, us.y, us.z, us.w};
                swiglu_store(gv, uv, hs, s, g, f, a.hperm, a.hperm16, a.hsum, bs1, lane);
                __syncwarp();
                if (lane == 0) red_release_gpu(hcnt + s * nC + g / 8, 1u);
                for (int kp = 0; kp < KP; ++kp) {  // consumed: back to the sentinel (after the release)
                    st_sentinel4(pg + kp * kstride0);
                    st_sentinel4(pg + f + kp * kstride0);
                }
                pu &= ~(1u << i);
                progress = true;
                fstamp_lane0(ftr, l, 8);  // released
            }
        }
        // ---- h chunks: each ready chunk lane copies its chunk
        if (pc) {
            bool ready = false;
            if ((pc >> lane) & 1u) {
                const int c = lane % nC;
                // seen complete: the acquire (one more round trip, only now) orders the copy after the units' h
                ready = cval >= static_cast<unsigned int>(min(8, Gf - 8 * c)) &&
                        ld_acquire_gpu(hcnt + lane) >= static_cast<unsigned int>(min(8, Gf - 8 * c));
            }
            if (ready) {
                const int s = lane / nC, c = lane - s * nC;
                const int nu = min(8, Gf - 8 * c);
                const bool p4 = T.p4[s] != 0;
                fence_proxy_async_global();
                uint64_t* bar = &hbar[s][c];
                mbar_expect_tx(bar, nu * 256 + (p4 ? 32 : 0));
                bulk_g2s(hres + static_cast<size_t>(s) * f * 2 + c * 2048,
                         (p4 ? a.hperm16 : a.hperm) + static_cast<size_t>(s) * f + c * 1024, nu * 256, bar);
                if (p4) bulk_g2s(hbias + s * bs1 + 8 * c, a.hsum + static_cast<size_t>(s) * bs1 + 8 * c, 32, bar);
            }
            const uint32_t rm = __ballot_sync(0xffffffffu, ready);
            pc &= ~rm;
            progress = progress || rm != 0;
            if (rm != 0 && pc == 0) fstamp_lane0(ftr, l, 9);
        }
        // ---- output tiles (their partials need every chunk): combine + residual,
        // polled by loading the partials themselves, two tiles' loads in flight together
        if (pr && pc == 0) {
            uint32_t todo = pr;
            while (todo) {
                const int i0 = __ffs(todo) - 1;
                todo &= todo - 1;
                const int i1 = todo ? __ffs(todo) - 1 : -1;
                if (i1 >= 0) todo &= todo - 1;
                const int q = lane >> 3, kg = lane & 7;
                int jx[2];
                float4 rr[2][2];
                bool miss[2] = {false, false};
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    const int i = h ? i1 : i0;
                    jx[h] = (b + (i < 0 ? 0 : i) * grid) * 16 + q * 4;
#pragma unroll
                    for (int jj = 0; jj < 2; ++jj)
                        rr[h][jj] = i >= 0 && jj < k ? sum_kparts_any(P1 + static_cast<size_t>(s_inv[jj]) * d + jx[h],
                                                                    kstride1, T.kp[1][s_inv[jj]], kg, &miss[h])
                                                     : make_float4(0.f, 0.f, 0.f, 0.f);
                }
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    const int i = h ? i1 : i0;
                    if (i < 0 || __any_sync(0xffffffffu, miss[h])) continue;
                    fstamp_lane0(ftr, l, 10);  // last tile's data complete
                    const int j = jx[h];
                    const uint2 xr = __ldcg(reinterpret_cast<const uint2*>(xl + j));
                    float acc[4] = {bf16_lo(xr.x), bf16_hi(xr.x), bf16_lo(xr.y), bf16_hi(xr.y)};
#pragma unroll
                    for (int jj = 0; jj < 2; ++jj) {
                        if (jj >= k) break;
                        const float4 r = rr[h][jj];
                        float4 s4;
                        s4.x = __shfl_sync(0xffffffffu, r.x, q * 8);
                        s4.y = __shfl_sync(0xffffffffu, r.y, q * 8);
                        s4.z = __shfl_sync(0xffffffffu, r.z, q * 8);
                        s4.w = __shfl_sync(0xffffffffu, r.w, q * 8);
#pragma unroll
                        for (int k2 = 1; k2 < kKG; ++k2) {
                            s4.x += __shfl_sync(0xffffffffu, r.x, q * 8 + k2);
                            s4.y += __shfl_sync(0xffffffffu, r.y, q * 8 + k2);
                            s4.z += __shfl_sync(0xffffffffu, r.z, q * 8 + k2);
                            s4.w += __shfl_sync(0xffffffffu, r.w, q * 8 + k2);
                        }
                        const float wj = s_w[jj];
                        acc[0] = __fmaf_rn(wj, s4.x, acc[0]);
                        acc[1] = __fmaf_rn(wj, s4.y, acc[1]);
                        acc[2] = __fmaf_rn(wj, s4.z, acc[2]);
                        acc[3] = __fmaf_rn(wj, s4.w, acc[3]);
                    }
                    if (kg == 0) {
                        const uint2 o = make_uint2(static_cast<uint32_t>(f2bf(acc[0])) | (static_cast<uint32_t>(f2bf(acc[1])) << 16),
                                                   static_cast<uint32_t>(f2bf(acc[2])) | (static_cast<uint32_t>(f2bf(acc[3])) << 16));
                        asm volatile("st.relaxed.gpu.global.v2.u32 [%0], {%1, %2};" ::"l"(yl + j), "r"(o.x), "r"(o.y)
                                     : "memory");
                    }
                    reset_tiles |= 1u << i;  // consumed: back to the sentinel after the release
                    fstamp_lane0(ftr, l, 11);  // last tile stored
                    pr &= ~(1u << i);
                    progress = true;
                }
            }
        }
        if (!progress && !(pc == 0 && pr != 0)) __nanosleep(128);  // the last tiles: poll without pause
    }
    // this finisher's output rows complete: one release per CTA and layer
    __syncwarp();
    if (lane == 0) red_release_gpu(xdone, 1u);
    for (uint32_t m = reset_tiles; m; m &= m - 1) {
        const int rt = b + (__ffs(m) - 1) * grid, q = lane >> 3, kg = lane & 7, j = rt * 16 + q * 4;
        for (int jj = 0; jj < k; ++jj) {
            const int slot = s_inv[jj];
            for (int kp = kg; kp < T.kp[1][slot]; kp += kKG)
                st_sentinel4(P1 + static_cast<size_t>(slot) * d + j + kp * kstride1);
        }
    }
    // every chunk copy into the resident h rows landed before the next layer reuses them
    for (int ch = lane; ch < nCh; ch += 32) mbar_wait(&hbar[ch / nC][ch % nC], static_cast<uint32_t>(l & 1));
    __syncwarp();
}

// NW streaming warps with NS ring stages each (+ the finisher warp)
template <class C, int NW, int NS>
__global__ void __launch_bounds__((NW + 1) * 32, 1) decode_flow_kernel(const __grid_constant__ DecodeArgs a) {
    constexpr int kStageBytes = kFlowStage;
    constexpr int kFlowWarps = NW;
    static_assert(NS == 1 || NS == 2, "one or two ring stages per warp");
    extern __shared__ __align__(128) uint8_t smem[];
    __shared__ FlowTab tab;
    __shared__ __align__(8) uint64_t bars[kFlowWarps][NS];
    __shared__ __align__(8) uint64_t hbar[2][kFlowMaxChunks];
    __shared__ __align__(16) moe_expert_weights s_ex[MOE_MAX_EXPERTS];
    __shared__ float lg_s[MOE_MAX_EXPERTS + 256];
    __shared__ int32_t s_inv[MOE_MAX_TOPK], s_topi[MOE_MAX_TOPK];
    __shared__ float s_w[MOE_MAX_TOPK];
    __shared__ __align__(16) uint16_t hs[128];
    __shared__ int s_last;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, tid = threadIdx.x;
    const int d = a.d, f = a.f, E = a.E, k = a.k;
    const int Gf = f / 128, RT1 = d / 16, f16 = f / 16;
    const int per_layer = flow_layer_words(k, d, f);
    unsigned long long* const ftr = g_fused_trace;
    if (lane == 0) {
        if (warp < kFlowWarps)
            for (int s2 = 0; s2 < NS; ++s2) mbar_init(&bars[warp][s2], 1);
        if (warp == kFlowWarps)
            for (int i = 0; i < 2 * kFlowMaxChunks; ++i) mbar_init(&hbar[i / kFlowMaxChunks][i % kFlowMaxChunks], 1);
        fence_mbar_init();
    }
    __syncthreads();
    const uint64_t pol = policy_evict_first();
    const int W = static_cast<int>(gridDim.x) * kFlowWarps;
    const int wid = warp * static_cast<int>(gridDim.x) + static_cast<int>(blockIdx.x);  // SM-fastest
    const int gr = lane >> 2, t4 = lane & 3;
    uint8_t* ring = smem + static_cast<size_t>(warp) * NS * kStageBytes;
    uint8_t* xres = smem + static_cast<size_t>(kFlowWarps) * NS * kStageBytes;  // bf16 row | fp16 row | bias
    const int bs0 = group_stride(d), bs1 = group_stride(f);
    uint8_t* hres = xres + 4 * d + 4 * bs0;                                             // k h rows | bias
    float* hbias = reinterpret_cast<float*>(hres + 2 * 2 * f);
    uint16_t* xs = reinterpret_cast<uint16_t*>(smem);  // routing scratch (rings idle)
    uint16_t* xn = xs + d;
    uint32_t phase_bits = 0;
    uint4 wpre[kPreChunks];
    if (warp < E) preload_w(wpre, a.wg + static_cast<size_t>(warp) * d, d, lane);  // the finisher warp routes too
    if (ftr != nullptr && tid == 0) {  // this SM's clock against the global timer (trace alignment)
        ftr[static_cast<size_t>(blockIdx.x) * kFusedStamps + 16] = gtimer();
        ftr[static_cast<size_t>(blockIdx.x) * kFusedStamps + 17] = clock64();
    }

    for (int l = 0; l < a.L; ++l) {
        const uint16_t* xl = l == 0 ? a.x_in : flow_xbuf(a, (l - 1) % 3);
        uint16_t* yl = l == a.L - 1 ? a.x_out : flow_xbuf(a, l % 3);
        const uint16_t* wgl = a.wg + static_cast<size_t>(l) * E * d;
        unsigned int* ctl = a.flow_ctl + static_cast<size_t>(l) * per_layer;
        fstamp(ftr, l, 0);
        // the layer's expert table while thread 0 waits for the previous layer's output
        for (int i = tid; i < E * static_cast<int>(sizeof(moe_expert_weights) / 8); i += blockDim.x)
            reinterpret_cast<uint2*>(s_ex)[i] = reinterpret_cast<const uint2*>(a.experts + static_cast<size_t>(l) * E)[i];
        __syncthreads();
        fstamp(ftr, l, 1);
        // ---- R: route the token (every CTA, identical results) --------------
        // x(l): every row load of the thread in flight at once; for l > 0 the
        // loads themselves wait for the previous layer (sentinel rows, above)
        {
            const int bd = static_cast<int>(blockDim.x) * 8;
            uint4 xv[4];
#pragma unroll
            for (int r = 0; r < 4; ++r)
                if (tid * 8 + r * bd < d)
                    xv[r] = l == 0 ? __ldcg(reinterpret_cast<const uint4*>(xl + tid * 8 + r * bd))
                                   : ld_relaxed_u4(xl + tid * 8 + r * bd);
            if (l > 0) {
                for (;;) {
                    bool miss = false;
#pragma unroll
                    for (int r = 0; r < 4; ++r)
                        if (tid * 8 + r * bd < d && has_x_sentinel(xv[r])) {
                            miss = true;
                            xv[r] = ld_relaxed_u4(xl + tid * 8 + r * bd);
                        }
                    if (!miss) break;
                }
            }
#pragma unroll
            for (int r = 0; r < 4; ++r)
                if (tid * 8 + r * bd < d) *reinterpret_cast<uint4*>(xs + tid * 8 + r * bd) = xv[r];
            for (int i = tid * 8 + 4 * bd; i < d; i += bd) {
                uint4 v = l == 0 ? __ldcg(reinterpret_cast<const uint4*>(xl + i)) : ld_relaxed_u4(xl + i);
                while (l > 0 && has_x_sentinel(v)) v = ld_relaxed_u4(xl + i);
                *reinterpret_cast<uint4*>(xs + i) = v;
            }
            if (l > 0) __threadfence();  // acquire: the writers' stores before their release fence
        }
        __syncthreads();
        if (ftr != nullptr && tid == 0)
            ftr[(static_cast<size_t>(l) * gridDim.x + blockIdx.x) * kFusedStamps + 12] = clock64();
        const uint16_t* xr = xs;
        if (a.norm_eps > 0.0f) {
            if (tid < 256) {
                float acc = 0.0f;  // route_kernel's pinned order
                for (int c = 0; c * 256 + tid < d; ++c) {
                    const float v = bf2f(xs[c * 256 + tid]);
                    acc = __fmaf_rn(v, v, acc);
                }
                lg_s[MOE_MAX_EXPERTS + tid] = acc;
            }
            __syncthreads();
            if (warp == 0) {  // the tree's levels 128, 64, 32 (one lane each), then the warp's shuffle levels
                const float* t = lg_s + MOE_MAX_EXPERTS;
                const float a0 = __fadd_rn(t[lane], t[lane + 128]), a1 = __fadd_rn(t[lane + 64], t[lane + 192]);
                const float a2 = __fadd_rn(t[lane + 32], t[lane + 160]), a3 = __fadd_rn(t[lane + 96], t[lane + 224]);
                float v = __fadd_rn(__fadd_rn(a0, a1), __fadd_rn(a2, a3));
#pragma unroll
                for (int s2 = 16; s2 >= 1; s2 >>= 1) v = __fadd_rn(v, __shfl_down_sync(0xffffffffu, v, s2));
                if (lane == 0) lg_s[MOE_MAX_EXPERTS] = v;
            }
            __syncthreads();
            const float rstd = __fdiv_rn(1.0f, __fsqrt_rn(__fadd_rn(__fdiv_rn(lg_s[MOE_MAX_EXPERTS], static_cast<float>(d)),
                                                                    a.norm_eps)));
            for (int i = tid * 8; i < d; i += blockDim.x * 8) {
                uint4 v = *reinterpret_cast<const uint4*>(xs + i);
                uint32_t w4[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
                for (int q = 0; q < 4; ++q)
                    w4[q] = static_cast<uint32_t>(f2bf(__fmul_rn(bf16_lo(w4[q]), rstd))) |
                            (static_cast<uint32_t>(f2bf(__fmul_rn(bf16_hi(w4[q]), rstd))) << 16);
                *reinterpret_cast<uint4*>(xn + i) = make_uint4(w4[0], w4[1], w4[2], w4[3]);
            }
            __syncthreads();
            xr = xn;
        }
        for (int e = warp; e < E; e += kFlowWarps + 1) {  // every warp, the finisher included: one logit each
            if (e != warp) preload_w(wpre, wgl + static_cast<size_t>(e) * d, d, lane);
            const float v = router_dot(xr, wpre, wgl + static_cast<size_t>(e) * d, d, lane);
            if (lane == 0) lg_s[e] = v;
        }
        __syncthreads();
        fstamp(ftr, l, 2);
        if (warp == 0) {
            route_tail_flow<C>(lg_s, s_ex, E, k, d, f, lane, s_topi, s_w, s_inv, tab);
            __syncwarp();
            if (blockIdx.x == 0 && lane < k) {
                a.idx[static_cast<size_t>(l) * a.idx_stride + lane] = s_topi[lane];
                a.wts[static_cast<size_t>(l) * a.idx_stride + lane] = s_w[lane];
            }
        } else if (warp < kFlowWarps) {
            // resident x row: K-permuted bf16, fp16 and the int4 bias terms
            uint16_t* rb = reinterpret_cast<uint16_t*>(xres);
            uint16_t* rh = rb + d;
            float* rx = reinterpret_cast<float*>(xres + 4 * d);
            const int G = d / 128, nw = kFlowWarps - 1;
            for (int g0 = (warp - 1) * 2; g0 < G; g0 += nw * 2) {
                const int g = g0 + (lane >> 4), c = lane & 15;
                uint4 cb = make_uint4(0, 0, 0, 0), ch = cb;
                float s_lo = 0.0f, s_hi = 0.0f, amax = 0.0f;
                if (g < G) permute_chunk(xr + g * 128, c, cb, ch, s_lo, s_hi, amax);
                numerics_group_check(amax, c == 0);
#pragma unroll
                for (int off = 8; off >= 1; off >>= 1) {
                    s_lo += __shfl_xor_sync(0xffffffffu, s_lo, off);
                    s_hi += __shfl_xor_sync(0xffffffffu, s_hi, off);
                }
                if (g < G) {
                    reinterpret_cast<uint4*>(rb + g * 128)[c] = cb;
                    reinterpret_cast<uint4*>(rh + g * 128)[c] = ch;
                    if (c == 0) rx[g] = int4_bias_term(s_lo, s_hi);
                }
            }
        }
        fence_proxy_async();  // routing scratch (generic) writes before the rings' bulk copies
        __syncthreads();
        fstamp(ftr, l, 3);
        if (l + 1 < a.L && blockIdx.x < 4 && tid == 0) {  // next layer's router weights -> L2
            const uint32_t chunk = static_cast<uint32_t>(E) * d * 2 / 4;
            if (chunk % 16 == 0)
                asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(wgl + static_cast<size_t>(E) * d +
                                                                            static_cast<size_t>(blockIdx.x) * chunk / 2),
                             "r"(chunk)
                             : "memory");
        }
        if (warp == kFlowWarps) {
            flow_finisher<C>(a, tab, l, ctl, hres, hbias, hbar, hs, s_inv, s_w, xl, yl, lane, ftr);
            if (ftr != nullptr) fstamp_lane0(ftr, l, 7);
            if (l + 1 < a.L && warp < E)
                preload_w(wpre, wgl + static_cast<size_t>(E) * d + static_cast<size_t>(warp) * d, d, lane);
            continue;
        }
        // ---- streaming: this warp's items of both passes, round-robin ------
        const FlowTab& T = tab;
        const int N = T.N0 + T.N1;
        // items [0, Ns) are dealt round-robin, the last quarter of the down pass is
        // handed out one item at a time from the layer's counter (grabbed one ahead)
        const int Ns = N - T.N1 / 4;
        const int nmine = wid < Ns ? (Ns - wid + W - 1) / W : 0;  // static items of this warp
        unsigned int* dctr = ctl + k * ((Gf + 7) / 8) + 1;
        unsigned int dgrab = 0;  // lane 0: the pre-grabbed dynamic index
        bool dstarted = false;
        // lane j holds the warp's item (batch*32 + j), packed
        int pk0 = 0, pk1 = -1;
        auto decode_batch = [&](int j0) {
            const int ix = wid + (j0 + lane) * W;
            pk1 = -1;
            if (j0 + lane < nmine) flow_pack(flow_item(T, ix, Gf, f16, RT1), pk0, pk1);
        };
        auto item_of = [&](int j) {
            if ((j & 31) == 0) decode_batch(j);
            return flow_unpack(__shfl_sync(0xffffffffu, pk0, j & 31), __shfl_sync(0xffffffffu, pk1, j & 31));
        };
        // the warp's j-th item (static, then dynamic); false when the layer is out of items
        auto next_of = [&](int j, FItem& it) -> bool {
            if (j < nmine) {
                it = item_of(j);
                if (j + 1 == nmine && lane == 0) {  // last static item: grab the first dynamic one now
                    dgrab = atomicAdd(dctr, 1u);
                    dstarted = true;
                }
                return true;
            }
            if (!dstarted) {
                if (lane == 0) dgrab = atomicAdd(dctr, 1u);
                dstarted = true;
            }
            const int ix = Ns + static_cast<int>(__shfl_sync(0xffffffffu, dgrab, 0));
            if (ix >= N) return false;
            if (lane == 0) dgrab = atomicAdd(dctr, 1u);
            it = flow_item(T, ix, Gf, f16, RT1);
            return true;
        };
        FItem it0{}, it1{};
        int issued = 0, computed = 0;
        bool more = true;
        if (next_of(0, it0)) {
            if (lane == 0) flow_issue<C>(T, it0, it0.pass ? f : d, ring, &bars[warp][0], pol);
            issued = 1;
            if (NS == 2) {
                if (next_of(1, it1)) {
                    if (lane == 0) flow_issue<C>(T, it1, it1.pass ? f : d, ring + kStageBytes, &bars[warp][1], pol);
                    issued = 2;
                } else {
                    more = false;
                }
            }
        } else {
            more = false;
        }
        bool first_down = true;
        while (computed < issued) {
            const int stage = NS == 2 ? computed & 1 : 0;
            const FItem it = stage ? it1 : it0;
            mbar_wait(&bars[warp][stage], (phase_bits >> stage) & 1u);
            phase_bits ^= 1u << stage;
            if (it.pass == 1) {
                if (first_down) {
                    first_down = false;
                    if (warp == 0) fstamp(ftr, l, 4);
                }
                mbar_wait(&hbar[it.s][it.c], static_cast<uint32_t>(l & 1));
            }
            uint8_t* sp = ring + stage * kStageBytes;
            float acc[4] = {0.f, 0.f, 0.f, 0.f};
            {
                const int gk = T.gk[it.pass][it.s];
                const bool p4 = T.p4[it.s] != 0;
                const uint8_t* bp;
                const float* x0;
                if (it.pass == 0) {
                    bp = xres + (p4 ? 2 * d : 0) + it.kp * gk * 256 + t4 * 16;
                    x0 = reinterpret_cast<const float*>(xres + 4 * d) + it.kp * gk;
                } else {
                    bp = hres + static_cast<size_t>(it.s) * f * 2 + it.kp * gk * 256 + t4 * 16;
                    x0 = hbias + it.s * bs1 + it.kp * gk;
                }
                flow_compute<C>(sp, bp, x0, gk, p4, lane, acc);
            }
            ++computed;
            fence_proxy_async();
            __syncwarp();
            FItem nit;
            if (more && next_of(issued, nit)) {
                if (lane == 0) flow_issue<C>(T, nit, nit.pass ? f : d, sp, &bars[warp][stage], pol);
                if (stage) it1 = nit; else it0 = nit;
                ++issued;
            } else {
                more = false;
            }
            const int rows = it.pass ? d : 2 * f;
            float* pp = (it.pass ? a.part1 + static_cast<size_t>(l & 1) * a.part1_stride
                                 : a.part0 + static_cast<size_t>(l & 1) * a.part0_stride) +
                        (static_cast<size_t>(it.kp) * k + it.s) * rows + it.rt * 16 + gr;
            if (t4 == 0) {
                st_relaxed_f32(pp, acc[0]);
                st_relaxed_f32(pp + 8, acc[2]);
            }
        }
        fence_proxy_async();  // resident rows / stages read (generic) before the next layer's bulk copies
        if (warp == 0) fstamp(ftr, l, 5);
        if (ftr != nullptr) fstamp_lane0(ftr, l, 15);  // the CTA's last streaming warp done (last writer wins)
        if (l + 1 < a.L && warp < E)
            preload_w(wpre, wgl + static_cast<size_t>(E) * d + static_cast<size_t>(warp) * d, d, lane);
    }
    // the last CTA out zeroes the counters for the next step
    __syncthreads();
    unsigned int* exitc = a.flow_ctl + static_cast<size_t>(a.L) * per_layer;
    if (tid == 0) {
        unsigned int old;
        asm volatile("atom.add.acq_rel.gpu.global.u32 %0, [%1], 1;" : "=r"(old) : "l"(exitc) : "memory");
        s_last = old == gridDim.x - 1;
    }
    __syncthreads();
    if (s_last) {
        const int words = a.L * per_layer;
        for (int i = tid; i < words / 4; i += blockDim.x) __stcg(reinterpret_cast<uint4*>(a.flow_ctl) + i, make_uint4(0, 0, 0, 0));
        for (int i = tid; i < 3 * (d / 8); i += blockDim.x)  // every row buffer back to the sentinel
            __stcg(reinterpret_cast<uint4*>(flow_xbuf(a, i / (d / 8))) + i % (d / 8),
                   make_uint4(0xffffffffu, 0xffffffffu, 0xffffffffu, 0xffffffffu));
        __syncthreads();
        if (tid == 0) *exitc = 0;
    }
}
}  // namespace moek

cudaError_t moek_debug_fused_trace(void* buf) {
    return cudaMemcpyToSymbol(moek::g_fused_trace, &buf, sizeof(buf));
}

size_t moek_decode_step_smem() {
    using C = moek::CfgDecode;
    return static_cast<size_t>(C::kWarps) * moek::kStages * C::kStageBytes + C::kResBytes;
}

bool moek_decode_step_supported(int E, int k, int d, int f) {
    // resident rows: <= 2 segments of K <= 14336 (CfgDecode's reserved area),
    // 256-thread routing, 32-output combine blocks
    return E >= 1 && E <= MOE_MAX_EXPERTS && k >= 1 && k <= 2 && k <= E && d % 256 == 0 && f % 128 == 0 &&
           d <= 14336 && f <= 14336 && moek::group_stride(f) <= 512 && moek::group_stride(d) <= 512 &&
           4 * d + 4 * moek::group_stride(d) <= moek::CfgDecode::kResBytes;
}

cudaError_t moek_decode_step(const MoeDecodeArgs& a, cudaStream_t stream) {
    using C = moek::CfgDecode;
    static int grid = 0;
    const size_t smem = moek_decode_step_smem();
    if (grid == 0) {
        MOE_CUDA_OK(cudaFuncSetAttribute(moek::decode_step_kernel<C>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(smem)));
        int dev = 0, sms = 0, per = 0;
        MOE_CUDA_OK(cudaGetDevice(&dev));
        MOE_CUDA_OK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
        MOE_CUDA_OK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, moek::decode_step_kernel<C>, C::kThreads, smem));
        if (per < 1) return cudaErrorCooperativeLaunchTooLarge;
        grid = sms;
    }
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(C::kThreads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = stream;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeCooperative;  // every CTA co-resident: the grid barriers rely on it
    attr[0].val.cooperative = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, moek::decode_step_kernel<C>, a);
}
int moek_group_stride(int K) { return moek::group_stride(K); }

namespace {
// streaming-warp x stage shapes of the dataflow step (MOE_FLOW_CFG picks one; A/B)
struct FlowShape {
    int nw, ns;
};
FlowShape flow_shape() {
    static FlowShape sh{0, 0};
    if (sh.nw == 0) {
        sh = FlowShape{7, 2};
        if (const char* e = getenv("MOE_FLOW_CFG")) {
            int nw = 0, ns = 0;
            if (sscanf(e, "%dx%d", &nw, &ns) == 2) sh = FlowShape{nw, ns};
        }
    }
    return sh;
}
template <int NW, int NS>
cudaError_t launch_flow(const MoeDecodeArgs& a, size_t smem, cudaStream_t stream) {
    using C = moek::CfgDecode;
    auto kern = moek::decode_flow_kernel<C, NW, NS>;
    static size_t smem_set = 0;
    static int grid = 0;
    if (smem > smem_set) {
        MOE_CUDA_OK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
        smem_set = smem;
    }
    if (grid == 0) {
        int dev = 0, sms = 0, per = 0;
        MOE_CUDA_OK(cudaGetDevice(&dev));
        MOE_CUDA_OK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
        MOE_CUDA_OK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, kern, (NW + 1) * 32, smem));
        if (per < 1) return cudaErrorCooperativeLaunchTooLarge;
        grid = sms;
    }
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3((NW + 1) * 32);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = stream;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeCooperative;  // every CTA co-resident: the readiness waits rely on it
    attr[0].val.cooperative = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, kern, a);
}
}  // namespace

size_t moek_decode_flow_smem(int d, int f) {
    const FlowShape sh = flow_shape();
    return static_cast<size_t>(sh.nw) * sh.ns * moek::kFlowStage + 4 * static_cast<size_t>(d) +
           4 * moek::group_stride(d) + 4 * static_cast<size_t>(f) + 8 * moek::group_stride(f);
}

size_t moek_decode_flow_ctl_words(int L, int k, int d, int f) {
    return static_cast<size_t>(L) * moek::flow_layer_words(k, d, f) + 32;
}

bool moek_decode_flow_supported(int E, int k, int d, int f, int sms) {
    if (!moek_decode_step_supported(E, k, d, f) || sms < 1) return false;
    const int Gf = f / 128, nC = (Gf + 7) / 8;
    // one finisher warp per CTA: <= 32 units, h chunks and output tiles each (a lane apiece)
    const bool fin = (k * Gf + sms - 1) / sms <= 32 && k * nC <= 32 && (d / 16 + sms - 1) / sms <= 32;
    return nC <= moek::kFlowMaxChunks && d / 128 <= 2 * 64 && Gf <= 2 * 64 && fin &&
           moek_decode_flow_smem(d, f) + 8 * 1024 <= 227 * 1024;
}

cudaError_t moek_decode_flow(const MoeDecodeArgs& a, cudaStream_t stream) {
    const size_t smem = moek_decode_flow_smem(a.d, a.f);
    const FlowShape sh = flow_shape();
    if (sh.nw == 15 && sh.ns == 1) return launch_flow<15, 1>(a, smem, stream);
    if (sh.nw == 15 && sh.ns == 2) return launch_flow<15, 2>(a, smem, stream);
    if (sh.nw == 11 && sh.ns == 2) return launch_flow<11, 2>(a, smem, stream);
    if (sh.nw == 11 && sh.ns == 1) return launch_flow<11, 1>(a, smem, stream);
    if (sh.nw == 7 && sh.ns == 2) return launch_flow<7, 2>(a, smem, stream);
    if (sh.nw == 8 && sh.ns == 2) return launch_flow<8, 2>(a, smem, stream);
    return cudaErrorInvalidValue;
}
// Largest T whose (active expert, 8-token tile) segments always fit the
// kernel's table: at most min(E, T*k) experts are active and their segments
// number at most min(E, T*k) + ceil(T*k / 8).
int moek_gemv_max_tokens(int E, int k) {
    if (E < 1 || k < 1) return 0;
    int T = 0;
    while (std::min(E, (T + 1) * k) + ((T + 1) * k + moek::kTile - 1) / moek::kTile <= moek::kMaxSegs) ++T;
    return T;
}
namespace moek {

template <class C>
cudaError_t launch_stream_cfg(const StreamArgs& a, bool pdl, cudaStream_t stream) {
    static int grid = 0;
    const size_t smem = static_cast<size_t>(C::kWarps) * kStages * C::kStageBytes + C::kResBytes;
    if (grid == 0) {
        MOE_CUDA_OK(cudaFuncSetAttribute(stream_kernel<C>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
        int dev = 0, sms = 0;
        MOE_CUDA_OK(cudaGetDevice(&dev));
        MOE_CUDA_OK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
        grid = sms;
    }
    if (pdl) return launch_pdl(stream_kernel<C>, dim3(grid), dim3(C::kThreads), smem, stream, a);
    stream_kernel<C><<<grid, C::kThreads, smem, stream>>>(a);
    return cudaGetLastError();
}

cudaError_t launch_stream(const StreamArgs& a, bool pdl, cudaStream_t stream) {
    static const bool dec = getenv("MOE_GEMV_CFG") == nullptr || atoi(getenv("MOE_GEMV_CFG")) != 0;
    // resident rows: one token, <= 2 segments (k <= 2), rows and bias fit the reserved area
    if (dec && a.T == 1 && a.k <= 2 && a.K <= 14336 && a.bstride <= 512) return launch_stream_cfg<CfgDecode>(a, pdl, stream);
    return launch_stream_cfg<CfgBatch>(a, pdl, stream);
}

}  // namespace moek

namespace {

size_t align256(size_t v) { return (v + 255) / 256 * 256; }

struct WsSizes {
    size_t xperm, xperm16, xsum, hperm, hperm16, hsum, part0, part1, kpslot, sched;
};

WsSizes ws_sizes(int T, int k, int d, int f) {
    const size_t slots = static_cast<size_t>(T) * k;
    WsSizes w;
    w.xperm = static_cast<size_t>(T) * d * 2;
    w.xperm16 = w.xperm;
    w.xsum = static_cast<size_t>(T) * moek::group_stride(d) * 4;
    w.hperm = slots * f * 2;
    w.hperm16 = w.hperm;
    w.hsum = slots * moek::group_stride(f) * 4;
    w.part0 = static_cast<size_t>(d / 128) * slots * 2 * f * 4;  // K-parts <= 128-K groups
    w.part1 = static_cast<size_t>(f / 128) * slots * d * 4;
    w.kpslot = slots * 2 * 4;
    w.sched = 16;
    return w;
}

}  // namespace

cudaError_t moek_debug_gemv_trace(void* buf) {
    return cudaMemcpyToSymbol(moek::g_gemv_trace, &buf, sizeof(buf));
}

cudaError_t moek_debug_layer_trace_router(void* buf, cudaStream_t stream);
cudaError_t moek_debug_layer_trace(void* buf, cudaStream_t stream) {
    // stream-ordered (pinned staging), so a trace can cover exactly one replay
    static void** host = nullptr;
    if (host == nullptr) MOE_CUDA_OK(cudaMallocHost(&host, 64 * sizeof(void*)));
    static int next = 0;
    void** h = host + (next++ & 63);
    *h = buf;
    MOE_CUDA_OK(cudaMemcpyToSymbolAsync(moek::g_layer_trace, h, sizeof(buf), 0, cudaMemcpyHostToDevice, stream));
    return moek_debug_layer_trace_router(h, stream);
}

size_t moek_gemv_workspace_bytes(int T, int k, int d, int f) {
    const WsSizes w = ws_sizes(T, k, d, f);
    return align256(w.xperm) + align256(w.xperm16) + align256(w.xsum) + align256(w.hperm) + align256(w.hperm16) +
           align256(w.hsum) + align256(w.part0) + align256(w.part1) + align256(w.kpslot) + align256(w.sched);
}

GemvWorkspace moek_gemv_workspace_view(void* base, int T, int k, int d, int f) {
    const WsSizes w = ws_sizes(T, k, d, f);
    char* p = static_cast<char*>(base);
    GemvWorkspace ws{};
    auto take = [&](size_t bytes) {
        char* r = p;
        p += align256(bytes);
        return r;
    };
    ws.xperm = take(w.xperm);
    ws.xperm16 = take(w.xperm16);
    ws.xsum = reinterpret_cast<float*>(take(w.xsum));
    ws.hperm = take(w.hperm);
    ws.hperm16 = take(w.hperm16);
    ws.hsum = reinterpret_cast<float*>(take(w.hsum));
    ws.part0 = reinterpret_cast<float*>(take(w.part0));
    ws.part1 = reinterpret_cast<float*>(take(w.part1));
    ws.kpslot = reinterpret_cast<int*>(take(w.kpslot));
    ws.sched = reinterpret_cast<unsigned int*>(take(w.sched));
    return ws;
}

cudaError_t moek_permute_rows(const void* x, int rows, int K, void* xperm, void* xperm16, float* xsum,
                              cudaStream_t stream) {
    const long long halves = static_cast<long long>(rows) * (K / 128);
    if (halves == 0) return cudaSuccess;
    return moek::launch_pdl(moek::permute_rows_kernel, dim3(static_cast<unsigned>((halves * 16 + 255) / 256)), dim3(256),
                            0, stream, static_cast<const uint16_t*>(x), rows, K, static_cast<uint16_t*>(xperm),
                            static_cast<uint16_t*>(xperm16), xsum, moek::group_stride(K));
}

cudaError_t moek_ffn_mma(const GemvWorkspace& ws, const void* x, const int32_t* perm, const int32_t* offsets,
                         const int32_t* inv, const float* wts, const void* resid, int T, int k,
                         const moe_expert_weights* experts, int E, int d, int f, uint64_t active_mask, void* out,
                         float* y, int xmode, cudaStream_t stream) {
    // every (active expert, 8-token tile) segment must fit the kernel's table
    if (moek_gemv_max_tokens(E, k) < T) return cudaErrorInvalidValue;
    if (d % (moek::kFinOQuads * 4) != 0 || f % 128 != 0) return cudaErrorInvalidValue;
    if (xmode == MOE_X_PERMUTE) MOE_CUDA_OK(moek_permute_rows(x, T, d, ws.xperm, ws.xperm16, ws.xsum, stream));
    const int nslots = T * k;
    moek::StreamArgs a{};
    a.offsets = offsets;
    a.perm = perm;
    a.T = T;
    a.k = k;
    a.kshift = (k & (k - 1)) == 0 ? __builtin_ctz(static_cast<unsigned>(k)) : -1;
    a.E = E;
    a.active_mask = active_mask;
    for (int e = 0; e < E; ++e) a.ex[e] = experts[e];
    // gate/up pass
    a.p = 0;
    a.rows = 2 * f;
    a.K = d;
    a.b16 = static_cast<const uint16_t*>(ws.xperm);
    a.b16h = static_cast<const uint16_t*>(ws.xperm16);
    a.bsum = ws.xsum;
    a.bstride = moek::group_stride(d);
    a.part = ws.part0;
    a.kpslot = ws.kpslot;
    a.sched = ws.sched;
    static const int dbg = getenv("MOE_GEMV_DBG") ? atoi(getenv("MOE_GEMV_DBG")) : 0;
    a.dbg = dbg;
    a.wait_first = xmode == MOE_X_ROUTED ? 1 : 0;
    MOE_CUDA_OK(moek::launch_stream(a, xmode != MOE_X_READY, stream));
    {
        MOE_CUDA_OK(moek::launch_pdl(moek::finalize_h_kernel, dim3(nslots * (f / 128)), dim3(moek::kFinHThreads), 0, stream,
                                     static_cast<const float*>(ws.part0), static_cast<const int*>(ws.kpslot), nslots, f,
                                     static_cast<uint16_t*>(ws.hperm), static_cast<uint16_t*>(ws.hperm16), ws.hsum,
                                     moek::group_stride(f), ws.sched));
    }
    // down pass
    a.p = 1;
    a.rows = d;
    a.K = f;
    a.b16 = static_cast<const uint16_t*>(ws.hperm);
    a.b16h = static_cast<const uint16_t*>(ws.hperm16);
    a.bsum = ws.hsum;
    a.bstride = moek::group_stride(f);
    a.part = ws.part1;
    a.kpslot = ws.kpslot + nslots;
    a.sched = ws.sched + 1;
    a.wait_first = 0;
    MOE_CUDA_OK(moek::launch_stream(a, true, stream));
    return moek::launch_pdl(moek::finalize_out_kernel,
                            dim3(static_cast<unsigned>((out ? T : nslots) * (d / (moek::kFinOQuads * 4)))),
                            dim3(moek::kFinOThreads), 0,
                            stream, static_cast<const float*>(ws.part1), static_cast<const int*>(ws.kpslot + nslots), T, k,
                            d, inv, wts, static_cast<const uint16_t*>(resid), static_cast<uint16_t*>(out), y,
                            ws.sched + 1);
}

MOE_NUMERICS_BINDER(gemv)

// Loads this unit's kernels now (cudaFuncGetAttributes).  Under lazy module
// loading (CUDA 12 default) a kernel's first launch may wait for the device
// to idle; the expert-parallel step has kernels that spin on a peer's flags,
// so every kernel it can launch must be resident before the first step.
cudaError_t moek_preload_gemv() {
    cudaFuncAttributes fa;
    MOE_CUDA_OK_PRELOAD(cudaFuncGetAttributes(&fa, moek::stream_kernel<moek::CfgBatch>));
    MOE_CUDA_OK_PRELOAD(cudaFuncGetAttributes(&fa, moek::stream_kernel<moek::CfgDecode>));
    MOE_CUDA_OK_PRELOAD(cudaFuncGetAttributes(&fa, moek::finalize_h_kernel));
    MOE_CUDA_OK_PRELOAD(cudaFuncGetAttributes(&fa, moek::finalize_out_kernel));
    MOE_CUDA_OK_PRELOAD(cudaFuncGetAttributes(&fa, moek::permute_rows_kernel));
    MOE_CUDA_OK_PRELOAD(cudaFuncGetAttributes(&fa, moek::decode_step_kernel<moek::CfgDecode>));
    MOE_CUDA_OK_PRELOAD(cudaFuncGetAttributes(&fa, moek::decode_flow_kernel<moek::CfgDecode, 7, 2>));
    return cudaSuccess;
}
