// tc_gemm.cu -- K3/K4 expert FFN on the 5th-generation tensor cores
// (tcgen05.mma, fp32 accumulators in TMEM) for batched decode / prefill,
// where an expert sees enough tokens that the contraction is a real GEMM.
//
// One CTA computes a 128-weight-row x (128 | 256)-token tile of one expert:
//   pass 0: D_gate, D_up = W_gate/up[rows] . X[tokens]^T -> fused SwiGLU
//           epilogue h = bf16(silu(g) * u) (+ its fp16 copy) for the tile
//   pass 1: D = W_down[rows] . H[tokens]^T -> y[slot][row] (fp32), combined
//           afterwards by the K5 combine kernel.
// Data path per 64-K chunk, warp-specialised, all hand-offs on mbarriers:
//   weights: HBM --bulk copy--> raw smem ring (fragment-block storage
//     layout) --converter warps--> canonical K-major SWIZZLE_128B A tiles;
//   tokens:  slot-ordered rows (gather kernel; h is slot-ordered already)
//     --TMA 2D boxes, 128-byte swizzle--> canonical B tiles;
//   one thread issues tcgen05.mma (M = 128, N = the tile's tokens rounded
//   to 16, K = 16 x 4) into TMEM; tcgen05.commit frees the stages.  bf16 experts run kind::f16 with BF16 operands; int4-g128 experts
//   are dequantised in the convert step to fp16 q*s (exact: <= 11
//   significant bits, for normal-range scales) and run with F16 operands
//   against an fp16 copy of the activations.
// The storage layout stays the GEMV's (fragment blocks), so one copy of the
// weights serves both paths.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <cstdlib>

#include <cstdio>
#include "common.cuh"
#include "launch.h"

namespace moek {
namespace tc {

constexpr int kM = 128;        // weight rows per tile (UMMA M)
constexpr int kKc = 64;        // K per chunk (one 128-byte swizzle atom of 16-bit values)
constexpr int kTileBytes = kM * kKc * 2;  // 16 KB (A tile; B tile is the same for kN = 128)
// raw stage: [A_gate raw 16 KB][A_up raw 16 KB][scales 2 x 256 B]
constexpr int kRawA = 16384;
constexpr int kRawS = 256;
constexpr int kRawBytes = 2 * kRawA + 2 * kRawS;  // weights only: token rows go straight to the canonical tile

struct TcArgs {
    // B operand tensor maps (2D: K x rows in slot order, 64 x 64 boxes,
    // SWIZZLE_128B): pass 0 the slot-ordered token rows (bf16 / fp16 copy),
    // pass 1 h (bf16 / fp16)
    CUtensorMap tmb;
    CUtensorMap tmb16;
    // fused persistent launch (tc_ffn_persist, fused = 1): the down pass's B maps (h),
    // and per (expert, token tile, K split) counters of finished gate/up tiles
    CUtensorMap tmh;
    CUtensorMap tmh16;
    unsigned int* dep;
    int dep_tt;               // token tiles per expert in dep's index
    const int32_t* offsets;   // [E+1]
    const int32_t* perm;      // [T*k]
    int T, k, E, kshift;
    int p;                    // 0 gate/up, 1 down
    int d, f;
    uint16_t* hout;           // pass 0: h [T*k][f] bf16
    uint16_t* hout16;         // pass 0: h [T*k][f] fp16
    float* y;                 // pass 1: y [T*k][d]
    uint64_t active_mask;
    int dbg;                  // MOE_TC_DBG (A/B and ablation switches, 0 in production):
                              // kernel ablations: bit0 skip convert, bit1 skip MMA, bit2 skip weight
                              // loads, bit5 bf16 halves as separate 2 KB reads, bit11 skip epilogue
                              // stores, bit12 skip B loads, bit13 plain arrives instead of commits,
                              // bit15 clock probe (-DMOE_TC_TRACE=1 builds), bit16/17 weight L2
                              // prefetch; dispatch: bit3/4 force 128/256-token tiles, bit8 per-tile
                              // (non-persistent) 128-token kernel, bit9 no down-pass K split, bit14
                              // no persistent wide kernel, bit18 single-CTA wide kernel, bit19
                              // release.cluster forwarder arrive, bit21 two launches instead of the
                              // fused one, bit22 split_reduce + combine, bit23 int4 wide tiles on
                              // tc_ffn_kernel<256>
    moe_expert_weights ex[MOE_MAX_EXPERTS];
};

MOE_DEVI uint32_t s32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }

MOE_DEVI void mbar_wait(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "W_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra W_%=;\n}" ::"r"(s32(bar)),
        "r"(parity)
        : "memory");
}

// SWIZZLE_128B K-major smem descriptor (sm100 version 1): start >> 4, LBO 16 B
// (unused for swizzled K-major), SBO 1024 B between 8-row groups.
MOE_DEVI uint64_t sdesc(uint32_t addr) {
    return static_cast<uint64_t>((addr >> 4) & 0x3FFFu) | (1ull << 16) | (64ull << 32) | (1ull << 46) | (2ull << 61);
}
// No-swizzle K-major descriptor over core-matrix storage (the bf16 weight
// blocks as bulk-copied: 8 x 8 core matrices of 128 contiguous bytes, 128 B
// apart along K (leading dimension), 1024 B apart along M (stride dimension)).
MOE_DEVI uint64_t sdesc_core(uint32_t addr) {
    return static_cast<uint64_t>((addr >> 4) & 0x3FFFu) | (8ull << 16) | (64ull << 32) | (1ull << 46);
}
// kind::f16 instruction descriptor: D f32, A/B format (0 f16, 1 bf16), K-major, N, M.
MOE_DEVI uint32_t idesc(int fmt, int n, int m) {
    return (1u << 4) | (static_cast<uint32_t>(fmt) << 7) | (static_cast<uint32_t>(fmt) << 10) |
           (static_cast<uint32_t>(n >> 3) << 17) | (static_cast<uint32_t>(m >> 4) << 24);
}
MOE_DEVI void umma(uint32_t dtmem, uint64_t a, uint64_t b, uint32_t id, uint32_t accum) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}" ::"r"(dtmem),
        "l"(a), "l"(b), "r"(id), "r"(accum)
        : "memory");
}
// SiLU for the tcgen05 epilogues (MUFU ex2 + fast divide, a few ulp of fp32,
// far inside the bf16 rounding of h): the pass-0 epilogue holds the
// accumulator while it runs, so its instruction count is on the critical path
MOE_DEVI float silu_fast(float g) { return __fdividef(g, 1.0f + __expf(-g)); }
// silu(g) = g/2 * (1 + tanh(g/2)): one MUFU op instead of two (ex2 + rcp) --
// the pass-0 drain of tc_ffn_wide is MUFU-bound; tanh.approx's ~2^-11
// relative error stays below h's bf16 rounding step (2^-8)
MOE_DEVI float silu_tanh(float g) {
    const float hg = 0.5f * g;
    float t;
    asm("tanh.approx.f32 %0, %1;" : "=f"(t) : "f"(hg));
    return __fmaf_rn(hg, t, hg);
}

// (lo, hi) -> packed bf16x2, round to nearest even (one F2FP; NaN -> 0x7fff, not f2bf's 0x7fc0)
MOE_DEVI uint32_t bf16x2_rn(float lo, float hi) {
    uint32_t r;
    asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(hi), "f"(lo));
    return r;
}

// One 64-K chunk of MMAs (4 k-steps x nmat matrices) and its two stage
// commits in ONE asm block under one elect.sync: descriptors advance by adds
// inside the block, so the issuing lane pays no per-MMA elect/branch/R2UR
// chain (at N = 64 the per-instruction issue cost, ~95 cycles with one asm
// statement per MMA, was 3x the tensor floor of 32).  a0/b0: the chunk's
// first descriptors; aj/bj: per-16-K steps; amat: the second matrix's offset.
MOE_DEVI void umma_chunk(int nmat, uint32_t d0, uint32_t d1, uint64_t a0, uint64_t amat, uint64_t aj, uint64_t b0,
                         uint64_t bj, uint32_t id, uint32_t acc0, uint64_t* bar_a, uint64_t* bar_b) {
    if (nmat == 2) {
        asm volatile(
            "{\n\t.reg .pred e, p, t;\n\t.reg .b64 a, b, m;\n\t"
            "elect.sync _|e, 0xffffffff;\n\tsetp.ne.b32 p, %8, 0;\n\tsetp.eq.u32 t, 0, 0;\n\t"
            "add.s64 m, %2, %3;\n\t"
            "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %2, %5, %7, p;\n\t"
            "@e tcgen05.mma.cta_group::1.kind::f16 [%1], m, %5, %7, p;\n\t"
            "add.s64 a, %2, %4;\n\tadd.s64 m, m, %4;\n\tadd.s64 b, %5, %6;\n\t"
            "@e tcgen05.mma.cta_group::1.kind::f16 [%0], a, b, %7, t;\n\t"
            "@e tcgen05.mma.cta_group::1.kind::f16 [%1], m, b, %7, t;\n\t"
            "add.s64 a, a, %4;\n\tadd.s64 m, m, %4;\n\tadd.s64 b, b, %6;\n\t"
            "@e tcgen05.mma.cta_group::1.kind::f16 [%0], a, b, %7, t;\n\t"
            "@e tcgen05.mma.cta_group::1.kind::f16 [%1], m, b, %7, t;\n\t"
            "add.s64 a, a, %4;\n\tadd.s64 m, m, %4;\n\tadd.s64 b, b, %6;\n\t"
            "@e tcgen05.mma.cta_group::1.kind::f16 [%0], a, b, %7, t;\n\t"
            "@e tcgen05.mma.cta_group::1.kind::f16 [%1], m, b, %7, t;\n\t"
            "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%9];\n\t"
            "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%10];\n}" ::"r"(d0),
            "r"(d1), "l"(a0), "l"(amat), "l"(aj), "l"(b0), "l"(bj), "r"(id), "r"(acc0), "r"(s32(bar_a)), "r"(s32(bar_b))
            : "memory");
    } else {
        asm volatile(
            "{\n\t.reg .pred e, p, t;\n\t.reg .b64 a, b;\n\t"
            "elect.sync _|e, 0xffffffff;\n\tsetp.ne.b32 p, %6, 0;\n\tsetp.eq.u32 t, 0, 0;\n\t"
            "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %3, %5, p;\n\t"
            "add.s64 a, %1, %2;\n\tadd.s64 b, %3, %4;\n\t"
            "@e tcgen05.mma.cta_group::1.kind::f16 [%0], a, b, %5, t;\n\t"
            "add.s64 a, a, %2;\n\tadd.s64 b, b, %4;\n\t"
            "@e tcgen05.mma.cta_group::1.kind::f16 [%0], a, b, %5, t;\n\t"
            "add.s64 a, a, %2;\n\tadd.s64 b, b, %4;\n\t"
            "@e tcgen05.mma.cta_group::1.kind::f16 [%0], a, b, %5, t;\n\t"
            "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%7];\n\t"
            "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%8];\n}" ::"r"(d0),
            "l"(a0), "l"(aj), "l"(b0), "l"(bj), "r"(id), "r"(acc0), "r"(s32(bar_a)), "r"(s32(bar_b))
            : "memory");
    }
}

// Warp-converged forms: every lane runs the issue loop with warp-uniform
// operands (kept in uniform registers, no per-MMA R2UR / elect waterfall) and
// one elected lane issues.
MOE_DEVI void umma_elect(uint32_t dtmem, uint64_t a, uint64_t b, uint32_t id, uint32_t accum) {
    asm volatile(
        "{\n\t.reg .pred p, e;\n\telect.sync _|e, 0xffffffff;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}" ::"r"(dtmem),
        "l"(a), "l"(b), "r"(id), "r"(accum)
        : "memory");
}
MOE_DEVI void umma_commit_elect(uint64_t* bar) {
    asm volatile(
        "{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
        "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n}" ::"r"(s32(bar))
        : "memory");
}
MOE_DEVI void umma_commit(uint64_t* bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(s32(bar))
                 : "memory");
}

// byte offset of (row, k) in a K-major SWIZZLE_128B tile of 64 16-bit values per row
MOE_DEVI int swz(int row, int kbyte) {
    return (row >> 3) * 1024 + (row & 7) * 128 + ((((kbyte >> 4) ^ (row & 7)) & 7) << 4) + (kbyte & 15);
}

#define TMEM_LD16(taddr, v)                                                                                       \
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];" \
                 : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),      \
                   "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]) \
                 : "r"(taddr))
#define TMEM_LD32(taddr, v)                                                                                       \
    asm volatile(                                                                                                 \
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17," \
        "%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"                                        \
        : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),       \
          "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]), \
          "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]),            \
          "=r"(v[23]), "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]),            \
          "=r"(v[30]), "=r"(v[31])                                                                              \
        : "r"(taddr))

struct Tile {
    int e, slot0, m, R0;  // expert, first slot, tokens in tile, first weight row
    int p;                // pass: 0 gate/up, 1 down (a.p, except in a fused launch)
};

// offs: the routing's expert offsets [E+1], staged in shared memory
template <int NT>
MOE_DEVI bool find_tile(const TcArgs& a, const int* offs, int RT, int b, Tile& tl) {
    constexpr int kN = NT;
    for (int e = 0; e < a.E; ++e) {
        if (!((a.active_mask >> e) & 1ull)) continue;
        const int o0 = offs[e], m = offs[e + 1] - o0;
        if (m == 0) continue;
        const int nt = (m + kN - 1) / kN;
        if (b < nt * RT) {
            // token tile fastest: the CTAs resident together share each weight
            // row tile through L2 (one HBM read serves every token tile)
            const int rt = b / nt, tt = b - rt * nt;
            tl.e = e;
            tl.slot0 = o0 + tt * kN;
            tl.m = min(kN, m - tt * kN);
            tl.R0 = rt * kM;
            tl.p = a.p;
            return true;
        }
        b -= nt * RT;
    }
    return false;
}

MOE_DEVI unsigned int ld_acquire_gpu_u32(const unsigned int* p) {
    unsigned int v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
MOE_DEVI void mbar_init_n(uint64_t* bar, uint32_t n) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(s32(bar)), "r"(n) : "memory");
}
MOE_DEVI void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(s32(bar)) : "memory");
}
MOE_DEVI void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(s32(bar)), "r"(bytes) : "memory");
}
MOE_DEVI void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(s32(dst)),
        "l"(src), "r"(bytes), "r"(s32(bar))
        : "memory");
}

// Warp roles (12 warps): 0 = bulk-copy producer of raw weight blocks, 1 =
// MMA issuer (one lane), 2 = TMA producer of the token-row (B) boxes, 4..11 =
// converters (raw -> canonical A tiles) and then the epilogue.  kRaw raw
// stages, kCan canonical A stages and kBst B stages, all handed over by
// mbarriers: the producers run ahead of the converters, the converters one
// canonical stage ahead of the tensor core.
constexpr int kThreads2 = 384;
constexpr int kConvThreads = 256;
constexpr int kRaw = 2, kCan = 2;
// bf16 tiles convert nothing: the canonical A stages serve as two more raw
// stages (a bf16 raw unit is 2 x 16 KB, the size of a canonical A stage)
constexpr int kRawB = kRaw + kCan;
constexpr int kCanA = 2 * kTileBytes;   // canonical A stage (gate + up)

// Raw stage layout: [A_gate raw 16 KB][A_up raw 16 KB][scales 2 x 256 B].
// bf16: the 64-K half (2 KB, core-matrix order) of each of the 8 row blocks
//       per matrix -- a canonical no-swizzle K-major A tile as it lands.
// int4: the whole 1 KB block per row tile (both K halves; the convert step
//       picks words 2hh, 2hh+1), 8 KB per matrix, + 8 x 32 B scales.
MOE_DEVI uint32_t raw_bytes(bool p4, int nmat) { return nmat * (p4 ? 8 * 1024 + 256 : 16384); }

MOE_DEVI void produce(const TcArgs& a, const Tile& tl, int nmat, int K, int kc, uint8_t* raw, uint64_t* bar,
                      int lane) {
    const moe_expert_weights& W = a.ex[tl.e];
    const int G = K / 128, g = kc >> 1, hh = kc & 1;
    const bool p4 = W.precision == MOE_P4;
    if (lane == 0) mbar_expect_tx(bar, raw_bytes(p4, nmat));
    __syncwarp();
    for (int mat = 0; mat < nmat; ++mat) {
        const int row0 = (tl.p == 0 && mat == 1) ? a.f + tl.R0 : tl.R0;
        const uint8_t* wb = static_cast<const uint8_t*>(tl.p == 0 ? W.w_gate_up : W.w_down);
        uint8_t* dst = raw + mat * kRawA;
        if (lane < 8) {
            const size_t blk = static_cast<size_t>(row0 / 16 + lane) * G + g;
            if (!p4) {
                bulk_g2s(dst + lane * 2048, wb + blk * 4096 + hh * 2048, 2048, bar);
            } else {
                const uint8_t* sb = static_cast<const uint8_t*>(tl.p == 0 ? W.s_gate_up : W.s_down);
                bulk_g2s(dst + lane * 1024, wb + blk * 1024, 1024, bar);
                bulk_g2s(raw + 2 * kRawA + mat * kRawS + lane * 32, sb + blk * 32, 32, bar);
            }
        }
    }
}

// bf16: chunks kc (even) and kc+1 = both halves of the same 4 KB blocks
MOE_DEVI void produce_pair(const TcArgs& a, const Tile& tl, int nmat, int K, int kc, uint8_t* raw0, uint8_t* raw1,
                           uint64_t* bar0, uint64_t* bar1, int lane) {
    const moe_expert_weights& W = a.ex[tl.e];
    const int G = K / 128, g = kc >> 1;
    if (lane == 0) {
        mbar_expect_tx(bar0, nmat * 16384);
        mbar_expect_tx(bar1, nmat * 16384);
    }
    __syncwarp();
    for (int mat = 0; mat < nmat; ++mat) {
        const int row0 = (tl.p == 0 && mat == 1) ? a.f + tl.R0 : tl.R0;
        const uint8_t* wb = static_cast<const uint8_t*>(tl.p == 0 ? W.w_gate_up : W.w_down);
        if (lane < 8) {
            const size_t blk = static_cast<size_t>(row0 / 16 + lane) * G + g;
            bulk_g2s(raw0 + mat * kRawA + lane * 2048, wb + blk * 4096, 2048, bar0);
            bulk_g2s(raw1 + mat * kRawA + lane * 2048, wb + blk * 4096 + 2048, 2048, bar1);
        }
    }
}

// One 64-K x 64-row box of the B tensor map into its SWIZZLE_128B canonical
// position (the TMA applies the same 16-byte-chunk XOR as swz(); the stage
// is 1024-byte aligned), completing on `bar`.
MOE_DEVI void tma_load_b(void* dst, const CUtensorMap* tm, int k0, int row0, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::
            "r"(s32(dst)),
        "l"(reinterpret_cast<uint64_t>(tm)), "r"(k0), "r"(row0), "r"(s32(bar))
        : "memory");
}

// per-converter-thread offsets (identical for every chunk).  A warp's 32
// threads are one item j: the 8 rows of a row half (lane = row % 8 * 4 + t),
// which is stmatrix's lane layout: word qi of the 4 lanes t of a row gives
// the row's 16-byte chunks 4qi .. 4qi+3 (nibble pairs u, gemv.cu group_int4),
// so one stmatrix.x4 per (j, qi) stores 4 whole 8 x 8 matrices (lane l
// supplies the address of row l % 8 of matrix l / 8 = chunk 4qi + l / 8).
struct ConvOffsets {
    int stm[2][2];  // int4: (item j, word qi) -> this lane's stmatrix row address
    int qrow[2];    // int4: item j -> raw word offset
    int qsc[2];     // int4: item j -> scale offset
};

MOE_DEVI void conv_offsets(int ct, int hh, ConvOffsets& o) {
    const int lane = ct & 31;
#pragma unroll
    for (int j = 0; j < 2; ++j) {
        const int it = ct + j * kConvThreads;
        const int i = it >> 6, hl = it & 63, half = hl >> 5, L = hl & 31;
        o.qrow[j] = i * 1024 + (hl * 4 + 2 * hh) * 4;
        o.qsc[j] = i * 32 + (L >> 2) * 4 + half * 2;
        const int srow = i * 16 + half * 8 + (lane & 7);  // row this lane addresses for stmatrix
#pragma unroll
        for (int qi = 0; qi < 2; ++qi) o.stm[j][qi] = swz(srow, (4 * qi + (lane >> 3)) * 16);
    }
}

MOE_DEVI void stmatrix_x4(uint32_t addr, uint32_t r0, uint32_t r1, uint32_t r2, uint32_t r3) {
    asm volatile("stmatrix.sync.aligned.m8n8.x4.shared.b16 [%0], {%1, %2, %3, %4};" ::"r"(addr), "r"(r0), "r"(r1), "r"(r2),
                 "r"(r3)
                 : "memory");
}

// int4 raw blocks -> fp16 q*s in the canonical SW128 A tile (bf16 blocks are
// already in core-matrix order and feed the MMA directly)
MOE_DEVI void convert_int4(int nmat, const uint8_t* raw, uint8_t* can, int ct, const ConvOffsets& o) {
    for (int mat = 0; mat < nmat; ++mat) {
        const uint8_t* src = raw + mat * kRawA;
        uint8_t* dst = can + mat * kTileBytes;
        const uint8_t* sc = raw + 2 * kRawA + mat * kRawS;
        const __half2 m1032 = __halves2half2(__ushort_as_half(0xE408), __ushort_as_half(0xE408));
        const __half2 m72 = __halves2half2(__ushort_as_half(0xD480), __ushort_as_half(0xD480));
        const __half2 r16 = __halves2half2(__ushort_as_half(0x2C00), __ushort_as_half(0x2C00));
#pragma unroll
        for (int j = 0; j < 2; ++j) {
            const uint2 w2 = *reinterpret_cast<const uint2*>(src + o.qrow[j]);
            const uint16_t sb = *reinterpret_cast<const uint16_t*>(sc + o.qsc[j]);
            if (f16_scale_bad(sb)) numerics_flag(MOE_NUM_F16_SCALE);
            const __half sh = __float2half_rn(bf2f(sb));  // exact for normal-range scales
            const __half2 s2 = __halves2half2(sh, sh);
#pragma unroll
            for (int qi = 0; qi < 2; ++qi) {
                const uint32_t w = qi ? w2.y : w2.x;
                uint32_t v[4] = {and_or(w, 0x000F000Fu, 0x64006400u), and_or(w, 0x00F000F0u, 0x64006400u),
                                 and_or(w >> 8, 0x000F000Fu, 0x64006400u), and_or(w >> 8, 0x00F000F0u, 0x64006400u)};
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    __half2 h = *reinterpret_cast<__half2*>(&v[u]);
                    h = (u & 1) ? __hfma2(h, r16, m72) : __hadd2(h, m1032);  // q exactly
                    h = __hmul2(h, s2);                                      // q*s exactly
                    v[u] = *reinterpret_cast<uint32_t*>(&h);
                }
                stmatrix_x4(s32(dst) + o.stm[j][qi], v[0], v[1], v[2], v[3]);
            }
        }
    }
}

template <int NT>
struct TcCfg {
    static constexpr int kN = NT;
    static constexpr int kBTile = NT * kKc * 2;        // B stage bytes
    static constexpr int kBst = NT == 256 ? 2 : 4;     // B stages
    static constexpr int kTmemCols = 2 * NT;           // gate + up accumulators
    static constexpr int kSmem = 1024 + kRaw * kRawBytes + kCan * kCanA + kBst * kBTile;
};

template <int NT>
__global__ void __launch_bounds__(kThreads2, 1) tc_ffn_kernel(const __grid_constant__ TcArgs a) {
    using Cf = TcCfg<NT>;
    constexpr int kN = Cf::kN, kBst = Cf::kBst;
    extern __shared__ uint8_t smem_raw[];
    // 1024-byte aligned base by pointer arithmetic (keeps the shared address
    // space, so the converters use LDS/STS, not generic loads/stores)
    uint8_t* smem = smem_raw + ((1024u - (s32(smem_raw) & 1023u)) & 1023u);
    __shared__ __align__(8) uint64_t raw_full[kRawB], raw_empty[kRawB], can_full[kCan], can_empty[kCan], b_full[kBst],
        b_empty[kBst], acc_full;
    __shared__ uint32_t tmem_slot;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    auto can = [&](int s) { return smem + s * kCanA; };
    auto bst = [&](int s) { return smem + kCan * kCanA + s * Cf::kBTile; };
    auto raw = [&](int s) {
        return s < kRaw ? smem + kCan * kCanA + kBst * Cf::kBTile + s * kRawBytes : smem + (s - kRaw) * kCanA;
    };

    pdl_wait();
    pdl_trigger();
    const int K = a.p == 0 ? a.d : a.f;
    const int RT = (a.p == 0 ? a.f : a.d) / kM;
    // the E+1 offsets in one parallel load instead of a dependent chain
    __shared__ int s_off[MOE_MAX_EXPERTS + 1];
    if (tid <= a.E) s_off[tid] = a.offsets[tid];
    __syncthreads();
    Tile tl;
    if (!find_tile<NT>(a, s_off, RT, blockIdx.x, tl)) return;
    const int nmat = a.p == 0 ? 2 : 1;
    const bool p4 = a.ex[tl.e].precision == MOE_P4;
    // UMMA N: the tile's tokens rounded up to 16 (M = 128 allows 16..256)
    const int nmma = min(kN, (tl.m + 15) / 16 * 16);
    if (tid == 0) {
        for (int s = 0; s < kRawB; ++s) {
            mbar_init_n(&raw_full[s], 1);  // producer expect_tx
            // int4: freed by the converter warps; bf16: by the MMA commit (the
            // raw core-matrix blocks are the A operand, no conversion)
            mbar_init_n(&raw_empty[s], p4 ? kConvThreads / 32 : 1);
        }
        for (int s = 0; s < kCan; ++s) {
            mbar_init_n(&can_full[s], kConvThreads / 32);  // converter warps
            mbar_init_n(&can_empty[s], 1);
        }
        for (int s = 0; s < kBst; ++s) {
            mbar_init_n(&b_full[s], 1);  // TMA expect_tx
            mbar_init_n(&b_empty[s], 1);
        }
        mbar_init_n(&acc_full, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 1) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(s32(&tmem_slot)),
                     "r"(Cf::kTmemCols)
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tmem = tmem_slot;
    const int nk = K / kKc;
    const int nraw = p4 ? kRaw : kRawB;  // raw stages in use

    if (warp == 0) {
        // ---- weight producer: kRaw chunks ahead of the converters ----
        // raw units: one 64-K chunk for bf16; a 128-K chunk pair for int4,
        // whose 1 KB blocks hold both K halves (loaded once, converted twice)
        for (int kc = 0; kc < nk; kc += p4 ? 2 : 1) {
            const int u = p4 ? kc >> 1 : kc;
            const int r = u % nraw, pass = u / nraw;
            if (pass > 0) mbar_wait(&raw_empty[r], (pass - 1) & 1);
            if (a.dbg & 4) {
                if (lane == 0) mbar_arrive(&raw_full[r]);
                __syncwarp();
            } else if (!p4 && !(a.dbg & 32) && (kc & 1) == 0 && kc + 1 < nk) {
                // both 64-K halves of each 4 KB bf16 block back to back: one
                // DRAM-contiguous 4 KB read per block instead of two 2 KB
                // reads a chunk apart
                const int r1 = (u + 1) % nraw, pass1 = (u + 1) / nraw;
                if (pass1 > 0) mbar_wait(&raw_empty[r1], (pass1 - 1) & 1);
                produce_pair(a, tl, nmat, K, kc, raw(r), raw(r1), &raw_full[r], &raw_full[r1], lane);
                ++kc;
            } else {
                produce(a, tl, nmat, K, kc, raw(r), &raw_full[r], lane);
            }
        }
    } else if (warp == 2) {
        // ---- B producer: TMA boxes of the slot-ordered rows, kBst chunks ahead ----
        if (lane == 0) {
            const CUtensorMap* tm = p4 ? &a.tmb16 : &a.tmb;
            const int nbox = (nmma + 63) / 64;
            for (int kb = 0; kb < nk; ++kb) {
                const int b = kb % kBst;
                if (kb >= kBst) mbar_wait(&b_empty[b], ((kb / kBst) - 1) & 1);
                if (a.dbg & 4096) {
                    mbar_arrive(&b_full[b]);
                    continue;
                }
                mbar_expect_tx(&b_full[b], static_cast<uint32_t>(nbox) * 64 * 128);
                for (int q = 0; q < nbox; ++q) tma_load_b(bst(b) + q * 8192, tm, kb * kKc, tl.slot0 + q * 64, &b_full[b]);
            }
        }
        __syncwarp();
    } else if (warp == 1) {
        // ---- MMA issuer ----
        const uint32_t id = idesc(p4 ? 0 : 1, nmma, kM);
        for (int kc = 0; kc < nk; ++kc) {
            const int c = kc % kCan, b = kc % kBst, r = kc % nraw;
            if (p4)
                mbar_wait(&can_full[c], (kc / kCan) & 1);
            else
                mbar_wait(&raw_full[r], (kc / nraw) & 1);
            mbar_wait(&b_full[b], (kc / kBst) & 1);
            asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
            {  // warp-converged issue (umma_elect)
                const uint32_t cb = s32(can(c)), rb = s32(raw(r)), bb = s32(bst(b));
#pragma unroll
                for (int j = 0; j < kKc / 16; ++j) {
                    if (a.dbg & 2) break;
                    const uint64_t bdesc = sdesc(bb + j * 32);
                    const uint32_t acc = (kc > 0 || j > 0) ? 1u : 0u;
                    // A: canonical SW128 tile (int4, converted) or the raw core-matrix blocks (bf16)
                    for (int mat = 0; mat < nmat; ++mat) {
                        const uint64_t adesc = p4 ? sdesc(cb + mat * kTileBytes + j * 32)
                                                  : sdesc_core(rb + mat * kRawA + j * 256);
                        umma_elect(tmem + mat * kN, adesc, bdesc, id, acc);
                    }
                }
                umma_commit_elect(p4 ? &can_empty[c] : &raw_empty[r]);
                umma_commit_elect(&b_empty[b]);
                if (kc == nk - 1) umma_commit_elect(&acc_full);
            }
        }
    } else if (warp >= 4) {
        // ---- converters, then the epilogue ----
        const int ct = tid - 128;
        ConvOffsets o0, o1;  // K halves hh = 0 / 1 (int4 word selection differs)
        conv_offsets(ct, 0, o0);
        conv_offsets(ct, 1, o1);
        for (int kc = 0; kc < (p4 ? nk : 0); ++kc) {  // bf16: nothing to convert
            const int u = kc >> 1;
            const int r = u % kRaw, c = kc % kCan;
            mbar_wait(&raw_full[r], (u / kRaw) & 1);
            if (kc >= kCan) mbar_wait(&can_empty[c], ((kc / kCan) - 1) & 1);
            if (!(a.dbg & 1)) convert_int4(nmat, raw(r), can(c), ct, (kc & 1) ? o1 : o0);
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            __syncwarp();
            if (lane == 0) {
                mbar_arrive(&can_full[c]);
                if (kc & 1) mbar_arrive(&raw_empty[r]);
            }
        }
        mbar_wait(&acc_full, 0);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const int row = (warp & 3) * 32 + lane;
        const uint32_t lane_base = static_cast<uint32_t>((warp & 3) * 32) << 16;
        const int c0 = ((warp - 4) >> 2) * (kN / 2);
        for (int cb = c0; cb < c0 + kN / 2 && !(a.dbg & 2048); cb += 32) {
            uint32_t g[32];
            TMEM_LD32(tmem + lane_base + cb, g);
            if (a.p == 0) {
                uint32_t u[32];
                TMEM_LD32(tmem + lane_base + kN + cb, u);
                asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
                for (int c = 0; c < 32; ++c) {
                    const int n = cb + c;
                    if (n < tl.m) {
                        const uint16_t hb = f2bf(silu_fast(__uint_as_float(g[c])) * __uint_as_float(u[c]));
                        const size_t o = static_cast<size_t>(tl.slot0 + n) * a.f + tl.R0 + row;
                        a.hout[o] = hb;
                        if (p4) {  // the fp16 copy feeds only an int4 down pass
                            if (f16_overflow(bf2f(hb))) numerics_flag(MOE_NUM_F16_ACT);
                            a.hout16[o] = __half_as_ushort(__float2half_rn(bf2f(hb)));
                        }
                    }
                }
            } else {
                asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
                for (int c = 0; c < 32; ++c) {
                    const int n = cb + c;
                    if (n < tl.m) a.y[static_cast<size_t>(tl.slot0 + n) * a.d + tl.R0 + row] = __uint_as_float(g[c]);
                }
            }
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (warp == 1)
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(Cf::kTmemCols) : "memory");
}

// ===========================================================================
// Persistent 128-token variant (tc_ffn_persist): one CTA per SM walks the
// tile list (t = blockIdx, blockIdx + grid, ...), every role running straight
// from one tile into the next -- no per-tile prologue, no pipeline drain, the
// epilogue of tile i overlapping the mainloop of tile i+1 through two TMEM
// accumulator buffers (512 columns).  Shared memory: region R (4 x 32 KB) is
// the bf16 raw ring, or for int4 tiles two canonical A stages + three compact
// raw units; region B holds four 16 KB B stages.  At a change of precision
// between consecutive tiles the weight producer waits for the previous
// tile's accumulators (so R is no longer read) before reusing R.
constexpr int kPRaw4Unit = 2 * 8192 + 2 * kRawS;  // compact int4 raw unit: [A_gate 8 KB][A_up 8 KB][scales]
#ifndef MOE_TCP_CAN
#define MOE_TCP_CAN 2
#endif
// MOE_TCP_WIDE: int4 canonical stages of a whole 128-K raw unit (both 64-K halves,
// 64 KB): one convert -> MMA hand-off per unit instead of per chunk
#ifndef MOE_TCP_WIDE
#define MOE_TCP_WIDE 0
#endif
constexpr bool kPWide = MOE_TCP_WIDE != 0;
constexpr int kPCan = kPWide ? 2 : MOE_TCP_CAN;     // int4 canonical A stages in R
constexpr int kPCanBytes = kPWide ? 65536 : 32768;
// MOE_TCP_RB: bf16 raw stages in R (32 KB each); MOE_TCP_B: B stages (16 KB; 0 = by kPCan)
// 5 + 4 measured best for batched decode (4+4: -1..4 %, 6+2: -7 %, 6+1: -30 %)
#ifndef MOE_TCP_RB
#define MOE_TCP_RB 5
#endif
#ifndef MOE_TCP_B
#define MOE_TCP_B 4
#endif
constexpr int kPRb = MOE_TCP_RB;
constexpr int kPBst = MOE_TCP_B ? MOE_TCP_B : (kPWide || kPCan == 3 ? 3 : 4);  // B stages
constexpr int kPR0 = kPWide ? 165888 : kPCan == 3 ? 5 * 32768 - 16384 : 4 * 32768;
constexpr int kPR = kPR0 > kPRb * 32768 ? kPR0 : kPRb * 32768;  // region R
constexpr int kPRaw4 = (kPR - kPCan * kPCanBytes) / kPRaw4Unit;  // int4 raw units in R after the canonical stages
constexpr int kPSmem = 1024 + kPR + kPBst * 128 * kKc * 2;  // R + B
static_assert(kPSmem + 1024 <= 232448 && kPRaw4 >= 2, "tc_ffn_persist stages exceed shared memory");

MOE_DEVI void produce4c(const TcArgs& a, const Tile& tl, int nmat, int K, int kc, uint8_t* raw, uint64_t* bar, int lane) {
    const moe_expert_weights& W = a.ex[tl.e];
    const int G = K / 128, g = kc >> 1;
    if (lane == 0) mbar_expect_tx(bar, nmat * (8 * 1024 + 256));
    __syncwarp();
    for (int mat = 0; mat < nmat; ++mat) {
        const int row0 = (tl.p == 0 && mat == 1) ? a.f + tl.R0 : tl.R0;
        const uint8_t* wb = static_cast<const uint8_t*>(tl.p == 0 ? W.w_gate_up : W.w_down);
        const uint8_t* sb = static_cast<const uint8_t*>(tl.p == 0 ? W.s_gate_up : W.s_down);
        if (lane < 8) {
            const size_t blk = static_cast<size_t>(row0 / 16 + lane) * G + g;
            bulk_g2s(raw + mat * 8192 + lane * 1024, wb + blk * 1024, 1024, bar);
            bulk_g2s(raw + 2 * 8192 + mat * kRawS + lane * 32, sb + blk * 32, 32, bar);
        }
    }
}

// convert_int4 over the compact raw unit layout.  Every raw word and scale of
// the chunk is loaded first, then converted and stored: the stores carry no
// memory clobber, so the loads are not serialised behind them (the
// canonical stage is read only by the tensor core, after the converters'
// proxy fence and barrier arrive, which are ordered asm statements).
MOE_DEVI void stmatrix_x4_nc(uint32_t addr, uint32_t r0, uint32_t r1, uint32_t r2, uint32_t r3) {
    asm volatile("stmatrix.sync.aligned.m8n8.x4.shared.b16 [%0], {%1, %2, %3, %4};" ::"r"(addr), "r"(r0), "r"(r1), "r"(r2),
                 "r"(r3));
}
MOE_DEVI void convert_int4c(int nmat, const uint8_t* raw, uint8_t* can, int ct, const ConvOffsets& o) {
    uint2 w2[2][2];
    uint16_t sb[2][2];
#pragma unroll
    for (int mat = 0; mat < 2; ++mat) {
        if (mat < nmat) {
#pragma unroll
            for (int j = 0; j < 2; ++j) {
                w2[mat][j] = *reinterpret_cast<const uint2*>(raw + mat * 8192 + o.qrow[j]);
                sb[mat][j] = *reinterpret_cast<const uint16_t*>(raw + 2 * 8192 + mat * kRawS + o.qsc[j]);
            }
        }
    }
    const __half2 m1032 = __halves2half2(__ushort_as_half(0xE408), __ushort_as_half(0xE408));
    const __half2 m72 = __halves2half2(__ushort_as_half(0xD480), __ushort_as_half(0xD480));
    const __half2 r16 = __halves2half2(__ushort_as_half(0x2C00), __ushort_as_half(0x2C00));
#pragma unroll
    for (int mat = 0; mat < 2; ++mat) {
        if (mat < nmat) {
            const uint32_t dst = s32(can + mat * kTileBytes);
#pragma unroll
            for (int j = 0; j < 2; ++j) {
                if (f16_scale_bad(sb[mat][j])) numerics_flag(MOE_NUM_F16_SCALE);
                const __half sh = __float2half_rn(bf2f(sb[mat][j]));
                const __half2 s2 = __halves2half2(sh, sh);
#pragma unroll
                for (int qi = 0; qi < 2; ++qi) {
                    const uint32_t w = qi ? w2[mat][j].y : w2[mat][j].x;
                    uint32_t v[4] = {and_or(w, 0x000F000Fu, 0x64006400u), and_or(w, 0x00F000F0u, 0x64006400u),
                                     and_or(w >> 8, 0x000F000Fu, 0x64006400u), and_or(w >> 8, 0x00F000F0u, 0x64006400u)};
#pragma unroll
                    for (int u = 0; u < 4; ++u) {
                        __half2 h = *reinterpret_cast<__half2*>(&v[u]);
                        h = (u & 1) ? __hfma2(h, r16, m72) : __hadd2(h, m1032);
                        h = __hmul2(h, s2);
                        v[u] = *reinterpret_cast<uint32_t*>(&h);
                    }
                    stmatrix_x4_nc(dst + o.stm[j][qi], v[0], v[1], v[2], v[3]);
                }
            }
        }
    }
}

// MOE_TC_DBG bit 15 (builds with -DMOE_TC_TRACE=1): CTA 0 stamps (SM clock) of its third tile's chunks -- chunks (tc_ffn_wide:
// weight issue, B issue, weight full seen by the MMA thread, B full seen, MMA
// committed; tc_ffn_persist int4 tiles: unit issue, converter start, converter
// done, MMA sees the canonical stage, MMA committed) -- printed at exit (latency probe)
#ifndef MOE_TC_TRACE
#define MOE_TC_TRACE 0  // the probe costs the int4 converter loop ~10 %: compiled in only on request
#endif
constexpr bool kTcTrace = MOE_TC_TRACE != 0;
__device__ unsigned int g_wtrace[6][64];
__device__ unsigned int g_wtrace2[2][4][64];  // tc_ffn_wide2: [rank][weight issue, forwarder, pair full, MMA][chunk]
MOE_DEVI unsigned int clk32() {
    unsigned int c;
    asm volatile("mov.u32 %0, %%clock;" : "=r"(c));
    return c;
}

// nsplit > 1 (down pass): tile (e, row tile, K split ks) covers chunks ks*nk/nsplit ..; its
// y rows go to ypart[ks] (summed in split order by split_reduce_kernel)
__global__ void __launch_bounds__(kThreads2, 1) tc_ffn_persist(const __grid_constant__ TcArgs a, int ntiles, int nsplit,
                                                               float* ypart, int fused) {
    constexpr int kN = 128, kBst = kPBst, kBTile = kN * kKc * 2;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = smem_raw + ((1024u - (s32(smem_raw) & 1023u)) & 1023u);
    __shared__ __align__(8) uint64_t rb_full[kPRb], rb_empty[kPRb], r4_full[kPRaw4], r4_empty[kPRaw4], cn_full[kPCan], cn_empty[kPCan],
        b_full[kBst], b_empty[kBst], acc_full[2], acc_empty[2];
    __shared__ uint32_t tmem_slot;
    __shared__ int s_off[MOE_MAX_EXPERTS + 1];
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    uint8_t* R = smem;
    uint8_t* Bst = smem + kPR;
    auto rawb = [&](int s) { return R + s * 32768; };
    auto can = [&](int s) { return R + s * kPCanBytes; };
    auto raw4 = [&](int s) { return R + kPCan * kPCanBytes + s * kPRaw4Unit; };
    auto bst = [&](int s) { return Bst + s * kBTile; };

    pdl_wait();
    pdl_trigger();
    // per-tile pass parameters (a fused launch walks the gate/up tiles, then the down tiles)
    auto K_of = [&](const Tile& t) { return t.p == 0 ? a.d : a.f; };
    auto nmat_of = [&](const Tile& t) { return t.p == 0 ? 2 : 1; };
    auto ns_of = [&](const Tile& t) { return t.p == 0 ? 1 : nsplit; };
    auto nks_of = [&](const Tile& t) { return K_of(t) / kKc / ns_of(t); };  // chunks per tile
    const int RT0 = a.f / kM;
    const int grid = static_cast<int>(gridDim.x);
    if (tid <= a.E) s_off[tid] = a.offsets[tid];
    if (tid == 0) {
        for (int s = 0; s < kPRb; ++s) {
            mbar_init_n(&rb_full[s], 1);
            mbar_init_n(&rb_empty[s], 1);  // MMA commit
        }
        for (int s = 0; s < kPRaw4; ++s) {
            mbar_init_n(&r4_full[s], 1);
            mbar_init_n(&r4_empty[s], kConvThreads / 32);
        }
        for (int s = 0; s < kPCan; ++s) {
            mbar_init_n(&cn_full[s], kConvThreads / 32);
            mbar_init_n(&cn_empty[s], 1);
        }
        for (int s = 0; s < 2; ++s) {
            mbar_init_n(&acc_full[s], 1);
            mbar_init_n(&acc_empty[s], kConvThreads / 32);
        }
        for (int s = 0; s < kBst; ++s) {
            mbar_init_n(&b_full[s], 1);
            mbar_init_n(&b_empty[s], 1);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 1) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(s32(&tmem_slot)), "r"(512)
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tmem = tmem_slot;
    // fused: the gate/up tiles come first, n0 of them
    int n0 = 0;
    if (fused)
        for (int e = 0; e < a.E; ++e)
            if ((a.active_mask >> e) & 1ull) n0 += (s_off[e + 1] - s_off[e] + kN - 1) / kN * RT0;
    // (row tile, K split) enumerated as one index: find_tile's R0 / 128 = rt * nsplit + ks
    auto tile_of = [&](int i, Tile& tl, int& kc0) {
        int t = static_cast<int>(blockIdx.x) + i * grid, p = a.p;
        if (fused) {
            p = t < n0 ? 0 : 1;
            if (p == 1) t -= n0;
        }
        const int nsp = p == 0 ? 1 : nsplit;
        if (!find_tile<128>(a, s_off, (p == 0 ? a.f : a.d) / kM * nsp, t, tl)) return false;
        tl.p = p;
        const int rtk = tl.R0 / kM, ks = rtk % nsp;
        tl.R0 = (rtk / nsp) * kM;
        kc0 = ks * nks_of(tl);
        return true;
    };
    // fused: counter of (expert, token tile, K split): the gate/up tiles whose h columns
    // fall in that split of the down pass's K; a down tile waits for RT0 / nsplit of them
    auto dep_of = [&](const Tile& t, int ks) {
        return a.dep + ((t.e * a.dep_tt + (t.slot0 - s_off[t.e]) / kN) * nsplit + ks);
    };
    auto is_p4 = [&](const Tile& tl) { return a.ex[tl.e].precision == MOE_P4; };
    const int my_tiles = static_cast<int>(blockIdx.x) < ntiles ? (ntiles - static_cast<int>(blockIdx.x) + grid - 1) / grid : 0;
    const bool trace = kTcTrace && (a.dbg & 32768) && blockIdx.x == 0;
    auto stamp = [&](int w, int i, int c) {
        if (trace && i == 2 && c < 64) g_wtrace[w][c] = clk32();
    };

    if (warp == 0) {
        // ---- weight producer ----
        int ub = 0, u4 = 0, prev = -1;
        for (int i = 0; i < my_tiles; ++i) {
            Tile tl;
            int kc0;
            if (!tile_of(i, tl, kc0)) break;  // past the routing's last tile
            const bool p4 = is_p4(tl);
            const int K = K_of(tl), nmat = nmat_of(tl), nks = nks_of(tl);
            if (prev >= 0 && prev != static_cast<int>(p4))  // region R changes role: the previous tile's MMAs first
                mbar_wait(&acc_full[(i - 1) & 1], static_cast<uint32_t>(((i - 1) >> 1) & 1));
            prev = p4;
            if (p4) {
                for (int kc = kc0; kc < kc0 + nks; kc += 2, ++u4) {
                    const int r = u4 % kPRaw4;
                    if (u4 >= kPRaw4) mbar_wait(&r4_empty[r], static_cast<uint32_t>(((u4 / kPRaw4) - 1) & 1));
                    if (lane == 0) stamp(0, i, kc - kc0);
                    produce4c(a, tl, nmat, K, kc, raw4(r), &r4_full[r], lane);
                }
            } else {
                for (int kc = kc0; kc < kc0 + nks; kc += 2, ub += 2) {  // both 64-K halves of each 4 KB block
                    const int r0 = ub % kPRb, r1 = (ub + 1) % kPRb;
                    if (ub >= kPRb) mbar_wait(&rb_empty[r0], static_cast<uint32_t>(((ub / kPRb) - 1) & 1));
                    if (ub + 1 >= kPRb) mbar_wait(&rb_empty[r1], static_cast<uint32_t>((((ub + 1) / kPRb) - 1) & 1));
                    produce_pair(a, tl, nmat, K, kc, rawb(r0), rawb(r1), &rb_full[r0], &rb_full[r1], lane);
                }
            }
        }
    } else if (warp == 2) {
        // ---- B producer ----
        if (lane == 0) {
            int kb = 0;
            for (int i = 0; i < my_tiles; ++i) {
                Tile tl;
                int kc0;
                if (!tile_of(i, tl, kc0)) break;
                const bool down_f = fused && tl.p == 1;
                const CUtensorMap* tm = down_f ? (is_p4(tl) ? &a.tmh16 : &a.tmh) : (is_p4(tl) ? &a.tmb16 : &a.tmb);
                const int nbox = (min(kN, (tl.m + 15) / 16 * 16) + 63) / 64;
                const int nks = nks_of(tl);
                if (down_f) {
                    // this token tile's h columns of this K split, written by other CTAs' gate/up tiles
                    const unsigned int* dp = dep_of(tl, kc0 / nks);
                    while (ld_acquire_gpu_u32(dp) < static_cast<unsigned int>(RT0 / nsplit)) __nanosleep(64);
                    asm volatile("fence.proxy.async.global;" ::: "memory");  // their generic stores before our TMA reads
                }
                for (int kc = kc0; kc < kc0 + nks; ++kc, ++kb) {
                    const int b = kb % kBst;
                    if (kb >= kBst) mbar_wait(&b_empty[b], static_cast<uint32_t>(((kb / kBst) - 1) & 1));
                    mbar_expect_tx(&b_full[b], static_cast<uint32_t>(nbox) * 64 * 128);
                    for (int q = 0; q < nbox; ++q) tma_load_b(bst(b) + q * 8192, tm, kc * kKc, tl.slot0 + q * 64, &b_full[b]);
                }
            }
        }
        __syncwarp();
    } else if (warp == 1) {
        // ---- MMA issuer ----
        int cb = 0, c4 = 0, kb = 0;
        for (int i = 0; i < my_tiles; ++i) {
            Tile tl;
            int kc0;
            if (!tile_of(i, tl, kc0)) break;  // past the routing's last tile
            const bool p4 = is_p4(tl);
            const int nmat = nmat_of(tl), nks = nks_of(tl);
            const int nmma = min(kN, (tl.m + 15) / 16 * 16);
            const uint32_t id = idesc(p4 ? 0 : 1, nmma, kM);
            const int buf = i & 1;
            if (i >= 2) mbar_wait(&acc_empty[buf], static_cast<uint32_t>(((i >> 1) - 1) & 1));
            asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
            const uint32_t dacc = tmem + buf * 256;
            for (int kc = kc0; kc < kc0 + nks; ++kc, ++kb) {
                const int b = kb % kBst;
                int slot;
                if (p4) {
                    const int cu = kPWide ? c4 >> 1 : c4;  // canonical stage use
                    slot = cu % kPCan;
                    if (!kPWide || (c4 & 1) == 0) mbar_wait(&cn_full[slot], static_cast<uint32_t>((cu / kPCan) & 1));
                    if (lane == 0) stamp(3, i, kc - kc0);
                } else {
                    slot = cb % kPRb;
                    mbar_wait(&rb_full[slot], static_cast<uint32_t>((cb / kPRb) & 1));
                }
                mbar_wait(&b_full[b], static_cast<uint32_t>((kb / kBst) & 1));
                if (lane == 0) stamp(5, i, kc - kc0);
                asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
                {
                    const uint32_t ab = s32(p4 ? can(slot) + (kPWide ? (c4 & 1) * 32768 : 0) : rawb(slot)), bb = s32(bst(b));
                    const bool rel = !p4 || !kPWide || (c4 & 1) == 1;  // the A stage is released with this chunk
                    if (!rel) {  // kPWide builds, first half of a canonical unit: only B is released
#pragma unroll
                        for (int j = 0; j < kKc / 16; ++j) {
                            const uint64_t bdesc = sdesc(bb + j * 32);
                            const uint32_t acc = (kc > kc0 || j > 0) ? 1u : 0u;
                            for (int mat = 0; mat < nmat; ++mat)
                                umma_elect(dacc + mat * kN, sdesc(ab + mat * kTileBytes + j * 32), bdesc, id, acc);
                        }
                        umma_commit_elect(&b_empty[b]);
                    } else {
                        umma_chunk(nmat, dacc, dacc + kN, p4 ? sdesc(ab) : sdesc_core(ab),
                                   p4 ? (kTileBytes >> 4) : (kRawA >> 4), p4 ? 2 : 16, sdesc(bb), 2, id,
                                   kc > kc0 ? 1u : 0u, p4 ? &cn_empty[slot] : &rb_empty[slot], &b_empty[b]);
                    }
                    if (kc == kc0 + nks - 1) umma_commit_elect(&acc_full[buf]);
                    if (lane == 0) stamp(4, i, kc - kc0);
                }
                if (p4) ++c4; else ++cb;
            }
        }
    } else if (warp >= 4) {
        // ---- converters (int4 tiles), then each tile's epilogue ----
        const int ct = tid - 128;
        ConvOffsets o0, o1;
        conv_offsets(ct, 0, o0);
        conv_offsets(ct, 1, o1);
        int u4 = 0, c4 = 0;
        const int row = (warp & 3) * 32 + lane;
        const uint32_t lane_base = static_cast<uint32_t>((warp & 3) * 32) << 16;
        const int c0 = ((warp - 4) >> 2) * (kN / 2);
        for (int i = 0; i < my_tiles; ++i) {
            Tile tl;
            int kc0;
            if (!tile_of(i, tl, kc0)) break;  // past the routing's last tile
            const int nmat = nmat_of(tl), nks = nks_of(tl);
            if (is_p4(tl) && kPWide) {
                for (int kc = kc0; kc < kc0 + nks; kc += 2, ++u4) {  // one hand-off per raw unit
                    const int r = u4 % kPRaw4, c = u4 % kPCan;
                    mbar_wait(&r4_full[r], static_cast<uint32_t>((u4 / kPRaw4) & 1));
                    if (u4 >= kPCan) mbar_wait(&cn_empty[c], static_cast<uint32_t>(((u4 / kPCan) - 1) & 1));
                    convert_int4c(nmat, raw4(r), can(c), ct, o0);
                    convert_int4c(nmat, raw4(r), can(c) + 32768, ct, o1);
                    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                    __syncwarp();
                    if (lane == 0) {
                        mbar_arrive(&cn_full[c]);
                        mbar_arrive(&r4_empty[r]);
                    }
                }
            } else if (is_p4(tl)) {
                for (int kc = kc0; kc < kc0 + nks; ++kc, ++c4) {
                    const int r = u4 % kPRaw4, c = c4 % kPCan;
                    if ((kc & 1) == 0) mbar_wait(&r4_full[r], static_cast<uint32_t>((u4 / kPRaw4) & 1));
                    if (c4 >= kPCan) mbar_wait(&cn_empty[c], static_cast<uint32_t>(((c4 / kPCan) - 1) & 1));
                    if (ct == 0) stamp(1, i, kc - kc0);
                    convert_int4c(nmat, raw4(r), can(c), ct, (kc & 1) ? o1 : o0);
                    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                    __syncwarp();
                    if (ct == 0) stamp(2, i, kc - kc0);
                    if (lane == 0) {
                        mbar_arrive(&cn_full[c]);
                        if (kc & 1) mbar_arrive(&r4_empty[r]);
                    }
                    if (kc & 1) ++u4;
                }
            }
            const int buf = i & 1;
            mbar_wait(&acc_full[buf], static_cast<uint32_t>((i >> 1) & 1));
            asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
            const uint32_t dacc = tmem + buf * 256;
            for (int cbk = c0; cbk < c0 + kN / 2; cbk += 32) {
                uint32_t g[32];
                TMEM_LD32(dacc + lane_base + cbk, g);
                if (tl.p == 0) {
                    uint32_t u[32];
                    TMEM_LD32(dacc + lane_base + kN + cbk, u);
                    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
                    for (int c = 0; c < 32; ++c) {
                        const int n = cbk + c;
                        if (n < tl.m) {
                            const uint16_t hb = f2bf(silu_fast(__uint_as_float(g[c])) * __uint_as_float(u[c]));
                            const size_t o = static_cast<size_t>(tl.slot0 + n) * a.f + tl.R0 + row;
                            a.hout[o] = hb;
                            if (is_p4(tl)) {  // the fp16 copy feeds only an int4 down pass
                                if (f16_overflow(bf2f(hb))) numerics_flag(MOE_NUM_F16_ACT);
                                a.hout16[o] = __half_as_ushort(__float2half_rn(bf2f(hb)));
                            }
                        }
                    }
                } else {
                    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
                    for (int c = 0; c < 32; ++c) {
                        const int n = cbk + c;
                        if (n < tl.m) {
                            float* yo = ns_of(tl) > 1 ? ypart + static_cast<size_t>(kc0 / nks) * a.T * a.k * a.d : a.y;
                            yo[static_cast<size_t>(tl.slot0 + n) * a.d + tl.R0 + row] = __uint_as_float(g[c]);
                        }
                    }
                }
            }
            asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
            __syncwarp();
            if (lane == 0) mbar_arrive(&acc_empty[buf]);
            if (fused && tl.p == 0) {
                // publish this tile's h columns to the down tiles that read them
                __threadfence();
                asm volatile("bar.sync 1, %0;" ::"r"(kConvThreads) : "memory");
                if (ct == 0) atomicAdd(dep_of(tl, (tl.R0 / kM) / (RT0 / nsplit)), 1u);
            }
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (warp == 1) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512) : "memory");
    if (trace && tid == 0 && my_tiles > 2) {
        const unsigned int t0 = g_wtrace[0][0];
        for (int c = 0; c < 64; ++c)
            printf("PTRACE p%d c %2d uiss %7d cstart %7d cdone %7d cfull %7d bfull %7d mma %7d\n", a.p, c,
                   g_wtrace[0][c] - t0, g_wtrace[1][c] - t0, g_wtrace[2][c] - t0, g_wtrace[3][c] - t0,
                   g_wtrace[5][c] - t0, g_wtrace[4][c] - t0);
    }
}

// y[slot][j] = sum over K splits of ypart[ks][slot][j], in split order, for the
// slots of this launch's experts only (other rows of y are left untouched, as
// the unsplit kernel leaves them).  One block per slot row (grid-stride).
__global__ void split_reduce_kernel(const float4* __restrict__ ypart, const int32_t* __restrict__ offsets, int E,
                                    uint64_t active_mask, int slots, int d4, int nsplit, float4* __restrict__ y) {
    __shared__ int s_off[MOE_MAX_EXPERTS + 1];
    pdl_wait();
    pdl_trigger();
    if (threadIdx.x <= E) s_off[threadIdx.x] = offsets[threadIdx.x];
    __syncthreads();
    const size_t plane = static_cast<size_t>(slots) * d4;
    for (int slot = blockIdx.x; slot < slots; slot += gridDim.x) {
        int e = 0;
        while (e < E && s_off[e + 1] <= slot) ++e;
        if (e >= E || !((active_mask >> e) & 1ull)) continue;
        for (int j = threadIdx.x; j < d4; j += blockDim.x) {
            const size_t i = static_cast<size_t>(slot) * d4 + j;
            float4 acc = __ldcg(ypart + i);
            for (int ks = 1; ks < nsplit; ++ks) {
                const float4 v = __ldcg(ypart + static_cast<size_t>(ks) * plane + i);
                acc.x += v.x; acc.y += v.y; acc.z += v.z; acc.w += v.w;
            }
            y[i] = acc;
        }
    }
}

// K5 from the down pass's split partials: y_slot = ypart[0] + ypart[1] + ... in split
// order (split_reduce_kernel's arithmetic), then combine_kernel's fma chain in j order.
__global__ void combine_splits_kernel(const float4* __restrict__ ypart, int slots, int nsplit,
                                      const int32_t* __restrict__ inv, const float* __restrict__ w,
                                      const uint16_t* __restrict__ res, int T, int d, int k, uint16_t* __restrict__ out) {
    pdl_wait();
    pdl_trigger();
    const int d4 = d / 4;
    const size_t plane = static_cast<size_t>(slots) * d4;
    const long long gid = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (gid >= static_cast<long long>(T) * d4) return;
    const int t = static_cast<int>(gid / d4), c4 = static_cast<int>(gid - static_cast<long long>(t) * d4);
    float acc[4] = {0.f, 0.f, 0.f, 0.f};
    if (res) {
        const uint2 r = *reinterpret_cast<const uint2*>(res + static_cast<size_t>(t) * d + c4 * 4);
        acc[0] = bf16_lo(r.x);
        acc[1] = bf16_hi(r.x);
        acc[2] = bf16_lo(r.y);
        acc[3] = bf16_hi(r.y);
    }
    for (int j = 0; j < k; ++j) {
        const float wj = w[t * k + j];
        const size_t i = static_cast<size_t>(inv[t * k + j]) * d4 + c4;
        float4 v = __ldcg(ypart + i);
        for (int ks = 1; ks < nsplit; ++ks) {
            const float4 q = __ldcg(ypart + static_cast<size_t>(ks) * plane + i);
            v.x += q.x; v.y += q.y; v.z += q.z; v.w += q.w;
        }
        acc[0] = __fmaf_rn(wj, v.x, acc[0]);
        acc[1] = __fmaf_rn(wj, v.y, acc[1]);
        acc[2] = __fmaf_rn(wj, v.z, acc[2]);
        acc[3] = __fmaf_rn(wj, v.w, acc[3]);
    }
    uint2 o;
    o.x = static_cast<uint32_t>(f2bf(acc[0])) | (static_cast<uint32_t>(f2bf(acc[1])) << 16);
    o.y = static_cast<uint32_t>(f2bf(acc[2])) | (static_cast<uint32_t>(f2bf(acc[3])) << 16);
    *reinterpret_cast<uint2*>(out + static_cast<size_t>(t) * d + c4 * 4) = o;
}

// ===========================================================================
// Persistent bf16 256-token variant (tc_ffn_wide): prefill-sized launches.
// One CTA per SM walks the tile list like tc_ffn_persist, at N = 256 (the
// operand bytes per MMA flop of a 128 x 256 tile are 3/4 of a 128 x 128
// tile's).  Shared memory: kWRaw 32 KB weight stages + kWB 32 KB B stages.
// TMEM: pass 0 needs gate + up = 512 columns, so one accumulator: the
// epilogue warps read their 128 columns of both into registers (h packed to
// bf16, 64 registers), release the accumulator, and store while the next
// tile's MMAs run; pass 1 (256 columns) double-buffers the accumulator.
#ifndef MOE_TCW_RAW
#define MOE_TCW_RAW 4
#endif
#ifndef MOE_TCW_B
#define MOE_TCW_B 3
#endif
#ifndef MOE_TCW_A1
#define MOE_TCW_A1 4
#endif
constexpr int kWRaw = MOE_TCW_RAW, kWB = MOE_TCW_B, kWA1 = MOE_TCW_A1;
constexpr int kWSmem = 1024 + kWRaw * 32768 + kWB * 256 * kKc * 2;
constexpr int kWB1 = (kWSmem - 1024 - kWA1 * 16384) / (256 * kKc * 2);  // pass-1 B stages
constexpr int kWMaxA = kWRaw > kWA1 ? kWRaw : kWA1, kWMaxB = kWB > kWB1 ? kWB : kWB1;
static_assert(kWB1 >= 1, "pass-1 stage split");
static_assert(kWSmem + 1024 <= 232448, "tc_ffn_wide stages exceed shared memory");
#ifndef MOE_TCW_PF
#define MOE_TCW_PF 0
#endif
constexpr int kWPf = MOE_TCW_PF;  // weight L2 prefetch distance (chunks; even, 0 = off)
static_assert(kWPf % 2 == 0, "prefetch whole 128-K blocks");


__global__ void __launch_bounds__(kThreads2, 1) tc_ffn_wide(const __grid_constant__ TcArgs a, int ntiles) {
    constexpr int kN = 256, kBTile = kN * kKc * 2;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = smem_raw + ((1024u - (s32(smem_raw) & 1023u)) & 1023u);
    __shared__ __align__(8) uint64_t rb_full[kWMaxA], rb_empty[kWMaxA], b_full[kWMaxB], b_empty[kWMaxB], acc_full[2],
        acc_empty[2];
    __shared__ uint32_t tmem_slot;
    __shared__ int s_off[MOE_MAX_EXPERTS + 1];
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int nmat = a.p == 0 ? 2 : 1;
    // pass 0: kWRaw 32 KB weight stages + kWB B stages; pass 1 (16 KB weight
    // stages): kWA1 weight stages and the rest of the pool as B stages
    const int nA = a.p == 0 ? kWRaw : kWA1, nB = a.p == 0 ? kWB : kWB1;
    const int sA = nmat * kRawA;
    auto rawb = [&](int s) { return smem + s * sA; };
    auto bst = [&](int s) { return smem + nA * sA + s * kBTile; };

    pdl_wait();
    pdl_trigger();
    const int K = a.p == 0 ? a.d : a.f;
    const int RT = (a.p == 0 ? a.f : a.d) / kM;
    const int nk = K / kKc;
    const int grid = static_cast<int>(gridDim.x);
    if (tid <= a.E) s_off[tid] = a.offsets[tid];
    if (tid == 0) {
        for (int s = 0; s < nA; ++s) {
            mbar_init_n(&rb_full[s], 1);
            mbar_init_n(&rb_empty[s], 1);  // MMA commit
        }
        for (int s = 0; s < nB; ++s) {
            mbar_init_n(&b_full[s], 1);
            mbar_init_n(&b_empty[s], 1);
        }
        for (int s = 0; s < 2; ++s) {
            mbar_init_n(&acc_full[s], 1);
            mbar_init_n(&acc_empty[s], kConvThreads / 32);  // the epilogue warps
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 1) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(s32(&tmem_slot)), "r"(512)
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tmem = tmem_slot;
    const int my_tiles = static_cast<int>(blockIdx.x) < ntiles ? (ntiles - static_cast<int>(blockIdx.x) + grid - 1) / grid : 0;
    auto tile_of = [&](int i, Tile& tl) { return find_tile<256>(a, s_off, RT, static_cast<int>(blockIdx.x) + i * grid, tl); };
    // accumulator use i: pass 0 has one buffer (use i waits for release i-1),
    // pass 1 two (use i waits for release i-2)
    const int nbuf = a.p == 0 ? 1 : 2;
    const bool trace = kTcTrace && (a.dbg & 32768) && blockIdx.x == 0;
    auto stamp = [&](int w, int i, int kc) {
        if (trace && i == 2 && kc < 64) g_wtrace[w][kc] = clk32();
    };

    if (warp == 0) {
        // ---- weight producer: both 64-K halves of each 4 KB block back to back ----
        int ub = 0;
        const bool unpaired = a.dbg & 32;  // one 2 KB read per block and chunk, each stage refilled as it frees
        const int pf = (a.dbg & 65536) ? 16 : kWPf;
        for (int i = 0; i < my_tiles; ++i) {
            Tile tl;
            if (!tile_of(i, tl)) break;
            const bool pf_cta = pf > 0 && (!(a.dbg & 131072) || tl.slot0 == s_off[tl.e]);  // bit 17: first token tile only
            for (int kc = 0; kc < nk; kc += unpaired ? 1 : 2, ub += unpaired ? 1 : 2) {
                const int r0 = ub % nA, r1 = (ub + 1) % nA;
                if (ub >= nA) mbar_wait(&rb_empty[r0], static_cast<uint32_t>(((ub / nA) - 1) & 1));
                if (!unpaired && ub + 1 >= nA) mbar_wait(&rb_empty[r1], static_cast<uint32_t>((((ub + 1) / nA) - 1) & 1));
                stamp(0, i, kc);
                if (pf_cta && (kc & 1) == 0 && kc + pf < nk && lane < 8) {
                    // the 4 KB blocks pf chunks ahead into L2: the smem ring then waits on L2, not DRAM
                    const moe_expert_weights& W = a.ex[tl.e];
                    const uint8_t* wb = static_cast<const uint8_t*>(a.p == 0 ? W.w_gate_up : W.w_down);
                    for (int mat = 0; mat < nmat; ++mat) {
                        const int row0 = (a.p == 0 && mat == 1) ? a.f + tl.R0 : tl.R0;
                        const size_t blk = static_cast<size_t>(row0 / 16 + lane) * (K / 128) + ((kc + pf) >> 1);
                        asm volatile("cp.async.bulk.prefetch.L2.global [%0], 4096;" ::"l"(wb + blk * 4096) : "memory");
                    }
                }
                if (a.dbg & 4) {
                    if (lane == 0) {
                        mbar_arrive(&rb_full[r0]);
                        if (!unpaired) mbar_arrive(&rb_full[r1]);
                    }
                    __syncwarp();
                } else if (unpaired) {
                    produce(a, tl, nmat, K, kc, rawb(r0), &rb_full[r0], lane);
                } else {
                    produce_pair(a, tl, nmat, K, kc, rawb(r0), rawb(r1), &rb_full[r0], &rb_full[r1], lane);
                }
            }
        }
    } else if (warp == 2) {
        // ---- B producer ----
        if (lane == 0) {
            int kb = 0;
            for (int i = 0; i < my_tiles; ++i) {
                Tile tl;
                if (!tile_of(i, tl)) break;
                const int nbox = (min(kN, (tl.m + 15) / 16 * 16) + 63) / 64;
                for (int kc = 0; kc < nk; ++kc, ++kb) {
                    const int b = kb % nB;
                    if (kb >= nB) mbar_wait(&b_empty[b], static_cast<uint32_t>(((kb / nB) - 1) & 1));
                    stamp(1, i, kc);
                    if (a.dbg & 4096) {
                        mbar_arrive(&b_full[b]);
                        continue;
                    }
                    mbar_expect_tx(&b_full[b], static_cast<uint32_t>(nbox) * 64 * 128);
                    for (int q = 0; q < nbox; ++q) tma_load_b(bst(b) + q * 8192, &a.tmb, kc * kKc, tl.slot0 + q * 64, &b_full[b]);
                }
            }
        }
        __syncwarp();
    } else if (warp == 1) {
        // ---- MMA issuer ----
        int kb = 0;
        for (int i = 0; i < my_tiles; ++i) {
            Tile tl;
            if (!tile_of(i, tl)) break;
            const int nmma = min(kN, (tl.m + 15) / 16 * 16);
            const uint32_t id = idesc(1, nmma, kM);
            const int buf = i % nbuf;
            if (i >= nbuf) mbar_wait(&acc_empty[buf], static_cast<uint32_t>(((i / nbuf) - 1) & 1));
            asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
            const uint32_t dacc = tmem + buf * kN;
            for (int kc = 0; kc < nk; ++kc, ++kb) {
                const int r = kb % nA, b = kb % nB;
                mbar_wait(&rb_full[r], static_cast<uint32_t>((kb / nA) & 1));
                if (lane == 0) stamp(2, i, kc);
                mbar_wait(&b_full[b], static_cast<uint32_t>((kb / nB) & 1));
                if (lane == 0) stamp(3, i, kc);
                asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
                const uint32_t ab = s32(rawb(r)), bb = s32(bst(b));
                if (a.dbg & 8192) {  // handshake probe: plain arrives instead of commits
                    if (lane == 0) {
                        mbar_arrive(&rb_empty[r]);
                        mbar_arrive(&b_empty[b]);
                        if (kc == nk - 1) mbar_arrive(&acc_full[buf]);
                    }
                } else {
                    if (!(a.dbg & 2)) {
#pragma unroll
                        for (int j = 0; j < kKc / 16; ++j) {
                            const uint64_t bdesc = sdesc(bb + j * 32);
                            const uint32_t acc = (kc > 0 || j > 0) ? 1u : 0u;
                            umma_elect(dacc, sdesc_core(ab + j * 256), bdesc, id, acc);
                            if (nmat == 2) umma_elect(dacc + kN, sdesc_core(ab + kRawA + j * 256), bdesc, id, acc);
                        }
                    }
                    umma_commit_elect(&rb_empty[r]);
                    umma_commit_elect(&b_empty[b]);
                    if (kc == nk - 1) umma_commit_elect(&acc_full[buf]);
                }
                if (lane == 0) stamp(4, i, kc);
                __syncwarp();
            }
        }
    } else if (warp >= 4) {
        // ---- epilogue ----
        const int row = (warp & 3) * 32 + lane;
        const uint32_t lane_base = static_cast<uint32_t>((warp & 3) * 32) << 16;
        const int c0 = ((warp - 4) >> 2) * (kN / 2);
        for (int i = 0; i < my_tiles; ++i) {
            Tile tl;
            if (!tile_of(i, tl)) break;
            const int buf = i % nbuf;
            mbar_wait(&acc_full[buf], static_cast<uint32_t>((i / nbuf) & 1));
            asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
            const uint32_t dacc = tmem + buf * kN;
            if (a.p == 0) {
                // h for this thread's row x 128 columns, packed, then the accumulator is free
                uint32_t hp[kN / 4];
#pragma unroll
                for (int q = 0; q < 8; ++q) {
                    uint32_t g[16], u[16];
                    TMEM_LD16(dacc + lane_base + c0 + q * 16, g);
                    TMEM_LD16(dacc + lane_base + kN + c0 + q * 16, u);
                    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
                    for (int c = 0; c < 16; c += 2) {
                        hp[q * 8 + c / 2] = bf16x2_rn(silu_tanh(__uint_as_float(g[c])) * __uint_as_float(u[c]),
                                                      silu_tanh(__uint_as_float(g[c + 1])) * __uint_as_float(u[c + 1]));
                    }
                }
                asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
                __syncwarp();
                if (lane == 0) mbar_arrive(&acc_empty[buf]);
                if (!(a.dbg & 2048)) {
                    uint16_t* ho = a.hout + static_cast<size_t>(tl.slot0 + c0) * a.f + tl.R0 + row;
#pragma unroll
                    for (int c = 0; c < kN / 2; ++c)
                        if (c0 + c < tl.m) ho[static_cast<size_t>(c) * a.f] = static_cast<uint16_t>(hp[c >> 1] >> ((c & 1) * 16));
                }
            } else {
                for (int cbk = c0; cbk < c0 + kN / 2 && cbk < tl.m && !(a.dbg & 2048); cbk += 32) {
                    uint32_t g[32];
                    TMEM_LD32(dacc + lane_base + cbk, g);
                    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
                    for (int c = 0; c < 32; ++c)
                        if (cbk + c < tl.m)
                            a.y[static_cast<size_t>(tl.slot0 + cbk + c) * a.d + tl.R0 + row] = __uint_as_float(g[c]);
                }
                asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
                __syncwarp();
                if (lane == 0) mbar_arrive(&acc_empty[buf]);
            }
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (warp == 1) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512) : "memory");
    if (trace && tid == 0 && my_tiles > 2) {
        const unsigned int t0 = g_wtrace[0][0];
        for (int kc = 0; kc < min(nk, 64); ++kc)
            printf("WTRACE p%d kc %2d wiss %7d biss %7d wfull %7d bfull %7d mma %7d\n", a.p, kc, g_wtrace[0][kc] - t0,
                   g_wtrace[1][kc] - t0, g_wtrace[2][kc] - t0, g_wtrace[3][kc] - t0, g_wtrace[4][kc] - t0);
    }
}

// ===========================================================================
// CTA-pair persistent variant (tc_ffn_wide2, clusters of 2): the same tile
// loop as tc_ffn_wide with tcgen05.mma.cta_group::2, M = 256.  CTA r of a
// pair holds rows R0 + 128r .. of the pair's 256-row tile (its own weights)
// and tokens [r N/2, (r+1) N/2) of the tile's B, and accumulates its 128 rows
// x N columns in its own TMEM.  Each SM's stages hold half of B, so the same
// shared memory keeps more chunks in flight (pass 0: 48 KB per chunk instead
// of 64, pass 1: 32 instead of 48) -- the operand streams are latency-bound.
// Hand-offs: each CTA loads its own stages on its own barriers; a forwarder
// lane per CTA arrives on the leader's pair barrier once both of its stages
// landed; the leader's MMA warp issues, and its commits multicast the stage
// releases and accumulator-ready signals to both CTAs; both CTAs' epilogue
// warps release the accumulator on the leader's barrier.
#ifndef MOE_TCW2_A0
#define MOE_TCW2_A0 5
#endif
#ifndef MOE_TCW2_A1
#define MOE_TCW2_A1 8
#endif
constexpr int kW2Pool = 224 * 1024;
constexpr int kW2A0 = MOE_TCW2_A0, kW2B0 = (kW2Pool - kW2A0 * 32768) / 16384;  // pass 0: 32 KB A, 16 KB B stages
constexpr int kW2A1 = MOE_TCW2_A1, kW2B1 = (kW2Pool - kW2A1 * 16384) / 16384;  // pass 1: 16 KB A, 16 KB B stages
constexpr int kW2MaxA = kW2A0 > kW2A1 ? kW2A0 : kW2A1, kW2MaxB = kW2B0 > kW2B1 ? kW2B0 : kW2B1;
constexpr int kW2R4 = 5;   // int4 raw units in region R (pass 0: 5, pass 1: 3 fit)
constexpr int kW2Np = 16;  // pair-barrier ring (> the chunks a forwarder can run ahead)
constexpr int kW2Smem = 1024 + kW2Pool;
static_assert(kW2MaxA < kW2Np && kW2MaxB < kW2Np && kW2B0 >= 2 && kW2B1 >= 2, "tc_ffn_wide2 stage split");

MOE_DEVI uint32_t cluster_ctarank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
MOE_DEVI void cluster_sync_all() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
MOE_DEVI uint32_t mapa_shared(uint32_t addr, uint32_t rank) {
    uint32_t r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(addr), "r"(rank));
    return r;
}
MOE_DEVI void mbar_arrive_remote(uint32_t cluster_addr) {
    asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr) : "memory");
}
MOE_DEVI void mbar_arrive_remote_relaxed(uint32_t cluster_addr) {
    asm volatile("mbarrier.arrive.relaxed.cluster.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr) : "memory");
}
MOE_DEVI void umma2_elect(uint32_t dtmem, uint64_t a, uint64_t b, uint32_t id, uint32_t accum) {
    asm volatile(
        "{\n\t.reg .pred p, e;\n\telect.sync _|e, 0xffffffff;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "@e tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n}" ::"r"(dtmem),
        "l"(a), "l"(b), "r"(id), "r"(accum)
        : "memory");
}
MOE_DEVI void umma2_commit_both_elect(uint64_t* bar) {
    asm volatile(
        "{\n\t.reg .pred e;\n\t.reg .b16 m;\n\telect.sync _|e, 0xffffffff;\n\tmov.b16 m, 3;\n\t"
        "@e tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], m;\n}" ::"r"(
            s32(bar))
        : "memory");
}

__global__ void __launch_bounds__(kThreads2, 1) tc_ffn_wide2(const __grid_constant__ TcArgs a, int ntiles) {
    constexpr int kN = 256, kBHalf = 128 * kKc * 2;  // 16 KB: 128 token rows x 64 K
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = smem_raw + ((1024u - (s32(smem_raw) & 1023u)) & 1023u);
    __shared__ __align__(8) uint64_t rb_full[kW2MaxA], rb_empty[kW2MaxA], b_full[kW2MaxB], b_empty[kW2MaxB],
        pair_full[kW2Np], acc_full[2], acc_empty[2], r4_full[kW2R4], r4_empty[kW2R4], cn_full[2], cn_empty[2];
    __shared__ uint32_t tmem_slot;
    __shared__ int s_off[MOE_MAX_EXPERTS + 1];
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const uint32_t rank = cluster_ctarank();
    const int nmat = a.p == 0 ? 2 : 1;
    const int nA = a.p == 0 ? kW2A0 : kW2A1, nB = a.p == 0 ? kW2B0 : kW2B1;
    const int sA = nmat * kRawA;
    auto rawb = [&](int s) { return smem + s * sA; };
    auto bst = [&](int s) { return smem + nA * sA + s * kBHalf; };
    // int4 tiles reuse region R (the bf16 weight ring): two canonical fp16 A stages, then
    // compact raw units (tc_ffn_persist's layout)
    const int nR4 = min(kW2R4, (nA * sA - 2 * 32768) / kPRaw4Unit);
    auto can = [&](int s) { return smem + s * 32768; };
    auto raw4 = [&](int s) { return smem + 2 * 32768 + s * kPRaw4Unit; };
    auto is_p4 = [&](const Tile& t) { return a.ex[t.e].precision == MOE_P4; };

    pdl_wait();
    pdl_trigger();
    const int K = a.p == 0 ? a.d : a.f;
    const int RP = (a.p == 0 ? a.f : a.d) / (2 * kM);  // 256-row pair tiles per expert
    const int nk = K / kKc;
    const int npair = static_cast<int>(gridDim.x) / 2, pair = static_cast<int>(blockIdx.x) / 2;
    if (tid <= a.E) s_off[tid] = a.offsets[tid];
    if (tid == 0) {
        for (int s = 0; s < nA; ++s) {
            mbar_init_n(&rb_full[s], 1);
            mbar_init_n(&rb_empty[s], 1);  // the leader's multicast commit
        }
        for (int s = 0; s < nB; ++s) {
            mbar_init_n(&b_full[s], 1);
            mbar_init_n(&b_empty[s], 1);
        }
        for (int s = 0; s < kW2Np; ++s) mbar_init_n(&pair_full[s], 2);  // one forwarder arrival per CTA
        for (int s = 0; s < 2; ++s) {
            mbar_init_n(&acc_full[s], 1);
            mbar_init_n(&acc_empty[s], 2 * (kConvThreads / 32));  // both CTAs' epilogue warps
            mbar_init_n(&cn_full[s], kConvThreads / 32);          // this CTA's converter warps
            mbar_init_n(&cn_empty[s], 1);                         // the leader's multicast commit
        }
        for (int s = 0; s < kW2R4; ++s) {
            mbar_init_n(&r4_full[s], 1);
            mbar_init_n(&r4_empty[s], kConvThreads / 32);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 1) {
        asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(s32(&tmem_slot)), "r"(512)
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    cluster_sync_all();  // the peer's barriers exist before any remote arrive or multicast commit
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tmem = tmem_slot;
    const int my_tiles = pair < ntiles ? (ntiles - pair + npair - 1) / npair : 0;
    // the pair's tile i: 256 rows (this CTA's 128 at R0) x up to 256 tokens; both CTAs agree
    auto tile_of = [&](int i, Tile& tl) {
        if (!find_tile<256>(a, s_off, RP, pair + i * npair, tl)) return false;
        tl.R0 = tl.R0 * 2 + static_cast<int>(rank) * kM;  // find_tile's R0 = pair-row-tile * 128
        return true;
    };
    auto n_of = [&](const Tile& tl) { return min(kN, (tl.m + 31) / 32 * 32); };  // both halves whole 16-column steps
    const int nbuf = a.p == 0 ? 1 : 2;
    const bool trace = kTcTrace && (a.dbg & 32768) && blockIdx.x < 2;
    auto stamp = [&](int w, int i, int kc) {
        if (trace && i == 2 && kc < 64) g_wtrace2[rank][w][kc] = clk32();
    };

    if (warp == 0) {
        // ---- this CTA's weight rows: bf16 both 64-K halves of each 4 KB block back to
        // back; int4 one compact raw unit per 128-K group ----
        int ub = 0, u4 = 0, prev = -1;
        for (int i = 0; i < my_tiles; ++i) {
            Tile tl;
            if (!tile_of(i, tl)) break;
            const bool p4 = is_p4(tl);
            if (prev >= 0 && prev != static_cast<int>(p4))  // region R changes role: the previous tile's MMAs first
                mbar_wait(&acc_full[(i - 1) % nbuf], static_cast<uint32_t>(((i - 1) / nbuf) & 1));
            prev = p4;
            if (p4) {
                for (int kc = 0; kc < nk; kc += 2, ++u4) {
                    const int r = u4 % nR4;
                    if (u4 >= nR4) mbar_wait(&r4_empty[r], static_cast<uint32_t>(((u4 / nR4) - 1) & 1));
                    produce4c(a, tl, nmat, K, kc, raw4(r), &r4_full[r], lane);
                }
                continue;
            }
            for (int kc = 0; kc < nk; kc += 2, ub += 2) {
                const int r0 = ub % nA, r1 = (ub + 1) % nA;
                if (ub >= nA) mbar_wait(&rb_empty[r0], static_cast<uint32_t>(((ub / nA) - 1) & 1));
                if (ub + 1 >= nA) mbar_wait(&rb_empty[r1], static_cast<uint32_t>((((ub + 1) / nA) - 1) & 1));
                if (lane == 0) stamp(0, i, kc);
                produce_pair(a, tl, nmat, K, kc, rawb(r0), rawb(r1), &rb_full[r0], &rb_full[r1], lane);
            }
        }
    } else if (warp == 2) {
        // ---- this CTA's half of the tile's tokens ----
        if (lane == 0) {
            int kb = 0;
            for (int i = 0; i < my_tiles; ++i) {
                Tile tl;
                if (!tile_of(i, tl)) break;
                const int halfn = n_of(tl) / 2, nbox = (halfn + 63) / 64;
                const int row0 = tl.slot0 + static_cast<int>(rank) * halfn;
                const CUtensorMap* tm = is_p4(tl) ? &a.tmb16 : &a.tmb;  // int4 tiles multiply fp16 activations
                for (int kc = 0; kc < nk; ++kc, ++kb) {
                    const int b = kb % nB;
                    if (kb >= nB) mbar_wait(&b_empty[b], static_cast<uint32_t>(((kb / nB) - 1) & 1));
                    mbar_expect_tx(&b_full[b], static_cast<uint32_t>(nbox) * 64 * 128);
                    for (int q = 0; q < nbox; ++q) tma_load_b(bst(b) + q * 8192, tm, kc * kKc, row0 + q * 64, &b_full[b]);
                }
            }
        }
        __syncwarp();
    } else if (warp == 3) {
        // ---- forwarder: both of this CTA's stages of chunk kb landed -> the leader's pair barrier ----
        if (lane == 0) {
            int kb = 0, cb = 0, c4 = 0;
            for (int i = 0; i < my_tiles; ++i) {
                Tile tl;
                if (!tile_of(i, tl)) break;
                const bool p4 = is_p4(tl);
                for (int kc = 0; kc < nk; ++kc, ++kb) {
                    if (p4) {
                        mbar_wait(&cn_full[c4 & 1], static_cast<uint32_t>((c4 >> 1) & 1));
                        ++c4;
                    } else {
                        mbar_wait(&rb_full[cb % nA], static_cast<uint32_t>((cb / nA) & 1));
                        ++cb;
                    }
                    mbar_wait(&b_full[kb % nB], static_cast<uint32_t>((kb / nB) & 1));
                    stamp(1, i, kc);
                    // relaxed: the stages' bytes already landed (this lane observed the
                    // complete_tx); a release at cluster scope costs ~1,400 cycles per
                    // chunk on the critical path (MOE_TC_DBG bit 19 selects it: 1193 -> 756 TF/s)
                    if (a.dbg & 524288)
                        mbar_arrive_remote(mapa_shared(s32(&pair_full[kb % kW2Np]), 0));
                    else
                        mbar_arrive_remote_relaxed(mapa_shared(s32(&pair_full[kb % kW2Np]), 0));
                }
            }
        }
        __syncwarp();
    } else if (warp == 1) {
        // ---- the leader's MMA warp ----
        if (rank == 0) {
            int kb = 0, cb = 0, c4 = 0;
            for (int i = 0; i < my_tiles; ++i) {
                Tile tl;
                if (!tile_of(i, tl)) break;
                const bool p4 = is_p4(tl);
                const uint32_t id = idesc(p4 ? 0 : 1, n_of(tl), 2 * kM);
                const int buf = i % nbuf;
                if (i >= nbuf) mbar_wait(&acc_empty[buf], static_cast<uint32_t>(((i / nbuf) - 1) & 1));
                asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
                const uint32_t dacc = tmem + buf * kN;
                for (int kc = 0; kc < nk; ++kc, ++kb) {
                    const int b = kb % nB;
                    mbar_wait(&pair_full[kb % kW2Np], static_cast<uint32_t>((kb / kW2Np) & 1));
                    if (lane == 0) stamp(2, i, kc);
                    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
                    const uint32_t bb = s32(bst(b));
                    if (p4) {  // canonical SW128 fp16 A stages written by the converters
                        const uint32_t ab = s32(can(c4 & 1));
#pragma unroll
                        for (int j = 0; j < kKc / 16; ++j) {
                            const uint64_t bdesc = sdesc(bb + j * 32);
                            const uint32_t acc = (kc > 0 || j > 0) ? 1u : 0u;
                            umma2_elect(dacc, sdesc(ab + j * 32), bdesc, id, acc);
                            if (nmat == 2) umma2_elect(dacc + kN, sdesc(ab + kTileBytes + j * 32), bdesc, id, acc);
                        }
                        umma2_commit_both_elect(&cn_empty[c4 & 1]);
                        ++c4;
                    } else {  // the raw bf16 core-matrix blocks
                        const uint32_t ab = s32(rawb(cb % nA));
#pragma unroll
                        for (int j = 0; j < kKc / 16; ++j) {
                            const uint64_t bdesc = sdesc(bb + j * 32);
                            const uint32_t acc = (kc > 0 || j > 0) ? 1u : 0u;
                            umma2_elect(dacc, sdesc_core(ab + j * 256), bdesc, id, acc);
                            if (nmat == 2) umma2_elect(dacc + kN, sdesc_core(ab + kRawA + j * 256), bdesc, id, acc);
                        }
                        umma2_commit_both_elect(&rb_empty[cb % nA]);
                        ++cb;
                    }
                    umma2_commit_both_elect(&b_empty[b]);
                    if (kc == nk - 1) umma2_commit_both_elect(&acc_full[buf]);
                    if (lane == 0) stamp(3, i, kc);
                }
            }
        }
        __syncwarp();
    } else if (warp >= 4) {
        // ---- epilogue: this CTA's 128 rows x the tile's tokens ----
        const int row = (warp & 3) * 32 + lane;
        const uint32_t lane_base = static_cast<uint32_t>((warp & 3) * 32) << 16;
        const int c0 = ((warp - 4) >> 2) * (kN / 2);
        const uint32_t leader_empty0 = mapa_shared(s32(&acc_empty[0]), 0), leader_empty1 = mapa_shared(s32(&acc_empty[1]), 0);
        const int ct = tid - 128;
        ConvOffsets o0, o1;
        conv_offsets(ct, 0, o0);
        conv_offsets(ct, 1, o1);
        int u4 = 0, c4 = 0;
        for (int i = 0; i < my_tiles; ++i) {
            Tile tl;
            if (!tile_of(i, tl)) break;
            const bool p4 = is_p4(tl);
            if (p4) {
                // ---- converters: this CTA's int4 rows -> fp16 q*s canonical A stages ----
                for (int kc = 0; kc < nk; ++kc, ++c4) {
                    const int r = u4 % nR4, c = c4 & 1;
                    if ((kc & 1) == 0) mbar_wait(&r4_full[r], static_cast<uint32_t>((u4 / nR4) & 1));
                    if (c4 >= 2) mbar_wait(&cn_empty[c], static_cast<uint32_t>(((c4 >> 1) - 1) & 1));
                    convert_int4c(nmat, raw4(r), can(c), ct, (kc & 1) ? o1 : o0);
                    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                    __syncwarp();
                    if (lane == 0) {
                        mbar_arrive(&cn_full[c]);
                        if (kc & 1) mbar_arrive(&r4_empty[r]);
                    }
                    if (kc & 1) ++u4;
                }
            }
            const int buf = i % nbuf;
            mbar_wait(&acc_full[buf], static_cast<uint32_t>((i / nbuf) & 1));
            asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
            const uint32_t dacc = tmem + buf * kN;
            if (a.p == 0) {
                uint32_t hp[kN / 4];
#pragma unroll
                for (int q = 0; q < 8; ++q) {
                    uint32_t g[16], u[16];
                    TMEM_LD16(dacc + lane_base + c0 + q * 16, g);
                    TMEM_LD16(dacc + lane_base + kN + c0 + q * 16, u);
                    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
                    for (int c = 0; c < 16; c += 2) {
                        hp[q * 8 + c / 2] = bf16x2_rn(silu_tanh(__uint_as_float(g[c])) * __uint_as_float(u[c]),
                                                      silu_tanh(__uint_as_float(g[c + 1])) * __uint_as_float(u[c + 1]));
                    }
                }
                asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
                __syncwarp();
                if (lane == 0) mbar_arrive_remote(buf ? leader_empty1 : leader_empty0);
                const size_t o = static_cast<size_t>(tl.slot0 + c0) * a.f + tl.R0 + row;
                uint16_t* ho = a.hout + o;
#pragma unroll
                for (int c = 0; c < kN / 2; ++c)
                    if (c0 + c < tl.m) ho[static_cast<size_t>(c) * a.f] = static_cast<uint16_t>(hp[c >> 1] >> ((c & 1) * 16));
                if (p4) {  // the fp16 copy feeds only an int4 down pass
                    uint16_t* h16 = a.hout16 + o;
#pragma unroll
                    for (int c = 0; c < kN / 2; ++c) {
                        if (c0 + c < tl.m) {
                            const float hv = bf2f(static_cast<uint16_t>(hp[c >> 1] >> ((c & 1) * 16)));
                            if (f16_overflow(hv)) numerics_flag(MOE_NUM_F16_ACT);
                            h16[static_cast<size_t>(c) * a.f] = __half_as_ushort(__float2half_rn(hv));
                        }
                    }
                }
            } else {
                for (int cbk = c0; cbk < c0 + kN / 2 && cbk < tl.m; cbk += 32) {
                    uint32_t g[32];
                    TMEM_LD32(dacc + lane_base + cbk, g);
                    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
                    for (int c = 0; c < 32; ++c)
                        if (cbk + c < tl.m)
                            a.y[static_cast<size_t>(tl.slot0 + cbk + c) * a.d + tl.R0 + row] = __uint_as_float(g[c]);
                }
                asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
                __syncwarp();
                if (lane == 0) mbar_arrive_remote(buf ? leader_empty1 : leader_empty0);
            }
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    cluster_sync_all();  // neither CTA frees TMEM while the pair's MMAs may still write it
    if (warp == 1) asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512) : "memory");
    if (trace && tid == 0 && rank == 0 && my_tiles > 2) {
        const unsigned int t0 = g_wtrace2[0][0][0];
        for (int kc = 0; kc < min(nk, 64); ++kc)
            printf("W2TRACE p%d kc %2d wiss0 %7d wiss1 %7d fwd0 %7d fwd1 %7d pfull %7d mma %7d\n", a.p, kc,
                   g_wtrace2[0][0][kc] - t0, g_wtrace2[1][0][kc] - t0, g_wtrace2[0][1][kc] - t0,
                   g_wtrace2[1][1][kc] - t0, g_wtrace2[0][2][kc] - t0, g_wtrace2[0][3][kc] - t0);
    }
}

// Pass-0 B operand in slot order: xs[slot] = x[token of slot] (bf16) and
// its fp16 copy (int4 experts), so every tile's token rows are one TMA box
// column.  One 16-byte chunk per thread.
__global__ void gather_rows_kernel(const uint16_t* __restrict__ x, const int32_t* __restrict__ perm, int slots, int d,
                                   int k, int kshift, uint16_t* __restrict__ xs, uint16_t* __restrict__ xs16,
                                   unsigned int* __restrict__ dep, int ndep) {
    pdl_wait();
    pdl_trigger();
    // the fused launch's tile counters (its PDL wait orders this before any use; the
    // previous layer's fused launch finished before our own wait returned)
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < ndep; i += gridDim.x * blockDim.x) dep[i] = 0u;
    const int cpr = d / 8;
    for (long long i = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
         i < static_cast<long long>(slots) * cpr; i += static_cast<long long>(gridDim.x) * blockDim.x) {
        const int slot = static_cast<int>(i / cpr), c = static_cast<int>(i - static_cast<long long>(slot) * cpr);
        const int pv = perm[slot];
        const int t = kshift >= 0 ? pv >> kshift : pv / k;
        const uint4 v = reinterpret_cast<const uint4*>(x + static_cast<size_t>(t) * d)[c];
        reinterpret_cast<uint4*>(xs + static_cast<size_t>(slot) * d)[c] = v;
        const uint32_t w[4] = {v.x, v.y, v.z, v.w};
        uint32_t h[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            h[q] = static_cast<uint32_t>(__half_as_ushort(__float2half_rn(bf16_lo(w[q])))) |
                   (static_cast<uint32_t>(__half_as_ushort(__float2half_rn(bf16_hi(w[q])))) << 16);
            if (f16_overflow(bf16_lo(w[q])) || f16_overflow(bf16_hi(w[q]))) numerics_flag(MOE_NUM_F16_ACT);
        }
        reinterpret_cast<uint4*>(xs16 + static_cast<size_t>(slot) * d)[c] = make_uint4(h[0], h[1], h[2], h[3]);
    }
}

// 2D tensor map over rows x K bf16/fp16 values (row stride K * 2 bytes),
// 64 x 64 boxes, 128-byte swizzle -- the canonical B tile layout.
cudaError_t encode_b(CUtensorMap* tm, const void* base, int K, int rows) {
    static PFN_cuTensorMapEncodeTiled_v12000 enc = nullptr;
    if (enc == nullptr) {
        cudaDriverEntryPointQueryResult q;
        void* fn = nullptr;
        MOE_CUDA_OK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q));
        if (fn == nullptr || q != cudaDriverEntryPointSuccess) return cudaErrorNotSupported;
        enc = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
    }
    const cuuint64_t dims[2] = {static_cast<cuuint64_t>(K), static_cast<cuuint64_t>(rows)};
    const cuuint64_t strides[1] = {static_cast<cuuint64_t>(K) * 2};
    const cuuint32_t box[2] = {static_cast<cuuint32_t>(kKc), 64};
    const cuuint32_t estr[2] = {1, 1};
    const CUresult r = enc(tm, CU_TENSOR_MAP_DATA_TYPE_UINT16, 2, const_cast<void*>(base), dims, strides, box, estr,
                           CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                           CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS ? cudaSuccess : cudaErrorInvalidValue;
}

}  // namespace tc
}  // namespace moek

#ifndef MOE_TC_DOWN_SPLIT
#define MOE_TC_DOWN_SPLIT 4
#endif
constexpr int kDownSplit = MOE_TC_DOWN_SPLIT;  // K splits of the down pass on the persistent kernel

size_t moek_tc_workspace_bytes(int T, int k, int d, int f) {
    const size_t slots = static_cast<size_t>(T) * k;
    // xs, xs16, h, h16, the down pass's split partials, the fused launch's tile counters
    return 2 * slots * d * 2 + 2 * slots * f * 2 + static_cast<size_t>(kDownSplit) * slots * d * 4 +
           static_cast<size_t>(MOE_MAX_EXPERTS) * (slots / 128 + 2) * kDownSplit * 4 + 1024;
}

// Grouped expert FFN on tcgen05 for every expert segment of a permutation:
// x natural [T][d] bf16 (already normalised), y_perm [T*k][d] fp32.
namespace {
struct TcCombine {  // optional K5 fused into the down pass's reduction (moek_ffn_tc_combine)
    const int32_t* inv;
    const float* w;
    const void* res;
    void* out;
};
cudaError_t ffn_tc_impl(void* ws, const void* x, const int32_t* perm, const int32_t* offsets, int T, int k,
                        const moe_expert_weights* experts, int E, int d, int f, uint64_t active_mask, float* y,
                        const TcCombine* cmb, bool* combined, cudaStream_t stream) {
    using namespace moek::tc;
    *combined = false;
    if (d % kM != 0 || f % kM != 0 || d % 128 != 0 || f % 128 != 0) return cudaErrorInvalidValue;
    static bool attr = false;
    if (!attr) {
        MOE_CUDA_OK(cudaFuncSetAttribute(tc_ffn_kernel<128>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         TcCfg<128>::kSmem));
        MOE_CUDA_OK(cudaFuncSetAttribute(tc_ffn_kernel<256>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         TcCfg<256>::kSmem));
        attr = true;
    }
    const size_t slots = static_cast<size_t>(T) * k;
    uint16_t* xs = static_cast<uint16_t*>(ws);
    uint16_t* xs16 = xs + slots * d;
    uint16_t* h = xs16 + slots * d;
    uint16_t* h16 = h + slots * f;
    float* ypart = reinterpret_cast<float*>(h16 + slots * f);
    unsigned int* dep = reinterpret_cast<unsigned int*>(ypart + static_cast<size_t>(kDownSplit) * slots * d);
    const int dep_tt = static_cast<int>(slots / 128 + 2);
    const int kshift = (k & (k - 1)) == 0 ? __builtin_ctz(static_cast<unsigned>(k)) : -1;
    TcArgs a{};
    a.offsets = offsets;
    a.perm = perm;
    a.T = T;
    a.k = k;
    a.E = E;
    a.kshift = (k & (k - 1)) == 0 ? __builtin_ctz(static_cast<unsigned>(k)) : -1;
    a.d = d;
    a.f = f;
    a.active_mask = active_mask;
    static const int dbg = getenv("MOE_TC_DBG") ? atoi(getenv("MOE_TC_DBG")) : 0;
    a.dbg = dbg;
    for (int e = 0; e < E; ++e) a.ex[e] = experts[e];
    // 256-token tiles once the average active expert sees at least 128 slots
    // (MOE_TC_DBG bit3 forces 128, bit4 forces 256)
    int nact = 0;
    for (int e = 0; e < E; ++e) nact += static_cast<int>((active_mask >> e) & 1ull);
    bool wide = nact > 0 && slots >= static_cast<size_t>(128) * nact;  // at 128 per expert the pair wins (bf16 +9 %)
    if (dbg & 8) wide = false;
    if (dbg & 16) wide = true;
    const int NT = wide ? 256 : 128;
    const int ntiles_max = static_cast<int>((slots + NT - 1) / NT) + E;
    auto kern = wide ? tc_ffn_kernel<256> : tc_ffn_kernel<128>;
    const int smem = wide ? TcCfg<256>::kSmem : TcCfg<128>::kSmem;
    // 128-token tiles: the persistent kernel over the exact tile count (MOE_TC_DBG bit 8 of 256: off)
    const bool persist = !wide && !(dbg & 256);
    static int sms = 0;
    if (sms == 0) {
        int dev = 0;
        MOE_CUDA_OK(cudaGetDevice(&dev));
        MOE_CUDA_OK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
        MOE_CUDA_OK(cudaFuncSetAttribute(tc_ffn_persist, cudaFuncAttributeMaxDynamicSharedMemorySize, kPSmem));
    }
    // wide launches: bf16 experts through the persistent tc_ffn_wide (MOE_TC_DBG
    // bit 14: off), int4 experts through tc_ffn_kernel<256>
    // (the CTA-pair kernel converts int4 tiles too: MOE_TC_DBG bit 23 sends them to
    // tc_ffn_kernel<256> instead)
    const bool wpair = !(dbg & 262144) && (f / kM) % 2 == 0 && (d / kM) % 2 == 0;  // MOE_TC_DBG bit 18: single-CTA tiles
    uint64_t mask16 = 0;
    for (int e = 0; e < E; ++e)
        if (((active_mask >> e) & 1ull) && (experts[e].precision != MOE_P4 || (wpair && !(dbg & 8388608))))
            mask16 |= 1ull << e;
    const bool wpers = wide && mask16 != 0 && !(dbg & 16384);
    const uint64_t mask_single = wpers ? (active_mask & ~mask16) : active_mask;
    static bool wide_attr = false;
    if (wpers && !wide_attr) {
        MOE_CUDA_OK(cudaFuncSetAttribute(tc_ffn_wide, cudaFuncAttributeMaxDynamicSharedMemorySize, kWSmem));
        wide_attr = true;
    }
    static bool pair_attr = false;
    if (wpers && wpair && !pair_attr) {
        MOE_CUDA_OK(cudaFuncSetAttribute(tc_ffn_wide2, cudaFuncAttributeMaxDynamicSharedMemorySize, kW2Smem));
        pair_attr = true;
    }
    auto launch_wide = [&](int rows) -> cudaError_t {
        TcArgs aw = a;
        aw.active_mask = mask16;
        if (wpair) {
            const int np = ntiles_max * (rows / kM / 2);
            cudaLaunchConfig_t cfg{};
            cfg.gridDim = dim3(static_cast<unsigned>(2 * std::min(np, sms / 2)));
            cfg.blockDim = dim3(kThreads2);
            cfg.dynamicSmemBytes = kW2Smem;
            cfg.stream = stream;
            cudaLaunchAttribute attr[2];
            attr[0].id = cudaLaunchAttributeClusterDimension;
            attr[0].val.clusterDim.x = 2;
            attr[0].val.clusterDim.y = 1;
            attr[0].val.clusterDim.z = 1;
            attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
            attr[1].val.programmaticStreamSerializationAllowed = 1;
            cfg.attrs = attr;
            cfg.numAttrs = 2;
            return cudaLaunchKernelEx(&cfg, tc_ffn_wide2, aw, np);
        }
        const int nt = ntiles_max * (rows / kM);
        return moek::launch_pdl(tc_ffn_wide, dim3(static_cast<unsigned>(std::min(nt, sms))), dim3(kThreads2), kWSmem,
                                stream, aw, nt);
    };
    // exact tile counts per pass need the routing (device); the persistent grid instead
    // walks tiles [0, ntiles_max * RT) and skips the empty ones (find_tile returns false)
    // pass 0: gate/up + SwiGLU -> h
    a.p = 0;
    MOE_CUDA_OK(encode_b(&a.tmb, xs, d, static_cast<int>(slots)));
    MOE_CUDA_OK(encode_b(&a.tmb16, xs16, d, static_cast<int>(slots)));
    a.hout = h;
    a.hout16 = h16;
    // K split of the persistent down pass in kDownSplit parts when every part keeps whole
    // int4 chunk pairs
    const int ns = (f / kKc) % (2 * kDownSplit) == 0 && !(dbg & 512) ? kDownSplit : 1;
    // one persistent launch for both passes (MOE_TC_DBG bit 21: two): the down tiles of
    // a (token tile, K split) start once its gate/up tiles are stored, so the last
    // gate/up wave shares the machine with the first down tiles
    const bool fuse = persist && !(dbg & 2097152) && (f / kM) % ns == 0;
    const int ndep = fuse ? E * dep_tt * ns : 0;
    const long long nch = static_cast<long long>(slots) * (d / 8);
    MOE_CUDA_OK(moek::launch_pdl(gather_rows_kernel, dim3(static_cast<unsigned>(std::min<long long>((nch + 255) / 256, 2368))),
                                 dim3(256), 0, stream, static_cast<const uint16_t*>(x), perm, static_cast<int>(slots), d, k,
                                 kshift, xs, xs16, dep, ndep));
    if (fuse) {
        MOE_CUDA_OK(encode_b(&a.tmb, xs, d, static_cast<int>(slots)));
        MOE_CUDA_OK(encode_b(&a.tmb16, xs16, d, static_cast<int>(slots)));
        MOE_CUDA_OK(encode_b(&a.tmh, h, f, static_cast<int>(slots)));
        MOE_CUDA_OK(encode_b(&a.tmh16, h16, f, static_cast<int>(slots)));
        a.p = 0;
        a.hout = h;
        a.hout16 = h16;
        a.y = y;
        a.dep = dep;
        a.dep_tt = dep_tt;
        const int nt = ntiles_max * (f / kM) + ntiles_max * (d / kM) * ns;
        MOE_CUDA_OK(moek::launch_pdl(tc_ffn_persist, dim3(static_cast<unsigned>(std::min(nt, sms))), dim3(kThreads2), kPSmem,
                                     stream, a, nt, ns, ypart, 1));
        if (ns == 1) return cudaSuccess;
        if (cmb != nullptr && !(dbg & 4194304)) {  // MOE_TC_DBG bit 22: split_reduce + combine instead
            *combined = true;
            const long long n = static_cast<long long>(T) * (d / 4);
            return moek::launch_pdl(combine_splits_kernel, dim3(static_cast<unsigned>((n + 255) / 256)), dim3(256), 0,
                                    stream, reinterpret_cast<const float4*>(ypart), static_cast<int>(slots), ns, cmb->inv,
                                    cmb->w, static_cast<const uint16_t*>(cmb->res), T, d, k,
                                    static_cast<uint16_t*>(cmb->out));
        }
        return moek::launch_pdl(split_reduce_kernel, dim3(static_cast<unsigned>(std::min<size_t>(slots, 2048))), dim3(256), 0,
                                stream, reinterpret_cast<const float4*>(ypart), offsets, E, active_mask,
                                static_cast<int>(slots), d / 4, ns, reinterpret_cast<float4*>(y));
    }
    if (persist) {
        const int nt0 = ntiles_max * (f / kM);
        MOE_CUDA_OK(moek::launch_pdl(tc_ffn_persist, dim3(static_cast<unsigned>(std::min(nt0, sms))), dim3(kThreads2), kPSmem,
                                     stream, a, nt0, 1, static_cast<float*>(nullptr), 0));
    } else {
        if (wpers) MOE_CUDA_OK(launch_wide(f));
        if (mask_single) {
            TcArgs as = a;
            as.active_mask = mask_single;
            MOE_CUDA_OK(moek::launch_pdl(kern, dim3(static_cast<unsigned>(ntiles_max * (f / kM))), dim3(kThreads2), smem,
                                         stream, as));
        }
    }
    // pass 1: down -> y
    a.p = 1;
    MOE_CUDA_OK(encode_b(&a.tmb, h, f, static_cast<int>(slots)));
    MOE_CUDA_OK(encode_b(&a.tmb16, h16, f, static_cast<int>(slots)));
    a.y = y;
    if (persist) {
        const int nt1 = ntiles_max * (d / kM) * ns;
        MOE_CUDA_OK(moek::launch_pdl(tc_ffn_persist, dim3(static_cast<unsigned>(std::min(nt1, sms))), dim3(kThreads2), kPSmem,
                                     stream, a, nt1, ns, ypart, 0));
        if (ns == 1) return cudaSuccess;
        return moek::launch_pdl(split_reduce_kernel, dim3(static_cast<unsigned>(std::min<size_t>(slots, 2048))), dim3(256), 0,
                                stream, reinterpret_cast<const float4*>(ypart), offsets, E, active_mask,
                                static_cast<int>(slots), d / 4, ns, reinterpret_cast<float4*>(y));
    }
    if (wpers) MOE_CUDA_OK(launch_wide(d));
    if (!mask_single) return cudaSuccess;
    TcArgs as = a;
    as.active_mask = mask_single;
    return moek::launch_pdl(kern, dim3(static_cast<unsigned>(ntiles_max * (d / kM))), dim3(kThreads2), smem, stream,
                            as);
}
}  // namespace

cudaError_t moek_ffn_tc(void* ws, const void* x, const int32_t* perm, const int32_t* offsets, int T, int k,
                        const moe_expert_weights* experts, int E, int d, int f, uint64_t active_mask, float* y,
                        cudaStream_t stream) {
    bool combined;
    return ffn_tc_impl(ws, x, perm, offsets, T, k, experts, E, d, f, active_mask, y, nullptr, &combined, stream);
}

cudaError_t moek_ffn_tc_combine(void* ws, const void* x, const int32_t* perm, const int32_t* offsets, int T, int k,
                                const moe_expert_weights* experts, int E, int d, int f, uint64_t active_mask,
                                float* y, const int32_t* inv, const float* w, const void* res, void* out,
                                cudaStream_t stream) {
    // every slot must come from this launch for the partials to hold the whole y
    const uint64_t all = E >= 64 ? ~0ull : ((1ull << E) - 1ull);
    const TcCombine cmb{inv, w, res, out};
    bool combined = false;
    MOE_CUDA_OK(ffn_tc_impl(ws, x, perm, offsets, T, k, experts, E, d, f, active_mask, y,
                            (active_mask & all) == all ? &cmb : nullptr, &combined, stream));
    if (combined) return cudaSuccess;
    return moek_combine(y, inv, w, res, T, d, k, out, stream);
}

MOE_NUMERICS_BINDER(tc)

// Loads this unit's kernels now (cudaFuncGetAttributes).  Under lazy module
// loading (CUDA 12 default) a kernel's first launch may wait for the device
// to idle; the expert-parallel step has kernels that spin on a peer's flags,
// so every kernel it can launch must be resident before the first step.
cudaError_t moek_preload_tc() {
    cudaFuncAttributes fa;
    MOE_CUDA_OK_PRELOAD(cudaFuncGetAttributes(&fa, moek::tc::tc_ffn_kernel<128>));
    MOE_CUDA_OK_PRELOAD(cudaFuncGetAttributes(&fa, moek::tc::tc_ffn_kernel<256>));
    MOE_CUDA_OK_PRELOAD(cudaFuncGetAttributes(&fa, moek::tc::tc_ffn_persist));
    MOE_CUDA_OK_PRELOAD(cudaFuncGetAttributes(&fa, moek::tc::split_reduce_kernel));
    MOE_CUDA_OK_PRELOAD(cudaFuncGetAttributes(&fa, moek::tc::combine_splits_kernel));
    MOE_CUDA_OK_PRELOAD(cudaFuncGetAttributes(&fa, moek::tc::tc_ffn_wide));
    MOE_CUDA_OK_PRELOAD(cudaFuncGetAttributes(&fa, moek::tc::tc_ffn_wide2));
    MOE_CUDA_OK_PRELOAD(cudaFuncGetAttributes(&fa, moek::tc::gather_rows_kernel));
    return cudaSuccess;
}
