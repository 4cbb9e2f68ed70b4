/*
 * moe_oracle.h -- CPU restatement of the MoE expert-layer hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and the
 * cpu_baseline / --impl reference legs of bench.py may load this library, and
 * only as the checker.  The product (paper_2407_14417_b200/) never links it.
 *
 * The reference (/root/reference, "moeserve") contains no tensor arithmetic
 * (SPEC.md:3, :13): its MoE-layer forward is the cost loop of simulate()
 * (simulator.cpp:89-110) and its router is a uniform draw (gating.cpp:43-51).
 * The numeric semantics restated here therefore come from
 *   - HF transformers 5.5.0 MixtralSparseMoeBlock / MixtralTopKRouter
 *     (modeling_mixtral.py:62-136; router :109-116, experts :90-96), and
 *   - the north star's int4 group-128 format,
 * anchored on the reference's own data-plane contracts: expert index
 * l*E+s (planner.hpp:29, simulator.cpp:92-94), ascending-slot trace records
 * (gating.cpp:48), Static miss semantics (simulator.cpp:98-106).
 * Tensor numerics are therefore "parity unpinned" by any reference test; the
 * control plane (plans, traces, counters) is pinned against the reference
 * compiled from source (oracle/_ref, see oracle/Makefile).
 *
 * Every definition below is the contract the CUDA kernels must meet; see
 * DESIGN.md section "Numeric contract".
 */
#pragma once
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- synthetic tensors (counter-based, so any element is reproducible) ---- */
/* r(seed, uid, i) = mix64(mix64(seed ^ uid*0xD1B54A32D192ED03) + (i+1)*golden) */
uint64_t orc_rand64(uint64_t seed, uint64_t uid, uint64_t i);
/* bf16 weights w_i = (int8)(r >> 56) * 2^-p  (exactly representable) */
void orc_synth_weight_bf16(uint64_t seed, uint64_t uid, int64_t n, int p, uint16_t* out);
/* bf16 activations x_i = ((r >> 32) % 129 - 64) / 64 */
void orc_synth_input_bf16(uint64_t seed, uint64_t uid, int64_t n, uint16_t* out);
/* shift p for a K-long dot so that the weights have std ~ 1/sqrt(K) */
int orc_weight_shift(int K);

/* ---- int4 group-128 format ---- */
/* q packed 8 per uint32 along K, element j of a word at bit 4*(j/2)+16*(j%2),
 * stored biased (u = q + 8).  One bf16 scale per (row, 128-K group).
 * quantize: s = bf16(absmax/7) (1 if absmax == 0); q = clamp(rint(w/s), -8, 7)
 * dequant : w = q * s, exact in fp32 (and in fp16: <= 11 significant bits) */
void orc_quantize_g128(const uint16_t* w, int rows, int cols, uint32_t* q, uint16_t* s);
void orc_dequant_g128(const uint32_t* q, const uint16_t* s, int rows, int cols, float* w_out);

/* ---- device storage layout ("fragment blocks") ----
 * The engine stores every expert matrix [R rows, K cols] (R % 16 == 0,
 * K % 128 == 0) as blocks of 16 rows x 128 K, block (rt, g) at index
 * rt*(K/128) + g.  Inside a group, K position k is permuted to
 *   pi(k) = t*32 + kk*4 + hi*2 + e   (kk = k/16, t = (k%8)/2, hi = (k%16)/8, e = k%2)
 * so that lane (gr, t) of an mma.m16n8k16 finds its fragments contiguous.
 * Element (row, k) with rr = row%16, gr = rr%8, half = rr/8,
 * p = pi(k%128), r = p%32, lane = gr*4 + p/32:
 *   bf16 block (4096 B): byte ((r/4)*32 + lane)*16 + (((r/2)%2)*2 + half)*4 + (r%2)*2
 *                        (part kk = r/4 is lane's {a0,a1,a2,a3} of MMA kk: one LDS.128)
 *   int4 block (1024 B): word ((half*32 + lane)*4 + r/8), nibble (r%8) placed
 *                        at bit 4*(j/2)+16*(j%2) with j = r%8, biased u=q+8
 *   int4 scales (32 B per block): bf16 at byte gr*4 + half*2
 * Activations fed to the GEMV (x / h) use the same pi within each group. */
int orc_perm_k(int k);                                    /* pi(k % 128) + 128*(k/128) */
void orc_pack_bf16_blocks(const uint16_t* w, int rows, int cols, uint16_t* out);
void orc_unpack_bf16_blocks(const uint16_t* blk, int rows, int cols, uint16_t* out);
/* q/s in the row-major format above -> block format (and back) */
void orc_pack_int4_blocks(const uint32_t* q, const uint16_t* s, int rows, int cols,
                          uint32_t* qb, uint16_t* sb);
void orc_unpack_int4_blocks(const uint32_t* qb, const uint16_t* sb, int rows, int cols,
                            uint32_t* q, uint16_t* s);

/* ---- K1 router: fp32 logits in the pinned lane/butterfly order, top-k on
 *      logits (ties -> lower index), softmax over the selected logits ---- */
void orc_gate_topk(const uint16_t* x, const uint16_t* wg, int T, int d, int E, int k,
                   int32_t* idx, float* w, float* logits /* [T,E] or NULL */);

/* ---- K2 stable counting sort of the T*k (token, j) pairs by expert ---- */
void orc_permute(const int32_t* idx, int T, int E, int k, int32_t* counts, int32_t* offsets,
                 int32_t* perm, int32_t* inv_perm);

/* ---- K3/K4 SwiGLU expert FFN over M rows of x.  wgu rows [0,f) = gate,
 *      [f,2f) = up; wd is [d,f].  h is rounded to bf16 before the down proj.
 *      fp32 accumulation; y is fp32. ---- */
void orc_ffn_bf16(const uint16_t* x, int M, const uint16_t* wgu, const uint16_t* wd, int d, int f,
                  float* y);
void orc_ffn_int4(const uint16_t* x, int M, const uint32_t* qgu, const uint16_t* sgu,
                  const uint32_t* qd, const uint16_t* sd, int d, int f, float* y);

/* ---- K5 combine: out[t] = bf16(res[t] + sum_j w[t,j] * y[inv[t*k+j]]),
 *      fp32 fmaf chain in j order (res may be NULL) ---- */
void orc_combine(const float* y_perm, const int32_t* inv_perm, const float* w,
                 const uint16_t* residual, int T, int d, int k, uint16_t* out);

/* ---- whole-layer / stack drivers over synthetic weights ---- */
typedef struct {
    int num_layers, num_experts, top_k, d_model, d_ffn;
    uint64_t seed;
    float norm_eps;   /* > 0: decoder-layer pre-MoE RMSNorm (unit weight) before the router and the
                         experts, residual = the un-normalised x; 0: the bare MoE block */
    int pad_;
} orc_model;

/* RMSNorm with unit weight (HF MixtralRMSNorm, modeling_mixtral.py), pinned
 * order: partial[i] = fmaf chain over x[c*256+i]^2 (c ascending), then the
 * pairwise tree partial[i] += partial[i+s] for s = 128, 64, ..., 1;
 * rstd = 1 / sqrtf(partial[0] / d + eps) (IEEE); out = bf16(x * rstd). */
void orc_rmsnorm(const uint16_t* x, int T, int d, float eps, uint16_t* out);

/* Materialises expert e = layer*E + slot: bf16 masters, quantised when int4. */
void orc_expert_bf16(const orc_model* m, int e, uint16_t* wgu, uint16_t* wd);
void orc_expert_int4(const orc_model* m, int e, uint32_t* qgu, uint16_t* sgu, uint32_t* qd,
                     uint16_t* sd);
void orc_router_weights(const orc_model* m, int layer, uint16_t* wg);
void orc_step_input(const orc_model* m, int step, int T, uint16_t* x);

/* Prepared weights of one expert (precision 0 = int4-g128, 1 = bf16). */
typedef struct {
    int precision;
    const void* w_gate_up;
    const void* s_gate_up;
    const void* w_down;
    const void* s_down;
} orc_expert;

/* One MoE layer over prepared weights (router wg [E,d], experts[E]); this is
 * the CPU baseline's timed call -- no weight generation inside. */
void orc_moe_layer_w(const orc_model* m, const uint16_t* wg, const orc_expert* experts,
                     const uint16_t* x, int T, uint16_t* out, int32_t* idx, float* w,
                     float* logits);

/* One MoE layer: x[T,d] -> out[T,d]; precision[e] = 0 (P4) / 1 (P16) for the
 * layer's E experts.  idx/w/logits optional. */
void orc_moe_layer(const orc_model* m, int layer, const int* precision, const uint16_t* x, int T,
                   uint16_t* out, int32_t* idx, float* w, float* logits);

/* Number of OpenMP threads the oracle uses. */
int orc_num_threads(void);

#ifdef __cplusplus
}
#endif
