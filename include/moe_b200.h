/*
 * moe_b200.h -- C ABI of the B200 MoE expert-layer hot path.
 *
 * This is the drop-in boundary under the reference's operator API
 * (/root/reference/proj/include/moeserve):
 *   router call           generate_trace   gating.hpp:33      -> moe_gate_topk (+ moe_generate_trace)
 *   placement config      make_plan        planner.hpp:71     -> moe_make_plan
 *   MoE-layer forward     simulate         simulator.hpp:58   -> moe_engine_* / moe_ffn / moe_combine
 *                                                                (+ moe_simulate for the cost model)
 * The reference has no FFI of its own (C++ headers only);
 * INTEGRATION.md shows the ctypes / C++ binding a maintainer would add.
 *
 * Conventions
 *   - plain pointers and sizes only; device pointers are caller-owned and the
 *     kernels are stream-ordered (cudaStream_t passed as void*); nothing in
 *     the kernel entry points allocates.
 *   - every entry point returns a status mirroring the reference CLI exit
 *     codes (cli.hpp:7-8): 0 ok, 1 internal (CUDA) error, 2 usage (bad
 *     shape / argument), 3 parse or validation error, 4 infeasible budget.
 *     moe_last_error() returns the thread's last message.
 *   - bf16 tensors are passed as void* (uint16 storage), int4-g128 weights
 *     as packed uint32 + bf16 scales (format in DESIGN.md, "int4 format").
 *   - no CPU fallback: without a CUDA device the kernel entry points return 1.
 */
#ifndef MOE_B200_H
#define MOE_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define MOE_MAX_EXPERTS 64
#define MOE_MAX_TOPK 8

enum { MOE_OK = 0, MOE_ERR_INTERNAL = 1, MOE_ERR_USAGE = 2, MOE_ERR_VALIDATION = 3,
       MOE_ERR_INFEASIBLE = 4 };
enum { MOE_P4 = 0, MOE_P16 = 1 };          /* Precision (profiles.hpp:17)   */
enum { MOE_GPU = 0, MOE_CPU = 1 };         /* Location  (planner.hpp:13)    */
enum { MOE_THROUGHPUT = 0, MOE_QUALITY = 1 };

const char* moe_last_error(void);
int moe_version(void);

/* ------------------------------------------------------------------------
 * Profiles and placement config (reference profiles.hpp / planner.hpp).
 * ---------------------------------------------------------------------- */
typedef struct {                 /* ModelProfile, profiles.hpp:29-43 */
    int32_t num_layers, experts_per_layer, top_k, pad_;
    int64_t size_nonexpert_bytes, size_expert16_bytes;
    double quant_ratio, compute_latency16_s, compute_penalty4, nonexpert_latency_s;
} moe_model_profile;

typedef struct {                 /* HardwareProfile, profiles.hpp:45-52 */
    int64_t gpu_mem_bytes;
    double transfer_bw_bytes_per_s;
} moe_hardware_profile;

typedef struct {                 /* TaskRequest, profiles.hpp:55-59 (n4_target -1 = none) */
    int32_t preference, n4_target;
    uint64_t seed;
} moe_task_request;

typedef struct {                 /* ExpertState, planner.hpp:22-26 */
    int32_t precision, location;
} moe_expert_state;

/* which: 0 mixtral-sec41, 1 mixtral-table1 (profiles.cpp:66-75) */
int moe_profile_builtin(int which, moe_model_profile* out);
/* Profile whose expert sizes equal the engine's allocations for d x f experts. */
int moe_profile_for_shape(int d_model, int d_ffn, int num_layers, int experts_per_layer, int top_k,
                          int64_t size_nonexpert_bytes, moe_model_profile* out);
int moe_load_profiles(const char* document, moe_model_profile* model, moe_hardware_profile* hw);
int64_t moe_parse_size(const char* text);                              /* -1 on error */
int64_t moe_expert_size(const moe_model_profile* p, int precision);
int moe_model_size(const moe_model_profile* p, int n4, int nonexpert_precision /*0 P4,1 P8,2 P16*/,
                   int64_t* out);
uint64_t moe_profile_fingerprint(const moe_model_profile* p);
int moe_num_experts_16(int64_t mem_gpu, const moe_model_profile* p);    /* Eq. 1 */
/* make_plan (planner.hpp:71): entries[num_experts] indexed layer*E + slot. */
int moe_make_plan(const moe_task_request* task, const moe_hardware_profile* hw,
                  const moe_model_profile* p, moe_expert_state* entries, int64_t* swap_slot_bytes);
int moe_assign_locations(const int32_t* precisions, const moe_hardware_profile* hw,
                         const moe_model_profile* p, uint64_t seed, moe_expert_state* entries,
                         int64_t* swap_slot_bytes);
int64_t moe_gpu_footprint(const moe_expert_state* entries, int64_t swap_slot_bytes,
                          const moe_model_profile* p);
/* Number of validate_plan() violations (0 = valid); messages joined by '\n'
 * into msg (capacity cap) when msg != NULL. */
int moe_validate_plan(const moe_expert_state* entries, int n_entries, int64_t swap_slot_bytes,
                      const moe_hardware_profile* hw, const moe_model_profile* p, char* msg,
                      int cap);
/* Plan artifact, `moeserve.plan.v1` JSON (serialize.hpp:18-19 write_plan /
 * read_plan).  write: returns the length (required length when cap is too
 * small; the text is copied only when it fits), -1 on error.  read: ParseError
 * (format marker, row shape, precision / location words) and ValidationError
 * (fingerprint, duplicate / missing / out-of-range expert) both return
 * MOE_ERR_VALIDATION, as in the CLI; moe_last_error() tells them apart.
 * entries holds L*E rows. */
int64_t moe_write_plan(const moe_expert_state* entries, int64_t swap_slot_bytes, uint64_t seed,
                       const moe_model_profile* p, char* buf, int64_t cap);
int moe_read_plan(const char* document, const moe_model_profile* p, moe_expert_state* entries,
                  int64_t* swap_slot_bytes, uint64_t* seed);

/* ------------------------------------------------------------------------
 * Routing records (gating.hpp) and the reference cost model (simulator.hpp).
 * ---------------------------------------------------------------------- */
/* Uniform stand-in router; slots[(t*L + l)*k + i], ascending per record. */
int moe_generate_trace(const moe_model_profile* p, int tokens, uint64_t seed, int32_t* slots,
                       uint64_t* fingerprint);
/* v1 text; returns length (required length when cap too small), -1 on error */
int64_t moe_write_trace(const moe_model_profile* p, int tokens, const int32_t* slots, char* buf,
                        int64_t cap);
int moe_read_trace(const char* document, int32_t dims[4] /*tokens,L,E,k*/, uint64_t* fingerprint,
                   int32_t* slots, int64_t slots_cap);

typedef struct {                 /* SimReport, simulator.hpp:33-53 */
    int64_t tokens, activations, hits, bytes_transferred, transfer_ns, compute_ns, nonexpert_ns;
} moe_sim_report;

/* lru_capacity 0 = Static policy */
int moe_simulate(const moe_expert_state* entries, int64_t swap_slot_bytes, const int32_t* slots,
                 int tokens, const moe_model_profile* p, const moe_hardware_profile* hw,
                 int lru_capacity, moe_sim_report* out);
double moe_expected_throughput(const moe_expert_state* entries, const moe_model_profile* p,
                               const moe_hardware_profile* hw);

/* Reconfiguration (reconfig.hpp:12-58): kinds 0 Offload, 1 Fetch, 2 Quantize,
 * 3 Dequantize; each action records the expert's entry in the target plan. */
typedef struct {
    int32_t kind, layer, slot, target_precision, target_location, pad_;
} moe_reconfig_action;
/* diff_plans (reconfig.cpp:19-55): writes min(n, cap) actions, *n_actions = n. */
int moe_diff_plans(const moe_expert_state* from, const moe_expert_state* to, uint64_t to_seed,
                   const moe_model_profile* p, const moe_hardware_profile* hw, moe_reconfig_action* actions,
                   int cap, int* n_actions, int64_t* bytes_moved, double* est_downtime_s);
/* apply (reconfig.cpp:84-168): checked replay; budget may be NULL. */
int moe_apply_reconfig(const moe_expert_state* plan, uint64_t plan_seed, const moe_reconfig_action* actions,
                       int n_actions, uint64_t target_seed, const moe_model_profile* p,
                       const moe_hardware_profile* budget, moe_expert_state* out, int64_t* out_swap,
                       uint64_t* out_seed);

/* moeserve.reconfig.v1 (serialize.cpp:160-206).  write: bytes_moved and
 * est_downtime_s are recomputed from the actions at hw (estimate_cost); returns
 * the length (see moe_write_plan).  read: as the reference (format ->
 * ParseError, fingerprint / bounds / stored bytes_moved -> ValidationError). */
int64_t moe_write_reconfig(const moe_reconfig_action* actions, int n_actions, uint64_t target_seed,
                           const moe_model_profile* p, const moe_hardware_profile* hw, char* buf, int64_t cap);
int moe_read_reconfig(const char* document, const moe_model_profile* p, const moe_hardware_profile* hw,
                      moe_reconfig_action* actions, int cap, int* n_actions, uint64_t* target_seed,
                      int64_t* bytes_moved, double* est_downtime_s);
/* SimReport as the reference's one-row CSV / JSON (serialize.cpp:218-243). */
int64_t moe_report_text(const moe_sim_report* r, int json, char* buf, int64_t cap);

/* Quality / memory / throughput sweep (pareto.hpp, cli.cpp:243-342).
 * Anchors: builtin name "wikitext2" | "ptb" | "c4" (Table 2), or an
 * INI document's [quality] section over a fallback (pareto.cpp:35-54). */
int moe_builtin_anchors(const char* name, double* ppl_all16, double* ppl_all4);
int moe_load_anchors(const char* document, double* ppl_all16, double* ppl_all4); /* in: fallback, out: result */
int moe_ppl_estimate(int n4, double ppl_all16, double ppl_all4, int num_e, double* out);
int moe_n4_for_budget(double ppl_budget, double ppl_all16, double ppl_all4, int num_e, int32_t* out);

typedef struct {                 /* ParetoRow, cli.cpp:243-251 */
    int64_t budget;
    int32_t n4, feasible, on_frontier, n_gpu;
    int64_t gpu_bytes;
    double ppl;
    moe_sim_report report;
} moe_pareto_row;
/* rows[g*n_budgets + b] for n4_grid[g] x budgets[b], frontier flags set. */
int moe_pareto_sweep(const int64_t* budgets, int n_budgets, const int32_t* n4_grid, int n_grid,
                     const moe_model_profile* p, const moe_hardware_profile* hw, int tokens, uint64_t seed,
                     double ppl_all16, double ppl_all4, moe_pareto_row* rows);
/* Frontier flags of arbitrary points (pareto.hpp:47-50). */
int moe_frontier_mask(int n, const double* throughput_tps, const double* ppl, const int64_t* gpu_bytes,
                      int32_t* on_frontier);
/* The sweep table; measured = NULL gives the reference schema exactly,
 * else 2 doubles per row (tok/s, hit rate; NaN = not measured) append
 * measured_tps,measured_hit_rate.  Returns the length (see moe_write_plan). */
int64_t moe_pareto_csv(const moe_pareto_row* rows, int n, const double* measured, char* buf, int64_t cap);

/* ------------------------------------------------------------------------
 * Kernels (sm_100a).  Stream-ordered; all pointers are device pointers.
 * ---------------------------------------------------------------------- */

/* K1: logits = x . wg^T in fp32 (pinned reduction order), top-k
 * on logits (ties -> lower index, output in descending logit order), weights
 * = softmax over the selected logits.  x [T,d] bf16, wg [E,d] bf16 ->
 * idx [T,k] int32, w [T,k] fp32, logits [T,E] fp32 (optional). */
int moe_gate_topk(const void* x, const void* wg, int T, int d, int E, int k, int32_t* idx,
                  float* w, float* logits, void* stream);

/* K1+K2 fused (the engine's route kernel): optional unit-weight RMSNorm
 * (norm_eps > 0, pinned order = oracle orc_rmsnorm) of x, the router and,
 * when counts != NULL, the stable permutation (offsets [E+1], perm, inv_perm;
 * `ticket` = 4 zeroed bytes, left zeroed).  xnat (optional) receives the
 * normalised rows [T,d] in natural order (the expert FFN input). */
int moe_route(const void* x, const void* wg, int T, int d, int E, int k, float norm_eps, int32_t* idx, float* w,
              float* logits, int32_t* counts, int32_t* offsets, int32_t* perm, int32_t* inv_perm, void* xnat,
              uint32_t* ticket, void* stream);

/* K2: stable expert-major counting sort of the T*k (token, j) pairs.
 * counts [E], offsets [E+1], perm [T*k] (perm[pos] = t*k + j),
 * inv_perm [T*k] (inv_perm[t*k + j] = pos).  Bit-exact, no atomics. */
int moe_permute(const int32_t* idx, int T, int E, int k, int32_t* counts, int32_t* offsets,
                int32_t* perm, int32_t* inv_perm, void* stream);

/* Weights of one expert as the kernels see them: every matrix [R rows, K]
 * in the fragment-block layout (16 rows x 128 K per block, DESIGN.md "HBM
 * layout"; produced by moe_pack_bf16_blocks / moe_quantize_g128). */
typedef struct {
    int32_t precision;        /* MOE_P4 (int4-g128) or MOE_P16 (bf16)                       */
    int32_t pad_;
    const void* w_gate_up;    /* [2f, d]: rows [0,f) gate, [f,2f) up; P16 bf16 blocks, P4 int4 blocks */
    const void* s_gate_up;    /* P4: bf16 scale blocks; P16: NULL                           */
    const void* w_down;       /* [d, f] blocks                                              */
    const void* s_down;       /* P4: bf16 scale blocks                                      */
} moe_expert_weights;

/* K3/K4: grouped SwiGLU FFN of every expert segment of a permutation, on the
 * streaming GEMV (experts whose w_gate_up is NULL -- another rank's shard --
 * are skipped and their y_perm rows left untouched), on the
 * tensor-core GEMV (<= 8 tokens per expert share each weight byte; larger
 * segments are tiled).  x [T,d] bf16 (natural order), offsets [E+1] (device),
 * experts[E] (host array of device pointers), y_perm [T*k, d] fp32.
 * Mixed precision per expert.  `workspace` (moe_ffn_workspace_bytes) must be
 * zero-filled before its first use; calls leave it reusable. */
size_t moe_ffn_workspace_bytes(int T, int k, int E, int d, int f);
int moe_ffn(const void* x, const int32_t* perm, const int32_t* offsets, int T, int k,
            const moe_expert_weights* experts, int E, int d, int f, void* workspace,
            size_t ws_bytes, float* y_perm, void* stream);
/* Survey-named single-precision wrappers of moe_ffn (all experts one format). */
int moe_ffn_int4(const void* x, const int32_t* perm, const int32_t* offsets, int T, int k,
                 const void* const* q_gate_up, const void* const* s_gate_up,
                 const void* const* q_down, const void* const* s_down, int E, int d, int f,
                 void* workspace, size_t ws_bytes, float* y_perm, void* stream);
int moe_ffn_bf16(const void* x, const int32_t* perm, const int32_t* offsets, int T, int k,
                 const void* const* w_gate_up, const void* const* w_down, int E, int d, int f,
                 void* workspace, size_t ws_bytes, float* y_perm, void* stream);
/* Largest T moe_ffn takes for E experts, top-k: its segment table holds
 * min(E, T*k) + ceil(T*k/8) <= 64 (active expert, 8-token tile) segments.
 * Larger batches belong on moe_ffn_tc. */
int moe_gemv_max_tokens(int E, int k);

/* fp16-operand range guard of the int4 paths (kernels/common.cuh).  Bit 0:
 * a bf16 activation (x or h) above 65504 was copied to fp16 (inf); bit 1: a
 * tcgen05 int4 dequantisation met a scale outside [2^-14, 8188] (q*s not
 * exact).  Process-wide, sticky until read with clear != 0.  MoeEngine
 * raises ValidationError (status 3) on it at sync for plans with int4
 * experts.  No reference counterpart (the reference has no tensor math). */
#define MOE_NUMERICS_F16_ACTIVATION 1u
#define MOE_NUMERICS_F16_SCALE 2u
int moe_numerics_status(int clear, uint32_t* flags);

/* K3/K4 on the 5th-generation tensor cores (tcgen05.mma, TMEM accumulators)
 * for batched decode / prefill: the same contract as moe_ffn (x [T,d] bf16
 * natural order, y_perm [T*k, d] fp32), 128-row x 128-token tiles per
 * expert, SwiGLU fused into the gate/up epilogue.  bf16 experts run BF16
 * operands; int4-g128 experts are dequantised on chip to fp16 q*s (exact
 * for normal-range scales) against an fp16 copy of the activations.
 * `workspace` needs moe_ffn_tc_workspace_bytes (no zero-fill needed). */
size_t moe_ffn_tc_workspace_bytes(int T, int k, int d, int f);
int moe_ffn_tc(const void* x, const int32_t* perm, const int32_t* offsets, int T, int k,
               const moe_expert_weights* experts, int E, int d, int f, void* workspace, size_t ws_bytes,
               float* y_perm, void* stream);

/* K5: out[t] = bf16(residual[t] + sum_j w[t,j] * y_perm[inv_perm[t*k+j]]),
 * fp32 fma chain in j order; residual may be NULL. */
int moe_combine(const float* y_perm, const int32_t* inv_perm, const float* w,
                const void* residual, int T, int d, int k, void* out, void* stream);

/* Expert-parallel combine: this rank's share of every
 * token's output, out[t] = sum over j with bit idx[t,j] of expert_mask of
 * w[t,j] * y_perm[inv_perm[t*k+j]] (fp32, j order).  The shares of all ranks
 * are summed by a reduce-scatter; moe_residual_add then forms
 * out = bf16(residual + sum). */
int moe_combine_partial(const float* y_perm, const int32_t* inv_perm, const float* w, const int32_t* idx,
                        uint64_t expert_mask, int T, int d, int k, float* out, void* stream);
int moe_residual_add(const void* residual, const float* part, int64_t n, void* out, void* stream);

/* int4-g128 quantiser: logical row-major bf16 [rows,cols] -> int4 fragment
 * blocks q (rows*cols/8 uint32) + scale blocks s (rows*cols/128 bf16); the
 * on-device "Quantize" action of the reconfiguration model (reconfig.hpp:12). */
int moe_quantize_g128(const void* w, int rows, int cols, uint32_t* q, void* s, void* stream);
/* logical row-major bf16 [rows,cols] -> bf16 fragment blocks */
int moe_pack_bf16_blocks(const void* w, int rows, int cols, void* out, void* stream);

/* Deterministic synthetic tensors (same generator as the oracle). */
int moe_synth_weight_bf16(uint64_t seed, uint64_t uid, int64_t n, int shift, void* out,
                          void* stream);
int moe_synth_input_bf16(uint64_t seed, uint64_t uid, int64_t n, void* out, void* stream);
int moe_weight_shift(int K);

/* Host-resident expert streaming: pinned H2D on a side stream, recorded on
 * `done_event` (cudaEvent_t as void*), which the compute stream waits on. */
int moe_stream_expert(void* dst_dev, const void* src_pinned, size_t bytes, void* copy_stream,
                      void* done_event);

/* ------------------------------------------------------------------------
 * Engine: one MoE layer stack on one device, owning weights laid out per a
 * placement plan (device-resident experts in HBM, host-resident experts in a
 * pinned arena streamed into the swap slot on a side stream, Static policy).
 * ---------------------------------------------------------------------- */
typedef struct moe_engine moe_engine;

typedef struct {
    int32_t num_layers, experts_per_layer, top_k, d_model, d_ffn;
    int32_t max_tokens;        /* largest decode batch T the engine is sized for */
    uint64_t seed;             /* synthetic weight seed                          */
    int32_t device;
    int32_t use_graphs;        /* capture decode steps in CUDA graphs            */
    float norm_eps;            /* > 0: Mixtral decoder-layer RMSNorm (unit weight) before every MoE
                                  block, out = x + MoE(RMSNorm(x)); 0: out = x + MoE(x) */
    int32_t tc_min_tokens;     /* decode batches T >= this use the tcgen05 expert GEMM, smaller ones
                                  the streaming GEMV (0: default 32, the measured crossover) */
    int32_t lru_capacity;      /* host-resident experts: 0 = Static (every activation re-streams into
                                  the single swap slot, simulator.cpp:98-106); C >= top_k = LRU cache of
                                  C device slots (simulator.cpp:37-62, the Mixtral-Offloading baseline) */
    int32_t keep_masters;      /* 1: pinned host copy of every expert in both precisions (the reconfig
                                  model's 16-bit CPU master, reconfig.hpp:39); needed by
                                  moe_engine_reconfigure */
    int32_t per_layer_decode;  /* 0 (default): a batch-1 decode step of an all-resident plan is ONE
                                  cooperative persistent launch (routing, both GEMV passes, SwiGLU and
                                  combine of every layer, grid barriers between phases); 1: five launches
                                  per layer (the same arithmetic, bit-identical output) */
    int32_t ep_rank, ep_world; /* expert parallelism: ep_world > 1 shards every layer's
                                  experts over ep_world engines (slot s on rank s*ep_world/E); this one
                                  holds only its own.  decode() then sends each routed token row to its
                                  expert's owner and gets the output back over peer memory (NVLink P2P /
                                  CUDA IPC; moe_engine_ep_buffer / moe_engine_ep_set_peers).  0/1: off */
} moe_engine_config;

int moe_engine_create(const moe_engine_config* cfg, const moe_expert_state* plan_entries,
                      moe_engine** out);
void moe_engine_destroy(moe_engine* eng);
/* Bytes of device memory held for experts / swap / workspaces. */
int moe_engine_memory(const moe_engine* eng, int64_t* expert_bytes, int64_t* swap_bytes,
                      int64_t* host_pinned_bytes, int64_t* workspace_bytes);
/* Device pointer to the layer input buffer [max_tokens, d] bf16. */
void* moe_engine_input(moe_engine* eng);
void* moe_engine_output(moe_engine* eng);
/* Fill the input buffer with the synthetic embedding of decode step `step`. */
int moe_engine_synth_input(moe_engine* eng, int step, int T);
/* One decode step of T tokens through all layers, input -> output, on the
 * engine's compute stream (async).  Routing of every layer is kept for
 * export. */
int moe_engine_decode(moe_engine* eng, int T);
/* Same, with host buffers: H2D of x_host, decode, D2H into out_host, synced. */
int moe_engine_decode_host(moe_engine* eng, const void* x_host, int T, void* out_host);
/* One layer: x (device [T,d]) -> out (device), routing outputs optional. */
int moe_engine_forward_layer(moe_engine* eng, int layer, const void* x, int T, void* out,
                             int32_t* idx_dev, float* w_dev, float* logits_dev);
int moe_engine_sync(moe_engine* eng);
/* Eager decode step with CUDA events around each layer's expert-FFN launches
 * (compute stream): ffn_ms[num_layers], algorithmic ffn_bytes[num_layers]
 * (selected experts' weights + activations), kernels launched per step. */
int moe_engine_profile_step(moe_engine* eng, int T, float* ffn_ms, int64_t* ffn_bytes,
                            int32_t* kernels_per_step);
/* The fused batch-1 step timed alone (one launch between CUDA events on the
 * engine stream): *ms its duration, *bytes the algorithmic bytes it moves
 * (every layer's distinct selected experts + activations).  Status 2 when
 * the engine does not use the fused step. */
int moe_engine_profile_fused(moe_engine* eng, float* ms, int64_t* bytes);
void* moe_engine_stream(moe_engine* eng);
/* Routing of the last decode step: slots [T, L, k] ascending per record
 * (GatingTrace layout, gating.hpp:22) -- host buffer. */
int moe_engine_last_routing(moe_engine* eng, int T, int32_t* slots_out);
/* Expert parallelism: this rank's exchange buffer -- its own cudaMalloc
 * allocation, to be shared with moe_ep_peer_ipc_handle -- and the G ranks'
 * buffer bases in rank order (its own at ep_rank) before the first decode.
 * Replaces nothing in the reference (single GPU): the north
 * star's EP over NVLink, with the exchange inside the engine's step. */
int moe_engine_ep_buffer(moe_engine* eng, void** base, int64_t* bytes);
int moe_engine_ep_set_peers(moe_engine* eng, const void* const* bases, int32_t world);
/* Cumulative SimReport counters of real runs (hits / bytes_transferred /
 * activations follow simulate() semantics for the engine's plan). */
int moe_engine_counters(const moe_engine* eng, moe_sim_report* out);

/* ------------------------------------------------------------------------
 * Expert-parallel exchange: NCCL over NVLink, loaded at
 * run time.  Per layer: moe_ep_dispatch all-gathers every rank's token rows
 * (bf16) into x_all[world*T_local][d]; the ranks route all rows and run their
 * own experts (moe_ffn / moe_ffn_tc with the other shards NULL), form their
 * shares (moe_combine_partial); moe_ep_combine reduce-scatters the fp32
 * shares so each rank gets the sum for its T_local tokens, then
 * moe_residual_add.  Errors: moe_ep_last_error().
 * ---------------------------------------------------------------------- */
#define MOE_EP_ID_BYTES 128
typedef struct moe_ep_comm moe_ep_comm;
const char* moe_ep_last_error(void);
int moe_ep_unique_id(char id[MOE_EP_ID_BYTES]);                       /* ncclGetUniqueId, on one rank */
int moe_ep_comm_init(const char id[MOE_EP_ID_BYTES], int world, int rank, int device, moe_ep_comm** out);
int moe_ep_comm_wrap(void* nccl_comm, int world, int rank, moe_ep_comm** out);  /* an existing ncclComm_t */
void moe_ep_comm_destroy(moe_ep_comm* comm);
int moe_ep_dispatch(moe_ep_comm* comm, const void* x_local, int T_local, int d, void* x_all, void* stream);
int moe_ep_combine(moe_ep_comm* comm, const float* part, int T_local, int d, float* mine, void* stream);

/* The same exchange fused into the kernels that produce it, over peer memory
 * (NVLink P2P / CUDA IPC) instead of collectives.  Each rank owns one zeroed
 * device buffer of moe_ep_peer_bytes and knows the G ranks' buffers (`bases`,
 * its own included; IPC handles via moe_ep_peer_ipc_*).  Per layer, epoch + 1:
 *   moe_ep_push_rows    own rows -> every peer's gather slot `rank`, release flag
 *   moe_ep_wait_rows    until every rank's rows arrived; gathered rows at
 *                       moe_ep_peer_rows(base) [G*T_local][d]
 *   (route + own experts on the gathered rows)
 *   moe_ep_push_shares  moe_combine_partial's share written straight into
 *                       each owner's receive slot `rank`, release flag
 *   moe_ep_reduce       out = bf16(x + sum over src in order) once all arrived */
size_t moe_ep_peer_bytes(int G, int T_local, int d);
/* A zeroed exchange buffer of its own cudaMalloc allocation (an IPC handle
 * maps whole allocations, so the buffer must start one). */
int moe_ep_peer_alloc(size_t bytes, void** base);
int moe_ep_peer_free(void* base);
void* moe_ep_peer_rows(void* base);
int moe_ep_peer_ipc_handle(const void* base, char handle[64]);
int moe_ep_peer_ipc_open(const char handle[64], void** peer_base);
int moe_ep_peer_ipc_close(void* peer_base);
int moe_ep_push_rows(const void* x_local, int T_local, int d, int rank, int G, const void* const* bases,
                     uint32_t epoch, void* stream);
int moe_ep_wait_rows(const void* my_base, int G, int T_local, int d, uint32_t epoch, void* stream);
int moe_ep_push_shares(const float* y_perm, const int32_t* inv_perm, const float* w, const int32_t* idx,
                       uint64_t expert_mask, int T_local, int d, int k, int rank, int G, const void* const* bases,
                       uint32_t epoch, void* stream);
int moe_ep_reduce(const void* x_local, int T_local, int d, int rank, int G, const void* const* bases,
                  uint32_t epoch, void* out, void* stream);
/* Execute diff_plans(current, target) on the device (needs keep_masters):
 * Offload releases HBM, Fetch / in-place Dequantize copy host copies in,
 * Quantize of a device-resident expert runs the int4-g128 quantiser on the
 * device.  transfer_bw prices the model's est_downtime_s. */
typedef struct {
    int32_t actions, pad_;
    int64_t bytes_moved;       /* model (estimate_cost)            */
    double est_downtime_s;     /* model: bytes_moved / transfer_bw */
    int64_t bytes_h2d;         /* measured bytes copied to the GPU */
    double measured_s;         /* measured wall time (events)      */
} moe_reconfig_report;
int moe_engine_reconfigure(moe_engine* eng, const moe_expert_state* target, uint64_t target_seed,
                           double transfer_bw_bytes_per_s, moe_reconfig_report* out);
int moe_engine_reset_counters(moe_engine* eng);
/* Per-expert device weight view (for tests); host-resident experts report
 * their pinned host pointers with location MOE_CPU. */
int moe_engine_expert(const moe_engine* eng, int layer, int slot, moe_expert_weights* out,
                      int32_t* location);
int moe_engine_router(const moe_engine* eng, int layer, const void** wg_dev);

/* Debug: device buffer receiving per-warp phase timestamps of the GEMV
 * kernels ([2 passes][148*12 warps][8] uint64: entry, after PDL wait, first
 * item ready, end, items, runs, epilogues, CTA); NULL disables. */
int moe_debug_gemv_trace(void* buf);
/* Debug: per layer kernel (route, permute_rows, gate/up stream, SwiGLU
 * finalize, down stream, output finalize) the earliest entry / post-PDL-wait
 * and latest end globaltimer stamps: [6][3] uint64, entry/wait slots must be
 * pre-filled with UINT64_MAX and end slots with 0; NULL disables.  Set in
 * stream order on `stream`, so it can bracket exactly one graph replay. */
int moe_debug_layer_trace(void* buf, void* stream);
/* Debug: device buffer [num_layers][#SMs][10] uint64 receiving, per layer and
 * CTA of the fused batch-1 step, globaltimer stamps at: layer start, routing
 * done, gate/up done, after barrier 1, SwiGLU done, after barrier 2, h rows
 * resident, down done, after barrier 3, combine done; NULL disables. */
int moe_debug_fused_trace(void* buf);
/* Debug: device pointer and size of one of the engine's GEMV workspace
 * buffers (0 gate/up partials, 1 down partials, 2 h bf16, 3 h fp16, 4 h bias). */
int moe_debug_engine_buffer(moe_engine* eng, int which, void** ptr, size_t* bytes);

#ifdef __cplusplus
}
#endif
#endif /* MOE_B200_H */
