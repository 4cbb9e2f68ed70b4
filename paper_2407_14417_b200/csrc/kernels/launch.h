// launch.h -- host-side launchers of the sm_100a kernels (internal).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "moe_b200.h"

cudaError_t moek_route(const void* x, const void* wg, int T, int d, int E, int k, int32_t* idx,
                       float* w, float* logits, int32_t* counts, int32_t* offsets, int32_t* perm,
                       int32_t* inv_perm, unsigned int* ticket, cudaStream_t stream, void* xperm = nullptr,
                       void* xperm16 = nullptr, float* xsum = nullptr, int xstride = 0, float norm_eps = 0.0f,
                       void* xnat = nullptr);
cudaError_t moek_permute(const int32_t* idx, int T, int E, int k, int32_t* counts, int32_t* offsets,
                         int32_t* perm, int32_t* inv_perm, cudaStream_t stream);
// Workspace of the tensor-core GEMV FFN (must be zeroed once; the kernels
// leave the arrival counters at zero).
struct GemvWorkspace {
    void* xperm;              // [T][d] bf16, K-permuted
    void* xperm16;            // [T][d] fp16 copy (B operand of int4 experts)
    float* xsum;              // [T][*] int4 bias term per activation group
    void* hperm;              // [T*k][f] bf16, K-permuted
    void* hperm16;            // [T*k][f] fp16 copy
    float* hsum;              // [T*k][*] int4 bias term per h group
    float* part0;             // gate/up partials [d/128][T*k][2f]
    float* part1;             // down partials [f/128][T*k][d]
    int* kpslot;              // [2][T*k] K-parts per slot of the last stream launches
    unsigned int* sched;      // tail-pool counters (reset by the finalize kernels)
};
// One zero-filled allocation of moek_gemv_workspace_bytes, carved by _view.
size_t moek_gemv_workspace_bytes(int T, int k, int d, int f);
GemvWorkspace moek_gemv_workspace_view(void* base, int T, int k, int d, int f);
cudaError_t moek_permute_rows(const void* x, int rows, int K, void* xperm, void* xperm16, float* xsum,
                              cudaStream_t stream);
// Expert FFN of every active expert segment (bit e of active_mask): gate/up
// GEMV + fused SwiGLU, down GEMV + fused combine (out != null: out[t] =
// bf16(resid[t] + sum_j w[t,j] y[inv[t*k+j]])) or per-slot y (out == null).
// xmode: how the K-permuted activations (ws.xperm*) come to be:
//   MOE_X_PERMUTE  run the permute_rows kernel first (route two launches back)
//   MOE_X_ROUTED   written by the route kernel launched immediately before
//   MOE_X_READY    written earlier on the stream; launch without PDL (e.g.
//                  after an event wait for a streamed expert)
enum { MOE_X_PERMUTE = 0, MOE_X_ROUTED = 1, MOE_X_READY = 2 };
int moek_group_stride(int K);
// Largest decode batch the streaming GEMV takes for E experts, top-k (segment table bound).
int moek_gemv_max_tokens(int E, int k);
cudaError_t moek_ffn_mma(const GemvWorkspace& ws, const void* x, const int32_t* perm,
                         const int32_t* offsets, const int32_t* inv, const float* wts,
                         const void* resid, int T, int k, const moe_expert_weights* experts, int E,
                         int d, int f, uint64_t active_mask, void* out, float* y, int xmode,
                         cudaStream_t stream);
// Fused batch-1 decode step (gemv.cu decode_step_kernel): the whole L-layer
// stack -- routing, gate/up GEMV, SwiGLU, down GEMV, combine + residual per
// layer -- in one cooperative persistent launch with grid barriers between
// the phases.  All experts device-resident; output bit-identical to the
// per-layer kernels.  Buffers are the engine's; sched [L][2] and bar [2]
// must be zero before the first launch (the kernel leaves them so).
struct MoeDecodeArgs {
    int L, E, k, d, f;
    float norm_eps;
    const moe_expert_weights* experts;  // [L*E] device table
    const uint16_t* wg;                 // [L][E][d]
    const uint16_t* x_in;               // [d]
    uint16_t* xbuf0;
    uint16_t* xbuf1;
    uint16_t* xbuf2;                    // decode_flow_kernel: third layer-output row (0xffff-filled, see gemv.cu)
    uint16_t* x_out;
    int32_t* idx;                       // [L][idx_stride] routing export
    float* wts;
    int idx_stride;
    float* part0;                       // [d/128][k][2f]
    float* part1;                       // [f/128][k][d]
    uint16_t* hperm;                    // [k][f]
    uint16_t* hperm16;
    float* hsum;                        // [k][group_stride(f)]
    unsigned int* sched;                // [L][2]
    unsigned long long* bar;            // grid-barrier arrival counter (monotonic)
    int bar_mode;                       // 0: release fetch-add; 1: fence + relaxed add (A/B)
    unsigned int* flow_ctl;             // decode_flow_kernel: moek_decode_flow_ctl_words() zeroed words
    size_t part0_stride, part1_stride;  // decode_flow_kernel: floats between the two (layer-parity) partial buffers
};
bool moek_decode_step_supported(int E, int k, int d, int f);
size_t moek_decode_step_smem();
cudaError_t moek_decode_step(const MoeDecodeArgs& a, cudaStream_t stream);
// Dataflow variant (counters instead of grid barriers); sms = the grid.
bool moek_decode_flow_supported(int E, int k, int d, int f, int sms);
size_t moek_decode_flow_smem(int d, int f);
size_t moek_decode_flow_ctl_words(int L, int k, int d, int f);
cudaError_t moek_decode_flow(const MoeDecodeArgs& a, cudaStream_t stream);
// Debug: [L][grid][10] u64 globaltimer stamps of the fused step's phases; null disables.
cudaError_t moek_debug_fused_trace(void* buf);
// tcgen05 grouped expert FFN (tc_gemm.cu): x natural [T][d] bf16 (already
// normalised), every active expert's segment -> y_perm [T*k][d] fp32.
size_t moek_tc_workspace_bytes(int T, int k, int d, int f);
cudaError_t moek_ffn_tc(void* ws, const void* x, const int32_t* perm, const int32_t* offsets, int T, int k,
                        const moe_expert_weights* experts, int E, int d, int f, uint64_t active_mask, float* y,
                        cudaStream_t stream);
// moek_ffn_tc followed by the K5 combine (out = bf16(res + sum_j w_j y_j), moek_combine's
// arithmetic): when the down pass ran K-split in the fused persistent launch, the combine
// reads the split partials directly (no y round trip, no split_reduce launch); otherwise
// y is written and moek_combine runs.  Bit-identical to moek_ffn_tc + moek_combine.
cudaError_t moek_ffn_tc_combine(void* ws, const void* x, const int32_t* perm, const int32_t* offsets, int T, int k,
                                const moe_expert_weights* experts, int E, int d, int f, uint64_t active_mask,
                                float* y, const int32_t* inv, const float* w, const void* res, void* out,
                                cudaStream_t stream);
// Host-resident expert streaming (engine.cpp): pinned H2D of one expert on
// the copy stream, recorded on `done` (may be null) for the compute stream.
cudaError_t moek_stream_expert(void* dst, const void* src_pinned, size_t bytes, cudaStream_t copy, cudaEvent_t done);
// fp16-operand range guard (common.cuh): bind each kernel translation unit
// to the process-wide flag word (mapped pinned host memory) on the current device.
cudaError_t moek_numerics_bind_gemv(unsigned int* p);
cudaError_t moek_numerics_bind_router(unsigned int* p);
cudaError_t moek_numerics_bind_tc(unsigned int* p);
enum { MOE_NUM_F16_ACT_BIT = 1, MOE_NUM_F16_SCALE_BIT = 2 };  // = common.cuh MOE_NUM_F16_*
// Binds the current device (once per device; engine.cpp) and reads / clears the word.
cudaError_t moek_numerics_bind_device();
unsigned int moek_numerics_status(int clear);
// Storage-layout converters (logical row-major -> fragment blocks).
// fragment blocks -> logical row-major bf16 (inverse of moek_pack_bf16_blocks)
cudaError_t moek_unpack_bf16_blocks(const void* in, int rows, int cols, void* w, cudaStream_t stream);
cudaError_t moek_pack_bf16_blocks(const void* w, int rows, int cols, void* out, cudaStream_t stream);
cudaError_t moek_quantize_blocks(const void* w, int rows, int cols, uint32_t* qb, void* sb,
                                 cudaStream_t stream);
// Expert-parallel all-to-all of routed rows over peer memory (ep_a2a.cu).
size_t moek_ep_a2a_bytes(int G, int C, int d);
size_t moek_ep_a2a_offset(int G, int C, int d, int which);  // 0 rows, 1 meta, 2 ret, 3 flags
cudaError_t moek_ep_a2a_dispatch(const void* xn, const int32_t* idx, int T, int k, int E, int d, int C, int rank,
                                 int G, const void* const* bases, const uint32_t* epoch_base, int layer,
                                 cudaStream_t stream);
cudaError_t moek_ep_a2a_wait(const void* my_base, int which, int G, int C, int d, const uint32_t* epoch_base,
                             int layer, cudaStream_t stream);
cudaError_t moek_ep_a2a_keys(const int32_t* meta, int n, int E, int32_t* keys, cudaStream_t stream);
cudaError_t moek_ep_a2a_return(const float* y, const int32_t* perm, const int32_t* offsets, int E, int d, int C,
                               int rank, int G, const void* const* bases, const uint32_t* epoch_base, int layer,
                               cudaStream_t stream);
cudaError_t moek_ep_a2a_gather(const void* rows, const int32_t* perm, const int32_t* offsets, int E, int d,
                               int max_rows, void* dense, cudaStream_t stream);
cudaError_t moek_ep_a2a_bump(uint32_t* epoch_base, int L, cudaStream_t stream);
// every kernel resident before the first expert-parallel step (lazy loading)
cudaError_t moek_preload_gemv();
cudaError_t moek_preload_router();
cudaError_t moek_preload_misc();
cudaError_t moek_preload_tc();
cudaError_t moek_preload_ep();
cudaError_t moek_combine(const float* y, const int32_t* inv, const float* w, const void* res, int T,
                         int d, int k, void* out, cudaStream_t stream);
cudaError_t moek_quantize(const void* w, int rows, int cols, uint32_t* q, void* s, cudaStream_t stream);
cudaError_t moek_combine_partial(const float* y, const int32_t* inv, const float* w, const int32_t* idx,
                                 unsigned long long mask, int T, int d, int k, float* out, cudaStream_t stream);
cudaError_t moek_residual_add(const void* res, const float* part, long long n, void* out, cudaStream_t stream);
cudaError_t moek_synth_weight(uint64_t seed, uint64_t uid, long long n, int shift, void* out,
                              cudaStream_t stream);
cudaError_t moek_synth_input(uint64_t seed, uint64_t uid, long long n, void* out, cudaStream_t stream);
int moek_weight_shift(int K);
// Debug: per-warp phase trace buffer for the GEMV kernels (null disables);
// [2 passes][148*warps][8] u64.
cudaError_t moek_debug_gemv_trace(void* buf);
// Debug: [6 kernels][entry, after wait, end] u64 globaltimer (min/min/max); null disables.
cudaError_t moek_debug_layer_trace(void* buf, cudaStream_t stream);

// Expert-parallel exchange over peer memory (ep_peer.cu): `bases` are the G
// ranks' exchange buffers (moek_ep_peer_bytes each, zeroed once), this
// rank's own included; epoch increases by one per layer step.
size_t moek_ep_peer_bytes(int G, int T_local, int d);
cudaError_t moek_ep_push_rows(const void* x_local, int T_local, int d, int rank, int G, const void* const* bases,
                              uint32_t epoch, cudaStream_t stream);
cudaError_t moek_ep_wait_rows(const void* my_base, int G, int T_local, int d, uint32_t epoch, cudaStream_t stream);
cudaError_t moek_ep_push_shares(const float* y, const int32_t* inv, const float* w, const int32_t* idx,
                                uint64_t mask, int T_local, int d, int k, int rank, int G, const void* const* bases,
                                uint32_t epoch, cudaStream_t stream);
cudaError_t moek_ep_reduce(const void* x_local, int T_local, int d, int rank, int G, const void* const* bases,
                           uint32_t epoch, void* out, cudaStream_t stream);
