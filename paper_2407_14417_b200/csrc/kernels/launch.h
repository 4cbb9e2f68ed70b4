// launch.h -- host-side launchers of the sm_100a kernels (internal).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "moe_b200.h"

cudaError_t moek_route(const void* x, const void* wg, int T, int d, int E, int k, int32_t* idx,
                       float* w, float* logits, int32_t* counts, int32_t* offsets, int32_t* perm,
                       int32_t* inv_perm, unsigned int* ticket, cudaStream_t stream);
cudaError_t moek_permute(const int32_t* idx, int T, int E, int k, int32_t* counts, int32_t* offsets,
                         int32_t* perm, int32_t* inv_perm, cudaStream_t stream);
// Workspace of the tensor-core GEMV FFN (must be zeroed once; the kernels
// leave the arrival counters at zero).
struct GemvWorkspace {
    void* xperm;              // [T][d] bf16, K-permuted
    float* xsum;              // [T][d/128] activation group sums
    void* hperm;              // [T*k][f] bf16, K-permuted
    float* hsum16;            // [T*k][f/16]
    float* hsum;              // [T*k][f/128]
    float* part;              // zeroed partial run sums
    unsigned int* counters;   // zeroed arrival counters
    unsigned int* gcounters;  // zeroed per-(segment, h group) counters
};
// One zero-filled allocation of moek_gemv_workspace_bytes, carved by _view.
size_t moek_gemv_workspace_bytes(int T, int k, int d, int f);
GemvWorkspace moek_gemv_workspace_view(void* base, int T, int k, int d, int f);
cudaError_t moek_permute_rows(const void* x, int rows, int K, void* xperm, float* xsum,
                              cudaStream_t stream);
// Expert FFN of every active expert segment (bit e of active_mask): gate/up
// GEMV + fused SwiGLU, down GEMV + fused combine (out != null: out[t] =
// bf16(resid[t] + sum_j w[t,j] y[inv[t*k+j]])) or per-slot y (out == null).
cudaError_t moek_ffn_mma(const GemvWorkspace& ws, const void* x, const int32_t* perm,
                         const int32_t* offsets, const int32_t* inv, const float* wts,
                         const void* resid, int T, int k, const moe_expert_weights* experts, int E,
                         int d, int f, uint64_t active_mask, void* out, float* y, bool xperm_ready,
                         cudaStream_t stream);
// Storage-layout converters (logical row-major -> fragment blocks).
cudaError_t moek_pack_bf16_blocks(const void* w, int rows, int cols, void* out, cudaStream_t stream);
cudaError_t moek_quantize_blocks(const void* w, int rows, int cols, uint32_t* qb, void* sb,
                                 cudaStream_t stream);
cudaError_t moek_combine(const float* y, const int32_t* inv, const float* w, const void* res, int T,
                         int d, int k, void* out, cudaStream_t stream);
cudaError_t moek_quantize(const void* w, int rows, int cols, uint32_t* q, void* s, cudaStream_t stream);
cudaError_t moek_synth_weight(uint64_t seed, uint64_t uid, long long n, int shift, void* out,
                              cudaStream_t stream);
cudaError_t moek_synth_input(uint64_t seed, uint64_t uid, long long n, void* out, cudaStream_t stream);
int moek_weight_shift(int K);
// Debug: per-warp phase trace buffer for the GEMV kernels (null disables);
// [2 passes][148*warps][8] u64.
cudaError_t moek_debug_gemv_trace(void* buf);
