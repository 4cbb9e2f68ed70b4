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
// active_mask: bit e set -> expert e's segments are computed by this launch.
cudaError_t moek_ffn_gemv(const void* x, const int32_t* perm, const int32_t* offsets, int T, int k,
                          const moe_expert_weights* experts, int E, int d, int f, void* h_ws,
                          float* y_perm, uint64_t active_mask, cudaStream_t stream);
cudaError_t moek_combine(const float* y, const int32_t* inv, const float* w, const void* res, int T,
                         int d, int k, void* out, cudaStream_t stream);
cudaError_t moek_quantize(const void* w, int rows, int cols, uint32_t* q, void* s, cudaStream_t stream);
cudaError_t moek_synth_weight(uint64_t seed, uint64_t uid, long long n, int shift, void* out,
                              cudaStream_t stream);
cudaError_t moek_synth_input(uint64_t seed, uint64_t uid, long long n, void* out, cudaStream_t stream);
int moek_weight_shift(int K);
