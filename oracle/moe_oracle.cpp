// moe_oracle.cpp -- CPU restatement of the MoE expert-layer hot path.
// TEST INFRASTRUCTURE ONLY (see moe_oracle.h).  Never linked by the product.
//
// Semantics sources (the reference has no tensor math):
//   router  : HF MixtralTopKRouter, modeling_mixtral.py:109-116 (softmax -> topk
//             -> renormalise == softmax over the selected logits)
//   experts : HF MixtralExperts, modeling_mixtral.py:90-96 (down(silu(gate)*up))
//   combine : HF index_add_ of routing-weighted expert outputs, :96
//   indexing: expert = layer*E + slot (reference planner.hpp:29,
//             simulator.cpp:92-94)
#include "moe_oracle.h"

#include <algorithm>
#include <cmath>
#include <cstring>
#include <vector>
#ifdef _OPENMP
#include <omp.h>
#endif

namespace {

inline uint64_t mix64(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}

inline float bf2f(uint16_t b) {
    uint32_t u = static_cast<uint32_t>(b) << 16;
    float f;
    std::memcpy(&f, &u, 4);
    return f;
}

inline uint16_t f2bf(float f) {
    uint32_t u;
    std::memcpy(&u, &f, 4);
    if ((u & 0x7fffffffu) > 0x7f800000u) return 0x7fc0;  // NaN
    u += 0x7fffu + ((u >> 16) & 1u);
    return static_cast<uint16_t>(u >> 16);
}

inline int nibble_shift(int j) { return 4 * (j >> 1) + 16 * (j & 1); }

inline float silu(float g) { return g / (1.0f + std::exp(-g)); }

// Dot products straight off the stored weights (bf16 or int4-g128), with the
// 16 independent fp32 partial sums (index mod 16) and a fixed pairwise fold;
// the order is part of the oracle's definition (FFN parity is tolerance based)
// and it vectorises without -ffast-math.  No dequantised copy is materialised.
inline float dot_bf16(const uint16_t* w, const float* x, int n) {
    float acc[16] = {0};
    int i = 0;
    for (; i + 16 <= n; i += 16)
        for (int l = 0; l < 16; ++l) acc[l] = std::fmaf(bf2f(w[i + l]), x[i + l], acc[l]);
    for (; i < n; ++i) acc[i & 15] = std::fmaf(bf2f(w[i]), x[i], acc[i & 15]);
    for (int h = 8; h >= 1; h >>= 1)
        for (int l = 0; l < h; ++l) acc[l] += acc[l + h];
    return acc[0];
}

inline float dot_int4(const uint32_t* q, const uint16_t* s, const float* x, int n) {
    float acc[16] = {0};
    for (int g = 0; g < n / 128; ++g) {
        const float sf = bf2f(s[g]);
        for (int i = g * 128; i < g * 128 + 128; i += 16)
            for (int l = 0; l < 16; ++l) {
                const int c = i + l;
                const int qv = static_cast<int>((q[c >> 3] >> nibble_shift(c & 7)) & 15u) - 8;
                acc[l] = std::fmaf(static_cast<float>(qv) * sf, x[c], acc[l]);
            }
    }
    for (int h = 8; h >= 1; h >>= 1)
        for (int l = 0; l < h; ++l) acc[l] += acc[l + h];
    return acc[0];
}

struct ExpertView {
    int precision;  // 0 int4, 1 bf16
    const void* gu;
    const uint16_t* sgu;
    const void* dn;
    const uint16_t* sd;
};

inline float row_dot(const ExpertView& w, bool down, int row, int K, const float* x) {
    if (w.precision == 1) {
        const uint16_t* base = static_cast<const uint16_t*>(down ? w.dn : w.gu);
        return dot_bf16(base + static_cast<size_t>(row) * K, x, K);
    }
    const uint32_t* base = static_cast<const uint32_t*>(down ? w.dn : w.gu);
    const uint16_t* sc = down ? w.sd : w.sgu;
    return dot_int4(base + static_cast<size_t>(row) * (K / 8), sc + static_cast<size_t>(row) * (K / 128), x, K);
}

// SwiGLU FFN of M rows: h = bf16(silu(gate . x) * (up . x)); y = down . h.
void ffn_rows(const uint16_t* x, int M, const ExpertView& w, int d, int f, float* y) {
    std::vector<float> xf(static_cast<size_t>(M) * d), h(static_cast<size_t>(M) * f);
    for (size_t i = 0; i < xf.size(); ++i) xf[i] = bf2f(x[i]);
#pragma omp parallel for schedule(static)
    for (int n = 0; n < f; ++n)
        for (int m = 0; m < M; ++m) {
            const float* xm = &xf[static_cast<size_t>(m) * d];
            const float g = row_dot(w, false, n, d, xm);
            const float u = row_dot(w, false, f + n, d, xm);
            h[static_cast<size_t>(m) * f + n] = bf2f(f2bf(silu(g) * u));
        }
#pragma omp parallel for schedule(static)
    for (int j = 0; j < d; ++j)
        for (int m = 0; m < M; ++m)
            y[static_cast<size_t>(m) * d + j] = row_dot(w, true, j, f, &h[static_cast<size_t>(m) * f]);
}

}  // namespace

extern "C" {

uint64_t orc_rand64(uint64_t seed, uint64_t uid, uint64_t i) {
    const uint64_t key = mix64(seed ^ (uid * 0xD1B54A32D192ED03ULL));
    return mix64(key + (i + 1) * 0x9E3779B97F4A7C15ULL);
}

void orc_synth_weight_bf16(uint64_t seed, uint64_t uid, int64_t n, int p, uint16_t* out) {
    const float scale = std::ldexp(1.0f, -p);
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < n; ++i) {
        const int8_t k = static_cast<int8_t>(orc_rand64(seed, uid, static_cast<uint64_t>(i)) >> 56);
        out[i] = f2bf(static_cast<float>(k) * scale);
    }
}

void orc_synth_input_bf16(uint64_t seed, uint64_t uid, int64_t n, uint16_t* out) {
    for (int64_t i = 0; i < n; ++i) {
        const int k = static_cast<int>((orc_rand64(seed, uid, static_cast<uint64_t>(i)) >> 32) % 129u) - 64;
        out[i] = f2bf(static_cast<float>(k) / 64.0f);
    }
}

int orc_weight_shift(int K) {
    // uniform int8 has std ~73.9; choose 2^-p ~ 1/(73.9*sqrt(K))
    return static_cast<int>(std::lround(std::log2(73.9 * std::sqrt(static_cast<double>(K)))));
}

void orc_quantize_g128(const uint16_t* w, int rows, int cols, uint32_t* q, uint16_t* s) {
    const int groups = cols / 128;
#pragma omp parallel for schedule(static)
    for (int r = 0; r < rows; ++r) {
        const uint16_t* row = w + static_cast<size_t>(r) * cols;
        uint32_t* qrow = q + static_cast<size_t>(r) * (cols / 8);
        for (int g = 0; g < groups; ++g) {
            float amax = 0.0f;
            for (int i = 0; i < 128; ++i) amax = std::max(amax, std::fabs(bf2f(row[g * 128 + i])));
            uint16_t sb = f2bf(amax / 7.0f);
            if (amax == 0.0f) sb = f2bf(1.0f);
            s[static_cast<size_t>(r) * groups + g] = sb;
            const float sf = bf2f(sb);
            for (int wd = 0; wd < 16; ++wd) {
                uint32_t word = 0;
                for (int j = 0; j < 8; ++j) {
                    float qv = std::rint(bf2f(row[g * 128 + wd * 8 + j]) / sf);
                    qv = std::min(7.0f, std::max(-8.0f, qv));
                    const uint32_t u = static_cast<uint32_t>(static_cast<int>(qv) + 8);
                    word |= u << nibble_shift(j);
                }
                qrow[g * 16 + wd] = word;
            }
        }
    }
}

void orc_dequant_g128(const uint32_t* q, const uint16_t* s, int rows, int cols, float* w_out) {
    const int groups = cols / 128;
#pragma omp parallel for schedule(static)
    for (int r = 0; r < rows; ++r) {
        for (int c = 0; c < cols; ++c) {
            const uint32_t word = q[static_cast<size_t>(r) * (cols / 8) + c / 8];
            const int qv = static_cast<int>((word >> nibble_shift(c & 7)) & 15u) - 8;
            const float sf = bf2f(s[static_cast<size_t>(r) * groups + c / 128]);
            w_out[static_cast<size_t>(r) * cols + c] = static_cast<float>(qv) * sf;  // exact
        }
    }
}

void orc_gate_topk(const uint16_t* x, const uint16_t* wg, int T, int d, int E, int k,
                   int32_t* idx, float* w, float* logits) {
    std::vector<float> lg(static_cast<size_t>(E));
    for (int t = 0; t < T; ++t) {
        const uint16_t* xt = x + static_cast<size_t>(t) * d;
        for (int e = 0; e < E; ++e) {
            const uint16_t* we = wg + static_cast<size_t>(e) * d;
            // Pinned order: lane l owns k = c*256 + l*8 + j (c outer, j inner),
            // sequential fmaf per lane, then an xor butterfly 16,8,4,2,1.
            float lane[32];
            for (int l = 0; l < 32; ++l) {
                float acc = 0.0f;
                for (int c = 0; c * 256 < d; ++c)
                    for (int j = 0; j < 8; ++j) {
                        const int kk = c * 256 + l * 8 + j;
                        if (kk < d) acc = std::fmaf(bf2f(xt[kk]), bf2f(we[kk]), acc);
                    }
                lane[l] = acc;
            }
            for (int off = 16; off >= 1; off >>= 1) {
                float nxt[32];
                for (int l = 0; l < 32; ++l) nxt[l] = lane[l] + lane[l ^ off];
                std::memcpy(lane, nxt, sizeof lane);
            }
            lg[static_cast<size_t>(e)] = lane[0];
            if (logits) logits[static_cast<size_t>(t) * E + e] = lane[0];
        }
        // top-k on logits, ties -> lower index, output in descending order
        std::vector<char> taken(static_cast<size_t>(E), 0);
        float sel[64];
        for (int j = 0; j < k; ++j) {
            int best = -1;
            for (int e = 0; e < E; ++e)
                if (!taken[e] && (best < 0 || lg[e] > lg[best])) best = e;
            taken[best] = 1;
            idx[static_cast<size_t>(t) * k + j] = best;
            sel[j] = lg[best];
        }
        float ex[64], sum = 0.0f;
        for (int j = 0; j < k; ++j) {
            ex[j] = std::exp(sel[j] - sel[0]);
            sum += ex[j];
        }
        for (int j = 0; j < k; ++j) w[static_cast<size_t>(t) * k + j] = ex[j] / sum;
    }
}

void orc_permute(const int32_t* idx, int T, int E, int k, int32_t* counts, int32_t* offsets,
                 int32_t* perm, int32_t* inv_perm) {
    const int n = T * k;
    for (int e = 0; e < E; ++e) counts[e] = 0;
    for (int i = 0; i < n; ++i) counts[idx[i]]++;
    offsets[0] = 0;
    for (int e = 0; e < E; ++e) offsets[e + 1] = offsets[e] + counts[e];
    std::vector<int32_t> cursor(offsets, offsets + E);
    for (int i = 0; i < n; ++i) {  // ascending (t, j) => stable
        const int pos = cursor[static_cast<size_t>(idx[i])]++;
        perm[pos] = i;
        inv_perm[i] = pos;
    }
}

void orc_ffn_bf16(const uint16_t* x, int M, const uint16_t* wgu, const uint16_t* wd, int d, int f,
                  float* y) {
    ffn_rows(x, M, ExpertView{1, wgu, nullptr, wd, nullptr}, d, f, y);
}

void orc_ffn_int4(const uint16_t* x, int M, const uint32_t* qgu, const uint16_t* sgu,
                  const uint32_t* qd, const uint16_t* sd, int d, int f, float* y) {
    ffn_rows(x, M, ExpertView{0, qgu, sgu, qd, sd}, d, f, y);
}

void orc_combine(const float* y_perm, const int32_t* inv_perm, const float* w,
                 const uint16_t* residual, int T, int d, int k, uint16_t* out) {
    for (int t = 0; t < T; ++t)
        for (int c = 0; c < d; ++c) {
            float acc = residual ? bf2f(residual[static_cast<size_t>(t) * d + c]) : 0.0f;
            for (int j = 0; j < k; ++j) {
                const int pos = inv_perm[t * k + j];
                acc = std::fmaf(w[t * k + j], y_perm[static_cast<size_t>(pos) * d + c], acc);
            }
            out[static_cast<size_t>(t) * d + c] = f2bf(acc);
        }
}

void orc_expert_bf16(const orc_model* m, int e, uint16_t* wgu, uint16_t* wd) {
    const int d = m->d_model, f = m->d_ffn;
    orc_synth_weight_bf16(m->seed, (static_cast<uint64_t>(e) << 4) | 1u,
                          static_cast<int64_t>(2) * f * d, orc_weight_shift(d), wgu);
    orc_synth_weight_bf16(m->seed, (static_cast<uint64_t>(e) << 4) | 2u,
                          static_cast<int64_t>(d) * f, orc_weight_shift(f), wd);
}

void orc_expert_int4(const orc_model* m, int e, uint32_t* qgu, uint16_t* sgu, uint32_t* qd,
                     uint16_t* sd) {
    const int d = m->d_model, f = m->d_ffn;
    std::vector<uint16_t> gu(static_cast<size_t>(2) * f * d), dn(static_cast<size_t>(d) * f);
    orc_expert_bf16(m, e, gu.data(), dn.data());
    orc_quantize_g128(gu.data(), 2 * f, d, qgu, sgu);
    orc_quantize_g128(dn.data(), d, f, qd, sd);
}

void orc_router_weights(const orc_model* m, int layer, uint16_t* wg) {
    orc_synth_weight_bf16(m->seed, (1ULL << 48) | static_cast<uint64_t>(layer),
                          static_cast<int64_t>(m->num_experts) * m->d_model,
                          orc_weight_shift(m->d_model), wg);
}

void orc_step_input(const orc_model* m, int step, int T, uint16_t* x) {
    orc_synth_input_bf16(m->seed, (2ULL << 48) | static_cast<uint64_t>(step),
                         static_cast<int64_t>(T) * m->d_model, x);
}

namespace {

void layer_forward(const orc_model* m, const uint16_t* wg, const ExpertView* ex, const uint16_t* x_res, int T,
                   uint16_t* out, int32_t* idx_out, float* w_out, float* logits) {
    const int d = m->d_model, f = m->d_ffn, E = m->num_experts, k = m->top_k;
    std::vector<uint16_t> xn;
    const uint16_t* x = x_res;
    if (m->norm_eps > 0.0f) {
        xn.resize(static_cast<size_t>(T) * d);
        orc_rmsnorm(x_res, T, d, m->norm_eps, xn.data());
        x = xn.data();
    }
    std::vector<int32_t> idx(static_cast<size_t>(T) * k), perm(idx.size()), inv(idx.size());
    std::vector<float> w(idx.size());
    orc_gate_topk(x, wg, T, d, E, k, idx.data(), w.data(), logits);
    std::vector<int32_t> counts(E), offsets(E + 1);
    orc_permute(idx.data(), T, E, k, counts.data(), offsets.data(), perm.data(), inv.data());
    std::vector<float> y_perm(static_cast<size_t>(T) * k * d);
    for (int s = 0; s < E; ++s) {
        const int M = counts[s];
        if (M == 0) continue;
        std::vector<uint16_t> xs(static_cast<size_t>(M) * d);
        for (int r = 0; r < M; ++r) {
            const int t = perm[offsets[s] + r] / k;
            std::memcpy(&xs[static_cast<size_t>(r) * d], x + static_cast<size_t>(t) * d, d * 2);
        }
        ffn_rows(xs.data(), M, ex[s], d, f, &y_perm[static_cast<size_t>(offsets[s]) * d]);
    }
    orc_combine(y_perm.data(), inv.data(), w.data(), x_res, T, d, k, out);
    if (idx_out) std::memcpy(idx_out, idx.data(), idx.size() * 4);
    if (w_out) std::memcpy(w_out, w.data(), w.size() * 4);
}

}  // namespace

void orc_rmsnorm(const uint16_t* x, int T, int d, float eps, uint16_t* out) {
    for (int t = 0; t < T; ++t) {
        const uint16_t* xr = x + static_cast<size_t>(t) * d;
        float part[256];
        for (int i = 0; i < 256; ++i) {
            float acc = 0.0f;
            for (int c = 0; c * 256 + i < d; ++c) {
                const float v = bf2f(xr[c * 256 + i]);
                acc = std::fmaf(v, v, acc);
            }
            part[i] = acc;
        }
        for (int s2 = 128; s2 >= 1; s2 >>= 1)
            for (int i = 0; i < s2; ++i) part[i] += part[i + s2];
        const float rstd = 1.0f / std::sqrt(part[0] / static_cast<float>(d) + eps);
        for (int j = 0; j < d; ++j) out[static_cast<size_t>(t) * d + j] = f2bf(bf2f(xr[j]) * rstd);
    }
}

void orc_moe_layer_w(const orc_model* m, const uint16_t* wg, const orc_expert* experts, const uint16_t* x,
                     int T, uint16_t* out, int32_t* idx, float* w, float* logits) {
    std::vector<ExpertView> ex(static_cast<size_t>(m->num_experts));
    for (int s = 0; s < m->num_experts; ++s)
        ex[s] = ExpertView{experts[s].precision, experts[s].w_gate_up,
                           static_cast<const uint16_t*>(experts[s].s_gate_up), experts[s].w_down,
                           static_cast<const uint16_t*>(experts[s].s_down)};
    layer_forward(m, wg, ex.data(), x, T, out, idx, w, logits);
}

void orc_moe_layer(const orc_model* m, int layer, const int* precision, const uint16_t* x, int T,
                   uint16_t* out, int32_t* idx_out, float* w_out, float* logits) {
    const int d = m->d_model, f = m->d_ffn, E = m->num_experts;
    std::vector<uint16_t> wg(static_cast<size_t>(E) * d);
    orc_router_weights(m, layer, wg.data());
    // Materialise the layer's experts (only the selected ones matter, but
    // materialising all keeps this driver simple; tests use small shapes or
    // one layer).
    std::vector<std::vector<uint16_t>> b_gu(E), b_dn(E), b_sgu(E), b_sd(E);
    std::vector<std::vector<uint32_t>> q_gu(E), q_dn(E);
    std::vector<orc_expert> ex(static_cast<size_t>(E));
    std::vector<int32_t> idx(static_cast<size_t>(T) * m->top_k);
    std::vector<float> wtmp(idx.size());
    std::vector<uint16_t> xn(static_cast<size_t>(T) * d);
    if (m->norm_eps > 0.0f) orc_rmsnorm(x, T, d, m->norm_eps, xn.data());
    orc_gate_topk(m->norm_eps > 0.0f ? xn.data() : x, wg.data(), T, d, E, m->top_k, idx.data(), wtmp.data(), nullptr);
    std::vector<char> used(static_cast<size_t>(E), 0);
    for (int32_t v : idx) used[static_cast<size_t>(v)] = 1;
    for (int s = 0; s < E; ++s) {
        ex[s].precision = precision[s];
        if (!used[s]) continue;
        const int e = layer * E + s;
        if (precision[s] == 1) {
            b_gu[s].resize(static_cast<size_t>(2) * f * d);
            b_dn[s].resize(static_cast<size_t>(d) * f);
            orc_expert_bf16(m, e, b_gu[s].data(), b_dn[s].data());
            ex[s].w_gate_up = b_gu[s].data();
            ex[s].w_down = b_dn[s].data();
        } else {
            q_gu[s].resize(static_cast<size_t>(2) * f * d / 8);
            q_dn[s].resize(static_cast<size_t>(d) * f / 8);
            b_sgu[s].resize(static_cast<size_t>(2) * f * d / 128);
            b_sd[s].resize(static_cast<size_t>(d) * f / 128);
            orc_expert_int4(m, e, q_gu[s].data(), b_sgu[s].data(), q_dn[s].data(), b_sd[s].data());
            ex[s].w_gate_up = q_gu[s].data();
            ex[s].s_gate_up = b_sgu[s].data();
            ex[s].w_down = q_dn[s].data();
            ex[s].s_down = b_sd[s].data();
        }
    }
    orc_moe_layer_w(m, wg.data(), ex.data(), x, T, out, idx_out, w_out, logits);
}

// ---- fragment-block storage layout (see moe_oracle.h) ----------------------
int orc_perm_k(int k) {
    const int g = k / 128, kin = k % 128;
    const int kk = kin / 16, t = (kin % 8) / 2, hi = (kin % 16) / 8, e = kin % 2;
    return g * 128 + t * 32 + kk * 4 + hi * 2 + e;
}

namespace {

struct BlockPos {
    size_t block;  // block index rt*G + g
    int lane, half, r, gr;
};

inline BlockPos block_pos(int row, int k, int cols) {
    const int G = cols / 128;
    const int rt = row / 16, rr = row % 16;
    const int p = orc_perm_k(k % 128);
    BlockPos b;
    b.block = static_cast<size_t>(rt) * G + k / 128;
    b.gr = rr % 8;
    b.half = rr / 8;
    b.r = p % 32;
    b.lane = b.gr * 4 + p / 32;
    return b;
}

// bf16 block = 16 rows x 128 K in UMMA "core matrix" order: [K half h][row
// half cr][8-K column cc][row r8][8 K values] -- an 8 x 8 core matrix is 128
// contiguous bytes, so a 64-K half is a canonical no-swizzle K-major tile
// (core stride 128 B along K, 1024 B along M) and ldmatrix.x4 yields the
// mma.m16n8k16 A fragments.
inline size_t bf16_block_index(int row, int k, int cols) {  // in uint16 units
    const size_t block = static_cast<size_t>(row / 16) * (cols / 128) + k / 128;
    const int kin = k % 128, rr = row % 16;
    return block * 2048 + static_cast<size_t>((kin / 64) * 1024 + (rr / 8) * 512 + ((kin % 64) / 8) * 64 + (rr % 8) * 8 +
                                              kin % 8);
}

inline size_t int4_block_word(const BlockPos& b) {  // in uint32 units
    return b.block * 256 + static_cast<size_t>((b.half * 32 + b.lane) * 4 + b.r / 8);
}

}  // namespace

void orc_pack_bf16_blocks(const uint16_t* w, int rows, int cols, uint16_t* out) {
#pragma omp parallel for schedule(static)
    for (int r = 0; r < rows; ++r)
        for (int c = 0; c < cols; ++c) out[bf16_block_index(r, c, cols)] = w[static_cast<size_t>(r) * cols + c];
}

void orc_unpack_bf16_blocks(const uint16_t* blk, int rows, int cols, uint16_t* out) {
#pragma omp parallel for schedule(static)
    for (int r = 0; r < rows; ++r)
        for (int c = 0; c < cols; ++c) out[static_cast<size_t>(r) * cols + c] = blk[bf16_block_index(r, c, cols)];
}

void orc_pack_int4_blocks(const uint32_t* q, const uint16_t* s, int rows, int cols, uint32_t* qb,
                          uint16_t* sb) {
    const int G = cols / 128;
    std::memset(qb, 0, static_cast<size_t>(rows) * cols / 2);
#pragma omp parallel for schedule(static)
    for (int rt = 0; rt < rows / 16; ++rt)
        for (int rr = 0; rr < 16; ++rr) {
            const int r = rt * 16 + rr;
            for (int c = 0; c < cols; ++c) {
                const uint32_t u = (q[static_cast<size_t>(r) * (cols / 8) + c / 8] >> nibble_shift(c & 7)) & 15u;
                const BlockPos b = block_pos(r, c, cols);
                qb[int4_block_word(b)] |= u << nibble_shift(b.r % 8);
            }
            for (int g = 0; g < G; ++g)
                sb[(static_cast<size_t>(rt) * G + g) * 16 + (rr % 8) * 2 + rr / 8] = s[static_cast<size_t>(r) * G + g];
        }
}

void orc_unpack_int4_blocks(const uint32_t* qb, const uint16_t* sb, int rows, int cols, uint32_t* q,
                            uint16_t* s) {
    const int G = cols / 128;
    std::memset(q, 0, static_cast<size_t>(rows) * cols / 2);
#pragma omp parallel for schedule(static)
    for (int r = 0; r < rows; ++r) {
        const int rt = r / 16, rr = r % 16;
        for (int c = 0; c < cols; ++c) {
            const BlockPos b = block_pos(r, c, cols);
            const uint32_t u = (qb[int4_block_word(b)] >> nibble_shift(b.r % 8)) & 15u;
            q[static_cast<size_t>(r) * (cols / 8) + c / 8] |= u << nibble_shift(c & 7);
        }
        for (int g = 0; g < G; ++g)
            s[static_cast<size_t>(r) * G + g] = sb[(static_cast<size_t>(rt) * G + g) * 16 + (rr % 8) * 2 + rr / 8];
    }
}

int orc_num_threads(void) {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}

}  // extern "C"
