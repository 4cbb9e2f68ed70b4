// engine.cu -- MoeEngine (see include/moeb200/engine.hpp).
//
// HBM layout: one device arena holds every GPU-resident expert back to back
// (256-byte aligned), one pinned host arena holds the CPU-resident experts,
// one swap slot of plan.swap_slot_bytes receives streamed experts.  Per
// expert (d = d_model, f = d_ffn):
//   bf16 : [w_gate_up 2f*d bf16][w_down d*f bf16]                  = 6df B
//   int4 : [q_gate_up 2f*d/8 u32][s_gate_up 2f*d/128 bf16]
//          [q_down d*f/8 u32][s_down d*f/128 bf16]                 = 99df/64 B
// which are exactly expert_size(P16) / expert_size(P4) of the profile made by
// profile_for_shape(), so bytes_transferred is the bytes really copied.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <list>
#include <map>
#include <mutex>
#include <stdexcept>
#include <string>

#include "kernels/launch.h"
#include "moeb200/engine.hpp"

#define MOE_CUDA_OK_HOST(expr)                      \
    do {                                            \
        cudaError_t err__ = (expr);                 \
        if (err__ != cudaSuccess) return err__;     \
    } while (0)

// ---- fp16-operand range guard (kernels/common.cuh) ----------------------
namespace {
std::mutex g_num_mu;
unsigned int* g_num_word = nullptr;  // mapped pinned host word, process-wide
uint64_t g_num_bound = 0;            // devices whose kernel TUs point at it
}  // namespace

cudaError_t moek_numerics_bind_device() {
    std::lock_guard<std::mutex> lk(g_num_mu);
    int dev = 0;
    MOE_CUDA_OK_HOST(cudaGetDevice(&dev));
    if (dev < 64 && ((g_num_bound >> dev) & 1ull)) return cudaSuccess;
    if (g_num_word == nullptr) {
        void* h = nullptr;
        MOE_CUDA_OK_HOST(cudaHostAlloc(&h, 64, cudaHostAllocMapped | cudaHostAllocPortable));
        g_num_word = static_cast<unsigned int*>(h);
        *g_num_word = 0;
    }
    void* dp = nullptr;
    MOE_CUDA_OK_HOST(cudaHostGetDevicePointer(&dp, g_num_word, 0));
    unsigned int* p = static_cast<unsigned int*>(dp);
    MOE_CUDA_OK_HOST(moek_numerics_bind_gemv(p));
    MOE_CUDA_OK_HOST(moek_numerics_bind_router(p));
    MOE_CUDA_OK_HOST(moek_numerics_bind_tc(p));
    if (dev < 64) g_num_bound |= 1ull << dev;
    return cudaSuccess;
}

cudaError_t moek_stream_expert(void* dst, const void* src_pinned, size_t bytes, cudaStream_t copy, cudaEvent_t done) {
    MOE_CUDA_OK_HOST(cudaMemcpyAsync(dst, src_pinned, bytes, cudaMemcpyHostToDevice, copy));
    return done != nullptr ? cudaEventRecord(done, copy) : cudaSuccess;
}

unsigned int moek_numerics_status(int clear) {
    std::lock_guard<std::mutex> lk(g_num_mu);
    if (g_num_word == nullptr) return 0;
    const unsigned int v = __atomic_load_n(g_num_word, __ATOMIC_ACQUIRE);
    if (clear) __atomic_and_fetch(g_num_word, ~v, __ATOMIC_ACQ_REL);
    return v;
}

namespace moeb200 {

namespace {

void ck(cudaError_t e, const char* what) {
    if (e != cudaSuccess)
        throw std::runtime_error(std::string("CUDA error in ") + what + ": " + cudaGetErrorString(e));
}

size_t align_up(size_t v, size_t a) { return (v + a - 1) / a * a; }

uint64_t uid_expert(int e, int tensor) { return (static_cast<uint64_t>(e) << 4) | static_cast<uint64_t>(tensor); }
uint64_t uid_router(int layer) { return (1ULL << 48) | static_cast<uint64_t>(layer); }
uint64_t uid_input(int step) { return (2ULL << 48) | static_cast<uint64_t>(step); }

}  // namespace

int weight_shift(int K) {
    return static_cast<int>(std::lround(std::log2(73.9 * std::sqrt(static_cast<double>(K)))));
}

struct MoeEngine::Impl {
    EngineConfig cfg;
    PlacementPlan plan;
    int L = 0, E = 0, K = 0, d = 0, f = 0, Tmax = 0;
    size_t size16 = 0, size4 = 0;

    cudaStream_t compute = nullptr, copy = nullptr;
    cudaEvent_t copy_done = nullptr;

    char* dev_arena = nullptr;
    size_t dev_bytes = 0;
    char* host_arena = nullptr;
    size_t host_bytes = 0;
    char* swap = nullptr;        // slot pool: 1 slot (Static) or lru_capacity slots (LRU)
    size_t swap_bytes = 0;       // bytes per slot
    int nslots = 1;
    std::vector<cudaEvent_t> slot_free;
    // LRU residency (simulator.cpp:37-62): host-resident experts cached in
    // device slots, least recently used evicted; plan-resident ones pinned
    // The accounting state (lru / lru_pos / lru_slot_of) is simulate()'s
    // cache and is emptied by reset_counters(), as simulate() starts cold;
    // slot_holds is the physical truth -- which expert's bytes each device
    // slot holds -- and survives it.
    std::list<int>* lru = nullptr;
    std::map<int, std::list<int>::iterator> lru_pos;
    std::map<int, int> lru_slot_of;   // cached expert -> slot
    std::vector<int> slot_holds;      // [nslots]: expert whose weights the slot holds (-1: none)
    void lru_clear() {
        if (!lru) return;
        lru->clear();
        lru_pos.clear();
        lru_slot_of.clear();
    }
    bool lru_touch(int e) {
        const auto it = lru_pos.find(e);
        if (it == lru_pos.end()) return false;
        lru->splice(lru->begin(), *lru, it->second);
        return true;
    }
    void lru_insert(int e) {
        int slot;
        if (static_cast<int>(lru_pos.size()) >= nslots) {  // evict the least recently used
            const int victim = lru->back();
            lru->pop_back();
            lru_pos.erase(victim);
            slot = lru_slot_of[victim];
            lru_slot_of.erase(victim);
        } else {
            slot = static_cast<int>(lru_pos.size());
        }
        lru->push_front(e);
        lru_pos[e] = lru->begin();
        lru_slot_of[e] = slot;
    }
    uint16_t* wg = nullptr;  // [L][E][d]

    std::vector<moe_expert_weights> weights;  // [L*E]
    // keep_masters: pinned [L*E][bf16 blocks | int4 blocks]; reconfigure()'s
    // device copies are per-expert allocations (`owned`), freed on release
    char* master_arena = nullptr;
    size_t master_stride = 0;
    std::vector<char*> owned;                 // [L*E]
    char* host_copy(int e, Precision p) const {
        char* b = master_arena + static_cast<size_t>(e) * master_stride;
        return p == Precision::P16 ? b : b + align_up(size16, 256);
    }
    std::vector<int> location;                // [L*E]
    std::vector<char> layer_has_cpu;

    uint16_t* xin = nullptr;
    uint16_t* xout = nullptr;
    uint16_t* xbuf[2] = {nullptr, nullptr};
    int32_t* idx = nullptr;   // [L][Tmax*K]
    float* wts = nullptr;     // [L][Tmax*K]
    int32_t* counts = nullptr;
    int32_t* offsets = nullptr;
    int32_t* perm = nullptr;
    int32_t* inv = nullptr;
    unsigned int* ticket = nullptr;
    float* y = nullptr;          // per-slot expert outputs (streamed-expert and tcgen05 paths)
    int Tgemv = 0;               // largest T of the streaming-GEMV path (workspace sizing)
    void* tcws = nullptr;        // tcgen05 path workspace (T >= tc_min_tokens)
    uint16_t* xn = nullptr;      // [Tmax][d] normalised rows in natural order (tcgen05 path)
    GemvWorkspace gws{};
    void* gws_base = nullptr;
    int32_t* idx_host = nullptr;  // pinned [Tmax*K]
    size_t ws_bytes = 0;
    // fused batch-1 step (decode_step_kernel)
    moe_expert_weights* dev_experts = nullptr;  // [L*E] device copy of `weights`
    unsigned int* fused_ctl = nullptr;          // [L*2 tail-pool counters][2 barrier words]
    bool fused_ok = false;
    unsigned int* flow_ctl = nullptr;           // decode_flow_kernel's per-layer completion counters
    float* flow_part = nullptr;                 // its partial buffers (sentinel-filled between uses)
    uint16_t* flow_x = nullptr;                 // its 3 layer-output rows (0xffff = not yet written)
    size_t flow_part0_floats = 0, flow_part1_floats = 0;
    bool flow_ok = false;                       // dataflow variant (default; MOE_FUSED=step: grid barriers)

    // expert parallelism (ep_a2a.cu): G ranks, this one owns slots s*G/E == rank
    bool ep = false;
    int G = 1, rank = 0, C = 0;          // C = entries per source rank (Tmax * K)
    std::vector<char> mine;              // [E] slot owned by this rank
    char* ep_buf = nullptr;              // rows | meta | ret | flags (peers write here)
    size_t ep_bytes = 0;
    std::vector<const void*> ep_peers;   // [G] exchange buffers, rank order
    uint32_t* ep_epoch = nullptr;
    int32_t *ep_keys = nullptr, *ep_counts = nullptr, *ep_offsets = nullptr, *ep_perm = nullptr, *ep_inv = nullptr,
            *ep_iota = nullptr;
    float* ep_y = nullptr;               // [G*C][d] per computed entry
    uint16_t* ep_dense = nullptr;        // GEMV path: received rows in slot order [G*ep_Tgemv*K][d]
    GemvWorkspace ep_gws{};
    void* ep_gws_base = nullptr;
    void* ep_tcws = nullptr;
    int ep_Tgemv = 0;                    // largest local T served by the GEMV on the received rows

    SimReport counters;
    std::map<int, cudaGraphExec_t> graphs;

    moe_expert_weights view(char* base, Precision p) const {
        moe_expert_weights w{};
        const size_t fd = static_cast<size_t>(f) * d;
        if (p == Precision::P16) {
            w.precision = MOE_P16;
            w.w_gate_up = base;
            w.w_down = base + 4 * fd;
        } else {
            w.precision = MOE_P4;
            w.w_gate_up = base;
            w.s_gate_up = base + fd;
            w.w_down = base + fd + fd / 32;
            w.s_down = base + fd + fd / 32 + fd / 2;
        }
        return w;
    }

    void dev_alloc(void** p, size_t bytes) {
        ck(cudaMalloc(p, bytes), "cudaMalloc");
        ws_bytes += bytes;
    }

    void init(const EngineConfig& c, const PlacementPlan& pl) {
        cfg = c;
        plan = pl;
        L = c.profile.num_layers;
        E = c.profile.experts_per_layer;
        K = c.profile.top_k;
        d = c.shape.d_model;
        f = c.shape.d_ffn;
        Tmax = c.max_tokens;
        validate_profile(c.profile);
        validate_shape(c.shape);
        if (E > MOE_MAX_EXPERTS) throw ValidationError("experts_per_layer exceeds MOE_MAX_EXPERTS");
        if (K > MOE_MAX_TOPK) throw ValidationError("top_k exceeds MOE_MAX_TOPK");
        if (Tmax < 1) throw ValidationError("max_tokens must be >= 1");
        G = c.ep_world;
        rank = c.ep_rank;
        ep = G > 1;
        if (G < 1 || G > 8 || rank < 0 || rank >= G) throw ValidationError("ep_world must be in [1, 8] and ep_rank in [0, ep_world)");
        if (ep && (E < G || E >= MOE_MAX_EXPERTS))
            throw ValidationError("expert parallelism needs ep_world <= experts_per_layer < MOE_MAX_EXPERTS");
        if (ep && (c.lru_capacity > 0 || c.keep_masters))
            throw UsageError("the expert-parallel engine serves device-resident experts (no LRU / reconfiguration masters)");
        mine.assign(static_cast<size_t>(E), 1);
        for (int s2 = 0; s2 < E; ++s2) mine[static_cast<size_t>(s2)] = !ep || s2 * G / E == rank;
        if (static_cast<int>(plan.entries.size()) != L * E)
            throw ValidationError("plan covers " + std::to_string(plan.entries.size()) +
                                  " experts, engine has " + std::to_string(L * E));
        size16 = static_cast<size_t>(expert_bytes_bf16(c.shape));
        size4 = static_cast<size_t>(expert_bytes_int4(c.shape));
        if (static_cast<size_t>(expert_size(c.profile, Precision::P16)) != size16 ||
            static_cast<size_t>(expert_size(c.profile, Precision::P4)) != size4)
            throw ValidationError("profile expert sizes do not match the tensor shape "
                                  "(build the profile with profile_for_shape)");
        int ndev = 0;
        if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0)
            throw std::runtime_error("no CUDA device: the MoE engine has no CPU fallback");
        ck(cudaSetDevice(c.device), "cudaSetDevice");
        ck(moek_numerics_bind_device(), "numerics guard");
        ck(cudaStreamCreateWithFlags(&compute, cudaStreamNonBlocking), "stream");
        if (c.keep_masters) {
            // reconfigure() allocates per-expert copies stream-ordered: keep
            // freed pool memory mapped instead of returning it at every sync
            cudaMemPool_t pool;
            ck(cudaDeviceGetDefaultMemPool(&pool, c.device), "mempool");
            uint64_t keep = UINT64_MAX;
            ck(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep), "mempool attr");
        }
        ck(cudaStreamCreateWithFlags(&copy, cudaStreamNonBlocking), "stream");
        ck(cudaEventCreateWithFlags(&copy_done, cudaEventDisableTiming), "event");
        if (c.lru_capacity > 0 && c.lru_capacity < c.profile.top_k)
            throw ValidationError("lru_capacity must be 0 (Static) or >= top_k");
        nslots = c.lru_capacity > 0 ? c.lru_capacity : 1;
        slot_free.resize(static_cast<size_t>(nslots));
        for (auto& ev : slot_free) ck(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming), "event");
        slot_holds.assign(static_cast<size_t>(nslots), -1);
        if (c.lru_capacity > 0) lru = new std::list<int>();

        // arenas
        std::vector<size_t> off(static_cast<size_t>(L * E));
        layer_has_cpu.assign(static_cast<size_t>(L), 0);
        location.assign(static_cast<size_t>(L * E), MOE_GPU);
        size_t swap_need = 0;
        for (int i = 0; i < L * E; ++i) {
            const ExpertState st = plan.entries[static_cast<size_t>(i)];
            const size_t sz = st.precision == Precision::P16 ? size16 : size4;
            if (!mine[static_cast<size_t>(i % E)]) continue;  // another rank's expert: not held here
            if (ep && st.location != Location::GPU)
                throw UsageError("the expert-parallel engine serves device-resident experts: plan expert " +
                                 std::to_string(i) + " is host-resident");
            if (st.location == Location::GPU) {
                off[static_cast<size_t>(i)] = dev_bytes;
                dev_bytes += align_up(sz, 256);
            } else {
                if (!c.keep_masters) {
                    off[static_cast<size_t>(i)] = host_bytes;
                    host_bytes += align_up(sz, 256);
                }
                layer_has_cpu[static_cast<size_t>(i / E)] = 1;
                location[static_cast<size_t>(i)] = MOE_CPU;
                swap_need = std::max(swap_need, sz);
            }
        }
        if (static_cast<size_t>(plan.swap_slot_bytes) < swap_need)
            throw ValidationError("plan swap_slot_bytes smaller than the largest CPU-resident expert");
        if (dev_bytes) ck(cudaMalloc(&dev_arena, dev_bytes), "cudaMalloc(expert arena)");
        if (host_bytes) ck(cudaHostAlloc(&host_arena, host_bytes, cudaHostAllocDefault), "cudaHostAlloc(host arena)");
        owned.assign(static_cast<size_t>(L * E), nullptr);
        if (c.keep_masters) {
            master_stride = align_up(size16, 256) + align_up(size4, 256);
            ck(cudaHostAlloc(&master_arena, master_stride * static_cast<size_t>(L * E), cudaHostAllocDefault),
               "cudaHostAlloc(master copies)");
        }
        swap_bytes = static_cast<size_t>(plan.swap_slot_bytes);
        if (swap_bytes) ck(cudaMalloc(&swap, swap_bytes * static_cast<size_t>(nslots)), "cudaMalloc(swap slots)");
        weights.resize(static_cast<size_t>(L * E));
        for (int i = 0; i < L * E; ++i) {
            const ExpertState st = plan.entries[static_cast<size_t>(i)];
            if (!mine[static_cast<size_t>(i % E)]) {
                weights[static_cast<size_t>(i)] = moe_expert_weights{};
                weights[static_cast<size_t>(i)].precision = st.precision == Precision::P16 ? MOE_P16 : MOE_P4;
                continue;
            }
            char* base = st.location == Location::GPU ? dev_arena + off[static_cast<size_t>(i)]
                         : c.keep_masters              ? host_copy(i, st.precision)
                                                       : host_arena + off[static_cast<size_t>(i)];
            weights[static_cast<size_t>(i)] = view(base, st.precision);
        }

        // workspaces
        const size_t TK = static_cast<size_t>(Tmax) * K;
        dev_alloc(reinterpret_cast<void**>(&wg), static_cast<size_t>(L) * E * d * 2);
        dev_alloc(reinterpret_cast<void**>(&xin), static_cast<size_t>(Tmax) * d * 2);
        dev_alloc(reinterpret_cast<void**>(&xout), static_cast<size_t>(Tmax) * d * 2);
        dev_alloc(reinterpret_cast<void**>(&xbuf[0]), static_cast<size_t>(Tmax) * d * 2);
        dev_alloc(reinterpret_cast<void**>(&xbuf[1]), static_cast<size_t>(Tmax) * d * 2);
        dev_alloc(reinterpret_cast<void**>(&idx), static_cast<size_t>(L) * TK * 4);
        dev_alloc(reinterpret_cast<void**>(&wts), static_cast<size_t>(L) * TK * 4);
        dev_alloc(reinterpret_cast<void**>(&counts), static_cast<size_t>(E) * 4);
        dev_alloc(reinterpret_cast<void**>(&offsets), static_cast<size_t>(E + 1) * 4);
        dev_alloc(reinterpret_cast<void**>(&perm), TK * 4);
        dev_alloc(reinterpret_cast<void**>(&inv), TK * 4);
        dev_alloc(reinterpret_cast<void**>(&ticket), 4);
        dev_alloc(reinterpret_cast<void**>(&y), TK * d * 4);
        // streaming GEMV below tc_min_tokens, tcgen05 GEMM from there on
        Tgemv = std::min(Tmax, std::max(1, cfg.tc_min_tokens - 1));
        if (Tgemv > moek_gemv_max_tokens(E, K))
            throw UsageError("decode batches below tc_min_tokens exceed the streaming GEMV's limit for " +
                             std::to_string(E) + " experts top-" + std::to_string(K) + " (moe_gemv_max_tokens = " +
                             std::to_string(moek_gemv_max_tokens(E, K)) + "): lower tc_min_tokens");
        const size_t ws_bytes = moek_gemv_workspace_bytes(Tgemv, K, d, f);
        dev_alloc(&gws_base, ws_bytes);
        ck(cudaMemsetAsync(gws_base, 0, ws_bytes, compute), "memset");
        gws = moek_gemv_workspace_view(gws_base, Tgemv, K, d, f);
        if (Tmax >= cfg.tc_min_tokens) {
            dev_alloc(&tcws, moek_tc_workspace_bytes(Tmax, K, d, f));
            dev_alloc(reinterpret_cast<void**>(&xn), static_cast<size_t>(Tmax) * d * 2);
        }
        ck(cudaMemsetAsync(ticket, 0, 4, compute), "memset");
        ck(cudaMemsetAsync(xin, 0, static_cast<size_t>(Tmax) * d * 2, compute), "memset");
        if (ep) ep_alloc();
        if (!ep && !cfg.per_layer_decode && moek_decode_step_supported(E, K, d, f)) {
            dev_alloc(reinterpret_cast<void**>(&dev_experts), static_cast<size_t>(L) * E * sizeof(moe_expert_weights));
            dev_alloc(reinterpret_cast<void**>(&fused_ctl), (static_cast<size_t>(L) * 2 + 2) * 4);
            ck(cudaMemsetAsync(fused_ctl, 0, (static_cast<size_t>(L) * 2 + 2) * 4, compute), "memset");
            fused_ok = true;
            int dev = 0, sms = 0;
            ck(cudaGetDevice(&dev), "cudaGetDevice");
            ck(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev), "attr");
            const char* mode = getenv("MOE_FUSED");
            if ((mode == nullptr || std::string(mode) != "step") && moek_decode_flow_supported(E, K, d, f, sms)) {
                const size_t words = moek_decode_flow_ctl_words(L, K, d, f);
                dev_alloc(reinterpret_cast<void**>(&flow_ctl), words * 4);
                ck(cudaMemsetAsync(flow_ctl, 0, words * 4, compute), "memset");
                // [d/128][K][2f] gate/up + [f/128][K][d] down partials, 0xffffffff = none pending
                // two of each (by layer parity)
                flow_part0_floats = static_cast<size_t>(d / 128) * K * 2 * f;
                flow_part1_floats = static_cast<size_t>(f / 128) * K * d;
                const size_t pf = 2 * (flow_part0_floats + flow_part1_floats);
                dev_alloc(reinterpret_cast<void**>(&flow_part), pf * 4);
                ck(cudaMemsetAsync(flow_part, 0xff, pf * 4, compute), "memset");
                dev_alloc(reinterpret_cast<void**>(&flow_x), static_cast<size_t>(3) * d * 2);
                ck(cudaMemsetAsync(flow_x, 0xff, static_cast<size_t>(3) * d * 2, compute), "memset");
                flow_ok = true;
            }
        }
        ck(cudaHostAlloc(reinterpret_cast<void**>(&idx_host), TK * 4, cudaHostAllocDefault), "cudaHostAlloc");

        materialize();
        upload_experts();
    }

    // the device expert table the fused step reads (after init / reconfigure)
    void upload_experts() {
        if (!dev_experts) return;
        ck(cudaMemcpyAsync(dev_experts, weights.data(), weights.size() * sizeof(moe_expert_weights),
                           cudaMemcpyHostToDevice, compute), "H2D expert table");
        ck(cudaStreamSynchronize(compute), "sync");
    }

    bool use_fused(int T) const {
        if (!fused_ok || T != 1) return false;
        for (char c : layer_has_cpu)
            if (c) return false;
        return true;
    }

    void launch_fused() {
        MoeDecodeArgs a{};
        a.L = L;
        a.E = E;
        a.k = K;
        a.d = d;
        a.f = f;
        a.norm_eps = cfg.norm_eps;
        a.experts = dev_experts;
        a.wg = wg;
        a.x_in = xin;
        a.xbuf0 = xbuf[0];
        a.xbuf1 = xbuf[1];
        a.x_out = xout;
        a.idx = idx;
        a.wts = wts;
        a.idx_stride = Tmax * K;
        a.part0 = gws.part0;
        a.part1 = gws.part1;
        a.hperm = static_cast<uint16_t*>(gws.hperm);
        a.hperm16 = static_cast<uint16_t*>(gws.hperm16);
        a.hsum = gws.hsum;
        a.sched = fused_ctl;
        a.bar = reinterpret_cast<unsigned long long*>(fused_ctl + static_cast<size_t>(L) * 2);
        static const int bar_mode = getenv("MOE_BAR_MODE") ? atoi(getenv("MOE_BAR_MODE")) : 0;
        a.bar_mode = bar_mode;
        a.flow_ctl = flow_ctl;
        if (flow_ok) {
            a.part0 = flow_part;
            a.part1 = flow_part + 2 * flow_part0_floats;
            a.part0_stride = flow_part0_floats;
            a.part1_stride = flow_part1_floats;
            a.xbuf0 = flow_x;
            a.xbuf1 = flow_x + d;
            a.xbuf2 = flow_x + 2 * static_cast<size_t>(d);
            ck(moek_decode_flow(a, compute), "decode_flow");
        } else {
            ck(moek_decode_step(a, compute), "decode_step");
        }
    }

    // Synthetic weights: bf16 masters from the counter-based generator,
    // quantised to int4-g128 on device for P4 experts (the same definitions
    // as oracle/moe_oracle.cpp), CPU-resident experts copied to the arena.
    void materialize() {
        const size_t fd = static_cast<size_t>(f) * d;
        const int sh_gu = weight_shift(d), sh_d = weight_shift(f);
        for (int l = 0; l < L; ++l)
            ck(moek_synth_weight(cfg.seed, uid_router(l), static_cast<long long>(E) * d, sh_gu,
                                 wg + static_cast<size_t>(l) * E * d, compute), "synth router");
        // logical (row-major) bf16 master -> fragment blocks (bf16 or int4)
        char* master = nullptr;
        char* stage = nullptr;
        ck(cudaMalloc(&master, size16), "cudaMalloc(master)");
        if (host_bytes || master_arena) ck(cudaMalloc(&stage, size16), "cudaMalloc(stage)");
        for (int e = 0; e < L * E; ++e) {
            const ExpertState st = plan.entries[static_cast<size_t>(e)];
            if (!mine[static_cast<size_t>(e % E)]) continue;  // another rank's expert
            ck(moek_synth_weight(cfg.seed, uid_expert(e, 1), static_cast<long long>(2 * fd), sh_gu, master, compute), "synth");
            ck(moek_synth_weight(cfg.seed, uid_expert(e, 2), static_cast<long long>(fd), sh_d, master + 4 * fd, compute), "synth");
            char* dst = st.location == Location::GPU ? static_cast<char*>(const_cast<void*>(weights[static_cast<size_t>(e)].w_gate_up))
                                                     : stage;
            moe_expert_weights v = view(dst, st.precision);
            if (st.precision == Precision::P16) {
                ck(moek_pack_bf16_blocks(master, 2 * f, d, const_cast<void*>(v.w_gate_up), compute), "pack");
                ck(moek_pack_bf16_blocks(master + 4 * fd, d, f, const_cast<void*>(v.w_down), compute), "pack");
            } else {
                ck(moek_quantize_blocks(master, 2 * f, d, static_cast<uint32_t*>(const_cast<void*>(v.w_gate_up)),
                                        const_cast<void*>(v.s_gate_up), compute), "quantize");
                ck(moek_quantize_blocks(master + 4 * fd, d, f, static_cast<uint32_t*>(const_cast<void*>(v.w_down)),
                                        const_cast<void*>(v.s_down), compute), "quantize");
            }
            if (master_arena) {
                // both host copies: the plan precision from dst first (dst may be
                // stage), then the other one made in stage
                const Precision other = st.precision == Precision::P16 ? Precision::P4 : Precision::P16;
                for (Precision p : {st.precision, other}) {
                    const size_t sz = p == Precision::P16 ? size16 : size4;
                    const void* src = dst;
                    if (p != st.precision) {
                        moe_expert_weights o = view(stage, p);
                        if (p == Precision::P16) {
                            ck(moek_pack_bf16_blocks(master, 2 * f, d, const_cast<void*>(o.w_gate_up), compute), "pack");
                            ck(moek_pack_bf16_blocks(master + 4 * fd, d, f, const_cast<void*>(o.w_down), compute), "pack");
                        } else {
                            ck(moek_quantize_blocks(master, 2 * f, d, static_cast<uint32_t*>(const_cast<void*>(o.w_gate_up)),
                                                    const_cast<void*>(o.s_gate_up), compute), "quantize");
                            ck(moek_quantize_blocks(master + 4 * fd, d, f, static_cast<uint32_t*>(const_cast<void*>(o.w_down)),
                                                    const_cast<void*>(o.s_down), compute), "quantize");
                        }
                        src = stage;
                    }
                    ck(cudaMemcpyAsync(host_copy(e, p), src, sz, cudaMemcpyDeviceToHost, compute), "D2H master");
                    ck(cudaStreamSynchronize(compute), "sync");  // stage reused
                }
            } else if (st.location == Location::CPU) {
                const size_t sz = st.precision == Precision::P16 ? size16 : size4;
                ck(cudaMemcpyAsync(const_cast<void*>(weights[static_cast<size_t>(e)].w_gate_up), stage, sz,
                                   cudaMemcpyDeviceToHost, compute), "D2H");
            }
            ck(cudaStreamSynchronize(compute), "sync");  // master / stage reused next iteration
        }
        cudaFree(master);
        if (stage) cudaFree(stage);
    }


    // ---- reconfiguration executor (reconfig.hpp; MoeEngine::reconfigure) ----
    void release_dev(int e) {
        // per-expert copies made by reconfigure are freed; arena copies stay
        // allocated (the arena is one block) until the engine is destroyed
        char*& p = owned[static_cast<size_t>(e)];
        if (p) ck(cudaFreeAsync(p, compute), "cudaFreeAsync");
        p = nullptr;
    }
    char* dev_new(int e, size_t bytes) {
        char* p = nullptr;
        ck(cudaMallocAsync(reinterpret_cast<void**>(&p), bytes, compute), "cudaMallocAsync(expert)");
        owned[static_cast<size_t>(e)] = p;
        return p;
    }

    ReconfigReport reconfigure(const PlacementPlan& target, const HardwareProfile& hw) {
        if (!master_arena)
            throw UsageError("reconfigure needs keep_masters (host copies of every expert, reconfig.hpp:39)");
        const ReconfigPlan rp = diff_plans(plan, target, cfg.profile, hw);
        const PlacementPlan next = apply(plan, rp, cfg.profile);  // checked replay (state, exclusivity)
        if (next.entries != target.entries) throw ValidationError("action list does not reach the target plan");
        ck(cudaStreamSynchronize(compute), "sync");
        ck(cudaStreamSynchronize(copy), "sync");
        for (auto& g : graphs) cudaGraphExecDestroy(g.second);  // expert pointers change
        graphs.clear();
        ReconfigReport rep;
        rep.actions = static_cast<int>(rp.actions.size());
        rep.bytes_moved = rp.bytes_moved;
        rep.est_downtime_s = rp.est_downtime_s;
        const size_t fd = static_cast<size_t>(f) * d;
        char* logical = nullptr;  // Quantize scratch: one expert's logical bf16 matrices
        cudaEvent_t t0, t1;
        ck(cudaEventCreate(&t0), "event");
        ck(cudaEventCreate(&t1), "event");
        ck(cudaEventRecord(t0, compute), "record");
        std::vector<ExpertState> cur = plan.entries;
        for (const ReconfigAction& a : rp.actions) {
            const int e = expert_index(cfg.profile, a.expert);
            ExpertState& st = cur[static_cast<size_t>(e)];
            moe_expert_weights& w = weights[static_cast<size_t>(e)];
            switch (a.kind) {
                case ActionKind::Offload:  // nothing moves toward the GPU: the host copy takes over
                    release_dev(e);
                    st.location = Location::CPU;
                    w = view(host_copy(e, st.precision), st.precision);
                    break;
                case ActionKind::Quantize:
                    st.precision = Precision::P4;
                    if (st.location == Location::GPU) {  // on-device int4-g128 from the 16-bit copy
                        if (!logical) ck(cudaMallocAsync(reinterpret_cast<void**>(&logical), size16, compute), "cudaMallocAsync");
                        ck(moek_unpack_bf16_blocks(w.w_gate_up, 2 * f, d, logical, compute), "unpack");
                        ck(moek_unpack_bf16_blocks(w.w_down, d, f, logical + 4 * fd, compute), "unpack");
                        char* prev = owned[static_cast<size_t>(e)];
                        owned[static_cast<size_t>(e)] = nullptr;
                        moe_expert_weights q = view(dev_new(e, size4), Precision::P4);
                        ck(moek_quantize_blocks(logical, 2 * f, d, static_cast<uint32_t*>(const_cast<void*>(q.w_gate_up)),
                                                const_cast<void*>(q.s_gate_up), compute), "quantize");
                        ck(moek_quantize_blocks(logical + 4 * fd, d, f, static_cast<uint32_t*>(const_cast<void*>(q.w_down)),
                                                const_cast<void*>(q.s_down), compute), "quantize");
                        if (prev) ck(cudaFreeAsync(prev, compute), "cudaFreeAsync");
                        w = q;
                    } else {
                        w = view(host_copy(e, Precision::P4), Precision::P4);
                    }
                    break;
                case ActionKind::Dequantize:
                    st.precision = Precision::P16;
                    if (st.location == Location::GPU) {  // in-place upgrade: pull the 16-bit master
                        char* prev = owned[static_cast<size_t>(e)];
                        owned[static_cast<size_t>(e)] = nullptr;
                        char* nb = dev_new(e, size16);
                        ck(cudaMemcpyAsync(nb, host_copy(e, Precision::P16), size16, cudaMemcpyHostToDevice, compute), "H2D");
                        rep.bytes_h2d += static_cast<bytes_t>(size16);
                        if (prev) ck(cudaFreeAsync(prev, compute), "cudaFreeAsync");
                        w = view(nb, Precision::P16);
                    } else {
                        w = view(host_copy(e, Precision::P16), Precision::P16);
                    }
                    break;
                case ActionKind::Fetch: {  // the host copy at its (destination) precision
                    st.location = Location::GPU;
                    const size_t sz = st.precision == Precision::P16 ? size16 : size4;
                    char* nb = dev_new(e, sz);
                    ck(cudaMemcpyAsync(nb, host_copy(e, st.precision), sz, cudaMemcpyHostToDevice, compute), "H2D");
                    rep.bytes_h2d += static_cast<bytes_t>(sz);
                    w = view(nb, st.precision);
                    break;
                }
            }
        }
        if (logical) ck(cudaFreeAsync(logical, compute), "cudaFreeAsync");
        ck(cudaEventRecord(t1, compute), "record");
        ck(cudaEventSynchronize(t1), "sync");
        float ms = 0.0f;
        ck(cudaEventElapsedTime(&ms, t0, t1), "elapsed");
        cudaEventDestroy(t0);
        cudaEventDestroy(t1);
        rep.measured_s = ms / 1e3;
        // the new plan: residency flags, swap slot(s), LRU state
        plan = next;
        layer_has_cpu.assign(static_cast<size_t>(L), 0);
        for (int i = 0; i < L * E; ++i) {
            const bool cpu = plan.entries[static_cast<size_t>(i)].location == Location::CPU;
            location[static_cast<size_t>(i)] = cpu ? MOE_CPU : MOE_GPU;
            if (cpu) layer_has_cpu[static_cast<size_t>(i / E)] = 1;
        }
        if (static_cast<size_t>(plan.swap_slot_bytes) > swap_bytes) {
            if (swap) ck(cudaFree(swap), "cudaFree(swap)");
            swap_bytes = static_cast<size_t>(plan.swap_slot_bytes);
            ck(cudaMalloc(&swap, swap_bytes * static_cast<size_t>(nslots)), "cudaMalloc(swap slots)");
        }
        lru_clear();
        slot_holds.assign(static_cast<size_t>(nslots), -1);  // slots may have been reallocated
        upload_experts();
        return rep;
    }

    void destroy() {
        for (auto& g : graphs) cudaGraphExecDestroy(g.second);
        graphs.clear();
        if (compute) cudaStreamSynchronize(compute);
        for (char* p : owned)
            if (p) cudaFree(p);
        owned.clear();
        if (master_arena) cudaFreeHost(master_arena);
        if (copy) cudaStreamSynchronize(copy);
        void* devp[] = {tcws, xn, dev_arena, swap, wg, xin, xout, xbuf[0], xbuf[1], idx, wts, counts, offsets, perm, inv, ticket, y,
                         gws_base, dev_experts, fused_ctl, flow_ctl, flow_part, flow_x, ep_buf, ep_epoch, ep_keys, ep_counts, ep_offsets, ep_perm,
                         ep_inv, ep_iota, ep_y, ep_gws_base, ep_tcws, ep_dense};
        for (void* p : devp)
            if (p) cudaFree(p);
        if (host_arena) cudaFreeHost(host_arena);
        if (idx_host) cudaFreeHost(idx_host);
        if (copy_done) cudaEventDestroy(copy_done);
        for (auto& ev : slot_free)
            if (ev) cudaEventDestroy(ev);
        delete lru;
        lru = nullptr;
        if (compute) cudaStreamDestroy(compute);
        if (copy) cudaStreamDestroy(copy);
    }

    void check_numerics() {
        // experiments that feed the kernels garbage on purpose (MOE_TC_DBG /
        // MOE_GEMV_DBG ablations) switch the guard off
        static const bool off = getenv("MOE_NUMERICS_CHECK_OFF") != nullptr;
        if (off) return;
        bool int4 = false;
        for (const ExpertState& st : plan.entries) int4 = int4 || st.precision == Precision::P4;
        if (!int4) return;
        const unsigned int v = moek_numerics_status(1);
        if (v & MOE_NUM_F16_ACT_BIT)
            throw ValidationError("int4 expert path: an activation (x or h) exceeds the fp16 range (|v| > 65504) "
                                  "of the int4 kernels' fp16 operand copy; its output is not finite");
        if (v & MOE_NUM_F16_SCALE_BIT)
            throw ValidationError("int4 expert path (tcgen05): an int4-g128 scale lies outside [2^-14, 8188], "
                                  "so the on-chip fp16 dequantisation q*s is inexact or infinite");
    }

    uint64_t mask_all() const { return E >= 64 ? ~0ull : ((1ull << E) - 1ull); }

    // One MoE layer: route -> FFN (streaming CPU-resident experts through the
    // swap slot(s)) -> combine with residual.  T < tc_min_tokens runs the
    // streaming GEMV, T >= tc_min_tokens the tcgen05 GEMM; both serve plans
    // with host-resident experts.
    void layer(int l, const uint16_t* x, int T, uint16_t* out, int32_t* idx_l, float* w_l, float* logits) {
        const moe_expert_weights* lw = weights.data() + static_cast<size_t>(l) * E;
        const bool tc = T >= cfg.tc_min_tokens;
        const bool host = layer_has_cpu[static_cast<size_t>(l)] != 0;
        if (!tc && T > Tgemv) throw UsageError("T exceeds the streaming-GEMV workspace (raise tc_min_tokens / max_tokens)");
        const uint16_t* xnorm = tc && cfg.norm_eps > 0.0f ? xn : x;  // tcgen05 B operand (natural order)
        if (tc) {
            // tcgen05 path: route writes the normalised rows in natural order
            ck(moek_route(x, wg + static_cast<size_t>(l) * E * d, T, d, E, K, idx_l, w_l, logits, counts, offsets,
                          perm, inv, ticket, compute, nullptr, nullptr, nullptr, 0, cfg.norm_eps,
                          cfg.norm_eps > 0.0f ? xn : nullptr),
               "route");
        } else {
            // route also writes the K-permuted activation copies the expert
            // GEMV reads (no separate permute kernel on the critical path)
            ck(moek_route(x, wg + static_cast<size_t>(l) * E * d, T, d, E, K, idx_l, w_l, logits, counts,
                          offsets, perm, inv, ticket, compute, gws.xperm, gws.xperm16, gws.xsum, moek_group_stride(d),
                          cfg.norm_eps),
               "route");
        }
        counters.activations += static_cast<int64_t>(T) * K;
        // expert FFN of the experts in `mask` into the per-slot outputs y
        auto ffn_y = [&](uint64_t mask, const moe_expert_weights* ew) {
            if (tc)
                ck(moek_ffn_tc(tcws, xnorm, perm, offsets, T, K, ew, E, d, f, mask, y, compute), "ffn_tc");
            else
                ck(moek_ffn_mma(gws, x, perm, offsets, inv, w_l, x, T, K, ew, E, d, f, mask, nullptr, y, MOE_X_READY,
                                compute), "ffn");
        };
        if (!host) {
            counters.hits += static_cast<int64_t>(T) * K;
            if (tc) {
                ck(moek_ffn_tc_combine(tcws, xnorm, perm, offsets, T, K, lw, E, d, f, mask_all(), y, inv, w_l, x, out,
                                       compute), "ffn_tc+combine");
            } else {
                ck(moek_ffn_mma(gws, x, perm, offsets, inv, w_l, x, T, K, lw, E, d, f, mask_all(), out, nullptr,
                                MOE_X_ROUTED, compute), "ffn");
            }
            return;
        }
        ck(cudaMemcpyAsync(idx_host, idx_l, static_cast<size_t>(T) * K * 4, cudaMemcpyDeviceToHost, compute), "D2H idx");
        ck(cudaStreamSynchronize(compute), "sync");
        // activation order of simulate(): tokens in order, each token's k
        // slots ascending (the GatingTrace record order, gating.cpp:48).  At
        // T > 1 this walks the batch inside the layer (the physical order of
        // a batched step); simulate() walks a trace token-major across layers,
        // so LRU hit counts equal it at T = 1 (Static at any T).
        std::vector<int32_t> order(idx_host, idx_host + static_cast<size_t>(T) * K);
        for (int t = 0; t < T; ++t) std::sort(order.begin() + t * K, order.begin() + (t + 1) * K);
        uint64_t sel = 0;
        for (int32_t s : order) sel |= 1ull << s;
        uint64_t resident = 0;
        for (int s = 0; s < E; ++s)
            if (((sel >> s) & 1ull) && location[static_cast<size_t>(l * E + s)] == MOE_GPU) resident |= 1ull << s;
        if (resident) ffn_y(resident, lw);
        std::vector<moe_expert_weights> tmp(lw, lw + E);
        uint64_t done = 0;
        for (int i = 0; i < T * K; ++i) {
            const int s = order[static_cast<size_t>(i)];
            const int e = l * E + s;
            const ExpertState st = plan.entries[static_cast<size_t>(e)];
            // simulate()'s per-activation rule (simulator.cpp:98-106):
            // GPU-resident, or (LRU) cached -> hit; else a transfer
            bool hit = st.location == Location::GPU;
            if (!hit && lru != nullptr) hit = lru_touch(e);
            if (hit) {
                ++counters.hits;
            } else {
                counters.bytes_transferred += static_cast<int64_t>(st.precision == Precision::P16 ? size16 : size4);
                if (lru != nullptr) lru_insert(e);
            }
            if (st.location == Location::GPU || ((done >> s) & 1ull)) continue;
            // first activation of host expert s in this layer: compute it now,
            // from the slot the accounting gives it (it is there at this point
            // of the walk; a later eviction in the same layer cannot affect a
            // computation already ordered on the stream).  The slot's bytes are
            // (re)streamed unless it already physically holds the expert.
            done |= 1ull << s;
            const moe_expert_weights& hw = lw[s];
            const size_t sz = hw.precision == MOE_P16 ? size16 : size4;
            const int slot = lru != nullptr ? lru_slot_of.at(e) : 0;
            char* dst = swap + static_cast<size_t>(slot) * swap_bytes;
            // Static re-streams every host activation (simulator.cpp:103-104)
            if (lru == nullptr || slot_holds[static_cast<size_t>(slot)] != e) {
                ck(cudaStreamWaitEvent(copy, slot_free[static_cast<size_t>(slot)], 0), "wait");
                ck(moek_stream_expert(dst, hw.w_gate_up, sz, copy, copy_done), "H2D expert");
                ck(cudaStreamWaitEvent(compute, copy_done, 0), "wait");
                slot_holds[static_cast<size_t>(slot)] = e;
            }
            tmp[static_cast<size_t>(s)] = view(dst, hw.precision == MOE_P16 ? Precision::P16 : Precision::P4);
            ffn_y(1ull << s, tmp.data());
            ck(cudaEventRecord(slot_free[static_cast<size_t>(slot)], compute), "record");
        }
        ck(moek_combine(y, inv, w_l, x, T, d, K, out, compute), "combine");
    }

    // ---- expert parallelism (ep_a2a.cu) ------------------------------------
    void ep_alloc() {
        // a rank's step spins on its peers' flags while the peers launch:
        // no kernel of the step may be loaded lazily (first-launch loading
        // can wait for the device to idle -> deadlock)
        ck(moek_preload_gemv(), "preload");
        ck(moek_preload_router(), "preload");
        ck(moek_preload_misc(), "preload");
        ck(moek_preload_tc(), "preload");
        ck(moek_preload_ep(), "preload");
        C = Tmax * K;
        const int Tp = G * C;  // received entries, sparse (one region per source rank)
        ep_bytes = moek_ep_a2a_bytes(G, C, d);
        ck(cudaMalloc(reinterpret_cast<void**>(&ep_buf), ep_bytes), "cudaMalloc(ep exchange)");  // own allocation: IPC maps it whole
        ck(cudaMemsetAsync(ep_buf, 0, ep_bytes, compute), "memset");
        dev_alloc(reinterpret_cast<void**>(&ep_epoch), 4);
        ck(cudaMemsetAsync(ep_epoch, 0, 4, compute), "memset");
        dev_alloc(reinterpret_cast<void**>(&ep_keys), static_cast<size_t>(Tp) * 4);
        dev_alloc(reinterpret_cast<void**>(&ep_counts), static_cast<size_t>(E + 1) * 4);
        dev_alloc(reinterpret_cast<void**>(&ep_offsets), static_cast<size_t>(E + 2) * 4);
        dev_alloc(reinterpret_cast<void**>(&ep_perm), static_cast<size_t>(Tp) * 4);
        dev_alloc(reinterpret_cast<void**>(&ep_inv), static_cast<size_t>(Tp) * 4);
        const int niota = std::max(C, Tp);
        dev_alloc(reinterpret_cast<void**>(&ep_iota), static_cast<size_t>(niota) * 4);
        dev_alloc(reinterpret_cast<void**>(&ep_y), static_cast<size_t>(Tp) * d * 4);
        std::vector<int32_t> io(static_cast<size_t>(niota));
        for (int i = 0; i < niota; ++i) io[static_cast<size_t>(i)] = i;
        ck(cudaMemcpy(ep_iota, io.data(), io.size() * 4, cudaMemcpyHostToDevice), "H2D iota");
        // owners run their experts on the received rows with k = 1: the GEMV
        // while the worst case (every rank's entries to this one) fits its
        // segment table, the tcgen05 GEMM from tc_min_tokens local tokens on
        ep_Tgemv = std::min(Tmax, std::max(1, cfg.tc_min_tokens - 1));
        while (ep_Tgemv > 0 && G * ep_Tgemv * K > moek_gemv_max_tokens(E, 1)) --ep_Tgemv;
        if (ep_Tgemv > 0) {
            const size_t b = moek_gemv_workspace_bytes(G * ep_Tgemv * K, 1, d, f);
            dev_alloc(&ep_gws_base, b);
            ck(cudaMemsetAsync(ep_gws_base, 0, b, compute), "memset");
            ep_gws = moek_gemv_workspace_view(ep_gws_base, G * ep_Tgemv * K, 1, d, f);
            dev_alloc(reinterpret_cast<void**>(&ep_dense), static_cast<size_t>(G) * ep_Tgemv * K * d * 2);
            ck(cudaMemsetAsync(ep_dense, 0, static_cast<size_t>(G) * ep_Tgemv * K * d * 2, compute), "memset");
        }
        if (Tmax > ep_Tgemv) dev_alloc(&ep_tcws, moek_tc_workspace_bytes(Tp, 1, d, f));
        if (!xn) dev_alloc(reinterpret_cast<void**>(&xn), static_cast<size_t>(Tmax) * d * 2);
        ck(cudaStreamSynchronize(compute), "sync");
    }

    uint64_t mine_mask() const {
        uint64_t m = 0;
        for (int s2 = 0; s2 < E; ++s2)
            if (mine[static_cast<size_t>(s2)]) m |= 1ull << s2;
        return m;
    }

    // One expert-parallel layer: route this rank's T tokens, send each routed
    // row to its expert's owner, run this rank's experts on what it received,
    // return the outputs to their sources, combine.  All on `compute`.
    void ep_layer(int l, const uint16_t* x, int T, uint16_t* out, int32_t* idx_l, float* w_l) {
        const int Tp = G * C;
        const uint16_t* xr = cfg.norm_eps > 0.0f ? xn : x;  // the experts' input rows (natural order)
        ck(moek_route(x, wg + static_cast<size_t>(l) * E * d, T, d, E, K, idx_l, w_l, nullptr, nullptr, nullptr,
                      nullptr, nullptr, ticket, compute, nullptr, nullptr, nullptr, 0, cfg.norm_eps,
                      cfg.norm_eps > 0.0f ? xn : nullptr),
           "route");
        const void* const* peers = ep_peers.data();
        ck(moek_ep_a2a_dispatch(xr, idx_l, T, K, E, d, C, rank, G, peers, ep_epoch, l, compute), "ep dispatch");
        ck(moek_ep_a2a_wait(ep_buf, 0, G, C, d, ep_epoch, l, compute), "ep wait rows");
        const int32_t* meta = reinterpret_cast<const int32_t*>(ep_buf + moek_ep_a2a_offset(G, C, d, 1));
        const void* rows = ep_buf + moek_ep_a2a_offset(G, C, d, 0);
        ck(moek_ep_a2a_keys(meta, Tp, E, ep_keys, compute), "ep keys");
        ck(moek_permute(ep_keys, Tp, E + 1, 1, ep_counts, ep_offsets, ep_perm, ep_inv, compute), "ep permute");
        const moe_expert_weights* lw = weights.data() + static_cast<size_t>(l) * E;
        if (T <= ep_Tgemv) {
            // received rows (G sparse regions of C entries) in slot order,
            // then the GEMV with the identity permutation over them
            const int Tg = G * ep_Tgemv * K;
            ck(moek_ep_a2a_gather(rows, ep_perm, ep_offsets, E, d, Tg, ep_dense, compute), "ep gather");
            ck(moek_ffn_mma(ep_gws, ep_dense, ep_iota, ep_offsets, ep_iota, nullptr, nullptr, Tg, 1, lw, E, d, f,
                            mine_mask(), nullptr, ep_y, MOE_X_PERMUTE, compute),
               "ep ffn");
        } else {
            ck(moek_ffn_tc(ep_tcws, rows, ep_perm, ep_offsets, Tp, 1, lw, E, d, f, mine_mask(), ep_y, compute), "ep ffn_tc");
        }
        ck(moek_ep_a2a_return(ep_y, ep_perm, ep_offsets, E, d, C, rank, G, peers, ep_epoch, l, compute), "ep return");
        ck(moek_ep_a2a_wait(ep_buf, 1, G, C, d, ep_epoch, l, compute), "ep wait returns");
        const float* ret = reinterpret_cast<const float*>(ep_buf + moek_ep_a2a_offset(G, C, d, 2));
        ck(moek_combine(ret, ep_iota, w_l, x, T, d, K, out, compute), "ep combine");
    }

    void run_layers(int T) {
        if (ep) {
            if (static_cast<int>(ep_peers.size()) != G) throw UsageError("expert-parallel engine: ep_set_peers first");
            const uint16_t* src = xin;
            const size_t TK = static_cast<size_t>(Tmax) * K;
            for (int l = 0; l < L; ++l) {
                uint16_t* dst = l == L - 1 ? xout : xbuf[l & 1];
                ep_layer(l, src, T, dst, idx + l * TK, wts + l * TK);
                src = dst;
            }
            ck(moek_ep_a2a_bump(ep_epoch, L, compute), "ep epoch");
            return;
        }
        if (use_fused(T)) {
            launch_fused();
            counters.activations += static_cast<int64_t>(T) * K * L;
            counters.hits += static_cast<int64_t>(T) * K * L;
            return;
        }
        const uint16_t* src = xin;
        const size_t TK = static_cast<size_t>(Tmax) * K;
        for (int l = 0; l < L; ++l) {
            uint16_t* dst = l == L - 1 ? xout : xbuf[l & 1];
            layer(l, src, T, dst, idx + l * TK, wts + l * TK, nullptr);
            src = dst;
        }
    }

    // Eager decode step with CUDA events (on the compute stream, where the
    // kernels are launched) bracketing each layer's expert-FFN launches.
    // Returns per-layer FFN milliseconds and the algorithmic bytes that FFN
    // must move: weights + scales of the distinct selected experts, the x
    // rows read, h written and read back, y written.
    void profile_step(int T, float* ffn_ms, int64_t* ffn_bytes, int* kernels_per_step) {
        if (T < 1 || T > Tmax) throw ValidationError("T must be in [1, max_tokens]");
        for (char c : layer_has_cpu)
            if (c) throw UsageError("profile_step needs an all-device-resident plan");
        std::vector<cudaEvent_t> ev(static_cast<size_t>(2 * L));
        for (auto& e : ev) ck(cudaEventCreate(&e), "event");
        const SimReport saved = counters;
        const uint16_t* src = xin;
        const size_t TK = static_cast<size_t>(Tmax) * K;
        for (int l = 0; l < L; ++l) {
            uint16_t* dst = l == L - 1 ? xout : xbuf[l & 1];
            const moe_expert_weights* lw = weights.data() + static_cast<size_t>(l) * E;
            const bool tc = T >= cfg.tc_min_tokens;
            ck(moek_route(src, wg + static_cast<size_t>(l) * E * d, T, d, E, K, idx + l * TK, wts + l * TK,
                          nullptr, counts, offsets, perm, inv, ticket, compute, tc ? nullptr : gws.xperm,
                          tc ? nullptr : gws.xperm16, tc ? nullptr : gws.xsum, moek_group_stride(d), cfg.norm_eps,
                          tc && cfg.norm_eps > 0.0f ? xn : nullptr), "route");
            ck(cudaEventRecord(ev[static_cast<size_t>(2 * l)], compute), "record");
            if (tc) {
                ck(moek_ffn_tc_combine(tcws, cfg.norm_eps > 0.0f ? xn : src, perm, offsets, T, K, lw, E, d, f,
                                       mask_all(), y, inv, wts + l * TK, src, dst, compute), "ffn_tc+combine");
            } else {
                ck(moek_ffn_mma(gws, src, perm, offsets, inv, wts + l * TK, src, T, K, lw, E, d, f, mask_all(), dst,
                                nullptr, MOE_X_ROUTED, compute), "ffn");
            }
            ck(cudaEventRecord(ev[static_cast<size_t>(2 * l + 1)], compute), "record");
            src = dst;
        }
        ck(cudaStreamSynchronize(compute), "sync");
        counters = saved;
        std::vector<int32_t> all(static_cast<size_t>(L) * TK);
        ck(cudaMemcpy(all.data(), idx, all.size() * 4, cudaMemcpyDeviceToHost), "D2H routing");
        for (int l = 0; l < L; ++l) {
            float ms = 0.0f;
            ck(cudaEventElapsedTime(&ms, ev[static_cast<size_t>(2 * l)], ev[static_cast<size_t>(2 * l + 1)]), "elapsed");
            ffn_ms[l] = ms;
            uint64_t sel = 0;
            for (int i = 0; i < T * K; ++i) sel |= 1ull << all[static_cast<size_t>(l) * TK + static_cast<size_t>(i)];
            int64_t bytes = 0;
            for (int s = 0; s < E; ++s)
                if ((sel >> s) & 1ull)
                    bytes += static_cast<int64_t>(plan.entries[static_cast<size_t>(l * E + s)].precision == Precision::P16 ? size16 : size4);
            bytes += static_cast<int64_t>(T) * K * d * 2      // x rows gathered
                     + static_cast<int64_t>(T) * K * f * 2 * 2  // h written + read
                     + static_cast<int64_t>(T) * K * d * 4;     // y written
            ffn_bytes[l] = bytes;
        }
        for (auto& e : ev) cudaEventDestroy(e);
        // GEMV: route(+x permute), gate/up stream, SwiGLU finalize, down stream, combine finalize
        // tcgen05: route, row gather, gate/up GEMM (+SwiGLU), down GEMM, combine
        if (kernels_per_step) *kernels_per_step = 5 * L;
    }

    bool profile_fused(float* ms, int64_t* bytes) {
        if (!use_fused(1)) return false;
        cudaEvent_t e0, e1;
        ck(cudaEventCreate(&e0), "event");
        ck(cudaEventCreate(&e1), "event");
        ck(cudaEventRecord(e0, compute), "record");
        launch_fused();
        ck(cudaEventRecord(e1, compute), "record");
        ck(cudaEventSynchronize(e1), "sync");
        ck(cudaEventElapsedTime(ms, e0, e1), "elapsed");
        cudaEventDestroy(e0);
        cudaEventDestroy(e1);
        const size_t TK = static_cast<size_t>(Tmax) * K;
        std::vector<int32_t> all(static_cast<size_t>(L) * TK);
        ck(cudaMemcpy(all.data(), idx, all.size() * 4, cudaMemcpyDeviceToHost), "D2H routing");
        int64_t b = 0;
        for (int l = 0; l < L; ++l) {
            uint64_t sel = 0;
            for (int i = 0; i < K; ++i) sel |= 1ull << all[static_cast<size_t>(l) * TK + static_cast<size_t>(i)];
            for (int s = 0; s < E; ++s)
                if ((sel >> s) & 1ull)
                    b += static_cast<int64_t>(plan.entries[static_cast<size_t>(l * E + s)].precision == Precision::P16 ? size16 : size4);
            b += static_cast<int64_t>(K) * d * 2 + static_cast<int64_t>(K) * f * 2 * 2 + static_cast<int64_t>(K) * d * 4;
        }
        *bytes = b;
        return true;
    }

    bool graphable() const {
        if (!cfg.use_graphs) return false;
        for (char c : layer_has_cpu)
            if (c) return false;
        return true;
    }

    void decode(int T) {
        if (T < 1 || T > Tmax) throw ValidationError("T must be in [1, max_tokens]");
        if (!graphable()) {
            run_layers(T);
            return;
        }
        auto it = graphs.find(T);
        if (it == graphs.end()) {
            // warm the launch-geometry caches outside capture
            const SimReport saved = counters;
            run_layers(T);
            ck(cudaStreamSynchronize(compute), "sync");
            counters = saved;
            cudaGraph_t g = nullptr;
            ck(cudaStreamBeginCapture(compute, cudaStreamCaptureModeThreadLocal), "capture");
            run_layers(T);
            ck(cudaStreamEndCapture(compute, &g), "capture end");
            counters = saved;
            cudaGraphExec_t ge = nullptr;
            ck(cudaGraphInstantiate(&ge, g, 0), "instantiate");
            cudaGraphDestroy(g);
            it = graphs.emplace(T, ge).first;
        }
        ck(cudaGraphLaunch(it->second, compute), "graph launch");
        counters.activations += static_cast<int64_t>(T) * K * L;
        counters.hits += static_cast<int64_t>(T) * K * L;
    }
};

MoeEngine::MoeEngine(const EngineConfig& cfg, const PlacementPlan& plan) : impl_(new Impl) {
    try {
        impl_->init(cfg, plan);
    } catch (...) {
        impl_->destroy();
        throw;
    }
}

MoeEngine::~MoeEngine() { impl_->destroy(); }

void* MoeEngine::input() { return impl_->xin; }
void* MoeEngine::output() { return impl_->xout; }
void* MoeEngine::stream() { return impl_->compute; }

void MoeEngine::synth_input(int step, int T) {
    if (T < 1 || T > impl_->Tmax) throw ValidationError("T must be in [1, max_tokens]");
    ck(moek_synth_input(impl_->cfg.seed, uid_input(step), static_cast<long long>(T) * impl_->d, impl_->xin,
                        impl_->compute), "synth input");
}

void* MoeEngine::ep_buffer(size_t* bytes) {
    if (bytes) *bytes = impl_->ep_bytes;
    return impl_->ep_buf;
}

void MoeEngine::ep_set_peers(const void* const* bases, int world) {
    Impl& m = *impl_;
    if (!m.ep) throw UsageError("ep_set_peers: the engine is not expert-parallel (ep_world = 1)");
    if (world != m.G || bases == nullptr) throw UsageError("ep_set_peers: expected " + std::to_string(m.G) + " buffer bases");
    if (bases[m.rank] != m.ep_buf) throw UsageError("ep_set_peers: bases[ep_rank] must be this engine's own ep_buffer");
    for (int r = 0; r < world; ++r)
        if (bases[r] == nullptr) throw UsageError("ep_set_peers: null base for rank " + std::to_string(r));
    m.ep_peers.assign(bases, bases + world);
    for (auto& g : m.graphs) cudaGraphExecDestroy(g.second);  // captured with the old bases
    m.graphs.clear();
}

void MoeEngine::decode(int T) {
    impl_->decode(T);
    impl_->counters.tokens += T;
}

void MoeEngine::decode_host(const void* x_host, int T, void* out_host) {
    if (T < 1 || T > impl_->Tmax) throw ValidationError("T must be in [1, max_tokens]");
    const size_t bytes = static_cast<size_t>(T) * impl_->d * 2;
    ck(cudaMemcpyAsync(impl_->xin, x_host, bytes, cudaMemcpyHostToDevice, impl_->compute), "H2D x");
    decode(T);
    ck(cudaMemcpyAsync(out_host, impl_->xout, bytes, cudaMemcpyDeviceToHost, impl_->compute), "D2H out");
    sync();
}

void MoeEngine::forward_layer(int layer, const void* x, int T, void* out, int32_t* idx, float* w,
                              float* logits) {
    if (layer < 0 || layer >= impl_->L) throw ValidationError("layer out of range");
    if (T < 1 || T > impl_->Tmax) throw ValidationError("T must be in [1, max_tokens]");
    // routing outputs are optional: default to the engine's own per-layer buffers
    const size_t TK = static_cast<size_t>(impl_->Tmax) * impl_->K;
    if (idx == nullptr) idx = impl_->idx + layer * TK;
    if (w == nullptr) w = impl_->wts + layer * TK;
    impl_->layer(layer, static_cast<const uint16_t*>(x), T, static_cast<uint16_t*>(out), idx, w, logits);
}

// Raises on the fp16-operand range guard when this engine's plan has int4
// experts (only their paths compute on fp16 copies); the word is cleared.
void MoeEngine::sync() {
    ck(cudaStreamSynchronize(impl_->compute), "sync");
    impl_->check_numerics();
}

bool MoeEngine::profile_fused(float* ms, int64_t* bytes) { return impl_->profile_fused(ms, bytes); }

void* MoeEngine::debug_buffer(int which, size_t* bytes) {
    Impl& m = *impl_;
    const size_t kd = static_cast<size_t>(m.K);
    switch (which) {
        case 0: *bytes = static_cast<size_t>(m.d / 128) * kd * 2 * m.f * 4; return m.gws.part0;
        case 1: *bytes = static_cast<size_t>(m.f / 128) * kd * m.d * 4; return m.gws.part1;
        case 2: *bytes = kd * m.f * 2; return m.gws.hperm;
        case 3: *bytes = kd * m.f * 2; return m.gws.hperm16;
        case 4: *bytes = kd * moek_group_stride(m.f) * 4; return m.gws.hsum;
        default: *bytes = 0; return nullptr;
    }
}
bool MoeEngine::fused() const { return impl_->use_fused(1); }

void MoeEngine::profile_step(int T, float* ffn_ms, int64_t* ffn_bytes, int* kernels_per_step) {
    impl_->profile_step(T, ffn_ms, ffn_bytes, kernels_per_step);
}

ReconfigReport MoeEngine::reconfigure(const PlacementPlan& target, const HardwareProfile& hw) {
    return impl_->reconfigure(target, hw);
}

const PlacementPlan& MoeEngine::plan() const { return impl_->plan; }

GatingTrace MoeEngine::last_routing(int T) {
    Impl& m = *impl_;
    sync();
    const size_t TK = static_cast<size_t>(m.Tmax) * m.K;
    std::vector<int32_t> all(static_cast<size_t>(m.L) * TK);
    ck(cudaMemcpy(all.data(), m.idx, all.size() * 4, cudaMemcpyDeviceToHost), "D2H routing");
    GatingTrace tr;
    tr.profile_fingerprint = profile_fingerprint(m.cfg.profile);
    tr.tokens = T;
    tr.num_layers = m.L;
    tr.experts_per_layer = m.E;
    tr.top_k = m.K;
    tr.slots.resize(static_cast<size_t>(T) * m.L * m.K);
    for (int t = 0; t < T; ++t)
        for (int l = 0; l < m.L; ++l) {
            int32_t* rec = tr.slots.data() + (static_cast<size_t>(t) * m.L + l) * m.K;
            for (int j = 0; j < m.K; ++j) rec[j] = all[static_cast<size_t>(l) * TK + static_cast<size_t>(t) * m.K + j];
            std::sort(rec, rec + m.K);
        }
    return tr;
}

const SimReport& MoeEngine::counters() const { return impl_->counters; }
// A new simulate() window: counters zeroed and the LRU accounting cache
// emptied (simulate() starts cold, simulator.cpp:66-87); the device slots keep
// their bytes, so an expert still physically present is not re-copied.
void MoeEngine::reset_counters() {
    impl_->counters = SimReport{};
    impl_->lru_clear();
}

moe_expert_weights MoeEngine::expert(int layer, int slot, int* location) const {
    const Impl& m = *impl_;
    if (layer < 0 || layer >= m.L || slot < 0 || slot >= m.E) throw ValidationError("expert id out of range");
    const size_t i = static_cast<size_t>(layer) * m.E + slot;
    if (location) *location = m.location[i];
    return m.weights[i];
}

const void* MoeEngine::router(int layer) const {
    if (layer < 0 || layer >= impl_->L) throw ValidationError("layer out of range");
    return impl_->wg + static_cast<size_t>(layer) * impl_->E * impl_->d;
}

void MoeEngine::memory(int64_t* expert_bytes, int64_t* swap_bytes, int64_t* host_bytes,
                       int64_t* workspace_bytes) const {
    if (expert_bytes) *expert_bytes = static_cast<int64_t>(impl_->dev_bytes);
    if (swap_bytes) *swap_bytes = static_cast<int64_t>(impl_->swap_bytes) * impl_->nslots;
    if (host_bytes) *host_bytes = static_cast<int64_t>(impl_->host_bytes);
    if (workspace_bytes) *workspace_bytes = static_cast<int64_t>(impl_->ws_bytes);
}

}  // namespace moeb200
