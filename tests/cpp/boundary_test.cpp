// boundary_test.cpp -- the drop-in boundary, compiled.
//
// Built against the reference's own headers and library (oracle/_ref,
// compiled from /root/reference/proj/src) and linked to libmoe_b200.so
// through integration/b200_backend.cpp:
//   moeserve::make_plan (reference planner, planner.hpp:71)
//     -> moe_engine_* (B200 engine via the C ABI, real kernels)
//     -> SimReport counters + the engine's real routing as a GatingTrace
//     -> moeserve::simulate on that trace (reference, simulator.hpp:56-58)
// and asserts the engine's counters equal the reference's, for Static and
// LRU residency on plans with host-resident experts.  Also drives
// moe_stream_expert (pinned H2D on a side stream + event) byte for byte.
// Exit 0 = pass.  Needs a CUDA device.
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "b200_backend.hpp"
#include "moe_b200.h"
#include "moeserve/errors.hpp"
#include "moeserve/planner.hpp"
#include "moeserve/simulator.hpp"

using namespace moeserve;

static int failures = 0;
#define EXPECT(cond, ...)                                  \
    do {                                                   \
        if (!(cond)) {                                     \
            std::fprintf(stderr, "FAIL %s:%d: ", __FILE__, __LINE__); \
            std::fprintf(stderr, __VA_ARGS__);             \
            std::fprintf(stderr, "\n");                    \
            ++failures;                                    \
        }                                                  \
    } while (0)

static void one_case(const char* name, double resident_frac, const ResidencyPolicy& policy, int steps) {
    const b200::EngineShape shape{512, 1792, 1e-5f};
    const ModelProfile model = b200::profile_for_shape(shape, 2, 8, 2, 1);
    TaskRequest task;
    task.preference = Preference::Quality;
    task.n4_target = 8;
    task.seed = 1;
    HardwareProfile hw;
    hw.gpu_mem_bytes = 1'000'000'000'000'000LL;
    const PlacementPlan full = make_plan(task, hw, model);
    const bytes_t s16 = model.size_expert16_bytes;
    hw.gpu_mem_bytes = model.size_nonexpert_bytes + s16 +
                       static_cast<bytes_t>(resident_frac * static_cast<double>(gpu_footprint(full, model) -
                                                                               model.size_nonexpert_bytes));
    const PlacementPlan plan = make_plan(task, hw, model);  // the reference planner
    int n_cpu = 0;
    for (const ExpertState& e : plan.entries) n_cpu += e.location == Location::CPU;
    GatingTrace routing;
    const SimReport got = b200::run_engine(plan, model, shape, policy, steps, 1, 11, &routing);
    const SimReport want = simulate(plan, routing, model, hw, policy);  // the reference cost model
    std::printf("%-24s cpu-resident %2d  engine: act %lld hits %lld bytes %lld | reference simulate(): act %lld "
                "hits %lld bytes %lld\n",
                name, n_cpu, static_cast<long long>(got.activations), static_cast<long long>(got.hits),
                static_cast<long long>(got.bytes_transferred), static_cast<long long>(want.activations),
                static_cast<long long>(want.hits), static_cast<long long>(want.bytes_transferred));
    EXPECT(resident_frac >= 1.0 || n_cpu > 0, "%s: plan has no host-resident experts", name);
    EXPECT(got.tokens == want.tokens, "%s: tokens %d vs %d", name, got.tokens, want.tokens);
    EXPECT(got.activations == want.activations, "%s: activations", name);
    EXPECT(got.hits == want.hits, "%s: hits %lld vs %lld", name, static_cast<long long>(got.hits),
           static_cast<long long>(want.hits));
    EXPECT(got.bytes_transferred == want.bytes_transferred, "%s: bytes_transferred", name);
}

static void stream_expert_case() {
    const size_t bytes = (90u << 20) + 4096 + 17;  // ~ one Mixtral int4 expert, odd tail
    unsigned char* host = nullptr;
    void* dev = nullptr;
    cudaStream_t copy;
    cudaEvent_t done;
    if (cudaHostAlloc(reinterpret_cast<void**>(&host), bytes, cudaHostAllocDefault) != cudaSuccess ||
        cudaMalloc(&dev, bytes) != cudaSuccess || cudaStreamCreateWithFlags(&copy, cudaStreamNonBlocking) != cudaSuccess ||
        cudaEventCreateWithFlags(&done, cudaEventDisableTiming) != cudaSuccess) {
        EXPECT(false, "CUDA setup failed");
        return;
    }
    for (size_t i = 0; i < bytes; ++i) host[i] = static_cast<unsigned char>((i * 2654435761u) >> 13);
    b200::check(moe_stream_expert(dev, host, bytes, copy, done));
    cudaEventSynchronize(done);
    std::vector<unsigned char> back(bytes);
    cudaMemcpy(back.data(), dev, bytes, cudaMemcpyDeviceToHost);
    EXPECT(std::memcmp(back.data(), host, bytes) == 0, "moe_stream_expert: bytes differ");
    // usage errors surface as the reference's UsageError through check()
    bool threw = false;
    try {
        b200::check(moe_stream_expert(nullptr, host, bytes, copy, done));
    } catch (const UsageError&) {
        threw = true;
    }
    EXPECT(threw, "moe_stream_expert(nullptr) must raise UsageError");
    std::printf("moe_stream_expert       %zu bytes pinned H2D on a side stream: %s\n", bytes,
                std::memcmp(back.data(), host, bytes) == 0 ? "identical" : "DIFFERENT");
    cudaFreeHost(host);
    cudaFree(dev);
    cudaStreamDestroy(copy);
    cudaEventDestroy(done);
}

int main() {
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess || n == 0) {
        std::fprintf(stderr, "no CUDA device\n");
        return 2;
    }
    try {
        one_case("all resident", 1.0, ResidencyPolicy::static_policy(), 6);
        one_case("static, 40% resident", 0.4, ResidencyPolicy::static_policy(), 12);
        one_case("static, 0% resident", 0.0, ResidencyPolicy::static_policy(), 8);
        one_case("lru(3), 30% resident", 0.3, ResidencyPolicy::lru(3), 16);
        one_case("lru(5), 10% resident", 0.1, ResidencyPolicy::lru(5), 16);
        stream_expert_case();
    } catch (const std::exception& e) {
        std::fprintf(stderr, "FAIL: exception %s\n", e.what());
        return 1;
    }
    if (failures) {
        std::fprintf(stderr, "%d failure(s)\n", failures);
        return 1;
    }
    std::printf("boundary ok\n");
    return 0;
}
