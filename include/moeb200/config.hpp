// config.hpp -- model / hardware / task descriptors of the MoE hot path.
//
// Same semantics as the reference's profiles module (profiles.hpp:29-100,
// profiles.cpp:66-256), re-implemented for the B200 engine, plus MoeShape,
// which the reference lacks (it carries byte sizes only, no d/f/g): the
// engine derives size_expert16_bytes = 6*d*f and quant_ratio = 128/33 from
// it so that expert_size(P4) equals the int4-g128 bytes the GPU allocates.
#pragma once

#include <cstdint>
#include <optional>
#include <stdexcept>
#include <string>
#include <string_view>
#include <utility>

namespace moeb200 {

using bytes_t = std::int64_t;

// Error taxonomy of errors.hpp:9-26; C-ABI status codes mirror the CLI exit
// codes of cli.hpp:7-8 (1 internal, 2 usage, 3 parse/validation, 4 infeasible).
struct ParseError : std::runtime_error {
    using std::runtime_error::runtime_error;
};
struct ValidationError : std::runtime_error {
    using std::runtime_error::runtime_error;
};
struct InfeasibleError : std::runtime_error {
    using std::runtime_error::runtime_error;
};
struct UsageError : std::runtime_error {
    using std::runtime_error::runtime_error;
};

enum class Precision { P4, P16 };
enum class NonexpertPrecision { P4, P8, P16 };
enum class Preference { Throughput, Quality };

// profiles.hpp:29-43.  Defaults: 32 layers x 8 experts, top-2, 336 MB bf16
// experts, 3.16 GB non-expert, latencies calibrated to 13.00 tok/s.
struct ModelProfile {
    int num_layers = 32;
    int experts_per_layer = 8;
    int top_k = 2;
    bytes_t size_nonexpert_bytes = 3'160'000'000;
    bytes_t size_expert16_bytes = 336'000'000;
    double quant_ratio = 4.0;
    double compute_latency16_s = 0.9 / (13.0 * 32.0 * 2.0);
    double compute_penalty4 = 1.15;
    double nonexpert_latency_s = 0.1 / 13.0;

    int num_experts() const { return num_layers * experts_per_layer; }
    friend bool operator==(const ModelProfile&, const ModelProfile&) = default;
};

// profiles.hpp:45-52
struct HardwareProfile {
    bytes_t gpu_mem_bytes = 80'000'000'000;
    double transfer_bw_bytes_per_s = 336'000'000.0 / 0.02735;
    friend bool operator==(const HardwareProfile&, const HardwareProfile&) = default;
};

// profiles.hpp:55-59
struct TaskRequest {
    Preference preference = Preference::Throughput;
    std::optional<int> n4_target;
    uint64_t seed = 0;
};

// Tensor shape of one expert (new; the reference has byte sizes only).
struct MoeShape {
    int d_model = 4096;
    int d_ffn = 14336;
    int group = 128;
    friend bool operator==(const MoeShape&, const MoeShape&) = default;
};

ModelProfile mixtral_sec41();
ModelProfile mixtral_table1();
HardwareProfile default_hardware();

// Profile whose byte sizes are exactly what the engine allocates for `shape`:
// bf16 expert = 3*d*f*2, int4-g128 expert = 3*d*f/2 + 3*d*f/128*2.
ModelProfile profile_for_shape(const MoeShape& shape, int num_layers, int experts_per_layer,
                               int top_k, bytes_t size_nonexpert_bytes);
bytes_t expert_bytes_bf16(const MoeShape& shape);
bytes_t expert_bytes_int4(const MoeShape& shape);

void validate_profile(const ModelProfile& profile);
void validate_hardware(const HardwareProfile& hw);
void validate_task(const TaskRequest& task, const ModelProfile& profile);
void validate_shape(const MoeShape& shape);

std::pair<ModelProfile, HardwareProfile> load_profiles(std::string_view document);
bytes_t parse_size(std::string_view text);

bytes_t expert_size(const ModelProfile& profile, Precision precision);
bytes_t model_size(const ModelProfile& profile, int n4, NonexpertPrecision nonexpert_precision);
bytes_t uniform_model_size(const ModelProfile& profile, NonexpertPrecision precision);

uint64_t profile_fingerprint(const ModelProfile& profile);
std::string fingerprint_hex(uint64_t fingerprint);

}  // namespace moeb200
