// serialize.cpp -- placement-plan artifact I/O.
//
// The engine reads and writes plans in the reference's own canonical JSON,
// `moeserve.plan.v1` (serialize.cpp:99-149): a format marker, the profile
// fingerprint, the seed, swap_slot_bytes, and one [layer, slot, "p4"|"p16",
// "gpu"|"cpu"] row per expert.
//
// - The writer reproduces nlohmann's dump(2) layout byte for byte
//   (tests/test_planner_parity.py compares it with the reference library).
// - The reader accepts any JSON layout of the same schema and applies the
//   reference's checks:
//   - format marker -> ParseError (serialize.cpp:31-35);
//   - fingerprint -> ValidationError (:37-43);
//   - rows [layer, slot, precision, location] -> ParseError (:131-133);
//   - duplicate / missing experts -> ValidationError (:135-147).
// There is no JSON library dependency: the schemas are small enough for the
// recursive-descent parser below.  It follows nlohmann/json 3.11.3, which the
// reference parses with: strict JSON numbers, no trailing content; get<int>()
// on a number or boolean converts (floats truncate), on anything else it is a
// type error -- an internal error (exit 1) in the reference CLI, here a
// std::runtime_error (MOE_ERR_INTERNAL).
//
// Also the reconfiguration artifact moeserve.reconfig.v1 (serialize.cpp:160-206)
// and the SimReport table / JSON (serialize.cpp:218-243).  Doubles are written
// as nlohmann does: shortest round-trip digits, fixed notation for decimal
// exponents -4 < n <= 15 (".0" on integral values), else d.ddde+XX.
#include <cctype>
#include <cerrno>
#include <charconv>
#include <cmath>
#include <cstdlib>
#include <stdexcept>
#include <string>
#include <string_view>
#include <vector>

#include "moeb200/config.hpp"
#include "moeb200/planner.hpp"
#include "moeb200/pareto.hpp"
#include "moeb200/serialize.hpp"

namespace moeb200 {

namespace {

constexpr const char* kPlanFormat = "moeserve.plan.v1";

struct JVal {
    enum Kind { Null, Bool, Num, Str, Arr, Obj } kind = Null;
    double num = 0.0;
    unsigned long long mag = 0;  // integer magnitude (is_int)
    bool neg = false;
    bool is_int = false;
    bool b = false;
    std::string str;
    std::vector<JVal> arr;
    std::vector<std::pair<std::string, JVal>> obj;
    const JVal* get(const std::string& k) const {
        for (const auto& kv : obj)
            if (kv.first == k) return &kv.second;
        return nullptr;
    }
};

struct Parser {
    std::string_view s;
    const char* what;
    size_t i = 0;
    [[noreturn]] void fail(const std::string& msg) const {
        throw ParseError(std::string(what) + ": " + msg + " at offset " + std::to_string(i));
    }
    void ws() {
        while (i < s.size() && std::isspace(static_cast<unsigned char>(s[i]))) ++i;
    }
    bool eat(char c) {
        ws();
        if (i < s.size() && s[i] == c) {
            ++i;
            return true;
        }
        return false;
    }
    std::string string_lit() {
        if (!eat('"')) fail("expected a string");
        std::string out;
        while (i < s.size() && s[i] != '"') {
            if (s[i] == '\\') {
                if (++i >= s.size()) break;
                const char e = s[i];
                out.push_back(e == 'n' ? '\n' : e == 't' ? '\t' : e);
            } else {
                out.push_back(s[i]);
            }
            ++i;
        }
        if (i >= s.size()) fail("unterminated string");
        ++i;
        return out;
    }
    JVal value() {
        ws();
        if (i >= s.size()) fail("unexpected end of document");
        JVal v;
        const char c = s[i];
        if (c == '{') {
            ++i;
            v.kind = JVal::Obj;
            if (eat('}')) return v;
            do {
                std::string k = string_lit();
                if (!eat(':')) fail("expected ':'");
                v.obj.emplace_back(std::move(k), value());
            } while (eat(','));
            if (!eat('}')) fail("expected '}'");
        } else if (c == '[') {
            ++i;
            v.kind = JVal::Arr;
            if (eat(']')) return v;
            do v.arr.push_back(value());
            while (eat(','));
            if (!eat(']')) fail("expected ']'");
        } else if (c == '"') {
            v.kind = JVal::Str;
            v.str = string_lit();
        } else if (s.compare(i, 4, "true") == 0 || s.compare(i, 5, "false") == 0) {
            v.kind = JVal::Bool;
            v.b = s[i] == 't';
            i += v.b ? 4 : 5;
        } else if (s.compare(i, 4, "null") == 0) {
            i += 4;
        } else {
            // RFC 8259 number: -?(0|[1-9][0-9]*)(.[0-9]+)?([eE][+-]?[0-9]+)?
            const size_t j = i;
            auto digits = [&]() {
                const size_t k = i;
                while (i < s.size() && std::isdigit(static_cast<unsigned char>(s[i]))) ++i;
                return i > k;
            };
            if (s[i] == '-') ++i;
            if (i < s.size() && s[i] == '0') ++i;
            else if (!digits()) fail("unexpected character");
            bool frac = false;
            if (i < s.size() && s[i] == '.') {
                ++i;
                frac = true;
                if (!digits()) fail("expected digits after '.'");
            }
            if (i < s.size() && (s[i] == 'e' || s[i] == 'E')) {
                ++i;
                frac = true;
                if (i < s.size() && (s[i] == '+' || s[i] == '-')) ++i;
                if (!digits()) fail("expected exponent digits");
            }
            const std::string num(s.substr(j, i - j));
            v.kind = JVal::Num;
            v.num = std::strtod(num.c_str(), nullptr);
            v.neg = num[0] == '-';
            if (!frac) {
                errno = 0;
                v.mag = std::strtoull(num.c_str() + (v.neg ? 1 : 0), nullptr, 10);
                // nlohmann keeps integers that fit int64 / uint64, else a float
                v.is_int = errno == 0 && (!v.neg || v.mag <= 9223372036854775808ull);
            }
        }
        return v;
    }
};

[[noreturn]] void type_error(const char* want, const JVal& v) {
    static const char* names[] = {"null", "boolean", "number", "string", "array", "object"};
    throw std::runtime_error(std::string("[json.exception.type_error.302] type must be ") + want + ", but is " +
                             names[v.kind]);
}

// nlohmann get<T>() for arithmetic T: numbers and booleans convert
template <class T>
T num_as(const JVal& v) {
    if (v.kind == JVal::Bool) return static_cast<T>(v.b);
    if (v.kind != JVal::Num) type_error("number", v);
    if (!v.is_int) return static_cast<T>(v.num);
    return v.neg ? static_cast<T>(-static_cast<long long>(v.mag)) : static_cast<T>(v.mag);
}

const std::string& str_of(const JVal& v) {
    if (v.kind != JVal::Str) type_error("string", v);
    return v.str;
}

JVal parse_doc(std::string_view doc, const char* what) {
    Parser p{doc, what};
    JVal j = p.value();
    p.ws();
    if (p.i != doc.size()) p.fail("unexpected trailing content");
    return j;
}

}  // namespace

std::string write_plan(const PlacementPlan& plan, const ModelProfile& profile) {
    const int E = profile.experts_per_layer;
    std::string out;
    out += "{\n  \"format\": \"";
    out += kPlanFormat;
    out += "\",\n  \"profile_fingerprint\": \"" + fingerprint_hex(profile_fingerprint(profile)) + "\",\n";
    out += "  \"seed\": " + std::to_string(plan.seed) + ",\n";
    out += "  \"swap_slot_bytes\": " + std::to_string(plan.swap_slot_bytes) + ",\n";
    out += "  \"experts\": [";
    for (size_t i = 0; i < plan.entries.size(); ++i) {
        const ExpertState& st = plan.entries[i];
        out += i ? ",\n    [\n" : "\n    [\n";
        out += "      " + std::to_string(static_cast<int>(i) / E) + ",\n";
        out += "      " + std::to_string(static_cast<int>(i) % E) + ",\n";
        out += std::string("      \"") + (st.precision == Precision::P4 ? "p4" : "p16") + "\",\n";
        out += std::string("      \"") + (st.location == Location::GPU ? "gpu" : "cpu") + "\"\n    ]";
    }
    out += plan.entries.empty() ? "]\n}\n" : "\n  ]\n}\n";
    return out;
}

namespace {

void check_format(const JVal& j, const char* expected, const char* what) {
    const JVal* fmt = j.kind == JVal::Obj ? j.get("format") : nullptr;
    if (fmt == nullptr || fmt->kind != JVal::Str || fmt->str != expected)
        throw ParseError(std::string(what) + ": missing or wrong format marker (expected '" + expected + "')");
}

void check_fingerprint(const JVal& j, const ModelProfile& profile, const char* what) {
    const std::string expected = fingerprint_hex(profile_fingerprint(profile));
    const JVal* fp = j.get("profile_fingerprint");
    const std::string got = fp ? str_of(*fp) : std::string();
    if (got != expected)
        throw ValidationError(std::string(what) + " was built for a different profile (fingerprint " + got +
                              ", expected " + expected + ")");
}

Precision precision_word(const JVal& v, const char* what) {
    const std::string& w = str_of(v);
    if (w == "p4") return Precision::P4;
    if (w == "p16") return Precision::P16;
    throw ParseError(std::string(what) + ": unknown precision '" + w + "'");
}

Location location_word(const JVal& v, const char* what) {
    const std::string& w = str_of(v);
    if (w == "gpu") return Location::GPU;
    if (w == "cpu") return Location::CPU;
    throw ParseError(std::string(what) + ": unknown location '" + w + "'");
}

constexpr const char* kReconfigFormat = "moeserve.reconfig.v1";
constexpr const char* kActionWord[] = {"offload", "fetch", "quantize", "dequantize"};

}  // namespace

PlacementPlan read_plan(std::string_view document, const ModelProfile& profile) {
    const JVal j = parse_doc(document, "plan file");
    check_format(j, kPlanFormat, "plan file");
    check_fingerprint(j, profile, "plan");
    const int n = profile.num_experts();
    PlacementPlan plan;
    if (const JVal* v = j.get("seed")) plan.seed = num_as<uint64_t>(*v);
    if (const JVal* v = j.get("swap_slot_bytes")) plan.swap_slot_bytes = num_as<bytes_t>(*v);
    const JVal* ex = j.get("experts");
    if (ex == nullptr || ex->kind != JVal::Arr) throw ParseError("plan file: missing experts array");
    plan.entries.resize(static_cast<size_t>(n));
    std::vector<char> seen(static_cast<size_t>(n), 0);
    for (const JVal& row : ex->arr) {
        if (row.kind != JVal::Arr || row.arr.size() != 4)
            throw ParseError("plan file: expert rows must be [layer, slot, precision, location]");
        const ExpertId id{num_as<int>(row.arr[0]), num_as<int>(row.arr[1])};
        const size_t idx = static_cast<size_t>(expert_index(profile, id));  // bounds: ValidationError
        if (seen[idx])
            throw ValidationError("plan file: duplicate entry for expert (" + std::to_string(id.layer) + "," +
                                  std::to_string(id.slot) + ")");
        seen[idx] = 1;
        plan.entries[idx] = {precision_word(row.arr[2], "plan file"), location_word(row.arr[3], "plan file")};
    }
    for (int i = 0; i < n; ++i)
        if (!seen[static_cast<size_t>(i)]) {
            const ExpertId id = expert_id_at(profile, i);
            throw ValidationError("plan file: missing entry for expert (" + std::to_string(id.layer) + "," +
                                  std::to_string(id.slot) + ")");
        }
    return plan;
}

std::string json_double(double v) {
    if (!std::isfinite(v)) return "null";
    if (v == 0.0) return std::signbit(v) ? "-0.0" : "0.0";
    char buf[64];
    const auto r = std::to_chars(buf, buf + sizeof buf, std::fabs(v), std::chars_format::scientific);
    const std::string sci(buf, r.ptr);  // d[.ddd]e(+|-)XX, shortest round trip
    const size_t e = sci.find('e');
    std::string digits = sci.substr(0, 1) + (e > 1 ? sci.substr(2, e - 2) : std::string());
    const int k = static_cast<int>(digits.size());
    const int n = std::atoi(sci.c_str() + e + 1) + 1;  // decimal point position
    std::string out = v < 0 ? "-" : "";
    if (k <= n && n <= 15) {
        out += digits + std::string(static_cast<size_t>(n - k), '0') + ".0";
    } else if (0 < n && n <= 15) {
        out += digits.substr(0, static_cast<size_t>(n)) + "." + digits.substr(static_cast<size_t>(n));
    } else if (-4 < n && n <= 0) {
        out += "0." + std::string(static_cast<size_t>(-n), '0') + digits;
    } else {
        out += digits.substr(0, 1);
        if (k > 1) out += "." + digits.substr(1);
        int x = n - 1;
        out += x < 0 ? "e-" : "e+";
        x = x < 0 ? -x : x;
        out += (x < 10 ? "0" : "") + std::to_string(x);
    }
    return out;
}

std::string write_reconfig(const ReconfigPlan& plan, const ModelProfile& profile) {
    std::string out = "{\n  \"format\": \"";
    out += kReconfigFormat;
    out += "\",\n  \"profile_fingerprint\": \"" + fingerprint_hex(profile_fingerprint(profile)) + "\",\n";
    out += "  \"target_seed\": " + std::to_string(plan.target_seed) + ",\n";
    out += "  \"bytes_moved\": " + std::to_string(plan.bytes_moved) + ",\n";
    out += "  \"est_downtime_s\": " + json_double(plan.est_downtime_s) + ",\n";
    out += "  \"actions\": [";
    for (size_t i = 0; i < plan.actions.size(); ++i) {
        const ReconfigAction& a = plan.actions[i];
        out += i ? ",\n    [\n" : "\n    [\n";
        out += std::string("      \"") + kActionWord[static_cast<int>(a.kind)] + "\",\n";
        out += "      " + std::to_string(a.expert.layer) + ",\n";
        out += "      " + std::to_string(a.expert.slot) + ",\n";
        out += std::string("      \"") + (a.target_precision == Precision::P4 ? "p4" : "p16") + "\",\n";
        out += std::string("      \"") + (a.target_location == Location::GPU ? "gpu" : "cpu") + "\"\n    ]";
    }
    out += plan.actions.empty() ? "]\n}\n" : "\n  ]\n}\n";
    return out;
}

ReconfigPlan read_reconfig(std::string_view document, const ModelProfile& profile, const HardwareProfile& hw) {
    const JVal j = parse_doc(document, "reconfig file");
    check_format(j, kReconfigFormat, "reconfig file");
    check_fingerprint(j, profile, "reconfig plan");
    ReconfigPlan plan;
    if (const JVal* v = j.get("target_seed")) plan.target_seed = num_as<uint64_t>(*v);
    const JVal* acts = j.get("actions");
    if (acts == nullptr || acts->kind != JVal::Arr) throw ParseError("reconfig file: missing actions array");
    for (const JVal& row : acts->arr) {
        if (row.kind != JVal::Arr || row.arr.size() != 5)
            throw ParseError("reconfig file: action rows must be [kind, layer, slot, precision, location]");
        const std::string& w = str_of(row.arr[0]);
        int kind = -1;
        for (int q = 0; q < 4; ++q)
            if (w == kActionWord[q]) kind = q;
        if (kind < 0) throw ParseError("reconfig plan: unknown action kind '" + w + "'");
        ReconfigAction a;
        a.kind = static_cast<ActionKind>(kind);
        a.expert = ExpertId{num_as<int>(row.arr[1]), num_as<int>(row.arr[2])};
        expert_index(profile, a.expert);  // bounds: ValidationError
        a.target_precision = precision_word(row.arr[3], "reconfig file");
        a.target_location = location_word(row.arr[4], "reconfig file");
        plan.actions.push_back(a);
    }
    std::tie(plan.bytes_moved, plan.est_downtime_s) = estimate_cost(plan, profile, hw);
    if (const JVal* v = j.get("bytes_moved")) {
        const bytes_t stored = num_as<bytes_t>(*v);
        if (stored != plan.bytes_moved)
            throw ValidationError("reconfig file: stored bytes_moved " + std::to_string(stored) +
                                  " disagrees with the action list (" + std::to_string(plan.bytes_moved) + ")");
    }
    return plan;
}

std::string report_csv(const SimReport& r) {
    std::string out =
        "tokens,total_time_s,throughput_tps,activations,hits,hit_rate,bytes_transferred,transfer_time_s,"
        "compute_time_s,nonexpert_time_s\n";
    out += std::to_string(r.tokens) + ',' + format_double(r.total_time_s()) + ',' + format_double(r.throughput_tps()) +
           ',' + std::to_string(r.activations) + ',' + std::to_string(r.hits) + ',' + format_double(r.hit_rate()) + ',' +
           std::to_string(r.bytes_transferred) + ',' + format_double(static_cast<double>(r.transfer_ns) / 1e9) + ',' +
           format_double(static_cast<double>(r.compute_ns) / 1e9) + ',' +
           format_double(static_cast<double>(r.nonexpert_ns) / 1e9) + '\n';
    return out;
}

std::string report_json(const SimReport& r) {
    std::string out = "{\n";
    out += "  \"tokens\": " + std::to_string(r.tokens) + ",\n";
    out += "  \"total_time_s\": " + json_double(r.total_time_s()) + ",\n";
    out += "  \"throughput_tps\": " + json_double(r.throughput_tps()) + ",\n";
    out += "  \"activations\": " + std::to_string(r.activations) + ",\n";
    out += "  \"hits\": " + std::to_string(r.hits) + ",\n";
    out += "  \"hit_rate\": " + json_double(r.hit_rate()) + ",\n";
    out += "  \"bytes_transferred\": " + std::to_string(r.bytes_transferred) + ",\n";
    out += "  \"transfer_time_s\": " + json_double(static_cast<double>(r.transfer_ns) / 1e9) + ",\n";
    out += "  \"compute_time_s\": " + json_double(static_cast<double>(r.compute_ns) / 1e9) + ",\n";
    out += "  \"nonexpert_time_s\": " + json_double(static_cast<double>(r.nonexpert_ns) / 1e9) + "\n}\n";
    return out;
}

}  // namespace moeb200
