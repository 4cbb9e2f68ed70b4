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
// There is no JSON library dependency: the schema is small enough for the
// recursive-descent parser below.
#include <cctype>
#include <cstdlib>
#include <string>
#include <string_view>
#include <vector>

#include "moeb200/config.hpp"
#include "moeb200/planner.hpp"

namespace moeb200 {

namespace {

constexpr const char* kPlanFormat = "moeserve.plan.v1";

struct JVal {
    enum Kind { Null, Bool, Num, Str, Arr, Obj } kind = Null;
    double num = 0.0;
    long long inum = 0;
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
    size_t i = 0;
    [[noreturn]] void fail(const std::string& what) const {
        throw ParseError("plan file: " + what + " at offset " + std::to_string(i));
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
            const size_t j = i;
            if (s[i] == '-' || s[i] == '+') ++i;
            bool frac = false;
            while (i < s.size() && (std::isdigit(static_cast<unsigned char>(s[i])) || s[i] == '.' || s[i] == 'e' ||
                                    s[i] == 'E' || s[i] == '-' || s[i] == '+')) {
                frac = frac || s[i] == '.' || s[i] == 'e' || s[i] == 'E';
                ++i;
            }
            if (i == j) fail("unexpected character");
            const std::string num(s.substr(j, i - j));
            v.kind = JVal::Num;
            v.num = std::strtod(num.c_str(), nullptr);
            v.is_int = !frac;
            if (!frac) v.inum = std::strtoll(num.c_str(), nullptr, 10);
        }
        return v;
    }
};

long long as_int(const JVal& v, const char* what) {
    if (v.kind != JVal::Num || !v.is_int) throw ParseError(std::string("plan file: ") + what + " must be an integer");
    return v.inum;
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

PlacementPlan read_plan(std::string_view document, const ModelProfile& profile) {
    Parser p{document};
    const JVal j = p.value();
    const JVal* fmt = j.kind == JVal::Obj ? j.get("format") : nullptr;
    if (fmt == nullptr || fmt->kind != JVal::Str || fmt->str != kPlanFormat)
        throw ParseError(std::string("plan file: missing or wrong format marker (expected '") + kPlanFormat + "')");
    const std::string expected = fingerprint_hex(profile_fingerprint(profile));
    const JVal* fp = j.get("profile_fingerprint");
    const std::string got = fp && fp->kind == JVal::Str ? fp->str : std::string();
    if (got != expected)
        throw ValidationError("plan was built for a different profile (fingerprint " + got + ", expected " +
                              expected + ")");
    const int E = profile.experts_per_layer, L = profile.num_layers, n = L * E;
    PlacementPlan plan;
    if (const JVal* v = j.get("seed")) plan.seed = static_cast<uint64_t>(as_int(*v, "seed"));
    if (const JVal* v = j.get("swap_slot_bytes")) plan.swap_slot_bytes = as_int(*v, "swap_slot_bytes");
    const JVal* ex = j.get("experts");
    if (ex == nullptr || ex->kind != JVal::Arr) throw ParseError("plan file: missing experts array");
    plan.entries.resize(static_cast<size_t>(n));
    std::vector<char> seen(static_cast<size_t>(n), 0);
    for (const JVal& row : ex->arr) {
        if (row.kind != JVal::Arr || row.arr.size() != 4)
            throw ParseError("plan file: expert rows must be [layer, slot, precision, location]");
        const long long layer = as_int(row.arr[0], "layer"), slot = as_int(row.arr[1], "slot");
        if (layer < 0 || layer >= L || slot < 0 || slot >= E)
            throw ValidationError("plan file: expert (" + std::to_string(layer) + "," + std::to_string(slot) +
                                  ") out of range");
        const size_t idx = static_cast<size_t>(layer * E + slot);
        if (seen[idx])
            throw ValidationError("plan file: duplicate entry for expert (" + std::to_string(layer) + "," +
                                  std::to_string(slot) + ")");
        seen[idx] = 1;
        const JVal &pr = row.arr[2], &lo = row.arr[3];
        if (pr.kind != JVal::Str || (pr.str != "p4" && pr.str != "p16"))
            throw ParseError("plan file: unknown precision '" + pr.str + "'");
        if (lo.kind != JVal::Str || (lo.str != "gpu" && lo.str != "cpu"))
            throw ParseError("plan file: unknown location '" + lo.str + "'");
        plan.entries[idx] = {pr.str == "p4" ? Precision::P4 : Precision::P16,
                             lo.str == "gpu" ? Location::GPU : Location::CPU};
    }
    for (int i = 0; i < n; ++i)
        if (!seen[static_cast<size_t>(i)])
            throw ValidationError("plan file: missing entry for expert (" + std::to_string(i / E) + "," +
                                  std::to_string(i % E) + ")");
    return plan;
}

}  // namespace moeb200
