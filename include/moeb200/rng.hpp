// rng.hpp -- the determinism contract shared with the reference's file
// formats (rng.hpp:11-14 there): xoshiro256** (Blackman & Vigna) seeded by
// four splitmix64 outputs, modulo bounded draws, partial Fisher-Yates subset.
// Plans and traces built with the same seed are bit-identical to the
// reference's (checked against oracle/_ref in tests/test_planner_parity.py).
#pragma once

#include <cstdint>
#include <vector>

namespace moeb200 {

class Xoshiro256 {
  public:
    explicit Xoshiro256(uint64_t seed) {
        uint64_t sm = seed;
        for (int i = 0; i < 4; ++i) {
            sm += 0x9E3779B97F4A7C15ULL;
            uint64_t z = sm;
            z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
            z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
            s_[i] = z ^ (z >> 31);
        }
    }

    uint64_t next() {
        const uint64_t out = rotl(s_[1] * 5u, 7) * 9u;
        const uint64_t shifted = s_[1] << 17;
        s_[2] ^= s_[0];
        s_[3] ^= s_[1];
        s_[1] ^= s_[2];
        s_[0] ^= s_[3];
        s_[2] ^= shifted;
        s_[3] = rotl(s_[3], 45);
        return out;
    }

    uint64_t below(uint64_t n) { return next() % n; }

  private:
    static uint64_t rotl(uint64_t v, int r) { return (v << r) | (v >> (64 - r)); }
    uint64_t s_[4];
};

// Uniform n-subset of [0, count), in draw order (partial Fisher-Yates).
inline std::vector<int> draw_subset(int count, int n, Xoshiro256& gen) {
    std::vector<int> pool(static_cast<size_t>(count));
    for (int i = 0; i < count; ++i) pool[static_cast<size_t>(i)] = i;
    for (int i = 0; i < n; ++i) {
        const auto pick = static_cast<size_t>(i) + gen.below(static_cast<uint64_t>(count - i));
        const int tmp = pool[static_cast<size_t>(i)];
        pool[static_cast<size_t>(i)] = pool[pick];
        pool[pick] = tmp;
    }
    pool.resize(static_cast<size_t>(n));
    return pool;
}

}  // namespace moeb200
