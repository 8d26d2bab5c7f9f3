// Storage dtypes and the deterministic RNG (reference proj/include/hlm/tensor.hpp:20,86-131).
#pragma once

#include <cmath>
#include <cstdint>
#include <random>

namespace hlm {
inline namespace b200 {

// BF16 / FP32: the reference store dtypes (how build_store rounds the initial
// weights). The B200 store always keeps an FP32 master + FP32 Adam moments
// and a BF16 shadow for transfer; Dtype::BF16 additionally means the master
// starts bf16-exact (identical to the reference bf16-store init).
enum class Dtype : std::uint8_t { BF16 = 0, FP32 = 1 };

inline const char* dtype_name(Dtype d) { return d == Dtype::BF16 ? "bf16" : "fp32"; }

// mt19937 + Box-Muller, bit-compatible with the reference stream.
class Rng {
public:
    explicit Rng(std::uint64_t seed) : gen_(static_cast<std::mt19937::result_type>(seed)) {}
    float uniform() { return static_cast<float>(gen_() >> 8) * (1.0f / 16777216.0f); }
    float normal() {
        if (have_spare_) {
            have_spare_ = false;
            return spare_;
        }
        float u1;
        do {
            u1 = uniform();
        } while (u1 <= 1e-12f);
        const float u2 = uniform();
        const float r = std::sqrt(-2.0f * std::log(u1));
        const float a = 6.2831853071795864769f * u2;
        spare_ = r * std::sin(a);
        have_spare_ = true;
        return r * std::cos(a);
    }
    float trunc_normal(float sd) {
        float v;
        do {
            v = normal() * sd;
        } while (v < -2.0f * sd || v > 2.0f * sd);
        return v;
    }
    std::uint32_t next_u32() { return gen_(); }
    std::int32_t uniform_int(std::int32_t n) {
        return static_cast<std::int32_t>(gen_() % static_cast<std::uint32_t>(n));
    }

private:
    std::mt19937 gen_;
    bool have_spare_ = false;
    float spare_ = 0.0f;
};

}  // inline namespace b200
}  // namespace hlm
