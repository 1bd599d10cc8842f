// Drop-in for stagger/rng.hpp (rng.hpp:19-62).  Host RNG of the precompute
// (identical sample order: mt19937_64, 53-bit uniforms, Box-Muller cos-first).
#pragma once

#include <cmath>
#include <cstdint>
#include <random>

#include "stagger/core.hpp"

namespace stagger {

class Rng {
  public:
    explicit Rng(std::uint64_t seed) : engine_(seed), seed_(seed) {}
    std::uint64_t next_u64() {
        ++draws_;
        return engine_();
    }
    double uniform() { return static_cast<double>(next_u64() >> 11) * 0x1.0p-53; }
    double gaussian() {
        if (has_spare_) {
            has_spare_ = false;
            return spare_;
        }
        const double u1 = uniform();
        const double u2 = uniform();
        const double r = std::sqrt(-2.0 * std::log1p(-u1));
        const double a = 2.0 * 3.14159265358979323846 * u2;
        spare_ = r * std::sin(a);
        has_spare_ = true;
        return r * std::cos(a);
    }
    // B200 build: the device SSF stream restarts mt19937_64 from this seed, so an
    // Rng handed to SsfState must not have been drawn from yet.
    std::uint64_t seed() const { return seed_; }
    bool fresh() const { return draws_ == 0 && !has_spare_; }

  private:
    std::mt19937_64 engine_;
    std::uint64_t seed_;
    std::uint64_t draws_ = 0;
    double spare_ = 0.0;
    bool has_spare_ = false;
};

inline Latent sample_gaussian(Rng& rng, std::size_t d) {
    if (d == 0) throw std::invalid_argument("sample_gaussian: d must be >= 1");
    Latent out(d);
    for (auto& x : out) x = rng.gaussian();
    return out;
}

inline std::uint64_t derive_seed(std::uint64_t seed, std::uint64_t stream_tag) {
    return sdx_derive_seed(seed, stream_tag);
}

inline constexpr std::uint64_t kStreamNoiseCache = 1;
inline constexpr std::uint64_t kStreamSsf = 2;
inline constexpr std::uint64_t kStreamSource = 3;
inline constexpr std::uint64_t kStreamCondition = 4;

}  // namespace stagger
