// Drop-in for stagger/ssf.hpp (ssf.hpp:14-42): the stochastic similarity gate
// on the device.  Payloads are u8-valued frames (0..255 per element); the
// cosine sums are exact integers on the GPU, so decisions are bit-identical
// to the reference's fp64 gate on the same values.
#pragma once

#include <cstdint>
#include <optional>
#include <vector>

#include "stagger/rng.hpp"

namespace stagger {

inline double skip_probability(double sim, double eta) {  // ssf.cpp:26-32
    if (!(eta >= 0.0 && eta < 1.0)) throw std::invalid_argument("skip_probability: eta must lie in [0,1)");
    const double p = (sim - eta) / (1.0 - eta);
    if (p <= 0.0) return 0.0;
    return p >= 1.0 ? 1.0 : p;
}

enum class GateDecision { process, skip };

namespace detail {
inline std::vector<std::uint8_t> to_u8(const Latent& v) {
    std::vector<std::uint8_t> o(v.size());
    for (size_t i = 0; i < v.size(); ++i) {
        const double x = v[i];
        if (!(x >= 0.0 && x <= 255.0) || x != std::floor(x))
            throw std::invalid_argument("device SSF: frame payloads must be u8-valued (0..255)");
        o[i] = static_cast<std::uint8_t>(x);
    }
    return o;
}
}  // namespace detail

class SsfState {
  public:
    // max_skip <= 0: the reference gate; > 0: the forced-process extension.
    SsfState(double eta, Rng rng, int max_skip = 0, int device = 0)
        : eta_(eta), seed_(rng.seed()), max_skip_(max_skip), device_(device) {
        if (!(eta >= 0.0 && eta < 1.0)) throw std::invalid_argument("SsfState: eta must lie in [0,1)");
        if (!rng.fresh()) throw std::invalid_argument("SsfState (device): pass a freshly seeded Rng");
    }
    ~SsfState() {
        if (h_) sdx_ssf_destroy(h_);
    }
    SsfState(const SsfState&) = delete;
    SsfState& operator=(const SsfState&) = delete;

    GateDecision gate(const Frame& frame) {
        const auto u8 = detail::to_u8(frame.payload);
        if (!h_) detail::check(sdx_ssf_create(eta_, seed_, max_skip_, static_cast<int64_t>(u8.size()), device_, &h_));
        else if (static_cast<int64_t>(u8.size()) != bytes_)
            throw std::invalid_argument("cosine_similarity: dimension mismatch");
        bytes_ = static_cast<int64_t>(u8.size());
        int d = 0;
        detail::check(sdx_ssf_gate(h_, u8.data(), 1, &d, nullptr));
        ref_ = d == SDX_GATE_PROCESS ? std::optional<Frame>(frame) : ref_;
        return d == SDX_GATE_SKIP ? GateDecision::skip : GateDecision::process;
    }

    double eta() const { return eta_; }
    std::uint64_t examined() const { return counters().first; }
    std::uint64_t skipped() const { return counters().second; }
    const std::optional<Frame>& ref_frame() const { return ref_; }

  private:
    std::pair<std::uint64_t, std::uint64_t> counters() const {
        std::uint64_t a = 0, b = 0;
        if (h_) detail::check(sdx_ssf_counters(h_, &a, &b));
        return {a, b};
    }
    double eta_;
    std::uint64_t seed_;
    int max_skip_;
    int device_;
    sdx_ssf* h_ = nullptr;
    int64_t bytes_ = 0;
    std::optional<Frame> ref_;
};

}  // namespace stagger
