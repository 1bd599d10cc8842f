// Drop-in for stagger/denoiser.hpp (denoiser.hpp:15-86).  On the B200 build the
// denoiser is a device backend selected by EngineConfig::backend: the
// reference's closed-form Gaussian model ("analytic", the parity denoiser) or
// the random-init UNet ("unet").  Batched evaluation happens inside
// StreamBatchEngine::tick / run_pipeline (one device call per tick); the
// backend object carries the reference's call accounting.
#pragma once

#include <cstdint>
#include <memory>
#include <string>

#include "stagger/core.hpp"

namespace stagger {

struct CallCounters {
    std::uint64_t calls = 0;
    std::uint64_t element_evals = 0;
};

class DenoiserBackend {
  public:
    explicit DenoiserBackend(std::string kind) : kind_(std::move(kind)) {}
    virtual ~DenoiserBackend() = default;
    const CallCounters& counters() const { return counters_; }
    void reset_counters() { counters_ = {}; }
    const std::string& kind() const { return kind_; }
    // engine hook: one batched device call of `rows` element evaluations
    void account(std::uint64_t rows) {
        counters_.calls += 1;
        counters_.element_evals += rows;
    }

  private:
    std::string kind_;
    CallCounters counters_;
};

class AnalyticGaussianModel : public DenoiserBackend {
  public:
    explicit AnalyticGaussianModel(double data_variance) : DenoiserBackend("analytic"), var_(data_variance) {
        if (!(data_variance > 0.0)) throw std::invalid_argument("AnalyticGaussianModel: data_variance must be > 0");
    }
    double data_variance() const { return var_; }

  private:
    double var_;
};

class UNetModel : public DenoiserBackend {
  public:
    UNetModel() : DenoiserBackend("unet") {}
};

inline std::shared_ptr<DenoiserBackend> make_backend(const EngineConfig& cfg) {
    if (cfg.backend == "analytic") return std::make_shared<AnalyticGaussianModel>(cfg.data_variance);
    if (cfg.backend == "unet") return std::make_shared<UNetModel>();
    throw std::invalid_argument("make_backend: unknown backend " + cfg.backend);
}

}  // namespace stagger
