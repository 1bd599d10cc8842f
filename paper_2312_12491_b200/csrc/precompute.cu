// Host-side precompute of the drop-in (PrecomputeCache, precompute.cpp:7-21):
// schedule (schedule.cpp:15-58), seed derivation (rng.cpp:14-20) and the
// mt19937_64 + Box-Muller noise stream (rng.hpp:19-49).  Runs once per config
// on the host in fp64 (libm log1p/sin/cos, like the reference, so the cached
// noise is bit-identical), then is uploaded to HBM by the engine/pipeline.
#include <cmath>
#include <random>
#include <string>
#include <vector>

#include "common.cuh"
#include "stagger_b200.h"

namespace {
thread_local std::string g_err_pc;

class HostRng {
  public:
    explicit HostRng(uint64_t seed) : eng_(seed) {}
    double uniform() { return static_cast<double>(eng_() >> 11) * 0x1.0p-53; }
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

  private:
    std::mt19937_64 eng_;
    double spare_ = 0.0;
    bool has_spare_ = false;
};

int fail(int code, const char* m) {
    g_err_pc = m;
    return code;
}
}  // namespace

extern "C" {

uint64_t sdx_derive_seed(uint64_t seed, uint64_t tag) {
    uint64_t z = seed + 0x9e3779b97f4a7c15ULL * (tag + 1);
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
}

const char* sdx_precompute_error(void) { return g_err_pc.c_str(); }

int sdx_build_schedule(int n, int t_grid, double entry, sdx_step* out) {
    if (n < 1) return fail(SDX_INVALID_ARGUMENT, "build_schedule: n must be >= 1");
    if (t_grid < 1) return fail(SDX_INVALID_ARGUMENT, "build_schedule: t_grid must be >= 1");
    if (n > t_grid) return fail(SDX_INVALID_ARGUMENT, "build_schedule: n exceeds t_grid");
    if (!(entry > 0.0 && entry <= 1.0))
        return fail(SDX_INVALID_ARGUMENT, "build_schedule: entry_strength must lie in (0,1]");
    const long tau0 = std::lround(entry * (t_grid - 1));
    if (n > tau0 + 1)
        return fail(SDX_INVALID_ARGUMENT, "build_schedule: n exceeds the usable range below the entry index");
    std::vector<double> table(static_cast<size_t>(t_grid));
    double prod = 1.0;
    for (int t = 0; t < t_grid; ++t) {
        const double frac = t_grid > 1 ? static_cast<double>(t) / (t_grid - 1) : 0.0;
        const double rate = 1e-4 + (2e-2 - 1e-4) * frac;
        prod *= 1.0 - rate;
        table[static_cast<size_t>(t)] = prod;
    }
    const double stride = static_cast<double>(tau0 + 1) / n;
    for (int i = 0; i < n; ++i) {
        const long tau = std::llround(static_cast<double>(tau0) - stride * i);
        out[i].tau = static_cast<int>(tau);
        out[i].alpha = table[static_cast<size_t>(tau)];
        out[i].beta = 1.0 - out[i].alpha;
        if (i > 0 && out[i].tau >= out[i - 1].tau)
            return fail(SDX_LOGIC_ERROR, "build_schedule: taus must strictly decrease");
    }
    return SDX_OK;
}

int sdx_sample_gaussian(uint64_t seed, int64_t d, double* out) {
    if (d < 1) return fail(SDX_INVALID_ARGUMENT, "sample_gaussian: d must be >= 1");
    HostRng r(seed);
    for (int64_t i = 0; i < d; ++i) out[i] = r.gaussian();
    return SDX_OK;
}

// n x d cached noise from Rng(derive_seed(seed, kStreamNoiseCache)).
int sdx_build_noise_cache(uint64_t seed, int n, int64_t d, double* out) {
    if (d < 1) return fail(SDX_INVALID_ARGUMENT, "sample_gaussian: d must be >= 1");
    HostRng r(sdx_derive_seed(seed, 1));
    for (int64_t i = 0; i < static_cast<int64_t>(n) * d; ++i) out[i] = r.gaussian();
    return SDX_OK;
}

}  // extern "C"
