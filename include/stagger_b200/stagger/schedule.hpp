// Drop-in for stagger/schedule.hpp (schedule.hpp:14-65): schedule types and
// build_schedule / lcm_coefficients.  The per-element transitions
// (forward_diffuse, predict_x0, consistency_step) run fused on the device
// inside StreamBatchEngine::tick and are not exposed as host vector ops.
#pragma once

#include <ostream>
#include <utility>
#include <vector>

#include "stagger/core.hpp"

namespace stagger {

struct ScheduleStep {
    int tau = 0;
    double alpha = 1.0;
    double beta = 0.0;
    bool is_terminal() const { return beta == 0.0; }
    static ScheduleStep terminal() { return ScheduleStep{0, 1.0, 0.0}; }
};

struct NoiseSchedule {
    std::vector<ScheduleStep> steps;
    int t_grid = 0;
    int n() const { return static_cast<int>(steps.size()); }
};

struct LcmParams {
    enum class Mode { exact, boundary_approx };
    double sigma_data = 0.5;
    double s = 10.0;
    Mode mode = Mode::exact;
};

inline NoiseSchedule build_schedule(int n, int t_grid, double entry_strength) {
    std::vector<sdx_step> buf(static_cast<size_t>(n > 0 ? n : 1));
    detail::check(sdx_build_schedule(n, t_grid, entry_strength, buf.data()), sdx_precompute_error());
    NoiseSchedule s;
    s.t_grid = t_grid;
    for (int i = 0; i < n; ++i) s.steps.push_back(ScheduleStep{buf[size_t(i)].tau, buf[size_t(i)].alpha, buf[size_t(i)].beta});
    return s;
}

inline std::pair<double, double> lcm_coefficients(const ScheduleStep& step, const LcmParams& p) {
    if (p.mode == LcmParams::Mode::boundary_approx) return step.tau == 0 ? std::pair{1.0, 0.0} : std::pair{0.0, 1.0};
    const double st = p.s * step.tau;
    const double sig2 = p.sigma_data * p.sigma_data;
    return {sig2 / (st * st + sig2), p.sigma_data * st / std::sqrt(sig2 + st * st)};
}

inline void dump_schedule_csv(const NoiseSchedule& schedule, std::ostream& os) {
    os << "i,tau,alpha,beta\n";
    os.precision(17);
    for (size_t i = 0; i < schedule.steps.size(); ++i) {
        const auto& s = schedule.steps[i];
        os << i << ',' << s.tau << ',' << s.alpha << ',' << s.beta << '\n';
    }
}

}  // namespace stagger
