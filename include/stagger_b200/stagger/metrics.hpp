// Drop-in for stagger/metrics.hpp (metrics.hpp:12-46): MetricsReport schema v1
// and its stable JSON rendering (field order and 2-space layout of
// report_to_json, metrics.cpp:10-36; doubles in shortest round-trip form).
#pragma once

#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <fstream>
#include <sstream>
#include <stdexcept>
#include <string>

namespace stagger {

struct MetricsReport {
    int schema_version = 1;
    std::string mode = "deterministic";
    bool incomplete = false;
    std::string error;
    std::uint64_t frames_in = 0, frames_out = 0, duplicates = 0, stale_skips = 0, input_drops = 0, output_drops = 0;
    std::uint64_t ticks = 0, denoiser_calls = 0, element_evals = 0;
    double work_units = 0.0;
    std::uint64_t ssf_examined = 0, ssf_skipped = 0;
    double skip_rate = 0.0;
    double latency_ticks_mean = 0.0;
    std::int64_t latency_ticks_min = 0, latency_ticks_max = 0;
    double mean_frame_time_ms = 0.0, throughput_fps = 0.0, wall_ms = 0.0;
};

namespace detail {
inline std::string json_double(double v) {
    char buf[64];
    for (int prec = 1; prec <= 17; ++prec) {
        std::snprintf(buf, sizeof buf, "%.*g", prec, v);
        if (std::strtod(buf, nullptr) == v) break;
    }
    std::string s(buf);
    if (s.find_first_of(".eEn") == std::string::npos) s += ".0";
    return s;
}
inline std::string json_string(const std::string& s) {
    std::string o = "\"";
    for (char c : s) {
        if (c == '"' || c == '\\') o += '\\', o += c;
        else if (c == '\n') o += "\\n";
        else o += c;
    }
    return o + "\"";
}
}  // namespace detail

inline std::string report_to_json(const MetricsReport& r) {
    std::ostringstream o;
    auto kv = [&](const char* k, const std::string& v, bool last = false) {
        o << "  \"" << k << "\": " << v << (last ? "\n" : ",\n");
    };
    o << "{\n";
    kv("schema_version", std::to_string(r.schema_version));
    kv("mode", detail::json_string(r.mode));
    kv("incomplete", r.incomplete ? "true" : "false");
    kv("error", detail::json_string(r.error));
    kv("frames_in", std::to_string(r.frames_in));
    kv("frames_out", std::to_string(r.frames_out));
    kv("duplicates", std::to_string(r.duplicates));
    kv("stale_skips", std::to_string(r.stale_skips));
    kv("input_drops", std::to_string(r.input_drops));
    kv("output_drops", std::to_string(r.output_drops));
    kv("ticks", std::to_string(r.ticks));
    kv("denoiser_calls", std::to_string(r.denoiser_calls));
    kv("element_evals", std::to_string(r.element_evals));
    kv("work_units", detail::json_double(r.work_units));
    kv("ssf_examined", std::to_string(r.ssf_examined));
    kv("ssf_skipped", std::to_string(r.ssf_skipped));
    kv("skip_rate", detail::json_double(r.skip_rate));
    kv("latency_ticks_mean", detail::json_double(r.latency_ticks_mean));
    kv("latency_ticks_min", std::to_string(r.latency_ticks_min));
    kv("latency_ticks_max", std::to_string(r.latency_ticks_max));
    kv("mean_frame_time_ms", detail::json_double(r.mean_frame_time_ms));
    kv("throughput_fps", detail::json_double(r.throughput_fps));
    kv("wall_ms", detail::json_double(r.wall_ms), true);
    o << "}\n";
    return o.str();
}

inline void write_report(const MetricsReport& report, const std::string& path) {
    std::ofstream out(path, std::ios::binary);
    if (!out) throw std::runtime_error("write_report: cannot open " + path);
    out << report_to_json(report);
}

}  // namespace stagger
