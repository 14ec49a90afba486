// splidar/reconstruct.hpp — drop-in replacement (B200 build) for the
// reference's reconstruct.hpp:20-491: the configuration types with the
// reference's defaults, validation messages and key=value keys, and the RT3D
// pipeline on the GPU.
//
//   detail::matched_filter_peaks  reconstruct.hpp:120-189  rt3d_matched_filter_peaks
//   init_matched_filter           reconstruct.hpp:197-249  rt3d_init_matched_filter
//   palm_step                     reconstruct.hpp:300-435  rt3d_palm_step
//   reconstruct                   reconstruct.hpp:457-489  rt3d_reconstruct (one CUDA
//                                 graph per frame, every decision on the device)
//
// Results equal the reference's within the north star's tolerances (peaks
// and init bit for bit); see DESIGN.md §2.
#pragma once

#include "splidar/b200_device.hpp"
#include "splidar/cloud.hpp"
#include "splidar/config.hpp"
#include "splidar/cube.hpp"
#include "splidar/denoise.hpp"
#include "splidar/likelihood.hpp"
#include "splidar/parallel.hpp"
#include "splidar/sensor.hpp"
#include "splidar/spatial_index.hpp"

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdint>
#include <map>
#include <set>
#include <stdexcept>
#include <string>
#include <vector>

namespace splidar {

inline constexpr double kBackgroundFloor = 1e-6;

struct InitParams {
    int max_returns = 3;          // K
    double peak_threshold = 0.5;  // matched-filter response, photons
    int min_separation = 3;       // bins between accepted peaks

    void validate() const {
        if (max_returns < 1) throw std::invalid_argument("InitParams: max_returns >= 1");
        if (min_separation < 1) throw std::invalid_argument("InitParams: min_separation >= 1");
        if (peak_threshold < 0.0) throw std::invalid_argument("InitParams: peak_threshold >= 0");
    }
};

/// A fixed step or "auto" (curvature preconditioned); backtracking guards both.
struct StepSize {
    bool automatic = true;
    double value = 1.0;

    static StepSize parse(const std::string& text) {
        StepSize s;
        if (text == "auto") return s;
        s.automatic = false;
        s.value = KeyValueFile::to_double(text, "step size");
        if (s.value <= 0.0) throw FormatError("step size must be positive or 'auto'");
        return s;
    }
    std::string str() const { return automatic ? "auto" : std::to_string(value); }
};

enum class BackgroundMode { Identity, Fft };

struct ReconConfig {
    int max_iters = 50;
    double stop_tol = 1e-4;
    StepSize step_t, step_r, step_b;
    double backtrack_beta = 0.5;
    ApssParams apss;
    int knn_k = 9;
    double r_min = 0.0;
    BackgroundMode background_mode = BackgroundMode::Identity;
    double fft_cutoff = 0.5;
    InitParams init;

    void validate() const {
        if (max_iters < 1) throw std::invalid_argument("ReconConfig: max_iters >= 1");
        if (stop_tol < 0.0) throw std::invalid_argument("ReconConfig: stop_tol >= 0");
        if (backtrack_beta <= 0.0 || backtrack_beta >= 1.0)
            throw std::invalid_argument("ReconConfig: backtrack_beta in (0,1)");
        if (knn_k < 1) throw std::invalid_argument("ReconConfig: knn_k >= 1");
        if (r_min < 0.0) throw std::invalid_argument("ReconConfig: r_min >= 0");
        apss.validate();
        init.validate();
    }

    static ReconConfig from_kv(const KeyValueFile& kv) {
        ReconConfig c;
        c.max_iters = kv.get_int("max_iters", c.max_iters);
        c.stop_tol = kv.get_double("stop_tol", c.stop_tol);
        c.step_t = StepSize::parse(kv.get_string("step_t", "auto"));
        c.step_r = StepSize::parse(kv.get_string("step_r", "auto"));
        c.step_b = StepSize::parse(kv.get_string("step_b", "auto"));
        c.backtrack_beta = kv.get_double("backtrack_beta", c.backtrack_beta);
        c.apss.kernel_radius = kv.get_double("apss_radius", c.apss.kernel_radius);
        c.apss.min_neighbors = kv.get_int("apss_min_neighbors", c.apss.min_neighbors);
        c.apss.sphere_degeneracy_eps = kv.get_double("apss_degeneracy_eps", c.apss.sphere_degeneracy_eps);
        c.knn_k = kv.get_int("knn_k", c.knn_k);
        c.r_min = kv.get_double("r_min", c.r_min);
        const std::string mode = kv.get_string("background_mode", "identity");
        if (mode == "fft") c.background_mode = BackgroundMode::Fft;
        else if (mode != "identity")
            throw FormatError("ReconConfig: background_mode must be identity or fft");
        c.fft_cutoff = kv.get_double("fft_cutoff", c.fft_cutoff);
        c.init.max_returns = kv.get_int("init_max_returns", c.init.max_returns);
        c.init.peak_threshold = kv.get_double("init_peak_threshold", c.init.peak_threshold);
        c.init.min_separation = kv.get_int("init_min_separation", c.init.min_separation);
        c.validate();
        return c;
    }
    static ReconConfig from_file(const std::string& path) {
        return from_kv(KeyValueFile::parse_file(path));
    }
};

struct BlockDiagnostics {
    double step_used = 0.0;
    int backtracks = 0;
    double nll_after_grad = 0.0;
    double nll_after_denoise = 0.0;
};

struct StepDiagnostics {
    double nll_before = 0.0;
    double nll_after = 0.0;
    std::size_t points_before = 0;
    std::size_t points_after = 0;
    BlockDiagnostics depth, intensity, background;
};

struct ReconReport {
    int iterations = 0;
    double init_nll = 0.0;
    double final_nll = 0.0;
    std::size_t points = 0;
    std::vector<double> nll_trace;  // init, then after each iteration
    std::vector<StepDiagnostics> steps;
    double init_seconds = 0.0;      // device timers (%globaltimer / CUDA events)
    double iterate_seconds = 0.0;
    double total_seconds = 0.0;
};

struct ReconResult {
    PointCloud cloud;
    BackgroundImage background;
    ReconReport report;
};

namespace detail {

inline constexpr int kMaxBacktracks = 30;

struct Peak {
    double t = 0.0;         // sub-bin refined position
    double response = 0.0;  // matched-filter response, photons
    double mass = 0.0;      // photons in the IRF-support window
};

inline std::vector<Peak> matched_filter_peaks(const Event* eb, const Event* ee, const Irf& irf,
                                              int n_bins, int k, double threshold, int min_sep) {
    const rt3d_irf iv = b200::irf_view(irf);
    std::vector<rt3d_peak> buf(k > 0 ? static_cast<std::size_t>(k) : 0u);
    std::int32_t n = 0;
    b200::check(rt3d_matched_filter_peaks(b200::session(), reinterpret_cast<const rt3d_event*>(eb),
                                          static_cast<std::uint64_t>(ee - eb), &iv, n_bins, k,
                                          threshold, min_sep, buf.data(), &n));
    std::vector<Peak> out(static_cast<std::size_t>(n));
    for (int q = 0; q < n; ++q) out[q] = Peak{buf[q].t, buf[q].response, buf[q].mass};
    return out;
}

inline rt3d_recon_config to_c(const ReconConfig& c) {
    rt3d_recon_config r{};
    r.max_iters = c.max_iters;
    r.knn_k = c.knn_k;
    r.stop_tol = c.stop_tol;
    r.step_t_auto = c.step_t.automatic;
    r.step_r_auto = c.step_r.automatic;
    r.step_b_auto = c.step_b.automatic;
    r.background_mode = c.background_mode == BackgroundMode::Fft ? 1 : 0;
    r.step_t = c.step_t.value;
    r.step_r = c.step_r.value;
    r.step_b = c.step_b.value;
    r.backtrack_beta = c.backtrack_beta;
    r.apss = rt3d_apss_params{c.apss.kernel_radius, c.apss.sphere_degeneracy_eps,
                              c.apss.min_neighbors, 0};
    r.r_min = c.r_min;
    r.fft_cutoff = c.fft_cutoff;
    r.init = rt3d_init_params{c.init.max_returns, c.init.min_separation, c.init.peak_threshold};
    return r;
}

inline StepDiagnostics from_c(const rt3d_step_diag& d) {
    auto blk = [](const rt3d_block_diag& b) {
        BlockDiagnostics o;
        o.step_used = b.step_used;
        o.backtracks = b.backtracks;
        o.nll_after_grad = b.nll_after_grad;
        o.nll_after_denoise = b.nll_after_denoise;
        return o;
    };
    StepDiagnostics o;
    o.nll_before = d.nll_before;
    o.nll_after = d.nll_after;
    o.points_before = static_cast<std::size_t>(d.points_before);
    o.points_after = static_cast<std::size_t>(d.points_after);
    o.depth = blk(d.depth);
    o.intensity = blk(d.intensity);
    o.background = blk(d.background);
    return o;
}

}  // namespace detail

inline SceneState init_matched_filter(const PhotonCube& cube, const SensorModel& sensor,
                                      const InitParams& params) {
    params.validate();
    b200::set_scene(cube, sensor);
    const rt3d_init_params p{params.max_returns, params.min_separation, params.peak_threshold};
    b200::check(rt3d_init_matched_filter(b200::session(), &p));
    PointCloud cloud;
    BackgroundImage bg;
    b200::download(sensor.n_rows, sensor.n_cols, cloud, bg);
    return SceneState(std::move(cloud), std::move(bg), &sensor);
}

/// One PALM iteration in place (the state as init_matched_filter / an
/// earlier palm_step leaves it: pixel-ordered, points at fine-pixel centres).
inline StepDiagnostics palm_step(SceneState& state, const PhotonCube& cube, const ReconConfig& cfg) {
    cfg.validate();
    detail::upload_state(state, cube);
    const rt3d_recon_config c = detail::to_c(cfg);
    rt3d_step_diag d{};
    b200::check(rt3d_palm_step(b200::session(), &c, &d));
    b200::download(state.sensor->n_rows, state.sensor->n_cols, state.cloud, state.background);
    state.refresh();
    return detail::from_c(d);
}

inline ReconResult reconstruct(const PhotonCube& cube, const SensorModel& sensor,
                               const ReconConfig& cfg) {
    cfg.validate();
    b200::set_scene(cube, sensor);
    const rt3d_recon_config c = detail::to_c(cfg);
    rt3d_session* s = b200::session();
    b200::check(rt3d_reconstruct(s, &c));
    rt3d_report info{};
    b200::check(rt3d_report_info(s, &info));
    ReconResult out;
    ReconReport& r = out.report;
    r.iterations = info.iterations;
    r.init_nll = info.init_nll;
    r.final_nll = info.final_nll;
    r.points = static_cast<std::size_t>(info.points);
    r.init_seconds = info.init_seconds;
    r.iterate_seconds = info.iterate_seconds;
    r.total_seconds = info.total_seconds;
    r.nll_trace.resize(static_cast<std::size_t>(info.iterations) + 1);
    std::vector<rt3d_step_diag> steps(static_cast<std::size_t>(info.iterations));
    b200::check(rt3d_report_copy(s, r.nll_trace.data(), steps.data()));
    for (const rt3d_step_diag& d : steps) r.steps.push_back(detail::from_c(d));
    b200::download(sensor.n_rows, sensor.n_cols, out.cloud, out.background);
    return out;
}

}  // namespace splidar
