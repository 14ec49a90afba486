// splidar/b200.hpp — drop-in B200 backend for splidar's reconstruction path.
//
// Include after the reference's own headers and call splidar::b200::X where
// the reference calls splidar::X: same argument types (PhotonCube,
// SensorModel, ReconConfig, SceneState, PointCloud, Grid2D ...), same result
// types, same exceptions.  Every function marshals its arguments into the
// plain C structs of rt3d.h, runs on the GPU behind an rt3d_session and copies
// the result back; there is no CPU fallback (no device -> b200::Error).
//
//   splidar::b200::reconstruct        <- splidar::reconstruct        reconstruct.hpp:308-340
//   splidar::b200::init_matched_filter<- splidar::init_matched_filter reconstruct.hpp:197-249
//   splidar::b200::matched_filter_peaks <- detail::matched_filter_peaks reconstruct.hpp:120-189
//   splidar::b200::palm_step          <- splidar::palm_step          reconstruct.hpp:300-435
//   splidar::b200::nll / grad_depth / grad_intensity / grad_background /
//                  block_curvatures   <- likelihood.hpp:136-333
//   splidar::b200::apss_project       <- splidar::apss_project       denoise.hpp:159-215
//   splidar::b200::knn_intensity_filter <- denoise.hpp:223-237
//   splidar::b200::prune              <- denoise.hpp:241-248
//   splidar::b200::fft_lowpass_filter / fft_background_denoise <- denoise.hpp:267-319
//   splidar::b200::baseline_xcorr     <- splidar::baseline_xcorr     eval.hpp:91-126
//   splidar::b200::evaluate           <- splidar::evaluate           eval.hpp:33-87
//   splidar::b200::encode_ply         <- splidar::encode_ply         io.hpp:162-179
//   splidar::b200::simulate_photons   <- simulate_cube's sampling    simulate.hpp:181-205
//
// The neighbour-search operators take the indexed cloud explicitly: the
// reference's SpatialIndex keeps its cloud private, and every reference call
// site indexes the cloud being filtered (reconstruct.hpp:355, :394), which is
// what the SpatialIndex overloads below assume.
#pragma once

#include "rt3d.h"

#include "splidar/cloud.hpp"
#include "splidar/config.hpp"
#include "splidar/cube.hpp"
#include "splidar/denoise.hpp"
#include "splidar/eval.hpp"
#include "splidar/likelihood.hpp"
#include "splidar/reconstruct.hpp"
#include "splidar/sensor.hpp"
#include "splidar/spatial_index.hpp"

#include <cstdint>
#include <memory>
#include <stdexcept>
#include <optional>
#include <string>
#include <vector>

namespace splidar::b200 {

/// CUDA / device failures (statuses with no reference exception type).
class Error : public std::runtime_error {
public:
    Error(rt3d_status st, const std::string& what) : std::runtime_error(what), status(st) {}
    rt3d_status status;
};

/// Status -> the exception the reference throws for the same condition.
inline void check(rt3d_status st) {
    if (st == RT3D_OK) return;
    std::string msg = rt3d_last_error();
    switch (st) {
    case RT3D_ERR_INVALID_ARGUMENT: throw std::invalid_argument(msg);
    case RT3D_ERR_FORMAT: throw FormatError(msg);
    case RT3D_ERR_OUT_OF_RANGE: throw std::out_of_range(msg);
    default: throw Error(st, msg);
    }
}

/// One device + one stream + resident buffers.  Reuse one per thread to keep
/// the device allocations warm across frames.
class Session {
public:
    explicit Session(int device = 0) {
        rt3d_session* s = nullptr;
        check(rt3d_session_create(device, &s));
        h_.reset(s);
    }
    rt3d_session* get() const { return h_.get(); }
    void synchronize() { check(rt3d_session_synchronize(get())); }

private:
    struct Del {
        void operator()(rt3d_session* s) const { rt3d_session_destroy(s); }
    };
    std::unique_ptr<rt3d_session, Del> h_;
};

/// The calling thread's session on device 0 (created on first use).
inline Session& default_session() {
    thread_local Session s(0);
    return s;
}

namespace detail {

inline rt3d_irf irf_view(const Irf& irf) {
    return rt3d_irf{irf.tau_min(), irf.dtau(), irf.samples().data(),
                    static_cast<std::uint64_t>(irf.samples().size())};
}

/// rt3d_sensor borrows the SensorModel's arrays; per_pixel keeps the IRF
/// views alive for the call.
struct SensorView {
    rt3d_sensor c{};
    std::vector<rt3d_irf> per_pixel;
    explicit SensorView(const SensorModel& s) {
        c.n_rows = s.n_rows;
        c.n_cols = s.n_cols;
        c.n_bins = s.n_bins;
        c.superres = s.superres;
        c.pixel_pitch = s.pixel_pitch;
        c.bin_resolution = s.bin_resolution;
        c.irf_shared = irf_view(s.irf_shared);
        for (const Irf& irf : s.irf_per_pixel) per_pixel.push_back(irf_view(irf));
        c.irf_per_pixel = per_pixel.empty() ? nullptr : per_pixel.data();
        c.gain = s.gain.data.data();
        c.dead = s.dead.data.data();
        if (s.gain.size() != std::size_t(s.n_rows) * s.n_cols ||
            s.dead.size() != std::size_t(s.n_rows) * s.n_cols)
            throw std::invalid_argument("SensorModel: gain/dead shape mismatch");
    }
};

static_assert(sizeof(Event) == sizeof(rt3d_event), "Event layout");

inline rt3d_cube cube_view(const PhotonCube& cube) {
    return rt3d_cube{cube.n_rows, cube.n_cols, cube.n_bins, 0, cube.bin_width_s,
                     cube.offsets.data(), reinterpret_cast<const rt3d_event*>(cube.events.data()),
                     static_cast<std::uint64_t>(cube.events.size())};
}

inline rt3d_point to_c(const Point& p) {
    rt3d_point q{};
    q.x = p.position.x();
    q.y = p.position.y();
    q.z = p.position.z();
    q.intensity = p.intensity;
    q.i = p.i;
    q.j = p.j;
    q.fi = p.fi;
    q.fj = p.fj;
    q.t = p.t;
    q.flags = p.flags;
    return q;
}

inline Point from_c(const rt3d_point& q) {
    Point p;
    p.position = Vec3(q.x, q.y, q.z);
    p.intensity = q.intensity;
    p.i = q.i;
    p.j = q.j;
    p.fi = q.fi;
    p.fj = q.fj;
    p.t = q.t;
    p.flags = q.flags;
    return p;
}

inline std::vector<rt3d_point> to_c(const PointCloud& c) {
    std::vector<rt3d_point> out(c.size());
    for (std::size_t n = 0; n < c.size(); ++n) out[n] = to_c(c[n]);
    return out;
}

inline PointCloud from_c(const std::vector<rt3d_point>& v) {
    PointCloud c;
    c.points.resize(v.size());
    for (std::size_t n = 0; n < v.size(); ++n) c.points[n] = from_c(v[n]);
    return c;
}

inline rt3d_init_params to_c(const InitParams& p) {
    return rt3d_init_params{p.max_returns, p.min_separation, p.peak_threshold};
}

inline rt3d_apss_params to_c(const ApssParams& p) {
    return rt3d_apss_params{p.kernel_radius, p.sphere_degeneracy_eps, p.min_neighbors, 0};
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
    r.apss = to_c(c.apss);
    r.r_min = c.r_min;
    r.fft_cutoff = c.fft_cutoff;
    r.init = to_c(c.init);
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

inline void set_scene(Session& s, const PhotonCube& cube, const SensorModel& sensor) {
    SensorView sv(sensor);
    check(rt3d_set_sensor(s.get(), &sv.c));
    rt3d_cube cv = cube_view(cube);
    check(rt3d_set_cube(s.get(), &cv));
}

inline void upload(Session& s, const SceneState& st, const PhotonCube& cube) {
    if (!st.sensor) throw std::invalid_argument("SceneState: null sensor");
    set_scene(s, cube, *st.sensor);
    std::vector<rt3d_point> pts = to_c(st.cloud);
    rt3d_state_view v{pts.data(), static_cast<std::uint64_t>(pts.size()),
                      st.background.data.data(), st.bucket_offsets.data(),
                      st.bucket_points.data()};
    check(rt3d_state_upload(s.get(), &v));
}

/// Session state -> (cloud, background).
inline void download(Session& s, int rows, int cols, PointCloud& cloud, BackgroundImage& bg) {
    std::uint64_t n = 0;
    check(rt3d_state_size(s.get(), &n));
    std::vector<rt3d_point> pts(n);
    bg = BackgroundImage(rows, cols, 0.0);
    check(rt3d_state_copy(s.get(), pts.data(), bg.data.data()));
    cloud = from_c(pts);
}

}  // namespace detail

// ---- full pipeline --------------------------------------------------------

inline ReconResult reconstruct(const PhotonCube& cube, const SensorModel& sensor,
                               const ReconConfig& cfg, Session& s = default_session()) {
    cfg.validate();
    detail::set_scene(s, cube, sensor);
    rt3d_recon_config c = detail::to_c(cfg);
    check(rt3d_reconstruct(s.get(), &c));
    rt3d_report info{};
    check(rt3d_report_info(s.get(), &info));
    ReconResult out;
    out.report.iterations = info.iterations;
    out.report.init_nll = info.init_nll;
    out.report.final_nll = info.final_nll;
    out.report.points = static_cast<std::size_t>(info.points);
    out.report.init_seconds = info.init_seconds;
    out.report.iterate_seconds = info.iterate_seconds;
    out.report.total_seconds = info.total_seconds;
    out.report.nll_trace.resize(std::size_t(info.iterations) + 1);
    std::vector<rt3d_step_diag> steps(info.iterations);
    check(rt3d_report_copy(s.get(), out.report.nll_trace.data(), steps.data()));
    for (const rt3d_step_diag& d : steps) out.report.steps.push_back(detail::from_c(d));
    detail::download(s, sensor.n_rows, sensor.n_cols, out.cloud, out.background);
    return out;
}

// ---- initialisation and baseline ----------------------------------------

inline SceneState init_matched_filter(const PhotonCube& cube, const SensorModel& sensor,
                                      const InitParams& params, Session& s = default_session()) {
    params.validate();
    detail::set_scene(s, cube, sensor);
    rt3d_init_params p = detail::to_c(params);
    check(rt3d_init_matched_filter(s.get(), &p));
    PointCloud cloud;
    BackgroundImage bg;
    detail::download(s, sensor.n_rows, sensor.n_cols, cloud, bg);
    return SceneState(std::move(cloud), std::move(bg), &sensor);
}

inline PointCloud baseline_xcorr(const PhotonCube& cube, const SensorModel& sensor,
                                 Session& s = default_session()) {
    detail::set_scene(s, cube, sensor);
    check(rt3d_baseline_xcorr(s.get()));
    PointCloud cloud;
    BackgroundImage bg;
    detail::download(s, sensor.n_rows, sensor.n_cols, cloud, bg);
    return cloud;
}

inline EvalResult evaluate(const PointCloud& est, const PointCloud& truth, double tau,
                           double pitch, Session& s = default_session()) {
    const std::vector<rt3d_point> e = detail::to_c(est), t = detail::to_c(truth);
    rt3d_eval r{};
    check(rt3d_evaluate(s.get(), e.data(), e.size(), t.data(), t.size(), tau, pitch, &r));
    EvalResult out;
    out.recall = r.recall;
    out.false_point_rate = r.false_point_rate;
    out.depth_rmse = r.depth_rmse;
    out.intensity_mae = r.intensity_mae;
    out.n_truth = r.n_truth;
    out.n_est = r.n_est;
    out.n_matched = r.n_matched;
    return out;
}

inline std::vector<splidar::detail::Peak> matched_filter_peaks(
    const Event* eb, const Event* ee, const Irf& irf, int n_bins, int k, double threshold,
    int min_sep, Session& s = default_session()) {
    rt3d_irf iv = detail::irf_view(irf);
    std::vector<rt3d_peak> buf(k > 0 ? std::size_t(k) : 0);
    std::int32_t n = 0;
    check(rt3d_matched_filter_peaks(s.get(), reinterpret_cast<const rt3d_event*>(eb),
                                    static_cast<std::uint64_t>(ee - eb), &iv, n_bins, k, threshold,
                                    min_sep, buf.data(), &n));
    std::vector<splidar::detail::Peak> out(n);
    for (int q = 0; q < n; ++q) out[q] = {buf[q].t, buf[q].response, buf[q].mass};
    return out;
}

// ---- likelihood ------------------------------------------------------------

inline double nll(const SceneState& state, const PhotonCube& cube, Session& s = default_session()) {
    detail::upload(s, state, cube);
    double v = 0.0;
    check(rt3d_nll(s.get(), &v));
    return v;
}

inline DepthGradient grad_depth(const SceneState& state, const PhotonCube& cube,
                                Session& s = default_session()) {
    detail::upload(s, state, cube);
    DepthGradient out;
    out.value.assign(state.cloud.size(), 0.0);
    std::vector<std::uint8_t> oog(state.cloud.size(), 0);
    check(rt3d_grad_depth(s.get(), out.value.data(), oog.data()));
    for (std::uint32_t n = 0; n < oog.size(); ++n)
        if (oog[n]) out.out_of_gate.push_back(n);
    return out;
}

inline std::vector<double> grad_intensity(const SceneState& state, const PhotonCube& cube,
                                          Session& s = default_session()) {
    detail::upload(s, state, cube);
    std::vector<double> out(state.cloud.size(), 0.0);
    check(rt3d_grad_intensity(s.get(), out.data()));
    return out;
}

inline Grid2D<double> grad_background(const SceneState& state, const PhotonCube& cube,
                                      Session& s = default_session()) {
    detail::upload(s, state, cube);
    Grid2D<double> out(state.sensor->n_rows, state.sensor->n_cols, 0.0);
    check(rt3d_grad_background(s.get(), out.data.data()));
    return out;
}

inline BlockCurvatures block_curvatures(const SceneState& state, const PhotonCube& cube,
                                        Session& s = default_session()) {
    detail::upload(s, state, cube);
    BlockCurvatures out;
    out.depth.assign(state.cloud.size(), 0.0);
    out.intensity.assign(state.cloud.size(), 0.0);
    out.background = Grid2D<double>(state.sensor->n_rows, state.sensor->n_cols, 0.0);
    check(rt3d_block_curvatures(s.get(), out.depth.data(), out.intensity.data(),
                                out.background.data.data()));
    return out;
}

// ---- one PALM iteration (state updated in place) ---------------------------

inline StepDiagnostics palm_step(SceneState& state, const PhotonCube& cube, const ReconConfig& cfg,
                                 Session& s = default_session()) {
    cfg.validate();
    detail::upload(s, state, cube);
    rt3d_recon_config c = detail::to_c(cfg);
    rt3d_step_diag d{};
    check(rt3d_palm_step(s.get(), &c, &d));
    PointCloud cloud;
    BackgroundImage bg;
    detail::download(s, state.sensor->n_rows, state.sensor->n_cols, cloud, bg);
    state.cloud = std::move(cloud);
    state.background = std::move(bg);
    state.refresh();
    return detail::from_c(d);
}

// ---- point-cloud denoisers ---------------------------------------------------

inline PointCloud apss_project(const PointCloud& cloud, const ApssParams& params,
                               const PointCloud& index_cloud, double index_cell,
                               Session& s = default_session()) {
    params.validate();
    std::vector<rt3d_point> in = detail::to_c(cloud), idx = detail::to_c(index_cloud);
    std::vector<rt3d_point> out(in.size());
    rt3d_apss_params p = detail::to_c(params);
    check(rt3d_apss_project(s.get(), in.data(), in.size(), &p, idx.data(), idx.size(), index_cell,
                            out.data()));
    return detail::from_c(out);
}

/// `index` must index `cloud` (as at every reference call site).
inline PointCloud apss_project(const PointCloud& cloud, const ApssParams& params,
                               const SpatialIndex& index, Session& s = default_session()) {
    return apss_project(cloud, params, cloud, index.cell_size(), s);
}

inline PointCloud knn_intensity_filter(const PointCloud& cloud, int k,
                                       const PointCloud& index_cloud, double index_cell,
                                       double radius, Session& s = default_session()) {
    std::vector<rt3d_point> in = detail::to_c(cloud), idx = detail::to_c(index_cloud);
    std::vector<rt3d_point> out(in.size());
    check(rt3d_knn_intensity_filter(s.get(), in.data(), in.size(), k, idx.data(), idx.size(),
                                    index_cell, radius, out.data()));
    return detail::from_c(out);
}

/// `index` must index `cloud` (as at every reference call site).
inline PointCloud knn_intensity_filter(const PointCloud& cloud, int k, const SpatialIndex& index,
                                       double radius, Session& s = default_session()) {
    return knn_intensity_filter(cloud, k, cloud, index.cell_size(), radius, s);
}

inline PointCloud prune(const PointCloud& cloud, double r_min, Session& s = default_session()) {
    std::vector<rt3d_point> in = detail::to_c(cloud), out(in.size());
    std::uint64_t n = 0;
    check(rt3d_prune(s.get(), in.data(), in.size(), r_min, out.data(), &n));
    out.resize(n);
    return detail::from_c(out);
}

// ---- background denoisers ----------------------------------------------------

inline Grid2D<double> fft_lowpass_filter(const Grid2D<double>& img, double cutoff,
                                         Session& s = default_session()) {
    Grid2D<double> out(img.rows, img.cols, 0.0);
    check(rt3d_fft_lowpass_filter(s.get(), img.data.data(), img.rows, img.cols, cutoff, 0,
                                  out.data.data()));
    return out;
}

inline BackgroundImage fft_background_denoise(const BackgroundImage& b, double cutoff,
                                              Session& s = default_session()) {
    BackgroundImage out(b.rows, b.cols, 0.0);
    check(rt3d_fft_lowpass_filter(s.get(), b.data.data(), b.rows, b.cols, cutoff, 1,
                                  out.data.data()));
    return out;
}

// ---- around the path: output and the forward simulator ----------------------

/// encode_ply (io.hpp:162-179), byte-identical; formatted on all host threads.
inline std::string encode_ply(const PointCloud& cloud, std::optional<double> pixel_pitch = {}) {
    const std::vector<rt3d_point> pts = detail::to_c(cloud);
    std::uint64_t n = 0;
    check(rt3d_encode_ply(pts.data(), pts.size(), pixel_pitch ? 1 : 0, pixel_pitch.value_or(0.0),
                          nullptr, 0, &n));
    std::string out(n, '\0');
    check(rt3d_encode_ply(pts.data(), pts.size(), pixel_pitch ? 1 : 0, pixel_pitch.value_or(0.0),
                          out.data(), n, &n));
    return out;
}

/// simulate_cube's photon sampling (simulate.hpp:181-205) on the device:
/// `truth` after the reflectivity scaling (SimReport::truth), `background`
/// = SimReport::background_truth.  The cube stays resident in `s` as well.
inline PhotonCube simulate_photons(const PointCloud& truth, const BackgroundImage& background,
                                   const SensorModel& sensor, std::uint64_t seed,
                                   Session& s = default_session()) {
    detail::SensorView sv(sensor);
    check(rt3d_set_sensor(s.get(), &sv.c));
    const std::vector<rt3d_point> pts = detail::to_c(truth);
    std::uint64_t n = 0, ph[2] = {0, 0};
    check(rt3d_simulate_cube(s.get(), pts.data(), pts.size(), background.data.data(), seed, &n,
                             ph));
    PhotonCube c(sensor.n_rows, sensor.n_cols, sensor.n_bins,
                 2.0 * sensor.bin_resolution / kSpeedOfLight);
    c.events.resize(n);
    static_assert(sizeof(Event) == sizeof(rt3d_event), "Event layout");
    check(rt3d_cube_copy(s.get(), c.offsets.data(),
                         reinterpret_cast<rt3d_event*>(c.events.data())));
    c.recount();
    return c;
}

}  // namespace splidar::b200
