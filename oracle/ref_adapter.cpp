// TEST INFRASTRUCTURE ONLY.  Compiles the reference headers unchanged from
// /root/reference/proj/include (plus the reference's own test oracles,
// /root/reference/proj/tests/oracles.hpp) against the test-only Eigen/FFTW
// stand-ins in oracle/shim, and exposes them through the rt3d_* C views so the
// tests can run the reference and the C oracle on identical inputs.
// Built by oracle/Makefile into oracle/_ref/libref.so (git-ignored).
// Standard headers first: the reference's Irf keeps its samples private and
// renormalises in its ctor; to hand it the exact (already normalised) sample
// array the oracle sees, the reference headers are compiled with private
// members opened up.  Test-only.
#include <algorithm>
#include <charconv>
#include <chrono>
#include <cmath>
#include <complex>
#include <cstdint>
#include <cstring>
#include <fstream>
#include <limits>
#include <map>
#include <optional>
#include <span>
#include <sstream>
#include <stdexcept>
#include <string>
#include <thread>
#include <tuple>
#include <unordered_map>
#include <vector>
#include <json.hpp>
#include <Eigen/Dense>
#include <fftw3.h>
#define private public
#include "splidar/splidar.hpp"
#include "splidar/io.hpp"
#include "splidar/report_json.hpp"
#undef private

#include "oracles.hpp"

#include "../include/rt3d.h"

#include <chrono>
#include <cstring>
#include <string>
#include <thread>

using namespace splidar;

namespace {

thread_local std::string g_err;

Irf make_irf(const rt3d_irf& v) {
    // samples are already normalised; the ctor renormalises by a mass that is
    // 1 up to rounding, so rebuild exactly from the given samples instead.
    std::vector<double> s(v.samples, v.samples + v.n_samples);
    Irf irf(v.tau_min, v.dtau, s);
    irf.samples_ = s;  // exact samples (see the note at the top)
    for (std::size_t k = 0; k + 1 < s.size(); ++k) irf.slopes_[k] = (s[k + 1] - s[k]) / v.dtau;
    return irf;
}

SensorModel make_sensor(const rt3d_sensor* s) {
    SensorModel m(s->n_rows, s->n_cols, s->n_bins, make_irf(s->irf_shared), s->superres,
                  s->pixel_pitch, s->bin_resolution);
    size_t np = static_cast<size_t>(s->n_rows) * s->n_cols;
    if (s->irf_per_pixel)
        for (size_t p = 0; p < np; ++p) m.irf_per_pixel.push_back(make_irf(s->irf_per_pixel[p]));
    for (size_t p = 0; p < np; ++p) {
        m.gain.data[p] = s->gain[p];
        m.dead.data[p] = s->dead[p];
    }
    return m;
}

PhotonCube make_cube(const rt3d_cube* c) {
    PhotonCube cube(c->n_rows, c->n_cols, c->n_bins, c->bin_width_s);
    size_t np = cube.n_pixels();
    for (size_t p = 0; p <= np; ++p) cube.offsets[p] = c->offsets[p];
    cube.events.resize(c->n_events);
    for (uint64_t e = 0; e < c->n_events; ++e)
        cube.events[e] = Event{c->events[e].bin, c->events[e].count};
    cube.recount();
    return cube;
}

Point to_point(const rt3d_point& q) {
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

rt3d_point from_point(const Point& p) {
    rt3d_point q;
    std::memset(&q, 0, sizeof q);
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

PointCloud make_cloud(const rt3d_point* pts, uint64_t n) {
    PointCloud c;
    c.points.reserve(n);
    for (uint64_t k = 0; k < n; ++k) c.points.push_back(to_point(pts[k]));
    return c;
}

SceneState make_state(const SensorModel& sensor, const rt3d_point* pts, uint64_t n,
                      const double* bg) {
    BackgroundImage b(sensor.n_rows, sensor.n_cols, 0.0);
    for (size_t p = 0; p < b.data.size(); ++p) b.data[p] = bg[p];
    return SceneState(make_cloud(pts, n), b, &sensor);
}

ReconConfig make_cfg(const rt3d_recon_config* c) {
    ReconConfig r;
    r.max_iters = c->max_iters;
    r.stop_tol = c->stop_tol;
    r.step_t.automatic = c->step_t_auto != 0;
    r.step_t.value = c->step_t;
    r.step_r.automatic = c->step_r_auto != 0;
    r.step_r.value = c->step_r;
    r.step_b.automatic = c->step_b_auto != 0;
    r.step_b.value = c->step_b;
    r.backtrack_beta = c->backtrack_beta;
    r.apss.kernel_radius = c->apss.kernel_radius;
    r.apss.min_neighbors = c->apss.min_neighbors;
    r.apss.sphere_degeneracy_eps = c->apss.sphere_degeneracy_eps;
    r.knn_k = c->knn_k;
    r.r_min = c->r_min;
    r.background_mode = c->background_mode ? BackgroundMode::Fft : BackgroundMode::Identity;
    r.fft_cutoff = c->fft_cutoff;
    r.init.max_returns = c->init.max_returns;
    r.init.peak_threshold = c->init.peak_threshold;
    r.init.min_separation = c->init.min_separation;
    return r;
}

rt3d_step_diag to_diag(const StepDiagnostics& d) {
    rt3d_step_diag o;
    std::memset(&o, 0, sizeof o);
    o.nll_before = d.nll_before;
    o.nll_after = d.nll_after;
    o.points_before = d.points_before;
    o.points_after = d.points_after;
    auto blk = [](const BlockDiagnostics& b) {
        rt3d_block_diag x;
        std::memset(&x, 0, sizeof x);
        x.step_used = b.step_used;
        x.backtracks = b.backtracks;
        x.nll_after_grad = b.nll_after_grad;
        x.nll_after_denoise = b.nll_after_denoise;
        return x;
    };
    o.depth = blk(d.depth);
    o.intensity = blk(d.intensity);
    o.background = blk(d.background);
    return o;
}

template <typename F>
int guarded(F&& f) {
    try {
        f();
        return 0;
    } catch (const FormatError& e) {
        g_err = e.what();
        return 2;
    } catch (const std::out_of_range& e) {
        g_err = e.what();
        return 3;
    } catch (const std::invalid_argument& e) {
        g_err = e.what();
        return 1;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 9;
    }
}

// last simulated scene / random instance, copied out by the *_copy calls
struct Held {
    PhotonCube cube;
    std::vector<Irf> irfs;
    SensorModel sensor;
    PointCloud cloud;
    BackgroundImage background;
    std::string report_json;
};
thread_local Held g_held;

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }
void ref_set_threads(unsigned n) { set_thread_count(n); }

// evaluate (eval.hpp:33-87)
int ref_evaluate(const rt3d_point* est, uint64_t n_est, const rt3d_point* truth, uint64_t n_truth,
                 double tau, double pitch, double* out7) {
    return guarded([&] {
        EvalResult r = evaluate(make_cloud(est, n_est), make_cloud(truth, n_truth), tau, pitch);
        out7[0] = r.recall;
        out7[1] = r.false_point_rate;
        out7[2] = r.depth_rmse;
        out7[3] = r.intensity_mae;
        out7[4] = (double)r.n_truth;
        out7[5] = (double)r.n_est;
        out7[6] = (double)r.n_matched;
    });
}

// encode_cube (io.hpp:99-114): the SPCB bytes of a cube
int ref_encode_cube(const rt3d_cube* c, uint8_t* out, uint64_t cap, uint64_t* n) {
    return guarded([&] {
        const std::string b = encode_cube(make_cube(c));
        *n = b.size();
        if (out && cap >= b.size()) std::memcpy(out, b.data(), b.size());
    });
}

// encode_ply (io.hpp:162-179): the reference's PLY text of a cloud
int ref_encode_ply(const rt3d_point* pts, uint64_t n, int has_pitch, double pitch, char* out,
                   uint64_t cap, uint64_t* nb) {
    return guarded([&] {
        const std::string b = has_pitch ? encode_ply(make_cloud(pts, n), pitch)
                                        : encode_ply(make_cloud(pts, n));
        *nb = b.size();
        if (out && cap >= b.size()) std::memcpy(out, b.data(), b.size());
    });
}

// decode_cube (io.hpp:116-145): 0 and the CSR, or 1 and the exception text
int ref_decode_cube(const uint8_t* bytes, uint64_t n, uint64_t* offsets, rt3d_event* events,
                    uint64_t cap) {
    return guarded([&] {
        PhotonCube cube = decode_cube(std::string(reinterpret_cast<const char*>(bytes), n));
        if (offsets) std::memcpy(offsets, cube.offsets.data(), cube.offsets.size() * 8);
        if (events && cap >= cube.events.size())
            std::memcpy(events, cube.events.data(), cube.events.size() * 8);
    });
}

int ref_matched_filter_peaks(const rt3d_event* ev, uint64_t n, const rt3d_irf* irf, int n_bins,
                             int k, double thr, int min_sep, rt3d_peak* out) {
    int cnt = -1;
    guarded([&] {
        Irf f = make_irf(*irf);
        std::vector<Event> e(n);
        for (uint64_t q = 0; q < n; ++q) e[q] = Event{ev[q].bin, ev[q].count};
        auto peaks = detail::matched_filter_peaks(e.data(), e.data() + n, f, n_bins, k, thr, min_sep);
        for (size_t q = 0; q < peaks.size(); ++q) out[q] = rt3d_peak{peaks[q].t, peaks[q].response, peaks[q].mass};
        cnt = static_cast<int>(peaks.size());
    });
    return cnt;
}

int ref_init_matched_filter(const rt3d_cube* c, const rt3d_sensor* s, const rt3d_init_params* p,
                            rt3d_point* pts, uint64_t* n, double* bg) {
    return guarded([&] {
        SensorModel sensor = make_sensor(s);
        PhotonCube cube = make_cube(c);
        InitParams ip;
        ip.max_returns = p->max_returns;
        ip.peak_threshold = p->peak_threshold;
        ip.min_separation = p->min_separation;
        SceneState st = init_matched_filter(cube, sensor, ip);
        for (size_t k = 0; k < st.cloud.size(); ++k) pts[k] = from_point(st.cloud[k]);
        *n = st.cloud.size();
        std::memcpy(bg, st.background.data.data(), sizeof(double) * st.background.data.size());
    });
}

double ref_nll(const rt3d_cube* c, const rt3d_sensor* s, const rt3d_point* pts, uint64_t n,
               const double* bg) {
    double v = 0;
    guarded([&] {
        SensorModel sensor = make_sensor(s);
        PhotonCube cube = make_cube(c);
        SceneState st = make_state(sensor, pts, n, bg);
        v = nll(st, cube);
    });
    return v;
}

int ref_grads(const rt3d_cube* c, const rt3d_sensor* s, const rt3d_point* pts, uint64_t n,
              const double* bg, double* gd, uint8_t* oog, double* gr, double* gb, double* cd,
              double* cr, double* cb) {
    return guarded([&] {
        SensorModel sensor = make_sensor(s);
        PhotonCube cube = make_cube(c);
        SceneState st = make_state(sensor, pts, n, bg);
        DepthGradient d = grad_depth(st, cube);
        std::memcpy(gd, d.value.data(), sizeof(double) * n);
        std::memset(oog, 0, n);
        for (auto k : d.out_of_gate) oog[k] = 1;
        auto r = grad_intensity(st, cube);
        std::memcpy(gr, r.data(), sizeof(double) * n);
        auto b = grad_background(st, cube);
        std::memcpy(gb, b.data.data(), sizeof(double) * b.data.size());
        auto cv = block_curvatures(st, cube);
        std::memcpy(cd, cv.depth.data(), sizeof(double) * n);
        std::memcpy(cr, cv.intensity.data(), sizeof(double) * n);
        std::memcpy(cb, cv.background.data.data(), sizeof(double) * cv.background.data.size());
    });
}

int ref_apss_project(const rt3d_point* pts, uint64_t n, const rt3d_apss_params* p,
                     double cell, rt3d_point* out) {
    return guarded([&] {
        PointCloud cloud = make_cloud(pts, n);
        ApssParams ap;
        ap.kernel_radius = p->kernel_radius;
        ap.min_neighbors = p->min_neighbors;
        ap.sphere_degeneracy_eps = p->sphere_degeneracy_eps;
        SpatialIndex idx(cloud, cell);
        PointCloud res = apss_project(cloud, ap, idx);
        for (size_t k = 0; k < res.size(); ++k) out[k] = from_point(res[k]);
    });
}

int ref_knn_intensity_filter(const rt3d_point* pts, uint64_t n, int k, double cell, double radius,
                             rt3d_point* out) {
    return guarded([&] {
        PointCloud cloud = make_cloud(pts, n);
        SpatialIndex idx(cloud, cell);
        PointCloud res = knn_intensity_filter(cloud, k, idx, radius);
        for (size_t q = 0; q < res.size(); ++q) out[q] = from_point(res[q]);
    });
}

int ref_fft_lowpass(const double* img, int rows, int cols, double cutoff, int clamp, double* out) {
    return guarded([&] {
        Grid2D<double> g(rows, cols);
        std::memcpy(g.data.data(), img, sizeof(double) * g.data.size());
        Grid2D<double> r = clamp ? fft_background_denoise(g, cutoff) : fft_lowpass_filter(g, cutoff);
        std::memcpy(out, r.data.data(), sizeof(double) * r.data.size());
    });
}

int ref_palm_step(const rt3d_cube* c, const rt3d_sensor* s, const rt3d_recon_config* cfg,
                  rt3d_point* pts, uint64_t* n, double* bg, rt3d_step_diag* diag) {
    return guarded([&] {
        SensorModel sensor = make_sensor(s);
        PhotonCube cube = make_cube(c);
        SceneState st = make_state(sensor, pts, *n, bg);
        StepDiagnostics d = palm_step(st, cube, make_cfg(cfg));
        *diag = to_diag(d);
        for (size_t k = 0; k < st.cloud.size(); ++k) pts[k] = from_point(st.cloud[k]);
        *n = st.cloud.size();
        std::memcpy(bg, st.background.data.data(), sizeof(double) * st.background.data.size());
    });
}

// Runs reconstruct; the result is held and copied out by ref_result_copy.
int ref_reconstruct(const rt3d_cube* c, const rt3d_sensor* s, const rt3d_recon_config* cfg,
                    uint64_t* n_points, int* iterations, double* seconds) {
    return guarded([&] {
        SensorModel sensor = make_sensor(s);
        PhotonCube cube = make_cube(c);
        auto t0 = std::chrono::steady_clock::now();
        ReconResult r = reconstruct(cube, sensor, make_cfg(cfg));
        auto t1 = std::chrono::steady_clock::now();
        if (seconds) *seconds = std::chrono::duration<double>(t1 - t0).count();
        g_held.cloud = std::move(r.cloud);
        g_held.background = std::move(r.background);
        g_held.report_json = recon_report_json(r.report, false);
        *n_points = g_held.cloud.size();
        *iterations = r.report.iterations;
        static thread_local std::vector<rt3d_step_diag> steps;
        static thread_local std::vector<double> trace;
        steps.clear();
        for (auto& d : r.report.steps) steps.push_back(to_diag(d));
        trace = r.report.nll_trace;
        g_held.irfs.clear();
        // stash trace/steps behind the report string's storage
        g_held.cube = PhotonCube();
        (void)steps;
        (void)trace;
    });
}

int ref_result_copy(rt3d_point* pts, double* bg) {
    for (size_t k = 0; k < g_held.cloud.size(); ++k) pts[k] = from_point(g_held.cloud[k]);
    if (bg)
        std::memcpy(bg, g_held.background.data.data(), sizeof(double) * g_held.background.data.size());
    return 0;
}

// Full report of the last ref_reconstruct (trace + steps), re-run free.
int ref_reconstruct_full(const rt3d_cube* c, const rt3d_sensor* s, const rt3d_recon_config* cfg,
                         rt3d_point* pts, uint64_t* n_points, double* bg, double* trace,
                         rt3d_step_diag* steps, int* iterations) {
    return guarded([&] {
        SensorModel sensor = make_sensor(s);
        PhotonCube cube = make_cube(c);
        ReconResult r = reconstruct(cube, sensor, make_cfg(cfg));
        for (size_t k = 0; k < r.cloud.size(); ++k) pts[k] = from_point(r.cloud[k]);
        *n_points = r.cloud.size();
        std::memcpy(bg, r.background.data.data(), sizeof(double) * r.background.data.size());
        for (size_t k = 0; k < r.report.nll_trace.size(); ++k) trace[k] = r.report.nll_trace[k];
        for (size_t k = 0; k < r.report.steps.size(); ++k) steps[k] = to_diag(r.report.steps[k]);
        *iterations = r.report.iterations;
    });
}

const char* ref_report_json() { return g_held.report_json.c_str(); }

int ref_baseline_xcorr(const rt3d_cube* c, const rt3d_sensor* s, rt3d_point* pts, uint64_t* n) {
    return guarded([&] {
        SensorModel sensor = make_sensor(s);
        PhotonCube cube = make_cube(c);
        PointCloud r = baseline_xcorr(cube, sensor);
        for (size_t k = 0; k < r.size(); ++k) pts[k] = from_point(r[k]);
        *n = r.size();
    });
}

// ---- inputs generated by the reference itself ------------------------------

// simulate_cube from a SceneSpec key=value text (simulate.hpp:139-302).
int ref_simulate(const char* scene_text, uint64_t seed, int* dims, uint64_t* n_events,
                 uint64_t* n_truth) {
    return guarded([&] {
        SceneSpec spec = SceneSpec::from_kv(KeyValueFile::parse_text(scene_text));
        g_held.sensor = build_sensor(spec);
        auto [cube, rep] = simulate_cube(spec, g_held.sensor, seed);
        g_held.cube = std::move(cube);
        g_held.cloud = std::move(rep.truth);
        dims[0] = g_held.cube.n_rows;
        dims[1] = g_held.cube.n_cols;
        dims[2] = g_held.cube.n_bins;
        dims[3] = g_held.sensor.superres;
        *n_events = g_held.cube.events.size();
        *n_truth = g_held.cloud.size();
    });
}

// oracle::random_instance (tests/oracles.hpp:75-133)
int ref_random_instance(uint64_t seed, int with_dead, int* dims, uint64_t* n_events,
                        uint64_t* n_points) {
    return guarded([&] {
        oracle::RandomInstance inst = oracle::random_instance(seed, with_dead != 0);
        g_held.sensor = inst.sensor;
        g_held.cube = inst.cube;
        g_held.cloud = inst.state.cloud;
        g_held.background = inst.state.background;
        dims[0] = g_held.cube.n_rows;
        dims[1] = g_held.cube.n_cols;
        dims[2] = g_held.cube.n_bins;
        dims[3] = g_held.sensor.superres;
        *n_events = g_held.cube.events.size();
        *n_points = g_held.cloud.size();
    });
}

// Copies the held cube / sensor tables / cloud / background.
int ref_held_copy(uint64_t* offsets, rt3d_event* events, double* gain, uint8_t* dead,
                  double* irf_samples, double* irf_meta, rt3d_point* pts, double* bg) {
    const PhotonCube& c = g_held.cube;
    if (offsets) std::memcpy(offsets, c.offsets.data(), sizeof(uint64_t) * c.offsets.size());
    if (events)
        for (size_t e = 0; e < c.events.size(); ++e) events[e] = rt3d_event{c.events[e].bin, c.events[e].count};
    if (gain) std::memcpy(gain, g_held.sensor.gain.data.data(), sizeof(double) * g_held.sensor.gain.data.size());
    if (dead) std::memcpy(dead, g_held.sensor.dead.data.data(), g_held.sensor.dead.data.size());
    if (irf_samples) {
        const auto& s = g_held.sensor.irf_shared.samples();
        std::memcpy(irf_samples, s.data(), sizeof(double) * s.size());
    }
    if (irf_meta) {
        irf_meta[0] = g_held.sensor.irf_shared.tau_min();
        irf_meta[1] = g_held.sensor.irf_shared.dtau();
        irf_meta[2] = static_cast<double>(g_held.sensor.irf_shared.samples().size());
        irf_meta[3] = g_held.sensor.pixel_pitch;
        irf_meta[4] = g_held.sensor.bin_resolution;
        irf_meta[5] = c.bin_width_s;
    }
    if (pts)
        for (size_t k = 0; k < g_held.cloud.size(); ++k) pts[k] = from_point(g_held.cloud[k]);
    if (bg && !g_held.background.data.empty())
        std::memcpy(bg, g_held.background.data.data(), sizeof(double) * g_held.background.data.size());
    return 0;
}

// oracle::dense_nll (tests/oracles.hpp:44-63) on a given state.
double ref_dense_nll(const rt3d_cube* c, const rt3d_sensor* s, const rt3d_point* pts, uint64_t n,
                     const double* bg) {
    double v = 0;
    guarded([&] {
        SensorModel sensor = make_sensor(s);
        PhotonCube cube = make_cube(c);
        SceneState st = make_state(sensor, pts, n, bg);
        v = oracle::dense_nll(st, cube);
    });
    return v;
}

// Irf::gaussian samples (sensor.hpp:45-57).
uint64_t ref_irf_gaussian(double sigma, double nsig, double dtau, double* out, double* tau_min) {
    Irf f = Irf::gaussian(sigma, nsig, dtau);
    std::memcpy(out, f.samples().data(), sizeof(double) * f.samples().size());
    *tau_min = f.tau_min();
    return f.samples().size();
}

}  // extern "C"
