// TEST INFRASTRUCTURE: the drop-in proof for include/splidar/b200.hpp.
// Built by oracle/Makefile (target `dropin`) against the reference's own
// headers (Eigen/FFTW stand-ins from oracle/shim), linked to librt3d.so, and
// run on a GPU box by tests/test_dropin.py.  Every check calls the reference
// function and its splidar::b200 counterpart on the same inputs:
//   bitwise      nll, gradients, curvatures, init, baseline, kNN, prune
//   tolerance    palm_step / reconstruct (APSS eigen-solver differs ~1e-11),
//                FFT (direct DFT stand-in vs device FFT)
//   exceptions   the reference's exception types for invalid inputs
#include "splidar/splidar.hpp"
#include "splidar/b200.hpp"
#include "oracles.hpp"

#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>

using namespace splidar;

static int g_fail = 0;
#define CHECK(cond, ...)                                              \
    do {                                                              \
        if (!(cond)) {                                                \
            std::printf("FAIL %s:%d: ", __FILE__, __LINE__);          \
            std::printf(__VA_ARGS__);                                 \
            std::printf("\n");                                        \
            ++g_fail;                                                 \
        }                                                             \
    } while (0)

static bool same(double a, double b) { return std::memcmp(&a, &b, sizeof a) == 0; }

static bool same_cloud(const PointCloud& a, const PointCloud& b) {
    if (a.size() != b.size()) return false;
    for (std::size_t n = 0; n < a.size(); ++n) {
        const Point &p = a[n], &q = b[n];
        if (!same(p.position.x(), q.position.x()) || !same(p.position.y(), q.position.y()) ||
            !same(p.position.z(), q.position.z()) || !same(p.intensity, q.intensity) ||
            p.i != q.i || p.j != q.j || p.fi != q.fi || p.fj != q.fj || !same(p.t, q.t) ||
            p.flags != q.flags)
            return false;
    }
    return true;
}

static void check_likelihood(std::uint64_t seed) {
    oracle::RandomInstance inst = oracle::random_instance(seed, seed % 2 == 1);
    const SceneState& st = inst.state;
    CHECK(same(nll(st, inst.cube), b200::nll(st, inst.cube)), "nll seed %llu",
          (unsigned long long)seed);
    DepthGradient a = grad_depth(st, inst.cube), b = b200::grad_depth(st, inst.cube);
    CHECK(a.out_of_gate == b.out_of_gate, "grad_depth oog seed %llu", (unsigned long long)seed);
    for (std::size_t n = 0; n < a.value.size(); ++n)
        CHECK(same(a.value[n], b.value[n]), "grad_depth[%zu]", n);
    auto gr = grad_intensity(st, inst.cube), gr2 = b200::grad_intensity(st, inst.cube);
    for (std::size_t n = 0; n < gr.size(); ++n) CHECK(same(gr[n], gr2[n]), "grad_intensity[%zu]", n);
    auto gb = grad_background(st, inst.cube), gb2 = b200::grad_background(st, inst.cube);
    for (std::size_t n = 0; n < gb.size(); ++n)
        CHECK(same(gb.data[n], gb2.data[n]), "grad_background[%zu]", n);
    auto c = block_curvatures(st, inst.cube), c2 = b200::block_curvatures(st, inst.cube);
    for (std::size_t n = 0; n < c.depth.size(); ++n)
        CHECK(same(c.depth[n], c2.depth[n]) && same(c.intensity[n], c2.intensity[n]),
              "curvature[%zu]", n);
    for (std::size_t n = 0; n < c.background.size(); ++n)
        CHECK(same(c.background.data[n], c2.background.data[n]), "curvature_b[%zu]", n);
}

static SceneSpec small_scene() {
    SceneSpec spec;
    spec.rows = 12;
    spec.cols = 12;
    spec.bins = 300;
    spec.superres = 3;
    spec.bin_resolution_m = 0.01;
    spec.pixel_pitch_m = 0.02 / 3;
    spec.target_ppp = 40;
    spec.target_sbr = 4;
    SurfaceSpec back;
    back.depth_m = 1.5;
    back.slope_x = 0.3;
    back.reflectivity = 0.8;
    SurfaceSpec bump;
    bump.kind = SurfaceSpec::Kind::Bump;
    bump.depth_m = 1.0;
    bump.bump_amp = -0.05;
    bump.bump_width = 0.03;
    bump.bump_cx = bump.bump_cy = 0.12;
    bump.region = {6, 6, 30, 30};
    spec.surfaces = {back, bump};
    spec.dead_pixels = {{0, 5}};
    return spec;
}

int main() {
    for (std::uint64_t seed = 1; seed <= 12; ++seed) check_likelihood(seed);

    SceneSpec spec = small_scene();
    SensorModel sensor = build_sensor(spec);
    PhotonCube cube = simulate_cube(spec, sensor, 7).first;

    ReconConfig cfg;
    cfg.max_iters = 6;
    cfg.stop_tol = 0.0;
    cfg.apss.kernel_radius = 0.02;
    cfg.knn_k = 9;
    cfg.r_min = 0.05;
    cfg.init.max_returns = 2;
    cfg.init.min_separation = 6;

    // forward simulator on the device: the same cube (counter-based RNG)
    {
        auto [ref_cube, rep] = simulate_cube(spec, sensor, 7);
        PhotonCube dev = b200::simulate_photons(rep.truth, rep.background_truth, sensor, 7);
        std::size_t diff = 0;
        if (dev.offsets != ref_cube.offsets || dev.events.size() != ref_cube.events.size()) {
            diff = 1;
        } else {
            for (std::size_t k = 0; k < dev.events.size(); ++k)
                diff += dev.events[k].bin != ref_cube.events[k].bin ||
                        dev.events[k].count != ref_cube.events[k].count;
        }
        CHECK(diff == 0, "simulate_photons differs (%zu)", diff);
        CHECK(dev.total_count == ref_cube.total_count, "simulate total count");
    }

    // init + baseline + peaks: bitwise
    SceneState s0 = init_matched_filter(cube, sensor, cfg.init);
    SceneState s1 = b200::init_matched_filter(cube, sensor, cfg.init);
    CHECK(same_cloud(s0.cloud, s1.cloud), "init cloud");
    CHECK(s0.background == s1.background, "init background");
    CHECK(same_cloud(baseline_xcorr(cube, sensor), b200::baseline_xcorr(cube, sensor)), "baseline");
    CHECK(encode_ply(s0.cloud, sensor.pixel_pitch) == b200::encode_ply(s0.cloud, sensor.pixel_pitch),
          "encode_ply");
    CHECK(encode_ply(s0.cloud) == b200::encode_ply(s0.cloud), "encode_ply without pitch");
    {
        const PointCloud bl = baseline_xcorr(cube, sensor);
        for (double tau : {0.01, 0.05, 0.3}) {
            const EvalResult e0 = evaluate(s0.cloud, bl, tau, sensor.pixel_pitch);
            const EvalResult e1 = b200::evaluate(s0.cloud, bl, tau, sensor.pixel_pitch);
            CHECK(same(e0.recall, e1.recall) && same(e0.false_point_rate, e1.false_point_rate) &&
                      same(e0.depth_rmse, e1.depth_rmse) &&
                      same(e0.intensity_mae, e1.intensity_mae) && e0.n_matched == e1.n_matched &&
                      e0.n_truth == e1.n_truth && e0.n_est == e1.n_est,
                  "evaluate tau %g", tau);
        }
    }
    for (int i = 0; i < cube.n_rows; ++i) {
        auto [eb, ee] = cube.pixel(i, i);
        auto p0 = splidar::detail::matched_filter_peaks(eb, ee, sensor.irf_shared, cube.n_bins, 3,
                                                        0.5, 6);
        auto p1 = b200::matched_filter_peaks(eb, ee, sensor.irf_shared, cube.n_bins, 3, 0.5, 6);
        CHECK(p0.size() == p1.size(), "peaks count pixel %d", i);
        for (std::size_t q = 0; q < p0.size() && q < p1.size(); ++q)
            CHECK(same(p0[q].t, p1[q].t) && same(p0[q].response, p1[q].response) &&
                      same(p0[q].mass, p1[q].mass),
                  "peak %zu pixel %d", q, i);
    }

    // denoisers on the init cloud
    SpatialIndex index(s0.cloud, cfg.apss.kernel_radius);
    CHECK(same_cloud(knn_intensity_filter(s0.cloud, 9, index, 0.02),
                     b200::knn_intensity_filter(s0.cloud, 9, index, 0.02)),
          "knn");
    CHECK(same_cloud(prune(s0.cloud, 0.3), b200::prune(s0.cloud, 0.3)), "prune");
    {
        PointCloud a = apss_project(s0.cloud, cfg.apss, index);
        PointCloud b = b200::apss_project(s0.cloud, cfg.apss, index);
        CHECK(a.size() == b.size(), "apss size");
        double worst = 0.0;
        for (std::size_t n = 0; n < a.size() && n < b.size(); ++n)
            worst = std::max(worst, (a[n].position - b[n].position).norm());
        CHECK(worst < 1e-9, "apss worst %.3g m", worst);
    }
    {
        auto a = fft_background_denoise(s0.background, 0.3);
        auto b = b200::fft_background_denoise(s0.background, 0.3);
        double worst = 0.0;
        for (std::size_t n = 0; n < a.size(); ++n)
            worst = std::max(worst, std::fabs(a.data[n] - b.data[n]));
        CHECK(worst < 1e-9, "fft worst %.3g", worst);
    }

    // one PALM step
    {
        SceneState a = s0, b = s0;
        StepDiagnostics da = palm_step(a, cube, cfg), db = b200::palm_step(b, cube, cfg);
        CHECK(a.cloud.size() == b.cloud.size(), "palm points %zu vs %zu", a.cloud.size(),
              b.cloud.size());
        CHECK(std::fabs(da.nll_after - db.nll_after) <= 1e-9 * std::fabs(da.nll_after),
              "palm nll %.17g vs %.17g", da.nll_after, db.nll_after);
        CHECK(da.depth.backtracks == db.depth.backtracks &&
                  da.intensity.backtracks == db.intensity.backtracks &&
                  da.background.backtracks == db.background.backtracks,
              "palm backtracks");
    }

    // full pipeline: north-star tolerances
    {
        ReconResult a = reconstruct(cube, sensor, cfg);
        ReconResult b = b200::reconstruct(cube, sensor, cfg);
        CHECK(a.report.iterations == b.report.iterations, "iterations %d vs %d",
              a.report.iterations, b.report.iterations);
        CHECK(a.cloud.size() == b.cloud.size(), "points %zu vs %zu", a.cloud.size(),
              b.cloud.size());
        double dt = 0.0, dr = 0.0;
        for (std::size_t n = 0; n < a.cloud.size() && n < b.cloud.size(); ++n) {
            dt = std::max(dt, std::fabs(a.cloud[n].t - b.cloud[n].t));
            dr = std::max(dr, std::fabs(a.cloud[n].intensity - b.cloud[n].intensity) /
                                  std::max(1e-12, std::fabs(a.cloud[n].intensity)));
        }
        CHECK(dt <= 1e-3, "reconstruct max |dt| %.3g bins", dt);
        CHECK(dr <= 1e-4, "reconstruct max rel |dr| %.3g", dr);
        CHECK(a.report.nll_trace.size() == b.report.nll_trace.size(), "trace size");
        CHECK(std::fabs(a.report.final_nll - b.report.final_nll) <=
                  1e-9 * std::fabs(a.report.final_nll),
              "final nll %.17g vs %.17g", a.report.final_nll, b.report.final_nll);
        std::printf("reconstruct: %zu points, %d iterations, max|dt| %.3g, max rel|dr| %.3g\n",
                    b.cloud.size(), b.report.iterations, dt, dr);
    }

    // exceptions
    {
        ReconConfig bad = cfg;
        bad.knn_k = 0;
        bool threw = false;
        try { b200::reconstruct(cube, sensor, bad); } catch (const std::invalid_argument&) { threw = true; }
        CHECK(threw, "invalid config must throw std::invalid_argument");
        SensorModel other(cube.n_rows + 1, cube.n_cols, cube.n_bins, Irf::gaussian(1.5));
        threw = false;
        try { b200::init_matched_filter(cube, other, cfg.init); } catch (const std::invalid_argument&) { threw = true; }
        CHECK(threw, "sensor/cube mismatch must throw std::invalid_argument");
    }

    if (g_fail) {
        std::printf("DROPIN FAILED (%d)\n", g_fail);
        return 1;
    }
    std::printf("DROPIN OK\n");
    return 0;
}
