// splidar/likelihood.hpp — drop-in replacement (B200 build) for the
// reference's likelihood.hpp:20-333.  SceneState and the per-pixel rate
// helpers of the forward model stay on the host (the simulator and the
// reference's tests call them); the likelihood sweeps — nll, grad_depth,
// grad_intensity, grad_background, block_curvatures — run on the GPU
// (rt3d_nll / rt3d_grad_* / rt3d_block_curvatures, one thread group per
// pixel, pairwise_sum's tree reproduced), bit-identical to the reference.
#pragma once

#include "splidar/b200_device.hpp"
#include "splidar/cloud.hpp"
#include "splidar/cube.hpp"
#include "splidar/grid.hpp"
#include "splidar/parallel.hpp"
#include "splidar/sensor.hpp"

#include <cmath>
#include <cstdint>
#include <limits>
#include <stdexcept>
#include <utility>
#include <vector>

namespace splidar {

/// The estimate (t, r, b) with its sensor and the per-pixel point buckets
/// (likelihood.hpp:20-62); refresh() after any cloud mutation.
struct SceneState {
    PointCloud cloud;
    BackgroundImage background;
    const SensorModel* sensor = nullptr;

    std::vector<std::uint32_t> bucket_offsets;  // n_pixels + 1
    std::vector<std::uint32_t> bucket_points;   // point indices grouped by pixel, cloud order

    SceneState() = default;
    SceneState(PointCloud c, BackgroundImage b, const SensorModel* s)
        : cloud(std::move(c)), background(std::move(b)), sensor(s) {
        if (!sensor) throw std::invalid_argument("SceneState: null sensor");
        if (background.rows != sensor->n_rows || background.cols != sensor->n_cols)
            throw std::invalid_argument("SceneState: background/sensor shape mismatch");
        refresh();
    }

    /// Stable counting sort of the points by home pixel.
    void refresh() {
        const std::size_t npix = static_cast<std::size_t>(sensor->n_rows) * sensor->n_cols;
        bucket_offsets.assign(npix + 1, 0);
        for (const Point& p : cloud) {
            if (p.i < 0 || p.i >= sensor->n_rows || p.j < 0 || p.j >= sensor->n_cols)
                throw std::invalid_argument("SceneState: point home pixel out of bounds");
            ++bucket_offsets[static_cast<std::size_t>(p.i) * sensor->n_cols + p.j + 1];
        }
        for (std::size_t q = 0; q < npix; ++q) bucket_offsets[q + 1] += bucket_offsets[q];
        bucket_points.assign(cloud.size(), 0);
        std::vector<std::uint32_t> fill(bucket_offsets.begin(), bucket_offsets.end() - 1);
        for (std::uint32_t n = 0; n < cloud.size(); ++n) {
            const Point& p = cloud[n];
            bucket_points[fill[static_cast<std::size_t>(p.i) * sensor->n_cols + p.j]++] = n;
        }
    }

    std::pair<const std::uint32_t*, const std::uint32_t*> pixel_points(int i, int j) const {
        const std::size_t q = static_cast<std::size_t>(i) * sensor->n_cols + j;
        return {bucket_points.data() + bucket_offsets[q], bucket_points.data() + bucket_offsets[q + 1]};
    }
};

/// lambda at (i, j, t): gain x (background + the pixel's points' IRF
/// contributions), likelihood.hpp:65-77.  Host: the forward model.
inline double rate(const SceneState& state, int i, int j, double t) {
    const SensorModel& sensor = *state.sensor;
    const double g = sensor.effective_gain(i, j);
    if (g == 0.0) return 0.0;
    const Irf& irf = sensor.irf(i, j);
    double lam = state.background(i, j);
    for (auto [b, e] = state.pixel_points(i, j); b != e; ++b)
        lam += state.cloud[*b].intensity * irf.value(t - state.cloud[*b].t);
    return g * lam;
}

/// rate() at every bin of one pixel (likelihood.hpp:80-95), accumulated
/// point by point over each point's IRF support.
inline std::vector<double> rate_profile(const SceneState& state, int i, int j) {
    const SensorModel& sensor = *state.sensor;
    std::vector<double> lam(sensor.n_bins, 0.0);
    const double g = sensor.effective_gain(i, j);
    if (g == 0.0) return lam;
    const double base = g * state.background(i, j);
    for (double& v : lam) v = base;
    const Irf& irf = sensor.irf(i, j);
    for (auto [b, e] = state.pixel_points(i, j); b != e; ++b) {
        const Point& p = state.cloud[*b];
        const auto [lo, hi] = irf.support_bins(p.t, sensor.n_bins);
        for (int k = lo; k <= hi; ++k) lam[k] += g * p.intensity * irf.value(k - p.t);
    }
    return lam;
}

namespace detail {

inline void check_dims(const SceneState& state, const PhotonCube& cube) {
    if (!state.sensor) throw std::invalid_argument("SceneState: null sensor");
    if (state.sensor->n_rows != cube.n_rows || state.sensor->n_cols != cube.n_cols ||
        state.sensor->n_bins != cube.n_bins)
        throw std::invalid_argument("likelihood: state/cube dimension mismatch");
}

/// The state and cube into the calling thread's device session.
inline void upload_state(const SceneState& state, const PhotonCube& cube) {
    check_dims(state, cube);
    b200::set_scene(cube, *state.sensor);
    const rt3d_state_view v{b200::c_points(state.cloud), static_cast<std::uint64_t>(state.cloud.size()),
                            state.background.data.data(), state.bucket_offsets.data(),
                            state.bucket_points.data()};
    b200::check(rt3d_state_upload(b200::session(), &v));
}

}  // namespace detail

/// Poisson negative log-likelihood up to the data-only constant
/// (likelihood.hpp:136-168): +inf for an active bin at zero rate.
inline double nll(const SceneState& state, const PhotonCube& cube) {
    detail::upload_state(state, cube);
    double v = 0.0;
    b200::check(rt3d_nll(b200::session(), &v));
    return v;
}

struct DepthGradient {
    std::vector<double> value;               // d nll / d t_n per point
    std::vector<std::uint32_t> out_of_gate;  // points whose IRF support misses the gate
};

inline DepthGradient grad_depth(const SceneState& state, const PhotonCube& cube) {
    detail::upload_state(state, cube);
    DepthGradient out;
    out.value.assign(state.cloud.size(), 0.0);
    std::vector<std::uint8_t> oog(state.cloud.size(), 0);
    b200::check(rt3d_grad_depth(b200::session(), out.value.data(), oog.data()));
    for (std::uint32_t n = 0; n < oog.size(); ++n)
        if (oog[n]) out.out_of_gate.push_back(n);
    return out;
}

inline std::vector<double> grad_intensity(const SceneState& state, const PhotonCube& cube) {
    detail::upload_state(state, cube);
    std::vector<double> out(state.cloud.size(), 0.0);
    b200::check(rt3d_grad_intensity(b200::session(), out.data()));
    return out;
}

inline Grid2D<double> grad_background(const SceneState& state, const PhotonCube& cube) {
    detail::upload_state(state, cube);
    Grid2D<double> out(cube.n_rows, cube.n_cols, 0.0);
    b200::check(rt3d_grad_background(b200::session(), out.data.data()));
    return out;
}

/// Gauss-Newton diagonals used to precondition "auto" steps.
struct BlockCurvatures {
    std::vector<double> depth;
    std::vector<double> intensity;
    Grid2D<double> background;
};

inline BlockCurvatures block_curvatures(const SceneState& state, const PhotonCube& cube) {
    detail::upload_state(state, cube);
    BlockCurvatures out;
    out.depth.assign(state.cloud.size(), 0.0);
    out.intensity.assign(state.cloud.size(), 0.0);
    out.background = Grid2D<double>(cube.n_rows, cube.n_cols, 0.0);
    b200::check(rt3d_block_curvatures(b200::session(), out.depth.data(), out.intensity.data(),
                                      out.background.data.data()));
    return out;
}

}  // namespace splidar
