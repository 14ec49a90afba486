// splidar/denoise.hpp — drop-in replacement (B200 build) for the reference's
// denoise.hpp:24-323: the plug-and-play denoisers of the PALM loop, on the
// GPU (no Eigen, no FFTW).
//
//   apss_project           denoise.hpp:159-217  rt3d_apss_project (Pratt sphere
//                                                fit by bisection, 1e-11 from QZ)
//   knn_intensity_filter   denoise.hpp:223-237  rt3d_knn_intensity_filter
//   prune                  denoise.hpp:241-248  rt3d_prune (stable compaction)
//   fft_lowpass_filter     denoise.hpp:267-311  rt3d_fft_lowpass_filter
//   fft_background_denoise denoise.hpp:315-319  (the same, clamped at zero)
//   identity_background    denoise.hpp:323
//
// The neighbour searches use the SpatialIndex's cloud and cell size: the
// device rebuilds the index's cell grid and answers its ball / kNN queries.
#pragma once

#include "splidar/b200_device.hpp"
#include "splidar/cloud.hpp"
#include "splidar/grid.hpp"
#include "splidar/spatial_index.hpp"

#include <cstdint>
#include <stdexcept>
#include <vector>

namespace splidar {

/// APSS kernel and fit parameters (denoise.hpp:24-45).
struct ApssParams {
    double kernel_radius = 0.1;           // metres
    int min_neighbors = 6;                // >= 4, the query point included
    double sphere_degeneracy_eps = 1e-3;  // |u_q| below this: plane

    void validate() const {
        if (kernel_radius <= 0.0)
            throw std::invalid_argument("ApssParams: kernel_radius must be positive");
        if (min_neighbors < 4) throw std::invalid_argument("ApssParams: min_neighbors must be >= 4");
        if (sphere_degeneracy_eps < 0.0)
            throw std::invalid_argument("ApssParams: sphere_degeneracy_eps must be >= 0");
    }

    /// (1 - (d / R)^2)^4 inside the kernel radius, 0 outside.
    double weight(double dist) const {
        const double x = dist / kernel_radius;
        if (x >= 1.0) return 0.0;
        double s = 1.0 - x * x;
        s *= s;
        return s * s;
    }
};

inline PointCloud apss_project(const PointCloud& cloud, const ApssParams& params,
                               const SpatialIndex& index) {
    params.validate();
    const PointCloud& idx = index.indexed_cloud();
    const rt3d_apss_params p{params.kernel_radius, params.sphere_degeneracy_eps,
                             params.min_neighbors, 0};
    PointCloud out;
    out.points.resize(cloud.size());
    b200::check(rt3d_apss_project(b200::session(), b200::c_points(cloud), cloud.size(), &p,
                                  b200::c_points(idx), idx.size(), index.cell_size(),
                                  b200::c_points(out)));
    return out;
}

inline PointCloud knn_intensity_filter(const PointCloud& cloud, int k, const SpatialIndex& index,
                                       double radius) {
    if (k < 1) throw std::invalid_argument("knn_intensity_filter: k must be >= 1");
    if (radius <= 0.0) throw std::invalid_argument("knn_intensity_filter: radius must be positive");
    const PointCloud& idx = index.indexed_cloud();
    PointCloud out;
    out.points.resize(cloud.size());
    b200::check(rt3d_knn_intensity_filter(b200::session(), b200::c_points(cloud), cloud.size(), k,
                                          b200::c_points(idx), idx.size(), index.cell_size(), radius,
                                          b200::c_points(out)));
    return out;
}

inline PointCloud prune(const PointCloud& cloud, double r_min) {
    if (r_min < 0.0) throw std::invalid_argument("prune: r_min must be >= 0");
    PointCloud out;
    out.points.resize(cloud.size());
    std::uint64_t n = 0;
    b200::check(rt3d_prune(b200::session(), b200::c_points(cloud), cloud.size(), r_min,
                           b200::c_points(out), &n));
    out.points.resize(n);
    return out;
}

inline Grid2D<double> fft_lowpass_filter(const Grid2D<double>& img, double cutoff) {
    Grid2D<double> out(img.rows, img.cols, 0.0);
    b200::check(rt3d_fft_lowpass_filter(b200::session(), img.data.data(), img.rows, img.cols, cutoff,
                                        0, out.data.data()));
    return out;
}

inline BackgroundImage fft_background_denoise(const BackgroundImage& b, double cutoff) {
    Grid2D<double> out(b.rows, b.cols, 0.0);
    b200::check(rt3d_fft_lowpass_filter(b200::session(), b.data.data(), b.rows, b.cols, cutoff, 1,
                                        out.data.data()));
    return out;
}

inline BackgroundImage identity_background(const BackgroundImage& b) { return b; }

}  // namespace splidar
