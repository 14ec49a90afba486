// splidar/cloud.hpp — drop-in replacement (B200 build) for the reference's
// proj/include/splidar/cloud.hpp: the same Point / PointCloud / PointFlags,
// with an Eigen-free Vec3 (the reference aliases Eigen::Vector3d,
// cloud.hpp:10) that offers the member API the reference's headers and tests
// use (x()/y()/z(), Zero(), norm(), squaredNorm(), dot(), arithmetic, ==).
//
// Put repo/include ahead of the reference's include directory: the
// hot-path headers (cloud, likelihood, spatial_index, denoise, reconstruct)
// then resolve to these, which run on the GPU through include/rt3d.h; the
// reference's other headers (cube, grid, sensor, parallel, config, io,
// simulate, eval, ...) are Eigen-free and compile unchanged against them.
#pragma once

#include <cmath>
#include <cstddef>
#include <cstdint>
#include <vector>

namespace splidar {

/// Three doubles, laid out like Eigen::Vector3d (24 bytes, x y z).  Norms
/// and dot products sum left to right, ((x x + y y) + z z).
class Vec3 {
public:
    Vec3() = default;
    Vec3(double x, double y, double z) : v_{x, y, z} {}
    static Vec3 Zero() { return Vec3(0.0, 0.0, 0.0); }

    double& x() { return v_[0]; }
    double& y() { return v_[1]; }
    double& z() { return v_[2]; }
    double x() const { return v_[0]; }
    double y() const { return v_[1]; }
    double z() const { return v_[2]; }
    double& operator[](std::size_t k) { return v_[k]; }
    double operator[](std::size_t k) const { return v_[k]; }
    double& operator()(std::size_t k) { return v_[k]; }
    double operator()(std::size_t k) const { return v_[k]; }

    double dot(const Vec3& o) const { return v_[0] * o.v_[0] + v_[1] * o.v_[1] + v_[2] * o.v_[2]; }
    double squaredNorm() const { return dot(*this); }
    double norm() const { return std::sqrt(squaredNorm()); }

    Vec3& operator+=(const Vec3& o) {
        for (int k = 0; k < 3; ++k) v_[k] += o.v_[k];
        return *this;
    }
    Vec3& operator-=(const Vec3& o) {
        for (int k = 0; k < 3; ++k) v_[k] -= o.v_[k];
        return *this;
    }
    Vec3& operator*=(double s) {
        for (double& c : v_) c *= s;
        return *this;
    }
    Vec3& operator/=(double s) {
        for (double& c : v_) c /= s;
        return *this;
    }
    friend Vec3 operator+(Vec3 a, const Vec3& b) { return a += b; }
    friend Vec3 operator-(Vec3 a, const Vec3& b) { return a -= b; }
    friend Vec3 operator-(const Vec3& a) { return Vec3(-a.v_[0], -a.v_[1], -a.v_[2]); }
    friend Vec3 operator*(Vec3 a, double s) { return a *= s; }
    friend Vec3 operator*(double s, Vec3 a) { return a *= s; }
    friend Vec3 operator/(Vec3 a, double s) { return a /= s; }
    friend bool operator==(const Vec3& a, const Vec3& b) {
        return a.v_[0] == b.v_[0] && a.v_[1] == b.v_[1] && a.v_[2] == b.v_[2];
    }
    friend bool operator!=(const Vec3& a, const Vec3& b) { return !(a == b); }

private:
    double v_[3] = {0.0, 0.0, 0.0};
};

enum PointFlags : std::uint8_t {
    kFlagIsolated = 1,    // fewer than min_neighbors inside the APSS kernel
    kFlagOutOfGate = 2,   // IRF support entirely outside the time gate
    kFlagDegenerate = 4,  // the sphere / plane fit was unusable
};

/// One surface point (cloud.hpp:18-25); 64 bytes, the layout of rt3d_point.
struct Point {
    Vec3 position = Vec3::Zero();  // world metres
    double intensity = 0.0;
    int i = 0, j = 0;              // home coarse pixel
    int fi = 0, fj = 0;            // fine transverse index
    double t = 0.0;                // depth in bins
    std::uint8_t flags = 0;
};

struct PointCloud {
    std::vector<Point> points;

    std::size_t size() const { return points.size(); }
    bool empty() const { return points.empty(); }
    Point& operator[](std::size_t n) { return points[n]; }
    const Point& operator[](std::size_t n) const { return points[n]; }
    auto begin() { return points.begin(); }
    auto end() { return points.end(); }
    auto begin() const { return points.begin(); }
    auto end() const { return points.end(); }
};

}  // namespace splidar
