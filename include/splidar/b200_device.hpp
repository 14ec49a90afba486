// splidar/b200_device.hpp — the device side of the drop-in headers: one
// rt3d_session per host thread (include/rt3d.h), marshalling of the
// reference's types into the C ABI's plain structs, and the mapping of the
// C ABI's status codes onto the exceptions the reference throws
// (std::invalid_argument, splidar::FormatError, std::out_of_range).
// There is no CPU fallback: without a device every call throws
// splidar::b200::Error (RT3D_ERR_NO_DEVICE).
#pragma once

#include "rt3d.h"

#include "splidar/cloud.hpp"
#include "splidar/cube.hpp"
#include "splidar/grid.hpp"
#include "splidar/sensor.hpp"

#include <cstddef>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

namespace splidar::b200 {

/// Device / CUDA failures (statuses without a reference exception type).
class Error : public std::runtime_error {
public:
    Error(rt3d_status st, const std::string& what) : std::runtime_error(what), status(st) {}
    rt3d_status status;
};

inline void check(rt3d_status st) {
    if (st == RT3D_OK) return;
    const std::string msg = rt3d_last_error();
    switch (st) {
    case RT3D_ERR_INVALID_ARGUMENT: throw std::invalid_argument(msg);
    case RT3D_ERR_FORMAT: throw FormatError(msg);
    case RT3D_ERR_OUT_OF_RANGE: throw std::out_of_range(msg);
    default: throw Error(st, msg);
    }
}

/// The calling thread's session (device RT3D_DEVICE, default 0), created on
/// first use and kept warm across calls.
inline rt3d_session* session() {
    struct Holder {
        rt3d_session* s = nullptr;
        ~Holder() {
            if (s) rt3d_session_destroy(s);
        }
    };
    thread_local Holder h;
    if (!h.s) {
        const char* dev = std::getenv("RT3D_DEVICE");
        check(rt3d_session_create(dev ? std::atoi(dev) : 0, &h.s));
    }
    return h.s;
}

static_assert(sizeof(Point) == sizeof(rt3d_point), "Point is laid out as rt3d_point");
static_assert(offsetof(Point, intensity) == offsetof(rt3d_point, intensity), "Point layout");
static_assert(offsetof(Point, i) == offsetof(rt3d_point, i), "Point layout");
static_assert(offsetof(Point, t) == offsetof(rt3d_point, t), "Point layout");
static_assert(offsetof(Point, flags) == offsetof(rt3d_point, flags), "Point layout");
static_assert(sizeof(Event) == sizeof(rt3d_event), "Event layout");

inline const rt3d_point* c_points(const PointCloud& c) {
    return reinterpret_cast<const rt3d_point*>(c.points.data());
}
inline rt3d_point* c_points(PointCloud& c) { return reinterpret_cast<rt3d_point*>(c.points.data()); }

inline rt3d_irf irf_view(const Irf& irf) {
    return rt3d_irf{irf.tau_min(), irf.dtau(), irf.samples().data(),
                    static_cast<std::uint64_t>(irf.samples().size())};
}

/// rt3d_sensor borrowing the SensorModel's arrays (per_pixel keeps the
/// per-pixel IRF views alive for the call).
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

inline rt3d_cube cube_view(const PhotonCube& cube) {
    return rt3d_cube{cube.n_rows, cube.n_cols, cube.n_bins, 0, cube.bin_width_s,
                     cube.offsets.data(), reinterpret_cast<const rt3d_event*>(cube.events.data()),
                     static_cast<std::uint64_t>(cube.events.size())};
}

inline void set_sensor(const SensorModel& sensor) {
    SensorView v(sensor);
    check(rt3d_set_sensor(session(), &v.c));
}

inline void set_scene(const PhotonCube& cube, const SensorModel& sensor) {
    set_sensor(sensor);
    const rt3d_cube c = cube_view(cube);
    check(rt3d_set_cube(session(), &c));
}

/// The session's state -> cloud (cloud order) and background.
inline void download(int rows, int cols, PointCloud& cloud, Grid2D<double>& bg) {
    std::uint64_t n = 0;
    check(rt3d_state_size(session(), &n));
    cloud.points.assign(n, Point{});
    bg = Grid2D<double>(rows, cols, 0.0);
    check(rt3d_state_copy(session(), c_points(cloud), bg.data.data()));
}

}  // namespace splidar::b200
