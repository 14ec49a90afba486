// Output formats after the path: the reconstructed
// cloud as the reference's ASCII PLY (encode_ply, io.hpp:162-179) and the
// background image as the CLI's CSV (tools/splidar_main.cpp:204-212).
//
// Text formatting is host work in the reference too; here the cloud comes
// off the device once (rt3d_state_copy) and the per-line snprintf calls are
// split over host threads in contiguous point ranges, each range formatted
// into its own buffer and the buffers concatenated in order, so the bytes are
// identical to the reference's single-threaded ostringstream for any thread
// count.  Two-call convention: buf == NULL (or cap too small) only reports
// the size in *n_bytes.
#include <algorithm>
#include <cstdio>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#include "../../include/rt3d.h"

namespace {

constexpr uint64_t kMinPerThread = 1u << 14;  // below this, threads cost more than they save

unsigned worker_count(uint64_t n) {
    unsigned hw = std::max(1u, std::thread::hardware_concurrency());
    uint64_t want = (n + kMinPerThread - 1) / kMinPerThread;
    return (unsigned)std::max<uint64_t>(1, std::min<uint64_t>(hw, want));
}

// Format items [0, n) with fmt_one(i, std::string&) over contiguous ranges.
template <class F>
std::string format_ranges(uint64_t n, F fmt_one) {
    const unsigned w = worker_count(n);
    std::vector<std::string> parts(w);
    auto run = [&](unsigned k) {
        const uint64_t lo = n * k / w, hi = n * (k + 1) / w;
        std::string& s = parts[k];
        s.reserve((hi - lo) * 64);
        for (uint64_t i = lo; i < hi; ++i) fmt_one(i, s);
    };
    if (w == 1) {
        run(0);
        return std::move(parts[0]);
    }
    std::vector<std::thread> th;
    for (unsigned k = 1; k < w; ++k) th.emplace_back(run, k);
    run(0);
    for (auto& t : th) t.join();
    size_t total = 0;
    for (auto& p : parts) total += p.size();
    std::string out;
    out.reserve(total);
    for (auto& p : parts) out += p;
    return out;
}

rt3d_status deliver(const std::string& s, char* buf, uint64_t cap, uint64_t* n_bytes) {
    *n_bytes = s.size();
    if (buf && cap >= s.size()) std::memcpy(buf, s.data(), s.size());
    return RT3D_OK;
}

}  // namespace

extern "C" {

// encode_ply (io.hpp:162-179)
rt3d_status rt3d_encode_ply(const rt3d_point* points, uint64_t n, int32_t has_pixel_pitch,
                            double pixel_pitch, char* buf, uint64_t cap, uint64_t* n_bytes) {
    if (!n_bytes || (n && !points)) return RT3D_ERR_INVALID_ARGUMENT;
    std::string head = "ply\nformat ascii 1.0\n";
    char line[160];
    if (has_pixel_pitch) {
        std::snprintf(line, sizeof line, "comment pixel_pitch %.17g\n", pixel_pitch);
        head += line;
    }
    head += "element vertex " + std::to_string(n) + "\n";
    head += "property float x\nproperty float y\nproperty float z\n"
            "property float intensity\nend_header\n";
    std::string body = format_ranges(n, [&](uint64_t i, std::string& s) {
        char b[160];
        const rt3d_point& p = points[i];
        int k = std::snprintf(b, sizeof b, "%.9g %.9g %.9g %.9g\n", p.x, p.y, p.z, p.intensity);
        s.append(b, (size_t)k);
    });
    return deliver(head + body, buf, cap, n_bytes);
}

// background CSV written by `splidar reconstruct --background-out`
// (tools/splidar_main.cpp:204-212): row-major, "%.9g", ',' between columns.
rt3d_status rt3d_encode_background_csv(const double* background, int32_t rows, int32_t cols,
                                       char* buf, uint64_t cap, uint64_t* n_bytes) {
    if (!n_bytes || rows < 0 || cols < 0 || (rows && cols && !background))
        return RT3D_ERR_INVALID_ARGUMENT;
    const uint64_t npix = (uint64_t)rows * (uint64_t)cols;
    std::string s = format_ranges(npix, [&](uint64_t i, std::string& out) {
        char b[64];
        int k = std::snprintf(b, sizeof b, "%.9g", background[i]);
        out.append(b, (size_t)k);
        out.push_back((int64_t)(i % (uint64_t)cols) + 1 == cols ? '\n' : ',');
    });
    return deliver(s, buf, cap, n_bytes);
}

}  // extern "C"
