// rt3d.cu — librt3d.so: the B200 RT3D path behind include/rt3d.h.
//
// One persistent cooperative kernel runs a whole frame (init + PALM
// iterations, reconstruct.hpp:457-489): every data-dependent decision of the
// reference (backtracking accept/reject, reconstruct.hpp:274-292; the stop
// rule, :475-477; prune counts) is taken on the device between grid
// barriers, so a frame is one launch with no host round trip.  The same
// device phases serve the fine-grained operators (nll, gradients, init,
// palm_step) through the program switch.
#include <cub/cub.cuh>
#include <cuda_runtime.h>
#include <nvtx3/nvToolsExt.h>

#include <algorithm>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/rt3d.h"
#include "rt3d_frame.cuh"
#include "rt3d_nbr.cuh"
#include "rt3d_stage.cuh"
#include "rt3d_sim.cuh"

namespace {
// NVTX range over a public entry point (header-only NVTX v3: a no-op unless a
// profiler injects itself), so an nsys/ncu timeline shows the API calls around
// the kernels and the graph replays.
struct NvtxRange {
    explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
    ~NvtxRange() { nvtxRangePop(); }
    NvtxRange(const NvtxRange&) = delete;
    NvtxRange& operator=(const NvtxRange&) = delete;
};
}  // namespace

using namespace rt3d;

static_assert(sizeof(StepDiagDev) == sizeof(rt3d_step_diag), "diag layout");
static_assert(sizeof(rt3d_point) == 64, "point layout");

// ===========================================================================
// device: persistent frame kernel
// ===========================================================================
namespace rt3d {

// the stage kernels of each lane-group configuration (rt3d_stage_g*.cu)
StageFn stage_fn_g4(int st);
StageFn stage_fn_g32(int st);
StageFn stage_fn_g3(int st);
StageFn stage_fn_g1(int st);

#define BATCH_FRAME(FB) (FB).f[(FB).n == 1 ? 0u : (FB).first + blockIdx.x / (FB).bpf]

#ifndef RT3D_APSS_MIN_BLOCKS
#define RT3D_APSS_MIN_BLOCKS 5
#endif
__global__ void __launch_bounds__(kNbrBlock, RT3D_APSS_MIN_BLOCKS) apss_kernel(const __grid_constant__ FrameBatch FB) {
    const Frame& F = BATCH_FRAME(FB);
    extern __shared__ __align__(16) unsigned char smem_raw[];
    if (ld_cg(&F.ctl->stop) || ld_cg(&F.ctl->abort)) return;
    stamp(F, PH_APSS);
    apss_moment_warps(F, reinterpret_cast<ApssWarpSm*>(smem_raw), ld_cg(&F.ctl->pbase),
                      ld_cg(&F.ctl->pown), ld_cg(&F.ctl->tc), ld_cg(&F.ctl->sc), kNbrWarps);
}

__global__ void __launch_bounds__(kFitBlock) apss_fit_kernel(const __grid_constant__ FrameBatch FB) {
    const Frame& F = BATCH_FRAME(FB);
    if (ld_cg(&F.ctl->stop) || ld_cg(&F.ctl->abort)) return;
    stamp(F, PH_APSS_FIT);
    apss_fit_threads(F, ld_cg(&F.ctl->pbase), ld_cg(&F.ctl->pown), ld_cg(&F.ctl->tc),
                     ld_cg(&F.ctl->sc));
}

// the fit of a latency-bound launch (one or two frames): eigenvalues and the
// Pratt solve on separate threads, side by side (apss_fit_split)
__global__ void __launch_bounds__(128) apss_fit_split_kernel(const __grid_constant__ FrameBatch FB) {
    const Frame& F = BATCH_FRAME(FB);
    if (ld_cg(&F.ctl->stop) || ld_cg(&F.ctl->abort)) return;
    stamp(F, PH_APSS_FIT);
    apss_fit_split(F, ld_cg(&F.ctl->pbase), ld_cg(&F.ctl->pown), ld_cg(&F.ctl->tc),
                   ld_cg(&F.ctl->sc));
}

__global__ void __launch_bounds__(kNbrBlock, 7) knn_kernel(const __grid_constant__ FrameBatch FB) {
    const Frame& F = BATCH_FRAME(FB);
    extern __shared__ __align__(16) unsigned char smem_raw[];
    if (ld_cg(&F.ctl->stop) || ld_cg(&F.ctl->abort)) return;
    stamp(F, PH_LAUNCH);
    // pairs by ticket on large clouds only: on small ones the one counter
    // per frame is contended (B, C: kNN +25-50 %)
    const uint32_t P = ld_cg(&F.ctl->pown);
    knn_warps<1>(F, reinterpret_cast<KnnWarpSm*>(smem_raw), ld_cg(&F.ctl->pbase), P, ld_cg(&F.ctl->tc),
                 ld_cg(&F.ctl->rc), ld_cg(&F.ctl->sc), P >= (1u << 20));
}

// every point to its final window in one kernel (superres frames: their
// first windows are small, and most points need the wider one)
__global__ void __launch_bounds__(kNbrBlock, 7) knn_full_kernel(const __grid_constant__ FrameBatch FB) {
    const Frame& F = BATCH_FRAME(FB);
    extern __shared__ __align__(16) unsigned char smem_raw[];
    if (ld_cg(&F.ctl->stop) || ld_cg(&F.ctl->abort)) return;
    stamp(F, PH_LAUNCH);
    const uint32_t P = ld_cg(&F.ctl->pown);
    knn_warps<0>(F, reinterpret_cast<KnnWarpSm*>(smem_raw), ld_cg(&F.ctl->pbase), P, ld_cg(&F.ctl->tc),
                 ld_cg(&F.ctl->rc), ld_cg(&F.ctl->sc), P >= (1u << 20));
}

// the points knn_kernel left for a wider window, over the full ball
__global__ void __launch_bounds__(kNbrBlock, 7) knn_rescan_kernel(const __grid_constant__ FrameBatch FB) {
    const Frame& F = BATCH_FRAME(FB);
    extern __shared__ __align__(16) unsigned char smem_raw[];
    if (ld_cg(&F.ctl->stop) || ld_cg(&F.ctl->abort)) return;
    if (ld_cg(&F.ctl->knn_nres) == 0u) return;
    knn_warps<2>(F, reinterpret_cast<KnnWarpSm*>(smem_raw), 0u, 0u, ld_cg(&F.ctl->tc),
                 ld_cg(&F.ctl->rc), ld_cg(&F.ctl->sc));
}

// Depth intervals of the blocks of F.zbs consecutive points of each pixel
// (thread per block) for the APSS scan's block culling (ball_scan_blocks)
__global__ void zblock_kernel(const __grid_constant__ FrameBatch FB) {
    const Frame& F = BATCH_FRAME(FB);
    if (ld_cg(&F.ctl->stop) || ld_cg(&F.ctl->abort)) return;
    const int tc = ld_cg(&F.ctl->tc), sc = ld_cg(&F.ctl->sc);
    const uint32_t nb = F.npix * F.zkb;
    const uint32_t* bo = F.bo[sc];
    const double* t = F.t[tc];
    for (uint32_t b = vblock(F) * blockDim.x + threadIdx.x; b < nb; b += vgrid(F) * blockDim.x) {
        const uint32_t p = b / F.zkb, k = b - p * F.zkb;
        const uint32_t n1 = bo[p + 1], lo = bo[p] + k * F.zbs;
        const uint32_t hi = lo + F.zbs < n1 ? lo + F.zbs : n1;
        double zmin = INFINITY, zmax = -INFINITY;
        for (uint32_t n = lo; n < hi; ++n) {
            const double z = t[n] * F.bres;
            zmin = z < zmin ? z : zmin;
            zmax = z > zmax ? z : zmax;
        }
        F.zb[b] = make_double2(zmin, zmax);
    }
}

// Row bands: every band keeps full-size arrays in the global
// index space (pixels and points), so a halo is a plain copy of the
// neighbouring bands' rows into this band's arrays at the same indices:
// the bucket offsets of the halo pixels and, for their points, t and the
// fine cells (what & 1: before APSS) and t and r (what & 2: before kNN).
// The neighbours' buffers are read directly (the same device here; peer
// memory over NVLink when the bands sit on different GPUs).
__global__ void halo_kernel(const __grid_constant__ FrameBatch FB, int what) {
    const uint32_t k = FB.first + blockIdx.x / FB.bpf;
    const Frame& F = FB.f[k];
    if (ld_cg(&F.ctl->stop) || ld_cg(&F.ctl->abort)) return;
    const uint32_t nth = FB.bpf * blockDim.x;
    const uint32_t tid = (blockIdx.x - F.blk0) * blockDim.x + threadIdx.x;
    const int tc = ld_cg(&F.ctl->tc), rc = ld_cg(&F.ctl->rc), sc = ld_cg(&F.ctl->sc);
    for (int side = 0; side < 2; ++side) {
        const int j = (int)k + (side ? 1 : -1);
        if (j < 0 || j >= (int)FB.n) continue;
        const Frame& N = FB.f[j];
        uint32_t p0, p1;  // the halo pixels, owned by band j
        if (side == 0) {
            p0 = F.bpix0 > F.halo_px ? F.bpix0 - F.halo_px : 0u;
            p1 = F.bpix0;
        } else {
            p0 = F.bpix1;
            p1 = F.bpix1 + F.halo_px < F.npix ? F.bpix1 + F.halo_px : F.npix;
        }
        const uint32_t* nbo = N.bo[sc];
        uint32_t* obo = F.bo[sc];
        if (what & 1)  // bo[p0 .. p1) above (bo[bpix0] is ours), bo(p0 .. p1] below
            for (uint32_t q = tid; q < p1 - p0; q += nth) {
                const uint32_t p = side ? p0 + 1 + q : p0 + q;
                obo[p] = ld_cg(&nbo[p]);
            }
        const uint32_t n0 = ld_cg(&nbo[p0]), n1 = ld_cg(&nbo[p1]);
        RT3D_CHECK(n0 <= n1 && n1 <= F.pcap && p1 <= F.npix);
        for (uint32_t n = n0 + tid; n < n1; n += nth) {
            F.t[tc][n] = ld_cg(&N.t[tc][n]);
            if (what & 2) F.r[rc][n] = ld_cg(&N.r[rc][n]);
            if (what & 1) {
                F.fi[sc][n] = ld_cg(&N.fi[sc][n]);
                F.fj[sc][n] = ld_cg(&N.fj[sc][n]);
            }
        }
    }
}

// FP64 vector throughput probe (the roof of the FP64-issue-bound kernels,
// rt3d_measure_fp64_peak): 8 independent DFMA chains per thread.
__global__ void fp64_peak_kernel(double* out, int iters, double a, double b) {
    double x[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) x[k] = 1e-3 * (threadIdx.x + k);
    for (int i = 0; i < iters; ++i)
#pragma unroll
        for (int k = 0; k < 8; ++k) x[k] = __fma_rn(x[k], a, b);
    double acc = 0.0;
#pragma unroll
    for (int k = 0; k < 8; ++k) acc += x[k];
    if (acc == 12345.678) out[blockIdx.x * blockDim.x + threadIdx.x] = acc;  // keeps the chains live
}

// ---------------------------------------------------------------------------
// Operators on arbitrary clouds (denoise.hpp:159-248) through a device
// SpatialIndex (spatial_index.hpp:18-77): the index cloud sorted by the
// reference's cell key (cell = the index's cell size, 21-bit packing), stably
// so a cell's points stay in ascending index order, plus the sorted unique
// keys and their start slots.  A query visits the 27 cells around q, merges
// their (ascending) slot runs by point index and keeps |q - p|^2 <= r^2: the
// ball in ascending index order, SpatialIndex::query's answer.
// ---------------------------------------------------------------------------
struct CloudSoA {
    const double* x;  // sorted slot order
    const double* y;
    const double* z;
    const double* r;
    uint32_t n;
    const uint32_t* order;         // slot -> point index
    const unsigned long long* ukey;  // ncell sorted unique cell keys
    const uint32_t* ustart;        // ncell + 1 slot starts
    uint32_t ncell;
    double cell;
};

__host__ __device__ __forceinline__ unsigned long long cell_pack(long long x, long long y, long long z) {
    auto u = [](long long v) {
        return (unsigned long long)(v + (1ll << 20)) & ((1ull << 21) - 1);
    };
    return (u(x) << 42) | (u(y) << 21) | u(z);
}
__device__ __forceinline__ long long cell_coord(double v, double cell) {
    return (long long)floor(v / cell);
}

template <typename Fn>
__device__ __forceinline__ void for_each_grid(const CloudSoA& c, const Pos& q, double r2, Fn fn) {
    uint32_t b[27], e[27];
    const long long cx = cell_coord(q.x, c.cell), cy = cell_coord(q.y, c.cell),
                    cz = cell_coord(q.z, c.cell);
    int nr = 0;
    for (long long a = cx - 1; a <= cx + 1; ++a)
        for (long long bb = cy - 1; bb <= cy + 1; ++bb)
            for (long long cc = cz - 1; cc <= cz + 1; ++cc) {
                const unsigned long long k = cell_pack(a, bb, cc);
                uint32_t lo = 0, hi = c.ncell;
                while (lo < hi) {
                    const uint32_t mid = (lo + hi) >> 1;
                    if (c.ukey[mid] < k) lo = mid + 1;
                    else hi = mid;
                }
                if (lo < c.ncell && c.ukey[lo] == k) {
                    b[nr] = c.ustart[lo];
                    e[nr] = c.ustart[lo + 1];
                    ++nr;
                }
            }
    for (;;) {  // merge the runs by point index
        int best = -1;
        uint32_t bi = 0xffffffffu;
        for (int t = 0; t < nr; ++t)
            if (b[t] < e[t] && c.order[b[t]] < bi) {
                bi = c.order[b[t]];
                best = t;
            }
        if (best < 0) break;
        const uint32_t slot = b[best]++;
        Pos o{c.x[slot], c.y[slot], c.z[slot]};
        const double dx = o.x - q.x, dy = o.y - q.y, dz = o.z - q.z;
        const double d2 = dx * dx + dy * dy + dz * dz;
        if (d2 <= r2) fn(bi, o, d2);
    }
}

// the grid: keys, then (after the sort) run starts and the slot-ordered SoA
__global__ void grid_keys_kernel(const rt3d_point* in, uint32_t n, double cell,
                                 unsigned long long* key, uint32_t* idx) {
    const uint32_t k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= n) return;
    key[k] = cell_pack(cell_coord(in[k].x, cell), cell_coord(in[k].y, cell), cell_coord(in[k].z, cell));
    idx[k] = k;
}
__global__ void grid_flags_kernel(const unsigned long long* key, uint32_t n, uint32_t* flag) {
    const uint32_t k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k < n) flag[k] = (k == 0 || key[k] != key[k - 1]) ? 1u : 0u;
}
__global__ void grid_fill_kernel(const rt3d_point* in, const unsigned long long* key,
                                 const uint32_t* order, const uint32_t* flag, const uint32_t* pos,
                                 uint32_t n, unsigned long long* ukey, uint32_t* ustart, double* x,
                                 double* y, double* z, double* r) {
    const uint32_t k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= n) return;
    if (flag[k]) {
        ukey[pos[k]] = key[k];
        ustart[pos[k]] = k;
    }
    if (k == n - 1) ustart[pos[k] + flag[k]] = n;
    const rt3d_point p = in[order[k]];
    x[k] = p.x;
    y[k] = p.y;
    z[k] = p.z;
    r[k] = p.intensity;
}

__global__ void apss_general_kernel(const rt3d_point* in, uint32_t n, CloudSoA idx, double R,
                                    int min_nbrs, double eps, rt3d_point* out) {
    uint32_t k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= n) return;
    rt3d_point p = in[k];
    Pos q{p.x, p.y, p.z};
    uint8_t fl = p.flags & (uint8_t)~(1u | 4u);
    Pos o;
    auto each = [&](double r2, auto fn) { for_each_grid(idx, q, r2, fn); };
    if (apss_point(each, q, R, min_nbrs, eps, fl, o)) {
        p.x = o.x;
        p.y = o.y;
        p.z = o.z;
    }
    p.flags = fl;
    out[k] = p;
}

__global__ void knn_general_kernel(const rt3d_point* in, uint32_t n, CloudSoA idx, int kk,
                                   double radius, const rt3d_point* index_aos, rt3d_point* out) {
    uint32_t k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= n) return;
    rt3d_point p = in[k];
    Pos q{p.x, p.y, p.z};
    auto each = [&](double r2, auto fn) { for_each_grid(idx, q, r2, fn); };
    p.intensity = knn_mean(each, kk, radius * radius, p.intensity,
                           [&](uint32_t m) { return index_aos[m].intensity; });
    out[k] = p;
}

__global__ void split_cloud_kernel(const rt3d_point* in, uint32_t n, double* x, double* y,
                                   double* z, double* r) {
    uint32_t k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= n) return;
    x[k] = in[k].x;
    y[k] = in[k].y;
    z[k] = in[k].z;
    r[k] = in[k].intensity;
}

// prune on an arbitrary cloud (denoise.hpp:241-248): keep flags, an
// exclusive scan (CUB), a stable scatter
__global__ void prune_flags_kernel(const rt3d_point* in, uint32_t n, double rmin, uint32_t* flag) {
    const uint32_t k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k < n) flag[k] = in[k].intensity >= rmin ? 1u : 0u;
}
__global__ void prune_scatter_kernel(const rt3d_point* in, uint32_t n, const uint32_t* flag,
                                     const uint32_t* pos, rt3d_point* out, uint32_t* total) {
    const uint32_t k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= n) return;
    if (flag[k]) out[pos[k]] = in[k];
    if (k == n - 1) *total = pos[k] + flag[k];
}

__global__ void fft_kernel(const double* img, double* out, double* re, double* im, double* re2,
                           double* im2, int nr, int nc, double cutoff, int clamp_nonneg) {
    cg::grid_group grid = cg::this_grid();
    const uint32_t nth = gridDim.x * blockDim.x;
    const uint32_t gtid = blockIdx.x * blockDim.x + threadIdx.x;
    if (fft_pow2(nr) && fft_pow2(nc)) {  // radix 2 (lines in dynamic shared memory)
        extern __shared__ double fft_smem[];
        double* s_re = fft_smem;
        double* s_im = fft_smem + kFftMax;
        fftp_rows_forward(img, re, im, nr, nc, s_re, s_im, blockIdx.x, gridDim.x);
        grid.sync();
        fftp_cols_mask(re, im, nr, nc, cutoff, s_re, s_im, blockIdx.x, gridDim.x);
        grid.sync();
        fftp_rows_backward(re, im, out, nr, nc, clamp_nonneg, s_re, s_im, blockIdx.x, gridDim.x);
        return;
    }
    fft_stage1(img, re, im, nr, nc, gtid, nth);
    grid.sync();
    fft_stage2(re, im, re2, im2, nr, nc, cutoff, gtid, nth);
    grid.sync();
    fft_stage3(re2, im2, re, im, nr, nc, gtid, nth);
    grid.sync();
    fft_stage4(re, im, out, nr, nc, clamp_nonneg, gtid, nth);
}

// SoA state -> AoS rt3d_point (cloud order), positions per world_from_lidar
// (sensor.hpp:200-203) or the baseline's coarse-centre placement
// (eval.hpp:116-118).
// SPCB events of pixel p (io.hpp:131-140) into the device CSR, with
// PhotonCube::validate's per-event checks (cube.hpp:94-106); the first error
// in pixel order is kept as (pixel << 2 | kind) in *err.  Pixel p's record
// starts after the 28-byte header, p + 1 count words and off[p] events.
__global__ void spcb_gather_kernel(const uint32_t* words, const uint32_t* off, uint32_t npix,
                                   uint32_t n_bins, uint2* ev, unsigned long long* err) {
    for (uint32_t p = blockIdx.x * blockDim.x + threadIdx.x; p < npix; p += gridDim.x * blockDim.x) {
        const uint32_t e0 = off[p], e1 = off[p + 1];
        const uint64_t w0 = 7ull + (uint64_t)(p + 1) + 2ull * e0;  // first event word
        uint32_t prev = 0;
        unsigned kind = 0;
        for (uint32_t k = 0; k < e1 - e0; ++k) {
            const uint32_t bin = words[w0 + 2ull * k], count = words[w0 + 2ull * k + 1];
            if (!kind) {
                if (bin >= n_bins) kind = 1;
                else if (count < 1) kind = 2;
                else if (k > 0 && bin <= prev) kind = 3;
            }
            prev = bin;
            ev[e0 + k] = make_uint2(bin, count);
        }
        if (kind) atomicMin(err, ((unsigned long long)p << 2) | kind);
    }
}

// rt3d_set_cube's checks on the device (PhotonCube::validate, cube.hpp:94-106,
// after the host checked the dimensions and the offsets' two ends): pixel p's
// offset range and events, the first error in pixel order (and, within a
// pixel, in event order) kept as (pixel << 3 | kind) in *err, kind 1 negative
// range, 2 bin out of range, 3 zero count, 4 bins not increasing; the 64-bit
// offsets narrowed into the device CSR's 32-bit table on the way.
__global__ void cube_check_kernel(const unsigned long long* off64, uint32_t npix,
                                  unsigned long long n_events, uint32_t n_bins, const uint2* ev,
                                  uint32_t* off32, unsigned long long* err) {
    for (uint32_t p = blockIdx.x * blockDim.x + threadIdx.x; p < npix; p += gridDim.x * blockDim.x) {
        const unsigned long long e0 = off64[p], e1 = off64[p + 1];
        off32[p] = (uint32_t)e0;
        if (p == 0) off32[npix] = (uint32_t)off64[npix];
        unsigned kind = 0;
        if (e0 > e1) {
            kind = 1;
        } else if (e1 <= n_events) {  // (else a later pixel's range is negative)
            uint32_t prev = 0;
            for (unsigned long long k = e0; k < e1 && !kind; ++k) {
                const uint2 e = ev[k];
                if (e.x >= n_bins) kind = 2;
                else if (e.y < 1) kind = 3;
                else if (k > e0 && e.x <= prev) kind = 4;
                prev = e.x;
            }
        }
        if (kind) atomicMin(err, ((unsigned long long)p << 3) | kind);
    }
}

// evaluate (eval.hpp:33-87): column key of every estimate / truth point
// (est first, then truth) -> (key, id); key order = std::map's (cx, cy) order
__global__ void eval_keys_kernel(const rt3d_point* pts, uint32_t n, double pitch,
                                 unsigned long long* keys, uint32_t* ids, unsigned int* bad) {
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        const double fx = floor(pts[i].x / pitch), fy = floor(pts[i].y / pitch);
        const long long cx = (long long)fx, cy = (long long)fy;
        if (!(fabs(fx) < 2147483648.0) || !(fabs(fy) < 2147483648.0)) atomicOr(bad, 1u);
        keys[i] = ((unsigned long long)(cx + 2147483648ll) << 32) |
                  (unsigned long long)(cy + 2147483648ll);
        ids[i] = i;
    }
}

// one thread per column (segment of equal keys): greedy one-to-one matching by
// (err, truth, est) within tau (eval.hpp:51-77); the k-th match of the column
// starting at sorted position p goes to out[p + k] = (err^2, |dr|), its count
// to cnt[p]
constexpr int kEvalCap = 64;
__global__ void eval_match_kernel(const rt3d_point* pts, uint32_t n_est, uint32_t n,
                                  const unsigned long long* keys, const uint32_t* ids, double tau,
                                  double2* out, uint32_t* cnt, unsigned int* bad) {
    for (uint32_t p = blockIdx.x * blockDim.x + threadIdx.x; p < n; p += gridDim.x * blockDim.x) {
        cnt[p] = 0;
        if (p > 0 && keys[p - 1] == keys[p]) continue;
        uint32_t q = p;
        while (q < n && keys[q] == keys[p]) ++q;
        uint32_t es[kEvalCap], ts[kEvalCap];
        int ne = 0, nt = 0;
        for (uint32_t k = p; k < q; ++k) {
            const uint32_t id = ids[k];
            if (id < n_est) {
                if (ne < kEvalCap) es[ne] = id;
                ++ne;
            } else {
                if (nt < kEvalCap) ts[nt] = id - n_est;
                ++nt;
            }
        }
        if (ne > kEvalCap || nt > kEvalCap) {
            atomicOr(bad, 2u);
            continue;
        }
        uint64_t eu = 0, tu = 0;  // used flags
        uint32_t m = 0;
        for (;;) {
            double be = INFINITY;
            uint32_t bt = 0xffffffffu, bs = 0xffffffffu;
            int bi = -1, bj = -1;
            for (int i = 0; i < ne; ++i) {
                if ((eu >> i) & 1u) continue;
                for (int j = 0; j < nt; ++j) {
                    if ((tu >> j) & 1u) continue;
                    const double err = fabs(pts[es[i]].z - pts[n_est + ts[j]].z);
                    if (!(err <= tau)) continue;
                    if (err < be || (err == be && (ts[j] < bt || (ts[j] == bt && es[i] < bs)))) {
                        be = err;
                        bt = ts[j];
                        bs = es[i];
                        bi = i;
                        bj = j;
                    }
                }
            }
            if (bi < 0) break;
            eu |= 1ull << bi;
            tu |= 1ull << bj;
            out[p + m] = make_double2(be * be, fabs(pts[bs].intensity - pts[n_est + bt].intensity));
            ++m;
        }
        cnt[p] = m;
    }
}

// end-of-frame copy for pipelined frames: the cloud (AoS), the background
// and the controller state into a result slot; P and the buffer toggles are
// read on the device, so nothing waits for the frame on the host
__global__ void gather_frame_kernel(Frame F, rt3d_point* out, double* bg, Ctl* ctl_out) {
    const Ctl* c = F.ctl;
    const uint32_t P = ld_cg(&c->P);
    const int tc = ld_cg(&c->tc), rc = ld_cg(&c->rc), bc = ld_cg(&c->bc), sc = ld_cg(&c->sc);
    const uint32_t nth = gridDim.x * blockDim.x;
    const uint32_t tid = blockIdx.x * blockDim.x + threadIdx.x;
    for (uint32_t n = tid; n < P; n += nth) {
        rt3d_point q;
        const uint32_t p = F.pix[sc][n];
        q.i = (int)(p / F.cols);
        q.j = (int)(p % F.cols);
        q.fi = F.fi[sc][n];
        q.fj = F.fj[sc][n];
        q.t = F.t[tc][n];
        q.intensity = F.r[rc][n];
        q.flags = F.fl[sc][n];
        for (int k = 0; k < 7; ++k) q.pad_[k] = 0;
        q.x = (q.fi + 0.5) * F.pitch;
        q.y = (q.fj + 0.5) * F.pitch;
        q.z = q.t * F.bres;
        out[n] = q;
    }
    for (uint32_t p = tid; p < F.npix; p += nth) bg[p] = F.b[bc][p];
    if (tid == 0) *ctl_out = *c;
}

__global__ void gather_points_kernel(Frame F, uint32_t pb, uint32_t P, int tc, int rc, int sc,
                                     int baseline, rt3d_point* out) {
    const uint32_t k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= P) return;
    const uint32_t n = pb + k;
    rt3d_point q;
    const uint32_t p = F.pix[sc][n];
    const int i = (int)(p / F.cols), j = (int)(p % F.cols);
    q.i = i;
    q.j = j;
    q.fi = F.fi[sc][n];
    q.fj = F.fj[sc][n];
    q.t = F.t[tc][n];
    q.intensity = F.r[rc][n];
    q.flags = F.fl[sc][n];
    for (int k = 0; k < 7; ++k) q.pad_[k] = 0;
    if (baseline) {
        const double coarse_pitch = F.pitch * F.s;
        q.x = (i + 0.5) * coarse_pitch;
        q.y = (j + 0.5) * coarse_pitch;
    } else {
        q.x = (q.fi + 0.5) * F.pitch;
        q.y = (q.fj + 0.5) * F.pitch;
    }
    q.z = q.t * F.bres;
    out[k] = q;
}

}  // namespace rt3d

// ===========================================================================
// host
// ===========================================================================
namespace {

thread_local std::string g_err;

rt3d_status fail(rt3d_status st, const char* fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    g_err = buf;
    return st;
}

#define CUDA_TRY(expr)                                                                  \
    do {                                                                                \
        cudaError_t e_ = (expr);                                                        \
        if (e_ != cudaSuccess)                                                          \
            return fail(RT3D_ERR_CUDA, "%s: %s (%s:%d)", #expr, cudaGetErrorString(e_), \
                        __FILE__, __LINE__);                                            \
    } while (0)

struct DevBuf {
    void* p = nullptr;
    size_t cap = 0;
    DevBuf() = default;
    DevBuf(const DevBuf&) = delete;
    DevBuf& operator=(const DevBuf&) = delete;
    ~DevBuf() { release(); }  // every member buffer goes with its session
    cudaError_t ensure(size_t bytes) {
        if (bytes <= cap && p) return cudaSuccess;
        const size_t old = p ? cap : 0;
        if (p) cudaFree(p);
        p = nullptr;
        cap = 0;
        // geometric growth: a stream of cubes of varying size reallocates a
        // few times, not at every larger one, so buffer addresses (and the
        // frame graphs cached by them) stay put
        size_t want = std::max<size_t>(bytes, 256);
        if (old) want = std::max(want, old + old / 2);
        want = (want + 65535) & ~(size_t)65535;
        cudaError_t e = cudaMalloc(&p, want);
        if (e == cudaSuccess) cap = want;
        return e;
    }
    template <typename T>
    T* as() const {
        return static_cast<T*>(p);
    }
    void release() {
        if (p) cudaFree(p);
        p = nullptr;
        cap = 0;
    }
};

}  // namespace

struct rt3d_session {
    int device = 0;
    int nsm = 0;
    cudaStream_t stream = nullptr;
    int grid_frame = 0;      // max over the configs (per-block scratch sizing)
    int grid_frame_c[4] = {0, 0, 0, 0};  // cooperative grid of stage_kernel per lane-group config
    int per_sm_c[4] = {0, 0, 0, 0};      // co-resident stage blocks per SM per config
    int want_per_sm = 2;              // RT3D_BLOCKS_PER_SM (lane-group configs 4, 32, 3)
    int want_per_sm_g1 = 0;           // RT3D_G1_BLOCKS_PER_SM (thread per pixel; 0: occupancy)
    int sharing = 1;                  // sessions running frames concurrently on the device
    int occ_apss = 1, occ_knn = 1, occ_fit = 1, occ_fit_split = 1;  // co-resident blocks per SM
    int grid_apss = 0, grid_knn = 0, grid_fit = 0, grid_fit_split = 0;
    int grid_fft = 0;
    // sensor
    bool have_sensor = false;
    int rows = 0, cols = 0, bins = 0, s = 1;
    double pitch = 1, bres = 1;
    bool per_pixel_irf = false;
    DevBuf irfs, irf_tab, irf_of_pix, gain, dead;
    // cube
    bool have_cube = false;
    int c_rows = 0, c_cols = 0, c_bins = 0;
    uint64_t n_events = 0;
    uint64_t lam_cap = 0;  // event capacity of the sweep spill slots (Frame::nev)
    DevBuf off, ev;
    // pipelined frames (rt3d_frame_submit / rt3d_frame_collect): a second
    // cube slot, a copy stream, result slots
    DevBuf off2, ev2;
    DevBuf eval_pts, eval_k[2], eval_v[2], eval_out, eval_cnt, eval_tmp;  // rt3d_evaluate
    DevBuf sim_boff, sim_bpts, sim_t, sim_r, sim_bg, sim_cnt, sim_tmp, sim_ph;  // rt3d_simulate_cube
    int cube_slot = 0;
    cudaStream_t cstream = nullptr;
    uint32_t* h_off[2] = {nullptr, nullptr};
    size_t h_off_cap[2] = {0, 0};
    cudaEvent_t cube_ready[2] = {nullptr, nullptr}, frame_done[2] = {nullptr, nullptr};
    DevBuf res_pts[2], res_bg[2], res_ctl[2];
    Ctl* h_res_ctl = nullptr;
    uint64_t next_ticket = 0;
    int inflight[2] = {0, 0};
    uint64_t slot_ticket[2] = {0, 0};
    size_t slot_npix[2] = {0, 0};  // background size of the frame in each slot
    // state
    DevBuf t[2], r[2], b[2], pix[2], fi[2], fj[2], fl[2], bo[2];
    size_t pcap = 0;
    DevBuf gt, ct, gr, cr, gb, cb, oog, lam, blk, bmax, cnt, btot, part, mig[2];
    DevBuf pk_t, pk_resp, pk_mass, pk_int, npk, nval, fft_re, fft_im, amom, zb, knn_list;
    DevBuf ctl, diag, trace, outpts, misc, prof, tblk, tbmax;
    bool profile = false;
    Ctl* h_ctl = nullptr;  // pinned staging
    // state description
    bool have_state = false;
    bool baseline_state = false;
    bool state_pinned = true;
    uint32_t P = 0;
    uint32_t pbase = 0;        // first point of the state (row bands: the band's own)
    int batch_hint = 1;        // frames per launch being prepared (build_frame's sweep layout)
    bool banded = false;       // the state is one row band of a frame (rt3d_reconstruct_bands)
    uint32_t band_pix0 = 0, band_pix1 = 0;
    int tc = 0, rc = 0, bc = 0, sc = 0;
    std::vector<uint32_t> perm;  // device order -> caller's cloud order (nll/grads API)
    uint32_t max_pts_per_pixel = 0;
    // last reconstruct report
    int iterations = 0;
    int report_iters_cap = 0;
    cudaEvent_t ev0 = nullptr, ev1 = nullptr;
    cudaEvent_t xev = nullptr;  // cross-stream ordering of batched frames
    cudaEvent_t oev = nullptr;  // rt3d_session_after's marker
    unsigned long long* h_dbg = nullptr;  // RT3D_DEBUG records (pinned copy)
    unsigned long long* d_dbg = nullptr;
    cudaStream_t side = nullptr;
    // kernel-class timing with CUDA events on the session stream (opt-in)
    bool time_kernels = false;
    struct Timed {
        int cls;
        cudaEvent_t a, b;
    };
    std::vector<Timed> timed;
    std::vector<cudaEvent_t> ev_pool;
    double kt_ms[RT3D_KERNEL_CLASSES] = {};
    uint64_t kt_n[RT3D_KERNEL_CLASSES] = {};
    // the last frame's launch sequence as a CUDA graph, replayed while the
    // frame (its Frame bytes: buffers, config, toggles) and timing mode match
    struct GraphCache {
        bool valid = false;
        int n = 0, first = 0, count = 0;  // frames of the batch; the ones launched
        uint32_t bpf = 0;
        bool zero_ctl = true;
        Frame F[kMaxBatch];
        cudaGraphExec_t exec = nullptr;
        uint64_t used = 0;
    } gc[4];  // pipelined frames alternate two cube slots: two live graphs
    uint64_t gc_clock = 0;
    uint64_t graph_captures = 0, graph_launches = 0;  // (rt3d_graph_counts)
};

namespace {

rt3d_status check_session(rt3d_session* s) {
    if (!s) return fail(RT3D_ERR_INVALID_ARGUMENT, "null session");
    return RT3D_OK;
}

int tree_depth(uint32_t npix) {
    int G = 0;
    while (((uint64_t)npix + (1ull << G) - 1) >> G > 32) ++G;
    return G;
}

rt3d_status ensure_state(rt3d_session* s, size_t pcap, size_t npix) {
    size_t pc = std::max<size_t>(pcap, 1);
    for (int k = 0; k < 2; ++k) {
        CUDA_TRY(s->t[k].ensure(pc * 8));
        CUDA_TRY(s->r[k].ensure(pc * 8));
        CUDA_TRY(s->pix[k].ensure(pc * 4));
        CUDA_TRY(s->fi[k].ensure(pc * 4));
        CUDA_TRY(s->fj[k].ensure(pc * 4));
        CUDA_TRY(s->fl[k].ensure(pc));
        CUDA_TRY(s->b[k].ensure(npix * 8));
        CUDA_TRY(s->bo[k].ensure((npix + 1) * 4));
    }
    CUDA_TRY(s->mig[0].ensure(pc * 8));
    CUDA_TRY(s->mig[1].ensure(pc * 8));
    CUDA_TRY(s->gt.ensure(pc * 8));
    CUDA_TRY(s->ct.ensure(pc * 8));
    CUDA_TRY(s->gr.ensure(pc * 8));
    CUDA_TRY(s->cr.ensure(pc * 8));
    CUDA_TRY(s->oog.ensure(pc));
    CUDA_TRY(s->gb.ensure(npix * 8));
    CUDA_TRY(s->cb.ensure(npix * 8));
    s->pcap = std::max(s->pcap, pc);
    return RT3D_OK;
}

// lane-group configs of the stage kernels (lanes per pixel 4, 32, 3, 1)
int cfg_index(int gsz) { return gsz == 4 ? 0 : gsz == 32 ? 1 : gsz == 3 ? 2 : 3; }

// stage blocks per SM a frame's cooperative grid uses for lane-group config c
int blocks_per_sm(const rt3d_session* s, int c) {
    if (c == 3) return s->want_per_sm_g1 > 0 ? s->want_per_sm_g1 : s->per_sm_c[3];
    return s->want_per_sm;
}

rt3d_status build_frame(rt3d_session* s, Frame& F, const Cfg& cfg, int max_iters) {
    if (!s->have_sensor) return fail(RT3D_ERR_INVALID_ARGUMENT, "rt3d: no sensor set");
    if (!s->have_cube) return fail(RT3D_ERR_INVALID_ARGUMENT, "rt3d: no cube set");
    if (s->rows != s->c_rows || s->cols != s->c_cols || s->bins != s->c_bins)
        return fail(RT3D_ERR_INVALID_ARGUMENT, "likelihood: state/cube dimension mismatch");
    std::memset(&F, 0, sizeof F);
    const uint32_t npix = (uint32_t)s->rows * (uint32_t)s->cols;
    F.rows = s->rows;
    F.cols = s->cols;
    F.bins = s->bins;
    F.s = s->s;
    // (APSS packs a member's fine cell into 16 + 16 bits)
    if ((uint64_t)s->rows * (uint64_t)s->s > 65535ull || (uint64_t)s->cols * (uint64_t)s->s > 65535ull)
        return fail(RT3D_ERR_UNSUPPORTED, "rt3d: fine grids of more than 65535 rows or columns are not supported");
    F.smag = s->s > 1 ? (uint32_t)(((1ull << 32) + (uint64_t)s->s - 1) / (uint64_t)s->s) : 0u;
    F.frows = s->rows * s->s;
    F.fcols = s->cols * s->s;
    F.pitch = s->pitch;
    F.bres = s->bres;
    F.tlim = (double)s->bins * (1.0 - 1e-12);  // reconstruct.hpp:331
    F.irfs = s->irfs.as<IrfDev>();
    F.irf_of_pix = s->per_pixel_irf ? s->irf_of_pix.as<uint32_t>() : nullptr;
    F.gain = s->gain.as<double>();
    F.dead = s->dead.as<uint8_t>();
    F.npix = npix;
    F.off = (s->cube_slot ? s->off2 : s->off).as<uint32_t>();
    F.ev = (s->cube_slot ? s->ev2 : s->ev).as<uint2>();
    F.G = tree_depth(npix);
    F.Gb = std::max(0, F.G - 3);
    F.wpb = 1 << (F.G - F.Gb);
    F.nbn = 1u << F.Gb;
    // scratch
    // per-event spill slots strided by a power-of-two capacity, not by this
    // cube's event count: the Frame bytes (the CUDA-graph cache key) then
    // stay the same across the frames of a stream
    while (s->lam_cap < s->n_events) s->lam_cap = s->lam_cap ? 2 * s->lam_cap : 4096;
    CUDA_TRY(s->lam.ensure(std::max<uint64_t>(s->lam_cap, 1) * 32));
    F.nev = s->lam_cap;
    F.pcap = (uint32_t)std::min<size_t>(s->pcap, 0xffffffffu);
    CUDA_TRY(s->blk.ensure((size_t)F.nbn * 8));
    CUDA_TRY(s->tblk.ensure((size_t)npix * 32 + 64));
    CUDA_TRY(s->tbmax.ensure((size_t)npix * 16 + 64));
    CUDA_TRY(s->part.ensure((size_t)npix * 8));
    F.part = s->part.as<double>();
    CUDA_TRY(s->bmax.ensure((size_t)s->grid_frame * 8));
    CUDA_TRY(s->cnt.ensure((size_t)npix * 4));
    CUDA_TRY(s->btot.ensure((size_t)s->grid_frame * 4));
    const size_t nslot = (size_t)npix * std::max(cfg.K, 1);
    CUDA_TRY(s->pk_t.ensure(nslot * 8));
    CUDA_TRY(s->pk_resp.ensure(nslot * 8));
    CUDA_TRY(s->pk_mass.ensure(nslot * 8));
    CUDA_TRY(s->pk_int.ensure(nslot * 8));
    CUDA_TRY(s->npk.ensure((size_t)npix * 4));
    CUDA_TRY(s->nval.ensure((size_t)npix * 4));
    if (cfg.bg_mode == 1) {
        CUDA_TRY(s->fft_re.ensure((size_t)npix * 16));
        CUDA_TRY(s->fft_im.ensure((size_t)npix * 16));
    }
    CUDA_TRY(s->ctl.ensure(sizeof(Ctl)));
    CUDA_TRY(s->diag.ensure(sizeof(StepDiagDev) * std::max(max_iters, 1)));
    CUDA_TRY(s->trace.ensure(8 * (std::max(max_iters, 1) + 1)));
    for (int k = 0; k < 2; ++k) {
        F.t[k] = s->t[k].as<double>();
        F.r[k] = s->r[k].as<double>();
        F.b[k] = s->b[k].as<double>();
        F.pix[k] = s->pix[k].as<uint32_t>();
        F.fi[k] = s->fi[k].as<int32_t>();
        F.fj[k] = s->fj[k].as<int32_t>();
        F.fl[k] = s->fl[k].as<uint8_t>();
        F.bo[k] = s->bo[k].as<uint32_t>();
    }
    F.mig[0] = s->mig[0].as<double>();
    F.mig[1] = s->mig[1].as<double>();
    F.gt = s->gt.as<double>();
    F.ct = s->ct.as<double>();
    F.gr = s->gr.as<double>();
    F.cr = s->cr.as<double>();
    F.gb = s->gb.as<double>();
    F.cb = s->cb.as<double>();
    F.oog = s->oog.as<uint8_t>();
    F.lam = s->lam.as<double>();
    F.blk = s->blk.as<double>();
    F.bmax = s->bmax.as<double>();
    F.cnt = s->cnt.as<uint32_t>();
    F.btot = s->btot.as<uint32_t>();
    F.pk_t = s->pk_t.as<double>();
    F.pk_resp = s->pk_resp.as<double>();
    F.pk_mass = s->pk_mass.as<double>();
    F.pk_int = s->pk_int.as<double>();
    F.npk = s->npk.as<uint32_t>();
    F.nval = s->nval.as<uint32_t>();
    F.fft_re = s->fft_re.as<double>();
    F.fft_im = s->fft_im.as<double>();
    CUDA_TRY(s->amom.ensure(std::max<size_t>(s->pcap, 1) * kMom * 8));
    F.amom = s->amom.as<double>();
    F.amom_stride = (uint32_t)std::max<size_t>(s->pcap, 1);
    // depth blocks for the neighbour scans of superres frames: blocks of s^2
    // points (one spawned surface), at most 4 per pixel
    F.zb = nullptr;
    F.zkb = F.zbs = 0;
    {
        const uint32_t bs = (uint32_t)(s->s * s->s);
        const uint32_t kb = (std::max<uint32_t>(s->max_pts_per_pixel, 1) + bs - 1) / bs;
        if (s->s > 1 && kb <= 4 && !getenv("RT3D_NO_ZBLOCKS")) {
            CUDA_TRY(s->zb.ensure((size_t)npix * kb * sizeof(double2)));
            F.zb = s->zb.as<double2>();
            F.zkb = kb;
            F.zbs = bs;
        }
    }
    CUDA_TRY(s->knn_list.ensure(std::max<size_t>(s->pcap, 1) * 4));
    F.knn_list = s->knn_list.as<uint32_t>();
    F.ctl = s->ctl.as<Ctl>();
    F.dbg = s->d_dbg;
    F.prof = nullptr;
    if (s->profile) {
        CUDA_TRY(s->prof.ensure(16ull * 128 * (std::max(max_iters, 1) + 1)));
        F.prof = s->prof.as<unsigned long long>();
    }
    F.diag = s->diag.as<StepDiagDev>();
    F.trace = s->trace.as<double>();
    F.cfg = cfg;
    F.cfg.blocktree = getenv("RT3D_TREE_OLD") ? 0 : 1;
    F.cfg.fuse_depth = getenv("RT3D_DEPTH_KERNEL") ? 0 : 1;
    // opt-in (RT3D_FUSED_ITER=1): measured slower on config B, the neighbour
    // phases run at the stage kernels' occupancy
    F.cfg.fused_iter = (F.cfg.fuse_depth && getenv("RT3D_FUSED_ITER")) ? 1 : 0;
    if (F.cfg.fused_iter) F.zb = nullptr;  // (no depth-block pass inside one-launch iterations)
    // two-candidate sweeps: bit 0 intensity, bit 1 depth (RT3D_TWO_CAND).
    // Default: two intensity candidates on frames below 2^20 events, where
    // the intensity block backtracks nearly every iteration and sweeps are
    // latency-bound; one candidate on large arrays, where backtracks are rare
    // and the second candidate is paid in full (config D: -5%,
    // profiles/r01_d_switch_sweep.jsonl)
    // Latency-bound launches (one or a few frames) also evaluate two depth
    // candidates: the depth block backtracks nearly every iteration at B and C
    // (B single frame +0.5 %, C +2.5 %; batches of 16: B -2 %).
    F.cfg.two_cand = getenv("RT3D_ONE_CAND") ? 0
                     : getenv("RT3D_TWO_CAND") ? atoi(getenv("RT3D_TWO_CAND"))
                     : (s->n_events >= (1ull << 20) ? 0 : (s->batch_hint < 4 ? 3 : 1));
    {
        // first kNN window: about k fine pixels; no pruning on huge grids
        // (the pruning margin assumes < 2^20 fine pixels, see knn_warps)
        // a window holding ~k cells; superres frames replicate each coarse
        // pixel's K peaks to all s^2 fine cells, so their cells hold K points
        // each (C: w0 = 1; kNN -13 % against w0 = 2)
        const double per_cell = s->s > 1 ? (double)std::max(cfg.K, 1) : 1.0;
        int w0 = (int)std::ceil(std::sqrt((double)std::max(cfg.knn_k, 1) / per_cell) / 2.0);
        w0 = std::max(w0, 1);
        if (F.frows >= (1 << 20) || F.fcols >= (1 << 20) || getenv("RT3D_KNN_NO_PRUNE")) w0 = cfg.W;
        if (const char* e = getenv("RT3D_KNN_W0")) w0 = std::max(1, atoi(e));
        F.cfg.knn_w0 = w0;
    }
    F.cfg.max_iters = max_iters;
    // lanes per pixel for the likelihood sweeps: 4 for sparse pixels (a few
    // events, <= 4 points), a warp otherwise
    {
        const uint32_t mpp = std::max<uint32_t>(s->max_pts_per_pixel, 1);
        const double mean_ev = npix ? (double)s->n_events / npix : 0.0;
        if (mpp > (uint32_t)SmemT<32>::kPvc)
            return fail(RT3D_ERR_UNSUPPORTED, "rt3d: more than %d points in one pixel",
                        SmemT<32>::kPvc);
        // sparse pixels: lane groups; groups of 3 (10 pixels per warp chunk)
        // when groups of 4 would leave more chunks than warps
        if (mpp <= (uint32_t)kThreadPts && s->batch_hint >= 4 && !getenv("RT3D_WARP_PER_PIXEL")) {
            // frames batched 4 or more to a launch (rt3d_reconstruct_batch):
            // each frame gets few blocks, and a thread per pixel at 3 blocks
            // per SM keeps more pixels in flight than lane groups at 2
            F.cfg.gsz = 1;
        } else if (mpp <= 4 && mean_ev <= 12.0 && !getenv("RT3D_WARP_PER_PIXEL")) {
            const uint64_t warps4 = (uint64_t)s->grid_frame_c[0] * kWarps;
            const uint64_t chunks4 = (npix + 7) / 8;
            F.cfg.gsz = (chunks4 > warps4 && !getenv("RT3D_G4")) ? 3 : 4;
        } else if (mpp <= (uint32_t)kThreadPts && npix >= (1u << 16) &&
                   !getenv("RT3D_WARP_PER_PIXEL")) {
            // large dense arrays (D, E): a thread per pixel, no staging, more
            // blocks per SM (sweep_node_thread)
            F.cfg.gsz = 1;
        } else {
            F.cfg.gsz = 32;
        }
        // test hook: force a lane-group config (1, 3, 4 need <= 4 points per pixel)
        if (const char* gs = getenv("RT3D_GSZ")) {
            const int g = atoi(gs);
            if (g == 32 || ((g == 1 || g == 3 || g == 4) && mpp <= 4)) F.cfg.gsz = g;
        }
        if (F.cfg.gsz == 1) F.cfg.fused_iter = 0;  // ST_ITER is not built for G == 1
    }
    {
        // blocktree block nodes: the shallowest depth <= G whose nodes hold at
        // most one chunk per warp (ceil(npix / 2^d) <= kWarps * 32/gsz)
        // Depths below G stay nodes of pairwise_sum's recursion while their
        // parents split (every parent has more than 8 pixels).
        const uint64_t cap = (uint64_t)kWarps * (uint64_t)(32 / F.cfg.gsz);
        int dmax = F.G;
        while (((uint64_t)npix >> dmax) > 8) ++dmax;  // depth dmax+1's parents would hold <= 8
        int d = 0;
        while (d < dmax && (((uint64_t)npix + (1ull << d) - 1) >> d) > cap) ++d;
        if (const char* e = getenv("RT3D_TBG")) d = std::max(d, std::min(atoi(e), F.G));
        F.tb_G = d;
        F.tb_nbn = 1u << d;
        F.tblk[0] = s->tblk.as<double>();
        F.tblk[1] = F.tblk[0] + F.tb_nbn;
        F.tbmax[0] = s->tbmax.as<double>();
        F.tbmax[1] = F.tbmax[0] + F.tb_nbn;
        F.tblk2[0] = F.tblk[0] + 2 * F.tb_nbn;
        F.tblk2[1] = F.tblk[0] + 3 * F.tb_nbn;
    }
    // one band: the whole frame
    F.nbands = 1;
    F.band = 0;
    F.bpix0 = 0;
    F.bpix1 = npix;
    F.bbn0 = 0;
    F.bbn1 = F.tb_nbn;
    {
        const int cfgi = cfg_index(F.cfg.gsz);
        if (std::min(s->per_sm_c[cfgi], blocks_per_sm(s, cfgi)) < s->sharing)
            return fail(RT3D_ERR_UNSUPPORTED,
                        "rt3d: this frame's stage kernels do not fit %d sessions per device",
                        s->sharing);
    }
    F.tc0 = s->tc;
    F.rc0 = s->rc;
    F.bc0 = s->bc;
    F.sc0 = s->sc;
    return RT3D_OK;
}

// lane-group configs of the stage kernels: lanes per pixel 4, 32, 3, 1
constexpr int kNumCfg = 4;
// dynamic shared memory of the stage kernels per config
static size_t stage_smem(int cfgi) {
    return cfgi == 0 ? sizeof(SmemT<4>) : cfgi == 1 ? sizeof(SmemT<32>)
                     : cfgi == 2 ? sizeof(SmemT<3>) : sizeof(SmemT<1>);
}
// [config][stage]
static StageFn stage_fn(int cfgi, int st) {
    return cfgi == 0 ? stage_fn_g4(st) : cfgi == 1 ? stage_fn_g32(st)
                     : cfgi == 2 ? stage_fn_g3(st) : stage_fn_g1(st);
}

cudaEvent_t pool_event(rt3d_session* s) {
    if (!s->ev_pool.empty()) {
        cudaEvent_t e = s->ev_pool.back();
        s->ev_pool.pop_back();
        return e;
    }
    cudaEvent_t e = nullptr;
    cudaEventCreate(&e);
    return e;
}

// fold completed event pairs into the per-class totals (synchronizes)
rt3d_status harvest_kernel_times(rt3d_session* s) {
    if (s->timed.empty()) return RT3D_OK;
    CUDA_TRY(cudaStreamSynchronize(s->stream));
    for (auto& t : s->timed) {
        float ms = 0.f;
        CUDA_TRY(cudaEventElapsedTime(&ms, t.a, t.b));
        s->kt_ms[t.cls] += ms;
        s->kt_n[t.cls] += 1;
        s->ev_pool.push_back(t.a);
        s->ev_pool.push_back(t.b);
    }
    s->timed.clear();
    return RT3D_OK;
}

// launch `fn` bracketed by CUDA events of class `cls` when timing is on
template <class Fn>
rt3d_status timed_launch(rt3d_session* s, int cls, Fn&& fn) {
    if (!s->time_kernels) return fn();
    if (s->timed.size() > 8192) {
        rt3d_status st = harvest_kernel_times(s);
        if (st) return st;
    }
    rt3d_session::Timed t{cls, pool_event(s), pool_event(s)};
    CUDA_TRY(cudaEventRecord(t.a, s->stream));
    rt3d_status st = fn();
    static const bool sync_each = getenv("RT3D_SYNC_EACH") != nullptr;  // (debugging: name the failing class)
    if (sync_each) {
        const cudaError_t e = cudaStreamSynchronize(s->stream);
        if (e != cudaSuccess)
            return fail(RT3D_ERR_CUDA, "kernel class %d: %s", cls, cudaGetErrorString(e));
    }
    CUDA_TRY(cudaEventRecord(t.b, s->stream));
    s->timed.push_back(t);
    return st;
}

// The batch of frames as one parameter block per kernel: frame k takes blocks
// [k bpf, (k+1) bpf) of the launch and its own barrier counters
// Row bands of one frame (Fs[k].nbands > 1) are coupled: one grid barrier
// over all bands' blocks (band 0's counters), one scan over all bands' blocks
// in band order (band 0's block totals).
static void make_batch(FrameBatch& FB, const Frame* Fs, int n, uint32_t bpf, int first = 0) {
    const bool coupled = Fs[0].nbands > 1;
    FB.n = (uint32_t)n;
    FB.bpf = bpf;
    FB.first = (uint32_t)first;
    for (int k = 0; k < n; ++k) {
        FB.f[k] = Fs[k];
        FB.f[k].blk0 = (uint32_t)(k - first) * bpf;  // (frames outside the launch: unused)
        FB.f[k].nblk = bpf;
        FB.f[k].barc = coupled ? Fs[0].ctl : Fs[k].ctl;
        FB.f[k].bar_n = coupled ? bpf * (uint32_t)n : bpf;
        FB.f[k].sblk0 = coupled ? (uint32_t)k * bpf : 0u;
        FB.f[k].sblk_n = coupled ? bpf * (uint32_t)n : bpf;
    }
}

// the frames as a stream-ordered kernel sequence on s's stream; every
// decision stays on the device (each frame's Ctl), so nothing here waits for
// the GPU.  The frames of a batch share every launch (same configuration).
// frames [first, first + count) of the n run on s's device; the others (row
// bands on other GPUs) only lend their buffers' addresses.  bpf: stage
// blocks per frame (0: the co-resident stage blocks split among count).
rt3d_status launch_frames_direct(rt3d_session* s, const Frame* Fs, int n, int first, int count,
                                 uint32_t bpf, bool zero_ctl = true) {
    const Frame& F = Fs[first];
    for (int k = first; k < first + count; ++k) {
        // (bands on several devices: the controllers were zeroed before any
        // device started, see rt3d_reconstruct_bands)
        if (zero_ctl) CUDA_TRY(cudaMemsetAsync(Fs[k].ctl, 0, sizeof(Ctl), s->stream));
        CUDA_TRY(cudaMemsetAsync(Fs[k].diag, 0,
                                 sizeof(StepDiagDev) * std::max(Fs[k].cfg.max_iters, 1), s->stream));
    }
    const int cfgi = cfg_index(F.cfg.gsz);
    static const int stage_cls[5] = {RT3D_KC_STAGE_FIRST, RT3D_KC_STAGE_DEPTH,
                                     RT3D_KC_STAGE_INTENSITY, RT3D_KC_STAGE_TAIL, RT3D_KC_ITER};
    // cooperative stage grids: the co-resident blocks split among the frames
    const uint32_t sbpf = bpf ? bpf : (uint32_t)std::max(1, s->grid_frame_c[cfgi] / count);
    static thread_local FrameBatch fb_stage, fb_apss, fb_fit, fb_knn, fb_halo;
    make_batch(fb_stage, Fs, n, sbpf, first);
    const bool bands = F.nbands > 1;
    if (bands) make_batch(fb_halo, Fs, n, (uint32_t)s->nsm, first);
    auto halo = [&](int what) -> rt3d_status {
        if (!bands) return RT3D_OK;
        halo_kernel<<<s->nsm * count, 256, 0, s->stream>>>(fb_halo, what);
        CUDA_TRY(cudaGetLastError());
        return RT3D_OK;
    };
    static thread_local FrameBatch fb_zb;
    const uint32_t zb_bpf = F.zb ? (F.npix * F.zkb + 255u) / 256u : 0u;
    if (F.zb) make_batch(fb_zb, Fs, n, zb_bpf, first);
    auto zblocks = [&]() -> rt3d_status {
        if (!F.zb) return RT3D_OK;
        // (timed with the APSS fit class)
        return timed_launch(s, RT3D_KC_APSS_FIT, [&]() -> rt3d_status {
            zblock_kernel<<<zb_bpf * (uint32_t)count, 256, 0, s->stream>>>(fb_zb);
            CUDA_TRY(cudaGetLastError());
            return RT3D_OK;
        });
    };
    make_batch(fb_apss, Fs, n, (uint32_t)s->grid_apss, first);
    // launches of at most ~two waves of split-fit blocks (one or two small
    // frames: latency-bound) take the split fit; batches and large frames
    // (throughput-bound) a thread per point
    static const bool fit_threads = getenv("RT3D_FIT_THREADS") != nullptr;
    const bool split_fit = !fit_threads &&
                           (uint64_t)count * F.pcap <= 2ull * 64ull * (uint64_t)s->grid_fit_split;
    make_batch(fb_fit, Fs, n, (uint32_t)(split_fit ? s->grid_fit_split : s->grid_fit), first);
    make_batch(fb_knn, Fs, n, (uint32_t)s->grid_knn, first);
    auto stage = [&](int st, int it) -> rt3d_status {
        return timed_launch(s, stage_cls[st], [&]() -> rt3d_status {
            void* args[] = {&fb_stage, &it};
            CUDA_TRY(cudaLaunchCooperativeKernel((const void*)stage_fn(cfgi, st),
                                                 dim3(sbpf * (uint32_t)count), dim3(kBlock), args,
                                                 stage_smem(cfgi), s->stream));
            return RT3D_OK;
        });
    };
    rt3d_status st;
    if ((st = stage(ST_FIRST, 0))) return st;
    const int prog = F.cfg.program;
    if (prog == PROG_RECON || prog == PROG_PALM) {
        for (int it = 0; it < F.cfg.max_iters; ++it) {
            if (F.cfg.fused_iter) {  // the whole iteration in one cooperative launch
                if ((st = stage(ST_ITER, it))) return st;
                continue;
            }
            if (!F.cfg.fuse_depth && (st = stage(ST_DEPTH, it))) return st;
            if ((st = halo(1))) return st;  // t, cells, buckets of the halo rows
            if ((st = zblocks())) return st;
            st = timed_launch(s, RT3D_KC_APSS, [&]() -> rt3d_status {
                apss_kernel<<<s->grid_apss * count, kNbrBlock, sizeof(ApssWarpSm) * kNbrWarps,
                              s->stream>>>(fb_apss);
                CUDA_TRY(cudaGetLastError());
                return RT3D_OK;
            });
            if (st) return st;
            st = timed_launch(s, RT3D_KC_APSS_FIT, [&]() -> rt3d_status {
                if (split_fit)
                    apss_fit_split_kernel<<<s->grid_fit_split * count, 128, 0, s->stream>>>(fb_fit);
                else
                    apss_fit_kernel<<<s->grid_fit * count, kFitBlock, 0, s->stream>>>(fb_fit);
                CUDA_TRY(cudaGetLastError());
                return RT3D_OK;
            });
            if (st) return st;
            if ((st = stage(ST_INTENSITY, it))) return st;
            if ((st = halo(2))) return st;  // t after APSS, r after the intensity step
            st = timed_launch(s, RT3D_KC_KNN, [&]() -> rt3d_status {
                // first windows then the deferred wider ones (no superres:
                // B kNN -11 %, E -7 %); superres frames in one kernel (C: the
                // split is +18 %)
                if (F.s > 1) {
                    knn_full_kernel<<<s->grid_knn * count, kNbrBlock, sizeof(KnnWarpSm) * kNbrWarps,
                                      s->stream>>>(fb_knn);
                    CUDA_TRY(cudaGetLastError());
                } else {
                    knn_kernel<<<s->grid_knn * count, kNbrBlock, sizeof(KnnWarpSm) * kNbrWarps,
                                 s->stream>>>(fb_knn);
                    CUDA_TRY(cudaGetLastError());
                    knn_rescan_kernel<<<s->grid_knn * count, kNbrBlock, sizeof(KnnWarpSm) * kNbrWarps,
                                        s->stream>>>(fb_knn);
                    CUDA_TRY(cudaGetLastError());
                }
                return RT3D_OK;
            });
            if (st) return st;
            if ((st = stage(ST_TAIL, it))) return st;
        }
    }
    return RT3D_OK;
}

static void graph_cache_drop(rt3d_session* s, int k) {
    auto& g = s->gc[k];
    if (!g.valid) return;
    cudaStreamSynchronize(s->stream);
    if (g.exec) cudaGraphExecDestroy(g.exec);
    g.exec = nullptr;
    g.valid = false;
}

// A frame is ~150 launches; replaying them as a CUDA graph removes the
// per-launch host cost and most of the inter-kernel gaps.  Graphs are cached
// by the Frame bytes of the batch (buffers, configuration, toggles), least
// recently used out.  Kernel timing (CUDA events around every launch) and the
// in-kernel profiler launch directly; so does RT3D_NO_GRAPH=1.
rt3d_status launch_frames(rt3d_session* s, Frame* Fs, int n, int first = 0, int count = -1,
                          uint32_t bpf = 0, bool zero_ctl = true) {
    if (count < 0) count = n;
    for (int k = 0; k < n; ++k) Fs[k].prof_cap = Fs[k].prof ? (uint32_t)(s->prof.cap / 16) : 0u;
    static const bool no_graph = getenv("RT3D_NO_GRAPH") != nullptr;
    if (no_graph || Fs[first].prof || s->time_kernels)
        return launch_frames_direct(s, Fs, n, first, count, bpf, zero_ctl);
    const int nc = (int)(sizeof(s->gc) / sizeof(s->gc[0]));
    int hit = -1, victim = 0;
    for (int k = 0; k < nc; ++k) {
        if (s->gc[k].valid && s->gc[k].n == n && s->gc[k].first == first &&
            s->gc[k].count == count && s->gc[k].bpf == bpf && s->gc[k].zero_ctl == zero_ctl &&
            std::memcmp(s->gc[k].F, Fs, sizeof(Frame) * (size_t)n) == 0)
            hit = k;
        if (!s->gc[k].valid || (s->gc[victim].valid && s->gc[k].used < s->gc[victim].used)) victim = k;
    }
    if (hit < 0) {
        hit = victim;
        graph_cache_drop(s, hit);
        auto& g = s->gc[hit];
        CUDA_TRY(cudaStreamBeginCapture(s->stream, cudaStreamCaptureModeThreadLocal));
        const rt3d_status st = launch_frames_direct(s, Fs, n, first, count, bpf, zero_ctl);
        cudaGraph_t graph = nullptr;
        const cudaError_t ce = cudaStreamEndCapture(s->stream, &graph);
        if (st) {
            if (graph) cudaGraphDestroy(graph);
            return st;
        }
        if (ce != cudaSuccess) return fail(RT3D_ERR_CUDA, "CUDA: stream capture: %s", cudaGetErrorString(ce));
        const cudaError_t ie = cudaGraphInstantiate(&g.exec, graph, 0);
        cudaGraphDestroy(graph);
        if (ie != cudaSuccess) return fail(RT3D_ERR_CUDA, "CUDA: graph instantiate: %s", cudaGetErrorString(ie));
        std::memcpy(g.F, Fs, sizeof(Frame) * (size_t)n);
        g.n = n;
        g.first = first;
        g.count = count;
        g.bpf = bpf;
        g.zero_ctl = zero_ctl;
        g.valid = true;
        ++s->graph_captures;
    }
    s->gc[hit].used = ++s->gc_clock;
    ++s->graph_launches;
    CUDA_TRY(cudaGraphLaunch(s->gc[hit].exec, s->stream));
    return RT3D_OK;
}

rt3d_status launch_frame(rt3d_session* s, Frame& F, uint32_t P_init) {
    // no host staging: back-to-back async launches must not race on it
    F.P0 = P_init;
    return launch_frames(s, &F, 1);
}

rt3d_status read_ctl(rt3d_session* s) {
    CUDA_TRY(cudaMemcpyAsync(s->h_ctl, s->ctl.p, sizeof(Ctl), cudaMemcpyDeviceToHost, s->stream));
    CUDA_TRY(cudaStreamSynchronize(s->stream));
    const Ctl& c = *s->h_ctl;
    if (c.abort)
        return fail(RT3D_ERR_CUDA,
                    "rt3d: grid barrier watchdog aborted the frame (block %u, op %d, iteration %d, "
                    "%u of %d blocks arrived, sweep %u)",
                    c.abort_block, c.abort_op, c.abort_it, c.abort_count, 0, c.abort_nsweep);
    return RT3D_OK;
}

Cfg cfg_from(const rt3d_recon_config* c, int program) {
    Cfg g;
    std::memset(&g, 0, sizeof g);
    g.program = program;
    g.max_iters = c->max_iters;
    g.stop_tol = c->stop_tol;
    g.step_auto[0] = c->step_t_auto != 0;
    g.step_auto[1] = c->step_r_auto != 0;
    g.step_auto[2] = c->step_b_auto != 0;
    g.step[0] = c->step_t;
    g.step[1] = c->step_r;
    g.step[2] = c->step_b;
    g.beta = c->backtrack_beta;
    g.R = c->apss.kernel_radius;
    g.eps = c->apss.sphere_degeneracy_eps;
    g.min_nbrs = c->apss.min_neighbors;
    g.knn_k = c->knn_k;
    g.r_min = c->r_min;
    g.bg_mode = c->background_mode;
    g.cutoff = c->fft_cutoff;
    g.K = c->init.max_returns;
    g.sep = c->init.min_separation;
    g.thr = c->init.peak_threshold;
    return g;
}

// ReconConfig::validate (reconstruct.hpp:68-77) + ApssParams/InitParams
rt3d_status validate_cfg(const rt3d_recon_config* c) {
    if (!c) return fail(RT3D_ERR_INVALID_ARGUMENT, "null config");
    if (c->max_iters < 1) return fail(RT3D_ERR_INVALID_ARGUMENT, "ReconConfig: max_iters >= 1");
    if (c->stop_tol < 0.0) return fail(RT3D_ERR_INVALID_ARGUMENT, "ReconConfig: stop_tol >= 0");
    if (c->backtrack_beta <= 0.0 || c->backtrack_beta >= 1.0)
        return fail(RT3D_ERR_INVALID_ARGUMENT, "ReconConfig: backtrack_beta in (0,1)");
    if (c->knn_k < 1) return fail(RT3D_ERR_INVALID_ARGUMENT, "ReconConfig: knn_k >= 1");
    if (c->r_min < 0.0) return fail(RT3D_ERR_INVALID_ARGUMENT, "ReconConfig: r_min >= 0");
    if (c->apss.kernel_radius <= 0.0)
        return fail(RT3D_ERR_INVALID_ARGUMENT, "ApssParams: kernel_radius must be positive");
    if (c->apss.min_neighbors < 4)
        return fail(RT3D_ERR_INVALID_ARGUMENT, "ApssParams: min_neighbors must be >= 4");
    if (c->apss.sphere_degeneracy_eps < 0.0)
        return fail(RT3D_ERR_INVALID_ARGUMENT, "ApssParams: sphere_degeneracy_eps must be >= 0");
    if (c->init.max_returns < 1) return fail(RT3D_ERR_INVALID_ARGUMENT, "InitParams: max_returns >= 1");
    if (c->init.min_separation < 1)
        return fail(RT3D_ERR_INVALID_ARGUMENT, "InitParams: min_separation >= 1");
    if (c->init.peak_threshold < 0.0)
        return fail(RT3D_ERR_INVALID_ARGUMENT, "InitParams: peak_threshold >= 0");
    if (c->init.max_returns > kMaxReturns)
        return fail(RT3D_ERR_UNSUPPORTED, "rt3d: max_returns > %d not supported on device",
                    kMaxReturns);
    if (c->background_mode == 1 && (c->fft_cutoff <= 0.0 || c->fft_cutoff > 1.0))
        return fail(RT3D_ERR_INVALID_ARGUMENT, "fft_lowpass_filter: cutoff must be in (0, 1]");
    return RT3D_OK;
}

rt3d_status require_device(rt3d_session* s) {
    rt3d_status st = check_session(s);
    if (st) return st;
    CUDA_TRY(cudaSetDevice(s->device));
    return RT3D_OK;
}

// window half-width for the pinned neighbourhood search
int window_w(double R, double pitch) { return (int)std::floor(R / pitch) + 1; }

template <typename T>
rt3d_status copy_per_point(rt3d_session* s, T* out, const void* dev) {
    if (!out || !s->P) return RT3D_OK;
    if (s->perm.empty()) {
        CUDA_TRY(cudaMemcpyAsync(out, dev, sizeof(T) * s->P, cudaMemcpyDeviceToHost, s->stream));
        CUDA_TRY(cudaStreamSynchronize(s->stream));
        return RT3D_OK;
    }
    std::vector<T> tmp(s->P);
    CUDA_TRY(cudaMemcpyAsync(tmp.data(), dev, sizeof(T) * s->P, cudaMemcpyDeviceToHost, s->stream));
    CUDA_TRY(cudaStreamSynchronize(s->stream));
    for (size_t k = 0; k < s->P; ++k) out[s->perm[k]] = tmp[k];
    return RT3D_OK;
}

}  // namespace

// ===========================================================================
// C ABI
// ===========================================================================
extern "C" {

int rt3d_abi_version(void) { return RT3D_ABI_VERSION; }
const char* rt3d_last_error(void) { return g_err.c_str(); }

int rt3d_device_count(void) {
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess) {
        cudaGetLastError();
        return 0;
    }
    return n;
}

// cooperative stage grids: `sharing` sessions running frames concurrently
// must fit on the device together (each cooperative grid co-resident)
static void set_frame_grids(rt3d_session* s) {
    // the neighbour kernels keep their full grids (grid-stride, no barrier):
    // halving them under sharing measured slower
    s->grid_apss = s->nsm * s->occ_apss;
    s->grid_knn = s->nsm * s->occ_knn;
    s->grid_fit = s->nsm * s->occ_fit;
    s->grid_fit_split = s->nsm * s->occ_fit_split;
    s->grid_frame = 0;
    for (int c = 0; c < kNumCfg; ++c) {
        const int per = std::max(1, std::min(s->per_sm_c[c], blocks_per_sm(s, c)) / std::max(1, s->sharing));
        s->grid_frame_c[c] = s->nsm * per;
        s->grid_frame = std::max(s->grid_frame, s->grid_frame_c[c]);
    }
}

rt3d_status rt3d_session_after(rt3d_session* s, rt3d_session* prior) {
    rt3d_status st = require_device(s);
    if (st) return st;
    if (!prior) return fail(RT3D_ERR_INVALID_ARGUMENT, "null prior session");
    if (prior == s) return RT3D_OK;
    // (recorded and waited on at once: the event can be re-recorded later)
    CUDA_TRY(cudaEventRecord(prior->oev, prior->stream));
    CUDA_TRY(cudaStreamWaitEvent(s->stream, prior->oev, 0));
    return RT3D_OK;
}

rt3d_status rt3d_session_set_sharing(rt3d_session* s, int n_sessions) {
    rt3d_status st = require_device(s);
    if (st) return st;
    if (n_sessions < 1) return fail(RT3D_ERR_INVALID_ARGUMENT, "sharing must be >= 1");
    for (int c = 0; c < 3; c += 2)  // lane-group configs (a warp per pixel: see build_frame)
        if (std::min(s->per_sm_c[c], s->want_per_sm) < n_sessions)
            return fail(RT3D_ERR_UNSUPPORTED,
                        "rt3d: %d sessions cannot share the device (%d stage blocks per SM)",
                        n_sessions, std::min(s->per_sm_c[c], s->want_per_sm));
    CUDA_TRY(cudaStreamSynchronize(s->stream));
    for (int k = 0; k < (int)(sizeof(s->gc) / sizeof(s->gc[0])); ++k) graph_cache_drop(s, k);
    const int old = s->grid_frame;
    s->sharing = n_sessions;
    set_frame_grids(s);
    if (s->grid_frame > old) {  // per-block scratch sized by the grid
        CUDA_TRY(s->bmax.ensure((size_t)s->grid_frame * 8));
        CUDA_TRY(s->btot.ensure((size_t)s->grid_frame * 4));
    }
    return RT3D_OK;
}

rt3d_status rt3d_session_create(int device, rt3d_session** out) {
    if (!out) return fail(RT3D_ERR_INVALID_ARGUMENT, "null out");
    *out = nullptr;
    int n = rt3d_device_count();
    if (n <= 0) return fail(RT3D_ERR_NO_DEVICE, "rt3d: no CUDA device (there is no CPU fallback)");
    if (device < 0 || device >= n) return fail(RT3D_ERR_INVALID_ARGUMENT, "bad device %d", device);
    CUDA_TRY(cudaSetDevice(device));
    cudaDeviceProp prop;
    CUDA_TRY(cudaGetDeviceProperties(&prop, device));
    if (prop.major < 10)
        return fail(RT3D_ERR_NO_DEVICE, "rt3d: built for sm_100a, device is sm_%d%d", prop.major,
                    prop.minor);
    rt3d_session* s = new rt3d_session();
    s->device = device;
    s->nsm = prop.multiProcessorCount;
    CUDA_TRY(cudaStreamCreateWithFlags(&s->stream, cudaStreamNonBlocking));
    int per_sm_c[kNumCfg] = {1 << 30, 1 << 30, 1 << 30, 1 << 30};
    for (int c = 0; c < kNumCfg; ++c)
        for (int st = 0; st < 5; ++st) {
            if (!stage_fn(c, st)) continue;  // ST_ITER is not built for G == 1
            int b = 0;
            const size_t sz = stage_smem(c);
            CUDA_TRY(cudaFuncSetAttribute((const void*)stage_fn(c, st),
                                          cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sz));
            CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(
                &b, (const void*)stage_fn(c, st), kBlock, sz));
            per_sm_c[c] = std::min(per_sm_c[c], b);
        }
    const int per_sm = std::min(std::min(per_sm_c[0], per_sm_c[1]), std::min(per_sm_c[2], per_sm_c[3]));
    {
        int a = 0, k = 0;
        CUDA_TRY(cudaFuncSetAttribute(apss_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      (int)(sizeof(ApssWarpSm) * kNbrWarps)));
        CUDA_TRY(cudaFuncSetAttribute(knn_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      (int)(sizeof(KnnWarpSm) * kNbrWarps)));
        CUDA_TRY(cudaFuncSetAttribute(knn_rescan_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      (int)(sizeof(KnnWarpSm) * kNbrWarps)));
        CUDA_TRY(cudaFuncSetAttribute(knn_full_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      (int)(sizeof(KnnWarpSm) * kNbrWarps)));
        CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&a, apss_kernel, kNbrBlock,
                                                               sizeof(ApssWarpSm) * kNbrWarps));
        CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&k, knn_kernel, kNbrBlock,
                                                               sizeof(KnnWarpSm) * kNbrWarps));
        int f = 0;
        CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&f, apss_fit_kernel, kFitBlock, 0));
        int fs = 0;
        CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&fs, apss_fit_split_kernel, 128, 0));
        s->occ_apss = std::max(a, 1);
        s->occ_knn = std::max(k, 1);
        s->occ_fit = std::max(f, 1);
        s->occ_fit_split = std::max(fs, 1);
    }
    if (per_sm < 1) {
        delete s;
        return fail(RT3D_ERR_CUDA, "rt3d: stage kernel does not fit on an SM");
    }
    const char* env = getenv("RT3D_BLOCKS_PER_SM");
    int want = env ? atoi(env) : 2;
    if (want < 1) want = 1;
    s->want_per_sm = want;
    if (const char* e1 = getenv("RT3D_G1_BLOCKS_PER_SM")) s->want_per_sm_g1 = std::max(1, atoi(e1));
    for (int c = 0; c < kNumCfg; ++c) s->per_sm_c[c] = per_sm_c[c];
    set_frame_grids(s);
    int per_sm_fft = 0;
    CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm_fft, fft_kernel, kBlock,
                                                           2 * kFftMax * sizeof(double)));
    s->grid_fft = s->nsm * std::max(1, per_sm_fft);
    CUDA_TRY(cudaMallocHost(&s->h_ctl, sizeof(Ctl)));
    if (getenv("RT3D_DEBUG")) {
        // device-resident records, read on a side stream (rt3d_debug_peek)
        CUDA_TRY(cudaMallocHost(&s->h_dbg, 8 * 4096));
        CUDA_TRY(cudaMalloc(&s->d_dbg, 8 * 4096));
        CUDA_TRY(cudaMemset(s->d_dbg, 0, 8 * 4096));
        CUDA_TRY(cudaStreamCreateWithFlags(&s->side, cudaStreamNonBlocking));
    }
    CUDA_TRY(cudaEventCreate(&s->ev0));
    CUDA_TRY(cudaEventCreate(&s->ev1));
    CUDA_TRY(cudaEventCreateWithFlags(&s->xev, cudaEventDisableTiming));
    CUDA_TRY(cudaEventCreateWithFlags(&s->oev, cudaEventDisableTiming));
    *out = s;
    return RT3D_OK;
}

rt3d_status rt3d_session_destroy(rt3d_session* s) {
    if (!s) return RT3D_OK;
    cudaSetDevice(s->device);
    cudaStreamSynchronize(s->stream);
    for (int k = 0; k < (int)(sizeof(s->gc) / sizeof(s->gc[0])); ++k) graph_cache_drop(s, k);
    for (auto& t : s->timed) {
        cudaEventDestroy(t.a);
        cudaEventDestroy(t.b);
    }
    for (cudaEvent_t e : s->ev_pool) cudaEventDestroy(e);
    if (s->cstream) {
        cudaStreamSynchronize(s->cstream);
        for (int k = 0; k < 2; ++k) {
            cudaEventDestroy(s->cube_ready[k]);
            cudaEventDestroy(s->frame_done[k]);
            if (s->h_off[k]) cudaFreeHost(s->h_off[k]);
        }
        cudaFreeHost(s->h_res_ctl);
        cudaStreamDestroy(s->cstream);
    }
    if (s->h_ctl) cudaFreeHost(s->h_ctl);
    if (s->h_dbg) cudaFreeHost(s->h_dbg);
    if (s->d_dbg) cudaFree(s->d_dbg);
    if (s->side) cudaStreamDestroy(s->side);
    if (s->ev0) cudaEventDestroy(s->ev0);
    if (s->ev1) cudaEventDestroy(s->ev1);
    if (s->xev) cudaEventDestroy(s->xev);
    if (s->oev) cudaEventDestroy(s->oev);
    if (s->stream) cudaStreamDestroy(s->stream);
    delete s;  // DevBuf members free their device memory
    return RT3D_OK;
}

void* rt3d_session_stream(rt3d_session* s) { return s ? (void*)s->stream : nullptr; }

rt3d_status rt3d_session_profile(rt3d_session* s, int enable) {
    if (!s) return fail(RT3D_ERR_INVALID_ARGUMENT, "null session");
    s->profile = enable != 0;
    return RT3D_OK;
}

void* rt3d_debug_buffer(rt3d_session* s) {
    // snapshot of the device records taken on a side stream, so it works
    // while the session stream is busy
    if (!s || !s->d_dbg) return nullptr;
    if (cudaMemcpyAsync(s->h_dbg, s->d_dbg, 8 * 4096, cudaMemcpyDeviceToHost, s->side) != cudaSuccess)
        return nullptr;
    cudaStreamSynchronize(s->side);
    return (void*)s->h_dbg;
}

rt3d_status rt3d_measure_fp64_peak(rt3d_session* s, double* tflops) {
    rt3d_status st = require_device(s);
    if (st) return st;
    if (!tflops) return fail(RT3D_ERR_INVALID_ARGUMENT, "null output");
    const int blocks = s->nsm * 16, threads = 128, iters = 1 << 14;
    CUDA_TRY(s->misc.ensure((size_t)blocks * threads * 8));
    fp64_peak_kernel<<<blocks, threads, 0, s->stream>>>(s->misc.as<double>(), 64, 0.999, 1e-3);
    CUDA_TRY(cudaGetLastError());
    float best = 1e30f;
    for (int rep = 0; rep < 5; ++rep) {
        CUDA_TRY(cudaEventRecord(s->ev0, s->stream));
        fp64_peak_kernel<<<blocks, threads, 0, s->stream>>>(s->misc.as<double>(), iters, 0.999, 1e-3);
        CUDA_TRY(cudaEventRecord(s->ev1, s->stream));
        CUDA_TRY(cudaEventSynchronize(s->ev1));
        float ms = 0.f;
        CUDA_TRY(cudaEventElapsedTime(&ms, s->ev0, s->ev1));
        best = std::min(best, ms);
    }
    *tflops = 2.0 * 8.0 * iters * (double)blocks * threads / (best * 1e-3) / 1e12;
    return RT3D_OK;
}

rt3d_status rt3d_session_time_kernels(rt3d_session* s, int enable) {
    rt3d_status st = require_device(s);
    if (st) return st;
    if ((st = harvest_kernel_times(s))) return st;
    s->time_kernels = enable != 0;
    for (int k = 0; k < RT3D_KERNEL_CLASSES; ++k) {
        s->kt_ms[k] = 0.0;
        s->kt_n[k] = 0;
    }
    return RT3D_OK;
}

rt3d_status rt3d_graph_counts(rt3d_session* s, uint64_t* captures, uint64_t* launches) {
    if (!s || !captures || !launches) return fail(RT3D_ERR_INVALID_ARGUMENT, "rt3d_graph_counts: null argument");
    *captures = s->graph_captures;
    *launches = s->graph_launches;
    return RT3D_OK;
}

rt3d_status rt3d_kernel_times(rt3d_session* s, double* ms, uint64_t* launches) {
    rt3d_status st = require_device(s);
    if (st) return st;
    if ((st = harvest_kernel_times(s))) return st;
    for (int k = 0; k < RT3D_KERNEL_CLASSES; ++k) {
        if (ms) ms[k] = s->kt_ms[k];
        if (launches) launches[k] = s->kt_n[k];
    }
    return RT3D_OK;
}

rt3d_status rt3d_profile_copy(rt3d_session* s, uint64_t* pairs, uint32_t cap, uint32_t* n) {
    rt3d_status st = require_device(s);
    if (st) return st;
    if ((st = read_ctl(s))) return st;
    uint32_t k = std::min(cap, s->h_ctl->nprof);
    if (k && pairs)
        CUDA_TRY(cudaMemcpy(pairs, s->prof.p, 16ull * k, cudaMemcpyDeviceToHost));
    if (n) *n = k;
    return RT3D_OK;
}

rt3d_status rt3d_session_synchronize(rt3d_session* s) {
    rt3d_status st = require_device(s);
    if (st) return st;
    CUDA_TRY(cudaStreamSynchronize(s->stream));
    return RT3D_OK;
}

// --- IRF tables (sensor.hpp:26-41, 63, reconstruct.hpp:126-127) ------------
static rt3d_status irf_check(const rt3d_irf& f) {
    if (f.dtau <= 0.0) return fail(RT3D_ERR_INVALID_ARGUMENT, "Irf: dtau must be positive");
    if (f.n_samples < 2 || !f.samples) return fail(RT3D_ERR_INVALID_ARGUMENT, "Irf: need >= 2 samples");
    for (uint64_t k = 0; k < f.n_samples; ++k)
        if (f.samples[k] < 0.0 || !std::isfinite(f.samples[k]))
            return fail(RT3D_ERR_INVALID_ARGUMENT, "Irf: samples must be finite and >= 0");
    return RT3D_OK;
}

rt3d_status rt3d_set_sensor(rt3d_session* s, const rt3d_sensor* v) {
    NvtxRange nvtx_("rt3d_set_sensor");
    rt3d_status st = require_device(s);
    if (st) return st;
    if (!v) return fail(RT3D_ERR_INVALID_ARGUMENT, "null sensor");
    if (v->n_rows <= 0 || v->n_cols <= 0 || v->n_bins <= 0)
        return fail(RT3D_ERR_INVALID_ARGUMENT, "SensorModel: dimensions must be positive");
    if (v->superres < 1) return fail(RT3D_ERR_INVALID_ARGUMENT, "SensorModel: superres must be >= 1");
    if (v->pixel_pitch <= 0.0 || v->bin_resolution <= 0.0)
        return fail(RT3D_ERR_INVALID_ARGUMENT, "SensorModel: pitch/bin resolution must be positive");
    if (!v->gain || !v->dead) return fail(RT3D_ERR_INVALID_ARGUMENT, "SensorModel: gain/dead required");
    const size_t npix = (size_t)v->n_rows * v->n_cols;
    if (npix >= (1ull << 31)) return fail(RT3D_ERR_UNSUPPORTED, "rt3d: too many pixels");
    const size_t nirf = v->irf_per_pixel ? npix : 1;
    std::vector<IrfDev> descs(nirf);
    size_t total = 0;
    for (size_t k = 0; k < nirf; ++k) {
        const rt3d_irf& f = v->irf_per_pixel ? v->irf_per_pixel[k] : v->irf_shared;
        if ((st = irf_check(f))) return st;
        total += 2 * f.n_samples;
    }
    if (!v->irf_per_pixel && (st = irf_check(v->irf_shared))) return st;
    std::vector<double> tab(total);
    size_t o = 0;
    std::vector<size_t> offs(nirf);
    for (size_t k = 0; k < nirf; ++k) {
        const rt3d_irf& f = v->irf_per_pixel ? v->irf_per_pixel[k] : v->irf_shared;
        offs[k] = o;
        double hmax = 0.0;
        for (uint64_t q = 0; q < f.n_samples; ++q) {
            tab[o + q] = f.samples[q];
            hmax = std::max(hmax, f.samples[q]);
        }
        for (uint64_t q = 0; q + 1 < f.n_samples; ++q)
            tab[o + f.n_samples + q] = (f.samples[q + 1] - f.samples[q]) / f.dtau;
        IrfDev& d = descs[k];
        d.tau_min = f.tau_min;
        d.dtau = f.dtau;
        d.tau_max = f.tau_min + f.dtau * (double)(f.n_samples - 1);
        d.h_max = hmax;
        d.n = (uint32_t)f.n_samples;
        int ex = 0;
        const double mant = std::frexp(f.dtau, &ex);
        d.pow2 = (mant == 0.5) ? 1u : 0u;
        d.inv_dtau = d.pow2 ? std::ldexp(1.0, 1 - ex) : 1.0 / f.dtau;  // (irf_x)
        d.lim = (double)(f.n_samples - 2);
        o += 2 * f.n_samples;
    }
    CUDA_TRY(s->irf_tab.ensure(total * 8));
    CUDA_TRY(s->irfs.ensure(nirf * sizeof(IrfDev)));
    for (size_t k = 0; k < nirf; ++k) {
        descs[k].s = s->irf_tab.as<double>() + offs[k];
        descs[k].d = s->irf_tab.as<double>() + offs[k] + descs[k].n;
    }
    CUDA_TRY(cudaMemcpyAsync(s->irf_tab.p, tab.data(), total * 8, cudaMemcpyHostToDevice, s->stream));
    CUDA_TRY(cudaMemcpyAsync(s->irfs.p, descs.data(), nirf * sizeof(IrfDev), cudaMemcpyHostToDevice,
                             s->stream));
    if (v->irf_per_pixel) {
        std::vector<uint32_t> idx(npix);
        for (size_t p = 0; p < npix; ++p) idx[p] = (uint32_t)p;
        CUDA_TRY(s->irf_of_pix.ensure(npix * 4));
        CUDA_TRY(cudaMemcpyAsync(s->irf_of_pix.p, idx.data(), npix * 4, cudaMemcpyHostToDevice, s->stream));
    }
    CUDA_TRY(s->gain.ensure(npix * 8));
    CUDA_TRY(s->dead.ensure(npix));
    CUDA_TRY(cudaMemcpyAsync(s->gain.p, v->gain, npix * 8, cudaMemcpyHostToDevice, s->stream));
    CUDA_TRY(cudaMemcpyAsync(s->dead.p, v->dead, npix, cudaMemcpyHostToDevice, s->stream));
    CUDA_TRY(cudaStreamSynchronize(s->stream));
    s->have_sensor = true;
    s->per_pixel_irf = v->irf_per_pixel != nullptr;
    s->rows = v->n_rows;
    s->cols = v->n_cols;
    s->bins = v->n_bins;
    s->s = v->superres;
    s->pitch = v->pixel_pitch;
    s->bres = v->bin_resolution;
    return RT3D_OK;
}

// PhotonCube::validate (cube.hpp:84-112) + the u32 offset table
static rt3d_status validate_cube(const rt3d_cube* c, uint32_t* off32) {
    if (!c) return fail(RT3D_ERR_INVALID_ARGUMENT, "null cube");
    if (c->n_rows <= 0 || c->n_cols <= 0 || c->n_bins <= 0)
        return fail(RT3D_ERR_FORMAT, "cube: non-positive dimensions");
    const size_t npix = (size_t)c->n_rows * c->n_cols;
    if (!c->offsets || c->offsets[0] != 0 || c->offsets[npix] != c->n_events)
        return fail(RT3D_ERR_FORMAT, "cube: bad offset table");
    if (c->n_events >= (1ull << 32)) return fail(RT3D_ERR_UNSUPPORTED, "rt3d: >= 2^32 events");
    for (size_t p = 0; p < npix; ++p) {
        if (c->offsets[p] > c->offsets[p + 1])
            return fail(RT3D_ERR_FORMAT, "cube: negative event range at pixel %zu", p);
        uint32_t prev = 0;
        bool first = true;
        for (uint64_t k = c->offsets[p]; k < c->offsets[p + 1]; ++k) {
            const rt3d_event& e = c->events[k];
            if (e.bin >= (uint32_t)c->n_bins)
                return fail(RT3D_ERR_FORMAT, "cube: bin out of range at pixel %zu", p);
            if (e.count < 1) return fail(RT3D_ERR_FORMAT, "cube: zero count at pixel %zu", p);
            if (!first && e.bin <= prev)
                return fail(RT3D_ERR_FORMAT, "cube: bins not strictly increasing at pixel %zu", p);
            prev = e.bin;
            first = false;
        }
        off32[p] = (uint32_t)c->offsets[p];
    }
    off32[npix] = (uint32_t)c->offsets[npix];
    return RT3D_OK;
}

rt3d_status rt3d_set_cube(rt3d_session* s, const rt3d_cube* c) {
    NvtxRange nvtx_("rt3d_set_cube");
    rt3d_status st = require_device(s);
    if (st) return st;
    if (!c) return fail(RT3D_ERR_INVALID_ARGUMENT, "null cube");
    if (c->n_rows <= 0 || c->n_cols <= 0 || c->n_bins <= 0)
        return fail(RT3D_ERR_FORMAT, "cube: non-positive dimensions");
    const size_t npix = (size_t)c->n_rows * c->n_cols;
    if (!c->offsets || c->offsets[0] != 0 || c->offsets[npix] != c->n_events)
        return fail(RT3D_ERR_FORMAT, "cube: bad offset table");
    if (c->n_events >= (1ull << 32)) return fail(RT3D_ERR_UNSUPPORTED, "rt3d: >= 2^32 events");
    if (npix >= (1ull << 32) - 1) return fail(RT3D_ERR_UNSUPPORTED, "rt3d: too many pixels");
    // the device may still read the other slot's / this slot's buffers
    CUDA_TRY(cudaStreamSynchronize(s->stream));
    s->cube_slot = 0;
    s->have_cube = false;
    CUDA_TRY(s->off.ensure((npix + 1) * 4));
    CUDA_TRY(s->ev.ensure(std::max<uint64_t>(c->n_events, 1) * 8));
    const size_t eo = (npix + 1) * 8;  // the error word after the 64-bit offsets
    CUDA_TRY(s->misc.ensure(eo + 8));
    unsigned long long* err = reinterpret_cast<unsigned long long*>(static_cast<char*>(s->misc.p) + eo);
    CUDA_TRY(cudaMemcpyAsync(s->misc.p, c->offsets, eo, cudaMemcpyHostToDevice, s->stream));
    if (c->n_events)
        CUDA_TRY(cudaMemcpyAsync(s->ev.p, c->events, c->n_events * 8, cudaMemcpyHostToDevice, s->stream));
    CUDA_TRY(cudaMemsetAsync(err, 0xff, 8, s->stream));
    cube_check_kernel<<<s->nsm * 8, 256, 0, s->stream>>>(
        s->misc.as<unsigned long long>(), (uint32_t)npix, c->n_events, (uint32_t)c->n_bins,
        s->ev.as<uint2>(), s->off.as<uint32_t>(), err);
    CUDA_TRY(cudaGetLastError());
    unsigned long long herr = 0;
    CUDA_TRY(cudaMemcpyAsync(&herr, err, 8, cudaMemcpyDeviceToHost, s->stream));
    CUDA_TRY(cudaStreamSynchronize(s->stream));
    if (herr != ~0ull) {
        const unsigned long long p = herr >> 3;
        const unsigned kind = (unsigned)(herr & 7u);
        return fail(RT3D_ERR_FORMAT, kind == 1   ? "cube: negative event range at pixel %llu"
                                     : kind == 2 ? "cube: bin out of range at pixel %llu"
                                     : kind == 3 ? "cube: zero count at pixel %llu"
                                                 : "cube: bins not strictly increasing at pixel %llu",
                    p);
    }
    s->have_cube = true;
    s->c_rows = c->n_rows;
    s->c_cols = c->n_cols;
    s->c_bins = c->n_bins;
    s->n_events = c->n_events;
    return RT3D_OK;
}

// decode_cube (io.hpp:116-145) straight into the session's device CSR: the
// host walks the per-pixel record headers only (O(pixels)); the events are
// copied once as raw bytes and gathered + validated on the device.
rt3d_status rt3d_set_cube_spcb(rt3d_session* s, const void* bytes, uint64_t n_bytes) {
    NvtxRange nvtx_("rt3d_set_cube_spcb");
    rt3d_status st = require_device(s);
    if (st) return st;
    if (!bytes) return fail(RT3D_ERR_INVALID_ARGUMENT, "null SPCB buffer");
    const unsigned char* b = static_cast<const unsigned char*>(bytes);
    uint64_t pos = 0;
    auto u32 = [&](const char* what, uint32_t& v) -> bool {
        if (n_bytes - pos < 4) {
            fail(RT3D_ERR_FORMAT, "SPCB: truncated while reading %s", what);
            return false;
        }
        v = (uint32_t)b[pos] | ((uint32_t)b[pos + 1] << 8) | ((uint32_t)b[pos + 2] << 16) |
            ((uint32_t)b[pos + 3] << 24);
        pos += 4;
        return true;
    };
    if (n_bytes < 4) return fail(RT3D_ERR_FORMAT, "SPCB: truncated while reading magic");
    if (std::memcmp(b, "SPCB", 4) != 0) return fail(RT3D_ERR_FORMAT, "SPCB: bad magic");
    pos = 4;
    uint32_t version, rows, cols, bins;
    if (!u32("version", version)) return RT3D_ERR_FORMAT;
    if (version != 1) return fail(RT3D_ERR_FORMAT, "SPCB: unsupported version %u", version);
    if (!u32("n_rows", rows) || !u32("n_cols", cols) || !u32("n_bins", bins)) return RT3D_ERR_FORMAT;
    if (n_bytes - pos < 8) return fail(RT3D_ERR_FORMAT, "SPCB: truncated while reading bin_width");
    double bin_width;
    std::memcpy(&bin_width, b + pos, 8);  // little-endian host
    pos += 8;
    if (rows == 0 || cols == 0 || bins == 0) return fail(RT3D_ERR_FORMAT, "SPCB: zero dimension");
    if (rows > 0x7fffffffu || cols > 0x7fffffffu || bins > 0x7fffffffu)
        return fail(RT3D_ERR_UNSUPPORTED, "rt3d: SPCB dimensions above 2^31");
    const uint64_t npix = (uint64_t)rows * cols;
    if (npix >= (1ull << 31)) return fail(RT3D_ERR_UNSUPPORTED, "rt3d: too many pixels");
    std::vector<uint32_t> off32(npix + 1);
    uint64_t ne = 0;
    for (uint64_t p = 0; p < npix; ++p) {
        uint32_t n;
        if (!u32("event count", n)) return RT3D_ERR_FORMAT;
        const uint64_t need = 8ull * n, have = n_bytes - pos;
        if (have < need)
            return fail(RT3D_ERR_FORMAT, "SPCB: truncated while reading %s",
                        (have % 8) >= 4 ? "event value" : "event bin");
        off32[p] = (uint32_t)ne;
        ne += n;
        if (ne >= (1ull << 32)) return fail(RT3D_ERR_UNSUPPORTED, "rt3d: >= 2^32 events");
        pos += need;
    }
    off32[npix] = (uint32_t)ne;
    if (pos != n_bytes) return fail(RT3D_ERR_FORMAT, "SPCB: trailing bytes");
    CUDA_TRY(cudaStreamSynchronize(s->stream));
    s->cube_slot = 0;
    CUDA_TRY(s->off.ensure((npix + 1) * 4));
    CUDA_TRY(s->ev.ensure(std::max<uint64_t>(ne, 1) * 8));
    const uint64_t eo = (n_bytes + 7) & ~7ull;  // the error word after the bytes
    CUDA_TRY(s->misc.ensure(eo + 8));
    CUDA_TRY(cudaMemcpyAsync(s->misc.p, b, n_bytes, cudaMemcpyHostToDevice, s->stream));
    CUDA_TRY(cudaMemcpyAsync(s->off.p, off32.data(), (npix + 1) * 4, cudaMemcpyHostToDevice, s->stream));
    unsigned long long* err =
        reinterpret_cast<unsigned long long*>(static_cast<char*>(s->misc.p) + eo);
    CUDA_TRY(cudaMemsetAsync(err, 0xff, 8, s->stream));
    spcb_gather_kernel<<<s->nsm * 8, 256, 0, s->stream>>>(
        s->misc.as<uint32_t>(), s->off.as<uint32_t>(), (uint32_t)npix, bins, s->ev.as<uint2>(), err);
    CUDA_TRY(cudaGetLastError());
    unsigned long long herr = 0;
    CUDA_TRY(cudaMemcpyAsync(&herr, err, 8, cudaMemcpyDeviceToHost, s->stream));
    CUDA_TRY(cudaStreamSynchronize(s->stream));
    if (herr != ~0ull) {
        const unsigned long long p = herr >> 2;
        const unsigned kind = (unsigned)(herr & 3u);
        s->have_cube = false;
        return fail(RT3D_ERR_FORMAT, kind == 1   ? "cube: bin out of range at pixel %llu"
                                     : kind == 2 ? "cube: zero count at pixel %llu"
                                                 : "cube: bins not strictly increasing at pixel %llu",
                    p);
    }
    s->have_cube = true;
    s->c_rows = (int)rows;
    s->c_cols = (int)cols;
    s->c_bins = (int)bins;
    s->n_events = ne;
    return RT3D_OK;
}

// validation, buffers and the Frame of an init-like program (reconstruct,
// init, baseline) on s's resident sensor and cube
static rt3d_status prepare_init_like(rt3d_session* s, const rt3d_recon_config* cfg, int program,
                                     Frame& F) {
    rt3d_status st = require_device(s);
    if (st) return st;
    if ((st = validate_cfg(cfg))) return st;
    // reconstruct -> palm_step -> fft_background_denoise (denoise.hpp:269-270)
    if (program == PROG_RECON && cfg->background_mode == 1 && s->have_sensor &&
        (s->rows < 2 || s->cols < 2))
        return fail(RT3D_ERR_INVALID_ARGUMENT, "fft_lowpass_filter: image must be at least 2x2");
    Cfg g = cfg_from(cfg, program);
    const size_t npix = (size_t)s->rows * s->cols;
    const size_t pcap = program == PROG_BASELINE
                            ? npix
                            : (size_t)cfg->init.max_returns * s->s * s->s * npix;
    if ((st = ensure_state(s, pcap, npix))) return st;
    g.W = window_w(cfg->apss.kernel_radius, s->pitch);
    g.set_oog_flags = 1;
    s->max_pts_per_pixel = program == PROG_BASELINE ? 1u : (uint32_t)cfg->init.max_returns * s->s * s->s;
    s->tc = s->rc = s->bc = s->sc = 0;
    if ((st = build_frame(s, F, g, program == PROG_RECON ? cfg->max_iters : 1))) return st;
    F.P0 = 0;
    return RT3D_OK;
}

static void finish_init_like(rt3d_session* s, const rt3d_recon_config* cfg, int program,
                             bool banded = false) {
    s->banded = banded;
    s->have_state = true;
    s->baseline_state = program == PROG_BASELINE;
    s->state_pinned = true;
    s->perm.clear();
    s->iterations = -1;  // resolved lazily (report / state queries)
    s->report_iters_cap = program == PROG_RECON ? cfg->max_iters : 0;
}

static rt3d_status run_init_like(rt3d_session* s, const rt3d_recon_config* cfg, int program) {
    Frame F;
    rt3d_status st = prepare_init_like(s, cfg, program, F);
    if (st) return st;
    CUDA_TRY(cudaEventRecord(s->ev0, s->stream));
    if ((st = launch_frames(s, &F, 1))) return st;
    CUDA_TRY(cudaEventRecord(s->ev1, s->stream));
    finish_init_like(s, cfg, program);
    return RT3D_OK;
}

// Host tree_node_range (rt3d_math.cuh): node k at depth d of pairwise_sum's
// recursion over n elements
static void host_node_range(uint32_t n, int d, uint32_t k, uint32_t& lo, uint32_t& size) {
    lo = 0;
    size = n;
    for (int b = d - 1; b >= 0; --b) {
        const uint32_t h = size / 2;
        if ((k >> b) & 1u) {
            lo += h;
            size -= h;
        } else {
            size = h;
        }
    }
}

static rt3d_status resolve_state(rt3d_session* s) {
    if (!s->have_state) return fail(RT3D_ERR_INVALID_ARGUMENT, "rt3d: no state in session");
    if (s->iterations != -1) return RT3D_OK;
    rt3d_status st = read_ctl(s);
    if (st) return st;
    const Ctl& c = *s->h_ctl;
    // a row band's state is its own points [pbase, pbase + pown)
    s->P = s->banded ? c.pown : c.P;
    s->pbase = s->banded ? c.pbase : 0u;
    s->tc = c.tc;
    s->rc = c.rc;
    s->bc = c.bc;
    s->sc = c.sc;
    s->iterations = c.iterations;
    return RT3D_OK;
}

rt3d_status rt3d_reconstruct(rt3d_session* s, const rt3d_recon_config* cfg) {
    NvtxRange nvtx_("rt3d_reconstruct");
    return run_init_like(s, cfg, PROG_RECON);
}

// n frames (one per session, each on its own resident cube) in one launch
// sequence on the first session's stream: every stage / neighbour kernel of
// the batch is one launch whose blocks split among the frames (FrameBatch),
// each frame with its own controller and grid barrier.  The sessions'
// streams are ordered before and after the batch, so their results read as
// after rt3d_reconstruct.
// One frame split into n row bands: session k owns
// the pixels of node k at depth log2(n) of pairwise_sum's tree, so each
// band's nll is an exact subtree and the combined tree is the single-GPU
// tree bit for bit.  Every session holds the same sensor and cube and
// full-size state arrays in the global index space; a band computes only its
// own pixels and points, and reads its neighbours' halo rows (ceil(W / s)
// coarse rows, W the APSS window) through halo_kernel before APSS and kNN.
// The bands' stage kernels are coupled: one grid barrier and one prune /
// spawn scan over all bands' blocks, one block-node array for the sweep
// trees.  Bands on one device run in one launch sequence; bands on several
// devices run one coupled launch sequence per device.  The result is
// identical to rt3d_reconstruct for any n.
rt3d_status rt3d_reconstruct_bands(rt3d_session* const* ss, int n, const rt3d_recon_config* cfg) {
    NvtxRange nvtx_("rt3d_reconstruct_bands");
    if (!ss || n < 1 || n > kMaxBatch || (n & (n - 1)))
        return fail(RT3D_ERR_INVALID_ARGUMENT, "rt3d: row bands: a power of two up to 16");
    for (int k = 0; k < n; ++k) {
        if (!ss[k]) return fail(RT3D_ERR_INVALID_ARGUMENT, "null session in bands");
        for (int j = 0; j < k; ++j)
            if (ss[j] == ss[k]) return fail(RT3D_ERR_INVALID_ARGUMENT, "rt3d: session twice in bands");
        if (!ss[k]->have_cube || !ss[k]->have_sensor)
            return fail(RT3D_ERR_INVALID_ARGUMENT, "rt3d: no sensor / cube set");
        if (ss[k]->rows != ss[0]->rows || ss[k]->cols != ss[0]->cols ||
            ss[k]->bins != ss[0]->bins || ss[k]->n_events != ss[0]->n_events)
            return fail(RT3D_ERR_INVALID_ARGUMENT, "rt3d: row bands need the same sensor and cube");
    }
    if (!cfg) return fail(RT3D_ERR_INVALID_ARGUMENT, "null config");
    if (n > 1 && cfg->background_mode != 0)
        return fail(RT3D_ERR_UNSUPPORTED, "rt3d: row bands need the identity background");
    rt3d_session* s0 = ss[0];
    static thread_local Frame Fs[kMaxBatch];
    rt3d_status st;
    for (int k = 0; k < n; ++k)
        if ((st = prepare_init_like(ss[k], cfg, PROG_RECON, Fs[k]))) return st;
    for (int k = 1; k < n; ++k)
        if (std::memcmp(&Fs[k].cfg, &Fs[0].cfg, sizeof(Cfg)) != 0)
            return fail(RT3D_ERR_UNSUPPORTED, "rt3d: bands built different sweep layouts");
    const uint32_t npix = Fs[0].npix, cols = (uint32_t)s0->cols;
    int d = 0;
    while ((1 << d) < n) ++d;
    if (n > 1) {
        if (!Fs[0].cfg.blocktree || !Fs[0].cfg.fuse_depth || Fs[0].cfg.fused_iter)
            return fail(RT3D_ERR_UNSUPPORTED, "rt3d: row bands need the default frame layout");
        if (Fs[0].tb_G < d)
            return fail(RT3D_ERR_UNSUPPORTED, "rt3d: frame too small for %d row bands", n);
    }
    const uint32_t hrows = (uint32_t)((Fs[0].cfg.W + s0->s - 1) / s0->s);
    const uint32_t halo_px = hrows * cols;
    for (int k = 0; k < n; ++k) {
        uint32_t lo, size;
        host_node_range(npix, d, (uint32_t)k, lo, size);
        if (n > 1 && (lo % cols != 0 || size < halo_px))
            return fail(RT3D_ERR_UNSUPPORTED,
                        "rt3d: row band %d [%u, %u) is not whole rows of at least %u rows", k, lo,
                        lo + size, hrows);
        Frame& F = Fs[k];
        F.nbands = n;
        F.band = k;
        if (n > 1) F.zb = nullptr;  // (the depth blocks would need halo rows too)
        F.bpix0 = lo;
        F.bpix1 = lo + size;
        F.bbn0 = (uint32_t)k * (F.tb_nbn / (uint32_t)n);
        F.bbn1 = F.bbn0 + F.tb_nbn / (uint32_t)n;
        F.halo_px = halo_px;
        // the sweep trees and the scans run over band 0's arrays
        for (int q = 0; q < 2; ++q) {
            F.tblk[q] = Fs[0].tblk[q];
            F.tbmax[q] = Fs[0].tbmax[q];
            F.tblk2[q] = Fs[0].tblk2[q];
        }
        F.btot = Fs[0].btot;
        ss[k]->band_pix0 = lo;
        ss[k]->band_pix1 = lo + size;
    }
    // bands on several GPUs: runs of consecutive bands on one device form a
    // launch on that device (its first session's stream), all launches with
    // the same stage blocks per band; the barrier, the scans and the halo
    // reads reach the other devices' buffers as peer memory over NVLink
    int gfirst[kMaxBatch], gcount[kMaxBatch], ng = 0, maxc = 0;
    for (int k = 0; k < n; ++k) {
        if (ng && ss[gfirst[ng - 1]]->device == ss[k]->device) {
            ++gcount[ng - 1];
        } else {
            gfirst[ng] = k;
            gcount[ng++] = 1;
        }
        maxc = std::max(maxc, gcount[ng - 1]);
    }
    for (int g = 0; g < ng; ++g)
        for (int h = 0; h < ng; ++h) {
            const int a = ss[gfirst[g]]->device, b = ss[gfirst[h]]->device;
            if (a == b) continue;
            int ok = 0;
            CUDA_TRY(cudaDeviceCanAccessPeer(&ok, a, b));
            if (!ok) return fail(RT3D_ERR_UNSUPPORTED, "rt3d: no peer access %d -> %d", a, b);
            CUDA_TRY(cudaSetDevice(a));
            const cudaError_t e = cudaDeviceEnablePeerAccess(b, 0);
            if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled)
                return fail(RT3D_ERR_CUDA, "CUDA: enable peer access: %s", cudaGetErrorString(e));
            cudaGetLastError();
        }
    const int cfgi = cfg_index(Fs[0].cfg.gsz);
    uint32_t bpf = 0xffffffffu;
    for (int g = 0; g < ng; ++g)
        bpf = std::min<uint32_t>(bpf, (uint32_t)std::max(1, ss[gfirst[g]]->grid_frame_c[cfgi] / maxc));
    for (int g = 0; g < ng; ++g) {
        rt3d_session* sl = ss[gfirst[g]];
        CUDA_TRY(cudaSetDevice(sl->device));
        for (int k = gfirst[g] + 1; k < gfirst[g] + gcount[g]; ++k) {
            CUDA_TRY(cudaEventRecord(ss[k]->xev, ss[k]->stream));
            CUDA_TRY(cudaStreamWaitEvent(sl->stream, ss[k]->xev, 0));
        }
        for (int k = gfirst[g]; k < gfirst[g] + gcount[g]; ++k)
            CUDA_TRY(cudaEventRecord(ss[k]->ev0, sl->stream));
    }
    // several devices: every controller (band 0's holds the barrier all
    // devices spin on) is zeroed before any device starts the frame
    if (ng > 1) {
        for (int k = 0; k < n; ++k) {
            CUDA_TRY(cudaSetDevice(ss[k]->device));
            CUDA_TRY(cudaStreamSynchronize(ss[k]->stream));
        }
        for (int g = 0; g < ng; ++g) {
            rt3d_session* sl = ss[gfirst[g]];
            CUDA_TRY(cudaSetDevice(sl->device));
            CUDA_TRY(cudaStreamSynchronize(sl->stream));
            for (int k = gfirst[g]; k < gfirst[g] + gcount[g]; ++k)
                CUDA_TRY(cudaMemsetAsync(Fs[k].ctl, 0, sizeof(Ctl), sl->stream));
            CUDA_TRY(cudaStreamSynchronize(sl->stream));
        }
    }
    // every device's launch sequence is issued before any waits: the coupled
    // cooperative kernels of all devices run concurrently
    for (int g = 0; g < ng; ++g) {
        rt3d_session* sl = ss[gfirst[g]];
        CUDA_TRY(cudaSetDevice(sl->device));
        if ((st = launch_frames(sl, Fs, n, gfirst[g], gcount[g], n > 1 ? bpf : 0u, ng == 1)))
            return st;
    }
    for (int g = 0; g < ng; ++g) {
        rt3d_session* sl = ss[gfirst[g]];
        CUDA_TRY(cudaSetDevice(sl->device));
        CUDA_TRY(cudaEventRecord(sl->xev, sl->stream));
        for (int k = gfirst[g]; k < gfirst[g] + gcount[g]; ++k) {
            CUDA_TRY(cudaEventRecord(ss[k]->ev1, sl->stream));
            if (k != gfirst[g]) CUDA_TRY(cudaStreamWaitEvent(ss[k]->stream, sl->xev, 0));
            finish_init_like(ss[k], cfg, PROG_RECON, n > 1);
        }
    }
    CUDA_TRY(cudaSetDevice(s0->device));
    return RT3D_OK;
}

// The row-band plan of rt3d_reconstruct_bands (host only): band k's pixels
// [begin[k], end[k]) = node k at depth log2(n) of pairwise_sum's tree, and
// the halo rows each band reads on either side (ceil(W / superres) rows of
// cols pixels, W = floor(R / pitch) + 1 fine pixels).
rt3d_status rt3d_band_plan(uint32_t n_rows, uint32_t n_cols, int32_t superres, double pixel_pitch,
                           double apss_radius, int32_t n, uint32_t* begin, uint32_t* end,
                           uint32_t* halo_rows) {
    if (n < 1 || n > kMaxBatch || (n & (n - 1)))
        return fail(RT3D_ERR_INVALID_ARGUMENT, "rt3d: row bands: a power of two up to 16");
    if (!begin || !end || !halo_rows || superres < 1 || !(pixel_pitch > 0.0) || !(apss_radius > 0.0))
        return fail(RT3D_ERR_INVALID_ARGUMENT, "rt3d: bad band plan arguments");
    int d = 0;
    while ((1 << d) < n) ++d;
    const uint32_t npix = n_rows * n_cols;
    const uint32_t hrows = (uint32_t)((window_w(apss_radius, pixel_pitch) + superres - 1) / superres);
    for (int k = 0; k < n; ++k) {
        uint32_t lo, size;
        host_node_range(npix, d, (uint32_t)k, lo, size);
        begin[k] = lo;
        end[k] = lo + size;
        if (n > 1 && (lo % n_cols != 0 || size < hrows * n_cols))
            return fail(RT3D_ERR_UNSUPPORTED,
                        "rt3d: row band %d [%u, %u) is not whole rows of at least %u rows", k, lo,
                        lo + size, hrows);
    }
    *halo_rows = hrows;
    return RT3D_OK;
}

rt3d_status rt3d_band_pixels(rt3d_session* s, uint32_t* pix0, uint32_t* pix1) {
    rt3d_status st = require_device(s);
    if (st) return st;
    if (!pix0 || !pix1) return fail(RT3D_ERR_INVALID_ARGUMENT, "null output");
    if (!s->have_state) return fail(RT3D_ERR_INVALID_ARGUMENT, "rt3d: no state in session");
    *pix0 = s->banded ? s->band_pix0 : 0u;
    *pix1 = s->banded ? s->band_pix1 : (uint32_t)(s->rows * s->cols);
    return RT3D_OK;
}

rt3d_status rt3d_reconstruct_batch(rt3d_session* const* ss, int n, const rt3d_recon_config* cfg) {
    NvtxRange nvtx_("rt3d_reconstruct_batch");
    if (!ss || n < 1 || n > kMaxBatch)
        return fail(RT3D_ERR_INVALID_ARGUMENT, "rt3d: batch of 1..%d sessions", kMaxBatch);
    for (int k = 0; k < n; ++k) {
        if (!ss[k]) return fail(RT3D_ERR_INVALID_ARGUMENT, "null session in batch");
        if (ss[k]->device != ss[0]->device)
            return fail(RT3D_ERR_INVALID_ARGUMENT, "rt3d: batched sessions must share a device");
        for (int j = 0; j < k; ++j)
            if (ss[j] == ss[k]) return fail(RT3D_ERR_INVALID_ARGUMENT, "rt3d: session twice in a batch");
    }
    rt3d_session* s0 = ss[0];
    static thread_local Frame Fs[kMaxBatch];
    rt3d_status st;
    for (int k = 0; k < n; ++k) {
        ss[k]->batch_hint = n;
        st = prepare_init_like(ss[k], cfg, PROG_RECON, Fs[k]);
        ss[k]->batch_hint = 1;
        if (st) return st;
    }
    for (int k = 1; k < n; ++k)
        if (std::memcmp(&Fs[k].cfg, &Fs[0].cfg, sizeof(Cfg)) != 0)
            return fail(RT3D_ERR_UNSUPPORTED,
                        "rt3d: batched frames need the same sweep layout (similar cubes)");
    for (int k = 1; k < n; ++k) {  // s0's stream after each session's uploads
        CUDA_TRY(cudaEventRecord(ss[k]->xev, ss[k]->stream));
        CUDA_TRY(cudaStreamWaitEvent(s0->stream, ss[k]->xev, 0));
    }
    for (int k = 0; k < n; ++k) CUDA_TRY(cudaEventRecord(ss[k]->ev0, s0->stream));
    if ((st = launch_frames(s0, Fs, n))) return st;
    CUDA_TRY(cudaEventRecord(s0->xev, s0->stream));
    for (int k = 0; k < n; ++k) {
        CUDA_TRY(cudaEventRecord(ss[k]->ev1, s0->stream));
        if (k) CUDA_TRY(cudaStreamWaitEvent(ss[k]->stream, s0->xev, 0));
        finish_init_like(ss[k], cfg, PROG_RECON);
    }
    return RT3D_OK;
}

static rt3d_status pipeline_init(rt3d_session* s) {
    if (s->cstream) return RT3D_OK;
    CUDA_TRY(cudaStreamCreateWithFlags(&s->cstream, cudaStreamNonBlocking));
    for (int k = 0; k < 2; ++k) {
        CUDA_TRY(cudaEventCreateWithFlags(&s->cube_ready[k], cudaEventDisableTiming));
        CUDA_TRY(cudaEventCreateWithFlags(&s->frame_done[k], cudaEventDisableTiming));
    }
    CUDA_TRY(cudaMallocHost(&s->h_res_ctl, sizeof(Ctl)));
    return RT3D_OK;
}

rt3d_status rt3d_frame_submit(rt3d_session* s, const rt3d_cube* c, const rt3d_recon_config* cfg,
                              uint64_t* ticket) {
    NvtxRange nvtx_("rt3d_frame_submit");
    rt3d_status st = require_device(s);
    if (st) return st;
    if (!c || !ticket) return fail(RT3D_ERR_INVALID_ARGUMENT, "null cube / ticket");
    if ((st = validate_cfg(cfg))) return st;
    if (!s->have_sensor) return fail(RT3D_ERR_INVALID_ARGUMENT, "rt3d: no sensor set");
    if (c->n_rows != s->rows || c->n_cols != s->cols || c->n_bins != s->bins)
        return fail(RT3D_ERR_INVALID_ARGUMENT, "likelihood: state/cube dimension mismatch");
    if ((st = pipeline_init(s))) return st;
    const int slot = (int)(s->next_ticket & 1u);
    if (s->inflight[slot])
        return fail(RT3D_ERR_INVALID_ARGUMENT, "rt3d: two frames in flight; collect ticket %llu first",
                    (unsigned long long)s->slot_ticket[slot]);
    const size_t npix = (size_t)c->n_rows * c->n_cols;
    if (s->h_off_cap[slot] < npix + 1) {
        if (s->h_off[slot]) cudaFreeHost(s->h_off[slot]);
        CUDA_TRY(cudaMallocHost(&s->h_off[slot], (npix + 1) * 4));
        s->h_off_cap[slot] = npix + 1;
    }
    if ((st = validate_cube(c, s->h_off[slot]))) return st;
    // H2D on the copy stream into this slot (its previous frame was collected)
    DevBuf& off = slot ? s->off2 : s->off;
    DevBuf& ev = slot ? s->ev2 : s->ev;
    CUDA_TRY(off.ensure((npix + 1) * 4));
    CUDA_TRY(ev.ensure(std::max<uint64_t>(c->n_events, 1) * 8));
    CUDA_TRY(cudaMemcpyAsync(off.p, s->h_off[slot], (npix + 1) * 4, cudaMemcpyHostToDevice, s->cstream));
    if (c->n_events)
        CUDA_TRY(cudaMemcpyAsync(ev.p, c->events, c->n_events * 8, cudaMemcpyHostToDevice, s->cstream));
    CUDA_TRY(cudaEventRecord(s->cube_ready[slot], s->cstream));
    CUDA_TRY(cudaStreamWaitEvent(s->stream, s->cube_ready[slot], 0));
    s->cube_slot = slot;
    s->have_cube = true;
    s->c_rows = c->n_rows;
    s->c_cols = c->n_cols;
    s->c_bins = c->n_bins;
    s->n_events = c->n_events;
    if ((st = run_init_like(s, cfg, PROG_RECON))) return st;
    // the frame's results into the slot, then the frame's completion event
    const size_t pcap = (size_t)cfg->init.max_returns * s->s * s->s * npix;
    CUDA_TRY(s->res_pts[slot].ensure(std::max<size_t>(pcap, 1) * sizeof(rt3d_point)));
    CUDA_TRY(s->res_bg[slot].ensure(npix * 8));
    CUDA_TRY(s->res_ctl[slot].ensure(sizeof(Ctl)));
    Frame F;
    Cfg g;
    std::memset(&g, 0, sizeof g);
    if ((st = build_frame(s, F, g, 1))) return st;
    gather_frame_kernel<<<s->nsm * 4, 256, 0, s->stream>>>(F, s->res_pts[slot].as<rt3d_point>(),
                                                          s->res_bg[slot].as<double>(),
                                                          s->res_ctl[slot].as<Ctl>());
    CUDA_TRY(cudaGetLastError());
    CUDA_TRY(cudaEventRecord(s->frame_done[slot], s->stream));
    s->inflight[slot] = 1;
    s->slot_ticket[slot] = s->next_ticket;
    s->slot_npix[slot] = npix;
    *ticket = s->next_ticket++;
    return RT3D_OK;
}

rt3d_status rt3d_frame_collect(rt3d_session* s, uint64_t ticket, rt3d_point* pts, uint64_t cap,
                               uint64_t* n_points, double* background, rt3d_report* info) {
    NvtxRange nvtx_("rt3d_frame_collect");
    rt3d_status st = require_device(s);
    if (st) return st;
    const int slot = (int)(ticket & 1u);
    if (!s->cstream || !s->inflight[slot] || s->slot_ticket[slot] != ticket)
        return fail(RT3D_ERR_INVALID_ARGUMENT, "rt3d: ticket %llu is not in flight",
                    (unsigned long long)ticket);
    CUDA_TRY(cudaStreamWaitEvent(s->cstream, s->frame_done[slot], 0));
    CUDA_TRY(cudaMemcpyAsync(s->h_res_ctl, s->res_ctl[slot].p, sizeof(Ctl), cudaMemcpyDeviceToHost,
                             s->cstream));
    CUDA_TRY(cudaStreamSynchronize(s->cstream));
    const Ctl& c = *s->h_res_ctl;
    if (n_points) *n_points = c.P;
    // a buffer too small keeps the frame in flight: collect it again with room
    if (pts && c.P > cap)
        return fail(RT3D_ERR_OUT_OF_RANGE, "rt3d: %u points do not fit in %llu", c.P,
                    (unsigned long long)cap);
    s->inflight[slot] = 0;
    if (c.abort)
        return fail(RT3D_ERR_CUDA, "rt3d: grid barrier watchdog aborted frame %llu",
                    (unsigned long long)ticket);
    const size_t npix = s->slot_npix[slot];
    if (pts && c.P)
        CUDA_TRY(cudaMemcpyAsync(pts, s->res_pts[slot].p, (size_t)c.P * sizeof(rt3d_point),
                                 cudaMemcpyDeviceToHost, s->cstream));
    if (background)
        CUDA_TRY(cudaMemcpyAsync(background, s->res_bg[slot].p, npix * 8, cudaMemcpyDeviceToHost,
                                 s->cstream));
    CUDA_TRY(cudaStreamSynchronize(s->cstream));
    if (info) {
        std::memset(info, 0, sizeof *info);
        info->iterations = c.iterations;
        info->points = c.P;
        info->init_nll = c.init_nll;
        info->final_nll = c.iterations > 0 ? c.prev : c.init_nll;
        const double init_s = (double)(c.t_init - c.t_start) * 1e-9;
        const double tot_s = (double)(c.t_end - c.t_start) * 1e-9;
        info->init_seconds = init_s;
        info->iterate_seconds = tot_s - init_s;
        info->total_seconds = tot_s;
    }
    return RT3D_OK;
}

rt3d_status rt3d_init_matched_filter(rt3d_session* s, const rt3d_init_params* p) {
    NvtxRange nvtx_("rt3d_init_matched_filter");
    if (!p) return fail(RT3D_ERR_INVALID_ARGUMENT, "null params");
    rt3d_recon_config c;
    std::memset(&c, 0, sizeof c);
    c.max_iters = 1;
    c.knn_k = 1;
    c.backtrack_beta = 0.5;
    c.apss.kernel_radius = 1.0;
    c.apss.min_neighbors = 6;
    c.init = *p;
    return run_init_like(s, &c, PROG_INIT);
}

rt3d_status rt3d_baseline_xcorr(rt3d_session* s) {
    rt3d_recon_config c;
    std::memset(&c, 0, sizeof c);
    c.max_iters = 1;
    c.knn_k = 1;
    c.backtrack_beta = 0.5;
    c.apss.kernel_radius = 1.0;
    c.apss.min_neighbors = 6;
    c.init.max_returns = 1;
    c.init.peak_threshold = 0.0;
    c.init.min_separation = 1;
    return run_init_like(s, &c, PROG_BASELINE);
}

rt3d_status rt3d_report_info(rt3d_session* s, rt3d_report* out) {
    rt3d_status st = require_device(s);
    if (st) return st;
    if (!out) return fail(RT3D_ERR_INVALID_ARGUMENT, "null out");
    if ((st = resolve_state(s))) return st;
    if ((st = read_ctl(s))) return st;
    const Ctl& c = *s->h_ctl;
    std::memset(out, 0, sizeof *out);
    out->iterations = c.iterations;
    out->points = c.P;
    out->init_nll = c.init_nll;
    out->final_nll = c.prev;
    out->init_seconds = c.t_init > c.t_start ? (c.t_init - c.t_start) * 1e-9 : 0.0;
    out->iterate_seconds = c.t_end > c.t_init ? (c.t_end - c.t_init) * 1e-9 : 0.0;
    float ms = 0.f;
    if (cudaEventElapsedTime(&ms, s->ev0, s->ev1) == cudaSuccess) out->total_seconds = ms * 1e-3;
    else cudaGetLastError();
    return RT3D_OK;
}

rt3d_status rt3d_report_copy(rt3d_session* s, double* trace, rt3d_step_diag* steps) {
    rt3d_status st = require_device(s);
    if (st) return st;
    if ((st = resolve_state(s))) return st;
    const int it = s->iterations;
    if (trace)
        CUDA_TRY(cudaMemcpyAsync(trace, s->trace.p, 8 * (it + 1), cudaMemcpyDeviceToHost, s->stream));
    if (steps && it > 0)
        CUDA_TRY(cudaMemcpyAsync(steps, s->diag.p, sizeof(rt3d_step_diag) * it,
                                 cudaMemcpyDeviceToHost, s->stream));
    CUDA_TRY(cudaStreamSynchronize(s->stream));
    return RT3D_OK;
}

rt3d_status rt3d_state_size(rt3d_session* s, uint64_t* n) {
    rt3d_status st = require_device(s);
    if (st) return st;
    if ((st = resolve_state(s))) return st;
    if (n) *n = s->P;
    return RT3D_OK;
}

rt3d_status rt3d_state_copy(rt3d_session* s, rt3d_point* pts, double* background) {
    NvtxRange nvtx_("rt3d_state_copy");
    rt3d_status st = require_device(s);
    if (st) return st;
    if ((st = resolve_state(s))) return st;
    const size_t npix = (size_t)s->rows * s->cols;
    if (pts && s->P) {
        Frame F;
        Cfg g;
        std::memset(&g, 0, sizeof g);
        if ((st = build_frame(s, F, g, 1))) return st;
        CUDA_TRY(s->outpts.ensure((size_t)s->P * sizeof(rt3d_point)));
        gather_points_kernel<<<(s->P + 255) / 256, 256, 0, s->stream>>>(
            F, s->pbase, s->P, s->tc, s->rc, s->sc, s->baseline_state ? 1 : 0,
            s->outpts.as<rt3d_point>());
        CUDA_TRY(cudaGetLastError());
        if (s->perm.empty()) {
            CUDA_TRY(cudaMemcpyAsync(pts, s->outpts.p, (size_t)s->P * sizeof(rt3d_point),
                                     cudaMemcpyDeviceToHost, s->stream));
        } else {
            std::vector<rt3d_point> tmp(s->P);
            CUDA_TRY(cudaMemcpyAsync(tmp.data(), s->outpts.p, (size_t)s->P * sizeof(rt3d_point),
                                     cudaMemcpyDeviceToHost, s->stream));
            CUDA_TRY(cudaStreamSynchronize(s->stream));
            for (size_t k = 0; k < s->P; ++k) pts[s->perm[k]] = tmp[k];
        }
    }
    if (background)
        CUDA_TRY(cudaMemcpyAsync(background, s->b[s->bc].p, npix * 8, cudaMemcpyDeviceToHost,
                                 s->stream));
    CUDA_TRY(cudaStreamSynchronize(s->stream));
    return RT3D_OK;
}

rt3d_status rt3d_state_upload(rt3d_session* s, const rt3d_state_view* v) {
    NvtxRange nvtx_("rt3d_state_upload");
    rt3d_status st = require_device(s);
    if (st) return st;
    if (!v) return fail(RT3D_ERR_INVALID_ARGUMENT, "null state");
    if (!s->have_sensor) return fail(RT3D_ERR_INVALID_ARGUMENT, "rt3d: no sensor set");
    const size_t npix = (size_t)s->rows * s->cols;
    const size_t n = v->n_points;
    if (n >= (1ull << 32)) return fail(RT3D_ERR_UNSUPPORTED, "rt3d: too many points");
    if (!v->background) return fail(RT3D_ERR_INVALID_ARGUMENT, "null background");
    // SceneState::refresh semantics (likelihood.hpp:38-55): stable counting
    // sort of the cloud by home pixel.
    std::vector<uint32_t> counts(npix, 0);
    for (size_t k = 0; k < n; ++k) {
        const rt3d_point& p = v->points[k];
        if (p.i < 0 || p.i >= s->rows || p.j < 0 || p.j >= s->cols)
            return fail(RT3D_ERR_INVALID_ARGUMENT, "SceneState: point home pixel out of bounds");
        ++counts[(size_t)p.i * s->cols + p.j];
    }
    std::vector<uint32_t> bo(npix + 1, 0);
    for (size_t p = 0; p < npix; ++p) bo[p + 1] = bo[p] + counts[p];
    std::vector<uint32_t> order(n);
    {
        std::vector<uint32_t> cur(bo.begin(), bo.end() - 1);
        for (size_t k = 0; k < n; ++k) {
            const rt3d_point& p = v->points[k];
            order[cur[(size_t)p.i * s->cols + p.j]++] = (uint32_t)k;
        }
    }
    bool identity = true;
    for (size_t k = 0; k < n && identity; ++k) identity = order[k] == k;
    uint32_t maxpp = 0;
    for (size_t p = 0; p < npix; ++p) maxpp = std::max(maxpp, counts[p]);
    s->max_pts_per_pixel = maxpp;
    bool pinned = true;
    std::vector<double> t(n), r(n);
    std::vector<uint32_t> pix(n);
    std::vector<int32_t> fi(n), fj(n);
    std::vector<uint8_t> fl(n);
    for (size_t k = 0; k < n; ++k) {
        const rt3d_point& p = v->points[order[k]];
        t[k] = p.t;
        r[k] = p.intensity;
        pix[k] = (uint32_t)((size_t)p.i * s->cols + p.j);
        fi[k] = p.fi;
        fj[k] = p.fj;
        fl[k] = p.flags;
        pinned = pinned && p.x == (p.fi + 0.5) * s->pitch && p.y == (p.fj + 0.5) * s->pitch &&
                 p.fi >= 0 && p.fj >= 0 && p.fi / s->s == p.i && p.fj / s->s == p.j;
    }
    if ((st = ensure_state(s, n, npix))) return st;
    s->tc = s->rc = s->bc = s->sc = 0;
    if (n) {
        CUDA_TRY(cudaMemcpyAsync(s->t[0].p, t.data(), n * 8, cudaMemcpyHostToDevice, s->stream));
        CUDA_TRY(cudaMemcpyAsync(s->r[0].p, r.data(), n * 8, cudaMemcpyHostToDevice, s->stream));
        CUDA_TRY(cudaMemcpyAsync(s->pix[0].p, pix.data(), n * 4, cudaMemcpyHostToDevice, s->stream));
        CUDA_TRY(cudaMemcpyAsync(s->fi[0].p, fi.data(), n * 4, cudaMemcpyHostToDevice, s->stream));
        CUDA_TRY(cudaMemcpyAsync(s->fj[0].p, fj.data(), n * 4, cudaMemcpyHostToDevice, s->stream));
        CUDA_TRY(cudaMemcpyAsync(s->fl[0].p, fl.data(), n, cudaMemcpyHostToDevice, s->stream));
    }
    CUDA_TRY(cudaMemcpyAsync(s->bo[0].p, bo.data(), (npix + 1) * 4, cudaMemcpyHostToDevice, s->stream));
    CUDA_TRY(cudaMemcpyAsync(s->b[0].p, v->background, npix * 8, cudaMemcpyHostToDevice, s->stream));
    CUDA_TRY(cudaStreamSynchronize(s->stream));
    s->have_state = true;
    s->baseline_state = false;
    s->state_pinned = pinned;
    s->P = (uint32_t)n;
    s->iterations = 0;
    s->perm.clear();
    if (!identity) s->perm = order;
    return RT3D_OK;
}

static rt3d_status run_sweeps(rt3d_session* s, int program) {
    rt3d_status st = require_device(s);
    if (st) return st;
    if ((st = resolve_state(s))) return st;
    if (s->banded)
        return fail(RT3D_ERR_UNSUPPORTED, "rt3d: a row band's state is a part of a frame");
    Cfg g;
    std::memset(&g, 0, sizeof g);
    g.program = program;
    g.max_iters = 1;
    Frame F;
    if ((st = build_frame(s, F, g, 1))) return st;
    if ((st = launch_frame(s, F, s->P))) return st;
    return RT3D_OK;
}

rt3d_status rt3d_nll(rt3d_session* s, double* out) {
    NvtxRange nvtx_("rt3d_nll");
    rt3d_status st = run_sweeps(s, PROG_NLL);
    if (st) return st;
    if ((st = read_ctl(s))) return st;
    if (out) *out = s->h_ctl->result;
    return RT3D_OK;
}

static rt3d_status run_grads(rt3d_session* s) { return run_sweeps(s, PROG_GRADS); }

rt3d_status rt3d_grad_depth(rt3d_session* s, double* value, uint8_t* oog) {
    NvtxRange nvtx_("rt3d_grad_depth");
    rt3d_status st = run_grads(s);
    if (st) return st;
    if ((st = copy_per_point(s, value, s->gt.p))) return st;
    return copy_per_point(s, oog, s->oog.p);
}

rt3d_status rt3d_grad_intensity(rt3d_session* s, double* out) {
    NvtxRange nvtx_("rt3d_grad_intensity");
    rt3d_status st = run_grads(s);
    if (st) return st;
    return copy_per_point(s, out, s->gr.p);
}

rt3d_status rt3d_grad_background(rt3d_session* s, double* out) {
    NvtxRange nvtx_("rt3d_grad_background");
    rt3d_status st = run_grads(s);
    if (st) return st;
    if (out) {
        CUDA_TRY(cudaMemcpyAsync(out, s->gb.p, (size_t)s->rows * s->cols * 8,
                                 cudaMemcpyDeviceToHost, s->stream));
        CUDA_TRY(cudaStreamSynchronize(s->stream));
    }
    return RT3D_OK;
}

rt3d_status rt3d_block_curvatures(rt3d_session* s, double* depth, double* intensity,
                                  double* background) {
    NvtxRange nvtx_("rt3d_block_curvatures");
    rt3d_status st = run_grads(s);
    if (st) return st;
    if ((st = copy_per_point(s, depth, s->ct.p))) return st;
    if ((st = copy_per_point(s, intensity, s->cr.p))) return st;
    if (background) {
        CUDA_TRY(cudaMemcpyAsync(background, s->cb.p, (size_t)s->rows * s->cols * 8,
                                 cudaMemcpyDeviceToHost, s->stream));
        CUDA_TRY(cudaStreamSynchronize(s->stream));
    }
    return RT3D_OK;
}

rt3d_status rt3d_palm_step(rt3d_session* s, const rt3d_recon_config* cfg, rt3d_step_diag* diag) {
    NvtxRange nvtx_("rt3d_palm_step");
    rt3d_status st = require_device(s);
    if (st) return st;
    if ((st = validate_cfg(cfg))) return st;
    if ((st = resolve_state(s))) return st;
    if (s->banded)
        return fail(RT3D_ERR_UNSUPPORTED, "rt3d: a row band's state is a part of a frame");
    if (!s->perm.empty())
        return fail(RT3D_ERR_UNSUPPORTED,
                    "rt3d: palm_step needs a pixel-ordered cloud (cloud order == bucket order)");
    if (!s->state_pinned || s->baseline_state)
        return fail(RT3D_ERR_UNSUPPORTED,
                    "rt3d: palm_step needs points at their fine-pixel centres (world_from_lidar)");
    Cfg g = cfg_from(cfg, PROG_PALM);
    g.W = window_w(cfg->apss.kernel_radius, s->pitch);
    g.set_oog_flags = 1;
    if (cfg->background_mode == 1 && (s->rows < 2 || s->cols < 2))
        return fail(RT3D_ERR_INVALID_ARGUMENT, "fft_lowpass_filter: image must be at least 2x2");
    Frame F;
    if ((st = build_frame(s, F, g, 1))) return st;
    if ((st = launch_frame(s, F, s->P))) return st;
    s->iterations = -1;
    if ((st = resolve_state(s))) return st;
    if (diag) {
        CUDA_TRY(cudaMemcpyAsync(diag, s->diag.p, sizeof(rt3d_step_diag), cudaMemcpyDeviceToHost,
                                 s->stream));
        CUDA_TRY(cudaStreamSynchronize(s->stream));
    }
    s->iterations = 0;
    return RT3D_OK;
}

rt3d_status rt3d_matched_filter_peaks(rt3d_session* s, const rt3d_event* events, uint64_t n,
                                      const rt3d_irf* irf, int32_t n_bins, int32_t k,
                                      double threshold, int32_t min_sep, rt3d_peak* out,
                                      int32_t* n_out) {
    NvtxRange nvtx_("rt3d_matched_filter_peaks");
    rt3d_status st = require_device(s);
    if (st) return st;
    if (!irf || !out || !n_out) return fail(RT3D_ERR_INVALID_ARGUMENT, "null argument");
    if (k > kMaxReturns) return fail(RT3D_ERR_UNSUPPORTED, "rt3d: k > %d", kMaxReturns);
    *n_out = 0;
    if (n == 0 || k < 1) return RT3D_OK;
    // a 1x1 sensor + cube holding the pixel; the session's own sensor/cube
    // are replaced (documented in rt3d.h usage of this test entry point)
    double gain = 1.0;
    uint8_t dead = 0;
    rt3d_sensor sv;
    std::memset(&sv, 0, sizeof sv);
    sv.n_rows = sv.n_cols = 1;
    sv.n_bins = n_bins;
    sv.superres = 1;
    sv.pixel_pitch = sv.bin_resolution = 1.0;
    sv.irf_shared = *irf;
    sv.gain = &gain;
    sv.dead = &dead;
    if ((st = rt3d_set_sensor(s, &sv))) return st;
    uint64_t offs[2] = {0, n};
    rt3d_cube cv;
    std::memset(&cv, 0, sizeof cv);
    cv.n_rows = cv.n_cols = 1;
    cv.n_bins = n_bins;
    cv.offsets = offs;
    cv.events = events;
    cv.n_events = n;
    if ((st = rt3d_set_cube(s, &cv))) return st;
    rt3d_recon_config c;
    std::memset(&c, 0, sizeof c);
    c.max_iters = 1;
    c.knn_k = 1;
    c.backtrack_beta = 0.5;
    c.apss.kernel_radius = 1.0;
    c.apss.min_neighbors = 6;
    c.init.max_returns = k;
    c.init.peak_threshold = threshold;
    c.init.min_separation = min_sep;
    Cfg g = cfg_from(&c, PROG_PEAKS);
    if ((st = ensure_state(s, 1, 1))) return st;
    Frame F;
    if ((st = build_frame(s, F, g, 1))) return st;
    if ((st = launch_frame(s, F, 0))) return st;
    uint32_t npk = 0;
    std::vector<double> t(k), rsp(k), mass(k);
    CUDA_TRY(cudaMemcpyAsync(&npk, s->npk.p, 4, cudaMemcpyDeviceToHost, s->stream));
    CUDA_TRY(cudaMemcpyAsync(t.data(), s->pk_t.p, 8 * k, cudaMemcpyDeviceToHost, s->stream));
    CUDA_TRY(cudaMemcpyAsync(rsp.data(), s->pk_resp.p, 8 * k, cudaMemcpyDeviceToHost, s->stream));
    CUDA_TRY(cudaMemcpyAsync(mass.data(), s->pk_mass.p, 8 * k, cudaMemcpyDeviceToHost, s->stream));
    CUDA_TRY(cudaStreamSynchronize(s->stream));
    for (uint32_t q = 0; q < npk; ++q) out[q] = rt3d_peak{t[q], rsp[q], mass[q]};
    *n_out = (int32_t)npk;
    s->have_state = false;
    return RT3D_OK;
}

// ---- arbitrary-cloud operators --------------------------------------------
// The device SpatialIndex of an index cloud (see for_each_grid): upload,
// cell keys, a stable radix sort of (key, index), run starts, the SoA in slot
// order.  `aos` keeps the index cloud in point order.
struct GridBufs {
    DevBuf aos, keys, idx, flag, pos, ukey, ustart, soa, tmp;
};
static rt3d_status build_grid(rt3d_session* s, const rt3d_point* cloud, uint64_t n, double cell,
                              GridBufs& g, CloudSoA& c) {
    const size_t nn = std::max<uint64_t>(n, 1);
    CUDA_TRY(g.aos.ensure(nn * sizeof(rt3d_point)));
    CUDA_TRY(g.keys.ensure(2 * nn * 8));
    CUDA_TRY(g.idx.ensure(2 * nn * 4));
    CUDA_TRY(g.flag.ensure(nn * 4));
    CUDA_TRY(g.pos.ensure(nn * 4));
    CUDA_TRY(g.ukey.ensure(nn * 8));
    CUDA_TRY(g.ustart.ensure((nn + 1) * 4));
    CUDA_TRY(g.soa.ensure(nn * 32));
    std::memset(&c, 0, sizeof c);
    c.cell = cell;
    c.n = (uint32_t)n;
    double* base = g.soa.as<double>();
    c.x = base;
    c.y = base + nn;
    c.z = base + 2 * nn;
    c.r = base + 3 * nn;
    c.ukey = g.ukey.as<unsigned long long>();
    c.ustart = g.ustart.as<uint32_t>();
    if (!n) return RT3D_OK;
    CUDA_TRY(cudaMemcpyAsync(g.aos.p, cloud, n * sizeof(rt3d_point), cudaMemcpyHostToDevice, s->stream));
    unsigned long long* k0 = g.keys.as<unsigned long long>();
    uint32_t* i0 = g.idx.as<uint32_t>();
    const uint32_t nb = (uint32_t)((n + 255) / 256);
    grid_keys_kernel<<<nb, 256, 0, s->stream>>>(g.aos.as<rt3d_point>(), (uint32_t)n, cell, k0, i0);
    CUDA_TRY(cudaGetLastError());
    cub::DoubleBuffer<unsigned long long> kb(k0, k0 + nn);
    cub::DoubleBuffer<uint32_t> vb(i0, i0 + nn);
    size_t tb = 0, ts = 0;
    CUDA_TRY(cub::DeviceRadixSort::SortPairs(nullptr, tb, kb, vb, (int)n, 0, 64, s->stream));
    CUDA_TRY(cub::DeviceScan::ExclusiveSum(nullptr, ts, g.flag.as<uint32_t>(), g.pos.as<uint32_t>(),
                                           (int)n, s->stream));
    CUDA_TRY(g.tmp.ensure(std::max(tb, ts)));
    tb = ts = g.tmp.cap;
    CUDA_TRY(cub::DeviceRadixSort::SortPairs(g.tmp.p, tb, kb, vb, (int)n, 0, 64, s->stream));
    grid_flags_kernel<<<nb, 256, 0, s->stream>>>(kb.Current(), (uint32_t)n, g.flag.as<uint32_t>());
    CUDA_TRY(cudaGetLastError());
    CUDA_TRY(cub::DeviceScan::ExclusiveSum(g.tmp.p, ts, g.flag.as<uint32_t>(), g.pos.as<uint32_t>(),
                                           (int)n, s->stream));
    grid_fill_kernel<<<nb, 256, 0, s->stream>>>(
        g.aos.as<rt3d_point>(), kb.Current(), vb.Current(), g.flag.as<uint32_t>(),
        g.pos.as<uint32_t>(), (uint32_t)n, g.ukey.as<unsigned long long>(), g.ustart.as<uint32_t>(),
        (double*)c.x, (double*)c.y, (double*)c.z, (double*)c.r);
    CUDA_TRY(cudaGetLastError());
    c.order = vb.Current();
    uint32_t last_pos = 0, last_flag = 0;
    CUDA_TRY(cudaMemcpyAsync(&last_pos, g.pos.as<uint32_t>() + (n - 1), 4, cudaMemcpyDeviceToHost, s->stream));
    CUDA_TRY(cudaMemcpyAsync(&last_flag, g.flag.as<uint32_t>() + (n - 1), 4, cudaMemcpyDeviceToHost, s->stream));
    CUDA_TRY(cudaStreamSynchronize(s->stream));
    c.ncell = last_pos + last_flag;
    return RT3D_OK;
}

static rt3d_status upload_points(rt3d_session* s, const rt3d_point* cloud, uint64_t n, DevBuf& aos) {
    CUDA_TRY(aos.ensure(std::max<uint64_t>(n, 1) * sizeof(rt3d_point)));
    if (n)
        CUDA_TRY(cudaMemcpyAsync(aos.p, cloud, n * sizeof(rt3d_point), cudaMemcpyHostToDevice,
                                 s->stream));
    return RT3D_OK;
}

rt3d_status rt3d_apss_project(rt3d_session* s, const rt3d_point* cloud, uint64_t n,
                              const rt3d_apss_params* prm, const rt3d_point* index_cloud,
                              uint64_t n_index, double cell, rt3d_point* out) {
    NvtxRange nvtx_("rt3d_apss_project");
    rt3d_status st = require_device(s);
    if (st) return st;
    if (!prm) return fail(RT3D_ERR_INVALID_ARGUMENT, "null params");
    if (prm->kernel_radius <= 0.0)
        return fail(RT3D_ERR_INVALID_ARGUMENT, "ApssParams: kernel_radius must be positive");
    if (prm->min_neighbors < 4)
        return fail(RT3D_ERR_INVALID_ARGUMENT, "ApssParams: min_neighbors must be >= 4");
    if (prm->sphere_degeneracy_eps < 0.0)
        return fail(RT3D_ERR_INVALID_ARGUMENT, "ApssParams: sphere_degeneracy_eps must be >= 0");
    if (cell <= 0.0) return fail(RT3D_ERR_INVALID_ARGUMENT, "SpatialIndex: cell size must be positive");
    if (n && prm->kernel_radius > cell * (1.0 + 1e-12))
        return fail(RT3D_ERR_INVALID_ARGUMENT, "SpatialIndex: query radius exceeds cell size");
    if (n >= (1ull << 32) || n_index >= (1ull << 32))
        return fail(RT3D_ERR_UNSUPPORTED, "rt3d: cloud too large");
    if (!n) return RT3D_OK;
    CloudSoA idx;
    DevBuf& aos_in = s->misc;
    static thread_local GridBufs grid;
    if ((st = build_grid(s, index_cloud, n_index, cell, grid, idx))) return st;
    if ((st = upload_points(s, cloud, n, aos_in))) return st;
    CUDA_TRY(s->outpts.ensure(n * sizeof(rt3d_point)));
    apss_general_kernel<<<(n + 127) / 128, 128, 0, s->stream>>>(
        aos_in.as<rt3d_point>(), (uint32_t)n, idx, prm->kernel_radius, prm->min_neighbors,
        prm->sphere_degeneracy_eps, s->outpts.as<rt3d_point>());
    CUDA_TRY(cudaGetLastError());
    CUDA_TRY(cudaMemcpyAsync(out, s->outpts.p, n * sizeof(rt3d_point), cudaMemcpyDeviceToHost,
                             s->stream));
    CUDA_TRY(cudaStreamSynchronize(s->stream));
    return RT3D_OK;
}

rt3d_status rt3d_knn_intensity_filter(rt3d_session* s, const rt3d_point* cloud, uint64_t n,
                                      int32_t k, const rt3d_point* index_cloud, uint64_t n_index,
                                      double cell, double radius, rt3d_point* out) {
    NvtxRange nvtx_("rt3d_knn_intensity_filter");
    rt3d_status st = require_device(s);
    if (st) return st;
    if (k < 1) return fail(RT3D_ERR_INVALID_ARGUMENT, "knn_intensity_filter: k must be >= 1");
    if (radius <= 0.0)
        return fail(RT3D_ERR_INVALID_ARGUMENT, "knn_intensity_filter: radius must be positive");
    if (cell <= 0.0) return fail(RT3D_ERR_INVALID_ARGUMENT, "SpatialIndex: cell size must be positive");
    if (n && radius > cell * (1.0 + 1e-12))
        return fail(RT3D_ERR_INVALID_ARGUMENT, "SpatialIndex: query radius exceeds cell size");
    if (n >= (1ull << 32) || n_index >= (1ull << 32))
        return fail(RT3D_ERR_UNSUPPORTED, "rt3d: cloud too large");
    if (!n) return RT3D_OK;
    CloudSoA idx;
    static thread_local GridBufs grid;
    if ((st = build_grid(s, index_cloud, n_index, cell, grid, idx))) return st;
    if ((st = upload_points(s, cloud, n, s->misc))) return st;
    CUDA_TRY(s->outpts.ensure(n * sizeof(rt3d_point)));
    knn_general_kernel<<<(n + 127) / 128, 128, 0, s->stream>>>(
        s->misc.as<rt3d_point>(), (uint32_t)n, idx, k, radius, grid.aos.as<rt3d_point>(),
        s->outpts.as<rt3d_point>());
    CUDA_TRY(cudaGetLastError());
    CUDA_TRY(cudaMemcpyAsync(out, s->outpts.p, n * sizeof(rt3d_point), cudaMemcpyDeviceToHost,
                             s->stream));
    CUDA_TRY(cudaStreamSynchronize(s->stream));
    return RT3D_OK;
}

rt3d_status rt3d_prune(rt3d_session* s, const rt3d_point* cloud, uint64_t n, double r_min,
                       rt3d_point* out, uint64_t* n_out) {
    NvtxRange nvtx_("rt3d_prune");
    rt3d_status st = require_device(s);
    if (st) return st;
    if (r_min < 0.0) return fail(RT3D_ERR_INVALID_ARGUMENT, "prune: r_min must be >= 0");
    if (!n_out) return fail(RT3D_ERR_INVALID_ARGUMENT, "null n_out");
    *n_out = 0;
    if (!n) return RT3D_OK;
    if (n >= (1ull << 32)) return fail(RT3D_ERR_UNSUPPORTED, "rt3d: cloud too large");
    CUDA_TRY(s->misc.ensure(n * sizeof(rt3d_point)));
    CUDA_TRY(s->outpts.ensure(n * sizeof(rt3d_point)));
    CUDA_TRY(cudaMemcpyAsync(s->misc.p, cloud, n * sizeof(rt3d_point), cudaMemcpyHostToDevice, s->stream));
    static thread_local DevBuf flags, tmp;
    CUDA_TRY(flags.ensure(8 * n + 16));
    uint32_t* flag = flags.as<uint32_t>();
    uint32_t* pos = flag + n;
    uint32_t* total = pos + n;
    const uint32_t nb = (uint32_t)((n + 255) / 256);
    prune_flags_kernel<<<nb, 256, 0, s->stream>>>(s->misc.as<rt3d_point>(), (uint32_t)n, r_min, flag);
    CUDA_TRY(cudaGetLastError());
    size_t tb = 0;
    CUDA_TRY(cub::DeviceScan::ExclusiveSum(nullptr, tb, flag, pos, (int)n, s->stream));
    CUDA_TRY(tmp.ensure(tb));
    tb = tmp.cap;
    CUDA_TRY(cub::DeviceScan::ExclusiveSum(tmp.p, tb, flag, pos, (int)n, s->stream));
    prune_scatter_kernel<<<nb, 256, 0, s->stream>>>(s->misc.as<rt3d_point>(), (uint32_t)n, flag, pos,
                                                    s->outpts.as<rt3d_point>(), total);
    CUDA_TRY(cudaGetLastError());
    uint32_t h_total = 0;
    CUDA_TRY(cudaMemcpyAsync(&h_total, total, 4, cudaMemcpyDeviceToHost, s->stream));
    CUDA_TRY(cudaStreamSynchronize(s->stream));
    if (h_total)
        CUDA_TRY(cudaMemcpy(out, s->outpts.p, (size_t)h_total * sizeof(rt3d_point), cudaMemcpyDeviceToHost));
    *n_out = h_total;
    return RT3D_OK;
}

rt3d_status rt3d_fft_lowpass_filter(rt3d_session* s, const double* img, int32_t rows, int32_t cols,
                                    double cutoff, int32_t clamp_nonneg, double* out) {
    NvtxRange nvtx_("rt3d_fft_lowpass_filter");
    rt3d_status st = require_device(s);
    if (st) return st;
    if (cutoff <= 0.0 || cutoff > 1.0)
        return fail(RT3D_ERR_INVALID_ARGUMENT, "fft_lowpass_filter: cutoff must be in (0, 1]");
    if (rows < 2 || cols < 2)
        return fail(RT3D_ERR_INVALID_ARGUMENT, "fft_lowpass_filter: image must be at least 2x2");
    const size_t total = (size_t)rows * cols;
    static thread_local DevBuf buf;
    CUDA_TRY(buf.ensure(total * 8 * 6));
    double* d = buf.as<double>();
    CUDA_TRY(cudaMemcpyAsync(d, img, total * 8, cudaMemcpyHostToDevice, s->stream));
    double *dimg = d, *dout = d + total, *re = d + 2 * total, *im = d + 3 * total,
           *re2 = d + 4 * total, *im2 = d + 5 * total;
    int nr = rows, nc = cols, cl = clamp_nonneg;
    void* args[] = {&dimg, &dout, &re, &im, &re2, &im2, &nr, &nc, &cutoff, &cl};
    CUDA_TRY(cudaLaunchCooperativeKernel((const void*)fft_kernel, dim3(s->grid_fft), dim3(kBlock),
                                         args, 2 * kFftMax * sizeof(double), s->stream));
    CUDA_TRY(cudaMemcpyAsync(out, dout, total * 8, cudaMemcpyDeviceToHost, s->stream));
    CUDA_TRY(cudaStreamSynchronize(s->stream));
    return RT3D_OK;
}

}  // extern "C"

rt3d_status rt3d_evaluate(rt3d_session* s, const rt3d_point* est, uint64_t n_est,
                          const rt3d_point* truth, uint64_t n_truth, double tau, double pitch,
                          rt3d_eval* out) {
    NvtxRange nvtx_("rt3d_evaluate");
    rt3d_status st = require_device(s);
    if (st) return st;
    if (!out) return fail(RT3D_ERR_INVALID_ARGUMENT, "null result");
    if (!(tau > 0.0)) return fail(RT3D_ERR_INVALID_ARGUMENT, "evaluate: tau must be positive");
    if (!(pitch > 0.0)) return fail(RT3D_ERR_INVALID_ARGUMENT, "evaluate: pitch must be positive");
    if ((n_est && !est) || (n_truth && !truth)) return fail(RT3D_ERR_INVALID_ARGUMENT, "null points");
    const uint64_t n = n_est + n_truth;
    if (n >= (1ull << 31)) return fail(RT3D_ERR_UNSUPPORTED, "rt3d: too many points");
    std::memset(out, 0, sizeof *out);
    out->n_est = n_est;
    out->n_truth = n_truth;
    if (n == 0 || n_est == 0 || n_truth == 0) {
        out->recall = n_truth ? 0.0 : 1.0;
        out->false_point_rate = n_est ? 1.0 : 0.0;
        return RT3D_OK;
    }
    CUDA_TRY(s->eval_pts.ensure(n * sizeof(rt3d_point)));
    for (int k = 0; k < 2; ++k) {
        CUDA_TRY(s->eval_k[k].ensure(n * 8));
        CUDA_TRY(s->eval_v[k].ensure(n * 4));
    }
    CUDA_TRY(s->eval_out.ensure(n * 16));
    CUDA_TRY(s->eval_cnt.ensure(n * 4 + 16));
    rt3d_point* dp = s->eval_pts.as<rt3d_point>();
    CUDA_TRY(cudaMemcpyAsync(dp, est, n_est * sizeof(rt3d_point), cudaMemcpyHostToDevice, s->stream));
    CUDA_TRY(cudaMemcpyAsync(dp + n_est, truth, n_truth * sizeof(rt3d_point), cudaMemcpyHostToDevice,
                             s->stream));
    unsigned int* bad = reinterpret_cast<unsigned int*>(s->eval_cnt.as<uint32_t>() + n);
    CUDA_TRY(cudaMemsetAsync(bad, 0, 4, s->stream));
    const int grid = s->nsm * 4;
    eval_keys_kernel<<<grid, 256, 0, s->stream>>>(dp, (uint32_t)n, pitch,
                                                 s->eval_k[0].as<unsigned long long>(),
                                                 s->eval_v[0].as<uint32_t>(), bad);
    CUDA_TRY(cudaGetLastError());
    cub::DoubleBuffer<unsigned long long> kb(s->eval_k[0].as<unsigned long long>(),
                                             s->eval_k[1].as<unsigned long long>());
    cub::DoubleBuffer<uint32_t> vb(s->eval_v[0].as<uint32_t>(), s->eval_v[1].as<uint32_t>());
    size_t tmp = 0;
    CUDA_TRY(cub::DeviceRadixSort::SortPairs(nullptr, tmp, kb, vb, (int)n, 0, 64, s->stream));
    CUDA_TRY(s->eval_tmp.ensure(tmp + 16));
    CUDA_TRY(cub::DeviceRadixSort::SortPairs(s->eval_tmp.p, tmp, kb, vb, (int)n, 0, 64, s->stream));
    eval_match_kernel<<<grid, 128, 0, s->stream>>>(dp, (uint32_t)n_est, (uint32_t)n, kb.Current(),
                                                  vb.Current(), tau, s->eval_out.as<double2>(),
                                                  s->eval_cnt.as<uint32_t>(), bad);
    CUDA_TRY(cudaGetLastError());
    std::vector<uint32_t> cnt(n + 1);
    std::vector<double2> val(n);
    CUDA_TRY(cudaMemcpyAsync(cnt.data(), s->eval_cnt.p, n * 4 + 4, cudaMemcpyDeviceToHost, s->stream));
    CUDA_TRY(cudaMemcpyAsync(val.data(), s->eval_out.p, n * 16, cudaMemcpyDeviceToHost, s->stream));
    CUDA_TRY(cudaStreamSynchronize(s->stream));
    if (cnt[n] & 1u) return fail(RT3D_ERR_UNSUPPORTED, "rt3d: evaluate column index beyond 2^31");
    if (cnt[n] & 2u)
        return fail(RT3D_ERR_UNSUPPORTED, "rt3d: evaluate column with more than %d points of a kind",
                    kEvalCap);
    // the sums in the reference's order: columns in key order, matches in order
    double sq_depth = 0.0, abs_intensity = 0.0;
    uint64_t matched = 0;
    for (uint64_t p = 0; p < n; ++p)
        for (uint32_t k = 0; k < cnt[p]; ++k) {
            sq_depth += val[p + k].x;
            abs_intensity += val[p + k].y;
            ++matched;
        }
    out->n_matched = matched;
    out->recall = (double)matched / (double)n_truth;
    out->false_point_rate = (double)(n_est - matched) / (double)n_est;
    out->depth_rmse = matched ? std::sqrt(sq_depth / (double)matched) : 0.0;
    out->intensity_mae = matched ? abs_intensity / (double)matched : 0.0;
    return RT3D_OK;
}


// simulate_cube's photon sampling (simulate.hpp:181-205) into the session's
// resident cube.  The truth buckets are a stable counting sort by coarse
// pixel (SceneState::refresh, likelihood.hpp:38-55) done on the host; the
// sampling, the offset scan and the event gather run on the device
// (rt3d_sim.cu).
rt3d_status rt3d_simulate_cube(rt3d_session* s, const rt3d_point* truth, uint64_t n_truth,
                               const double* background, uint64_t seed, uint64_t* n_events,
                               uint64_t* photons) {
    NvtxRange nvtx_("rt3d_simulate_cube");
    rt3d_status st = require_device(s);
    if (st) return st;
    if (!s->have_sensor) return fail(RT3D_ERR_INVALID_ARGUMENT, "simulate: no sensor set");
    if ((n_truth && !truth) || !background)
        return fail(RT3D_ERR_INVALID_ARGUMENT, "simulate: null truth / background");
    if (n_truth >= (1ull << 32)) return fail(RT3D_ERR_UNSUPPORTED, "rt3d: >= 2^32 truth points");
    const size_t npix = (size_t)s->rows * s->cols;
    std::vector<uint32_t> boff(npix + 1, 0), bpts(std::max<uint64_t>(n_truth, 1));
    std::vector<double> tt(std::max<uint64_t>(n_truth, 1)), rr(std::max<uint64_t>(n_truth, 1));
    for (uint64_t k = 0; k < n_truth; ++k) {
        const rt3d_point& q = truth[k];
        if (q.i < 0 || q.i >= s->rows || q.j < 0 || q.j >= s->cols)
            return fail(RT3D_ERR_OUT_OF_RANGE, "simulate: truth point %llu outside the sensor",
                        (unsigned long long)k);
        ++boff[(size_t)q.i * s->cols + q.j + 1];
        tt[k] = q.t;
        rr[k] = q.intensity;
    }
    for (size_t p = 0; p < npix; ++p) boff[p + 1] += boff[p];
    {
        std::vector<uint32_t> cur(boff.begin(), boff.end() - 1);
        for (uint64_t k = 0; k < n_truth; ++k)
            bpts[cur[(size_t)truth[k].i * s->cols + truth[k].j]++] = (uint32_t)k;
    }
    CUDA_TRY(cudaStreamSynchronize(s->stream));
    CUDA_TRY(s->sim_boff.ensure((npix + 1) * 4));
    CUDA_TRY(s->sim_bpts.ensure(bpts.size() * 4));
    CUDA_TRY(s->sim_t.ensure(tt.size() * 8));
    CUDA_TRY(s->sim_r.ensure(rr.size() * 8));
    CUDA_TRY(s->sim_bg.ensure(npix * 8));
    CUDA_TRY(s->sim_cnt.ensure((npix + 1) * 4));
    CUDA_TRY(s->sim_ph.ensure(16));
    CUDA_TRY(s->off.ensure((npix + 1) * 4));
    CUDA_TRY(cudaMemcpyAsync(s->sim_boff.p, boff.data(), (npix + 1) * 4, cudaMemcpyHostToDevice, s->stream));
    CUDA_TRY(cudaMemcpyAsync(s->sim_bpts.p, bpts.data(), bpts.size() * 4, cudaMemcpyHostToDevice, s->stream));
    CUDA_TRY(cudaMemcpyAsync(s->sim_t.p, tt.data(), tt.size() * 8, cudaMemcpyHostToDevice, s->stream));
    CUDA_TRY(cudaMemcpyAsync(s->sim_r.p, rr.data(), rr.size() * 8, cudaMemcpyHostToDevice, s->stream));
    CUDA_TRY(cudaMemcpyAsync(s->sim_bg.p, background, npix * 8, cudaMemcpyHostToDevice, s->stream));
    SimArgs a;
    a.irfs = s->irfs.as<IrfDev>();
    a.irf_of_pix = s->per_pixel_irf ? s->irf_of_pix.as<uint32_t>() : nullptr;
    a.gain = s->gain.as<double>();
    a.dead = s->dead.as<uint8_t>();
    a.background = s->sim_bg.as<double>();
    a.boff = s->sim_boff.as<uint32_t>();
    a.bpts = s->sim_bpts.as<uint32_t>();
    a.pt_t = s->sim_t.as<double>();
    a.pt_r = s->sim_r.as<double>();
    a.rows = s->rows;
    a.cols = s->cols;
    a.bins = s->bins;
    a.seed = seed;
    size_t tmp = 0;
    CUDA_TRY(sim_count(a, s->sim_cnt.as<uint32_t>(), s->off.as<uint32_t>(), nullptr, nullptr, &tmp,
                       s->stream));
    CUDA_TRY(s->sim_tmp.ensure(std::max<size_t>(tmp, 16)));
    CUDA_TRY(sim_count(a, s->sim_cnt.as<uint32_t>(), s->off.as<uint32_t>(),
                       s->sim_ph.as<unsigned long long>(), s->sim_tmp.p, &tmp, s->stream));
    uint32_t total = 0;
    unsigned long long ph[2] = {0, 0};
    CUDA_TRY(cudaMemcpyAsync(&total, s->off.as<uint32_t>() + npix, 4, cudaMemcpyDeviceToHost, s->stream));
    CUDA_TRY(cudaMemcpyAsync(ph, s->sim_ph.p, 16, cudaMemcpyDeviceToHost, s->stream));
    CUDA_TRY(cudaStreamSynchronize(s->stream));
    CUDA_TRY(s->ev.ensure(std::max<uint64_t>(total, 1) * 8));
    CUDA_TRY(sim_write(a, s->off.as<uint32_t>(), s->ev.as<uint2>(), s->stream));
    CUDA_TRY(cudaStreamSynchronize(s->stream));
    s->cube_slot = 0;
    s->have_cube = true;
    s->c_rows = s->rows;
    s->c_cols = s->cols;
    s->c_bins = s->bins;
    s->n_events = total;
    if (n_events) *n_events = total;
    if (photons) {
        photons[0] = ph[0];
        photons[1] = ph[1];
    }
    return RT3D_OK;
}

// The session's resident cube back to the host (PhotonCube CSR, cube.hpp:24-40).
rt3d_status rt3d_cube_copy(rt3d_session* s, uint64_t* offsets, rt3d_event* events) {
    NvtxRange nvtx_("rt3d_cube_copy");
    rt3d_status st = require_device(s);
    if (st) return st;
    if (!s->have_cube) return fail(RT3D_ERR_INVALID_ARGUMENT, "no cube set");
    const size_t npix = (size_t)s->c_rows * s->c_cols;
    const DevBuf& off = s->cube_slot ? s->off2 : s->off;
    const DevBuf& ev = s->cube_slot ? s->ev2 : s->ev;
    CUDA_TRY(cudaStreamSynchronize(s->stream));
    if (offsets) {
        std::vector<uint32_t> o(npix + 1);
        CUDA_TRY(cudaMemcpy(o.data(), off.p, (npix + 1) * 4, cudaMemcpyDeviceToHost));
        for (size_t p = 0; p <= npix; ++p) offsets[p] = o[p];
    }
    if (events && s->n_events)
        CUDA_TRY(cudaMemcpy(events, ev.p, s->n_events * 8, cudaMemcpyDeviceToHost));
    return RT3D_OK;
}
