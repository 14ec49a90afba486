// rt3d_nbr.cuh — APSS (denoise.hpp:159-217 + the pinning of
// reconstruct.hpp:352-363) and the kNN intensity filter (denoise.hpp:223-237)
// as stand-alone high-occupancy kernels, launched between the cooperative
// stage kernels of a frame.
//
// Work mapping: one warp per point.  Inside PALM every point sits at its
// fine-pixel centre, so SpatialIndex::query's ball (spatial_index.hpp:31-47,
// exact |q-p|^2 <= R^2, ascending index) is found among the points of the
// coarse pixels under the fine window [fi-W, fi+W] x [fj-W, fj+W],
// W = floor(R/pitch)+1.  The window's rows are contiguous index ranges (the
// cloud is pixel-major); the warp concatenates them and scans 32 candidates
// at a time (coalesced loads), compacting the members of each chunk with a
// ballot in ascending index order.  Every sum of the reference is then
// accumulated sequentially in that order by one lane per accumulator, so the
// result is bit-identical to the sequential loops of denoise.hpp.  The fit
// tail (3x3 eigenvalues, Pratt pencil, projection) runs one lane per point
// over the warp's batch of points.
#pragma once

#include "rt3d_frame.cuh"

namespace rt3d {

constexpr int kNbrBlock = 128;
constexpr int kNbrWarps = kNbrBlock / 32;
constexpr int kChunkStride = 9;  // doubles per staged member (odd: no bank conflicts)
constexpr int kMom = 25;         // wsum, mean(3), cov(6), M(15)
constexpr int kKnnCap = 512;     // per-warp ball list for the kNN selection

struct RowTab {
    uint32_t pre[33];  // exclusive prefix of the window rows' candidate counts
    uint32_t m0[32];   // first candidate index of each row
};
constexpr int kApssList = 256;  // ball members kept per warp (x, y, z, w)
struct ApssWarpSm {
    double chunk[32][kChunkStride];
    double list[kApssList][4];
    double mom[32][kMom];
    int32_t stat[32];
    RowTab rt;
};
struct KnnWarpSm {
    double d2[kKnnCap];
    uint32_t idx[kKnnCap];
    RowTab rt;
};

__device__ __forceinline__ uint32_t lanemask_lt() {
    uint32_t m;
    asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
    return m;
}

// Ball of q over the window; visit(rank, mm, pos, d2) on member lanes,
// flush(n_members) once per chunk (warp-synchronous).
template <typename Visit, typename Flush>
__device__ __forceinline__ void ball_scan(const Frame& F, int tc, int sc, RowTab& rt, int fi,
                                          int fj, const Pos& q, double r2, Visit visit,
                                          Flush flush) {
    const int lane = threadIdx.x & 31;
    const int W = F.cfg.W, s = F.s;
    const double rw = F.cfg.R / F.pitch;
    const double lim2 = rw * rw * (1.0 + 1e-9);
    int a0 = fi - W, a1 = fi + W;
    a0 = a0 < 0 ? 0 : a0;
    a1 = a1 > F.frows - 1 ? F.frows - 1 : a1;
    const int ci0 = a0 / s, ci1 = a1 / s;
    const uint32_t* bo = F.bo[sc];
    const double* tt = F.t[tc];
    const int32_t* FI = F.fi[sc];
    const int32_t* FJ = F.fj[sc];
    for (int rb = ci0; rb <= ci1; rb += 32) {
        // one window row per lane: its candidate range (disc-culled columns)
        const int ci = rb + lane;
        uint32_t m0 = 0, len = 0;
        if (ci <= ci1) {
            const int r_lo = ci * s, r_hi = r_lo + s - 1;
            const int dmin = fi < r_lo ? r_lo - fi : (fi > r_hi ? fi - r_hi : 0);
            const double rem = lim2 - (double)dmin * (double)dmin;
            if (rem >= 0.0) {
                int wj = (int)floor(sqrt(rem)) + 1;
                wj = wj > W ? W : wj;
                int b0 = fj - wj, b1 = fj + wj;
                b0 = b0 < 0 ? 0 : b0;
                b1 = b1 > F.fcols - 1 ? F.fcols - 1 : b1;
                const uint32_t prow = (uint32_t)ci * F.cols;
                m0 = bo[prow + b0 / s];
                len = bo[prow + b1 / s + 1] - m0;
            }
        }
        uint32_t inc = len;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, inc, o);
            if (lane >= o) inc += y;
        }
        rt.pre[lane] = inc - len;
        rt.m0[lane] = m0;
        const uint32_t total = __shfl_sync(0xffffffffu, inc, 31);
        if (lane == 31) rt.pre[32] = total;
        __syncwarp();
        // chunks of 32 candidates; the next chunk's loads are issued before
        // the current chunk is processed (software pipelining)
        int j = 0;
        auto locate = [&](uint32_t f) -> uint32_t {
            while (rt.pre[j + 1] <= f) ++j;
            return rt.m0[j] + (f - rt.pre[j]);
        };
        bool v = (uint32_t)lane < total;
        uint32_t mm = v ? locate(lane) : 0u;
        int cfi = v ? FI[mm] : 0, cfj = v ? FJ[mm] : 0;
        double ctt = v ? tt[mm] : 0.0;
        for (uint32_t fb = 0; fb < total; fb += 32) {
            const uint32_t f2 = fb + 32 + lane;
            const bool v2 = f2 < total;
            const uint32_t mm2 = v2 ? locate(f2) : 0u;
            const int nfi = v2 ? FI[mm2] : 0, nfj = v2 ? FJ[mm2] : 0;
            const double ntt = v2 ? tt[mm2] : 0.0;
            bool ok = false;
            Pos o;
            double d2 = 0.0;
            if (v) {
                o.x = (cfi + 0.5) * F.pitch;
                o.y = (cfj + 0.5) * F.pitch;
                o.z = ctt * F.bres;
                const double dx = o.x - q.x, dy = o.y - q.y, dz = o.z - q.z;
                d2 = dx * dx + dy * dy + dz * dz;
                ok = d2 <= r2;
            }
            const uint32_t bal = __ballot_sync(0xffffffffu, ok);
            if (bal) {
                if (ok) visit(__popc(bal & lanemask_lt()), mm, o, d2);
                __syncwarp();
                flush(__popc(bal));
                __syncwarp();
            }
            v = v2;
            mm = mm2;
            cfi = nfi;
            cfj = nfj;
            ctt = ntt;
        }
        __syncwarp();
    }
}

__device__ __forceinline__ void tri_index(int a, int& r, int& c) {
    r = 0;
    while ((r + 1) * (r + 2) / 2 <= a) ++r;
    c = a - r * (r + 1) / 2;
}

// APSS over the current state (toggles in ctl); writes t[tc^1] and flags.
__device__ void apss_warps(const Frame& F, ApssWarpSm* wsm) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    ApssWarpSm& A = wsm[warp];
    const Ctl* ctl = F.ctl;
    const uint32_t P = ld_cg(&ctl->P);
    const int tc = ld_cg(&ctl->tc), sc = ld_cg(&ctl->sc);
    const uint32_t gw = blockIdx.x * kNbrWarps + warp, nw = gridDim.x * kNbrWarps;
    const double R = F.cfg.R, r2 = R * R;
    // pass-B accumulator of this lane: lanes 0..5 covariance (lower, row-major),
    // lanes 6..20 the Pratt moments M (lower, row-major)
    int ar = 0, ac = 0;
    tri_index(lane < 6 ? lane : lane - 6, ar, ac);
    for (uint32_t first = gw; first < P; first += nw * 32u) {
        int nb = 0;
        for (int j = 0; j < 32; ++j) {
            const uint32_t n = first + (uint32_t)j * nw;
            if (n >= P) break;
            ++nb;
            const int fi = F.fi[sc][n], fj = F.fj[sc][n];
            const Pos q{(fi + 0.5) * F.pitch, (fj + 0.5) * F.pitch, F.t[tc][n] * F.bres};
            // pass A: ball size, wsum, weighted mean (denoise.hpp:172-186);
            // members (x, y, z, w) kept in the warp's list for pass B
            double accA = 0.0;
            unsigned int cnt = 0;
            ball_scan(
                F, tc, sc, A.rt, fi, fj, q, r2,
                [&](int rank, uint32_t, const Pos& o, double d2) {
                    const double w = apss_weight(R, sqrt(d2));
                    double* c = A.chunk[rank];
                    c[0] = w;
                    c[1] = o.x;
                    c[2] = o.y;
                    c[3] = o.z;
                    const unsigned int slot = cnt + (unsigned int)rank;
                    if (slot < (unsigned int)kApssList) {
                        A.list[slot][0] = o.x;
                        A.list[slot][1] = o.y;
                        A.list[slot][2] = o.z;
                        A.list[slot][3] = w;
                    }
                },
                [&](int nm) {
                    if (lane == 0) {
#pragma unroll 4
                        for (int k = 0; k < nm; ++k) accA += A.chunk[k][0];
                    } else if (lane < 4) {
#pragma unroll 4
                        for (int k = 0; k < nm; ++k) accA += A.chunk[k][0] * A.chunk[k][lane];
                    }
                    cnt += (unsigned int)nm;
                });
            const double wsum = __shfl_sync(0xffffffffu, accA, 0);
            double m0 = __shfl_sync(0xffffffffu, accA, 1);
            double m1 = __shfl_sync(0xffffffffu, accA, 2);
            double m2 = __shfl_sync(0xffffffffu, accA, 3);
            int st = 0;
            if (cnt < (unsigned int)F.cfg.min_nbrs) st = 1;  // isolated
            else if (wsum <= 0.0) st = 2;                    // degenerate
            if (st) {
                if (lane == 0) A.stat[j] = st;
                continue;
            }
            m0 /= wsum;
            m1 /= wsum;
            m2 /= wsum;
            // pass B: covariance (denoise.hpp:190-195) and the fit moments
            // M (denoise.hpp:73-80), centred on the mean
            double accB = 0.0;
            auto stage_member = [&](int rank, double x, double y, double z, double w) {
                const double y0 = x - m0, y1 = y - m1, y2 = z - m2;
                double* c = A.chunk[rank];
                c[0] = w;
                c[1] = 1.0;
                c[2] = y0;
                c[3] = y1;
                c[4] = y2;
                c[5] = y0 * y0 + y1 * y1 + y2 * y2;
            };
            auto flush_b = [&](int nm) {
                if (lane < 6) {  // (w*d_r)*d_c over every member
#pragma unroll 4
                    for (int k = 0; k < nm; ++k) {
                        const double* c = A.chunk[k];
                        accB += c[0] * c[2 + ar] * c[2 + ac];
                    }
                } else if (lane < 21) {  // (w*d5_r)*d5_c over members with w > 0
#pragma unroll 4
                    for (int k = 0; k < nm; ++k) {
                        const double* c = A.chunk[k];
                        const double w = c[0];
                        const double tm = w * c[1 + ar] * c[1 + ac];
                        if (w > 0.0) accB += tm;
                    }
                }
            };
            if (cnt <= (unsigned int)kApssList) {
                for (unsigned int base = 0; base < cnt; base += 32) {
                    const unsigned int k = base + lane;
                    if (k < cnt) stage_member(lane, A.list[k][0], A.list[k][1], A.list[k][2], A.list[k][3]);
                    __syncwarp();
                    flush_b((int)min(32u, cnt - base));
                    __syncwarp();
                }
            } else {  // ball larger than the list: walk the window again
                ball_scan(
                    F, tc, sc, A.rt, fi, fj, q, r2,
                    [&](int rank, uint32_t, const Pos& o, double d2) {
                        stage_member(rank, o.x, o.y, o.z, apss_weight(R, sqrt(d2)));
                    },
                    flush_b);
            }
            if (lane < 21) A.mom[j][4 + lane] = accB;
            if (lane == 0) {
                A.mom[j][0] = wsum;
                A.mom[j][1] = m0;
                A.mom[j][2] = m1;
                A.mom[j][3] = m2;
                A.stat[j] = 0;
            }
        }
        __syncwarp();
        // fit tail, one lane per point of the batch (denoise.hpp:186-214)
        if (lane < nb) {
            const uint32_t n = first + (uint32_t)lane * nw;
            const int fi = F.fi[sc][n], fj = F.fj[sc][n];
            const Pos q{(fi + 0.5) * F.pitch, (fj + 0.5) * F.pitch, F.t[tc][n] * F.bres};
            uint8_t fl = F.fl[sc][n] & (uint8_t)~(1u | 4u);
            double z = q.z;
            const int st = A.stat[lane];
            if (st == 1) {
                fl |= 1u;
            } else if (st == 2) {
                fl |= 4u;
            } else {
                const double* mo = A.mom[lane];
                const double wsum = mo[0];
                const double c00 = mo[4] / wsum, c10 = mo[5] / wsum, c11 = mo[6] / wsum,
                             c20 = mo[7] / wsum, c21 = mo[8] / wsum, c22 = mo[9] / wsum;
                double e0, e1, e2;
                sym3_eigenvalues(c00, c10, c11, c20, c21, c22, e0, e1, e2);
                Sphere sp;
                Pos o;
                if (e2 <= 0.0 || e1 <= 1e-12 * e2) {
                    fl |= 4u;
                } else {
                    double M[15];
#pragma unroll
                    for (int k = 0; k < 15; ++k) M[k] = mo[10 + k];
                    if (!sphere_from_moments(M, mo[1], mo[2], mo[3], sp) ||
                        !project_sphere(sp, F.cfg.eps, q.x, q.y, q.z, o.x, o.y, o.z))
                        fl |= 4u;
                    else
                        z = o.z;
                }
            }
            // reconstruct.hpp:359: t = clamp(z / bin_res, 0, T(1-1e-12))
            F.t[tc ^ 1][n] = std_clamp(z / F.bres, 0.0, F.tlim);
            F.fl[sc][n] = fl;
        }
        __syncwarp();
    }
}

// kNN intensity filter over the current state; writes r[rc^1].
__device__ void knn_warps(const Frame& F, KnnWarpSm* wsm) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    KnnWarpSm& K = wsm[warp];
    const Ctl* ctl = F.ctl;
    const uint32_t P = ld_cg(&ctl->P);
    const int tc = ld_cg(&ctl->tc), rc = ld_cg(&ctl->rc), sc = ld_cg(&ctl->sc);
    const uint32_t gw = blockIdx.x * kNbrWarps + warp, nw = gridDim.x * kNbrWarps;
    const double R = F.cfg.R, r2 = R * R;
    const double* rr = F.r[rc];
    const int k = F.cfg.knn_k;
    for (uint32_t n = gw; n < P; n += nw) {
        const int fi = F.fi[sc][n], fj = F.fj[sc][n];
        const Pos q{(fi + 0.5) * F.pitch, (fj + 0.5) * F.pitch, F.t[tc][n] * F.bres};
        unsigned int cnt = 0;
        ball_scan(
            F, tc, sc, K.rt, fi, fj, q, r2,
            [&](int rank, uint32_t mm, const Pos&, double d2) {
                const unsigned int slot = cnt + (unsigned int)rank;
                if (slot < (unsigned int)kKnnCap) {
                    K.d2[slot] = d2;
                    K.idx[slot] = mm;
                }
            },
            [&](int nm) { cnt += (unsigned int)nm; });
        // k smallest (d^2, index) in rank order (spatial_index.hpp:51-62),
        // averaged in that order (denoise.hpp:233-234)
        double last_d = 0.0, acc = 0.0;
        uint32_t last_i = 0;
        int taken = 0;
        const bool listed = cnt <= (unsigned int)kKnnCap;
        for (; taken < k && (unsigned int)taken < cnt; ++taken) {
            double bd = INFINITY;
            uint32_t bi = 0xffffffffu;
            auto consider = [&](double d, uint32_t i) {
                const bool after = taken == 0 || d > last_d || (d == last_d && i > last_i);
                if (after && (d < bd || (d == bd && i < bi))) {
                    bd = d;
                    bi = i;
                }
            };
            if (listed) {
                for (unsigned int e = lane; e < cnt; e += 32) consider(K.d2[e], K.idx[e]);
            } else {  // list overflow: rescan the ball
                ball_scan(
                    F, tc, sc, K.rt, fi, fj, q, r2,
                    [&](int, uint32_t mm, const Pos&, double d2) { consider(d2, mm); },
                    [&](int) {});
            }
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
                const double od = __shfl_xor_sync(0xffffffffu, bd, o);
                const uint32_t oi = __shfl_xor_sync(0xffffffffu, bi, o);
                if (od < bd || (od == bd && oi < bi)) {
                    bd = od;
                    bi = oi;
                }
            }
            acc += rr[bi];
            last_d = bd;
            last_i = bi;
        }
        const double result = cnt == 0 ? rr[n] : acc / (double)taken;
        if (lane == 0) F.r[rc ^ 1][n] = result;
        __syncwarp();
    }
}

}  // namespace rt3d

namespace rt3d {

// ---------------------------------------------------------------------------
// Tiled variant: a block owns a tile of TH x TW coarse pixels; the points of
// the tile plus a halo of ceil(W/s) coarse pixels are staged in shared memory
// (positions exactly as the reference computes them, global indices,
// per-staged-pixel offsets) with coalesced loads.  One thread per point then
// walks its window from shared memory in ascending global index and forms
// every sum sequentially, exactly like the loops of denoise.hpp.
// ---------------------------------------------------------------------------
constexpr int kTileThreads = 64;

struct TileView {
    double* x;
    double* y;
    double* z;
    uint32_t* gi;
    uint32_t* po;       // staged pixel -> first staged point (srows*scols + 1)
    uint32_t* rowpre;   // tile rows -> prefix of the tile's own points (TH + 1)
    int sr0, sc0, srows, scols;
};

__host__ __device__ __forceinline__ size_t tile_smem_bytes(int cap, int maxpix, int th) {
    return (size_t)cap * (3 * 8 + 4) + (size_t)(maxpix + 1) * 4 + (size_t)(th + 1) * 4 + 64;
}

// Window rows of (fi, fj) in the staged tile: fn(k0, k1) per row, ascending.
template <typename Fn>
__device__ __forceinline__ void tile_rows(const Frame& F, const TileView& T, int fi, int fj,
                                          Fn fn) {
    const int W = F.cfg.W, s = F.s;
    const double rw = F.cfg.R / F.pitch;
    const double lim2 = rw * rw * (1.0 + 1e-9);
    int a0 = fi - W, a1 = fi + W;
    a0 = a0 < 0 ? 0 : a0;
    a1 = a1 > F.frows - 1 ? F.frows - 1 : a1;
    const int ci0 = a0 / s, ci1 = a1 / s;
    for (int ci = ci0; ci <= ci1; ++ci) {
        const int r_lo = ci * s, r_hi = r_lo + s - 1;
        const int dmin = fi < r_lo ? r_lo - fi : (fi > r_hi ? fi - r_hi : 0);
        const double rem = lim2 - (double)dmin * (double)dmin;
        if (rem < 0.0) continue;
        int wj = (int)floor(sqrt(rem)) + 1;
        wj = wj > W ? W : wj;
        int b0 = fj - wj, b1 = fj + wj;
        b0 = b0 < 0 ? 0 : b0;
        b1 = b1 > F.fcols - 1 ? F.fcols - 1 : b1;
        const int sp = (ci - T.sr0) * T.scols - T.sc0;
        fn(T.po[sp + b0 / s], T.po[sp + b1 / s + 1]);
    }
}

// Ball of q, 4 candidates at a time: fn(k[4], d2[4], ok[4]) with the batch
// in ascending index (slots past the row end have ok = false).
template <typename Fn>
__device__ __forceinline__ void tile_ball4(const Frame& F, const TileView& T, int fi, int fj,
                                           const Pos& q, double r2, Fn fn) {
    tile_rows(F, T, fi, fj, [&](uint32_t k0, uint32_t k1) {
        for (uint32_t k = k0; k < k1; k += 4) {
            uint32_t kk[4];
            double d2[4];
            bool ok[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                kk[u] = k + u < k1 ? k + u : k1 - 1;
                const double dx = T.x[kk[u]] - q.x, dy = T.y[kk[u]] - q.y, dz = T.z[kk[u]] - q.z;
                d2[u] = dx * dx + dy * dy + dz * dz;
                ok[u] = (k + u < k1) && d2[u] <= r2;
            }
            fn(kk, d2, ok);
        }
    });
}

template <typename Fn>
__device__ __forceinline__ void tile_ball(const Frame& F, const TileView& T, int fi, int fj,
                                          const Pos& q, double r2, Fn fn) {
    tile_ball4(F, T, fi, fj, q, r2, [&](const uint32_t* kk, const double* d2, const bool* ok) {
#pragma unroll
        for (int u = 0; u < 4; ++u)
            if (ok[u]) fn(kk[u], d2[u]);
    });
}

// APSS + pinning of point n (denoise.hpp:163-214, reconstruct.hpp:357-361):
// pass 1 the mean, pass 2 covariance and fit moments, each in ascending index
__device__ __forceinline__ void apss_thread(const Frame& F, const TileView& T, int tc, int sc,
                                            uint32_t n) {
    const double R = F.cfg.R, r2 = R * R;
    const int fi = F.fi[sc][n], fj = F.fj[sc][n];
    const Pos q{(fi + 0.5) * F.pitch, (fj + 0.5) * F.pitch, F.t[tc][n] * F.bres};
    uint8_t fl = F.fl[sc][n] & (uint8_t)~(1u | 4u);
    double z = q.z;
    unsigned int cnt = 0;
    double wsum = 0.0, m0 = 0.0, m1 = 0.0, m2 = 0.0;
    // Branch-free batches of 4 candidates (in ascending index): weights first
    // (independent sqrt/div), then the sums in order.  A non-member adds
    // exactly +0.0 (w = 0): every accumulator starts at +0.0 and can never be
    // -0.0, so the sums equal the reference's member-only loops bit for bit.
    tile_ball4(F, T, fi, fj, q, r2, [&](const uint32_t* kk, const double* d2, const bool* ok) {
        double w[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const double wu = apss_weight(R, sqrt(d2[u]));
            w[u] = ok[u] ? wu : 0.0;
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            cnt += ok[u] ? 1u : 0u;
            wsum += w[u];
            m0 += w[u] * T.x[kk[u]];
            m1 += w[u] * T.y[kk[u]];
            m2 += w[u] * T.z[kk[u]];
        }
    });
    if (cnt < (unsigned int)F.cfg.min_nbrs) {
        fl |= 1u;
    } else if (wsum <= 0.0) {
        fl |= 4u;
    } else {
        m0 /= wsum;
        m1 /= wsum;
        m2 /= wsum;
        double c00 = 0, c10 = 0, c11 = 0, c20 = 0, c21 = 0, c22 = 0;
        double M[15];
#pragma unroll
        for (int k = 0; k < 15; ++k) M[k] = 0.0;
        tile_ball4(F, T, fi, fj, q, r2, [&](const uint32_t* kk, const double* d2, const bool* ok) {
            double w[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const double wu = apss_weight(R, sqrt(d2[u]));
                w[u] = ok[u] ? wu : 0.0;
            }
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                // d (= y) of non-members is zeroed so their terms are +0.0
                const double y0 = ok[u] ? T.x[kk[u]] - m0 : 0.0;
                const double y1 = ok[u] ? T.y[kk[u]] - m1 : 0.0;
                const double y2 = ok[u] ? T.z[kk[u]] - m2 : 0.0;
                const double w0 = w[u] * y0, w1 = w[u] * y1, w2 = w[u] * y2;
                c00 += w0 * y0;
                c10 += w1 * y0;
                c11 += w1 * y1;
                c20 += w2 * y0;
                c21 += w2 * y1;
                c22 += w2 * y2;
                // M: members with w <= 0 are skipped (denoise.hpp:75): wm = 0
                const double wm = w[u] > 0.0 ? w[u] : 0.0;
                const double dv[5] = {1.0, y0, y1, y2, y0 * y0 + y1 * y1 + y2 * y2};
#pragma unroll
                for (int a = 0; a < 5; ++a) {
                    const double wa = wm * dv[a];
#pragma unroll
                    for (int c = 0; c <= a; ++c) M[lt(a, c)] += wa * dv[c];
                }
            }
        });
        c00 /= wsum;
        c10 /= wsum;
        c11 /= wsum;
        c20 /= wsum;
        c21 /= wsum;
        c22 /= wsum;
        double e0, e1, e2;
        sym3_eigenvalues(c00, c10, c11, c20, c21, c22, e0, e1, e2);
        Sphere sp;
        Pos o;
        if (e2 <= 0.0 || e1 <= 1e-12 * e2) {
            fl |= 4u;
        } else if (!sphere_from_moments(M, m0, m1, m2, sp) ||
                   !project_sphere(sp, F.cfg.eps, q.x, q.y, q.z, o.x, o.y, o.z)) {
            fl |= 4u;
        } else {
            z = o.z;
        }
    }
    F.t[tc ^ 1][n] = std_clamp(z / F.bres, 0.0, F.tlim);
    F.fl[sc][n] = fl;
}

// kNN mean of point n (denoise.hpp:228-235; spatial_index.hpp:51-62)
__device__ __forceinline__ void knn_thread(const Frame& F, const TileView& T, int tc, int rc,
                                           int sc, uint32_t n) {
    const double R = F.cfg.R, r2 = R * R;
    const int fi = F.fi[sc][n], fj = F.fj[sc][n];
    const Pos q{(fi + 0.5) * F.pitch, (fj + 0.5) * F.pitch, F.t[tc][n] * F.bres};
    const double* rr = F.r[rc];
    auto each = [&](double rr2, auto fn) {
        tile_ball(F, T, fi, fj, q, rr2, [&](uint32_t k, double d2) {
            Pos o{T.x[k], T.y[k], T.z[k]};
            fn(T.gi[k], o, d2);
        });
    };
    F.r[rc ^ 1][n] = knn_mean(each, F.cfg.knn_k, r2, rr[n], [&](uint32_t m) { return rr[m]; });
}

// Launch: one block per tile (grid = number of tiles), tile edge from Cfg.
template <int MODE>
__device__ void nbr_tile_block(const Frame& F, unsigned char* smem, int cap) {
    const Ctl* ctl = F.ctl;
    const int tc = ld_cg(&ctl->tc), rc = ld_cg(&ctl->rc), sc = ld_cg(&ctl->sc);
    const int TH = F.cfg.tile_h, TW = F.cfg.tile_w, h = F.cfg.halo;
    const int tcols = (F.cols + TW - 1) / TW;
    const int r0 = (int)(blockIdx.x / tcols) * TH, c0 = (int)(blockIdx.x % tcols) * TW;
    TileView T;
    T.sr0 = r0 - h < 0 ? 0 : r0 - h;
    T.sc0 = c0 - h < 0 ? 0 : c0 - h;
    const int sr1 = r0 + TH + h > F.rows ? F.rows : r0 + TH + h;
    const int sc1 = c0 + TW + h > F.cols ? F.cols : c0 + TW + h;
    T.srows = sr1 - T.sr0;
    T.scols = sc1 - T.sc0;
    const int npix = T.srows * T.scols;
    T.x = reinterpret_cast<double*>(smem);
    T.y = T.x + cap;
    T.z = T.y + cap;
    T.gi = reinterpret_cast<uint32_t*>(T.z + cap);
    T.po = T.gi + cap;
    T.rowpre = T.po + (npix + 1);
    __shared__ int32_t s_rowbase[128];
    const uint32_t* bo = F.bo[sc];
    // staged rows: contiguous global ranges; their local bases by a serial scan
    if (threadIdx.x == 0) {
        int acc = 0;
        for (int r = 0; r < T.srows; ++r) {
            const uint32_t prow = (uint32_t)(T.sr0 + r) * F.cols + T.sc0;
            s_rowbase[r] = acc;
            acc += (int)(bo[prow + T.scols] - bo[prow]);
        }
        // the tile's own rows: prefix of their point counts
        const int tr1 = r0 + TH > F.rows ? F.rows : r0 + TH;
        const int tc1 = c0 + TW > F.cols ? F.cols : c0 + TW;
        uint32_t pre = 0;
        for (int r = r0; r <= tr1; ++r) {
            T.rowpre[r - r0] = pre;
            if (r < tr1) pre += bo[(uint32_t)r * F.cols + tc1] - bo[(uint32_t)r * F.cols + c0];
        }
    }
    __syncthreads();
    for (int qp = threadIdx.x; qp < npix; qp += blockDim.x) {
        const int r = qp / T.scols, c = qp % T.scols;
        const uint32_t prow = (uint32_t)(T.sr0 + r) * F.cols + T.sc0;
        T.po[qp] = (uint32_t)s_rowbase[r] + (bo[prow + c] - bo[prow]);
    }
    if (threadIdx.x == 0) {
        const uint32_t prow = (uint32_t)(T.sr0 + T.srows - 1) * F.cols + T.sc0;
        T.po[npix] = (uint32_t)s_rowbase[T.srows - 1] + (bo[prow + T.scols] - bo[prow]);
    }
    for (int r = 0; r < T.srows; ++r) {
        const uint32_t prow = (uint32_t)(T.sr0 + r) * F.cols + T.sc0;
        const uint32_t m0 = bo[prow], m1 = bo[prow + T.scols];
        const int base = s_rowbase[r];
        for (uint32_t mm = m0 + threadIdx.x; mm < m1; mm += blockDim.x) {
            const int k = base + (int)(mm - m0);
            T.x[k] = (F.fi[sc][mm] + 0.5) * F.pitch;
            T.y[k] = (F.fj[sc][mm] + 0.5) * F.pitch;
            T.z[k] = F.t[tc][mm] * F.bres;
            T.gi[k] = mm;
        }
    }
    __syncthreads();
    // the tile's own points, row by row
    const int tr1 = r0 + TH > F.rows ? F.rows : r0 + TH;
    const int tc1 = c0 + TW > F.cols ? F.cols : c0 + TW;
    const uint32_t total = T.rowpre[tr1 - r0];
    for (uint32_t k = threadIdx.x; k < total; k += blockDim.x) {
        int r = r0;
        while (T.rowpre[r - r0 + 1] <= k) ++r;
        const uint32_t n = bo[(uint32_t)r * F.cols + c0] + (k - T.rowpre[r - r0]);
        if (MODE == 0) apss_thread(F, T, tc, sc, n);
        else knn_thread(F, T, tc, rc, sc, n);
    }
}

}  // namespace rt3d
