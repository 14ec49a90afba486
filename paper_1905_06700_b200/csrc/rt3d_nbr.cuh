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
struct ApssWarpSm {
    double chunk[32][kChunkStride];
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
        int j = 0;
        for (uint32_t fb = 0; fb < total; fb += 32) {
            const uint32_t f = fb + lane;
            bool ok = false;
            Pos o;
            double d2 = 0.0;
            uint32_t mm = 0;
            if (f < total) {
                while (rt.pre[j + 1] <= f) ++j;
                mm = rt.m0[j] + (f - rt.pre[j]);
                o.x = (FI[mm] + 0.5) * F.pitch;
                o.y = (FJ[mm] + 0.5) * F.pitch;
                o.z = tt[mm] * F.bres;
                const double dx = o.x - q.x, dy = o.y - q.y, dz = o.z - q.z;
                d2 = dx * dx + dy * dy + dz * dz;
                ok = d2 <= r2;
            }
            const uint32_t bal = __ballot_sync(0xffffffffu, ok);
            if (!bal) continue;
            if (ok) visit(__popc(bal & lanemask_lt()), mm, o, d2);
            __syncwarp();
            flush(__popc(bal));
            __syncwarp();
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
            // pass A: ball size, wsum, weighted mean (denoise.hpp:172-186)
            double accA = 0.0;
            unsigned int cnt = 0;
            ball_scan(
                F, tc, sc, A.rt, fi, fj, q, r2,
                [&](int rank, uint32_t, const Pos& o, double d2) {
                    const double w = apss_weight(R, sqrt(d2));
                    double* c = A.chunk[rank];
                    c[0] = w;
                    c[1] = w * o.x;
                    c[2] = w * o.y;
                    c[3] = w * o.z;
                },
                [&](int nm) {
                    if (lane < 4)
                        for (int k = 0; k < nm; ++k) accA += A.chunk[k][lane];
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
            ball_scan(
                F, tc, sc, A.rt, fi, fj, q, r2,
                [&](int rank, uint32_t, const Pos& o, double d2) {
                    const double w = apss_weight(R, sqrt(d2));
                    const double y0 = o.x - m0, y1 = o.y - m1, y2 = o.z - m2;
                    double* c = A.chunk[rank];
                    c[0] = w;
                    c[1] = 1.0;
                    c[2] = y0;
                    c[3] = y1;
                    c[4] = y2;
                    c[5] = y0 * y0 + y1 * y1 + y2 * y2;
                },
                [&](int nm) {
                    if (lane < 6) {  // (w*d_r)*d_c over every member
                        for (int k = 0; k < nm; ++k) {
                            const double* c = A.chunk[k];
                            accB += c[0] * c[2 + ar] * c[2 + ac];
                        }
                    } else if (lane < 21) {  // (w*d5_r)*d5_c over members with w > 0
                        for (int k = 0; k < nm; ++k) {
                            const double* c = A.chunk[k];
                            const double w = c[0];
                            if (w <= 0.0) continue;
                            accB += w * c[1 + ar] * c[1 + ac];
                        }
                    }
                });
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
