// rt3d_nbr.cuh — APSS (denoise.hpp:159-217 + the pinning of
// reconstruct.hpp:352-363) and the kNN intensity filter (denoise.hpp:223-237)
// as stand-alone high-occupancy kernels, launched between the cooperative
// stage kernels of a frame.
//
// Work mapping: 16 lanes per point, two points per warp (APSS and kNN); two
// points in the same or adjacent fine cells share one 32-lane scan of their
// windows' union (APSS).  Inside PALM every point sits at its fine-pixel centre, so
// SpatialIndex::query's ball (spatial_index.hpp:31-47, exact |q-p|^2 <= R^2,
// ascending index) is found among the points of the coarse pixels under the
// fine window [fi-W, fi+W] x [fj-W, fj+W], W = floor(R/pitch)+1.  The
// window's rows are contiguous index ranges (the cloud is pixel-major); the
// group concatenates them and scans one candidate per lane at a time
// (coalesced loads), compacting the members of each chunk with a ballot in
// ascending index order.
//
// APSS moments: ball member m (ascending index) is accumulated by the group's
// lane m mod 16, sequentially; the 16 lane partials are combined by the
// halving tree p[l] += p[l+o], o = 8..1.  The oracle uses the same order
// (oracle/rt3d_oracle.c, lane_tree, APSS_LANES), so device and oracle agree
// bit for bit.  The sphere fit and projection then run one thread per point
// (apss_fit_kernel; apss_fit_split_kernel for single small frames) from the
// moments staged in L2.
#pragma once

#include "rt3d_frame.cuh"

namespace rt3d {

constexpr int kNbrBlock = 128;
constexpr int kNbrWarps = kNbrBlock / 32;
constexpr int kKnnCap = 192;     // per-point ball list for the kNN selection (two per warp)
constexpr int kFitBlock = 128;

// Lane groups of GW lanes scanning one point's window each: GW = 32 (kNN, a
// warp per point) or 16 (APSS, two points per warp).  Warp-collective
// operations run over the whole warp; each group reads its own field of a
// ballot, and every loop that contains one runs to the larger of the two
// groups' trip counts (the shorter group idles, predicated off).
template <int GW>
struct Grp {
    static_assert(GW == 16 || GW == 32, "lane groups of 16 or 32");
    __device__ static __forceinline__ int gl() { return (int)(threadIdx.x & (GW - 1)); }
    __device__ static __forceinline__ int base() { return GW == 32 ? 0 : (int)(threadIdx.x & 16u); }
    // this group's bits of a full-warp ballot
    __device__ static __forceinline__ uint32_t field(uint32_t b) {
        return GW == 32 ? b : (b >> base()) & 0xFFFFu;
    }
    __device__ static __forceinline__ uint32_t lt() { return (1u << gl()) - 1u; }
    __device__ static __forceinline__ uint32_t le() { return (2u << gl()) - 1u; }
    // the larger of the two groups' values (warp-uniform)
    __device__ static __forceinline__ uint32_t wmax(uint32_t v) {
        return GW == 32 ? v : max(v, __shfl_xor_sync(0xffffffffu, v, 16));
    }
};

struct RowTab {
    // the batch's non-empty rows, compacted in row order
    uint32_t pre[32];  // rank of the row's first candidate (strictly increasing)
    uint32_t m0[32];   // index of the row's first candidate
    uint32_t n;        // number of non-empty rows
};

// APSS: two points per warp, 16 lanes each (see apss_moment_warps)
constexpr int kApssGW = kApssLanes;
// ball members kept per point for the dense passes (larger balls take
// chunk-by-chunk rescans): 208 keeps the warp's scratch at 10.9 KB, so five
// 4-warp blocks share an SM (the balls of B and E hold <= ~206)
constexpr int kApssCap = 208;
struct ApssList {
    double z[kApssCap], w[kApssCap];  // member depth, d^2 then weight
    uint32_t fij[kApssCap];           // member fine cell, fi << 16 | fj
};
struct ApssWarpSm {
    union {
        ApssList list[2];            // one per lane group
        double red[32][kRedStride];  // lane partials, after the lists are consumed
    } u;
    double chunk[32][4];  // the current scan chunk's members (w, x, y, z), a group's 16 slots
    RowTab rt[2];
    uint2 rng[2][64];  // depth-block candidate ranges (ball_scan_blocks)
};
struct KnnList {              // one lane group's ball list
    double d2[kKnnCap];
    uint32_t idx[kKnnCap];
    uint32_t sel[kKnnCap];  // the selection in rank order
    double kth;
};
struct KnnWarpSm {
    KnnList l[2];
    RowTab rt[2];
};

__device__ __forceinline__ uint32_t lanemask_lt() {
    uint32_t m;
    asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
    return m;
}

// Window rows of point (fi, fj): coarse rows ci0..ci1 (fine window of
// half-width W, clipped).
__device__ __forceinline__ void window_rows(const Frame& F, int fi, int W, int& ci0, int& ci1) {
    int a0 = fi - W, a1 = fi + W;
    a0 = a0 < 0 ? 0 : a0;
    a1 = a1 > F.frows - 1 ? F.frows - 1 : a1;
    ci0 = coarse_of(F, a0);
    ci1 = coarse_of(F, a1);
}

// Candidate range of window row ci = rb + (lane in group) (disc-culled
// columns): the global loads of a row batch, kept in registers until
// rows_finish.
template <int GW>
__device__ __forceinline__ void rows_load(const Frame& F, int sc, int fi, int fj, int W, int rb,
                                          int ci1, uint32_t& m0, uint32_t& len) {
    const int s = F.s;
    const double rw = F.cfg.R / F.pitch;
    const double lim2 = rw * rw * (1.0 + 1e-9);
    const int ci = rb + Grp<GW>::gl();
    m0 = 0;
    len = 0;
    if (ci <= ci1) {
        const int r_lo = ci * s, r_hi = r_lo + s - 1;
        const int dmin = fi < r_lo ? r_lo - fi : (fi > r_hi ? fi - r_hi : 0);
        const double rem = lim2 - (double)dmin * (double)dmin;
        if (rem >= 0.0) {
            // a member at column offset b has (b pitch)^2 <= R^2 - (a pitch)^2
            // up to rounding far below the 1e-9 margin of lim2, so
            // |b| <= floor(sqrt(rem)) bounds every member of this row
            int wj = (int)floor(sqrt(rem));
            wj = wj > W ? W : wj;
            int b0 = fj - wj, b1 = fj + wj;
            b0 = b0 < 0 ? 0 : b0;
            b1 = b1 > F.fcols - 1 ? F.fcols - 1 : b1;
            const uint32_t prow = (uint32_t)ci * F.cols;
            const uint32_t* bo = F.bo[sc];
            const int c0 = coarse_of(F, b0), c1 = coarse_of(F, b1);
            m0 = bo[prow + c0];
            len = bo[prow + c1 + 1] - m0;
        }
    }
}

// prefix of the group's row batch into rt (non-empty rows compacted);
// returns the batch's candidate count
template <int GW>
__device__ __forceinline__ uint32_t rows_finish(RowTab& rt, uint32_t m0, uint32_t len) {
    using G = Grp<GW>;
    const int gl = G::gl();
    uint32_t inc = len;
#pragma unroll
    for (int o = 1; o < GW; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, inc, o, GW);
        if (gl >= o) inc += y;
    }
    const uint32_t ne = G::field(__ballot_sync(0xffffffffu, len != 0u));
    if (len) {
        const int cp = __popc(ne & G::lt());
        rt.pre[cp] = inc - len;
        rt.m0[cp] = m0;
    }
    const uint32_t total = __shfl_sync(0xffffffffu, inc, GW - 1, GW);
    if (gl == 0) rt.n = (uint32_t)__popc(ne);
    __syncwarp();
    return total;
}

// The candidates of the group's row batch (rt, total) against q: visit(rank,
// mm, pos, d2, fi, fj) on member lanes, flush(n_members) once per chunk of GW
// candidates (warp-synchronous); the next chunk's loads are issued before the
// current chunk is processed.  kXLane: flush reads what other lanes' visits
// wrote (warp barriers around it); list builders that only write their own
// slots skip those barriers and synchronise once after the scan.
template <int GW, bool kXLane, typename Visit, typename Flush>
__device__ __forceinline__ void rows_scan(const Frame& F, int tc, int sc, const RowTab& rt,
                                          uint32_t total, const Pos& q, double r2, Visit visit,
                                          Flush flush) {
    using G = Grp<GW>;
    const int gl = G::gl();
    const double* tt = F.t[tc];
    const int32_t* FI = F.fi[sc];
    const int32_t* FJ = F.fj[sc];
    // lane k of the group holds non-empty row k: its first rank pk and
    // rank -> index offset dk.  The row of candidate fb + l is the row
    // holding fb plus the rows starting in (fb, fb + l]: a ballot, an
    // OR-reduction of the start offsets inside the chunk and a popcount,
    // then one shuffle.
    const bool hr = (uint32_t)gl < rt.n;
    const uint32_t pk = hr ? rt.pre[gl] : 0xffffffffu;
    const uint32_t dk = hr ? rt.m0[gl] - pk : 0u;
    const uint32_t lanes_le = G::le();
    auto locate = [&](uint32_t fb) -> uint32_t {  // warp-collective: candidate fb + gl
        const int j0 = __popc(G::field(__ballot_sync(0xffffffffu, pk <= fb))) - 1;
        const uint32_t bit = (pk > fb && pk - fb < (uint32_t)GW) ? 1u << (pk - fb + G::base()) : 0u;
        const int j = j0 + __popc(G::field(__reduce_or_sync(0xffffffffu, bit)) & lanes_le);
        return fb + (uint32_t)gl + __shfl_sync(0xffffffffu, dk, j & (GW - 1), GW);
    };
    const uint32_t tmax = G::wmax(total);
    bool v = (uint32_t)gl < total;
    uint32_t mm = locate(0u);
    RT3D_CHECK(!v || mm < F.pcap);
    int cfi = v ? FI[mm] : 0, cfj = v ? FJ[mm] : 0;
    double ctt = v ? tt[mm] : 0.0;
    for (uint32_t fb = 0; fb < tmax; fb += GW) {
        const uint32_t f2 = fb + GW + (uint32_t)gl;
        const bool v2 = f2 < total;
        const uint32_t mm2 = locate(fb + GW);
        RT3D_CHECK(!v2 || mm2 < F.pcap);
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
        const uint32_t wb = __ballot_sync(0xffffffffu, ok);
        if (wb) {
            const uint32_t bal = G::field(wb);
            if (ok) visit(__popc(bal & G::lt()), mm, o, d2, cfi, cfj);
            if (kXLane) __syncwarp();
            flush(__popc(bal));
            if (kXLane) __syncwarp();
        }
        v = v2;
        mm = mm2;
        cfi = nfi;
        cfj = nfj;
        ctt = ntt;
    }
    __syncwarp();
}

// Ball of q over the window, all row batches (act false: an empty window,
// the group only takes part in the warp's collectives).
template <int GW, bool kXLane, typename Visit, typename Flush>
__device__ __forceinline__ void ball_scan(const Frame& F, int tc, int sc, RowTab& rt, int fi,
                                          int fj, const Pos& q, double r2, Visit visit,
                                          Flush flush, int Wq = -1, bool act = true) {
    // Wq < W restricts the scan to the fine window of half-width Wq (kNN)
    const int W = Wq >= 0 && Wq < F.cfg.W ? Wq : F.cfg.W;
    int ci0, ci1;
    window_rows(F, fi, W, ci0, ci1);
    if (!act) {
        ci0 = 0;
        ci1 = -1;
    }
    const uint32_t nb = ci1 >= ci0 ? (uint32_t)((ci1 - ci0) / GW + 1) : 0u;
    const uint32_t nbm = Grp<GW>::wmax(nb);
    for (uint32_t b = 0; b < nbm; ++b) {
        const int rb = ci0 + (int)b * GW;
        uint32_t m0, len;
        rows_load<GW>(F, sc, fi, fj, W, rb, ci1, m0, len);
        const uint32_t total = rows_finish<GW>(rt, m0, len);
        rows_scan<GW, kXLane>(F, tc, sc, rt, total, q, r2, visit, flush);
    }
}

// Ball of q over the window through the depth blocks (superres frames,
// F.zb): the window's (coarse row, coarse pixel) pairs one per lane, each
// pixel's blocks of F.zbs consecutive points whose depth interval reaches
// [q.z - R, q.z + R] become candidate ranges (adjacent kept blocks merged),
// compacted in ascending index order and scanned GW ranges at a time.  A
// block is dropped only when fl(zmin - q.z) or fl(q.z - zmax) exceeds
// R (1 + 1e-9): by monotone rounding every point in it has dz beyond that,
// so d^2 >= fl(dz^2) > R^2 (1 + 2^-53) >= fl(R R): no member is lost, and the
// members come in the same ascending index order as ball_scan's.
template <int GW, bool kXLane, typename Visit, typename Flush>
__device__ __forceinline__ void ball_scan_blocks(const Frame& F, int tc, int sc, RowTab& rt,
                                                 uint2* rng, int fi, int fj, const Pos& q,
                                                 double r2, Visit visit, Flush flush, int Wq = -1,
                                                 bool act = true) {
    using G = Grp<GW>;
    const int gl = G::gl();
    const int W = Wq >= 0 && Wq < F.cfg.W ? Wq : F.cfg.W;
    const double rw = F.cfg.R / F.pitch;
    const double lim2 = rw * rw * (1.0 + 1e-9);
    const double zc = F.cfg.R * (1.0 + 1e-9);
    const uint32_t* bo = F.bo[sc];
    const uint32_t KB = F.zkb, BS = F.zbs;
    const int s = F.s;
    const uint32_t lanes_le = G::le();
    int ci0, ci1;
    window_rows(F, fi, W, ci0, ci1);
    if (!act) {
        ci0 = 0;
        ci1 = -1;
    }
    const uint32_t nrb = ci1 >= ci0 ? (uint32_t)((ci1 - ci0) / GW + 1) : 0u;
    const uint32_t nrbm = G::wmax(nrb);
    for (uint32_t rbi = 0; rbi < nrbm; ++rbi) {
        // lane r: coarse row rb + r and its disc-culled coarse columns
        // [c0, c0 + npx) (rows_load's bounds)
        const int rb = ci0 + (int)rbi * GW;
        const int ci = rb + gl;
        int c0 = 0;
        uint32_t npx = 0;
        if (ci <= ci1) {
            const int r_lo = ci * s, r_hi = r_lo + s - 1;
            const int dmin = fi < r_lo ? r_lo - fi : (fi > r_hi ? fi - r_hi : 0);
            const double rem = lim2 - (double)dmin * (double)dmin;
            if (rem >= 0.0) {
                int wj = (int)floor(sqrt(rem));
                wj = wj > W ? W : wj;
                int b0 = fj - wj, b1 = fj + wj;
                b0 = b0 < 0 ? 0 : b0;
                b1 = b1 > F.fcols - 1 ? F.fcols - 1 : b1;
                c0 = coarse_of(F, b0);
                npx = (uint32_t)(coarse_of(F, b1) - c0 + 1);
            }
        }
        uint32_t inc = npx;
#pragma unroll
        for (int o = 1; o < GW; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, inc, o, GW);
            if (gl >= o) inc += y;
        }
        const uint32_t ppre = inc - npx, P = __shfl_sync(0xffffffffu, inc, GW - 1, GW);
        // rows with pixels are a contiguous run of lanes from the first one
        const uint32_t pk = npx ? ppre : 0xffffffffu;
        const uint32_t nem = G::field(__ballot_sync(0xffffffffu, npx != 0u));
        const int fne = nem ? __ffs((int)nem) - 1 : 0;
        const uint32_t Pm = G::wmax(P);
        for (uint32_t ub = 0; ub < Pm; ub += GW) {
            // pair ub + gl: its row lane (locate's ballot / OR-reduction)
            const int j0 = __popc(G::field(__ballot_sync(0xffffffffu, pk <= ub))) - 1;
            const uint32_t bit = (pk > ub && pk - ub < (uint32_t)GW) ? 1u << (pk - ub + G::base()) : 0u;
            const int L = fne + j0 + __popc(G::field(__reduce_or_sync(0xffffffffu, bit)) & lanes_le);
            const uint32_t Lpre = __shfl_sync(0xffffffffu, ppre, L & (GW - 1), GW);
            const int Lc0 = __shfl_sync(0xffffffffu, c0, L & (GW - 1), GW);
            const uint32_t u = ub + (uint32_t)gl;
            // the pixel's kept blocks as a bit mask (empty blocks hold
            // (+inf, -inf) and are never kept), runs of kept blocks merged
            uint32_t n0 = 0, n1 = 0, keep = 0;
            if (u < P) {
                const uint32_t p = (uint32_t)(rb + L) * (uint32_t)F.cols + (uint32_t)Lc0 + (u - Lpre);
                const double2* zp = F.zb + (size_t)p * KB;
#pragma unroll
                for (uint32_t k = 0; k < 4u; ++k) {
                    if (k < KB) {
                        const double2 zz = zp[k];
                        if (!(zz.x - q.z > zc || q.z - zz.y > zc)) keep |= 1u << k;
                    }
                }
                n0 = bo[p];
                n1 = bo[p + 1];
            }
            const uint32_t starts = keep & ~(keep << 1);
            const uint32_t kc = (uint32_t)__popc(starts);
            uint32_t kinc = kc;
#pragma unroll
            for (int o = 1; o < GW; o <<= 1) {
                const uint32_t y = __shfl_up_sync(0xffffffffu, kinc, o, GW);
                if (gl >= o) kinc += y;
            }
            const uint32_t KT = __shfl_sync(0xffffffffu, kinc, GW - 1, GW);
            uint32_t wpos = kinc - kc;
            for (uint32_t st = starts; st; st &= st - 1u) {
                const int a = __ffs((int)st) - 1;
                const int e = __ffs((int)(~keep & ~((1u << a) - 1u))) - 1;  // first dropped block after a
                const uint32_t lo = n0 + (uint32_t)a * BS;
                const uint32_t hi = min(n0 + (uint32_t)e * BS, n1);
                rng[wpos++] = make_uint2(lo, hi - lo);
            }
            __syncwarp();
            const uint32_t KTm = G::wmax(KT);
            for (uint32_t gb = 0; gb < KTm; gb += GW) {
                const uint32_t g = gb + (uint32_t)gl;
                const uint2 rg = g < KT ? rng[g] : make_uint2(0u, 0u);
                const uint32_t total = rows_finish<GW>(rt, rg.x, rg.y);
                rows_scan<GW, kXLane>(F, tc, sc, rt, total, q, r2, visit, flush);
            }
            __syncwarp();
        }
    }
}

// Candidate range of window row ci = rb + lane for two points in the same
// or adjacent fine cells: the union of their disc-culled column ranges
// (contiguous: each holds its own point's column, and those differ by at most
// one); a row outside one point's disc takes the other's range.
__device__ __forceinline__ void rows_load_union(const Frame& F, int sc, int fiA, int fjA, int fiB,
                                                int fjB, int W, int rb, int ci1, uint32_t& m0,
                                                uint32_t& len) {
    const int s = F.s;
    const double rw = F.cfg.R / F.pitch;
    const double lim2 = rw * rw * (1.0 + 1e-9);
    const int ci = rb + (int)(threadIdx.x & 31);
    m0 = 0;
    len = 0;
    if (ci > ci1) return;
    int c0 = 0x7fffffff, c1 = -1;
#pragma unroll
    for (int p = 0; p < 2; ++p) {
        const int fi = p ? fiB : fiA, fj = p ? fjB : fjA;
        const int r_lo = ci * s, r_hi = r_lo + s - 1;
        const int dmin = fi < r_lo ? r_lo - fi : (fi > r_hi ? fi - r_hi : 0);
        const double rem = lim2 - (double)dmin * (double)dmin;
        if (rem >= 0.0) {  // (rows_load's bound for this point)
            int wj = (int)floor(sqrt(rem));
            wj = wj > W ? W : wj;
            int b0 = fj - wj, b1 = fj + wj;
            b0 = b0 < 0 ? 0 : b0;
            b1 = b1 > F.fcols - 1 ? F.fcols - 1 : b1;
            const int a = coarse_of(F, b0), e = coarse_of(F, b1);
            c0 = a < c0 ? a : c0;
            c1 = e > c1 ? e : c1;
        }
    }
    if (c1 >= 0) {
        const uint32_t prow = (uint32_t)ci * F.cols;
        const uint32_t* bo = F.bo[sc];
        m0 = bo[prow + c0];
        len = bo[prow + c1 + 1] - m0;
    }
}

// The warp's two points in the same or adjacent fine cells (consecutive
// points of a pixel, or of neighbouring pixels): one 32-lane scan of the
// union of their windows with two memberships per candidate, each formed
// with its own point exactly as ball_scan forms it (a candidate outside a
// point's own window lies outside its ball and fails the test), each member
// going to its point's list in ascending index order:
// put(g, slot, index, z, d^2, fine cell).
// The candidates of a 32-lane row batch (rt, total) against two points,
// each membership formed with its own point exactly as rows_scan forms it;
// members go to put(g, slot, index, z, d^2, fine cell) in ascending index
// order (slot = the point's member count before it).
template <typename Put>
__device__ __forceinline__ void rows_scan_pair(const Frame& F, int tc, int sc, const RowTab& rt,
                                               uint32_t total, const Pos& qA, const Pos& qB,
                                               double r2, Put put, unsigned int& c0,
                                               unsigned int& c1) {
    using G = Grp<32>;
    const int lane = threadIdx.x & 31;
    const double* tt = F.t[tc];
    const int32_t* FI = F.fi[sc];
    const int32_t* FJ = F.fj[sc];
    const uint32_t lt = G::lt(), le = G::le();
    const bool hr = (uint32_t)lane < rt.n;
    const uint32_t pk = hr ? rt.pre[lane] : 0xffffffffu;
    const uint32_t dk = hr ? rt.m0[lane] - pk : 0u;
    auto locate = [&](uint32_t fb) -> uint32_t {  // (rows_scan's)
        const int j0 = __popc(__ballot_sync(0xffffffffu, pk <= fb)) - 1;
        const uint32_t bit = (pk > fb && pk - fb < 32u) ? 1u << (pk - fb) : 0u;
        const int j = j0 + __popc(__reduce_or_sync(0xffffffffu, bit) & le);
        return fb + (uint32_t)lane + __shfl_sync(0xffffffffu, dk, j & 31);
    };
    bool v = (uint32_t)lane < total;
    uint32_t mm = locate(0u);
    RT3D_CHECK(!v || mm < F.pcap);
    int cfi = v ? FI[mm] : 0, cfj = v ? FJ[mm] : 0;
    double ctt = v ? tt[mm] : 0.0;
    for (uint32_t fb = 0; fb < total; fb += 32) {
        const uint32_t f2 = fb + 32 + (uint32_t)lane;
        const bool v2 = f2 < total;
        const uint32_t mm2 = locate(fb + 32);
        RT3D_CHECK(!v2 || mm2 < F.pcap);
        const int nfi = v2 ? FI[mm2] : 0, nfj = v2 ? FJ[mm2] : 0;
        const double ntt = v2 ? tt[mm2] : 0.0;
        bool ok0 = false, ok1 = false;
        double oz = 0.0, d20 = 0.0, d21 = 0.0;
        if (v) {
            const double ox = (cfi + 0.5) * F.pitch, oy = (cfj + 0.5) * F.pitch;
            oz = ctt * F.bres;
            const double dxA = ox - qA.x, dyA = oy - qA.y, dzA = oz - qA.z;
            const double dxB = ox - qB.x, dyB = oy - qB.y, dzB = oz - qB.z;
            d20 = dxA * dxA + dyA * dyA + dzA * dzA;
            d21 = dxB * dxB + dyB * dyB + dzB * dzB;
            ok0 = d20 <= r2;
            ok1 = d21 <= r2;
        }
        const uint32_t b0 = __ballot_sync(0xffffffffu, ok0), b1 = __ballot_sync(0xffffffffu, ok1);
        const uint32_t cf = ((uint32_t)cfi << 16) | (uint32_t)cfj;
        if (ok0) put(0, c0 + (unsigned int)__popc(b0 & lt), mm, oz, d20, cf);
        if (ok1) put(1, c1 + (unsigned int)__popc(b1 & lt), mm, oz, d21, cf);
        c0 += (unsigned int)__popc(b0);
        c1 += (unsigned int)__popc(b1);
        v = v2;
        mm = mm2;
        cfi = nfi;
        cfj = nfj;
        ctt = ntt;
    }
    __syncwarp();
}

template <typename Put>
__device__ __forceinline__ void ball_scan_pair(const Frame& F, int tc, int sc, RowTab& rt,
                                               int fiA, int fjA, int fiB, int fjB, const Pos& qA,
                                               const Pos& qB, double r2, int W, Put put,
                                               unsigned int& c0, unsigned int& c1) {
    int ci0, ci1, di0, di1;
    window_rows(F, fiA, W, ci0, ci1);
    window_rows(F, fiB, W, di0, di1);
    ci0 = di0 < ci0 ? di0 : ci0;
    ci1 = di1 > ci1 ? di1 : ci1;
    for (int rb = ci0; rb <= ci1; rb += 32) {
        uint32_t m0r, lenr;
        rows_load_union(F, sc, fiA, fjA, fiB, fjB, W, rb, ci1, m0r, lenr);
        const uint32_t total = rows_finish<32>(rt, m0r, lenr);
        rows_scan_pair(F, tc, sc, rt, total, qA, qB, r2, put, c0, c1);
    }
}

// ball_scan_pair through the depth blocks (superres frames, F.zb): the union
// window's (coarse row, coarse pixel) pairs one per lane, a block kept when
// its depth interval reaches either point's [z - R, z + R] (the culling test
// of ball_scan_blocks, per point), kept runs merged into ranges.
template <typename Put>
__device__ __forceinline__ void ball_scan_blocks_pair(const Frame& F, int tc, int sc, RowTab& rt,
                                                      uint2* rng, int fiA, int fjA, int fiB,
                                                      int fjB, const Pos& qA, const Pos& qB,
                                                      double r2, Put put, unsigned int& c0,
                                                      unsigned int& c1) {
    using G = Grp<32>;
    const int lane = threadIdx.x & 31;
    const int W = F.cfg.W;
    const double rw = F.cfg.R / F.pitch;
    const double lim2 = rw * rw * (1.0 + 1e-9);
    const double zc = F.cfg.R * (1.0 + 1e-9);
    const uint32_t* bo = F.bo[sc];
    const uint32_t KB = F.zkb, BS = F.zbs;
    const int s = F.s;
    const uint32_t le = G::le();
    int ci0, ci1, di0, di1;
    window_rows(F, fiA, W, ci0, ci1);
    window_rows(F, fiB, W, di0, di1);
    ci0 = di0 < ci0 ? di0 : ci0;
    ci1 = di1 > ci1 ? di1 : ci1;
    for (int rb = ci0; rb <= ci1; rb += 32) {
        // lane r: coarse row rb + r, the union of both points' disc-culled
        // coarse columns (rows_load_union's)
        const int ci = rb + lane;
        int c0c = 0;
        uint32_t npx = 0;
        if (ci <= ci1) {
            int a0 = 0x7fffffff, a1 = -1;
#pragma unroll
            for (int p = 0; p < 2; ++p) {
                const int fi = p ? fiB : fiA, fj = p ? fjB : fjA;
                const int r_lo = ci * s, r_hi = r_lo + s - 1;
                const int dmin = fi < r_lo ? r_lo - fi : (fi > r_hi ? fi - r_hi : 0);
                const double rem = lim2 - (double)dmin * (double)dmin;
                if (rem >= 0.0) {
                    int wj = (int)floor(sqrt(rem));
                    wj = wj > W ? W : wj;
                    int b0 = fj - wj, b1 = fj + wj;
                    b0 = b0 < 0 ? 0 : b0;
                    b1 = b1 > F.fcols - 1 ? F.fcols - 1 : b1;
                    const int x0 = coarse_of(F, b0), x1 = coarse_of(F, b1);
                    a0 = x0 < a0 ? x0 : a0;
                    a1 = x1 > a1 ? x1 : a1;
                }
            }
            if (a1 >= 0) {
                c0c = a0;
                npx = (uint32_t)(a1 - a0 + 1);
            }
        }
        uint32_t inc = npx;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, inc, o);
            if (lane >= o) inc += y;
        }
        const uint32_t ppre = inc - npx, P = __shfl_sync(0xffffffffu, inc, 31);
        const uint32_t pk = npx ? ppre : 0xffffffffu;
        const uint32_t nem = __ballot_sync(0xffffffffu, npx != 0u);
        const int fne = nem ? __ffs((int)nem) - 1 : 0;
        for (uint32_t ub = 0; ub < P; ub += 32) {
            const int j0 = __popc(__ballot_sync(0xffffffffu, pk <= ub)) - 1;
            const uint32_t bit = (pk > ub && pk - ub < 32u) ? 1u << (pk - ub) : 0u;
            const int L = fne + j0 + __popc(__reduce_or_sync(0xffffffffu, bit) & le);
            const uint32_t Lpre = __shfl_sync(0xffffffffu, ppre, L & 31);
            const int Lc0 = __shfl_sync(0xffffffffu, c0c, L & 31);
            const uint32_t u = ub + (uint32_t)lane;
            uint32_t n0 = 0, n1 = 0, keep = 0;
            if (u < P) {
                const uint32_t p = (uint32_t)(rb + L) * (uint32_t)F.cols + (uint32_t)Lc0 + (u - Lpre);
                const double2* zp = F.zb + (size_t)p * KB;
#pragma unroll
                for (uint32_t k = 0; k < 4u; ++k) {
                    if (k < KB) {
                        const double2 zz = zp[k];
                        const bool kA = !(zz.x - qA.z > zc || qA.z - zz.y > zc);
                        const bool kB = !(zz.x - qB.z > zc || qB.z - zz.y > zc);
                        if (kA || kB) keep |= 1u << k;
                    }
                }
                n0 = bo[p];
                n1 = bo[p + 1];
            }
            const uint32_t starts = keep & ~(keep << 1);
            const uint32_t kc = (uint32_t)__popc(starts);
            uint32_t kinc = kc;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const uint32_t y = __shfl_up_sync(0xffffffffu, kinc, o);
                if (lane >= o) kinc += y;
            }
            const uint32_t KT = __shfl_sync(0xffffffffu, kinc, 31);
            uint32_t wpos = kinc - kc;
            for (uint32_t st = starts; st; st &= st - 1u) {
                const int a = __ffs((int)st) - 1;
                const int e = __ffs((int)(~keep & ~((1u << a) - 1u))) - 1;
                const uint32_t lo = n0 + (uint32_t)a * BS;
                const uint32_t hi = min(n0 + (uint32_t)e * BS, n1);
                rng[wpos++] = make_uint2(lo, hi - lo);
            }
            __syncwarp();
            for (uint32_t gb = 0; gb < KT; gb += 32) {
                const uint32_t g = gb + (uint32_t)lane;
                const uint2 rg = g < KT ? rng[g] : make_uint2(0u, 0u);
                const uint32_t total = rows_finish<32>(rt, rg.x, rg.y);
                rows_scan_pair(F, tc, sc, rt, total, qA, qB, r2, put, c0, c1);
            }
            __syncwarp();
        }
    }
}

// p[l] = p[l] + p[l+o], o = GW/2..1, over the group's lanes; the sum lands
// in the group's lane 0 and is broadcast (oracle: lane_tree)
template <int GW>
__device__ __forceinline__ double group_halving_sum(double v) {
#pragma unroll
    for (int o = GW / 2; o > 0; o >>= 1) v = v + __shfl_down_sync(0xffffffffu, v, o, GW);
    return __shfl_sync(0xffffffffu, v, 0, GW);
}

// APSS moments over the current state, two points per warp (16 lanes each:
// the per-point work that does not scale with the ball, row tables, the
// reductions, the stores, is issued once for both), results to F.amom (kMom
// doubles per point): [0] wsum (-1: isolated), [1..3] mean, [4..18] M (lower,
// row-major; the covariance is read off M, see apss_pass_b).  Summation
// order: ball member m (ascending index) on the group's lane m mod 16, the 16
// lane partials combined by the halving tree (oracle: APSS_LANES 16).
// Points [pb, pb + P) (a band's own points; pb = 0 for a whole frame); wpb:
// warps per block taking part (the rest return).
static __device__ void apss_moment_warps(const Frame& F, ApssWarpSm* wsm, uint32_t pb, uint32_t P,
                                         int tc, int sc, uint32_t wpb) {
    using G = Grp<kApssGW>;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if ((uint32_t)warp >= wpb) return;
    const int gl = G::gl(), grp = lane >> 4;
    ApssWarpSm& A = wsm[warp];
    ApssList& L = A.u.list[grp];
    const uint32_t gw = vblock(F) * wpb + warp, nw = vgrid(F) * wpb;
    const double R = F.cfg.R, r2 = R * R, Rinv = 1.0 / R;
    const double pitch = F.pitch;
    // the warp's pairs gw + j nw, points 2 pair + group: positions preloaded
    // 16 pairs at a time (lane 2 i + g holds pair jbase + i's point g)
    int pfi = 0, pfj = 0;
    double pt = 0.0;
    uint32_t jbase = 0xffffffffu;
    for (uint32_t j = 0;; ++j) {
        const uint32_t pair = gw + j * nw;
        if (2u * pair >= P) break;  // (warp-uniform)
        if ((j & ~15u) != jbase) {
            jbase = j & ~15u;
            const uint32_t nl = 2u * (gw + (jbase + (uint32_t)(lane >> 1)) * nw) + (uint32_t)(lane & 1);
            if (nl < P) {
                pfi = F.fi[sc][pb + nl];
                pfj = F.fj[sc][pb + nl];
                pt = F.t[tc][pb + nl];
            }
        }
        const int src = (int)((j & 15u) << 1) | grp;
        const int fi = __shfl_sync(0xffffffffu, pfi, src);
        const int fj = __shfl_sync(0xffffffffu, pfj, src);
        const double tq = __shfl_sync(0xffffffffu, pt, src);
        const uint32_t nl = 2u * pair + (uint32_t)grp;
        const bool act = nl < P;
        const uint32_t n = pb + nl;
        RT3D_CHECK(!act || n < F.pcap);
        const Pos q{(fi + 0.5) * pitch, (fj + 0.5) * pitch, tq * F.bres};
        // pass A (denoise.hpp:172-186): the scan only collects the ball (member
        // rank order = ascending index) with its d^2 into the group's list;
        // the weights and the weighted sums then run densely over the list,
        // member m on the group's lane m mod 16 in increasing m
        unsigned int cnt = 0;
        auto visitA = [&](int rank, uint32_t, const Pos& o, double d2, int mfi, int mfj) {
            const unsigned int g = cnt + (unsigned int)rank;
            if (g < (unsigned int)kApssCap) {
                L.z[g] = o.z;
                L.w[g] = d2;
                L.fij[g] = ((uint32_t)mfi << 16) | (uint32_t)mfj;
            }
        };
        auto flushA = [&](int nm) { cnt += (unsigned int)nm; };
        // the two points in the same or adjacent fine cells (consecutive
        // points of a pixel or of neighbouring pixels): one shared 32-lane
        // scan of the union of their windows
        const int ofi = __shfl_xor_sync(0xffffffffu, fi, 16), ofj = __shfl_xor_sync(0xffffffffu, fj, 16);
        const bool share = __all_sync(0xffffffffu, act && abs(fi - ofi) <= 1 && abs(fj - ofj) <= 1);
        if (share) {
            const int fiA = __shfl_sync(0xffffffffu, fi, 0), fjA = __shfl_sync(0xffffffffu, fj, 0);
            const int fiB = __shfl_sync(0xffffffffu, fi, 16), fjB = __shfl_sync(0xffffffffu, fj, 16);
            const Pos qA{(fiA + 0.5) * pitch, (fjA + 0.5) * pitch, __shfl_sync(0xffffffffu, q.z, 0)};
            const Pos qB{(fiB + 0.5) * pitch, (fjB + 0.5) * pitch, __shfl_sync(0xffffffffu, q.z, 16)};
            unsigned int c0 = 0, c1 = 0;
            auto put = [&](int g, unsigned int slot, uint32_t, double oz, double d2, uint32_t cf) {
                if (slot < (unsigned int)kApssCap) {
                    A.u.list[g].z[slot] = oz;
                    A.u.list[g].w[slot] = d2;
                    A.u.list[g].fij[slot] = cf;
                }
            };
            if (F.zb)  // (rng[0..1] as one 128-range scratch)
                ball_scan_blocks_pair(F, tc, sc, A.rt[0], &A.rng[0][0], fiA, fjA, fiB, fjB, qA, qB, r2,
                                      put, c0, c1);
            else
                ball_scan_pair(F, tc, sc, A.rt[0], fiA, fjA, fiB, fjB, qA, qB, r2, F.cfg.W, put, c0, c1);
            cnt = grp ? c1 : c0;
        } else if (F.zb) {
            ball_scan_blocks<kApssGW, false>(F, tc, sc, A.rt[grp], A.rng[grp], fi, fj, q, r2, visitA,
                                             flushA, -1, act);
        } else {
            ball_scan<kApssGW, false>(F, tc, sc, A.rt[grp], fi, fj, q, r2, visitA, flushA, -1, act);
        }
        const bool over = cnt > (unsigned int)kApssCap;
        double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
        if (!over) {
            // (the scans end with a warp barrier; pass B reads back only the
            // entries this lane rewrote)
            for (unsigned int g = gl; g < cnt; g += kApssGW) {
                const double w = apss_weight_d2(R, Rinv, L.w[g]);
                const uint32_t c = L.fij[g];
                L.w[g] = w;
                a0 += w;
                a1 = __fma_rn(w, ((double)(int)(c >> 16) + 0.5) * pitch, a1);
                a2 = __fma_rn(w, ((double)(int)(c & 0xFFFFu) + 0.5) * pitch, a2);
                a3 = __fma_rn(w, L.z[g], a3);
            }
        }
        // ball larger than the list (either group): accumulate chunk by chunk
        // on a rescan, the other group idle
        const bool anyover = __any_sync(0xffffffffu, over);
        auto chunk_visit = [&](int rank, uint32_t, const Pos& o, double d2, int, int) {
            double* c = A.chunk[G::base() + rank];
            c[0] = apss_weight_d2(R, Rinv, d2);
            c[1] = o.x;
            c[2] = o.y;
            c[3] = o.z;
        };
        if (anyover) {
            unsigned int c1 = 0;
            ball_scan<kApssGW, true>(
                F, tc, sc, A.rt[grp], fi, fj, q, r2, chunk_visit,
                [&](int nm) {
                    const int r = (gl - (int)c1) & (kApssGW - 1);  // member c1 + r: lane (c1 + r) mod 16
                    if (r < nm) {
                        const double* c = A.chunk[G::base() + r];
                        const double w = c[0];
                        a0 += w;
                        a1 = __fma_rn(w, c[1], a1);
                        a2 = __fma_rn(w, c[2], a2);
                        a3 = __fma_rn(w, c[3], a3);
                    }
                    c1 += (unsigned int)nm;
                },
                -1, act && over);
        }
        const double wsum = group_halving_sum<kApssGW>(a0);
        double m0 = group_halving_sum<kApssGW>(a1), m1 = group_halving_sum<kApssGW>(a2),
               m2 = group_halving_sum<kApssGW>(a3);
        const bool isol = cnt < (unsigned int)F.cfg.min_nbrs;
        const bool skip = !act || isol || wsum <= 0.0;
        if (act && (isol || wsum <= 0.0) && gl == 0) F.amom[(size_t)n * kMom] = isol ? -1.0 : wsum;
        if (__all_sync(0xffffffffu, skip)) continue;
        {  // (the three divisions by wsum share its reciprocal)
            const double winv = 1.0 / wsum;
            m0 = div_rcp(m0, wsum, winv);
            m1 = div_rcp(m1, wsum, winv);
            m2 = div_rcp(m2, wsum, winv);
        }
        // pass B: covariance and fit moments
        double b[kRedStride];
#pragma unroll
        for (int e = 0; e < kRedStride; ++e) b[e] = 0.0;
        if (!skip && !over) {
            for (unsigned int g = gl; g < cnt; g += kApssGW) {
                const uint32_t c = L.fij[g];
                apss_pass_b(b, L.w[g], ((double)(int)(c >> 16) + 0.5) * pitch,
                            ((double)(int)(c & 0xFFFFu) + 0.5) * pitch, L.z[g], m0, m1, m2);
            }
        }
        if (anyover) {  // walk the window again
            unsigned int c2 = 0;
            ball_scan<kApssGW, true>(
                F, tc, sc, A.rt[grp], fi, fj, q, r2, chunk_visit,
                [&](int nm) {
                    const int r = (gl - (int)c2) & (kApssGW - 1);
                    if (r < nm) {
                        const double* c = A.chunk[G::base() + r];
                        apss_pass_b(b, c[0], c[1], c[2], c[3], m0, m1, m2);
                    }
                    c2 += (unsigned int)nm;
                },
                -1, act && over && !skip);
        }
        __syncwarp();  // the lists are consumed: their storage takes the partials
#pragma unroll
        for (int e = 0; e < kRedStride; ++e) A.u.red[lane][e] = b[e];
        __syncwarp();
        if (!skip) {
            if (gl < kRedStride) {
                double v[kApssGW];
#pragma unroll
                for (int l = 0; l < kApssGW; ++l) v[l] = A.u.red[G::base() + l][gl];
#pragma unroll
                for (int o = kApssGW / 2; o > 0; o >>= 1)
#pragma unroll
                    for (int l = 0; l < o; ++l) v[l] = v[l] + v[l + o];
                F.amom[(size_t)n * kMom + 4 + gl] = v[0];  // M, lower row-major
            } else {
                F.amom[(size_t)n * kMom + 0] = wsum;
                F.amom[(size_t)n * kMom + 1] = m0;
                F.amom[(size_t)n * kMom + 2] = m1;
                F.amom[(size_t)n * kMom + 3] = m2;
            }
        }
        __syncwarp();
    }
}

// sphere fit, projection and pinning, one thread per point
// (denoise.hpp:186-214, reconstruct.hpp:352-363); writes t[tc^1] and flags
static __device__ void apss_fit_threads(const Frame& F, uint32_t pb, uint32_t P, int tc, int sc) {
    (void)F.amom_stride;
    for (uint32_t nl = vblock(F) * blockDim.x + threadIdx.x; nl < P; nl += vgrid(F) * blockDim.x) {
        const uint32_t n = pb + nl;
        RT3D_CHECK(n < F.pcap);
        const int fi = F.fi[sc][n], fj = F.fj[sc][n];
        const Pos q{(fi + 0.5) * F.pitch, (fj + 0.5) * F.pitch, F.t[tc][n] * F.bres};
        uint8_t fl = F.fl[sc][n] & (uint8_t)~(1u | 4u);
        double z = q.z;
        const double* mo = F.amom + (size_t)n * kMom;
        const double wsum = mo[0];
        if (wsum < 0.0) {
            fl |= 1u;  // isolated
        } else if (wsum <= 0.0) {
            fl |= 4u;
        } else {
            double M[15], cv[6];
#pragma unroll
            for (int k = 0; k < 15; ++k) M[k] = mo[4 + k];
            cov_from_moments(M, wsum, cv);
            if (cov_degenerate(cv)) {
                fl |= 4u;
            } else {
                Sphere sp;
                Pos o;
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
}

// The fit of apss_fit_threads for latency-bound launches (a single frame):
// 64 points per 128-thread block, the first 64 threads run the covariance
// eigenvalues and finish the point, the other 64 the Pratt pencil solve with
// the two-step bisection, side by side; the same operations as
// apss_fit_threads, so the same results.
static __device__ void apss_fit_split(const Frame& F, uint32_t pb, uint32_t P, int tc, int sc) {
    __shared__ double s_sp[64][5];
    __shared__ int s_ok[64], s_deg[64];
    const int t = (int)threadIdx.x, k = t & 63;
    const bool solver = t >= 64;
    for (uint32_t b0 = vblock(F) * 64u; b0 < P; b0 += vgrid(F) * 64u) {
        const uint32_t nl = b0 + (uint32_t)k;
        const bool act = nl < P;
        const uint32_t n = pb + nl;
        RT3D_CHECK(!act || n < F.pcap);
        const double* mo = F.amom + (size_t)n * kMom;
        const double wsum = act ? mo[0] : -1.0;
        if (wsum > 0.0) {
            double M[15];
#pragma unroll
            for (int e = 0; e < 15; ++e) M[e] = mo[4 + e];
            if (solver) {
                Sphere sp;
                s_ok[k] = sphere_from_moments<true>(M, mo[1], mo[2], mo[3], sp) ? 1 : 0;
                s_sp[k][0] = sp.u0;
                s_sp[k][1] = sp.ul0;
                s_sp[k][2] = sp.ul1;
                s_sp[k][3] = sp.ul2;
                s_sp[k][4] = sp.uq;
            } else {
                double cv[6];
                cov_from_moments(M, wsum, cv);
                s_deg[k] = cov_degenerate(cv) ? 1 : 0;
            }
        }
        __syncthreads();
        if (!solver && act) {
            const int fi = F.fi[sc][n], fj = F.fj[sc][n];
            const Pos q{(fi + 0.5) * F.pitch, (fj + 0.5) * F.pitch, F.t[tc][n] * F.bres};
            uint8_t fl = F.fl[sc][n] & (uint8_t)~(1u | 4u);
            double z = q.z;
            if (wsum < 0.0) {
                fl |= 1u;  // isolated
            } else if (wsum <= 0.0 || s_deg[k]) {
                fl |= 4u;
            } else {
                const Sphere sp{s_sp[k][0], s_sp[k][1], s_sp[k][2], s_sp[k][3], s_sp[k][4]};
                Pos o;
                if (!s_ok[k] || !project_sphere(sp, F.cfg.eps, q.x, q.y, q.z, o.x, o.y, o.z))
                    fl |= 4u;
                else
                    z = o.z;
            }
            F.t[tc ^ 1][n] = std_clamp(z / F.bres, 0.0, F.tlim);
            F.fl[sc][n] = fl;
        }
        __syncthreads();
    }
}

// ascending bitonic sort of one u32 per lane across each lane group
template <int GW>
__device__ __forceinline__ uint32_t group_sort(uint32_t x) {
    const int gl = Grp<GW>::gl();
#pragma unroll
    for (int size = 2; size <= GW; size <<= 1) {
#pragma unroll
        for (int j = size >> 1; j > 0; j >>= 1) {
            const uint32_t y = __shfl_xor_sync(0xffffffffu, x, j);
            const bool up = (gl & size) == 0 || size == GW;  // this pair sorts ascending
            const bool low = (gl & j) == 0;                  // this lane keeps the smaller
            x = (low == up) ? min(x, y) : max(x, y);
        }
    }
    return x;
}

// k smallest (d^2, index) keys of the group's list in rank order
// (spatial_index.hpp:51-62) -> L.sel[0..taken), L.kth = the last key's d^2.
// Warp-collective: both groups call it, a group with act false does nothing.
// The list is in ascending index order, so the (d^2, index) order is
// (d^2, slot).
constexpr int kKnnGW = 16;       // lanes per point: two points per warp
constexpr int kKnnKeys = 6;      // keys per lane of the threshold path (lists <= 96)
__device__ __forceinline__ int knn_select(KnnList& L, unsigned int cnt, int k, bool act) {
    using G = Grp<kKnnGW>;
    const int gl = G::gl();
    const int taken = act ? ((unsigned int)k < cnt ? k : (int)cnt) : 0;
    constexpr unsigned int kThr = kKnnKeys * kKnnGW;
    static_assert(2 * kThr <= kKnnCap, "kNN threshold path: list and compacted keys");
    const int mode = !act ? -1 : (cnt <= (unsigned int)kKnnGW ? 0 : (cnt <= kThr ? 1 : 2));
    if (__any_sync(0xffffffffu, mode == 0)) {  // rank by counting, one key per lane
        if (mode == 0 && (unsigned int)gl < cnt) {
            const double my = L.d2[gl];
            int rank = 0;
            for (unsigned int e = 0; e < cnt; ++e) {
                const double d = L.d2[e];
                rank += (d < my || (d == my && e < (unsigned int)gl)) ? 1 : 0;
            }
            if (rank < taken) L.sel[rank] = L.idx[gl];
            if (rank == taken - 1) L.kth = my;
        }
    }
    if (__any_sync(0xffffffffu, mode == 1)) {
        // A threshold from the lane minima (a lane holds slots gl + 16 e) on
        // the high words of the keys' bits (d^2 >= 0, so the high word is
        // monotone in d^2): at least k keys have a high word at or below the
        // k-th smallest minimum's, so the keys above it rank >= k.  The keys
        // at or below it are compacted in slot order (typically ~k of them)
        // and ranked by counting; ranks are a permutation.
        const bool on = mode == 1;
        double a[kKnnKeys];
        uint32_t h[kKnnKeys];
        uint32_t hmin = 0xffffffffu;
#pragma unroll
        for (int e = 0; e < kKnnKeys; ++e) {
            const bool v = on && (unsigned int)(gl + kKnnGW * e) < cnt;
            a[e] = v ? L.d2[gl + kKnnGW * e] : INFINITY;
            h[e] = v ? (uint32_t)((unsigned long long)__double_as_longlong(a[e]) >> 32) : 0xffffffffu;
            hmin = min(hmin, h[e]);
        }
        const uint32_t srt = group_sort<kKnnGW>(hmin);
        const uint32_t tau =
            k <= kKnnGW ? __shfl_sync(0xffffffffu, srt, (k - 1) & (kKnnGW - 1), kKnnGW) : 0xffffffffu;
        // the compacted keys go to slots [kThr, kThr + c) of the list
        double* cd = L.d2 + kThr;
        uint32_t* ci = L.idx + kThr;
        unsigned int c = 0;
#pragma unroll
        for (int e = 0; e < kKnnKeys; ++e) {
            const bool in = on && (unsigned int)(gl + kKnnGW * e) < cnt && h[e] <= tau;
            const uint32_t bal = G::field(__ballot_sync(0xffffffffu, in));
            if (in) {
                const unsigned int p = c + (unsigned int)__popc(bal & G::lt());
                cd[p] = a[e];
                ci[p] = L.idx[gl + kKnnGW * e];
            }
            c += (unsigned int)__popc(bal);
        }
        __syncwarp();
        if (on) {
            for (unsigned int sl = (unsigned int)gl; sl < c; sl += kKnnGW) {
                const double my = cd[sl];
                int rank = 0;
                for (unsigned int e = 0; e < c; ++e) {
                    const double d = cd[e];
                    rank += (d < my || (d == my && e < sl)) ? 1 : 0;
                }
                if (rank < taken) L.sel[rank] = ci[sl];
                if (rank == taken - 1) L.kth = my;
            }
        }
    }
    if (__any_sync(0xffffffffu, mode == 2)) {  // successive minima over the list
        const bool on = mode == 2;
        double last_d = 0.0;
        uint32_t last_i = 0;
        const int kr = (int)G::wmax((uint32_t)(on ? taken : 0));
        for (int tk = 0; tk < kr; ++tk) {
            double bd = INFINITY;
            uint32_t bi = 0xffffffffu;
            if (on)
                for (unsigned int e = gl; e < cnt; e += kKnnGW) {
                    const double d = L.d2[e];
                    const uint32_t i = L.idx[e];
                    const bool after = tk == 0 || d > last_d || (d == last_d && i > last_i);
                    if (after && (d < bd || (d == bd && i < bi))) {
                        bd = d;
                        bi = i;
                    }
                }
#pragma unroll
            for (int o = kKnnGW / 2; o > 0; o >>= 1) {
                const double od = __shfl_xor_sync(0xffffffffu, bd, o);
                const uint32_t oi = __shfl_xor_sync(0xffffffffu, bi, o);
                if (od < bd || (od == bd && oi < bi)) {
                    bd = od;
                    bi = oi;
                }
            }
            if (on && tk < taken && gl == 0) {
                L.sel[tk] = bi;
                if (tk == taken - 1) L.kth = bd;
            }
            last_d = bd;
            last_i = bi;
        }
    }
    __syncwarp();
    return taken;
}

// kNN intensity filter over the current state, two points per warp (16
// lanes each); writes r[rc^1].
//
// Window pruning (exact): a member whose fine pixel lies outside the window
// of half-width w differs by >= w+1 pixels along one axis, so its d^2 is at
// least ((w+1) pitch)^2 (1 - 1e-9) (d^2 = (dx^2 + dy^2) + dz^2 only grows with
// the added squares; the margin covers the rounding of the pixel-centre
// coordinates for grids below 2^20 fine pixels).  The scan starts with the
// small window knn_w0; if the k-th key found there is below that bound for
// the next ring, no member outside can enter the top k and the selection is
// final; otherwise the window grows to the first ring whose bound exceeds
// the k-th key (at most W, the full ball).  The two groups grow their
// windows independently; the warp rescans until both are final.
// MODE 0: every point to its final window (one kernel).  MODE 1 (knn_kernel):
// every point's first window; a point that needs a wider one is appended to
// F.knn_list (its result left to MODE 2).  MODE 2 (knn_rescan_kernel): the
// listed points over the full ball W, which holds every candidate of any
// window the growth could stop at, so the selection is the same.
template <int MODE = 0>
static __device__ void knn_warps(const Frame& F, KnnWarpSm* wsm, uint32_t pb, uint32_t P, int tc,
                                 int rc, int sc, bool dyn = false) {
    using G = Grp<kKnnGW>;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int gl = G::gl(), grp = lane >> 4;
    KnnWarpSm& K = wsm[warp];
    KnnList& L = K.l[grp];
    const uint32_t wpb = blockDim.x >> 5;
    const uint32_t gw = vblock(F) * wpb + warp, nw = vgrid(F) * wpb;
    const double R = F.cfg.R, r2 = R * R;
    const double* rr = F.r[rc];
    const int k = F.cfg.knn_k, Wfull = F.cfg.W;
    const double pitch = F.pitch;
    const int w0 = F.cfg.knn_w0 < Wfull ? F.cfg.knn_w0 : Wfull;
    // the warp's pairs gw + j nw, points 2 pair + group: positions preloaded
    // 16 pairs at a time (lane 2 i + g holds pair jbase + i's point g)
    int pfi = 0, pfj = 0;
    double pt = 0.0;
    uint32_t jbase = 0xffffffffu;
    auto point = [&](uint32_t j, int& fi, int& fj, double& t) {  // (warp-collective)
        if ((j & ~15u) != jbase) {
            jbase = j & ~15u;
            const uint32_t nl = 2u * (gw + (jbase + (uint32_t)(lane >> 1)) * nw) + (uint32_t)(lane & 1);
            if (nl < P) {
                pfi = F.fi[sc][pb + nl];
                pfj = F.fj[sc][pb + nl];
                pt = F.t[tc][pb + nl];
            }
        }
        const int src = (int)((j & 15u) << 1) | grp;
        fi = __shfl_sync(0xffffffffu, pfi, src);
        fj = __shfl_sync(0xffffffffu, pfj, src);
        t = __shfl_sync(0xffffffffu, pt, src);
    };
    // dyn (the stand-alone kernel): pairs by ticket (F.ctl->knn_next), so a
    // warp that drew points needing wider windows does not hold up the
    // launch; the next ticket and its positions are fetched while the current
    // pair is filtered.  Otherwise the warp's pairs gw + j nw.
    unsigned int* const tkt = &F.ctl->knn_next;
    uint32_t pair = gw;
    int dfi = 0, dfj = 0;
    double dtq = 0.0;
    auto load_pos = [&](uint32_t pr) {
        const uint32_t nl = 2u * pr + (uint32_t)grp;
        if (nl < P) {
            dfi = F.fi[sc][pb + nl];
            dfj = F.fj[sc][pb + nl];
            dtq = F.t[tc][pb + nl];
        }
    };
    if (MODE == 2) {  // the listed points
        P = ld_cg(&F.ctl->knn_nres);
        dyn = false;
    }
    if (dyn) {
        unsigned int t0 = 0;
        if (lane == 0) t0 = atomicAdd(tkt, 1u);
        pair = __shfl_sync(0xffffffffu, t0, 0);
        load_pos(pair);
    }
    unsigned int kept = 0;
    for (uint32_t j = 0;; ++j) {
        if (!dyn) pair = gw + j * nw;
        if (2u * pair >= P) break;  // (warp-uniform)
        unsigned int nxt = 0;
        if (dyn && lane == 0) nxt = atomicAdd(tkt, 1u);
        int fi = 0, fj = 0;
        double tq = 0.0;
        const uint32_t nl = 2u * pair + (uint32_t)grp;
        const bool act = nl < P;
        uint32_t n = pb + nl;
        if (MODE == 2) {
            n = act ? F.knn_list[nl] : 0u;
            if (act) {
                fi = F.fi[sc][n];
                fj = F.fj[sc][n];
                tq = F.t[tc][n];
            }
        } else if (dyn) {
            fi = dfi;
            fj = dfj;
            tq = dtq;
        } else {
            point(j, fi, fj, tq);
        }
        RT3D_CHECK(!act || n < F.pcap);
        const Pos q{(fi + 0.5) * pitch, (fj + 0.5) * pitch, tq * F.bres};
        int w = MODE == 2 ? Wfull : w0;
        bool deferred = false;
        int taken = 0;
        unsigned int cnt = 0;
        bool done = !act, over = false;
        while (!__all_sync(0xffffffffu, done)) {
            unsigned int c = 0;
            auto visitK = [&](int rank, uint32_t mm, const Pos&, double d2, int, int) {
                const unsigned int slot = c + (unsigned int)rank;
                if (slot < (unsigned int)kKnnCap) {
                    L.d2[slot] = d2;
                    L.idx[slot] = mm;
                }
            };
            auto flushK = [&](int nm) { c += (unsigned int)nm; };
            ball_scan<kKnnGW, false>(F, tc, sc, K.rt[grp], fi, fj, q, r2, visitK, flushK, w, !done);
            const bool sel = !done && c <= (unsigned int)kKnnCap;
            if (!done) cnt = c;
            if (!done && !sel) {  // overflow: exact rescans below
                over = true;
                done = true;
            }
            const int tk = knn_select(L, cnt, k, sel);
            if (sel) {
                taken = tk;
                if (w >= Wfull) {
                    done = true;
                } else if (taken < k) {  // too few in the small window: take the full ball
                    w = Wfull;
                } else {
                    const double kth = L.kth;
                    int wn = w;
                    while (wn < Wfull) {
                        const double b = (double)(wn + 1) * pitch;
                        if (b * b * (1.0 - 1e-9) > kth) break;
                        ++wn;
                    }
                    if (wn == w) done = true;  // nothing outside the window can enter the top k
                    else w = wn;
                }
            }
            if (MODE == 1 && !done) {  // a wider window: the rescan kernel's
                deferred = true;
                done = true;
            }
        }
        if (MODE == 1 && deferred && gl == 0) F.knn_list[atomicAdd(&F.ctl->knn_nres, 1u)] = n;
        if (dyn) {  // the next pair's positions load during the selection's tail
            const uint32_t np = __shfl_sync(0xffffffffu, nxt, 0);
            load_pos(np);
        }
        double result = 0.0;
        if (__any_sync(0xffffffffu, over)) {
            // list overflow (full window): successive minima over rescans
            double last_d = 0.0, acc = 0.0;
            uint32_t last_i = 0;
            const int kr = (int)G::wmax((uint32_t)(over ? (k < (int)cnt ? k : (int)cnt) : 0));
            int tkn = 0;
            for (int tk = 0; tk < kr; ++tk) {
                const bool on = over && tk < k && (unsigned int)tk < cnt;
                double bd = INFINITY;
                uint32_t bi = 0xffffffffu;
                ball_scan<kKnnGW, true>(
                    F, tc, sc, K.rt[grp], fi, fj, q, r2,
                    [&](int, uint32_t mm, const Pos&, double d, int, int) {
                        const bool after = tk == 0 || d > last_d || (d == last_d && mm > last_i);
                        if (after && (d < bd || (d == bd && mm < bi))) {
                            bd = d;
                            bi = mm;
                        }
                    },
                    [&](int) {}, w, on);
#pragma unroll
                for (int o = kKnnGW / 2; o > 0; o >>= 1) {
                    const double od = __shfl_xor_sync(0xffffffffu, bd, o);
                    const uint32_t oi = __shfl_xor_sync(0xffffffffu, bi, o);
                    if (od < bd || (od == bd && oi < bi)) {
                        bd = od;
                        bi = oi;
                    }
                }
                if (on) {
                    acc += rr[bi];
                    ++tkn;
                }
                last_d = bd;
                last_i = bi;
            }
            if (over) result = cnt == 0 ? rr[n] : acc / (double)tkn;
        }
        // mean over the selection in rank order (denoise.hpp:233-234): the
        // loads in parallel, the sum in rank order
        {
            double acc = 0.0;
            const int tm = (int)G::wmax((uint32_t)(over || deferred ? 0 : taken));
            for (int t0 = 0; t0 < tm; t0 += kKnnGW) {
                const double v = !over && !deferred && t0 + gl < taken ? rr[L.sel[t0 + gl]] : 0.0;
                const int nb = tm - t0 < kKnnGW ? tm - t0 : kKnnGW;  // (warp-uniform)
                for (int t = 0; t < nb; ++t) {
                    const double x = __shfl_sync(0xffffffffu, v, t, kKnnGW);
                    if (t0 + t < taken) acc += x;
                }
            }
            if (act && !over) result = taken == 0 ? rr[n] : acc / (double)taken;
        }
        if (act && !deferred && gl == 0) {
            F.r[rc ^ 1][n] = result;
            kept += (result >= F.cfg.r_min) ? 1u : 0u;  // prune's test (denoise.hpp:246)
        }
        __syncwarp();
        if (dyn) pair = __shfl_sync(0xffffffffu, nxt, 0);
    }
    // survivors of the coming prune, one integer atomic per group (exact, any order)
    if (gl == 0 && kept) atomicAdd(&F.ctl->keep, kept);
}

constexpr uint32_t kApssStageWarps = (uint32_t)(kNbrBlockBytes / sizeof(ApssWarpSm));
static_assert(kApssStageWarps >= 2, "APSS warp scratch exceeds the stage union");
static_assert(kWarps * sizeof(KnnWarpSm) <= (size_t)kNbrBlockBytes, "kNN warp scratch exceeds the stage union");

}  // namespace rt3d
