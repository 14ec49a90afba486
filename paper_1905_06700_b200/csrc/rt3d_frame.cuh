// rt3d_frame.cuh — device phases of one RT3D frame and the persistent
// cooperative kernel that runs them (init + PALM iterations) with grid-wide
// barriers instead of host round trips.
//
// Data layout in HBM (all SoA, points in cloud order = pixel-major, so the
// SceneState buckets of likelihood.hpp:38-55 are contiguous ranges bo[p] ..
// bo[p+1] and bucket_points is the identity):
//   cube      off[npix+1] u32, ev[E] {bin,count} u32x2          (read-only)
//   points    t[2][P] f64, r[2][P] f64, pix/fi/fj[2][P] i32, fl[2][P] u8
//   buckets   bo[2][npix+1] u32
//   pixels    b[2][npix] f64, gb/cb[npix] f64
// Double buffers hold (current, candidate) for the backtracking line search
// and (in, out) for the Jacobi-style denoisers and the prune compaction.
#pragma once

#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>

#include "rt3d_math.cuh"

namespace rt3d {

namespace cg = cooperative_groups;

constexpr int kBlock = 256;
constexpr int kWarps = kBlock / 32;
constexpr int kLamCap = 16;        // per-lane rate slots kept in shared memory
constexpr int kMaxReturns = 16;    // InitParams::max_returns supported on device
constexpr int kKnnFast = 32;       // knn_k handled with an in-register top-k list
constexpr int kIrfSmem = 256;      // shared IRF samples kept in shared memory

enum Program : int {
    PROG_RECON = 0,   // reconstruct (reconstruct.hpp:457-489)
    PROG_INIT = 1,    // init_matched_filter (reconstruct.hpp:197-249)
    PROG_PALM = 2,    // one palm_step on the resident state (reconstruct.hpp:300-435)
    PROG_NLL = 3,     // nll (likelihood.hpp:136-168)
    PROG_GRADS = 4,   // grad_depth/intensity/background + block_curvatures
    PROG_BASELINE = 5,// baseline_xcorr (eval.hpp:91-126)
    PROG_PEAKS = 6,   // matched_filter_peaks on every pixel, no spawn
};

enum Kind : int {
    K_NLL = 0,
    K_CAND_T = 1,
    K_CAND_R = 2,
    K_CAND_B = 3,
    K_GRAD_T = 4,
    K_GRAD_R = 5,
    K_GRAD_B = 6,
};

enum Op : int {
    OP_RESULT = 0,
    OP_GRAD_T_FIRST = 1,
    OP_GRAD_T_END = 2,
    OP_GRAD_R = 3,
    OP_GRAD_B_PRUNED = 4,
    OP_GRAD_B_EMPTY = 5,
    OP_CAND_T = 6,
    OP_CAND_R = 7,
    OP_CAND_B = 8,
};

// phase ids of the optional in-kernel timer (Frame::prof)
enum Phase : int {
    PH_INIT_PEAKS = 1, PH_SCAN = 2, PH_SPAWN = 3, PH_GRAD_T = 4, PH_CAND_T = 5, PH_APSS = 6,
    PH_GRAD_R = 7, PH_CAND_R = 8, PH_KNN = 9, PH_PRUNE_A = 10, PH_PRUNE_B = 11, PH_GRAD_B = 12,
    PH_CAND_B = 13, PH_FFT = 14, PH_LAUNCH = 15, PH_APSS_FIT = 16,
};

struct BlockDiagDev {
    double step_used, nll_after_grad, nll_after_denoise;
    int32_t backtracks, pad_;
};
struct StepDiagDev {  // layout of rt3d_step_diag
    double nll_before, nll_after;
    unsigned long long points_before, points_after;
    BlockDiagDev blk[3];
};

struct Ctl {
    unsigned int ticket;   // last-block election
    unsigned int P;        // current point count
    int iterations;
    int stop;
    int done, accept, bt, pad0_;
    double nll_cur, prev, init_nll, result, alpha, cmax;
    unsigned long long t_start, t_init, t_end;  // %globaltimer stamps (ns)
    unsigned int nprof, prof_cap;
    int tc, rc, bc, sc;    // current buffer of t, r, b and the point structure
    double red_total, red_max;  // barrier-tree fallback: the last block's results
    // grid barrier (gbar) and its watchdog: a barrier that waits longer than
    // kBarrierTimeoutNs aborts the frame instead of hanging the device
    unsigned int bar_count, bar_gen, abort, abort_block;
    unsigned int keep, pad1_;  // points the kNN filter left at r >= r_min (prune skip test)
    unsigned int pown, pbase;  // this frame's (band's) own points [pbase, pbase + pown)
    int abort_op, abort_it;
    unsigned int abort_count, abort_nsweep;
    // blocktree sweeps: block nodes handed out by ticket (by sweep parity);
    // the last block to leave a sweep resets them
    unsigned int wq_ticket[2], wq_done[2];
    unsigned int knn_next;  // kNN: the next pair of points by ticket (reset by every stage kernel)
    unsigned int knn_nres;  // kNN: points deferred to the rescan kernel (reset likewise)
};
constexpr unsigned long long kBarrierTimeoutNs = 2000000000ull;
#ifndef RT3D_BARRIER_SLEEP_NS
#define RT3D_BARRIER_SLEEP_NS 32
#endif
constexpr unsigned int kBarrierSleepNs = RT3D_BARRIER_SLEEP_NS;

struct Cfg {
    int program;
    int max_iters;
    double stop_tol;
    int step_auto[3];
    double step[3];
    double beta;
    double R;          // apss kernel radius (= SpatialIndex cell)
    double eps;        // sphere degeneracy eps
    int min_nbrs;
    int knn_k;
    double r_min;
    int bg_mode;
    double cutoff;
    int K, sep;
    double thr;
    int W;             // fine-pixel window half-width floor(R/pitch)+1
    int knn_w0;        // first kNN window half-width (see knn_warps)
    int set_oog_flags; // palm: OR out-of-gate into flags
    int blocktree;     // sweeps: block-node aligned phase 1 + replicated top tree
    int two_cand;      // depth / intensity candidate sweeps evaluate alpha and alpha * beta
    int fuse_depth;    // depth block at the end of ST_FIRST / ST_TAIL (no ST_DEPTH launch)
    int fused_iter;    // one ST_ITER launch per iteration (APSS, fit, kNN as grid phases)
    int gsz;           // lanes per pixel in the likelihood sweeps (1, 3, 4 or 32)
};

struct Frame {
    // sensor (sensor.hpp:131-170)
    int rows, cols, bins, s;
    int frows, fcols;
    uint32_t smag;  // ceil(2^32 / s) (s > 1): a / s == umulhi(a, smag) for 0 <= a < 2^20
    double pitch, bres, tlim;
    const IrfDev* irfs;
    const uint32_t* irf_of_pix;  // nullptr: irfs[0] for every pixel
    const double* gain;
    const uint8_t* dead;
    // cube
    uint32_t npix;
    uint64_t nev;      // events (E)
    const uint32_t* off;
    const uint2* ev;
    // pairwise tree geometry over pixels
    int G, Gb, wpb;
    uint32_t nbn;
    // state
    double* t[2];
    double* r[2];
    double* b[2];
    uint32_t* pix[2];
    int32_t* fi[2];
    int32_t* fj[2];
    uint8_t* fl[2];
    uint32_t* bo[2];
    int tc0, rc0, bc0, sc0;  // initial buffer toggles
    uint32_t P0;             // initial point count (resident state)
    uint32_t prof_cap;
    uint32_t pcap;           // point capacity of the state buffers (bounds checks)
    // scratch
    double* mig[2];   // per point mass_in_gate(t) of the current t (see SweepCtx)
    double* gt;
    double* ct;
    double* gr;
    double* cr;
    double* gb;
    double* cb;
    uint8_t* oog;
    double* lam;      // 4*E per-event slots (rate + 3 terms) for pixels above
                      // the lane group's shared-memory capacity
    double* part;     // npix per-pixel nll partials (sweep -> tree reduction)
    double* blk;      // nbn block-node sums
    double* bmax;     // gridDim block maxima
    // blocktree sweeps: block nodes at depth tb_G, sums / maxima by sweep parity
    int tb_G;
    uint32_t tb_nbn;
    double* tblk[2];
    double* tbmax[2];
    double* tblk2[2];  // second-candidate block-node sums
    uint32_t* cnt;    // npix prefix scratch
    uint32_t* btot;   // gridDim block totals
    double* pk_t;
    double* pk_resp;
    double* pk_mass;
    double* pk_int;   // intensity, < 0 marks a peak with no in-gate IRF mass
    uint32_t* npk;
    uint32_t* nval;
    double* amom;     // APSS moments, kMom x amom_stride (SoA): apss_kernel -> apss_fit_kernel
    uint32_t amom_stride;
    // depth blocks (superres frames): each pixel's points in blocks of zbs
    // consecutive points (spawned surface by surface, s^2 per surface), the
    // block's depth interval [min z, max z] at zb[p * zkb + k] (zblock_kernel,
    // before each APSS launch; empty blocks (+inf, -inf)); nullptr: off
    double2* zb;
    uint32_t zkb, zbs;
    uint32_t* knn_list;  // points the kNN's first windows left to the rescan kernel
    double* fft_re;   // 2*npix complex scratch (fft background mode)
    double* fft_im;
    // launch geometry: this frame's blocks are blk0 .. blk0 + nblk - 1 of the
    // launch (a batch of frames shares one launch, FrameBatch); the grid
    // barrier counts bar_n blocks on barc's counters (led by scan slot 0)
    uint32_t blk0, nblk, bar_n, pad_launch_;
    Ctl* barc;
    // row bands (large arrays): this frame owns pixels
    // [bpix0, bpix1) and the block nodes [bbn0, bbn1) of the pairwise tree;
    // the prune / spawn scans run over all bands' blocks in band order
    // (scan block sblk0 + vblock of sblk_n); global values (point count,
    // barrier) live in barc.  One band: the whole frame.
    int nbands, band;
    uint32_t bpix0, bpix1, bbn0, bbn1, sblk0, sblk_n;
    uint32_t halo_px;  // pixels of the halo rows on each side (ceil(W / s) rows)
    // control / report
    unsigned long long* prof;  // optional (id, %globaltimer) pairs after each barrier
    volatile unsigned long long* dbg;  // mapped host memory: progress / fault records
    Ctl* ctl;
    StepDiagDev* diag;
    double* trace;
    Cfg cfg;
};

// frames of one launch (a batch shares each stage / neighbour kernel): block
// b serves frame b / bpf; kernels take the batch as a __grid_constant__
// parameter and keep a reference to their frame
constexpr int kMaxBatch = 32;
struct FrameBatch {
    uint32_t n, bpf;
    uint32_t first, pad_;  // this launch runs frames first .. first + gridDim.x / bpf - 1
    Frame f[kMaxBatch];
};

// this block's index / the block count within its frame
// coarse index a / F.s of a fine index 0 <= a < 2^20 without an integer
// division: with m = ceil(2^32 / s) = (2^32 + e) / s, 0 <= e < s,
// a m / 2^32 = a / s + a e / (s 2^32) and a e < 2^32 keeps the floor exact
__device__ __forceinline__ int coarse_of(const Frame& F, int a) {
    return F.s == 1 ? a : (int)__umulhi((uint32_t)a, F.smag);
}

__device__ __forceinline__ uint32_t vblock(const Frame& F) { return blockIdx.x - F.blk0; }
__device__ __forceinline__ uint32_t vgrid(const Frame& F) { return F.nblk; }
// the frame's global point count (all bands)
__device__ __forceinline__ uint32_t global_P(const Frame& F) { return __ldcg(&F.barc->P); }

// Likelihood sweep staging: a warp owns a tree node of <= 32 consecutive
// pixels; their events and points are contiguous CSR ranges, copied into
// shared memory with coalesced loads in batches of <= kEvc events and
// <= kPvc points, then processed by lane groups (one pixel per group).
// Staging capacities: lane groups of 4 (sparse frames, <= 4 points and ~12
// events per pixel) stage 8 pixels per batch; a warp per pixel stages up to
// 32 (176 events: two warp-per-pixel blocks still share an SM, see the
// static_assert below SmemT).  The smaller footprint lets two 256-thread
// blocks share an SM.
// (G == 1, thread per pixel, reads the CSR directly: no staging)
template <int G>
struct SweepDims {
    static constexpr int EVC = G >= 32 ? 176 : G == 1 ? 1 : 64;
    static constexpr int PVC = G >= 32 ? 128 : G == 1 ? 1 : 32;
};
template <int EVC, int PVC>
struct WarpSweepSmT {
    uint2 ev[EVC];
    double lam[EVC], tn[EVC], t1[EVC], t2[EVC];
    uint32_t mk[EVC + 1];  // warp-per-pixel sweeps: the points whose support holds each event
    double pt[PVC], pr[PVC], pmig[PVC];
    int2 plh[PVC];
    uint32_t me0[32], mm[32], mn0[32], mnp[32];
    double mb[32], mgain[32];
    uint32_t mdead[32];
    double vals[32];
};
constexpr int kTopMin = 1024;  // top-of-tree values always reducible in shared memory
constexpr int kInitCap = 256;  // matched-filter candidate lags cached per warp
// APSS / kNN scratch inside the stage kernels (ST_ITER): a block's worth, the
// kNN's 8 warps or the APSS's first kNbrBlockBytes / sizeof(ApssWarpSm) warps
constexpr int kNbrBlockBytes = 57344;
struct InitWarpSm {
    int lag[kInitCap];
    double resp[kInitCap];
    uint32_t pre[33];
    int lo[32];
};
template <int G>
struct SmemT {
    static constexpr int kEvc = SweepDims<G>::EVC;
    static constexpr int kPvc = SweepDims<G>::PVC;
    using Warp = WarpSweepSmT<kEvc, kPvc>;
    union {
        struct {
            Warp w[kWarps];
        } sw;
        double top[kTopMin];
        InitWarpSm init[kWarps];
        // APSS / kNN phases of ST_ITER (not instantiated for G == 1, whose
        // small footprint lets more blocks share an SM)
        alignas(16) unsigned char nbr[G == 1 ? 16 : kNbrBlockBytes];
    } u;
    double node[kWarps];
    double wmax[kWarps];
    unsigned int scan[kWarps + 1];
    int is_last;
    unsigned int nsweep;  // sweeps run by this kernel (blocktree buffer parity)
    unsigned int wq;      // the block's next block-node ticket
    int aborted;          // the frame was aborted by the barrier watchdog
    Ctl c;                // this block's replica of the controller state
    double bpart[kWarps * 32];  // blocktree: the block node's pixel partials
    double bpart2[kWarps * 32]; // ... for the second candidate of two-candidate sweeps
    double node2[32];
    double node2b[32];
    IrfDev irf0;
    double irf_tab[2 * kIrfSmem];
};

// two blocks per SM: 228 KB of shared memory, 1 KB reserved per block
static_assert(2 * (sizeof(SmemT<32>) + 1024) <= 233472, "warp-per-pixel stage blocks no longer pair on an SM");
static_assert(2 * (sizeof(SmemT<4>) + 1024) <= 233472, "lane-group stage blocks no longer pair on an SM");

// Bounds checks of the checked build (make checked: -DRT3D_CHECKS, the
// librt3d_checked.so the test suite runs under with RT3D_LIB): a violated
// index bound prints its site and traps, so the test fails with a CUDA error
// instead of reading or writing out of bounds.  Compiled out otherwise.
#ifdef RT3D_CHECKS
#define RT3D_CHECK(cond)                                                                     \
    do {                                                                                     \
        if (!(cond)) {                                                                       \
            printf("rt3d check failed: %s (%s:%d) block %d thread %d\n", #cond, __FILE__,     \
                   __LINE__, (int)blockIdx.x, (int)threadIdx.x);                             \
            __trap();                                                                        \
        }                                                                                    \
    } while (0)
#else
#define RT3D_CHECK(cond) \
    do {                 \
    } while (0)
#endif

__device__ __forceinline__ unsigned long long globaltimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

template <typename T>
__device__ __forceinline__ T ld_cg(const T* p) {
    return __ldcg(p);
}

// profiling stamp from the calling thread (sweep-internal sub-phases)
__device__ __forceinline__ void sub_stamp(const Frame& F, int id) {
    if (F.prof) {
        unsigned int k = F.ctl->nprof;
        if (k < F.ctl->prof_cap) {
            F.prof[2 * k] = (unsigned long long)id;
            F.prof[2 * k + 1] = globaltimer();
            F.ctl->nprof = k + 1;
        }
    }
}

// sweep sub-phase stamps (tools/sweep_profile.py), compiled in with
// -DRT3D_SWEEP_PROF only: they cost registers in the hot loops
#ifdef RT3D_SWEEP_PROF
#define SWEEP_STAMP(who, id) \
    do {                     \
        if (who) sub_stamp(F, id); \
    } while (0)
#else
#define SWEEP_STAMP(who, id) \
    do {                     \
        (void)(who);         \
    } while (0)
#endif



template <class SM>
__device__ __forceinline__ const IrfDev& pixel_irf(const Frame& F, const SM& sm, uint32_t p) {
    return F.irf_of_pix ? F.irfs[F.irf_of_pix[p]] : sm.irf0;
}

__device__ __forceinline__ uint32_t lower_bound_bin(const uint2* ev, uint32_t lo, uint32_t hi,
                                                    uint32_t key) {
    while (lo < hi) {
        uint32_t mid = lo + (hi - lo) / 2;
        if (__ldg(&ev[mid].x) < key) lo = mid + 1;
        else hi = mid;
    }
    return lo;
}

// ---------------------------------------------------------------------------
// block-wide exclusive scan of one u32 per thread
// ---------------------------------------------------------------------------
template <class SM>
__device__ __forceinline__ unsigned int block_exclusive_scan(unsigned int v, SM& sm,
                                                             unsigned int& total) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    unsigned int x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        unsigned int y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) sm.scan[warp] = x;
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned int acc = 0;
        for (int w = 0; w < kWarps; ++w) {
            unsigned int t = sm.scan[w];
            sm.scan[w] = acc;
            acc += t;
        }
        sm.scan[kWarps] = acc;
    }
    __syncthreads();
    unsigned int ex = sm.scan[warp] + x - v;
    total = sm.scan[kWarps];
    __syncthreads();
    return ex;
}

// ---------------------------------------------------------------------------
// Matched filter (reconstruct.hpp:120-189), warp per pixel
// ---------------------------------------------------------------------------
// the `response` lambda, reconstruct.hpp:129-138
__device__ __forceinline__ double mf_response(const uint2* ev, uint32_t e0, uint32_t m,
                                              const IrfDev& f, double t0) {
    uint32_t first = (uint32_t)std_max(0.0, ceil(t0 + f.tau_min));
    uint32_t k = lower_bound_bin(ev, e0, e0 + m, first);
    double c = 0.0;
    const double top = t0 + f.tau_max;
    for (; k < e0 + m; ++k) {
        uint2 e = __ldg(&ev[k]);
        if (!((double)e.x <= top)) break;
        c += (double)e.y * irf_value(f, (double)e.x - t0);
    }
    return c / f.h_max;
}

template <class SM>
__device__ void phase_init_peaks(const Frame& F, SM& sm) {
    const int lane = threadIdx.x & 31;
    const uint32_t nwarps = vgrid(F) * kWarps;
    const int K = F.cfg.K, sep = F.cfg.sep, T = F.bins;
    const double thr = F.cfg.thr;
    for (uint32_t p = F.bpix0 + vblock(F) * kWarps + (threadIdx.x >> 5); p < F.bpix1; p += nwarps) {
        const double g = F.dead[p] ? 0.0 : F.gain[p];
        const uint32_t e0 = F.off[p], e1 = F.off[p + 1], m = e1 - e0;
        if (g == 0.0 || m == 0) {
            if (lane == 0) {
                F.npk[p] = 0;
                F.nval[p] = 0;
                F.b[0][p] = kBackgroundFloor;
            }
            continue;
        }
        const IrfDev& f = pixel_irf(F, sm, p);
        int taken[kMaxReturns];
        double tresp[kMaxReturns];
        int nt = 0;
        // candidate lags (reconstruct.hpp:141-148): per event the lags whose
        // IRF support reaches it, minus the previous event's range, so the
        // ranges are disjoint and increasing; one lane per candidate computes
        // its response once, then K greedy rounds pick the best non-clashing
        // candidate (= the reference's sorted greedy scan, :154-170)
        InitWarpSm& I = sm.u.init[threadIdx.x >> 5];
        uint32_t C = 0;
        bool listed = true;
        // Per-lane top-K (sep <= 16, K <= 8): candidate g (in increasing lag
        // order) belongs to lane g mod 32, so one lane's candidates lie >= 32
        // lags apart and a taken peak excludes at most one of them (|dlag| <
        // sep <= 16).  After r rounds a lane has lost at most r candidates, so
        // its best non-clashing candidate is among its best r + 1 <= K: each
        // lane keeps its K best (response desc, lag asc) at or above the
        // threshold, every response is computed once, and the K rounds below
        // give the reference's greedy picks (reconstruct.hpp:154-170).
        const bool topk = sep <= 16 && K <= 8;
        int nl = 0;  // this lane's list length (slots I.lag / I.resp [lane * 8, + K))
        for (uint32_t eb = 0; eb < m; eb += 32) {
            const uint32_t e = eb + lane;
            int lo = 0, hi = -1;
            if (e < m) {
                const uint32_t bin = __ldg(&F.ev[e0 + e].x);
                lo = (int)ceil((double)bin - f.tau_max);
                lo = lo < 0 ? 0 : lo;
                hi = (int)floor((double)bin - f.tau_min);
                hi = hi > T - 1 ? T - 1 : hi;
                if (e > 0) {
                    const uint32_t pb = __ldg(&F.ev[e0 + e - 1].x);
                    int phi = (int)floor((double)pb - f.tau_min);
                    phi = phi > T - 1 ? T - 1 : phi;
                    if (phi + 1 > lo) lo = phi + 1;
                }
            }
            const uint32_t len = hi >= lo ? (uint32_t)(hi - lo + 1) : 0u;
            uint32_t inc = len;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const uint32_t y = __shfl_up_sync(0xffffffffu, inc, o);
                if (lane >= o) inc += y;
            }
            const uint32_t total = __shfl_sync(0xffffffffu, inc, 31);
            if (!topk && C + total > (uint32_t)kInitCap) {
                listed = false;
                break;
            }
            I.pre[lane] = inc - len;
            I.lo[lane] = lo;
            if (lane == 31) I.pre[32] = total;
            __syncwarp();
            int j = 0;
            if (topk) {
                for (uint32_t c = (uint32_t)((lane - (int)C) & 31); c < total; c += 32) {
                    while (I.pre[j + 1] <= c) ++j;
                    const int t0 = I.lo[j] + (int)(c - I.pre[j]);
                    const double rr = mf_response(F.ev, e0, m, f, (double)t0);
                    if (!(rr >= thr)) continue;
                    int pos = nl < K ? nl : K;
                    if (pos == K && !(rr > I.resp[lane * 8 + K - 1])) continue;  // not in the top K
                    if (nl < K) ++nl;
                    if (pos == K) pos = K - 1;
                    while (pos > 0 && rr > I.resp[lane * 8 + pos - 1]) {
                        I.resp[lane * 8 + pos] = I.resp[lane * 8 + pos - 1];
                        I.lag[lane * 8 + pos] = I.lag[lane * 8 + pos - 1];
                        --pos;
                    }
                    I.resp[lane * 8 + pos] = rr;
                    I.lag[lane * 8 + pos] = t0;
                }
            } else {
                for (uint32_t c = lane; c < total; c += 32) {
                    while (I.pre[j + 1] <= c) ++j;
                    const int t0 = I.lo[j] + (int)(c - I.pre[j]);
                    I.lag[C + c] = t0;
                    I.resp[C + c] = mf_response(F.ev, e0, m, f, (double)t0);
                }
            }
            C += total;
            __syncwarp();
        }
        for (int round = 0; round < K; ++round) {
            double best_r = -INFINITY;
            int best_l = 0x7fffffff;
            if (topk) {
                for (int q = 0; q < nl; ++q) {  // first non-clashing entry of the lane's list
                    const int t0 = I.lag[lane * 8 + q];
                    bool clash = false;
                    for (int u = 0; u < nt; ++u) {
                        const int dd = taken[u] - t0;
                        if ((dd < 0 ? -dd : dd) < sep) clash = true;
                    }
                    if (clash) continue;
                    best_r = I.resp[lane * 8 + q];
                    best_l = t0;
                    break;
                }
            } else if (listed) {
                for (uint32_t c = lane; c < C; c += 32) {
                    const int t0 = I.lag[c];
                    bool clash = false;
                    for (int q = 0; q < nt; ++q) {
                        int dd = taken[q] - t0;
                        if ((dd < 0 ? -dd : dd) < sep) clash = true;
                    }
                    if (clash) continue;
                    const double rr = I.resp[c];
                    if (rr >= thr && (rr > best_r || (rr == best_r && t0 < best_l))) {
                        best_r = rr;
                        best_l = t0;
                    }
                }
            } else {  // more candidates than the cache: recompute per round
                for (uint32_t e = lane; e < m; e += 32) {
                    const uint32_t bin = __ldg(&F.ev[e0 + e].x);
                    int lo = (int)ceil((double)bin - f.tau_max);
                    lo = lo < 0 ? 0 : lo;
                    int hi = (int)floor((double)bin - f.tau_min);
                    hi = hi > T - 1 ? T - 1 : hi;
                    if (e > 0) {
                        const uint32_t pb = __ldg(&F.ev[e0 + e - 1].x);
                        int phi = (int)floor((double)pb - f.tau_min);
                        phi = phi > T - 1 ? T - 1 : phi;
                        if (phi + 1 > lo) lo = phi + 1;
                    }
                    for (int t0 = lo; t0 <= hi; ++t0) {
                        bool clash = false;
                        for (int q = 0; q < nt; ++q) {
                            int dd = taken[q] - t0;
                            if ((dd < 0 ? -dd : dd) < sep) clash = true;
                        }
                        if (clash) continue;
                        double rr = mf_response(F.ev, e0, m, f, (double)t0);
                        if (rr >= thr && (rr > best_r || (rr == best_r && t0 < best_l))) {
                            best_r = rr;
                            best_l = t0;
                        }
                    }
                }
            }
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
                double orr = __shfl_xor_sync(0xffffffffu, best_r, o);
                int ol = __shfl_xor_sync(0xffffffffu, best_l, o);
                if (orr > best_r || (orr == best_r && ol < best_l)) {
                    best_r = orr;
                    best_l = ol;
                }
            }
            if (best_r == -INFINITY) break;
            taken[nt] = best_l;
            tresp[nt] = best_r;
            ++nt;
        }
        __syncwarp();
        if (lane == 0) {
            double pt[kMaxReturns], pm[kMaxReturns], pr[kMaxReturns];
            for (int q = 0; q < nt; ++q) {
                const int t0 = taken[q];
                const double c0 = tresp[q];
                double cm = t0 > 0 ? mf_response(F.ev, e0, m, f, (double)(t0 - 1)) : 0.0;
                double cp = t0 < T - 1 ? mf_response(F.ev, e0, m, f, (double)(t0 + 1)) : 0.0;
                double denom = cm - 2.0 * c0 + cp;
                double delta = fabs(denom) > 1e-12 ? 0.5 * (cm - cp) / denom : 0.0;
                double tt = t0 + std_clamp(delta, -0.5, 0.5);
                int wlo, whi;
                irf_support(f, tt, T, wlo, whi);
                double mass = 0.0;
                for (uint32_t k = e0; k < e1; ++k) {
                    uint2 e = __ldg(&F.ev[k]);
                    if (e.x >= (uint32_t)wlo && e.x <= (uint32_t)whi) mass += (double)e.y;
                }
                // stable insertion by t (std::sort on <= 16 elements)
                int pos = q;
                while (pos > 0 && tt < pt[pos - 1]) {
                    pt[pos] = pt[pos - 1];
                    pm[pos] = pm[pos - 1];
                    pr[pos] = pr[pos - 1];
                    --pos;
                }
                pt[pos] = tt;
                pm[pos] = mass;
                pr[pos] = c0;
            }
            double claimed = 0.0;
            uint32_t nv = 0;
            for (int q = 0; q < nt; ++q) {
                const double irf_mass = irf_mass_in_gate(f, pt[q], T);
                double inten = -1.0;
                if (irf_mass > 0.0) {
                    inten = pm[q] / (g * irf_mass);
                    claimed += pm[q];
                    ++nv;
                }
                const size_t slot = (size_t)p * K + q;
                F.pk_t[slot] = pt[q];
                F.pk_resp[slot] = pr[q];
                F.pk_mass[slot] = pm[q];
                F.pk_int[slot] = inten;
            }
            double total = 0.0;
            for (uint32_t k = e0; k < e1; ++k) total += (double)__ldg(&F.ev[k].y);
            double residual = std_max(0.0, total - std_min(claimed, total));
            F.b[0][p] = std_max(kBackgroundFloor, residual / (g * T));
            F.npk[p] = (uint32_t)nt;
            F.nval[p] = nv;
        }
    }
}

// ---------------------------------------------------------------------------
// chunked grid scan: stage A writes per-pixel block-local prefixes, stage B
// adds the block base (after a grid barrier)
// ---------------------------------------------------------------------------
// this block's chunk of the band's pixels [bpix0, bpix1)
__device__ __forceinline__ void chunk_range(const Frame& F, uint32_t& c0, uint32_t& c1) {
    const uint32_t n = F.bpix1 - F.bpix0;
    uint32_t chunk = (n + vgrid(F) - 1) / vgrid(F);
    c0 = vblock(F) * chunk;
    c1 = c0 + chunk;
    if (c0 > n) c0 = n;
    if (c1 > n) c1 = n;
    c0 += F.bpix0;
    c1 += F.bpix0;
}
// this block's slot in the (all-band) scan
__device__ __forceinline__ uint32_t scan_block(const Frame& F) { return F.sblk0 + vblock(F); }

template <class SM, typename CountFn>
__device__ void scan_stage_a(const Frame& F, SM& sm, CountFn count) {
    uint32_t c0, c1;
    chunk_range(F, c0, c1);
    unsigned int carry = 0;
    for (uint32_t base = c0; base < c1; base += kBlock) {
        uint32_t p = base + threadIdx.x;
        unsigned int v = p < c1 ? count(p) : 0u, tot;
        unsigned int ex = block_exclusive_scan(v, sm, tot);
        if (p < c1) F.cnt[p] = carry + ex;
        carry += tot;
    }
    if (threadIdx.x == 0) F.btot[scan_block(F)] = carry;
}

// returns this block's base (over all bands' scan blocks); the band's first
// index in *band_base, the band's end in *band_end (the band's last block),
// the total over all bands in *total_out (the scan's last block)
template <class SM>
__device__ unsigned int scan_stage_b_base(const Frame& F, SM& sm, unsigned int* total_out,
                                          unsigned int* band_base = nullptr,
                                          unsigned int* band_end = nullptr) {
    const uint32_t sb = scan_block(F);
    unsigned int part = 0, bpart = 0;
    for (uint32_t b = threadIdx.x; b < sb; b += kBlock) {
        const unsigned int v = ld_cg(&F.btot[b]);
        part += v;
        if (b < F.sblk0) bpart += v;
    }
    unsigned int tot, btot_band;
    (void)block_exclusive_scan(part, sm, tot);
    (void)block_exclusive_scan(bpart, sm, btot_band);
    const unsigned int mine = ld_cg(&F.btot[sb]);
    if (threadIdx.x == 0) {
        if (sb == F.sblk_n - 1) *total_out = tot + mine;
        if (band_base) *band_base = btot_band;
        if (band_end) *band_end = tot + mine;
    }
    return tot;
}

// block-wide sum of one u32 per thread, returned to every thread
template <class SM>
__device__ __forceinline__ unsigned int block_sum_u32(unsigned int v, SM& sm) {
    unsigned int tot;
    (void)block_exclusive_scan(v, sm, tot);
    return tot;
}

// spawn points of init_matched_filter (reconstruct.hpp:219-237, 245-247)
template <class SM>
__device__ void phase_spawn(const Frame& F, SM& sm, bool baseline) {
    unsigned int total = 0, band_base = 0, band_end = 0;
    unsigned int base = scan_stage_b_base(F, sm, &total, &band_base, &band_end);
    uint32_t c0, c1;
    chunk_range(F, c0, c1);
    const int s = F.s, K = F.cfg.K;
    for (uint32_t p = c0 + threadIdx.x; p < c1; p += kBlock) {
        uint32_t o = base + ld_cg(&F.cnt[p]);
        F.bo[0][p] = o;
        const int i = (int)(p / F.cols), j = (int)(p % F.cols);
        const uint32_t nt = F.npk[p];
        RT3D_CHECK(o + F.nval[p] * (uint32_t)(s * s) <= F.pcap && nt <= (uint32_t)K);
        for (uint32_t q = 0; q < nt; ++q) {
            const size_t slot = (size_t)p * K + q;
            const double inten = F.pk_int[slot];
            if (!(inten >= 0.0)) continue;
            if (baseline) {
                // eval.hpp:107-120: one point, first peak, coarse-centre cell
                F.t[0][o] = F.pk_t[slot];
                F.r[0][o] = inten;
                F.pix[0][o] = p;
                F.fi[0][o] = i * s + s / 2;
                F.fj[0][o] = j * s + s / 2;
                F.fl[0][o] = 0;
                ++o;
                break;
            }
            const double rr = inten / (double)(s * s);
            for (int a = 0; a < s; ++a)
                for (int c = 0; c < s; ++c) {
                    F.t[0][o] = F.pk_t[slot];
                    F.r[0][o] = rr;
                    F.pix[0][o] = p;
                    F.fi[0][o] = i * s + a;
                    F.fj[0][o] = j * s + c;
                    F.fl[0][o] = 0;
                    ++o;
                }
        }
    }
    if (vblock(F) == vgrid(F) - 1 && threadIdx.x == 0) {
        F.bo[0][F.bpix1] = band_end;
        F.ctl->pbase = band_base;
        F.ctl->pown = band_end - band_base;
    }
    if (scan_block(F) == F.sblk_n - 1 && threadIdx.x == 0) F.barc->P = total;
}

// ---------------------------------------------------------------------------
// Likelihood sweep of one pixel (likelihood.hpp:100-333, reconstruct.hpp:
// 312-347,382-389,415-421).  Returns the pixel's nll partial.
// ---------------------------------------------------------------------------
struct SweepCtx {
    double alpha;
    double alpha2;   // two-candidate sweeps: the next backtracking step alpha * beta
    int two;         // evaluate alpha2 as well (K_CAND_T / K_CAND_R, blocktree)
    double cfloor;   // 1e-3 * max(curv) + 1e-30 (reconstruct.hpp:315)
    int tc, rc, bc, sc;
    int apply_floor; // background floor of reconstruct.hpp:427 before the sweep
    int mig_cached;  // mass_in_gate(t) of the current t is in F.mig[sc]
};

// Irf::value / deriv (sensor.hpp:69-82), branch-free so that independent
// evaluations overlap: for in-range tau, 0 <= x <= n-1, so the saturating
// conversion min((uint32)x, n-2) is the reference's segment
// min((size_t)x, n-2), and converting it back gives the same x - k; out of
// range taus read a clamped segment (the conversion saturates: negative and
// NaN give 0) and are discarded by the final select.
__device__ __forceinline__ double irf_value_fast(const IrfDev& f, double tau) {
    const bool in = (tau >= f.tau_min) && (tau <= f.tau_max);
    const double x = irf_x(f, tau);
    const uint32_t k = min(__double2uint_rz(x), f.n - 2u);
    const double fr = x - (double)k;
    const double s0 = f.s[k], s1 = f.s[k + 1];
    const double v = s0 + fr * (s1 - s0);
    return in ? v : 0.0;
}
__device__ __forceinline__ double irf_deriv_fast(const IrfDev& f, double tau) {
    const bool in = (tau > f.tau_min) && (tau < f.tau_max);
    const double x = irf_x(f, tau);
    const double v = f.d[min(__double2uint_rz(x), f.n - 2u)];
    return in ? v : 0.0;
}
// sum of -deriv over the support bins (likelihood.hpp:205), evaluations
// independent, subtraction sequential
__device__ __forceinline__ double neg_deriv_sum(const IrfDev& f, double t, int lo, int hi) {
    double acc = 0.0;
    int b = lo;
    for (; b + 3 <= hi; b += 4) {
        const double v0 = irf_deriv_fast(f, (double)b - t);
        const double v1 = irf_deriv_fast(f, (double)(b + 1) - t);
        const double v2 = irf_deriv_fast(f, (double)(b + 2) - t);
        const double v3 = irf_deriv_fast(f, (double)(b + 3) - t);
        acc -= v0;
        acc -= v1;
        acc -= v2;
        acc -= v3;
    }
    for (; b <= hi; ++b) acc -= irf_deriv_fast(f, (double)b - t);
    return acc;
}
// mass_in_gate, sensor.hpp:93-98: evaluations independent, sum sequential
__device__ __forceinline__ double mig_fast(const IrfDev& f, double t, int lo, int hi) {
    double m = 0.0;
    int b = lo;
    for (; b + 3 <= hi; b += 4) {
        const double v0 = irf_value_fast(f, (double)b - t);
        const double v1 = irf_value_fast(f, (double)(b + 1) - t);
        const double v2 = irf_value_fast(f, (double)(b + 2) - t);
        const double v3 = irf_value_fast(f, (double)(b + 3) - t);
        m += v0;
        m += v1;
        m += v2;
        m += v3;
    }
    for (; b <= hi; ++b) m += irf_value_fast(f, (double)b - t);
    return m;
}

// first event index (relative) with bin >= key, over the pixel's events
__device__ __forceinline__ uint32_t first_event_ge(const uint2* ev, uint32_t e0, uint32_t m,
                                                   uint32_t key) {
    return lower_bound_bin(ev, e0, e0 + m, key) - e0;
}

// Likelihood sweep of one staged pixel by a group of G lanes
// (likelihood.hpp:100-333).  Lanes compute per-event terms in parallel; every
// sum the reference forms sequentially is accumulated by one lane in the
// reference's order.  Returns the pixel's nll partial on the group leader.
template <int KIND, int G>
__device__ __forceinline__ double sweep_staged_pixel(const Frame& F, typename SmemT<G>::Warp& W,
                                                     const SweepCtx& X, const IrfDev& f, int q,
                                                     const uint2* EV, double* LAM, double* TN,
                                                     double* T1, double* T2, uint32_t pbase,
                                                     int gl, unsigned gmask, double& cmax) {
    const uint32_t m = W.mm[q];
    const uint32_t np = W.mnp[q];
    const bool dead = W.mdead[q] != 0;
    const double gain = W.mgain[q];
    const double g = dead ? 0.0 : gain;
    const double b = W.mb[q];
    const int T = F.bins;
    const double* pt = W.pt + pbase;
    const double* pr = W.pr + pbase;
    const int2* plh = W.plh + pbase;

    // A warp per pixel (<= 32 points, events staged): the points whose IRF
    // support holds event k as a bit mask MK[k], so each event visits only
    // those points, still in cloud order.  Events are sorted by bin, so a
    // point's support [lo, hi] is the event range [lower_bound(lo),
    // lower_bound(hi + 1)); its bit is toggled at both ends and a prefix XOR
    // over the events (a contiguous run per lane, then across lanes) gives
    // the masks.
    const bool use_mask = G == 32 && np <= 32u && m <= (uint32_t)SmemT<G>::kEvc && g != 0.0;
    uint32_t* MK = W.mk;
    if (use_mask) {
        for (uint32_t k = gl; k <= m; k += G) MK[k] = 0u;
        __syncwarp(gmask);
        if ((uint32_t)gl < np) {
            const int2 lh = plh[gl];
            if (lh.x <= lh.y) {
                uint32_t a = 0, hi = m;
                while (a < hi) {
                    const uint32_t mid = (a + hi) >> 1;
                    if ((int)EV[mid].x < lh.x) a = mid + 1;
                    else hi = mid;
                }
                uint32_t c = a;
                hi = m;
                while (c < hi) {
                    const uint32_t mid = (c + hi) >> 1;
                    if ((int)EV[mid].x <= lh.y) c = mid + 1;
                    else hi = mid;
                }
                if (a < c) {
                    atomicXor(&MK[a], 1u << gl);
                    atomicXor(&MK[c], 1u << gl);
                }
            }
        }
        __syncwarp(gmask);
        const uint32_t per = (m + 31u) >> 5;
        const uint32_t c0 = min((uint32_t)gl * per, m), c1 = min(c0 + per, m);
        uint32_t x = 0;
        for (uint32_t k = c0; k < c1; ++k) x ^= MK[k];
        uint32_t inc = x;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(gmask, inc, o);
            if (gl >= o) inc ^= y;
        }
        uint32_t run = inc ^ x;  // exclusive
        for (uint32_t k = c0; k < c1; ++k) {
            run ^= MK[k];
            MK[k] = run;
        }
        __syncwarp(gmask);
    }

    // rates at the active bins (detail::active_rates, likelihood.hpp:100-121)
    bool bad = false;  // an active bin at rate <= 0 (the nll is +inf)
    for (uint32_t k = gl; k < m; k += G) {
        const uint2 e = EV[k];
        double l = 0.0;
        if (g != 0.0) {
            l = g * b;
            if (use_mask) {
                for (uint32_t mk = MK[k]; mk; mk &= mk - 1u) {
                    const int qq = __ffs((int)mk) - 1;
                    l += g * pr[qq] * irf_value_fast(f, (double)e.x - pt[qq]);
                }
            } else {
                for (uint32_t qq = 0; qq < np; ++qq) {
                    const int2 lh = plh[qq];
                    if ((int)e.x >= lh.x && (int)e.x <= lh.y)
                        l += g * pr[qq] * irf_value_fast(f, (double)e.x - pt[qq]);
                }
            }
        }
        LAM[k] = l;
        bad |= l <= 0.0;
        const double z = (double)e.y;
        TN[k] = (l > 0.0) ? z * log(l) : 0.0;
        if (KIND == K_GRAD_B) {  // zero terms where the reference skips the bin
            T1[k] = (l > 0.0) ? g * z / l : 0.0;
            T2[k] = (l > 0.0) ? g * g * z / (l * l) : 0.0;
        }
    }
    const bool any_bad = __any_sync(gmask, bad);
    __syncwarp(gmask);

    // nll partial, likelihood.hpp:141-165 (leader, reference order): +inf at
    // the first bin with rate <= 0, else the sequential subtraction, now free
    // of the per-bin branch so the shared-memory loads pipeline
    double part = 0.0;
    if (gl == 0 && !dead) {
        double mass = T * b;
        for (uint32_t qq = 0; qq < np; ++qq) mass += pr[qq] * W.pmig[pbase + qq];
        double acc = gain * mass;
        if (any_bad) {
            acc = INFINITY;
        } else {
            for (uint32_t k = 0; k < m; ++k) acc -= TN[k];
        }
        part = acc;
    }

    if (KIND == K_GRAD_T || KIND == K_GRAD_R) {  // per point (owner lanes)
        const bool skip = (np == 0) || g == 0.0;
        const uint32_t n0 = W.mn0[q];
        for (uint32_t k = gl; k < np; k += G) {
            const uint32_t n = n0 + k;
            double gval = 0.0, cv = 0.0;
            uint8_t og = 0;
            if (!skip) {
                const double t = pt[k], r = pr[k];
                const int2 lh = plh[k];
                // first staged event with bin >= lo (binary search)
                uint32_t kk = 0;
                if (lh.x <= lh.y) {
                    uint32_t hi = m;
                    while (kk < hi) {
                        const uint32_t mid = (kk + hi) >> 1;
                        if (EV[mid].x < (uint32_t)lh.x) kk = mid + 1;
                        else hi = mid;
                    }
                }
                if (KIND == K_GRAD_T) {  // grad_depth + curvature().depth
                    if (lh.x > lh.y) {
                        og = 1;
                    } else {
                        const double grr = g * r;
                        double acc = 0.0;
                        acc = neg_deriv_sum(f, t, lh.x, lh.y);
                        for (; kk < m; ++kk) {
                            const uint2 e = EV[kk];
                            if (e.x > (uint32_t)lh.y) break;
                            const double l = LAM[kk];
                            const double dv = irf_deriv_fast(f, (double)e.x - t);
                            if (l > 0.0) acc += dv * (double)e.y / l;
                            if (!(l <= 0.0)) {  // likelihood.hpp:320
                                const double zl2 = (double)e.y / (l * l);
                                const double dh = grr * dv;
                                cv += dh * dh * zl2;
                            }
                        }
                        if (r != 0.0) gval = grr * acc;
                    }
                } else {  // grad_intensity + curvature().intensity
                    double acc = W.pmig[pbase + k];
                    if (lh.x <= lh.y) {
                        for (; kk < m; ++kk) {
                            const uint2 e = EV[kk];
                            if (e.x > (uint32_t)lh.y) break;
                            const double l = LAM[kk];
                            const double hv = irf_value_fast(f, (double)e.x - t);
                            if (l > 0.0) acc -= hv * (double)e.y / l;
                            if (!(l <= 0.0)) {
                                const double zl2 = (double)e.y / (l * l);
                                const double h = g * hv;
                                cv += h * h * zl2;
                            }
                        }
                    }
                    gval = g * acc;
                }
            }
            if (KIND == K_GRAD_T) {
                F.gt[n] = gval;
                F.ct[n] = cv;
                F.oog[n] = og;
                if (og && F.cfg.set_oog_flags) F.fl[X.sc][n] |= 2u;
            } else {
                F.gr[n] = gval;
                F.cr[n] = cv;
            }
            cmax = std_max(cmax, cv);
        }
    }
    if (KIND == K_GRAD_B && gl == 0) {  // grad_background + curvature().background
        double gval = 0.0, bs = 0.0;
        if (g != 0.0) {
            double acc = g * T;
            for (uint32_t k = 0; k < m; ++k) {  // T1 = T2 = 0 where LAM <= 0: same sums
                acc -= T1[k];
                bs += T2[k];
            }
            gval = acc;
        }
        cmax = std_max(cmax, bs);
        // b and gain of pixel q are in registers: hand the results to the
        // caller (which knows the pixel id) through the same slots
        W.mb[q] = gval;
        W.mgain[q] = bs;
    }
    __syncwarp(gmask);
    return part;
}

// candidate values of the depth / intensity steps (reconstruct.hpp:324-347,
// 373-389): dir = grad, or grad / (curv + floor) for "auto" steps
__device__ __forceinline__ double cand_t_value(const Frame& F, const SweepCtx& X, uint32_t n,
                                               double t0, double alpha) {
    double dir = F.gt[n];
    if (F.cfg.step_auto[0]) dir = dir / (F.ct[n] + X.cfloor);
    return std_clamp(t0 - alpha * dir, 0.0, F.tlim);
}
__device__ __forceinline__ double cand_r_value(const Frame& F, const SweepCtx& X, uint32_t n,
                                               double r0, double alpha) {
    double dir = F.gr[n];
    if (F.cfg.step_auto[1]) dir = dir / (F.cr[n] + X.cfloor);
    return std_max(0.0, r0 - alpha * dir);
}

// One warp processes tree node pixels [lo, lo+size): meta (lane per pixel),
// then batches staged in shared memory, then lane groups per pixel.
template <int KIND, int G>
__device__ __forceinline__ void sweep_node(const Frame& F, SmemT<G>& sm, const SweepCtx& X,
                                           uint32_t lo, uint32_t size, double& cmax,
                                           double* spart = nullptr, double* spart2 = nullptr) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    typename SmemT<G>::Warp& W = sm.u.sw.w[warp];
    constexpr int kEvc = SmemT<G>::kEvc, kPvc = SmemT<G>::kPvc;
    const int gl = lane % G, grp = lane / G;
    constexpr int NG = 32 / G;
    const unsigned gmask = (G == 32) ? 0xffffffffu : (((1u << G) - 1u) << (grp * G));
    const bool w0t0 = vblock(F) == 0 && threadIdx.x == 0;
    SWEEP_STAMP(w0t0, 110);
    // ---- meta, lane per pixel
    if ((uint32_t)lane < size) {
        const uint32_t p = lo + lane;
        RT3D_CHECK(p >= F.bpix0 && p < F.bpix1);
        const uint32_t e0 = F.off[p], e1 = F.off[p + 1];
        const uint32_t* bo = F.bo[X.sc];
        const uint32_t n0 = bo[p], n1 = bo[p + 1];
        RT3D_CHECK(e0 <= e1 && e1 <= F.off[F.npix] && n0 <= n1 && n1 <= F.pcap);
        const bool dead = F.dead[p] != 0;
        double b;
        if (KIND == K_CAND_B) {
            double dir = F.gb[p];
            if (F.cfg.step_auto[2]) dir = dir / (F.cb[p] + X.cfloor);
            b = std_max(0.0, F.b[X.bc][p] - X.alpha * dir);
            F.b[X.bc ^ 1][p] = b;
        } else {
            b = F.b[X.bc][p];
            if (X.apply_floor) {
                b = (b < kBackgroundFloor) ? kBackgroundFloor : b;
                F.b[X.bc][p] = b;
            }
        }
        W.me0[lane] = e0;
        W.mm[lane] = e1 - e0;
        W.mn0[lane] = n0;
        W.mnp[lane] = n1 - n0;
        W.mb[lane] = b;
        W.mgain[lane] = F.gain[p];
        W.mdead[lane] = dead ? 1u : 0u;
    }
    __syncwarp();
    SWEEP_STAMP(w0t0, 111);
    const double* tcur = F.t[X.tc];
    const double* rcur = F.r[X.rc];
    for (uint32_t q0 = 0; q0 < size;) {
        // batch [q0, q1): events <= kEvc and points <= kPvc (at least 1 pixel)
        uint32_t q1 = q0, ne = 0, npt = 0;
        while (q1 < size) {
            const uint32_t a = W.mm[q1], c = W.mnp[q1];
            if (q1 > q0 && (ne + a > (uint32_t)kEvc || npt + c > (uint32_t)kPvc)) break;
            ne += a;
            npt += c;
            ++q1;
        }
        const bool ev_smem = ne <= (uint32_t)kEvc;
        const uint32_t E0 = W.me0[q0], N0 = W.mn0[q0];
        RT3D_CHECK(npt <= (uint32_t)kPvc && (ev_smem || q1 == q0 + 1));
        if (ev_smem)
            for (uint32_t k = lane; k < ne; k += 32) W.ev[k] = __ldg(&F.ev[E0 + k]);
        const int ncand = ((KIND == K_CAND_T || KIND == K_CAND_R) && X.two) ? 2 : 1;
        for (int cand = 0; cand < ncand; ++cand) {
        const double alpha = cand ? X.alpha2 : X.alpha;
        (void)alpha;
        // points: candidate values, support, mass_in_gate (lane per point)
        for (uint32_t k = lane; k < npt; k += 32) {
            const uint32_t n = N0 + k;
            uint32_t qk = q0;
            if (F.irf_of_pix)
                while (qk + 1 < q1 && W.mn0[qk + 1] - N0 <= k) ++qk;
            const IrfDev& f = pixel_irf(F, sm, lo + qk);
            double t = tcur[n], r = rcur[n];
            if (KIND == K_CAND_T) {
                t = cand_t_value(F, X, n, t, alpha);
                if (!X.two) F.t[X.tc ^ 1][n] = t;
            }
            if (KIND == K_CAND_R) {
                r = cand_r_value(F, X, n, r, alpha);
                if (!X.two) F.r[X.rc ^ 1][n] = r;
            }
            int plo, phi;
            irf_support(f, t, F.bins, plo, phi);
            W.pt[k] = t;
            W.pr[k] = r;
            W.plh[k] = make_int2(plo, phi);
            // mass_in_gate(t): recomputed when t is a candidate or was just
            // moved by APSS, else read back (t is unchanged since then)
            constexpr bool kCompute = KIND == K_CAND_T || KIND == K_GRAD_R || KIND == K_NLL ||
                                      KIND == K_GRAD_T;
            double mg;
            if (kCompute && !(KIND == K_GRAD_T && X.mig_cached)) {
                mg = mig_fast(f, t, plo, phi);
                if (KIND == K_GRAD_R) F.mig[X.sc][n] = mg;
            } else {
                mg = F.mig[X.sc][n];
            }
            W.pmig[k] = mg;
        }
        __syncwarp();
        SWEEP_STAMP(w0t0, 112);
        for (uint32_t qb = q0; qb < q1; qb += NG) {
            const uint32_t q = qb + grp;
            if (q < q1) {
                const uint32_t eoff = W.me0[q] - E0;
                const uint2* EV;
                double *LAM, *TN, *T1, *T2;
                if (ev_smem) {
                    EV = W.ev + eoff;
                    LAM = W.lam + eoff;
                    TN = W.tn + eoff;
                    T1 = W.t1 + eoff;
                    T2 = W.t2 + eoff;
                } else {  // a single pixel above kEvc events: global slots
                    const uint32_t e0 = W.me0[q];
                    EV = F.ev + e0;
                    LAM = F.lam + e0;
                    TN = F.lam + F.nev + e0;
                    T1 = F.lam + 2 * F.nev + e0;
                    T2 = F.lam + 3 * F.nev + e0;
                }
                const IrfDev& f = pixel_irf(F, sm, lo + q);
                const double part = sweep_staged_pixel<KIND, G>(F, W, X, f, (int)q, EV, LAM, TN,
                                                                T1, T2, W.mn0[q] - N0, gl, gmask,
                                                                cmax);
                if (gl == 0) {
                    double* sp = cand ? spart2 : spart;
                    if (sp) sp[q] = part;
                    else F.part[lo + q] = part;
                    if (KIND == K_GRAD_B) {
                        F.gb[lo + q] = W.mb[q];
                        F.cb[lo + q] = W.mgain[q];
                    }
                }
            }
        }
        __syncwarp();
        }
        __syncwarp();
        SWEEP_STAMP(w0t0, 113);
        q0 = q1;
    }
}

// ---------------------------------------------------------------------------
// Thread-per-pixel likelihood sweep (G == 1) for dense large arrays (configs
// D/E: tens of events per pixel, <= kThreadPts points per pixel).  Each
// thread runs one pixel exactly as the reference's per-pixel loop body does
// (likelihood.hpp:100-333): events read straight from the CSR in order, the
// rate of every event formed point by point in cloud order, the nll partial,
// the background gradient and each point's gradient / curvature summed
// sequentially in the reference's order, so every result is bit-identical to
// the staged lane-group sweep (sweep_node) and to the reference.  Rates are
// recomputed in the per-point loops instead of being stored: a few FP64
// operations per support event against 8 B of HBM traffic per event.
// ---------------------------------------------------------------------------
constexpr int kThreadPts = 4;

struct TpPoints {
    double t[kThreadPts], r[kThreadPts], mig[kThreadPts];
    int lo[kThreadPts], hi[kThreadPts];
};

// detail::active_rates (likelihood.hpp:111-119) at one event
__device__ __forceinline__ double tp_rate(const IrfDev& f, double g, double b, int np,
                                          const TpPoints& P, uint32_t bin) {
    if (g == 0.0) return 0.0;
    double l = g * b;
#pragma unroll
    for (int q = 0; q < kThreadPts; ++q)
        if (q < np && (int)bin >= P.lo[q] && (int)bin <= P.hi[q])
            l += g * P.r[q] * irf_value_fast(f, (double)bin - P.t[q]);
    return l;
}

template <int KIND, class SM>
__device__ __forceinline__ void sweep_node_thread(const Frame& F, SM& sm, const SweepCtx& X,
                                                  uint32_t lo, uint32_t size, double& cmax,
                                                  double* spart, double* spart2) {
    const int lane = threadIdx.x & 31;
    if ((uint32_t)lane >= size) return;
    const uint32_t p = lo + (uint32_t)lane;
    RT3D_CHECK(p >= F.bpix0 && p < F.bpix1);
    const uint32_t e0 = F.off[p], m = F.off[p + 1] - e0;
    const uint32_t* bo = F.bo[X.sc];
    const uint32_t n0 = bo[p];
    const int np = (int)(bo[p + 1] - n0);
    RT3D_CHECK(e0 + m <= F.off[F.npix] && n0 + (uint32_t)np <= F.pcap && np <= kThreadPts);
    const bool dead = F.dead[p] != 0;
    const double gain = F.gain[p];
    const double g = dead ? 0.0 : gain;
    double b;
    if (KIND == K_CAND_B) {
        double dir = F.gb[p];
        if (F.cfg.step_auto[2]) dir = dir / (F.cb[p] + X.cfloor);
        b = std_max(0.0, F.b[X.bc][p] - X.alpha * dir);
        F.b[X.bc ^ 1][p] = b;
    } else {
        b = F.b[X.bc][p];
        if (X.apply_floor) {
            b = (b < kBackgroundFloor) ? kBackgroundFloor : b;
            F.b[X.bc][p] = b;
        }
    }
    const IrfDev& f = pixel_irf(F, sm, p);
    const int T = F.bins;
    const uint2* ev = F.ev + e0;
    const int ncand = ((KIND == K_CAND_T || KIND == K_CAND_R) && X.two) ? 2 : 1;
    for (int cand = 0; cand < ncand; ++cand) {
        const double alpha = cand ? X.alpha2 : X.alpha;
        (void)alpha;
        TpPoints P;
#pragma unroll
        for (int k = 0; k < kThreadPts; ++k) {
            P.t[k] = P.r[k] = P.mig[k] = 0.0;
            P.lo[k] = 1;
            P.hi[k] = 0;
            if (k < np) {
                const uint32_t n = n0 + (uint32_t)k;
                double t = F.t[X.tc][n], r = F.r[X.rc][n];
                if (KIND == K_CAND_T) {
                    t = cand_t_value(F, X, n, t, alpha);
                    if (!X.two) F.t[X.tc ^ 1][n] = t;
                }
                if (KIND == K_CAND_R) {
                    r = cand_r_value(F, X, n, r, alpha);
                    if (!X.two) F.r[X.rc ^ 1][n] = r;
                }
                int a, c;
                irf_support(f, t, T, a, c);
                constexpr bool kCompute = KIND == K_CAND_T || KIND == K_GRAD_R || KIND == K_NLL ||
                                          KIND == K_GRAD_T;
                double mg;
                if (kCompute && !(KIND == K_GRAD_T && X.mig_cached)) {
                    mg = mig_fast(f, t, a, c);
                    if (KIND == K_GRAD_R) F.mig[X.sc][n] = mg;
                } else {
                    mg = F.mig[X.sc][n];
                }
                P.t[k] = t;
                P.r[k] = r;
                P.lo[k] = a;
                P.hi[k] = c;
                P.mig[k] = mg;
            }
        }
        // events in order: rates, the nll partial (likelihood.hpp:141-165)
        // and the background gradient / curvature (:256-277, :300-307)
        double acc = 0.0, gbv = g * T, bs = 0.0;
        bool inf = false;
        if (!dead) {
            double mass = T * b;
            for (int q = 0; q < np && q < kThreadPts; ++q) mass += P.r[q] * P.mig[q];
            acc = gain * mass;
        }
        // the pixel's events in groups of 4, the next group's loads issued
        // before this group's arithmetic (each thread walks its own pixel, so
        // the loads would otherwise wait one by one)
        uint2 nxt[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) nxt[j] = (uint32_t)j < m ? __ldg(&ev[j]) : make_uint2(0u, 0u);
        for (uint32_t k0 = 0; k0 < m; k0 += 4) {
            uint2 cur[4];
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                cur[j] = nxt[j];
                nxt[j] = k0 + 4 + j < m ? __ldg(&ev[k0 + 4 + j]) : make_uint2(0u, 0u);
            }
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                if (k0 + j >= m) break;
                const uint2 e = cur[j];
                const double l = tp_rate(f, g, b, np, P, e.x);
                const double z = (double)e.y;
                if (!dead && !inf) {
                    if (l <= 0.0) inf = true;
                    else acc -= (l > 0.0) ? z * log(l) : 0.0;
                }
                if (KIND == K_GRAD_B && l > 0.0) {
                    gbv -= g * z / l;
                    bs += g * g * z / (l * l);
                }
            }
        }
        const double part = dead ? 0.0 : (inf ? INFINITY : acc);
        double* sp = cand ? spart2 : spart;
        if (sp) sp[lane] = part;
        else F.part[p] = part;
        if (KIND == K_GRAD_B) {
            const double gval = g != 0.0 ? gbv : 0.0;
            const double bsv = g != 0.0 ? bs : 0.0;
            F.gb[p] = gval;
            F.cb[p] = bsv;
            cmax = std_max(cmax, bsv);
        }
        if (KIND == K_GRAD_T || KIND == K_GRAD_R) {  // per point (likelihood.hpp:178-253)
            const bool skip = (np == 0) || g == 0.0;
            for (int k = 0; k < np && k < kThreadPts; ++k) {
                const uint32_t n = n0 + (uint32_t)k;
                double gval = 0.0, cv = 0.0;
                uint8_t og = 0;
                if (!skip) {
                    double t = 0.0, r = 0.0, mgk = 0.0;
                    int plo = 1, phi = 0;
#pragma unroll
                    for (int q = 0; q < kThreadPts; ++q)
                        if (q == k) {
                            t = P.t[q];
                            r = P.r[q];
                            mgk = P.mig[q];
                            plo = P.lo[q];
                            phi = P.hi[q];
                        }
                    uint32_t kk = m;
                    if (plo <= phi) kk = first_event_ge(F.ev, e0, m, (uint32_t)plo);
                    if (KIND == K_GRAD_T) {
                        if (plo > phi) {
                            og = 1;
                        } else {
                            const double grr = g * r;
                            double a = neg_deriv_sum(f, t, plo, phi);
                            for (; kk < m; ++kk) {
                                const uint2 e = __ldg(&ev[kk]);
                                if (e.x > (uint32_t)phi) break;
                                const double l = tp_rate(f, g, b, np, P, e.x);
                                const double dv = irf_deriv_fast(f, (double)e.x - t);
                                if (l > 0.0) a += dv * (double)e.y / l;
                                if (!(l <= 0.0)) {
                                    const double zl2 = (double)e.y / (l * l);
                                    const double dh = grr * dv;
                                    cv += dh * dh * zl2;
                                }
                            }
                            if (r != 0.0) gval = grr * a;
                        }
                    } else {
                        double a = mgk;
                        if (plo <= phi) {
                            for (; kk < m; ++kk) {
                                const uint2 e = __ldg(&ev[kk]);
                                if (e.x > (uint32_t)phi) break;
                                const double l = tp_rate(f, g, b, np, P, e.x);
                                const double hv = irf_value_fast(f, (double)e.x - t);
                                if (l > 0.0) a -= hv * (double)e.y / l;
                                if (!(l <= 0.0)) {
                                    const double zl2 = (double)e.y / (l * l);
                                    const double h = g * hv;
                                    cv += h * h * zl2;
                                }
                            }
                        }
                        gval = g * a;
                    }
                }
                if (KIND == K_GRAD_T) {
                    F.gt[n] = gval;
                    F.ct[n] = cv;
                    F.oog[n] = og;
                    if (og && F.cfg.set_oog_flags) F.fl[X.sc][n] |= 2u;
                } else {
                    F.gr[n] = gval;
                    F.cr[n] = cv;
                }
                cmax = std_max(cmax, cv);
            }
        }
    }
}

// ---------------------------------------------------------------------------
// Controller: runs on thread 0 of the last block after each grid reduction
// ---------------------------------------------------------------------------
// The controller state is replicated: every block runs the same decisions on
// the same reduced values (its own Ctl copy in shared memory); only block 0
// (`writer`) records the diagnostics and trace, and writes the state back to
// F.ctl at the end of the kernel.
static __device__ void set_block(const Frame& F, Ctl* c, bool writer, int blk, double cmax, int it) {
    c->cmax = cmax;
    c->alpha = F.cfg.step_auto[blk] ? 1.0 : F.cfg.step[blk];
    c->bt = 0;
    c->accept = 0;
    c->done = 0;
    if (c->alpha <= 0.0) {  // safeguarded_step's empty-step exit (reconstruct.hpp:278-281)
        c->alpha = 0.0;
        c->done = 1;
        if (it >= 0 && writer) {
            BlockDiagDev& d = F.diag[it].blk[blk];
            d.step_used = 0.0;
            d.backtracks = 0;
            d.nll_after_grad = c->nll_cur;
        }
    }
}

static __device__ void controller(const Frame& F, Ctl* c, bool writer, int op, int it, double v,
                           double cmax) {
    switch (op) {
        case OP_RESULT:
            c->result = v;
            c->cmax = cmax;
            break;
        case OP_GRAD_T_FIRST:
            c->nll_cur = v;
            c->init_nll = v;
            c->prev = v;
            if (writer) F.trace[0] = v;
            set_block(F, c, writer, 0, cmax, 0);
            break;
        case OP_GRAD_T_END: {
            if (writer) {
                StepDiagDev& d = F.diag[it];
                d.blk[2].nll_after_denoise = v;
                d.nll_after = v;
                d.points_after = global_P(F);
                F.trace[it + 1] = v;
            }
            c->iterations = it + 1;
            // stop rule, reconstruct.hpp:475-477
            double rel = fabs(c->prev - v) / std_max(1.0, fabs(c->prev));
            c->prev = v;
            c->stop = rel < F.cfg.stop_tol;
            c->nll_cur = v;
            set_block(F, c, writer, 0, cmax, it + 1 < F.cfg.max_iters ? it + 1 : -1);
            break;
        }
        case OP_GRAD_R:
            if (writer) F.diag[it].blk[0].nll_after_denoise = v;
            c->nll_cur = v;
            set_block(F, c, writer, 1, cmax, it);
            break;
        case OP_GRAD_B_PRUNED:
            if (writer) F.diag[it].blk[1].nll_after_denoise = v;
            c->nll_cur = v;
            set_block(F, c, writer, 2, cmax, it);
            break;
        case OP_GRAD_B_EMPTY:
            set_block(F, c, writer, 2, cmax, it);
            break;
        case OP_CAND_T:
        case OP_CAND_R:
        case OP_CAND_B: {
            const int blk = op - OP_CAND_T;
            // safeguarded_step, reconstruct.hpp:282-291
            if (v <= c->nll_cur) {
                c->nll_cur = v;
                c->accept = 1;
                c->done = 1;
            } else {
                c->alpha *= F.cfg.beta;
                c->bt += 1;
                if (c->bt >= kMaxBacktracks) {
                    c->alpha = 0.0;
                    c->accept = 0;
                    c->done = 1;
                }
            }
            if (c->done && writer) {
                BlockDiagDev& d = F.diag[it].blk[blk];
                d.step_used = c->alpha;
                d.backtracks = c->bt;
                d.nll_after_grad = c->nll_cur;
            }
            break;
        }
    }
}

__device__ __forceinline__ unsigned int ld_volatile(const unsigned int* p) {
    return *reinterpret_cast<const volatile unsigned int*>(p);
}

// Grid barrier of the cooperative stage kernels (all blocks co-resident):
// arrival counter + generation, with a watchdog.  Returns true when the frame
// has been aborted (a barrier waited longer than kBarrierTimeoutNs); every
// later barrier then returns immediately so that all blocks run out.
template <class SM>
__device__ bool gbar(const Frame& F, SM& sm, int op = -1, int it = -1) {
    __syncthreads();
    if (threadIdx.x == 0 && !sm.aborted) {
        // one word: block 0 adds 2^31 - (n - 1), the others 1, so the top bit
        // flips exactly when the last block arrives and the low bits return
        // to where they were
        // (row bands may sit on several GPUs: system-scope fences and atomics
        // on band 0's counters, reached through peer memory)
        Ctl* c = F.barc;
        const bool sys = F.nbands > 1;
        const unsigned int inc = scan_block(F) == 0 ? 0x80000000u - (F.bar_n - 1u) : 1u;
        if (sys) __threadfence_system();
        else __threadfence();
        const unsigned int old = sys ? atomicAdd_system(&c->bar_count, inc) : atomicAdd(&c->bar_count, inc);
        const unsigned long long t0 = globaltimer();
        unsigned int spins = 0;
        while (((ld_volatile(&c->bar_count) ^ old) & 0x80000000u) == 0u) {
            // back off once the wait is long: the poll loop's issue slots
            // belong to the other warps on the SM (and to concurrent frames)
            if (spins > 32u) __nanosleep(kBarrierSleepNs);
            if (((++spins) & 255u) == 0u) {
                if (ld_volatile(&c->abort)) {
                    sm.aborted = 1;
                    break;
                }
                if (globaltimer() - t0 > kBarrierTimeoutNs) {
                    if ((sys ? atomicExch_system(&c->abort, 1u) : atomicExch(&c->abort, 1u)) == 0u) {
                        c->abort_block = blockIdx.x;
                        if (F.ctl != c) atomicExch(&F.ctl->abort, 1u);
                        c->abort_op = op;
                        c->abort_it = it;
                        c->abort_count = ld_volatile(&c->bar_count);
                        c->abort_nsweep = sm.nsweep;
                    }
                    sm.aborted = 1;
                    break;
                }
            }
        }
        if (sys) __threadfence_system();
        else __threadfence();
    }
    __syncthreads();
    return sm.aborted != 0;
}

// In-place perfect-tree reduction over v[0..w) (pairs (2q, 2q+1) at every
// level) by the whole block: every level is read into registers before any
// thread writes, so no thread reads an element another thread of the same
// level has already overwritten.  w <= 8 * kBlock.
__device__ __forceinline__ void block_tree_levels(double* v, uint32_t w) {
    while (w > 1) {
        const uint32_t h = w / 2;
        double tmp[8];
        int k = 0;
        for (uint32_t q = threadIdx.x; q < h; q += kBlock) tmp[k++] = v[2 * q] + v[2 * q + 1];
        __syncthreads();
        k = 0;
        for (uint32_t q = threadIdx.x; q < h; q += kBlock) v[q] = tmp[k++];
        __syncthreads();
        w = h;
    }
}
__device__ __forceinline__ void block_tree_levels_g(double* v, uint32_t w) {
    while (w > 1) {
        const uint32_t h = w / 2;
        for (uint32_t q0 = 0; q0 < h; q0 += 8u * kBlock) {
            double tmp[8];
            int k = 0;
            const uint32_t qe = q0 + 8u * kBlock < h ? q0 + 8u * kBlock : h;
            for (uint32_t q = q0 + threadIdx.x; q < qe; q += kBlock)
                tmp[k++] = ld_cg(&v[2 * q]) + ld_cg(&v[2 * q + 1]);
            __syncthreads();
            k = 0;
            for (uint32_t q = q0 + threadIdx.x; q < qe; q += kBlock) v[q] = tmp[k++];
            __threadfence_block();
            __syncthreads();
        }
        w = h;
    }
}

// pairwise tree over the nbn block-node sums, in the last block
template <class SM>
__device__ double top_tree(const Frame& F, SM& sm) {
    const uint32_t nb = F.nbn;
    double* v = reinterpret_cast<double*>(&sm.u);
    if (nb <= (uint32_t)(sizeof(sm.u) / sizeof(double)) && nb <= 8u * kBlock) {
        for (uint32_t q = threadIdx.x; q < nb; q += kBlock) v[q] = ld_cg(&F.blk[q]);
        __syncthreads();
        block_tree_levels(v, nb);
        double r = v[0];
        __syncthreads();
        return r;
    }
    block_tree_levels_g(F.blk, nb);
    double r = ld_cg(&F.blk[0]);
    __syncthreads();
    return r;
}

// sum over a perfect binary tree (pairs (2q, 2q+1) at every level) of nb
// values (a power of two) and their max, in every block (all threads return
// both).  Up to kBlock values are loaded one per thread; above that each
// thread first reduces a contiguous power-of-two run with the binary-counter
// form of the same tree.
// perfect binary tree over nb values (a power of two <= 32 * kWarps), two
// arrays at once: warp w reduces values [32w, 32w + 32) with shuffles (pairs
// (2q, 2q+1) at every level), then thread 0 combines the warp sums (only
// thread 0's results are defined).
template <class SM>
__device__ void top_small(const double* vals, const double* vals2, const double* mx, uint32_t nb,
                          SM& sm, double& total, double& total2, double& gm) {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t span = nb < 32u ? nb : 32u;
    const uint32_t nw = nb / span;
    if ((uint32_t)warp < nw) {
        const uint32_t i = (uint32_t)warp * span + (uint32_t)lane;
        const bool in = (uint32_t)lane < span;
        double v = in ? ld_cg(&vals[i]) : 0.0;
        double v2 = (vals2 && in) ? ld_cg(&vals2[i]) : 0.0;
        double m = in ? ld_cg(&mx[i]) : 0.0;
        for (uint32_t o = 1; o < span; o <<= 1) {
            v = v + __shfl_down_sync(0xffffffffu, v, o);
            v2 = v2 + __shfl_down_sync(0xffffffffu, v2, o);
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) m = std_max(m, __shfl_xor_sync(0xffffffffu, m, o));
        if (lane == 0) {
            sm.node[warp] = v;
            sm.node2b[warp] = v2;
            sm.wmax[warp] = m;
        }
    }
    __syncthreads();
    // the warp sums' tree by thread 0 (the caller's controller thread); the
    // caller's closing block barrier orders the next reuse of sm.node
    if (threadIdx.x == 0) {
        double t[kWarps], t2[kWarps];
        double g = 0.0;
#pragma unroll
        for (int w = 0; w < kWarps; ++w) {
            t[w] = (uint32_t)w < nw ? sm.node[w] : 0.0;
            t2[w] = (uint32_t)w < nw ? sm.node2b[w] : 0.0;
            g = (uint32_t)w < nw ? std_max(g, sm.wmax[w]) : g;
        }
        // the perfect tree over the nw (a power of two) warp sums
#pragma unroll
        for (int w = kWarps; w > 1; w >>= 1)
            if ((uint32_t)w <= nw) {
#pragma unroll
                for (int q = 0; q < w / 2; ++q) {
                    t[q] = t[2 * q] + t[2 * q + 1];
                    t2[q] = t2[2 * q] + t2[2 * q + 1];
                }
            }
        total = t[0];
        total2 = t2[0];
        gm = g;
    }
}

// sum over a perfect binary tree (pairs (2q, 2q+1) at every level) of nb
// values (a power of two) and their max, in every block (defined in thread 0,
// which runs the controller).  Up to 32 * kWarps values: top_small; above that each thread first
// reduces a contiguous power-of-two run with the binary-counter form of the
// same tree, then the block reduces the thread sums.
template <class SM>
__device__ void top_all(const double* vals, const double* mx, uint32_t nb, SM& sm, double& total,
                        double& gm, const double* vals2 = nullptr, double* total2 = nullptr) {
    if (nb <= 32u * kWarps) {
        double t2 = 0.0;
        top_small(vals, vals2, mx, nb, sm, total, t2, gm);
        if (total2) *total2 = t2;
        return;
    }
    if (vals2) {
        double g2;
        top_all(vals2, mx, nb, sm, *total2, g2);
    }
    double* v = reinterpret_cast<double*>(&sm.u);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    double m = 0.0;
    const uint32_t per = nb / kBlock;
    double st[16];
    const uint32_t base = threadIdx.x * per;
    for (uint32_t j = 0; j < per; ++j) {
        double x = ld_cg(&vals[base + j]);
        m = std_max(m, ld_cg(&mx[base + j]));
        int l = 0;
        for (uint32_t bb = j; bb & 1u; bb >>= 1, ++l) x = st[l] + x;
        st[l] = x;
    }
    int L = 0;
    while ((1u << L) < per) ++L;
    v[threadIdx.x] = st[L];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) m = std_max(m, __shfl_xor_sync(0xffffffffu, m, o));
    if (lane == 0) sm.wmax[warp] = m;
    __syncthreads();
    block_tree_levels(v, kBlock);
    total = v[0];
    m = 0.0;
    for (int k = 0; k < kWarps; ++k) m = std_max(m, sm.wmax[k]);
    gm = m;
    __syncthreads();
}

// One likelihood sweep over all pixels in pairwise_sum's tree order
// (parallel.hpp:52-61), ending with the controller decision in every block.
//
// blocktree (default): block b owns the block nodes b, b + grid, ... at depth
// tb_G (each at most one chunk per warp); its warps sweep the node's chunks
// into shared memory, the block reduces the node (pw32 per depth-G node, then
// their perfect tree) and publishes it; one grid barrier; then every block
// reduces the block-node sums itself (top_all) and runs its replica of the
// controller, so the next sweep starts without a second barrier.  Ownership
// of pixels and points is the same in every sweep, so per-point scratch
// (gradients, candidates, mass_in_gate) is block-private between barriers.
//
// fallback: chunks over all warps, barrier, block nodes at depth Gb, last
// block reduces the top and publishes it, barrier, every block reads it.
template <int KIND, int G>
__device__ void tree_sweep_g(const Frame& F, SmemT<G>& sm, const SweepCtx& X,
                             int op, int it) {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    constexpr uint32_t NG = 32 / G;
    const bool b0t0 = vblock(F) == 0 && threadIdx.x == 0;
    SWEEP_STAMP(b0t0, 100);
    if (threadIdx.x == 0 && F.dbg)
        F.dbg[64 + vblock(F)] = ((unsigned long long)it << 40) | ((unsigned long long)op << 32) |
                                 (unsigned long long)sm.nsweep;
    double total = 0.0, gm = 0.0, total2 = 0.0;
    if (F.cfg.blocktree) {
        const uint32_t par = sm.nsweep & 1u;
        double* blk = F.tblk[par];
        double* bmx = F.tbmax[par];
        double* blk2 = F.tblk2[par];
        const bool two = (KIND == K_CAND_T || KIND == K_CAND_R) && X.two;
        // block nodes above depth G hold 2^dG depth-G nodes; at or below it
        // (small dense frames) a block node is itself a node of pairwise_sum's
        // recursion of <= 32 pixels
        const int dG = F.G > F.tb_G ? F.G - F.tb_G : 0;
        const bool sub = F.tb_G >= F.G;
        // Many block nodes per block (large frames): nodes by ticket (results
        // are keyed by node, so who computes which does not matter), uneven
        // pixels even out across blocks; the next ticket is fetched while the
        // current node is swept.  Few nodes per block: the static
        // round-robin (a ticket's latency would sit on the critical path).
        unsigned int* const wt = &F.ctl->wq_ticket[par];
        const uint32_t nn = F.bbn1 - F.bbn0;
        const bool dyn = nn >= 8u * vgrid(F);
        if (threadIdx.x == 0) sm.wq = dyn ? atomicAdd(wt, 1u) : vblock(F);
        __syncthreads();
        for (uint32_t tk = sm.wq; tk < nn; tk = sm.wq) {
            unsigned int nxt = 0;
            if (threadIdx.x == 0) nxt = dyn ? atomicAdd(wt, 1u) : tk + vgrid(F);
            const uint32_t bn = F.bbn0 + tk;
            uint32_t blo, bsz;
            tree_node_range(F.npix, F.tb_G, bn, blo, bsz);
            const uint32_t nch = (bsz + NG - 1) / NG;
            double cm = 0.0;
            for (uint32_t c = warp; c < nch; c += kWarps) {
                const uint32_t lo = blo + c * NG;
                const uint32_t size = blo + bsz - lo < NG ? blo + bsz - lo : NG;
                if constexpr (G == 1)
                    sweep_node_thread<KIND>(F, sm, X, lo, size, cm, sm.bpart + (lo - blo),
                                            two ? sm.bpart2 + (lo - blo) : nullptr);
                else
                    sweep_node<KIND, G>(F, sm, X, lo, size, cm, sm.bpart + (lo - blo),
                                        two ? sm.bpart2 + (lo - blo) : nullptr);
            }
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) cm = std_max(cm, __shfl_xor_sync(0xffffffffu, cm, o));
            if (lane == 0) sm.wmax[warp] = cm;
            __syncthreads();
            if (threadIdx.x < (1u << dG)) {
                uint32_t lo = blo, size = bsz;
                if (!sub) tree_node_range(F.npix, F.G, (bn << dG) | threadIdx.x, lo, size);
                sm.node2[threadIdx.x] = pw32(sm.bpart, (int)(lo - blo), (int)size);
            } else if (two && threadIdx.x >= 32 && threadIdx.x - 32 < (1u << dG)) {
                uint32_t lo = blo, size = bsz;
                if (!sub) tree_node_range(F.npix, F.G, (bn << dG) | (threadIdx.x - 32), lo, size);
                sm.node2b[threadIdx.x - 32] = pw32(sm.bpart2, (int)(lo - blo), (int)size);
            }
            __syncthreads();
            if (two && threadIdx.x == 32) {
                for (uint32_t w = 1u << dG; w > 1; w >>= 1)
                    for (uint32_t q = 0; q < w / 2; ++q)
                        sm.node2b[q] = sm.node2b[2 * q] + sm.node2b[2 * q + 1];
                blk2[bn] = sm.node2b[0];
            }
            if (threadIdx.x == 0) {
                for (uint32_t w = 1u << dG; w > 1; w >>= 1)
                    for (uint32_t q = 0; q < w / 2; ++q)
                        sm.node2[q] = sm.node2[2 * q] + sm.node2[2 * q + 1];
                blk[bn] = sm.node2[0];
                double bm = 0.0;
                for (int w = 0; w < kWarps; ++w) bm = std_max(bm, sm.wmax[w]);
                bmx[bn] = bm;
                sm.wq = nxt;
            }
            __syncthreads();
        }
        // every block has drawn its closing ticket: the last one out resets
        // this parity's counters (its next use is two sweeps and a grid
        // barrier away)
        if (dyn && threadIdx.x == 0 && atomicAdd(&F.ctl->wq_done[par], 1u) == vgrid(F) - 1) {
            atomicExch(wt, 0u);
            atomicExch(&F.ctl->wq_done[par], 0u);
        }
        SWEEP_STAMP(b0t0, 101);
        if (gbar(F, sm, op, it)) {
            if (threadIdx.x == 0) sm.c.done = 1;
            __syncthreads();
            return;
        }
        SWEEP_STAMP(b0t0, 102);
        top_all(blk, bmx, F.tb_nbn, sm, total, gm, two ? blk2 : nullptr, &total2);
    } else {
        double cmax = 0.0;
        {
            const uint32_t gw = vblock(F) * kWarps + warp, nw = vgrid(F) * kWarps;
            const uint32_t nchunks = (F.npix + NG - 1) / NG;
            for (uint32_t c = gw; c < nchunks; c += nw) {
                const uint32_t lo = c * NG;
                const uint32_t size = F.npix - lo < NG ? F.npix - lo : NG;
                if constexpr (G == 1)
                    sweep_node_thread<KIND>(F, sm, X, lo, size, cmax, nullptr, nullptr);
                else
                    sweep_node<KIND, G>(F, sm, X, lo, size, cmax);
            }
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) cmax = std_max(cmax, __shfl_xor_sync(0xffffffffu, cmax, o));
        if (lane == 0) sm.wmax[warp] = cmax;
        __syncthreads();
        if (threadIdx.x == 0) {
            double bm = 0.0;
            for (int w = 0; w < kWarps; ++w) bm = std_max(bm, sm.wmax[w]);
            F.bmax[vblock(F)] = bm;
        }
        if (gbar(F, sm, op, it)) {
            if (threadIdx.x == 0) sm.c.done = 1;
            __syncthreads();
            return;
        }
        for (uint32_t bn = vblock(F); bn < F.nbn; bn += vgrid(F)) {
            if (warp < F.wpb) {
                uint32_t lo, size;
                tree_node_range(F.npix, F.G, bn * (uint32_t)F.wpb + warp, lo, size);
                double* v = sm.u.sw.w[warp].vals;
                if ((uint32_t)lane < size) v[lane] = ld_cg(&F.part[lo + lane]);
                __syncwarp();
                if (lane == 0) sm.node[warp] = pw32(v, 0, (int)size);
            }
            __syncthreads();
            if (threadIdx.x == 0) {
                double v[kWarps];
                for (int w = 0; w < F.wpb; ++w) v[w] = sm.node[w];
                for (int w = F.wpb; w > 1; w >>= 1)
                    for (int q = 0; q < w / 2; ++q) v[q] = v[2 * q] + v[2 * q + 1];
                F.blk[bn] = v[0];
            }
            __syncthreads();
        }
        if (threadIdx.x == 0) {
            __threadfence();
            unsigned int tk = atomicAdd(&F.ctl->ticket, 1u);
            sm.is_last = (tk == vgrid(F) - 1);
        }
        __syncthreads();
        if (sm.is_last) {
            __threadfence();
            double t = top_tree(F, sm);
            double g = 0.0;
            for (uint32_t b = threadIdx.x; b < vgrid(F); b += kBlock) g = std_max(g, ld_cg(&F.bmax[b]));
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) g = std_max(g, __shfl_xor_sync(0xffffffffu, g, o));
            if (lane == 0) sm.wmax[warp] = g;
            __syncthreads();
            if (threadIdx.x == 0) {
                g = 0.0;
                for (int w = 0; w < kWarps; ++w) g = std_max(g, sm.wmax[w]);
                F.ctl->ticket = 0;
                F.ctl->red_total = t;
                F.ctl->red_max = g;
            }
        }
        if (gbar(F, sm, op, it)) {
            if (threadIdx.x == 0) sm.c.done = 1;
            __syncthreads();
            return;
        }
        total = ld_cg(&F.ctl->red_total);
        gm = ld_cg(&F.ctl->red_max);
    }
    if (threadIdx.x == 0) {
        controller(F, &sm.c, vblock(F) == 0, op, it, total, gm);
        // the second candidate is the next backtracking step: taken exactly
        // when the first was rejected and the search goes on
        if ((KIND == K_CAND_T || KIND == K_CAND_R) && X.two && F.cfg.blocktree && !sm.c.done)
            controller(F, &sm.c, vblock(F) == 0, op, it, total2, gm);
        sm.nsweep += 1u;
    }
    SWEEP_STAMP(b0t0, 103);
    __syncthreads();
}

// ---------------------------------------------------------------------------
// Neighbourhoods on the pinned fine grid.  Inside PALM every point sits at
// its fine-pixel centre (reconstruct.hpp:233,357-361), so the SpatialIndex
// ball (spatial_index.hpp:31-47: exact |q-p|^2 <= R^2, ascending index) is
// the set of points of the coarse pixels covering the fine window
// [fi-W, fi+W] x [fj-W, fj+W], W = floor(R/pitch)+1, visited in raster
// order (= ascending index, the cloud being pixel-major).
// ---------------------------------------------------------------------------
struct Pos {
    double x, y, z;
};

template <typename Fn>
__device__ __forceinline__ void for_each_pinned_neighbor(const Frame& F, int tc, int sc, int fi,
                                                         int fj, const Pos& q, double r2, Fn fn) {
    const int W = F.cfg.W, s = F.s;
    int a0 = fi - W, a1 = fi + W, b0 = fj - W, b1 = fj + W;
    a0 = a0 < 0 ? 0 : a0;
    b0 = b0 < 0 ? 0 : b0;
    a1 = a1 > F.frows - 1 ? F.frows - 1 : a1;
    b1 = b1 > F.fcols - 1 ? F.fcols - 1 : b1;
    const int ci0 = coarse_of(F, a0), ci1 = coarse_of(F, a1), cj0 = coarse_of(F, b0),
              cj1 = coarse_of(F, b1);
    const uint32_t* bo = F.bo[sc];
    const double* tt = F.t[tc];
    const int32_t* FI = F.fi[sc];
    const int32_t* FJ = F.fj[sc];
    for (int ci = ci0; ci <= ci1; ++ci) {
        const uint32_t prow = (uint32_t)ci * F.cols;
        const uint32_t m0 = bo[prow + cj0], m1 = bo[prow + cj1 + 1];
        for (uint32_t mm = m0; mm < m1; ++mm) {
            Pos o;
            o.x = (FI[mm] + 0.5) * F.pitch;
            o.y = (FJ[mm] + 0.5) * F.pitch;
            o.z = tt[mm] * F.bres;
            const double dx = o.x - q.x, dy = o.y - q.y, dz = o.z - q.z;
            const double d2 = dx * dx + dy * dy + dz * dz;
            if (d2 <= r2) fn(mm, o, d2);
        }
    }
}

constexpr int kMom = 19;        // APSS moments: wsum, mean(3), M(15)
// APSS summation lanes: ball member m is accumulated into lane partial
// m mod kApssLanes, the partials combined by the halving tree (the oracle's
// APSS_LANES); the device kernel runs 16 lanes per point
constexpr int kApssLanes = 16;
constexpr int kRedStride = 15;  // APSS pass-B partials per lane (M, lower triangle)

// Pratt moments of one member centred on the mean, (w d_r) d_c with
// d = (1, y, |y|^2) (denoise.hpp:73-80), into this lane's partials.  The
// weighted covariance of denoise.hpp:190-195 is (w y_r) y_c = M(r+1, c+1)
// term by term, so it is read off M: members with w == 0 add signed zeros,
// which leave a partial sum unchanged (partials start at +0 and are never
// -0), hence including them here and skipping them in M (denoise.hpp:75)
// give the same bits.
__device__ __forceinline__ void apss_pass_b(double (&b)[kRedStride], double w, double x, double y,
                                            double z, double m0, double m1, double m2) {
    const double y0 = x - m0, y1 = y - m1, y2 = z - m2;
    const double dv[5] = {1.0, y0, y1, y2, y0 * y0 + y1 * y1 + y2 * y2};
    int e = 0;
#pragma unroll
    for (int r = 0; r < 5; ++r) {
        const double wa = w * dv[r];
#pragma unroll
        for (int c = 0; c <= r; ++c) {  // fused multiply-add (the oracle's fma)
            b[e] = __fma_rn(wa, dv[c], b[e]);
            ++e;
        }
    }
}

// covariance (lower, row-major) from the Pratt moments
__device__ __forceinline__ void cov_from_moments(const double* M, double wsum, double cv[6]) {
    cv[0] = M[lt(1, 1)] / wsum;
    cv[1] = M[lt(2, 1)] / wsum;
    cv[2] = M[lt(2, 2)] / wsum;
    cv[3] = M[lt(3, 1)] / wsum;
    cv[4] = M[lt(3, 2)] / wsum;
    cv[5] = M[lt(3, 3)] / wsum;
}

// apss_project's degeneracy test on the covariance (denoise.hpp:197-203),
// the Jacobi sweeps skipped where the answer is provably "no"
// (cov_clearly_nondegenerate)
__device__ __forceinline__ bool cov_degenerate(const double cv[6]) {
    if (cov_clearly_nondegenerate(cv)) return false;
    double e0, e1, e2;
    sym3_eigenvalues(cv[0], cv[1], cv[2], cv[3], cv[4], cv[5], e0, e1, e2);
    return e2 <= 0.0 || e1 <= 1e-12 * e2;
}

// the halving tree over kApssLanes lane partials (column `col` of
// p[kApssLanes][stride]): p[l] = p[l] + p[l+o], o = kApssLanes/2..1 (oracle:
// lane_tree)
__device__ __forceinline__ double halving_sum_lanes(double* p, int stride, int col) {
    for (int o = kApssLanes / 2; o > 0; o >>= 1)
        for (int l = 0; l < o; ++l) p[l * stride + col] = p[l * stride + col] + p[(l + o) * stride + col];
    return p[col];
}

// apss_project for one point (denoise.hpp:163-214), neighbour enumerator
// supplied by the caller, in the lane-strided summation order of the warp
// kernel (rt3d_nbr.cuh) emulated sequentially.  Returns the new position in
// `out` when the fit projected it; updates flags.
template <typename Enum>
__device__ __forceinline__ bool apss_point(Enum&& each, const Pos& q, double R, int min_nbrs,
                                           double eps, uint8_t& flags, Pos& out) {
    const double r2 = R * R, Rinv = 1.0 / R;
    unsigned int cnt = 0;
    double pa[kApssLanes][4];
    for (int l = 0; l < kApssLanes; ++l) pa[l][0] = pa[l][1] = pa[l][2] = pa[l][3] = 0.0;
    each(r2, [&](uint32_t, const Pos& o, double d2) {
        const double w = apss_weight_d2(R, Rinv, d2);
        double* a = pa[cnt % (unsigned int)kApssLanes];
        ++cnt;
        a[0] += w;
        a[1] = __fma_rn(w, o.x, a[1]);
        a[2] = __fma_rn(w, o.y, a[2]);
        a[3] = __fma_rn(w, o.z, a[3]);
    });
    if (cnt < (unsigned int)min_nbrs) {
        flags |= 1u;
        return false;
    }
    const double wsum = halving_sum_lanes(&pa[0][0], 4, 0);
    double m0 = halving_sum_lanes(&pa[0][0], 4, 1), m1 = halving_sum_lanes(&pa[0][0], 4, 2),
           m2 = halving_sum_lanes(&pa[0][0], 4, 3);
    if (wsum <= 0.0) {
        flags |= 4u;
        return false;
    }
    m0 /= wsum;
    m1 /= wsum;
    m2 /= wsum;
    double pb[kApssLanes][kRedStride];
    for (int l = 0; l < kApssLanes; ++l)
        for (int e = 0; e < kRedStride; ++e) pb[l][e] = 0.0;
    unsigned int c2 = 0;
    each(r2, [&](uint32_t, const Pos& o, double d2) {
        apss_pass_b(pb[c2 % (unsigned int)kApssLanes], apss_weight_d2(R, Rinv, d2), o.x, o.y, o.z, m0, m1, m2);
        ++c2;
    });
    double cv[6], M[15];
    for (int e = 0; e < 15; ++e) M[e] = halving_sum_lanes(&pb[0][0], kRedStride, e);
    cov_from_moments(M, wsum, cv);
    if (cov_degenerate(cv)) {
        flags |= 4u;
        return false;
    }
    Sphere sp;
    if (!sphere_from_moments(M, m0, m1, m2, sp) ||
        !project_sphere(sp, eps, q.x, q.y, q.z, out.x, out.y, out.z)) {
        flags |= 4u;
        return false;
    }
    return true;
}

// top-k by (d^2, index), spatial_index.hpp:51-62, then the mean
// (denoise.hpp:228-235)
template <typename Enum, typename RFn>
__device__ __forceinline__ double knn_mean(Enum&& each, int k, double r2, double self_r, RFn rof) {
    if (k <= kKnnFast) {
        double kd[kKnnFast];
        uint32_t ki[kKnnFast];
        int cnt = 0;
        each(r2, [&](uint32_t mm, const Pos&, double d2) {
            if (cnt == k && !(d2 < kd[cnt - 1] || (d2 == kd[cnt - 1] && mm < ki[cnt - 1]))) return;
            int pos = cnt < k ? cnt : k - 1;
            while (pos > 0 && (d2 < kd[pos - 1] || (d2 == kd[pos - 1] && mm < ki[pos - 1]))) {
                kd[pos] = kd[pos - 1];
                ki[pos] = ki[pos - 1];
                --pos;
            }
            kd[pos] = d2;
            ki[pos] = mm;
            if (cnt < k) ++cnt;
        });
        if (cnt == 0) return self_r;
        double acc = 0.0;
        for (int q = 0; q < cnt; ++q) acc += rof(ki[q]);
        return acc / (double)cnt;
    }
    // large k: successive minimum selection
    double last_d = -1.0;
    uint32_t last_i = 0;
    bool have_last = false;
    double acc = 0.0;
    int cnt = 0;
    for (; cnt < k; ++cnt) {
        double bd = INFINITY;
        uint32_t bi = 0xffffffffu;
        bool found = false;
        each(r2, [&](uint32_t mm, const Pos&, double d2) {
            if (have_last && !(d2 > last_d || (d2 == last_d && mm > last_i))) return;
            if (!found || d2 < bd || (d2 == bd && mm < bi)) {
                bd = d2;
                bi = mm;
                found = true;
            }
        });
        if (!found) break;
        acc += rof(bi);
        last_d = bd;
        last_i = bi;
        have_last = true;
    }
    if (cnt == 0) return self_r;
    return acc / (double)cnt;
}

// prune (denoise.hpp:241-248) + SceneState::refresh (likelihood.hpp:38-55):
// per-pixel survivor counts, grid scan, stable scatter into the other buffers
template <class SM>
__device__ void phase_prune_a(const Frame& F, SM& sm, int rc, int sc) {
    const uint32_t* bo = F.bo[sc];
    const double* r = F.r[rc];
    const double rmin = F.cfg.r_min;
    scan_stage_a(F, sm, [&](uint32_t p) {
        unsigned int c = 0;
        for (uint32_t n = bo[p]; n < bo[p + 1]; ++n) c += (r[n] >= rmin) ? 1u : 0u;
        return c;
    });
}

template <class SM>
__device__ void phase_prune_b(const Frame& F, SM& sm, int tc, int rc, int sc) {
    unsigned int total = 0, band_base = 0, band_end = 0;
    unsigned int base = scan_stage_b_base(F, sm, &total, &band_base, &band_end);
    uint32_t c0, c1;
    chunk_range(F, c0, c1);
    const uint32_t* bo = F.bo[sc];
    const double rmin = F.cfg.r_min;
    for (uint32_t p = c0 + threadIdx.x; p < c1; p += kBlock) {
        uint32_t o = base + ld_cg(&F.cnt[p]);
        RT3D_CHECK(o <= F.pcap && bo[p] <= bo[p + 1] && bo[p + 1] <= F.pcap);
        F.bo[sc ^ 1][p] = o;
        for (uint32_t n = bo[p]; n < bo[p + 1]; ++n) {
            const double rv = F.r[rc][n];
            if (!(rv >= rmin)) continue;
            F.t[tc ^ 1][o] = F.t[tc][n];
            F.r[rc ^ 1][o] = rv;
            F.pix[sc ^ 1][o] = F.pix[sc][n];
            F.fi[sc ^ 1][o] = F.fi[sc][n];
            F.fj[sc ^ 1][o] = F.fj[sc][n];
            F.fl[sc ^ 1][o] = F.fl[sc][n];
            F.mig[sc ^ 1][o] = F.mig[sc][n];
            ++o;
        }
    }
    if (vblock(F) == vgrid(F) - 1 && threadIdx.x == 0) {
        F.bo[sc ^ 1][F.bpix1] = band_end;
        F.ctl->pbase = band_base;
        F.ctl->pown = band_end - band_base;
    }
    if (scan_block(F) == F.sblk_n - 1 && threadIdx.x == 0) F.barc->P = total;
}

// ---------------------------------------------------------------------------
// FFT background low-pass (denoise.hpp:254-319): unnormalised forward 2-D
// DFT, radial raised-cosine mask, backward DFT / (nr*nc), clamp >= 0.
// Separable direct DFTs (exactly reduced twiddle phases), three stages.
// ---------------------------------------------------------------------------
__device__ __forceinline__ double lowpass_mask(double rho, double cutoff) {
    if (cutoff >= 1.0) return 1.0;
    double w = std_min(0.2 * cutoff, 1.0 - cutoff);
    double lo = cutoff - w;
    if (rho <= lo) return 1.0;
    if (rho >= cutoff) return 0.0;
    return 0.5 * (1.0 + cospi((rho - lo) / w));
}

// stage 1: forward DFT along every row of img (real) -> (re, im)
static __device__ void fft_stage1(const double* img, double* re, double* im, int nr, int nc,
                           uint32_t gtid, uint32_t nth) {
    for (uint32_t idx = gtid; idx < (uint32_t)(nr * nc); idx += nth) {
        const int a = idx / nc, k = idx % nc;
        double ar = 0.0, ai = 0.0;
        for (int x = 0; x < nc; ++x) {
            const int ph = (int)(((long long)k * x) % nc);
            double sn, cs;
            sincospi(2.0 * ph / nc, &sn, &cs);
            const double v = img[(size_t)a * nc + x];
            ar += v * cs;
            ai -= v * sn;
        }
        re[idx] = ar;
        im[idx] = ai;
    }
}

// stage 2: per column: forward DFT along rows, mask, backward DFT along rows
static __device__ void fft_stage2(double* re, double* im, double* re2, double* im2, int nr, int nc,
                           double cutoff, uint32_t gtid, uint32_t nth) {
    const double fmax_r = (double)(nr / 2) / nr;
    const double fmax_c = (double)(nc / 2) / nc;
    const double rho_max = sqrt(fmax_r * fmax_r + fmax_c * fmax_c);
    for (uint32_t idx = gtid; idx < (uint32_t)(nr * nc); idx += nth) {
        // idx = (ka, b): forward along rows at frequency ka for column b
        const int ka = idx / nc, b = idx % nc;
        double ar = 0.0, ai = 0.0;
        for (int x = 0; x < nr; ++x) {
            const int ph = (int)(((long long)ka * x) % nr);
            double sn, cs;
            sincospi(2.0 * ph / nr, &sn, &cs);
            const double xr = re[(size_t)x * nc + b], xi = im[(size_t)x * nc + b];
            ar += xr * cs + xi * sn;
            ai += xi * cs - xr * sn;
        }
        const int far = (ka <= nr / 2) ? ka : ka - nr;
        const int fac = (b <= nc / 2) ? b : b - nc;
        const double fr = (double)far / nr, fc = (double)fac / nc;
        const double mval = lowpass_mask(sqrt(fr * fr + fc * fc) / rho_max, cutoff);
        re2[idx] = ar * mval;
        im2[idx] = ai * mval;
    }
}

static __device__ void fft_stage3(const double* re2, const double* im2, double* re, double* im, int nr,
                           int nc, uint32_t gtid, uint32_t nth) {
    // backward along rows (column direction) for each (a, b)
    for (uint32_t idx = gtid; idx < (uint32_t)(nr * nc); idx += nth) {
        const int a = idx / nc, b = idx % nc;
        double ar = 0.0, ai = 0.0;
        for (int k = 0; k < nr; ++k) {
            const int ph = (int)(((long long)k * a) % nr);
            double sn, cs;
            sincospi(2.0 * ph / nr, &sn, &cs);
            const double xr = re2[(size_t)k * nc + b], xi = im2[(size_t)k * nc + b];
            ar += xr * cs - xi * sn;
            ai += xr * sn + xi * cs;
        }
        re[idx] = ar;
        im[idx] = ai;
    }
}

static __device__ void fft_stage4(const double* re, const double* im, double* out, int nr, int nc,
                           int clamp_nonneg, uint32_t gtid, uint32_t nth) {
    const double total = (double)nr * nc;
    for (uint32_t idx = gtid; idx < (uint32_t)(nr * nc); idx += nth) {
        const int a = idx / nc, y = idx % nc;
        double ar = 0.0;
        for (int k = 0; k < nc; ++k) {
            const int ph = (int)(((long long)k * y) % nc);
            double sn, cs;
            sincospi(2.0 * ph / nc, &sn, &cs);
            ar += re[(size_t)a * nc + k] * cs - im[(size_t)a * nc + k] * sn;
        }
        const double v = ar / total;
        out[idx] = clamp_nonneg ? std_max(0.0, v) : v;
    }
}

// Radix-2 path for power-of-two images (both sides <= kFftMax): per line an
// in-place Cooley-Tukey FFT in shared memory (bit reversal, log2 n butterfly
// passes, exact twiddle phases pos / len), O(n^2 log n) for an n x n image.
// Three grid phases: forward along every row; per column forward, mask,
// backward (in place); backward along every row, / (nr nc), clamp.  Agrees
// with the direct DFT to rounding (~1e-16 relative).
constexpr int kFftMax = 1024;
__device__ __forceinline__ bool fft_pow2(int n) { return n >= 2 && n <= kFftMax && !(n & (n - 1)); }

__device__ __forceinline__ void fft_line(double* re, double* im, int n, double sign) {
    const int logn = __ffs(n) - 1;
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
        const int j = (int)(__brev((unsigned)i) >> (32 - logn));
        if (j > i) {
            const double a = re[i], b = im[i];
            re[i] = re[j];
            im[i] = im[j];
            re[j] = a;
            im[j] = b;
        }
    }
    __syncthreads();
    for (int len = 2; len <= n; len <<= 1) {
        const int half = len >> 1;
        for (int k = threadIdx.x; k < n / 2; k += blockDim.x) {
            const int pos = k & (half - 1);
            const int i0 = (k - pos) * 2 + pos, i1 = i0 + half;
            double sn, cs;
            sincospi(2.0 * pos / len, &sn, &cs);
            const double wr = cs, wi = sign * sn;
            const double tr = re[i1] * wr - im[i1] * wi, ti = re[i1] * wi + im[i1] * wr;
            re[i1] = re[i0] - tr;
            im[i1] = im[i0] - ti;
            re[i0] = re[i0] + tr;
            im[i0] = im[i0] + ti;
        }
        __syncthreads();
    }
}

// phase 1: forward FFT along every row of the real image
static __device__ void fftp_rows_forward(const double* img, double* re, double* im, int nr, int nc,
                                  double* s_re, double* s_im, uint32_t blk, uint32_t nblk) {
    for (uint32_t a = blk; a < (uint32_t)nr; a += nblk) {
        for (int x = threadIdx.x; x < nc; x += blockDim.x) {
            s_re[x] = img[(size_t)a * nc + x];
            s_im[x] = 0.0;
        }
        __syncthreads();
        fft_line(s_re, s_im, nc, -1.0);
        for (int x = threadIdx.x; x < nc; x += blockDim.x) {
            re[(size_t)a * nc + x] = s_re[x];
            im[(size_t)a * nc + x] = s_im[x];
        }
        __syncthreads();
    }
}

// phase 2: per column, forward FFT, the radial raised-cosine mask, backward FFT
static __device__ void fftp_cols_mask(double* re, double* im, int nr, int nc, double cutoff, double* s_re,
                               double* s_im, uint32_t blk, uint32_t nblk) {
    const double fmax_r = (double)(nr / 2) / nr;
    const double fmax_c = (double)(nc / 2) / nc;
    const double rho_max = sqrt(fmax_r * fmax_r + fmax_c * fmax_c);
    for (uint32_t b = blk; b < (uint32_t)nc; b += nblk) {
        for (int x = threadIdx.x; x < nr; x += blockDim.x) {
            s_re[x] = re[(size_t)x * nc + b];
            s_im[x] = im[(size_t)x * nc + b];
        }
        __syncthreads();
        fft_line(s_re, s_im, nr, -1.0);
        const int fac = ((int)b <= nc / 2) ? (int)b : (int)b - nc;
        const double fc = (double)fac / nc;
        for (int ka = threadIdx.x; ka < nr; ka += blockDim.x) {
            const int far = (ka <= nr / 2) ? ka : ka - nr;
            const double fr = (double)far / nr;
            const double mval = lowpass_mask(sqrt(fr * fr + fc * fc) / rho_max, cutoff);
            s_re[ka] *= mval;
            s_im[ka] *= mval;
        }
        __syncthreads();
        fft_line(s_re, s_im, nr, 1.0);
        for (int x = threadIdx.x; x < nr; x += blockDim.x) {
            re[(size_t)x * nc + b] = s_re[x];
            im[(size_t)x * nc + b] = s_im[x];
        }
        __syncthreads();
    }
}

// phase 3: backward FFT along every row, / (nr nc), optional clamp at zero
static __device__ void fftp_rows_backward(const double* re, const double* im, double* out, int nr, int nc,
                                   int clamp_nonneg, double* s_re, double* s_im, uint32_t blk,
                                   uint32_t nblk) {
    const double total = (double)nr * nc;
    for (uint32_t a = blk; a < (uint32_t)nr; a += nblk) {
        for (int x = threadIdx.x; x < nc; x += blockDim.x) {
            s_re[x] = re[(size_t)a * nc + x];
            s_im[x] = im[(size_t)a * nc + x];
        }
        __syncthreads();
        fft_line(s_re, s_im, nc, 1.0);
        for (int y = threadIdx.x; y < nc; y += blockDim.x) {
            const double v = s_re[y] / total;
            out[(size_t)a * nc + y] = clamp_nonneg ? std_max(0.0, v) : v;
        }
        __syncthreads();
    }
}

}  // namespace rt3d
