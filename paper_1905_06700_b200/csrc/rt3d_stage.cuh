// rt3d_stage.cuh — the cooperative stage kernels of a frame (init + PALM
// blocks between grid barriers).  Instantiated per lane-group configuration
// in rt3d_stage_g{3,4,32}.cu so the three heavy instantiation sets compile in
// parallel; rt3d.cu reaches them through stage_fn_g*().
#pragma once

#include "rt3d_frame.cuh"
#include "rt3d_nbr.cuh"

#ifndef RT3D_G1_MIN_BLOCKS
#define RT3D_G1_MIN_BLOCKS 3
#endif

namespace rt3d {

// grid barrier + optional phase stamp (leader thread, after the barrier)
template <class SM>
__device__ __forceinline__ void gsync(SM& sm, const Frame& F, int phase) {
    gbar(F, sm, 1000 + phase);
    if (F.prof && vblock(F) == 0 && threadIdx.x == 0) {
        unsigned int k = F.ctl->nprof;
        if (k < F.ctl->prof_cap) {
            F.prof[2 * k] = (unsigned long long)phase;
            F.prof[2 * k + 1] = globaltimer();
            F.ctl->nprof = k + 1;
        }
    }
}

__device__ __forceinline__ void stamp(const Frame& F, int phase) {
    if (F.prof && vblock(F) == 0 && threadIdx.x == 0) {
        unsigned int k = F.ctl->nprof;
        if (k < F.ctl->prof_cap) {
            F.prof[2 * k] = (unsigned long long)phase;
            F.prof[2 * k + 1] = globaltimer();
            F.ctl->nprof = k + 1;
        }
    }
}

template <int KIND, int G>
__device__ void cand_loop(const Frame& F, SmemT<G>& sm, int tc, int rc, int bc, int sc, int op,
                          int it) {
    // sm.c is this block's controller replica: every block sees the same
    // decisions after each sweep (tree_sweep_g ends with a block barrier)
    // (the depth block backtracks about half the time on config B, the
    // intensity block nearly always: two candidates pay for the latter)
    const bool two = F.cfg.blocktree && ((KIND == K_CAND_R && (F.cfg.two_cand & 1)) ||
                                         (KIND == K_CAND_T && (F.cfg.two_cand & 2)));
    SweepCtx X;
    X.cfloor = 1e-3 * sm.c.cmax + 1e-30;
    X.tc = tc;
    X.rc = rc;
    X.bc = bc;
    X.sc = sc;
    X.apply_floor = 0;
    X.mig_cached = 0;
    while (!sm.c.done) {
        X.alpha = sm.c.alpha;
        // two candidates per sweep (alpha, alpha * beta) while another
        // backtrack is allowed; the controller consumes them in order
        X.two = two && sm.c.bt + 1 < kMaxBacktracks;
        X.alpha2 = X.alpha * F.cfg.beta;
        tree_sweep_g<KIND, G>(F, sm, X, op, it);
        stamp(F, KIND == K_CAND_T ? PH_CAND_T : KIND == K_CAND_R ? PH_CAND_R : PH_CAND_B);
    }
    if (two && sm.c.accept) {
        // two-candidate sweeps do not store their candidates: write the
        // accepted one for this block's own points (same expressions)
        const double a = sm.c.alpha;
        for (uint32_t bn = F.bbn0 + vblock(F); bn < F.bbn1; bn += vgrid(F)) {
            uint32_t blo, bsz;
            tree_node_range(F.npix, F.tb_G, bn, blo, bsz);
            const uint32_t n0 = F.bo[sc][blo], n1 = F.bo[sc][blo + bsz];
            for (uint32_t n = n0 + threadIdx.x; n < n1; n += kBlock) {
                if (KIND == K_CAND_T) F.t[tc ^ 1][n] = cand_t_value(F, X, n, F.t[tc][n], a);
                else F.r[rc ^ 1][n] = cand_r_value(F, X, n, F.r[rc][n], a);
            }
        }
        __syncthreads();
    }
}

enum Stage : int { ST_FIRST = 0, ST_DEPTH = 1, ST_INTENSITY = 2, ST_TAIL = 3, ST_ITER = 4 };

// depth block of iteration it, reconstruct.hpp:320-350: safeguarded gradient
// step; returns the new t toggle.  Runs at the end of the stage kernel that
// computed the depth gradients (ST_FIRST for iteration 0, ST_TAIL for the
// next iteration), so it needs no launch of its own.
template <int G>
__device__ int depth_block(const Frame& F, SmemT<G>& sm, int it, int tc, int rc, int bc, int sc) {
    const uint32_t P = global_P(F);
    if (vblock(F) == 0 && threadIdx.x == 0) {
        StepDiagDev& d = F.diag[it];
        d.nll_before = sm.c.nll_cur;
        d.points_before = P;
        if (P == 0) {
            d.blk[0].nll_after_grad = d.blk[0].nll_after_denoise = d.nll_before;
            d.blk[1].nll_after_grad = d.blk[1].nll_after_denoise = d.nll_before;
        }
    }
    if (P > 0) {
        cand_loop<K_CAND_T, G>(F, sm, tc, rc, bc, sc, OP_CAND_T, it);
        if (sm.c.accept) tc ^= 1;
    }
    return tc;
}

// blocks per SM the register budget is sized for: 2 (128 registers) for the
// lane-group sweeps, more for the thread-per-pixel sweeps of large arrays
template <int G>
struct StageOcc {
    static constexpr int kBlocks = G == 1 ? RT3D_G1_MIN_BLOCKS : 2;
};

template <int STAGE, int G>
__global__ void __launch_bounds__(kBlock, StageOcc<G>::kBlocks)
    stage_kernel(const __grid_constant__ FrameBatch FB, int it);

// One stage of a frame: a cooperative kernel whose phases are separated by
// grid barriers.  Buffer toggles live in Ctl between kernels; every block
// reads them at entry, the leader writes them back at exit (after at least
// one barrier, so no block still reads them).
template <int STAGE, int G>
__global__ void __launch_bounds__(kBlock, StageOcc<G>::kBlocks)
    stage_kernel(const __grid_constant__ FrameBatch FB, int it) {
    const Frame& F = FB.f[FB.n == 1 ? 0u : FB.first + blockIdx.x / FB.bpf];
    constexpr int stage = STAGE;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    SmemT<G>& sm = *reinterpret_cast<SmemT<G>*>(smem_raw);
    const bool leader = vblock(F) == 0 && threadIdx.x == 0;
    const int prog = F.cfg.program;
    if (STAGE != ST_FIRST && (ld_cg(&F.ctl->stop) || ld_cg(&F.ctl->abort))) return;
    if (!F.irf_of_pix) {  // shared IRF: tables in shared memory
        const IrfDev f0 = F.irfs[0];
        if (f0.n <= (uint32_t)kIrfSmem) {
            for (uint32_t k = threadIdx.x; k < f0.n; k += kBlock) {
                sm.irf_tab[k] = f0.s[k];
                if (k + 1 < f0.n) sm.irf_tab[kIrfSmem + k] = f0.d[k];
            }
        }
        if (threadIdx.x == 0) {
            sm.irf0 = f0;
            if (f0.n <= (uint32_t)kIrfSmem) {
                sm.irf0.s = sm.irf_tab;
                sm.irf0.d = sm.irf_tab + kIrfSmem;
            }
        }
    }
    if (threadIdx.x == 0) {
        sm.nsweep = 0;
        sm.aborted = 0;
        // controller replica: zero for a new frame, else the state the
        // previous kernel's block 0 wrote back
        uint64_t* d = reinterpret_cast<uint64_t*>(&sm.c);
        const uint64_t* g = reinterpret_cast<const uint64_t*>(F.ctl);
        for (int k = 0; k < (int)(sizeof(Ctl) / 8); ++k) d[k] = stage == ST_FIRST ? 0ull : ld_cg(&g[k]);
        if (stage == ST_FIRST) sm.c.P = F.P0;
    }
    __syncthreads();
    int tc, rc, bc, sc;
    if (stage == ST_FIRST) {
        tc = F.tc0;
        rc = F.rc0;
        bc = F.bc0;
        sc = F.sc0;
        if (leader) {
            // Ctl was zeroed by cudaMemsetAsync; nothing else reads these
            // before the first barrier.
            const unsigned long long t0 = globaltimer();
            F.ctl->t_start = t0;
            F.ctl->P = F.P0;
            F.ctl->pown = F.P0;
            F.ctl->pbase = 0;
            F.ctl->prof_cap = F.prof_cap;
            if (F.prof && F.prof_cap) {
                F.prof[0] = 0;
                F.prof[1] = t0;
                F.ctl->nprof = 1;
            }
        }
    } else {
        tc = ld_cg(&F.ctl->tc);
        rc = ld_cg(&F.ctl->rc);
        bc = ld_cg(&F.ctl->bc);
        sc = ld_cg(&F.ctl->sc);
        stamp(F, stage == ST_INTENSITY ? PH_APSS : stage == ST_TAIL ? PH_KNN : PH_LAUNCH);
    }
    SweepCtx X0;
    X0.alpha = 0.0;
    X0.cfloor = 0.0;
    X0.apply_floor = 0;
    X0.mig_cached = 0;

    if constexpr (STAGE == ST_FIRST) {
        if (prog == PROG_RECON || prog == PROG_INIT || prog == PROG_BASELINE ||
            prog == PROG_PEAKS) {
            phase_init_peaks(F, sm);
            gsync(sm, F, PH_INIT_PEAKS);
            if (prog == PROG_PEAKS) return;
            const bool baseline = prog == PROG_BASELINE;
            const int s2 = F.s * F.s;
            scan_stage_a(F, sm, [&](uint32_t p) {
                uint32_t nv = F.nval[p];
                return baseline ? (nv > 0 ? 1u : 0u) : nv * (uint32_t)s2;
            });
            gsync(sm, F, PH_SCAN);
            phase_spawn(F, sm, baseline);
            gsync(sm, F, PH_SPAWN);
            tc = rc = bc = sc = 0;
        }
        if (leader) F.ctl->t_init = globaltimer();
        X0.tc = tc;
        X0.rc = rc;
        X0.bc = bc;
        X0.sc = sc;
        if (prog == PROG_NLL) {
            tree_sweep_g<K_NLL, G>(F, sm, X0, OP_RESULT, 0);
        } else if (prog == PROG_GRADS) {
            tree_sweep_g<K_GRAD_T, G>(F, sm, X0, OP_RESULT, 0);
            tree_sweep_g<K_GRAD_R, G>(F, sm, X0, OP_RESULT, 0);
            tree_sweep_g<K_GRAD_B, G>(F, sm, X0, OP_RESULT, 0);
        } else if (prog == PROG_RECON || prog == PROG_PALM) {
            // nll at the initial state + depth gradients (reconstruct.hpp:466)
            tree_sweep_g<K_GRAD_T, G>(F, sm, X0, OP_GRAD_T_FIRST, 0);
            stamp(F, PH_GRAD_T);
            if (F.cfg.fuse_depth) tc = depth_block<G>(F, sm, 0, tc, rc, bc, sc);
        }
    } else if constexpr (STAGE == ST_DEPTH) {
        tc = depth_block<G>(F, sm, it, tc, rc, bc, sc);
    }
    if constexpr (STAGE == ST_ITER) {
        // a whole iteration in one launch: the APSS moments and fit as grid
        // phases between barriers (same device functions as apss_kernel /
        // apss_fit_kernel, warp scratch in the stage union)
        const uint32_t P = global_P(F);
        if (P > 0) {
            apss_moment_warps(F, reinterpret_cast<ApssWarpSm*>(sm.u.nbr), ld_cg(&F.ctl->pbase),
                              ld_cg(&F.ctl->pown), tc, sc, kApssStageWarps);
            gsync(sm, F, PH_APSS);
            apss_fit_threads(F, ld_cg(&F.ctl->pbase), ld_cg(&F.ctl->pown), tc, sc);
            gsync(sm, F, PH_APSS_FIT);
        }
    }
    if constexpr (STAGE == ST_INTENSITY || STAGE == ST_ITER) {
        // APSS wrote t[tc^1]; intensity block, :371-392
        const uint32_t P = global_P(F);
        if (P > 0) {
            tc ^= 1;
            SweepCtx X = X0;
            X.tc = tc;
            X.rc = rc;
            X.bc = bc;
            X.sc = sc;
            tree_sweep_g<K_GRAD_R, G>(F, sm, X, OP_GRAD_R, it);
            stamp(F, PH_GRAD_R);
            cand_loop<K_CAND_R, G>(F, sm, tc, rc, bc, sc, OP_CAND_R, it);
            if (sm.c.accept) rc ^= 1;
        }
    }
    if constexpr (STAGE == ST_ITER) {
        // the kNN filter as a grid phase (knn_kernel's device function); it
        // counts the points prune will keep into ctl->keep (reset by the
        // previous kernel's write-back)
        const uint32_t P = global_P(F);
        if (P > 0) {
            gsync(sm, F, PH_GRAD_R);  // the accepted intensity candidates of every block
            knn_warps(F, reinterpret_cast<KnnWarpSm*>(sm.u.nbr), ld_cg(&F.ctl->pbase),
                      ld_cg(&F.ctl->pown), tc, rc, sc);
            gsync(sm, F, PH_KNN);
        }
    }
    if constexpr (STAGE == ST_TAIL || STAGE == ST_ITER) {
        // kNN wrote r[rc^1] (knn_kernel); prune + refresh (:395-397), then
        // the background block (:405-429) and the nll that ends the iteration
        const uint32_t P = global_P(F);
        SweepCtx X = X0;
        if (P > 0) {
            rc ^= 1;
            // the kNN kernel counted the points at r >= r_min: when prune keeps
            // them all the compaction is the identity and the buffers stay
            // (row bands always compact: the count is per band)
            if (F.nbands > 1 || ld_cg(&F.ctl->keep) != P) {
                phase_prune_a(F, sm, rc, sc);
                gsync(sm, F, PH_PRUNE_A);
                phase_prune_b(F, sm, tc, rc, sc);
                gsync(sm, F, PH_PRUNE_B);
                tc ^= 1;
                rc ^= 1;
                sc ^= 1;
            }
            X.tc = tc;
            X.rc = rc;
            X.bc = bc;
            X.sc = sc;
            tree_sweep_g<K_GRAD_B, G>(F, sm, X, OP_GRAD_B_PRUNED, it);
            stamp(F, PH_GRAD_B);
        } else {
            X.tc = tc;
            X.rc = rc;
            X.bc = bc;
            X.sc = sc;
            tree_sweep_g<K_GRAD_B, G>(F, sm, X, OP_GRAD_B_EMPTY, it);
            stamp(F, PH_GRAD_B);
        }
        cand_loop<K_CAND_B, G>(F, sm, tc, rc, bc, sc, OP_CAND_B, it);
        if (sm.c.accept) bc ^= 1;
        if (F.cfg.bg_mode == 1) {
            const uint32_t nth = vgrid(F) * kBlock;
            const uint32_t gtid = vblock(F) * kBlock + threadIdx.x;
            const int nr = F.rows, nc = F.cols;
            double* re = F.fft_re;
            double* im = F.fft_im;
            double* re2 = F.fft_re + F.npix;
            double* im2 = F.fft_im + F.npix;
            if (fft_pow2(nr) && fft_pow2(nc) &&
                2 * kFftMax * sizeof(double) <= sizeof(sm.u)) {  // radix 2, lines in shared memory
                double* s_re = reinterpret_cast<double*>(&sm.u);
                double* s_im = s_re + kFftMax;
                fftp_rows_forward(F.b[bc], re, im, nr, nc, s_re, s_im, vblock(F), vgrid(F));
                gsync(sm, F, PH_FFT);
                fftp_cols_mask(re, im, nr, nc, F.cfg.cutoff, s_re, s_im, vblock(F), vgrid(F));
                gsync(sm, F, PH_FFT);
                fftp_rows_backward(re, im, F.b[bc], nr, nc, 1, s_re, s_im, vblock(F), vgrid(F));
                gsync(sm, F, PH_FFT);
            } else {
            fft_stage1(F.b[bc], re, im, nr, nc, gtid, nth);
            gsync(sm, F, PH_FFT);
            fft_stage2(re, im, re2, im2, nr, nc, F.cfg.cutoff, gtid, nth);
            gsync(sm, F, PH_FFT);
            fft_stage3(re2, im2, re, im, nr, nc, gtid, nth);
            gsync(sm, F, PH_FFT);
            fft_stage4(re, im, F.b[bc], nr, nc, 1, gtid, nth);
            gsync(sm, F, PH_FFT);
            }
        }
        X.bc = bc;
        X.apply_floor = 1;
        // t unchanged since GRAD_R (APSS output): mass_in_gate is cached,
        // unless the cloud was empty (no GRAD_R ran)
        X.mig_cached = global_P(F) > 0 ? 1 : 0;
        tree_sweep_g<K_GRAD_T, G>(F, sm, X, OP_GRAD_T_END, it);
        stamp(F, PH_GRAD_T);
        // the next iteration's depth block (skipped by the stop rule)
        if (F.cfg.fuse_depth && it + 1 < F.cfg.max_iters && !sm.c.stop)
            tc = depth_block<G>(F, sm, it + 1, tc, rc, bc, sc);
    }
    // row bands: every band's writes of this stage (the accepted candidates
    // included) are complete before any band's next kernel reads its halo
    if (F.nbands > 1) gsync(sm, F, PH_LAUNCH);
    if (leader && !sm.aborted) {
        // the controller replica back to F.ctl for the next kernel and the host
        Ctl* c = F.ctl;
        c->iterations = sm.c.iterations;
        c->stop = sm.c.stop;
        c->done = sm.c.done;
        c->accept = sm.c.accept;
        c->bt = sm.c.bt;
        c->nll_cur = sm.c.nll_cur;
        c->prev = sm.c.prev;
        c->init_nll = sm.c.init_nll;
        c->result = sm.c.result;
        c->alpha = sm.c.alpha;
        c->cmax = sm.c.cmax;
        c->keep = 0;  // the next kNN pass counts from zero
        c->knn_next = 0;
        c->knn_nres = 0;
        c->P = global_P(F);  // (row bands: all bands' points, from barc)
        F.ctl->tc = tc;
        F.ctl->rc = rc;
        F.ctl->bc = bc;
        F.ctl->sc = sc;
        F.ctl->t_end = globaltimer();
    }
}

using StageFn = void (*)(FrameBatch, int);
enum { kNumStages = 5 };

}  // namespace rt3d
