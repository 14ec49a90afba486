/*
 * rt3d_oracle.h — TEST INFRASTRUCTURE ONLY.
 *
 * A plain-C restatement of the reference RT3D path (splidar, header-only C++,
 * /root/reference/proj/include/splidar), used exclusively by tests/, by
 * __graft_entry__.smoke() and by bench.py's cpu_baseline leg as the checker.
 * Nothing in the product (paper_1905_06700_b200/, include/) links or calls it.
 *
 * Every function cites the reference file:line it follows.  Floating-point
 * expressions keep the reference's evaluation order; the library is compiled
 * with -ffp-contract=off and no -march (the reference's Release build has no
 * FMA), so on the same inputs the results are bit-identical to the compiled
 * reference except where the reference calls Eigen (APSS eigen-solves, see
 * oracle_apss_project) or FFTW (oracle_fft_lowpass_filter).
 *
 * Parity is pinned by tests/test_oracle.py: the reference's own known-answer
 * and property tests (tests/test_likelihood.cpp, test_denoise.cpp,
 * test_init.cpp, test_palm.cpp, acceptance C1-C3) restated against this
 * library, plus a bit-for-bit comparison against the reference headers
 * compiled here (oracle/_ref, built by oracle/Makefile with test-only Eigen /
 * FFTW stand-ins) on seeded simulator scenes.
 */
#ifndef RT3D_ORACLE_H
#define RT3D_ORACLE_H

#include "../include/rt3d.h"

#ifdef __cplusplus
extern "C" {
#endif

/* Irf::gaussian + Irf normalisation (sensor.hpp:26-57).  Writes the
 * normalised samples; returns the sample count (0 if cap is too small). */
uint64_t oracle_irf_gaussian(double sigma_bins, double n_sigmas, double dtau, double* samples,
                             uint64_t cap, double* tau_min);
/* Irf ctor normalisation of raw samples in place (sensor.hpp:26-41). */
int oracle_irf_normalise(double* samples, uint64_t n, double dtau);
double oracle_irf_value(const rt3d_irf* irf, double tau);
double oracle_irf_deriv(const rt3d_irf* irf, double tau);
double oracle_irf_mass_in_gate(const rt3d_irf* irf, double t, int n_bins);

/* parallel.hpp:52-61 */
double oracle_pairwise_sum(const double* v, uint64_t n);

/* reconstruct.hpp:120-189; returns the peak count (<= k). */
int oracle_matched_filter_peaks(const rt3d_event* events, uint64_t n_events, const rt3d_irf* irf,
                                int n_bins, int k, double threshold, int min_sep,
                                rt3d_peak* out);

/* reconstruct.hpp:197-249.  points must hold max_returns*s*s*n_pixels. */
int oracle_init_matched_filter(const rt3d_cube* cube, const rt3d_sensor* sensor,
                               const rt3d_init_params* params, rt3d_point* points,
                               uint64_t* n_points, double* background);

/* likelihood.hpp:136-333 on a state given as (points, n, background) — the
 * buckets are rebuilt with SceneState::refresh (likelihood.hpp:38-55). */
double oracle_nll(const rt3d_cube* cube, const rt3d_sensor* sensor, const rt3d_point* points,
                  uint64_t n, const double* background);
void oracle_grad_depth(const rt3d_cube* cube, const rt3d_sensor* sensor,
                       const rt3d_point* points, uint64_t n, const double* background,
                       double* value, uint8_t* out_of_gate);
void oracle_grad_intensity(const rt3d_cube* cube, const rt3d_sensor* sensor,
                           const rt3d_point* points, uint64_t n, const double* background,
                           double* out);
void oracle_grad_background(const rt3d_cube* cube, const rt3d_sensor* sensor,
                            const rt3d_point* points, uint64_t n, const double* background,
                            double* out);
void oracle_block_curvatures(const rt3d_cube* cube, const rt3d_sensor* sensor,
                             const rt3d_point* points, uint64_t n, const double* background,
                             double* depth, double* intensity, double* bg_curv);

/* denoise.hpp:159-217 with SpatialIndex (spatial_index.hpp:18-77) built over
 * index_cloud with cell size `cell`.  Returns 0, or -1 (invalid_argument). */
int oracle_apss_project(const rt3d_point* cloud, uint64_t n, const rt3d_apss_params* params,
                        const rt3d_point* index_cloud, uint64_t n_index, double cell,
                        rt3d_point* out);
/* denoise.hpp:223-237 */
int oracle_knn_intensity_filter(const rt3d_point* cloud, uint64_t n, int k,
                                const rt3d_point* index_cloud, uint64_t n_index, double cell,
                                double radius, rt3d_point* out);
/* denoise.hpp:241-248; returns survivors. */
uint64_t oracle_prune(const rt3d_point* cloud, uint64_t n, double r_min, rt3d_point* out);
/* evaluate (eval.hpp:33-87); out7 = recall, false_point_rate, depth_rmse,
   intensity_mae, n_truth, n_est, n_matched; returns 0, or 1 for tau/pitch <= 0 */
int oracle_evaluate(const rt3d_point* est, uint64_t n_est, const rt3d_point* truth, uint64_t n_truth,
                    double tau, double pitch, double* out7);
/* denoise.hpp:254-319 (direct DFT instead of FFTW). */
int oracle_fft_lowpass_filter(const double* img, int rows, int cols, double cutoff,
                              int clamp_nonneg, double* out);

/* reconstruct.hpp:300-435 in place on (points, *n, background). */
int oracle_palm_step(const rt3d_cube* cube, const rt3d_sensor* sensor,
                     const rt3d_recon_config* cfg, rt3d_point* points, uint64_t* n,
                     double* background, rt3d_step_diag* diag);

/* reconstruct.hpp:457-489.  points: capacity max_returns*s*s*n_pixels;
 * nll_trace: max_iters+1; steps: max_iters. */
int oracle_reconstruct(const rt3d_cube* cube, const rt3d_sensor* sensor,
                       const rt3d_recon_config* cfg, rt3d_point* points, uint64_t* n_points,
                       double* background, double* nll_trace, rt3d_step_diag* steps,
                       int* iterations);

/* eval.hpp:91-126 */
int oracle_baseline_xcorr(const rt3d_cube* cube, const rt3d_sensor* sensor, rt3d_point* points,
                          uint64_t* n_points);

/* Stage-level hooks used by the parity tests: the 5x5 Pratt pencil solve and
 * the 3x3 covariance eigenvalues of the APSS fit. */
int oracle_pratt_smallest(const double m[25], double u[5]);
void oracle_sym3_eigenvalues(const double c[9], double ev[3]);

#ifdef __cplusplus
}
#endif

#endif
