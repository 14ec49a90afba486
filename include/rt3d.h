/*
 * rt3d.h — C ABI of the B200 RT3D reconstruction path (librt3d.so).
 *
 * This is the drop-in boundary for the hot path of the reference library
 * `splidar` (header-only C++20, /root/reference/proj/include/splidar).  The
 * reference has no ABI of its own: every entry point below replaces one of its
 * inline C++ functions, cited as file:line.  The C++ headers under
 * include/splidar/ keep the reference's names and signatures and forward to
 * these functions; see INTEGRATION.md for the binding.
 *
 * Conventions
 *  - Plain pointers + sizes only; no C++ or torch types cross the boundary.
 *  - Every function returns rt3d_status.  On failure rt3d_last_error() holds a
 *    thread-local message.  The status maps onto the reference's exception
 *    types: INVALID_ARGUMENT -> std::invalid_argument, FORMAT ->
 *    splidar::FormatError, OUT_OF_RANGE -> std::out_of_range.
 *  - Inputs are caller-owned and only read during the call.  Device copies
 *    live in an rt3d_session (one CUDA device + one stream).  Results of
 *    init / palm_step / reconstruct / baseline stay resident in the session
 *    until copied out with rt3d_state_copy / rt3d_report_copy.
 *  - There is no CPU fallback: without a usable CUDA device every compute
 *    entry point returns RT3D_ERR_NO_DEVICE.
 *  - Results are deterministic run to run (no floating-point atomics).
 */
#ifndef RT3D_H
#define RT3D_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define RT3D_ABI_VERSION 1

typedef enum rt3d_status {
    RT3D_OK = 0,
    RT3D_ERR_INVALID_ARGUMENT = 1, /* std::invalid_argument                 */
    RT3D_ERR_FORMAT = 2,           /* splidar::FormatError (cube.hpp:11-14)  */
    RT3D_ERR_OUT_OF_RANGE = 3,     /* std::out_of_range (sensor.hpp:186-191) */
    RT3D_ERR_CUDA = 4,             /* CUDA runtime failure                   */
    RT3D_ERR_NCCL = 5,             /* collective failure (multi-GPU)         */
    RT3D_ERR_UNSUPPORTED = 6,      /* input outside what the device path handles */
    RT3D_ERR_NO_DEVICE = 7         /* no CUDA device: there is no CPU fallback */
} rt3d_status;

/* Point flags, reference cloud.hpp:12-16. */
#define RT3D_FLAG_ISOLATED 1u
#define RT3D_FLAG_OUT_OF_GATE 2u
#define RT3D_FLAG_DEGENERATE 4u

/* splidar::Event (cube.hpp:16-20): one active bin. */
typedef struct rt3d_event {
    uint32_t bin;
    uint32_t count;
} rt3d_event;

/* splidar::Point (cloud.hpp:18-25) with Vec3 = three doubles.  64 bytes, the
 * same layout as the drop-in header's Point, so clouds cross without copies. */
typedef struct rt3d_point {
    double x, y, z;       /* world metres */
    double intensity;     /* r >= 0 */
    int32_t i, j;         /* home coarse pixel */
    int32_t fi, fj;       /* fine transverse index */
    double t;             /* depth, bin units */
    uint8_t flags;
    uint8_t pad_[7];
} rt3d_point;

/* splidar::Irf (sensor.hpp:21-126).  `samples` are the NORMALISED samples
 * exactly as Irf::samples() returns them (the constructor's rescale,
 * sensor.hpp:33-37, happens on the host); slopes are derived on upload with
 * the reference's expression (sensor.hpp:38-40). */
typedef struct rt3d_irf {
    double tau_min;
    double dtau;
    const double* samples;
    uint64_t n_samples;
} rt3d_irf;

/* splidar::SensorModel (sensor.hpp:131-170). */
typedef struct rt3d_sensor {
    int32_t n_rows, n_cols, n_bins, superres;
    double pixel_pitch;    /* metres per fine pixel */
    double bin_resolution; /* metres per bin */
    rt3d_irf irf_shared;
    const rt3d_irf* irf_per_pixel; /* NULL, or n_rows*n_cols row-major */
    const double* gain;            /* n_rows*n_cols */
    const uint8_t* dead;           /* n_rows*n_cols, nonzero = dead */
} rt3d_sensor;

/* splidar::PhotonCube (cube.hpp:24-115), CSR. */
typedef struct rt3d_cube {
    int32_t n_rows, n_cols, n_bins, pad_;
    double bin_width_s;
    const uint64_t* offsets; /* n_rows*n_cols + 1 */
    const rt3d_event* events;
    uint64_t n_events;
} rt3d_cube;

/* splidar::SceneState (likelihood.hpp:20-62) as a host view. */
typedef struct rt3d_state_view {
    const rt3d_point* points;
    uint64_t n_points;
    const double* background;       /* n_rows*n_cols */
    const uint32_t* bucket_offsets; /* n_rows*n_cols + 1 */
    const uint32_t* bucket_points;  /* n_points */
} rt3d_state_view;

/* splidar::InitParams (reconstruct.hpp:25-35). */
typedef struct rt3d_init_params {
    int32_t max_returns;
    int32_t min_separation;
    double peak_threshold;
} rt3d_init_params;

/* splidar::ApssParams (denoise.hpp:24-45). */
typedef struct rt3d_apss_params {
    double kernel_radius;
    double sphere_degeneracy_eps;
    int32_t min_neighbors;
    int32_t pad_;
} rt3d_apss_params;

/* splidar::ReconConfig (reconstruct.hpp:56-107).  step_*_auto != 0 is
 * StepSize "auto" (reconstruct.hpp:39-52); otherwise step_* is the value. */
typedef struct rt3d_recon_config {
    int32_t max_iters;
    int32_t knn_k;
    double stop_tol;
    int32_t step_t_auto, step_r_auto, step_b_auto;
    int32_t background_mode; /* 0 identity, 1 fft (reconstruct.hpp:54) */
    double step_t, step_r, step_b;
    double backtrack_beta;
    rt3d_apss_params apss;
    double r_min;
    double fft_cutoff;
    rt3d_init_params init;
} rt3d_recon_config;

/* splidar::detail::Peak (reconstruct.hpp:111-115). */
typedef struct rt3d_peak {
    double t;
    double response;
    double mass;
} rt3d_peak;

/* splidar::BlockDiagnostics / StepDiagnostics (reconstruct.hpp:251-264). */
typedef struct rt3d_block_diag {
    double step_used;
    double nll_after_grad;
    double nll_after_denoise;
    int32_t backtracks;
    int32_t pad_;
} rt3d_block_diag;

typedef struct rt3d_step_diag {
    double nll_before;
    double nll_after;
    uint64_t points_before;
    uint64_t points_after;
    rt3d_block_diag depth, intensity, background;
} rt3d_step_diag;

/* splidar::ReconReport scalars (reconstruct.hpp:437-447).  seconds are the
 * device time of the frame (CUDA events), split init / iterate. */
typedef struct rt3d_report {
    int32_t iterations;
    int32_t pad_;
    uint64_t points;
    double init_nll;
    double final_nll;
    double init_seconds;
    double iterate_seconds;
    double total_seconds;
} rt3d_report;

/* EvalResult (eval.hpp:20-28) */
typedef struct rt3d_eval {
    double recall;
    double false_point_rate;
    double depth_rmse;
    double intensity_mae;
    uint64_t n_truth;
    uint64_t n_est;
    uint64_t n_matched;
} rt3d_eval;

typedef struct rt3d_session rt3d_session;

/* ---- library / session ------------------------------------------------ */
int rt3d_abi_version(void);
const char* rt3d_last_error(void);
int rt3d_device_count(void);
rt3d_status rt3d_session_create(int device, rt3d_session** out);
rt3d_status rt3d_session_destroy(rt3d_session* s);
rt3d_status rt3d_session_synchronize(rt3d_session* s);
/* Size the session's cooperative grids so that n_sessions sessions can run
 * frames concurrently on the device (one per stream, e.g. alternate frames
 * of a video): each gets 1/n of the co-resident stage blocks.  Default 1. */
rt3d_status rt3d_session_set_sharing(rt3d_session* s, int n_sessions);
/* Device-side ordering, no host wait: the work queued on s from now on starts
 * after the work queued so far on prior (an event on prior's stream).  With
 * two groups of full-grid sessions alternating batches, one group's uploads
 * and downloads overlap the other group's frames while the frames themselves
 * run one after another. */
rt3d_status rt3d_session_after(rt3d_session* s, rt3d_session* prior);
/* The session's CUDA stream (a cudaStream_t), for callers that time the
 * stream-ordered entry points with their own CUDA events. */
void* rt3d_session_stream(rt3d_session* s);
/* Phase timer: when enabled, the frame kernel stamps (phase id,
 * %globaltimer ns) after every grid barrier; rt3d_profile_copy reads the
 * pairs of the last launch.  Off by default (bench.py's breakdown only). */
rt3d_status rt3d_session_profile(rt3d_session* s, int enable);
rt3d_status rt3d_profile_copy(rt3d_session* s, uint64_t* pairs, uint32_t cap, uint32_t* n);
/* Measured FP64 vector throughput of the session's device (DFMA chains,
 * best of 5, TFLOP/s): the roof the bench reports FP64-bound kernels against. */
rt3d_status rt3d_measure_fp64_peak(rt3d_session* s, double* tflops);
/* Kernel-class timing: with it enabled every launch of a frame is bracketed
 * by CUDA events recorded on the session stream; rt3d_kernel_times
 * synchronizes and returns the summed milliseconds and launch counts per
 * class since the last rt3d_session_time_kernels call. */
enum {
    RT3D_KC_STAGE_FIRST = 0,     /* init peaks/spawn + first sweeps          */
    RT3D_KC_STAGE_DEPTH = 1,     /* depth block: grad/curv + backtracking    */
    RT3D_KC_APSS = 2,            /* APSS ball moments (denoise.hpp:159-195)  */
    RT3D_KC_STAGE_INTENSITY = 3, /* intensity block                          */
    RT3D_KC_KNN = 4,             /* kNN intensity filter (denoise.hpp:223)   */
    RT3D_KC_STAGE_TAIL = 5,      /* prune, background block, stop rule       */
    RT3D_KC_APSS_FIT = 6,        /* APSS sphere fit + projection + pinning   */
    RT3D_KC_ITER = 7,            /* a whole PALM iteration in one launch     */
    RT3D_KERNEL_CLASSES = 8
};
rt3d_status rt3d_session_time_kernels(rt3d_session* s, int enable);
/* Debug aid (RT3D_DEBUG set at session creation): mapped host memory with
 * per-block progress records and fault records; NULL otherwise. */
void* rt3d_debug_buffer(rt3d_session* s);
rt3d_status rt3d_kernel_times(rt3d_session* s, double* ms, uint64_t* launches);
/* Frames replay cached CUDA graphs (keyed by the launch's frame parameters:
 * buffers, configuration and sweep layout, not the cube's contents): the
 * graphs captured and the graph launches made by this session so far. */
rt3d_status rt3d_graph_counts(rt3d_session* s, uint64_t* captures, uint64_t* launches);

/* Upload the sensor (IRF tables, gain, dead mask) and the photon cube.  They
 * stay resident until replaced.  Validation follows SensorModel's ctor
 * (sensor.hpp:138-148) and PhotonCube::validate (cube.hpp:84-112); the cube's
 * per-pixel checks run on the device after the upload, so a cube rejected
 * there (RT3D_ERR_FORMAT "... at pixel p") leaves the session without one. */
rt3d_status rt3d_set_sensor(rt3d_session* s, const rt3d_sensor* sensor);
rt3d_status rt3d_set_cube(rt3d_session* s, const rt3d_cube* cube);
/* decode_cube / read_cube (io.hpp:116-150) from an SPCB byte buffer straight
 * into the session's device CSR (the file's bytes, e.g. read or mmapped by the
 * caller).  Same errors as the reference (RT3D_ERR_FORMAT with its messages). */
rt3d_status rt3d_set_cube_spcb(rt3d_session* s, const void* bytes, uint64_t n_bytes);

/* ---- hot path ----------------------------------------------------------- */
/* splidar::reconstruct (reconstruct.hpp:457-489): matched-filter init + PALM
 * iterations, one persistent device kernel per frame, stream-ordered on the
 * session stream (returns before the frame finishes). */
rt3d_status rt3d_reconstruct(rt3d_session* s, const rt3d_recon_config* cfg);
rt3d_status rt3d_report_info(rt3d_session* s, rt3d_report* out);
/* A batch of frames: reconstruct (reconstruct.hpp:457-489) on each of the n
 * (<= 32) sessions' resident cubes, all in one launch sequence on sessions[0]'s
 * stream (a frame axis in every kernel's grid; video streams).
 * Sessions share the device and the configuration; each session's report and
 * state then read exactly as after rt3d_reconstruct on that session.
 * RT3D_ERR_UNSUPPORTED when the cubes need different sweep layouts. */
rt3d_status rt3d_reconstruct_batch(rt3d_session* const* sessions, int32_t n,
                                   const rt3d_recon_config* cfg);
/* Row bands of ONE large frame: n in {1,2,4,8,16,32}
 * sessions holding the same sensor and cube; session k reconstructs the
 * pixels of node k at depth log2(n) of parallel::pairwise_sum's tree
 * (parallel.hpp:52-61; whole rows), reading its neighbours' halo rows before
 * APSS and kNN (reconstruct.hpp:352-397) and combining the sweep sums over all
 * bands with the reference's tree, so the frame equals rt3d_reconstruct's bit
 * for bit.  Afterwards rt3d_state_size / rt3d_state_copy of session k give
 * its own points (the frame's cloud = the bands' clouds in order) and the
 * background of its pixels rt3d_band_pixels(). */
rt3d_status rt3d_reconstruct_bands(rt3d_session* const* sessions, int32_t n,
                                   const rt3d_recon_config* cfg);
rt3d_status rt3d_band_pixels(rt3d_session* s, uint32_t* pixel_begin, uint32_t* pixel_end);
/* The band plan (host only, no device): band k's pixels [begin[k], end[k])
 * and the halo rows every band reads on either side; RT3D_ERR_UNSUPPORTED
 * when the bands are not whole rows at least halo_rows tall. */
rt3d_status rt3d_band_plan(uint32_t n_rows, uint32_t n_cols, int32_t superres, double pixel_pitch,
                           double apss_radius, int32_t n, uint32_t* begin, uint32_t* end,
                           uint32_t* halo_rows);

/* Pipelined frames (a video stream through one session):
 * rt3d_frame_submit validates `cube`, copies it (pinned host memory avoids a
 * staging copy) on the session's copy stream into one of two device slots
 * and enqueues reconstruct (reconstruct.hpp:457-489) plus an end-of-frame copy
 * of the cloud and background into a result slot; it returns at once with a
 * ticket.  rt3d_frame_collect waits for that frame and copies its cloud,
 * background and report out; *n_points receives the count.  A cloud of more
 * than cap points returns RT3D_ERR_OUT_OF_RANGE and copies nothing: the frame
 * stays in flight and can be collected again with a larger buffer.  At most
 * two frames are in flight; `cube` must stay valid until its frame is
 * collected. */
rt3d_status rt3d_frame_submit(rt3d_session* s, const rt3d_cube* cube, const rt3d_recon_config* cfg,
                              uint64_t* ticket);
rt3d_status rt3d_frame_collect(rt3d_session* s, uint64_t ticket, rt3d_point* points, uint64_t cap,
                               uint64_t* n_points, double* background, rt3d_report* info);
/* nll_trace holds iterations+1 values, steps holds iterations entries. */
rt3d_status rt3d_report_copy(rt3d_session* s, double* nll_trace, rt3d_step_diag* steps);

/* Current device SceneState (after init / palm_step / reconstruct /
 * baseline): point count, then copy out (points in cloud order, background
 * n_rows*n_cols).  Either output pointer may be NULL. */
rt3d_status rt3d_state_size(rt3d_session* s, uint64_t* n_points);
rt3d_status rt3d_state_copy(rt3d_session* s, rt3d_point* points, double* background);

/* ---- operators the reference's own tests call -------------------------- */
/* detail::matched_filter_peaks (reconstruct.hpp:120-189) on one pixel's
 * events.  `out` must hold k peaks; *n_out receives the count. */
rt3d_status rt3d_matched_filter_peaks(rt3d_session* s, const rt3d_event* events, uint64_t n_events,
                                      const rt3d_irf* irf, int32_t n_bins, int32_t k,
                                      double threshold, int32_t min_sep, rt3d_peak* out,
                                      int32_t* n_out);
/* init_matched_filter (reconstruct.hpp:197-249) -> session state. */
rt3d_status rt3d_init_matched_filter(rt3d_session* s, const rt3d_init_params* params);
/* baseline_xcorr (eval.hpp:91-126) -> session state (background = floor). */
rt3d_status rt3d_baseline_xcorr(rt3d_session* s);
/* Upload a host SceneState as the session state (used by palm_step etc.). */
rt3d_status rt3d_state_upload(rt3d_session* s, const rt3d_state_view* state);

/* Likelihood sweeps on the session state (likelihood.hpp:136-333). */
rt3d_status rt3d_nll(rt3d_session* s, double* out);
rt3d_status rt3d_grad_depth(rt3d_session* s, double* value, uint8_t* out_of_gate);
rt3d_status rt3d_grad_intensity(rt3d_session* s, double* out);
rt3d_status rt3d_grad_background(rt3d_session* s, double* out);
rt3d_status rt3d_block_curvatures(rt3d_session* s, double* depth, double* intensity,
                                  double* background);

/* palm_step (reconstruct.hpp:300-435) on the session state, in place. */
rt3d_status rt3d_palm_step(rt3d_session* s, const rt3d_recon_config* cfg, rt3d_step_diag* diag);

/* Point-cloud denoisers on arbitrary clouds (denoise.hpp:159-248).  The
 * neighbour set is SpatialIndex::query / query_knn over `index_cloud`
 * (spatial_index.hpp:31-62) with cell size `index_cell`. */
rt3d_status rt3d_apss_project(rt3d_session* s, const rt3d_point* cloud, uint64_t n,
                              const rt3d_apss_params* params, const rt3d_point* index_cloud,
                              uint64_t n_index, double index_cell, rt3d_point* out);
rt3d_status rt3d_knn_intensity_filter(rt3d_session* s, const rt3d_point* cloud, uint64_t n,
                                      int32_t k, const rt3d_point* index_cloud, uint64_t n_index,
                                      double index_cell, double radius, rt3d_point* out);
rt3d_status rt3d_prune(rt3d_session* s, const rt3d_point* cloud, uint64_t n, double r_min,
                       rt3d_point* out, uint64_t* n_out);

/* fft_lowpass_filter / fft_background_denoise (denoise.hpp:267-319). */
rt3d_status rt3d_fft_lowpass_filter(rt3d_session* s, const double* img, int32_t rows,
                                    int32_t cols, double cutoff, int32_t clamp_nonneg,
                                    double* out);

/* evaluate (eval.hpp:33-87): points grouped into transverse columns of the
 * given pitch (floor(x / pitch), floor(y / pitch)), matched one-to-one per
 * column greedily by (|dz|, truth index, estimate index) within tau.  Columns
 * and matches on the device; the error sums in the reference's order on the
 * host, so the result is bit-identical. */
rt3d_status rt3d_evaluate(rt3d_session* s, const rt3d_point* est, uint64_t n_est,
                          const rt3d_point* truth, uint64_t n_truth, double tau, double pitch,
                          rt3d_eval* out);

/* ---- forward simulator (device) ----------------------------------------- */
/* simulate_cube's photon sampling (simulate.hpp:181-205: rate_profile,
 * likelihood.hpp:80-95, and CounterRng::next_poisson keyed by (seed, pixel,
 * bin, stream), rng.hpp:11-98) on the device, into the session's resident
 * cube (as if rt3d_set_cube had been called).  `truth` is the scene's truth
 * cloud after the reflectivity scaling (simulate.hpp:145-159; i, j, t and
 * intensity are read), `background` the true background per pixel and bin
 * (simulate.hpp:172-177).  Uses the session's sensor (IRF, gain, dead).
 * photons[2] receives {signal, background} photon totals.  Sampled events
 * must stay below 2^32. */
rt3d_status rt3d_simulate_cube(rt3d_session* s, const rt3d_point* truth, uint64_t n_truth,
                               const double* background, uint64_t seed, uint64_t* n_events,
                               uint64_t* photons);
/* The session's resident cube (CSR, cube.hpp:24-40) back to the host:
 * offsets u64[rows*cols+1], events[n_events] (n_events from
 * rt3d_simulate_cube or the cube that was set).  Either pointer may be NULL. */
rt3d_status rt3d_cube_copy(rt3d_session* s, uint64_t* offsets, rt3d_event* events);

/* ---- output formats (host only, no session) ---------------------------- */
/* encode_ply (io.hpp:162-179): ASCII PLY of a cloud (e.g. from
 * rt3d_state_copy / rt3d_frame_collect), byte-identical to the reference's;
 * has_pixel_pitch != 0 adds the "comment pixel_pitch" line.  Two calls: with
 * buf NULL (or cap too small) only *n_bytes is set. */
rt3d_status rt3d_encode_ply(const rt3d_point* points, uint64_t n, int32_t has_pixel_pitch,
                            double pixel_pitch, char* buf, uint64_t cap, uint64_t* n_bytes);
/* The background CSV of `splidar reconstruct --background-out`
 * (tools/splidar_main.cpp:204-212): rows lines of cols "%.9g" values. */
rt3d_status rt3d_encode_background_csv(const double* background, int32_t rows, int32_t cols,
                                       char* buf, uint64_t cap, uint64_t* n_bytes);

#ifdef __cplusplus
}
#endif

#endif /* RT3D_H */
