/*
 * rt3d_scene.h — synthetic photon cubes for benchmarks and tests
 * (libscene.so, host C).  A restatement of the reference's forward simulator,
 * simulate.hpp:20-223 with CounterRng (rng.hpp:11-98): the same scene
 * description, the same counter-based RNG keyed by (seed, pixel, bin,
 * stream), so the cubes are bit-identical to the reference's simulate_cube
 * (checked in tests/test_scene.py) and reproducible under any threading.
 * It is the input side of the path, not the path itself.
 */
#ifndef RT3D_SCENE_H
#define RT3D_SCENE_H

#include <stdint.h>

#include "rt3d.h"

#ifdef __cplusplus
extern "C" {
#endif

/* SurfaceSpec (simulate.hpp:20-42) */
typedef struct rt3d_surface {
    int32_t kind; /* 0 plane, 1 bump */
    int32_t checker_period;
    double depth_m, slope_x, slope_y;
    double bump_amp, bump_cx, bump_cy, bump_width;
    double reflectivity, checker_contrast;
    int32_t region[4]; /* x0,y0,x1,y1 on the fine grid; x1 < 0 = full grid */
    int32_t n_holes;
    int32_t pad_;
    const int32_t* holes; /* n_holes * 4 */
} rt3d_surface;

/* SceneSpec (simulate.hpp:47-65) */
typedef struct rt3d_scene_spec {
    int32_t rows, cols, bins, superres;
    double bin_resolution_m, pixel_pitch_m, irf_sigma_bins, irf_support_sigmas;
    double ambient_per_bin, target_ppp, target_sbr;
    int32_t n_surfaces, n_dead;
    const rt3d_surface* surfaces;
    const int32_t* dead_pixels; /* n_dead * 2 */
} rt3d_scene_spec;

typedef struct rt3d_scene rt3d_scene;

/* simulate_cube (simulate.hpp:139-223) with `threads` workers (0 = all).
 * Returns 0, or -1 with a message in rt3d_scene_error(). */
int rt3d_scene_simulate(const rt3d_scene_spec* spec, uint64_t seed, int threads,
                        rt3d_scene** out);
const char* rt3d_scene_error(void);
/* sizes: events, truth points, irf samples */
void rt3d_scene_sizes(const rt3d_scene* s, uint64_t* n_events, uint64_t* n_truth,
                      uint64_t* n_irf);
/* copies; any pointer may be NULL.  meta = {tau_min, dtau, bin_width_s,
 * signal_photons, background_photons}. */
void rt3d_scene_copy(const rt3d_scene* s, uint64_t* offsets, rt3d_event* events,
                     double* irf_samples, rt3d_point* truth, uint8_t* dead, double* meta);
/* background_truth (simulate.hpp:172-177): ambient + hot pixels, f64[rows*cols] */
void rt3d_scene_background(const rt3d_scene* s, double* out);
void rt3d_scene_free(rt3d_scene* s);

#ifdef __cplusplus
}
#endif

#endif
