/*
 * scene.c — libscene.so: synthetic photon cubes (scenegen/rt3d_scene.h).
 * Restates the reference's forward simulator (simulate.hpp:139-223) and its
 * counter-based RNG (rng.hpp:11-98) so that benchmark inputs of the named
 * shapes can be made on the GPU box, bit-identical to the reference's cubes.
 * Compiled without FMA contraction, like the reference's Release build.
 */
#include "rt3d_scene.h"

#include <math.h>
#include <pthread.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <unistd.h>

static _Thread_local char g_err[256];

static int fail(const char* msg) {
    snprintf(g_err, sizeof g_err, "%s", msg);
    return -1;
}
const char* rt3d_scene_error(void) { return g_err; }

/* ---- CounterRng, rng.hpp:11-98 ---------------------------------------- */
#define KGAMMA 0x9E3779B97F4A7C15ull
static inline uint64_t mix64(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}
typedef struct {
    uint64_t base, counter;
} crng;
static inline crng crng_make(uint64_t a, uint64_t b, uint64_t c, uint64_t d) {
    crng r;
    r.base = mix64(a + KGAMMA);
    r.base = mix64(r.base ^ mix64(b + 2 * KGAMMA));
    r.base = mix64(r.base ^ mix64(c + 3 * KGAMMA));
    r.base = mix64(r.base ^ mix64(d + 5 * KGAMMA));
    r.counter = 0;
    return r;
}
static inline uint64_t crng_u64(crng* r) { return mix64(r->base + (++r->counter) * KGAMMA); }
static inline double crng_unit(crng* r) {
    return ((double)(crng_u64(r) >> 11) + 0.5) * 0x1.0p-53;
}
static uint32_t poisson_inversion(crng* r, double lambda) {
    const double limit = exp(-lambda);
    uint32_t k = 0;
    double p = 1.0;
    do {
        ++k;
        p *= crng_unit(r);
    } while (p > limit);
    return k - 1;
}
static uint32_t poisson_ptrd(crng* r, double lambda) {
    const double slam = sqrt(lambda);
    const double loglam = log(lambda);
    const double b = 0.931 + 2.53 * slam;
    const double a = -0.059 + 0.02483 * b;
    const double inv_alpha = 1.1239 + 1.1328 / (b - 3.4);
    const double vr = 0.9277 - 3.6224 / (b - 2.0);
    for (;;) {
        double u;
        double v = crng_unit(r);
        if (v <= 0.86 * vr) {
            u = v / vr - 0.43;
            return (uint32_t)floor((2.0 * a / (0.5 - fabs(u)) + b) * u + lambda + 0.445);
        }
        if (v >= vr) {
            u = crng_unit(r) - 0.5;
        } else {
            u = v / vr - 0.93;
            u = (u < 0 ? -0.5 : 0.5) - u;
            v = crng_unit(r) * vr;
        }
        const double us = 0.5 - fabs(u);
        if (us < 0.013 && v > us) continue;
        const double kf = floor((2.0 * a / us + b) * u + lambda + 0.445);
        v = v * inv_alpha / (a / (us * us) + b);
        if (kf >= 10.0) {
            const double log_sqrt_2pi = 0.91893853320467267;
            if (log(v * slam) <= (kf + 0.5) * log(lambda / kf) - lambda - log_sqrt_2pi + kf -
                                      (1.0 / 12.0 - 1.0 / (360.0 * kf * kf)) / kf)
                return (uint32_t)kf;
        } else if (kf >= 0.0) {
            if (log(v) <= kf * loglam - lambda - lgamma(kf + 1.0)) return (uint32_t)kf;
        }
    }
}
static inline uint32_t next_poisson(crng* r, double lambda) {
    if (!(lambda > 0.0)) return 0;
    if (lambda < 10.0) return poisson_inversion(r, lambda);
    return poisson_ptrd(r, lambda);
}

/* ---- Irf::gaussian + interpolation, sensor.hpp:26-98 --------------------- */
typedef struct {
    double tau_min, dtau, tau_max;
    int n;
    double* s;
} irf_t;

static int irf_gaussian(double sigma, double nsig, double dtau, irf_t* f) {
    if (sigma <= 0.0) return -1;
    double half = nsig * sigma;
    int n = (int)ceil(2.0 * half / dtau);
    n = (n < 2 ? 2 : n) + 1;
    f->s = (double*)malloc(sizeof(double) * n);
    for (int k = 0; k < n; ++k) {
        double tau = -half + k * dtau;
        f->s[k] = exp(-0.5 * tau * tau / (sigma * sigma));
    }
    f->s[0] = 0.0;
    f->s[n - 1] = 0.0;
    double mass = 0.0;
    for (int k = 0; k < n; ++k) mass += f->s[k];
    mass *= dtau;
    if (mass <= 0.0) return -1;
    for (int k = 0; k < n; ++k) f->s[k] /= mass;
    f->tau_min = -half;
    f->dtau = dtau;
    f->n = n;
    f->tau_max = f->tau_min + dtau * (double)(n - 1);
    return 0;
}
static inline double irf_value(const irf_t* f, double tau) {
    if (tau < f->tau_min || tau > f->tau_max) return 0.0;
    double x = (tau - f->tau_min) / f->dtau;
    uint64_t k = (uint64_t)x;
    if (k > (uint64_t)(f->n - 2)) k = f->n - 2;
    double fr = x - (double)k;
    return f->s[k] + fr * (f->s[k + 1] - f->s[k]);
}
static inline void irf_support(const irf_t* f, double t, int n_bins, int* lo, int* hi) {
    int a = (int)ceil(t + f->tau_min), b = (int)floor(t + f->tau_max);
    *lo = a < 0 ? 0 : a;
    *hi = b > n_bins - 1 ? n_bins - 1 : b;
}
static double irf_mass_in_gate(const irf_t* f, double t, int n_bins) {
    int lo, hi;
    irf_support(f, t, n_bins, &lo, &hi);
    double m = 0.0;
    for (int b = lo; b <= hi; ++b) m += irf_value(f, (double)b - t);
    return m;
}

/* ---- scene ------------------------------------------------------------- */
struct rt3d_scene {
    int rows, cols, bins, s;
    irf_t irf;
    uint64_t* offsets;
    rt3d_event* events;
    uint64_t n_events;
    rt3d_point* truth;
    uint64_t n_truth;
    uint8_t* dead;
    double bin_width_s;
    uint64_t sig, bgp;
    double* bg; /* background_truth, simulate.hpp:172-177 */
};

/* SurfaceSpec::depth_at, simulate.hpp:37-41 */
static double depth_at(const rt3d_surface* s, double x, double y) {
    if (s->kind == 0) return s->depth_m + s->slope_x * x + s->slope_y * y;
    double dx = x - s->bump_cx, dy = y - s->bump_cy;
    return s->depth_m +
           s->bump_amp * exp(-(dx * dx + dy * dy) / (2.0 * s->bump_width * s->bump_width));
}

typedef struct {
    const rt3d_scene_spec* spec;
    rt3d_scene* sc;
    const double* bgimg;
    const uint32_t* boff;
    const uint32_t* bpts;
    uint64_t seed;
    size_t p0, p1;
    rt3d_event** ev;
    uint32_t* nev;
    uint64_t sig, bgp;
} job_t;

static void* sim_worker(void* arg) {
    job_t* J = (job_t*)arg;
    rt3d_scene* sc = J->sc;
    const int T = sc->bins;
    double* lam = (double*)malloc(sizeof(double) * T);
    for (size_t p = J->p0; p < J->p1; ++p) {
        J->nev[p] = 0;
        J->ev[p] = NULL;
        double g = sc->dead[p] ? 0.0 : 1.0; /* gain 1 (build_sensor) */
        if (g == 0.0) continue;
        /* rate_profile, likelihood.hpp:80-95 */
        double bg = g * J->bgimg[p];
        for (int t = 0; t < T; ++t) lam[t] = bg;
        for (uint32_t k = J->boff[p]; k < J->boff[p + 1]; ++k) {
            const rt3d_point* pt = &sc->truth[J->bpts[k]];
            int lo, hi;
            irf_support(&sc->irf, pt->t, T, &lo, &hi);
            for (int b = lo; b <= hi; ++b)
                lam[b] += g * pt->intensity * irf_value(&sc->irf, (double)b - pt->t);
        }
        const double lam_bg = g * J->bgimg[p];
        uint32_t cap = 0, n = 0;
        rt3d_event* out = NULL;
        for (int t = 0; t < T; ++t) {
            double d = lam[t] - lam_bg;
            double lam_sig = (0.0 < d) ? d : 0.0;
            crng rs = crng_make(J->seed, p, (uint64_t)t, 1);
            crng rb = crng_make(J->seed, p, (uint64_t)t, 2);
            uint32_t zs = lam_sig > 0.0 ? next_poisson(&rs, lam_sig) : 0;
            uint32_t zb = lam_bg > 0.0 ? next_poisson(&rb, lam_bg) : 0;
            J->sig += zs;
            J->bgp += zb;
            if (zs + zb > 0) {
                if (n == cap) {
                    cap = cap ? 2 * cap : 16;
                    out = (rt3d_event*)realloc(out, sizeof(rt3d_event) * cap);
                }
                out[n].bin = (uint32_t)t;
                out[n].count = zs + zb;
                ++n;
            }
        }
        J->ev[p] = out;
        J->nev[p] = n;
    }
    free(lam);
    return NULL;
}

int rt3d_scene_simulate(const rt3d_scene_spec* spec, uint64_t seed, int threads,
                        rt3d_scene** out) {
    *out = NULL;
    if (spec->rows <= 0 || spec->cols <= 0 || spec->bins <= 0 || spec->superres < 1)
        return fail("scene: bad grid dimensions");
    rt3d_scene* sc = (rt3d_scene*)calloc(1, sizeof(rt3d_scene));
    sc->rows = spec->rows;
    sc->cols = spec->cols;
    sc->bins = spec->bins;
    sc->s = spec->superres;
    if (irf_gaussian(spec->irf_sigma_bins, spec->irf_support_sigmas, 0.25, &sc->irf)) {
        free(sc);
        return fail("Irf: sigma must be positive");
    }
    const size_t npix = (size_t)spec->rows * spec->cols;
    sc->dead = (uint8_t*)calloc(npix, 1);
    for (int k = 0; k < spec->n_dead; ++k) {
        int i = spec->dead_pixels[2 * k], j = spec->dead_pixels[2 * k + 1];
        if (i < 0 || i >= spec->rows || j < 0 || j >= spec->cols) {
            rt3d_scene_free(sc);
            return fail("scene: dead pixel out of bounds");
        }
        sc->dead[(size_t)i * spec->cols + j] = 1;
    }
    const int frows = spec->rows * spec->superres, fcols = spec->cols * spec->superres;
    const double pitch = spec->pixel_pitch_m, bres = spec->bin_resolution_m;

    /* build_truth, simulate.hpp:197-230 */
    size_t cap = 1024;
    sc->truth = (rt3d_point*)malloc(sizeof(rt3d_point) * cap);
    for (int q = 0; q < spec->n_surfaces; ++q) {
        const rt3d_surface* sf = &spec->surfaces[q];
        int x0 = sf->region[0], y0 = sf->region[1], x1 = sf->region[2], y1 = sf->region[3];
        if (x1 < 0) {
            x0 = 0;
            y0 = 0;
            x1 = frows;
            y1 = fcols;
        }
        for (int fi = x0; fi < x1; ++fi)
            for (int fj = y0; fj < y1; ++fj) {
                int holed = 0;
                for (int h = 0; h < sf->n_holes; ++h) {
                    const int32_t* r = sf->holes + 4 * h;
                    if (fi >= r[0] && fi < r[2] && fj >= r[1] && fj < r[3]) {
                        holed = 1;
                        break;
                    }
                }
                if (holed) continue;
                double x = (fi + 0.5) * pitch, y = (fj + 0.5) * pitch;
                double z = depth_at(sf, x, y);
                rt3d_point p;
                memset(&p, 0, sizeof p);
                p.x = x;
                p.y = y;
                p.z = z;
                p.intensity = sf->reflectivity;
                if (sf->checker_contrast != 0.0) {
                    int par = (fi / sf->checker_period + fj / sf->checker_period) & 1;
                    p.intensity *= 1.0 + (par ? sf->checker_contrast : -sf->checker_contrast);
                }
                /* map_world_to_lidar, sensor.hpp:181-197 */
                double fx = floor(p.x / pitch), fy = floor(p.y / pitch);
                if (fx < 0 || fx >= frows || fy < 0 || fy >= fcols) {
                    rt3d_scene_free(sc);
                    return fail("scene: surface leaves the gate: x/y outside frustum");
                }
                p.t = p.z / bres;
                if (p.t < 0 || p.t >= spec->bins) {
                    rt3d_scene_free(sc);
                    return fail("scene: surface leaves the gate: z outside depth gate");
                }
                p.fi = (int)fx;
                p.fj = (int)fy;
                p.i = p.fi / spec->superres;
                p.j = p.fj / spec->superres;
                if (sc->n_truth == cap) {
                    cap *= 2;
                    sc->truth = (rt3d_point*)realloc(sc->truth, sizeof(rt3d_point) * cap);
                }
                sc->truth[sc->n_truth++] = p;
            }
    }

    /* reflectivity scaling and ambient level, simulate.hpp:245-278 */
    double total_expected = 0.0;
    for (uint64_t k = 0; k < sc->n_truth; ++k) {
        const rt3d_point* p = &sc->truth[k];
        double g = sc->dead[(size_t)p->i * spec->cols + p->j] ? 0.0 : 1.0;
        total_expected += g * p->intensity * irf_mass_in_gate(&sc->irf, p->t, spec->bins);
    }
    const double n_pix = (double)spec->rows * spec->cols;
    if (spec->target_ppp > 0.0 && total_expected > 0.0) {
        double scale = spec->target_ppp * n_pix / total_expected;
        for (uint64_t k = 0; k < sc->n_truth; ++k) sc->truth[k].intensity *= scale;
        total_expected *= scale;
    }
    double ambient = spec->ambient_per_bin;
    double gain_sum = 0.0;
    for (size_t p = 0; p < npix; ++p) gain_sum += sc->dead[p] ? 0.0 : 1.0;
    if (spec->target_sbr > 0.0) {
        double bg_total = total_expected / spec->target_sbr;
        double den = gain_sum * spec->bins;
        ambient = bg_total / ((den < 1e-300) ? 1e-300 : den);
    }
    if (ambient < 0.0) {
        rt3d_scene_free(sc);
        return fail("scene: negative ambient");
    }
    double* bgimg = (double*)malloc(sizeof(double) * npix);
    for (size_t p = 0; p < npix; ++p) bgimg[p] = ambient;

    /* SceneState buckets, likelihood.hpp:38-55 */
    uint32_t* boff = (uint32_t*)calloc(npix + 1, sizeof(uint32_t));
    uint32_t* bpts = (uint32_t*)malloc(sizeof(uint32_t) * (sc->n_truth ? sc->n_truth : 1));
    for (uint64_t k = 0; k < sc->n_truth; ++k)
        ++boff[(size_t)sc->truth[k].i * spec->cols + sc->truth[k].j + 1];
    for (size_t p = 0; p < npix; ++p) boff[p + 1] += boff[p];
    uint32_t* cur = (uint32_t*)malloc(sizeof(uint32_t) * npix);
    memcpy(cur, boff, sizeof(uint32_t) * npix);
    for (uint64_t k = 0; k < sc->n_truth; ++k)
        bpts[cur[(size_t)sc->truth[k].i * spec->cols + sc->truth[k].j]++] = (uint32_t)k;
    free(cur);

    /* per-pixel Poisson draws, simulate.hpp:286-305 */
    int nt = threads > 0 ? threads : (int)sysconf(_SC_NPROCESSORS_ONLN);
    if (nt < 1) nt = 1;
    if ((size_t)nt > npix) nt = (int)npix;
    rt3d_event** ev = (rt3d_event**)calloc(npix, sizeof(rt3d_event*));
    uint32_t* nev = (uint32_t*)calloc(npix, sizeof(uint32_t));
    job_t* jobs = (job_t*)calloc(nt, sizeof(job_t));
    pthread_t* th = (pthread_t*)calloc(nt, sizeof(pthread_t));
    size_t chunk = (npix + nt - 1) / nt;
    for (int w = 0; w < nt; ++w) {
        job_t* J = &jobs[w];
        J->spec = spec;
        J->sc = sc;
        J->bgimg = bgimg;
        J->boff = boff;
        J->bpts = bpts;
        J->seed = seed;
        J->p0 = w * chunk;
        J->p1 = J->p0 + chunk < npix ? J->p0 + chunk : npix;
        if (J->p0 > npix) J->p0 = npix;
        J->ev = ev;
        J->nev = nev;
        pthread_create(&th[w], NULL, sim_worker, J);
    }
    for (int w = 0; w < nt; ++w) {
        pthread_join(th[w], NULL);
        sc->sig += jobs[w].sig;
        sc->bgp += jobs[w].bgp;
    }
    sc->offsets = (uint64_t*)malloc(sizeof(uint64_t) * (npix + 1));
    sc->offsets[0] = 0;
    for (size_t p = 0; p < npix; ++p) sc->offsets[p + 1] = sc->offsets[p] + nev[p];
    sc->n_events = sc->offsets[npix];
    sc->events = (rt3d_event*)malloc(sizeof(rt3d_event) * (sc->n_events ? sc->n_events : 1));
    for (size_t p = 0; p < npix; ++p) {
        if (nev[p]) memcpy(sc->events + sc->offsets[p], ev[p], sizeof(rt3d_event) * nev[p]);
        free(ev[p]);
    }
    sc->bin_width_s = 2.0 * bres / 299792458.0;
    free(ev);
    free(nev);
    free(jobs);
    free(th);
    sc->bg = bgimg;
    free(boff);
    free(bpts);
    *out = sc;
    return 0;
}

void rt3d_scene_sizes(const rt3d_scene* s, uint64_t* n_events, uint64_t* n_truth,
                      uint64_t* n_irf) {
    if (n_events) *n_events = s->n_events;
    if (n_truth) *n_truth = s->n_truth;
    if (n_irf) *n_irf = (uint64_t)s->irf.n;
}

void rt3d_scene_copy(const rt3d_scene* s, uint64_t* offsets, rt3d_event* events,
                     double* irf_samples, rt3d_point* truth, uint8_t* dead, double* meta) {
    const size_t npix = (size_t)s->rows * s->cols;
    if (offsets) memcpy(offsets, s->offsets, sizeof(uint64_t) * (npix + 1));
    if (events && s->n_events) memcpy(events, s->events, sizeof(rt3d_event) * s->n_events);
    if (irf_samples) memcpy(irf_samples, s->irf.s, sizeof(double) * s->irf.n);
    if (truth && s->n_truth) memcpy(truth, s->truth, sizeof(rt3d_point) * s->n_truth);
    if (dead) memcpy(dead, s->dead, npix);
    if (meta) {
        meta[0] = s->irf.tau_min;
        meta[1] = s->irf.dtau;
        meta[2] = s->bin_width_s;
        meta[3] = (double)s->sig;
        meta[4] = (double)s->bgp;
    }
}

void rt3d_scene_free(rt3d_scene* s) {
    if (!s) return;
    free(s->irf.s);
    free(s->offsets);
    free(s->events);
    free(s->truth);
    free(s->dead);
    free(s->bg);
    free(s);
}

void rt3d_scene_background(const rt3d_scene* s, double* out) {
    if (s->bg) memcpy(out, s->bg, sizeof(double) * (size_t)s->rows * s->cols);
}
