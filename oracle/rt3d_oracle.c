/*
 * rt3d_oracle.c — TEST INFRASTRUCTURE ONLY (see rt3d_oracle.h).
 *
 * Plain-C restatement of the reference RT3D path.  Each function names the
 * reference file:line (relative to /root/reference/proj/include/splidar) it
 * restates.  Expressions keep the reference's operand order; compile with
 * -ffp-contract=off and no -march so no FMA is formed (the reference's
 * Release build, CMakeLists.txt:6-8,18, has none either).
 *
 * Third-party arithmetic: the reference calls Eigen's GeneralizedEigenSolver
 * (QZ) and SelfAdjointEigenSolver inside APSS (denoise.hpp:86-87,196) and
 * FFTW (denoise.hpp:278-306).  Neither library is present here.  Their
 * published contracts are restated instead:
 *  - pencil (M, N): the reference keeps the smallest eigenvalue eta >=
 *    -1e-9 tr(M) whose eigenvector lies in the feasible cone u'Nu > 0
 *    (denoise.hpp:92-112).  For symmetric PSD M and the Pratt matrix N
 *    (inertia 4+,1-) that is the smallest non-negative eigenvalue, which is
 *    also sup{ sigma >= 0 : M - sigma N positive definite }.  It is found by
 *    bisection on a division-free definiteness test (pd5), and its
 *    eigenvector by inverse iteration on an LDL' factor of the last definite
 *    shift (pratt_smallest below);
 *  - only the eigenVALUES of the 3x3 covariance decide anything
 *    (denoise.hpp:197-203; the eigenvector only orients the sign of u, and the
 *    projection is invariant under u -> -u), computed by cyclic Jacobi;
 *  - FFTW's unnormalised forward/backward DFT is evaluated directly.
 */
#include "rt3d_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

#ifndef M_PI
#define M_PI 3.14159265358979323846
#endif

static const double kBackgroundFloor = 1e-6; /* reconstruct.hpp:23 */
static const int kMaxBacktracks = 30;        /* reconstruct.hpp:268 */

/* ------------------------------------------------------------------------ */
/* std:: helpers with the reference's exact semantics                        */
/* ------------------------------------------------------------------------ */
static inline double std_max(double a, double b) { return (a < b) ? b : a; }
static inline double std_min(double a, double b) { return (b < a) ? b : a; }
static inline double std_clamp(double v, double lo, double hi) {
    return (v < lo) ? lo : (hi < v) ? hi : v;
}
static inline int imax(int a, int b) { return a < b ? b : a; }
static inline int imin(int a, int b) { return b < a ? b : a; }

/* ------------------------------------------------------------------------ */
/* Irf (sensor.hpp:21-126)                                                   */
/* ------------------------------------------------------------------------ */
typedef struct irf_t {
    double tau_min, dtau, tau_max;
    uint64_t n;
    const double* s;
    double* d; /* slopes, n-1 */
} irf_t;

static void irf_make(irf_t* o, const rt3d_irf* in) {
    o->tau_min = in->tau_min;
    o->dtau = in->dtau;
    o->n = in->n_samples;
    o->s = in->samples;
    /* tau_max(): tau_min_ + dtau_ * (samples_.size() - 1)   sensor.hpp:63 */
    o->tau_max = in->tau_min + in->dtau * (double)(in->n_samples - 1);
    o->d = (double*)malloc(sizeof(double) * (in->n_samples > 1 ? in->n_samples - 1 : 1));
    /* sensor.hpp:38-40 */
    for (uint64_t k = 0; k + 1 < in->n_samples; ++k)
        o->d[k] = (in->samples[k + 1] - in->samples[k]) / in->dtau;
}
static void irf_free(irf_t* o) { free(o->d); }

/* sensor.hpp:69-75 */
static inline double irf_value(const irf_t* f, double tau) {
    if (tau < f->tau_min || tau > f->tau_max) return 0.0;
    double x = (tau - f->tau_min) / f->dtau;
    uint64_t k = (uint64_t)x;
    if (k > f->n - 2) k = f->n - 2;
    double fr = x - (double)k;
    return f->s[k] + fr * (f->s[k + 1] - f->s[k]);
}
/* sensor.hpp:77-82 */
static inline double irf_deriv(const irf_t* f, double tau) {
    if (tau <= f->tau_min || tau >= f->tau_max) return 0.0;
    double x = (tau - f->tau_min) / f->dtau;
    uint64_t k = (uint64_t)x;
    if (k > f->n - 2) k = f->n - 2;
    return f->d[k];
}
/* sensor.hpp:86-90 */
static inline void irf_support(const irf_t* f, double t, int n_bins, int* lo, int* hi) {
    *lo = imax(0, (int)ceil(t + f->tau_min));
    *hi = imin(n_bins - 1, (int)floor(t + f->tau_max));
}
/* sensor.hpp:93-98 */
static double irf_mass_in_gate(const irf_t* f, double t, int n_bins) {
    int lo, hi;
    irf_support(f, t, n_bins, &lo, &hi);
    double m = 0.0;
    for (int b = lo; b <= hi; ++b) m += irf_value(f, (double)b - t);
    return m;
}

double oracle_irf_value(const rt3d_irf* irf, double tau) {
    irf_t f;
    irf_make(&f, irf);
    double v = irf_value(&f, tau);
    irf_free(&f);
    return v;
}
double oracle_irf_deriv(const rt3d_irf* irf, double tau) {
    irf_t f;
    irf_make(&f, irf);
    double v = irf_deriv(&f, tau);
    irf_free(&f);
    return v;
}
double oracle_irf_mass_in_gate(const rt3d_irf* irf, double t, int n_bins) {
    irf_t f;
    irf_make(&f, irf);
    double v = irf_mass_in_gate(&f, t, n_bins);
    irf_free(&f);
    return v;
}

/* sensor.hpp:26-41 (normalisation part of the ctor) */
int oracle_irf_normalise(double* s, uint64_t n, double dtau) {
    if (dtau <= 0.0 || n < 2) return -1;
    double mass = 0.0;
    for (uint64_t k = 0; k < n; ++k) {
        if (s[k] < 0.0 || !isfinite(s[k])) return -1;
    }
    for (uint64_t k = 0; k < n; ++k) mass += s[k];
    mass *= dtau;
    if (mass <= 0.0) return -1;
    for (uint64_t k = 0; k < n; ++k) s[k] /= mass;
    return 0;
}

/* sensor.hpp:45-57 */
uint64_t oracle_irf_gaussian(double sigma_bins, double n_sigmas, double dtau, double* samples,
                             uint64_t cap, double* tau_min) {
    if (sigma_bins <= 0.0) return 0;
    double half = n_sigmas * sigma_bins;
    int n = imax(2, (int)ceil(2.0 * half / dtau)) + 1;
    if ((uint64_t)n > cap) return 0;
    for (int k = 0; k < n; ++k) {
        double tau = -half + k * dtau;
        samples[k] = exp(-0.5 * tau * tau / (sigma_bins * sigma_bins));
    }
    samples[0] = 0.0;
    samples[n - 1] = 0.0;
    if (oracle_irf_normalise(samples, (uint64_t)n, dtau) != 0) return 0;
    *tau_min = -half;
    return (uint64_t)n;
}

/* ------------------------------------------------------------------------ */
/* parallel.hpp:52-61                                                        */
/* ------------------------------------------------------------------------ */
double oracle_pairwise_sum(const double* v, uint64_t n) {
    if (n == 0) return 0.0;
    if (n <= 8) {
        double s = 0.0;
        for (uint64_t k = 0; k < n; ++k) s += v[k];
        return s;
    }
    uint64_t half = n / 2;
    return oracle_pairwise_sum(v, half) + oracle_pairwise_sum(v + half, n - half);
}

/* ------------------------------------------------------------------------ */
/* Sensor / state                                                            */
/* ------------------------------------------------------------------------ */
typedef struct sensor_t {
    int rows, cols, bins, s;
    double pitch, bres;
    irf_t shared;
    irf_t* pp; /* per pixel or NULL */
    const double* gain;
    const uint8_t* dead;
} sensor_t;

static void sensor_make(sensor_t* o, const rt3d_sensor* in) {
    o->rows = in->n_rows;
    o->cols = in->n_cols;
    o->bins = in->n_bins;
    o->s = in->superres;
    o->pitch = in->pixel_pitch;
    o->bres = in->bin_resolution;
    irf_make(&o->shared, &in->irf_shared);
    o->pp = NULL;
    if (in->irf_per_pixel) {
        size_t np = (size_t)in->n_rows * in->n_cols;
        o->pp = (irf_t*)malloc(sizeof(irf_t) * np);
        for (size_t p = 0; p < np; ++p) irf_make(&o->pp[p], &in->irf_per_pixel[p]);
    }
    o->gain = in->gain;
    o->dead = in->dead;
}
static void sensor_free(sensor_t* o) {
    irf_free(&o->shared);
    if (o->pp) {
        size_t np = (size_t)o->rows * o->cols;
        for (size_t p = 0; p < np; ++p) irf_free(&o->pp[p]);
        free(o->pp);
    }
}
/* sensor.hpp:160-169 */
static inline const irf_t* sensor_irf(const sensor_t* s, size_t p) {
    return s->pp ? &s->pp[p] : &s->shared;
}
static inline double effective_gain(const sensor_t* s, size_t p) {
    return s->dead[p] ? 0.0 : s->gain[p];
}

typedef struct state_t {
    rt3d_point* pts;
    uint64_t n;
    double* bg;
    uint32_t* boff; /* n_pix + 1 */
    uint32_t* bpts; /* n */
    const sensor_t* sensor;
} state_t;

/* SceneState::refresh, likelihood.hpp:38-55.  Returns -1 on a home pixel out
 * of bounds (invalid_argument). */
static int state_refresh(state_t* st) {
    const sensor_t* s = st->sensor;
    size_t n_pix = (size_t)s->rows * s->cols;
    uint32_t* counts = (uint32_t*)calloc(n_pix, sizeof(uint32_t));
    for (uint64_t k = 0; k < st->n; ++k) {
        const rt3d_point* p = &st->pts[k];
        if (p->i < 0 || p->i >= s->rows || p->j < 0 || p->j >= s->cols) {
            free(counts);
            return -1;
        }
        ++counts[(size_t)p->i * s->cols + p->j];
    }
    st->boff[0] = 0;
    for (size_t p = 0; p < n_pix; ++p) st->boff[p + 1] = st->boff[p] + counts[p];
    for (size_t p = 0; p < n_pix; ++p) counts[p] = st->boff[p];
    for (uint64_t k = 0; k < st->n; ++k) {
        size_t p = (size_t)st->pts[k].i * s->cols + st->pts[k].j;
        st->bpts[counts[p]++] = (uint32_t)k;
    }
    free(counts);
    return 0;
}

static int state_make(state_t* st, const sensor_t* s, rt3d_point* pts, uint64_t n, double* bg,
                      uint64_t cap) {
    size_t n_pix = (size_t)s->rows * s->cols;
    st->pts = pts;
    st->n = n;
    st->bg = bg;
    st->sensor = s;
    st->boff = (uint32_t*)malloc(sizeof(uint32_t) * (n_pix + 1));
    st->bpts = (uint32_t*)malloc(sizeof(uint32_t) * (cap > 0 ? cap : 1));
    return state_refresh(st);
}
static void state_free(state_t* st) {
    free(st->boff);
    free(st->bpts);
}

/* detail::active_rates, likelihood.hpp:100-121 */
static int active_rates(const state_t* st, const rt3d_cube* cube, size_t p, double* lam) {
    const sensor_t* s = st->sensor;
    double g = effective_gain(s, p);
    uint64_t eb = cube->offsets[p], ee = cube->offsets[p + 1];
    for (uint64_t e = eb; e < ee; ++e) lam[e - eb] = 0.0;
    if (g == 0.0) return 0;
    double bg = st->bg[p];
    for (uint64_t e = eb; e < ee; ++e) lam[e - eb] = g * bg;
    const irf_t* irf = sensor_irf(s, p);
    for (uint32_t k = st->boff[p]; k < st->boff[p + 1]; ++k) {
        const rt3d_point* pt = &st->pts[st->bpts[k]];
        int lo, hi;
        irf_support(irf, pt->t, s->bins, &lo, &hi);
        uint64_t e = eb;
        while (e != ee && cube->events[e].bin < (uint32_t)lo) ++e;
        for (; e != ee && cube->events[e].bin <= (uint32_t)hi; ++e)
            lam[e - eb] += g * pt->intensity * irf_value(irf, (double)cube->events[e].bin - pt->t);
    }
    return 1;
}

static uint64_t max_events_per_pixel(const rt3d_cube* cube) {
    size_t np = (size_t)cube->n_rows * cube->n_cols;
    uint64_t m = 1;
    for (size_t p = 0; p < np; ++p) {
        uint64_t c = cube->offsets[p + 1] - cube->offsets[p];
        if (c > m) m = c;
    }
    return m;
}

/* nll, likelihood.hpp:136-168 */
static double state_nll(const state_t* st, const rt3d_cube* cube) {
    const sensor_t* s = st->sensor;
    size_t n_pix = (size_t)cube->n_rows * cube->n_cols;
    double* partial = (double*)calloc(n_pix, sizeof(double));
    double* lam = (double*)malloc(sizeof(double) * max_events_per_pixel(cube));
    for (size_t p = 0; p < n_pix; ++p) {
        if (s->dead[p]) continue;
        double g = s->gain[p];
        const irf_t* irf = sensor_irf(s, p);
        double mass = cube->n_bins * st->bg[p];
        for (uint32_t k = st->boff[p]; k < st->boff[p + 1]; ++k) {
            const rt3d_point* pt = &st->pts[st->bpts[k]];
            mass += pt->intensity * irf_mass_in_gate(irf, pt->t, cube->n_bins);
        }
        double acc = g * mass;
        active_rates(st, cube, p, lam);
        uint64_t eb = cube->offsets[p], ee = cube->offsets[p + 1];
        for (uint64_t e = eb; e < ee; ++e) {
            double l = lam[e - eb];
            if (l <= 0.0) {
                acc = INFINITY;
                break;
            }
            acc -= (double)cube->events[e].count * log(l);
        }
        partial[p] = acc;
    }
    double v = oracle_pairwise_sum(partial, n_pix);
    free(partial);
    free(lam);
    return v;
}

/* grad_depth, likelihood.hpp:178-219 */
static void state_grad_depth(const state_t* st, const rt3d_cube* cube, double* value,
                             uint8_t* oog) {
    const sensor_t* s = st->sensor;
    size_t n_pix = (size_t)cube->n_rows * cube->n_cols;
    for (uint64_t k = 0; k < st->n; ++k) {
        value[k] = 0.0;
        oog[k] = 0;
    }
    double* lam = (double*)malloc(sizeof(double) * max_events_per_pixel(cube));
    for (size_t p = 0; p < n_pix; ++p) {
        uint32_t pb = st->boff[p], pe = st->boff[p + 1];
        if (pb == pe) continue;
        double g = effective_gain(s, p);
        if (g == 0.0) continue;
        const irf_t* irf = sensor_irf(s, p);
        active_rates(st, cube, p, lam);
        uint64_t eb = cube->offsets[p], ee = cube->offsets[p + 1];
        for (uint32_t k = pb; k < pe; ++k) {
            uint32_t n = st->bpts[k];
            const rt3d_point* pt = &st->pts[n];
            int lo, hi;
            irf_support(irf, pt->t, cube->n_bins, &lo, &hi);
            if (lo > hi) {
                oog[n] = 1;
                continue;
            }
            if (pt->intensity == 0.0) continue;
            double acc = 0.0;
            for (int b = lo; b <= hi; ++b) acc -= irf_deriv(irf, (double)b - pt->t);
            uint64_t e = eb;
            while (e != ee && cube->events[e].bin < (uint32_t)lo) ++e;
            for (; e != ee && cube->events[e].bin <= (uint32_t)hi; ++e) {
                double l = lam[e - eb];
                if (l > 0.0)
                    acc += irf_deriv(irf, (double)cube->events[e].bin - pt->t) *
                           (double)cube->events[e].count / l;
            }
            value[n] = g * pt->intensity * acc;
        }
    }
    free(lam);
}

/* grad_intensity, likelihood.hpp:222-253 */
static void state_grad_intensity(const state_t* st, const rt3d_cube* cube, double* out) {
    const sensor_t* s = st->sensor;
    size_t n_pix = (size_t)cube->n_rows * cube->n_cols;
    for (uint64_t k = 0; k < st->n; ++k) out[k] = 0.0;
    double* lam = (double*)malloc(sizeof(double) * max_events_per_pixel(cube));
    for (size_t p = 0; p < n_pix; ++p) {
        uint32_t pb = st->boff[p], pe = st->boff[p + 1];
        if (pb == pe) continue;
        double g = effective_gain(s, p);
        if (g == 0.0) continue;
        const irf_t* irf = sensor_irf(s, p);
        active_rates(st, cube, p, lam);
        uint64_t eb = cube->offsets[p], ee = cube->offsets[p + 1];
        for (uint32_t k = pb; k < pe; ++k) {
            uint32_t n = st->bpts[k];
            const rt3d_point* pt = &st->pts[n];
            double acc = irf_mass_in_gate(irf, pt->t, cube->n_bins);
            int lo, hi;
            irf_support(irf, pt->t, cube->n_bins, &lo, &hi);
            uint64_t e = eb;
            while (e != ee && cube->events[e].bin < (uint32_t)lo) ++e;
            for (; e != ee && cube->events[e].bin <= (uint32_t)hi; ++e) {
                double l = lam[e - eb];
                if (l > 0.0)
                    acc -= irf_value(irf, (double)cube->events[e].bin - pt->t) *
                           (double)cube->events[e].count / l;
            }
            out[n] = g * acc;
        }
    }
    free(lam);
}

/* grad_background, likelihood.hpp:256-277 */
static void state_grad_background(const state_t* st, const rt3d_cube* cube, double* out) {
    const sensor_t* s = st->sensor;
    size_t n_pix = (size_t)cube->n_rows * cube->n_cols;
    double* lam = (double*)malloc(sizeof(double) * max_events_per_pixel(cube));
    for (size_t p = 0; p < n_pix; ++p) {
        out[p] = 0.0;
        double g = effective_gain(s, p);
        if (g == 0.0) continue;
        active_rates(st, cube, p, lam);
        uint64_t eb = cube->offsets[p], ee = cube->offsets[p + 1];
        double acc = g * cube->n_bins;
        for (uint64_t e = eb; e < ee; ++e) {
            double l = lam[e - eb];
            if (l > 0.0) acc -= g * (double)cube->events[e].count / l;
        }
        out[p] = acc;
    }
    free(lam);
}

/* block_curvatures, likelihood.hpp:288-333 */
static void state_curvatures(const state_t* st, const rt3d_cube* cube, double* depth,
                             double* intensity, double* bgc) {
    const sensor_t* s = st->sensor;
    size_t n_pix = (size_t)cube->n_rows * cube->n_cols;
    for (uint64_t k = 0; k < st->n; ++k) {
        depth[k] = 0.0;
        intensity[k] = 0.0;
    }
    double* lam = (double*)malloc(sizeof(double) * max_events_per_pixel(cube));
    for (size_t p = 0; p < n_pix; ++p) {
        bgc[p] = 0.0;
        double g = effective_gain(s, p);
        if (g == 0.0) continue;
        const irf_t* irf = sensor_irf(s, p);
        active_rates(st, cube, p, lam);
        uint64_t eb = cube->offsets[p], ee = cube->offsets[p + 1];
        double bsum = 0.0;
        for (uint64_t e = eb; e < ee; ++e) {
            double l = lam[e - eb];
            if (l > 0.0) bsum += g * g * (double)cube->events[e].count / (l * l);
        }
        bgc[p] = bsum;
        for (uint32_t k = st->boff[p]; k < st->boff[p + 1]; ++k) {
            uint32_t n = st->bpts[k];
            const rt3d_point* pt = &st->pts[n];
            int lo, hi;
            irf_support(irf, pt->t, cube->n_bins, &lo, &hi);
            double stt = 0.0, sr = 0.0;
            uint64_t e = eb;
            while (e != ee && cube->events[e].bin < (uint32_t)lo) ++e;
            for (; e != ee && cube->events[e].bin <= (uint32_t)hi; ++e) {
                double l = lam[e - eb];
                if (l <= 0.0) continue;
                double tau = (double)cube->events[e].bin - pt->t;
                double zl2 = (double)cube->events[e].count / (l * l);
                double dh = g * pt->intensity * irf_deriv(irf, tau);
                double h = g * irf_value(irf, tau);
                stt += dh * dh * zl2;
                sr += h * h * zl2;
            }
            depth[n] = stt;
            intensity[n] = sr;
        }
    }
    free(lam);
}

/* Public state-level wrappers. */
#define WITH_STATE(body)                                                   \
    sensor_t sn;                                                           \
    sensor_make(&sn, sensor);                                              \
    state_t st;                                                            \
    state_make(&st, &sn, (rt3d_point*)points, n, (double*)background, n); \
    body;                                                                  \
    state_free(&st);                                                       \
    sensor_free(&sn);

double oracle_nll(const rt3d_cube* cube, const rt3d_sensor* sensor, const rt3d_point* points,
                  uint64_t n, const double* background) {
    double v = 0.0;
    WITH_STATE(v = state_nll(&st, cube));
    return v;
}
void oracle_grad_depth(const rt3d_cube* cube, const rt3d_sensor* sensor,
                       const rt3d_point* points, uint64_t n, const double* background,
                       double* value, uint8_t* out_of_gate) {
    WITH_STATE(state_grad_depth(&st, cube, value, out_of_gate));
}
void oracle_grad_intensity(const rt3d_cube* cube, const rt3d_sensor* sensor,
                           const rt3d_point* points, uint64_t n, const double* background,
                           double* out) {
    WITH_STATE(state_grad_intensity(&st, cube, out));
}
void oracle_grad_background(const rt3d_cube* cube, const rt3d_sensor* sensor,
                            const rt3d_point* points, uint64_t n, const double* background,
                            double* out) {
    WITH_STATE(state_grad_background(&st, cube, out));
}
void oracle_block_curvatures(const rt3d_cube* cube, const rt3d_sensor* sensor,
                             const rt3d_point* points, uint64_t n, const double* background,
                             double* depth, double* intensity, double* bg_curv) {
    WITH_STATE(state_curvatures(&st, cube, depth, intensity, bg_curv));
}

/* ------------------------------------------------------------------------ */
/* Matched filter, reconstruct.hpp:120-189                                   */
/* ------------------------------------------------------------------------ */
typedef struct mf_ctx {
    const rt3d_event* eb;
    uint64_t n;
    const irf_t* irf;
    double h_max;
} mf_ctx;

/* the `response` lambda, reconstruct.hpp:129-138 */
static double mf_response(const mf_ctx* c, double t0) {
    uint32_t first = (uint32_t)std_max(0.0, ceil(t0 + c->irf->tau_min));
    /* std::lower_bound: first event with bin >= first */
    uint64_t lo = 0, hi = c->n;
    while (lo < hi) {
        uint64_t mid = lo + (hi - lo) / 2;
        if (c->eb[mid].bin < first) lo = mid + 1;
        else hi = mid;
    }
    double acc = 0.0;
    for (uint64_t e = lo; e != c->n && (double)c->eb[e].bin <= t0 + c->irf->tau_max; ++e)
        acc += (double)c->eb[e].count * irf_value(c->irf, (double)c->eb[e].bin - t0);
    return acc / c->h_max;
}

static int cmp_int(const void* a, const void* b) {
    int x = *(const int*)a, y = *(const int*)b;
    return (x > y) - (x < y);
}

typedef struct rank_t {
    double resp;
    int lag;
} rank_t;
static int cmp_rank(const void* a, const void* b) {
    const rank_t* x = (const rank_t*)a;
    const rank_t* y = (const rank_t*)b;
    if (x->resp != y->resp) return x->resp > y->resp ? -1 : 1;
    return (x->lag > y->lag) - (x->lag < y->lag);
}

static int mf_peaks(const rt3d_event* eb, uint64_t n_ev, const irf_t* irf, int n_bins, int k,
                    double threshold, int min_sep, rt3d_peak* out) {
    if (n_ev == 0) return 0;
    mf_ctx c = {eb, n_ev, irf, 0.0};
    for (uint64_t q = 0; q < irf->n; ++q) c.h_max = std_max(c.h_max, irf->s[q]);

    /* candidate lags, reconstruct.hpp:141-148 */
    size_t cap = 16, nc = 0;
    int* cand = (int*)malloc(sizeof(int) * cap);
    for (uint64_t e = 0; e < n_ev; ++e) {
        int lo = imax(0, (int)ceil((double)eb[e].bin - irf->tau_max));
        int hi = imin(n_bins - 1, (int)floor((double)eb[e].bin - irf->tau_min));
        for (int t0 = lo; t0 <= hi; ++t0) {
            if (nc == cap) {
                cap *= 2;
                cand = (int*)realloc(cand, sizeof(int) * cap);
            }
            cand[nc++] = t0;
        }
    }
    qsort(cand, nc, sizeof(int), cmp_int);
    size_t nu = 0;
    for (size_t q = 0; q < nc; ++q)
        if (nu == 0 || cand[q] != cand[nu - 1]) cand[nu++] = cand[q];

    /* responses + ranking, reconstruct.hpp:150-159 */
    rank_t* order = (rank_t*)malloc(sizeof(rank_t) * (nu ? nu : 1));
    for (size_t q = 0; q < nu; ++q) {
        order[q].resp = mf_response(&c, (double)cand[q]);
        order[q].lag = cand[q];
    }
    qsort(order, nu, sizeof(rank_t), cmp_rank);

    /* greedy pick + refine, reconstruct.hpp:161-186 */
    int n_out = 0;
    int* taken = (int*)malloc(sizeof(int) * (k > 0 ? k : 1));
    int n_taken = 0;
    for (size_t q = 0; q < nu; ++q) {
        if (n_out >= k) break;
        if (order[q].resp < threshold) break;
        int t0 = order[q].lag;
        int clash = 0;
        for (int m = 0; m < n_taken; ++m)
            if (abs(taken[m] - t0) < min_sep) {
                clash = 1;
                break;
            }
        if (clash) continue;
        taken[n_taken++] = t0;

        rt3d_peak pk;
        pk.response = order[q].resp;
        pk.mass = 0.0;
        double c0 = order[q].resp;
        double cm = t0 > 0 ? mf_response(&c, (double)(t0 - 1)) : 0.0;
        double cp = t0 < n_bins - 1 ? mf_response(&c, (double)(t0 + 1)) : 0.0;
        double denom = cm - 2.0 * c0 + cp;
        double delta = fabs(denom) > 1e-12 ? 0.5 * (cm - cp) / denom : 0.0;
        pk.t = t0 + std_clamp(delta, -0.5, 0.5);
        int wlo, whi;
        irf_support(irf, pk.t, n_bins, &wlo, &whi);
        for (uint64_t e = 0; e < n_ev; ++e)
            if (eb[e].bin >= (uint32_t)wlo && eb[e].bin <= (uint32_t)whi)
                pk.mass += (double)eb[e].count;
        out[n_out++] = pk;
    }
    /* std::sort by t (insertion sort for n <= 16: stable), reconstruct.hpp:187 */
    for (int a = 1; a < n_out; ++a) {
        rt3d_peak v = out[a];
        int b = a;
        while (b > 0 && v.t < out[b - 1].t) {
            out[b] = out[b - 1];
            --b;
        }
        out[b] = v;
    }
    free(cand);
    free(order);
    free(taken);
    return n_out;
}

int oracle_matched_filter_peaks(const rt3d_event* events, uint64_t n_events, const rt3d_irf* irf,
                                int n_bins, int k, double threshold, int min_sep,
                                rt3d_peak* out) {
    irf_t f;
    irf_make(&f, irf);
    int n = mf_peaks(events, n_events, &f, n_bins, k, threshold, min_sep, out);
    irf_free(&f);
    return n;
}

/* world_from_lidar, sensor.hpp:200-203 */
static inline void world_from_lidar(int fi, int fj, double t, const sensor_t* s, double* x,
                                    double* y, double* z) {
    *x = (fi + 0.5) * s->pitch;
    *y = (fj + 0.5) * s->pitch;
    *z = t * s->bres;
}

/* init_matched_filter, reconstruct.hpp:197-249 */
static int init_impl(const rt3d_cube* cube, const sensor_t* sn, const rt3d_init_params* prm,
                     rt3d_point* points, uint64_t* n_points, double* background) {
    if (prm->max_returns < 1 || prm->min_separation < 1 || prm->peak_threshold < 0.0) return -1;
    if (sn->rows != cube->n_rows || sn->cols != cube->n_cols || sn->bins != cube->n_bins)
        return -1;
    size_t n_pix = (size_t)cube->n_rows * cube->n_cols;
    int s = sn->s;
    rt3d_peak* peaks = (rt3d_peak*)malloc(sizeof(rt3d_peak) * prm->max_returns);
    uint64_t np = 0;
    for (size_t p = 0; p < n_pix; ++p) {
        int i = (int)p / sn->cols, j = (int)p % sn->cols;
        background[p] = kBackgroundFloor;
        double g = effective_gain(sn, p);
        if (g == 0.0) continue;
        uint64_t eb = cube->offsets[p], ee = cube->offsets[p + 1];
        if (eb == ee) continue;
        const irf_t* irf = sensor_irf(sn, p);
        int npk = mf_peaks(cube->events + eb, ee - eb, irf, cube->n_bins, prm->max_returns,
                           prm->peak_threshold, prm->min_separation, peaks);
        double claimed = 0.0;
        for (int q = 0; q < npk; ++q) {
            double irf_mass = irf_mass_in_gate(irf, peaks[q].t, cube->n_bins);
            if (irf_mass <= 0.0) continue;
            double intensity = peaks[q].mass / (g * irf_mass);
            claimed += peaks[q].mass;
            for (int a = 0; a < s; ++a)
                for (int c = 0; c < s; ++c) {
                    rt3d_point* pt = &points[np++];
                    memset(pt, 0, sizeof(*pt));
                    pt->fi = i * s + a;
                    pt->fj = j * s + c;
                    pt->i = i;
                    pt->j = j;
                    pt->t = peaks[q].t;
                    world_from_lidar(pt->fi, pt->fj, pt->t, sn, &pt->x, &pt->y, &pt->z);
                    pt->intensity = intensity / (double)(s * s);
                }
        }
        double total = 0.0;
        for (uint64_t e = eb; e < ee; ++e) total += (double)cube->events[e].count;
        double residual = std_max(0.0, total - std_min(claimed, total));
        background[p] = std_max(kBackgroundFloor, residual / (g * cube->n_bins));
    }
    free(peaks);
    *n_points = np;
    return 0;
}

int oracle_init_matched_filter(const rt3d_cube* cube, const rt3d_sensor* sensor,
                               const rt3d_init_params* params, rt3d_point* points,
                               uint64_t* n_points, double* background) {
    sensor_t sn;
    sensor_make(&sn, sensor);
    int rc = init_impl(cube, &sn, params, points, n_points, background);
    sensor_free(&sn);
    return rc;
}

/* ------------------------------------------------------------------------ */
/* SpatialIndex, spatial_index.hpp:18-77                                     */
/* ------------------------------------------------------------------------ */
typedef struct sidx_t {
    const rt3d_point* cloud;
    uint64_t n;
    double cell;
    uint64_t* keys;  /* sorted */
    uint32_t* order; /* point ids sorted by (key, id) */
} sidx_t;

static inline int64_t sidx_coord(const sidx_t* x, double v) { return (int64_t)floor(v / x->cell); }
static inline uint64_t sidx_u(int64_t v) {
    return (uint64_t)(v + (1ll << 20)) & ((1ull << 21) - 1);
}
static inline uint64_t sidx_pack(int64_t a, int64_t b, int64_t c) {
    return (sidx_u(a) << 42) | (sidx_u(b) << 21) | sidx_u(c);
}

static const uint64_t* g_sort_keys;
static int cmp_key_id(const void* a, const void* b) {
    uint32_t x = *(const uint32_t*)a, y = *(const uint32_t*)b;
    uint64_t kx = g_sort_keys[x], ky = g_sort_keys[y];
    if (kx != ky) return kx < ky ? -1 : 1;
    return (x > y) - (x < y);
}

static void sidx_build(sidx_t* x, const rt3d_point* cloud, uint64_t n, double cell) {
    x->cloud = cloud;
    x->n = n;
    x->cell = cell;
    uint64_t* k = (uint64_t*)malloc(sizeof(uint64_t) * (n ? n : 1));
    x->order = (uint32_t*)malloc(sizeof(uint32_t) * (n ? n : 1));
    x->keys = (uint64_t*)malloc(sizeof(uint64_t) * (n ? n : 1));
    for (uint64_t q = 0; q < n; ++q) {
        k[q] = sidx_pack(sidx_coord(x, cloud[q].x), sidx_coord(x, cloud[q].y),
                         sidx_coord(x, cloud[q].z));
        x->order[q] = (uint32_t)q;
    }
    g_sort_keys = k;
    qsort(x->order, n, sizeof(uint32_t), cmp_key_id);
    for (uint64_t q = 0; q < n; ++q) x->keys[q] = k[x->order[q]];
    free(k);
}
static void sidx_free(sidx_t* x) {
    free(x->keys);
    free(x->order);
}

/* Vec3 (a - b).squaredNorm(), Eigen evaluation order ((dx*dx + dy*dy) + dz*dz) */
static inline double sqdist(double ax, double ay, double az, double bx, double by, double bz) {
    double dx = ax - bx, dy = ay - by, dz = az - bz;
    return dx * dx + dy * dy + dz * dz;
}

static int cmp_u32(const void* a, const void* b) {
    uint32_t x = *(const uint32_t*)a, y = *(const uint32_t*)b;
    return (x > y) - (x < y);
}

/* query, spatial_index.hpp:31-47; returns count, fills *out (malloc'd). */
static uint64_t sidx_query(const sidx_t* x, double qx, double qy, double qz, double radius,
                           uint32_t** out, uint64_t* cap) {
    uint64_t cnt = 0;
    const double r2 = radius * radius;
    int64_t cx = sidx_coord(x, qx), cy = sidx_coord(x, qy), cz = sidx_coord(x, qz);
    for (int64_t dx = -1; dx <= 1; ++dx)
        for (int64_t dy = -1; dy <= 1; ++dy)
            for (int64_t dz = -1; dz <= 1; ++dz) {
                uint64_t key = sidx_pack(cx + dx, cy + dy, cz + dz);
                uint64_t lo = 0, hi = x->n;
                while (lo < hi) {
                    uint64_t mid = lo + (hi - lo) / 2;
                    if (x->keys[mid] < key) lo = mid + 1;
                    else hi = mid;
                }
                for (uint64_t q = lo; q < x->n && x->keys[q] == key; ++q) {
                    uint32_t m = x->order[q];
                    const rt3d_point* p = &x->cloud[m];
                    if (sqdist(p->x, p->y, p->z, qx, qy, qz) <= r2) {
                        if (cnt == *cap) {
                            *cap = *cap ? *cap * 2 : 64;
                            *out = (uint32_t*)realloc(*out, sizeof(uint32_t) * *cap);
                        }
                        (*out)[cnt++] = m;
                    }
                }
            }
    qsort(*out, cnt, sizeof(uint32_t), cmp_u32);
    return cnt;
}

/* ------------------------------------------------------------------------ */
/* APSS, denoise.hpp:24-217                                                  */
/* ------------------------------------------------------------------------ */

/* ApssParams::weight, denoise.hpp:38-44 */
static inline double apss_weight(double radius, double dist) {
    double x = dist / radius;
    if (x >= 1.0) return 0.0;
    double s = 1.0 - x * x;
    s *= s;
    return s * s;
}

/* Eigenvalues of a symmetric 3x3 (row-major, lower triangle read) by cyclic
 * Jacobi, ascending.  Stand-in for SelfAdjointEigenSolver<Matrix3d>
 * (denoise.hpp:196); only the eigenvalues are used (denoise.hpp:198-199). */
void oracle_sym3_eigenvalues(const double c[9], double ev[3]) {
    double a[3][3];
    for (int r = 0; r < 3; ++r)
        for (int q = 0; q <= r; ++q) a[r][q] = a[q][r] = c[r * 3 + q];
    for (int sweep = 0; sweep < 12; ++sweep) {
        double off = fabs(a[1][0]) + fabs(a[2][0]) + fabs(a[2][1]);
        if (off == 0.0) break;
        for (int p = 0; p < 2; ++p)
            for (int q = p + 1; q < 3; ++q) {
                double apq = a[q][p];
                if (apq == 0.0) continue;
                double app = a[p][p], aqq = a[q][q];
                double theta = (aqq - app) / (2.0 * apq);
                double t;
                if (fabs(theta) > 1e150) {
                    t = 0.5 / theta;
                } else {
                    t = 1.0 / (fabs(theta) + sqrt(theta * theta + 1.0));
                    if (theta < 0.0) t = -t;
                }
                double cs = 1.0 / sqrt(t * t + 1.0);
                double sn = t * cs;
                a[p][p] = app - t * apq;
                a[q][q] = aqq + t * apq;
                a[p][q] = a[q][p] = 0.0;
                int r = 3 - p - q;
                double arp = a[r][p], arq = a[r][q];
                a[r][p] = a[p][r] = cs * arp - sn * arq;
                a[r][q] = a[q][r] = sn * arp + cs * arq;
            }
    }
    double d0 = a[0][0], d1 = a[1][1], d2 = a[2][2], tmp;
    if (d1 < d0) { tmp = d0; d0 = d1; d1 = tmp; }
    if (d2 < d1) { tmp = d1; d1 = d2; d2 = tmp; }
    if (d1 < d0) { tmp = d0; d0 = d1; d1 = tmp; }
    ev[0] = d0;
    ev[1] = d1;
    ev[2] = d2;
}

/* LDL' of the lower triangle of a symmetric 5x5; 1 if all pivots > 0. */
static int ldlt5(const double a[5][5], double L[5][5], double d[5]) {
    for (int j = 0; j < 5; ++j) {
        double s = a[j][j];
        for (int k = 0; k < j; ++k) s -= L[j][k] * L[j][k] * d[k];
        if (!(s > 0.0)) return 0;
        d[j] = s;
        for (int i = j + 1; i < 5; ++i) {
            double v = a[i][j];
            for (int k = 0; k < j; ++k) v -= L[i][k] * L[j][k] * d[k];
            L[i][j] = v / s;
        }
    }
    return 1;
}

/* Positive definiteness of the lower triangle of a symmetric 5x5 without
 * divisions: Gaussian elimination with each Schur update scaled by the
 * (positive) pivot, a[i][j] <- a[k][k] a[i][j] - a[i][k] a[j][k]; the pivots
 * keep the signs of the LDL' pivots. */
static int pd5(double a[5][5]) {
    for (int k = 0; k < 5; ++k) {
        const double akk = a[k][k];
        if (!(akk > 0.0)) return 0;
        for (int i = k + 1; i < 5; ++i)
            for (int j = k + 1; j <= i; ++j) a[i][j] = akk * a[i][j] - a[i][k] * a[j][k];
    }
    return 1;
}

/* M - sigma N with the Pratt matrix N (denoise.hpp:82-84). */
static void pencil_shift(const double m[5][5], double sigma, double a[5][5]) {
    memcpy(a, m, sizeof(double) * 25);
    a[1][1] = m[1][1] - sigma;
    a[2][2] = m[2][2] - sigma;
    a[3][3] = m[3][3] - sigma;
    a[4][0] = m[4][0] + 2.0 * sigma;
    a[0][4] = a[4][0];
}

/* Smallest admissible generalized eigenpair of (M, N) — the eigenvector the
 * reference's loop over GeneralizedEigenSolver results keeps
 * (denoise.hpp:86-112), before normalisation.  Returns 0 if none. */
int oracle_pratt_smallest(const double mflat[25], double u[5]) {
    double m[5][5], a[5][5], L[5][5], d[5];
    for (int r = 0; r < 5; ++r)
        for (int q = 0; q <= r; ++q) m[r][q] = m[q][r] = mflat[r * 5 + q];
    const double scale = std_max(m[0][0] + m[1][1] + m[2][2] + m[3][3] + m[4][4], 1e-300);
    double sigma;
    pencil_shift(m, 0.0, a);
    double hi = std_min(std_min(m[1][1], m[2][2]), m[3][3]);
    if (pd5(a) && hi > 0.0) {
        double lo = 0.0;
        for (int it = 0; it < 200; ++it) {
            double mid = 0.5 * (lo + hi);
            if (!(mid > lo && mid < hi)) break;
            pencil_shift(m, mid, a);
            if (pd5(a)) lo = mid;
            else hi = mid;
            /* bracket to 1e-9 relative: the inverse iteration below converges
             * from there (ratio ~1e-9 / gap per step) */
            if (hi - lo <= 1e-9 * hi) break;
        }
        sigma = lo;
    } else {
        /* M (numerically) singular: eta* ~ 0; step just below it. */
        double delta = 1e-15 * scale;
        int ok = 0;
        for (int k = 0; k < 12 && !ok; ++k) {
            pencil_shift(m, -delta, a);
            if (pd5(a)) ok = 1;
            else delta *= 10.0;
        }
        if (!ok) return 0;
        sigma = -delta;
    }
    /* the factor of the last definite shift; the division-free test and the
     * LDL' can disagree within rounding of eta*, so step below if needed */
    {
        const double base = sigma;
        double delta = 1e-15 * scale;
        int ok = 0;
        for (int k = 0; k < 14; ++k) {
            pencil_shift(m, sigma, a);
            if (ldlt5(a, L, d)) {
                ok = 1;
                break;
            }
            sigma = base - delta;
            delta *= 10.0;
        }
        if (!ok) return 0;
    }
    /* inverse iteration (M - sigma N) x_{k+1} = N x_k */
    double x[5] = {1.0, 1.0, 1.0, 1.0, 1.0};
    for (int it = 0; it < 4; ++it) {
        double y[5];
        y[0] = -2.0 * x[4];
        y[1] = x[1];
        y[2] = x[2];
        y[3] = x[3];
        y[4] = -2.0 * x[0];
        for (int i = 0; i < 5; ++i) {
            double v = y[i];
            for (int k = 0; k < i; ++k) v -= L[i][k] * y[k];
            y[i] = v;
        }
        for (int i = 0; i < 5; ++i) y[i] = y[i] / d[i];
        for (int i = 4; i >= 0; --i) {
            double v = y[i];
            for (int k = i + 1; k < 5; ++k) v -= L[k][i] * y[k];
            y[i] = v;
        }
        double nrm = sqrt(y[0] * y[0] + y[1] * y[1] + y[2] * y[2] + y[3] * y[3] + y[4] * y[4]);
        if (!(nrm > 0.0) || !isfinite(nrm)) return 0;
        for (int i = 0; i < 5; ++i) x[i] = y[i] / nrm;
    }
    for (int i = 0; i < 5; ++i) u[i] = x[i];
    return 1;
}

typedef struct sphere_t {
    double u0, ul[3], uq;
    int valid;
} sphere_t;

/* fit_algebraic_sphere, denoise.hpp:66-125 */
/* fit_algebraic_sphere (denoise.hpp:66-125) from its moment matrix M
 * (lower triangle, row-major 5x5), accumulated by the caller */
static sphere_t fit_sphere(const double M[25], const double centre[3]) {
    sphere_t best;
    memset(&best, 0, sizeof(best));
    double v[5];
    if (!oracle_pratt_smallest(M, v)) return best;
    double vn2 = v[0] * v[0] + v[1] * v[1] + v[2] * v[2] + v[3] * v[3] + v[4] * v[4];
    if (sqrt(vn2) < 1e-300) return best;
    double nrm = v[1] * v[1] + v[2] * v[2] + v[3] * v[3] - 4.0 * v[0] * v[4];
    if (nrm <= 1e-14 * vn2) return best;
    double sq = sqrt(nrm);
    for (int i = 0; i < 5; ++i) v[i] /= sq;
    best.u0 = v[0];
    best.ul[0] = v[1];
    best.ul[1] = v[2];
    best.ul[2] = v[3];
    best.uq = v[4];
    best.valid = 1;
    /* undo the centring, denoise.hpp:116-117 */
    double dot = best.ul[0] * centre[0] + best.ul[1] * centre[1] + best.ul[2] * centre[2];
    double csq = centre[0] * centre[0] + centre[1] * centre[1] + centre[2] * centre[2];
    best.u0 = best.u0 - dot + best.uq * csq;
    double tq = 2.0 * best.uq;
    for (int a = 0; a < 3; ++a) best.ul[a] = best.ul[a] - tq * centre[a];
    /* orientation by the PCA normal (denoise.hpp:119-123) flips (u0,ul,uq)
     * together; project_onto_sphere is exactly invariant under that flip, so
     * it is not restated. */
    return best;
}

static inline double sphere_eval(const sphere_t* s, const double p[3]) {
    return s->u0 + (s->ul[0] * p[0] + s->ul[1] * p[1] + s->ul[2] * p[2]) +
           s->uq * (p[0] * p[0] + p[1] * p[1] + p[2] * p[2]);
}

/* project_onto_sphere, denoise.hpp:128-150 */
static int project_sphere(const sphere_t* s, double eps, const double p[3], double out[3]) {
    double g2 = s->ul[0] * s->ul[0] + s->ul[1] * s->ul[1] + s->ul[2] * s->ul[2];
    if (fabs(s->uq) < eps) {
        if (g2 < 1e-20) return 0;
        double f = sphere_eval(s, p) / g2;
        for (int a = 0; a < 3; ++a) out[a] = p[a] - f * s->ul[a];
        return 1;
    }
    double c[3];
    double tq = 2.0 * s->uq;
    for (int a = 0; a < 3; ++a) c[a] = -s->ul[a] / tq;
    double disc = g2 - 4.0 * s->u0 * s->uq;
    if (disc <= 0.0) {
        if (g2 < 1e-20) return 0;
        double f = sphere_eval(s, p) / g2;
        for (int a = 0; a < 3; ++a) out[a] = p[a] - f * s->ul[a];
        return 1;
    }
    double radius = sqrt(disc) / (2.0 * fabs(s->uq));
    double d[3] = {p[0] - c[0], p[1] - c[1], p[2] - c[2]};
    double dn = sqrt(d[0] * d[0] + d[1] * d[1] + d[2] * d[2]);
    if (dn < 1e-14) return 0;
    double f = radius / dn;
    for (int a = 0; a < 3; ++a) out[a] = c[a] + f * d[a];
    return 1;
}

#define APSS_LANES 16
/* the halving tree over APSS_LANES lane partials: p[l] += p[l + o], o = APSS_LANES/2 .. 1 */
static double lane_tree(const double* base, int stride, int col) {
    double p[APSS_LANES];
    for (int l = 0; l < APSS_LANES; ++l) p[l] = base[l * stride + col];
    for (int o = APSS_LANES / 2; o > 0; o >>= 1)
        for (int l = 0; l < o; ++l) p[l] = p[l] + p[l + o];
    return p[0];
}

/* apss_project, denoise.hpp:159-217 */
int oracle_apss_project(const rt3d_point* cloud, uint64_t n, const rt3d_apss_params* prm,
                        const rt3d_point* index_cloud, uint64_t n_index, double cell,
                        rt3d_point* out) {
    if (prm->kernel_radius <= 0.0 || prm->min_neighbors < 4 || prm->sphere_degeneracy_eps < 0.0)
        return -1;
    if (cell <= 0.0) return -1;
    if (prm->kernel_radius > cell * (1.0 + 1e-12) && n > 0) return -1;
    sidx_t idx;
    sidx_build(&idx, index_cloud, n_index, cell);
    memmove(out, cloud, sizeof(rt3d_point) * n);
    uint32_t* nb = NULL;
    uint64_t cap = 0;
    double* q = NULL;
    double* w = NULL;
    uint64_t qcap = 0;
    const double R = prm->kernel_radius;
    for (uint64_t k = 0; k < n; ++k) {
        const rt3d_point* pt = &cloud[k];
        uint8_t flags = pt->flags & (uint8_t)~(RT3D_FLAG_ISOLATED | RT3D_FLAG_DEGENERATE);
        out[k].flags = flags;
        uint64_t cnt = sidx_query(&idx, pt->x, pt->y, pt->z, R, &nb, &cap);
        if (cnt < (uint64_t)prm->min_neighbors) {
            out[k].flags = flags | RT3D_FLAG_ISOLATED;
            continue;
        }
        if (cnt > qcap) {
            qcap = cnt;
            q = (double*)realloc(q, sizeof(double) * 3 * qcap);
            w = (double*)realloc(w, sizeof(double) * qcap);
        }
        /* Summation order (shared with the device kernel, rt3d_nbr.cuh): ball
         * member m (ascending index) is accumulated into lane m mod APSS_LANES (16),
         * sequentially; the lane partials are then combined by the halving
         * tree of lane_tree().  The reference sums each moment sequentially
         * (denoise.hpp:174-180, 191-194, 74-80); the reassociation moves the
         * moments at the 1e-16 relative level, far below the eigen-solver
         * difference. */
        double pa[APSS_LANES][4];
        memset(pa, 0, sizeof(pa));
        for (uint64_t m = 0; m < cnt; ++m) {
            const rt3d_point* o = &index_cloud[nb[m]];
            double* a = pa[m % APSS_LANES];
            q[3 * m] = o->x;
            q[3 * m + 1] = o->y;
            q[3 * m + 2] = o->z;
            w[m] = apss_weight(R, sqrt(sqdist(o->x, o->y, o->z, pt->x, pt->y, pt->z)));
            a[0] += w[m];
            for (int c = 0; c < 3; ++c) a[1 + c] = fma(w[m], q[3 * m + c], a[1 + c]);
        }
        double wsum = lane_tree(&pa[0][0], 4, 0), mean[3];
        for (int c = 0; c < 3; ++c) mean[c] = lane_tree(&pa[0][0], 4, 1 + c);
        if (wsum <= 0.0) {
            out[k].flags = flags | RT3D_FLAG_DEGENERATE;
            continue;
        }
        for (int a = 0; a < 3; ++a) mean[a] /= wsum;
        /* covariance (denoise.hpp:190-195) and the Pratt moments M
         * (denoise.hpp:73-80, members with w > 0), both centred on the mean */
        double pb[APSS_LANES][21];
        memset(pb, 0, sizeof(pb));
        for (uint64_t m = 0; m < cnt; ++m) {
            double* b = pb[m % APSS_LANES];
            double d[3] = {q[3 * m] - mean[0], q[3 * m + 1] - mean[1], q[3 * m + 2] - mean[2]};
            /* the moment sums by fused multiply-add, as the device
             * (apss_pass_b): one rounding per accumulation instead of two */
            int e = 0;
            for (int r = 0; r < 3; ++r) {
                double wr = w[m] * d[r];
                for (int c = 0; c <= r; ++c) {
                    b[e] = fma(wr, d[c], b[e]);
                    ++e;
                }
            }
            if (w[m] > 0.0) {
                double dv[5] = {1.0, d[0], d[1], d[2], d[0] * d[0] + d[1] * d[1] + d[2] * d[2]};
                for (int r = 0; r < 5; ++r) {
                    double wr = w[m] * dv[r];
                    for (int c = 0; c <= r; ++c) {
                        b[e] = fma(wr, dv[c], b[e]);
                        ++e;
                    }
                }
            }
        }
        double cov[9], M[25];
        memset(cov, 0, sizeof(cov));
        memset(M, 0, sizeof(M));
        {
            int e = 0;
            for (int r = 0; r < 3; ++r)
                for (int c = 0; c <= r; ++c) cov[r * 3 + c] = lane_tree(&pb[0][0], 21, e++) / wsum;
            for (int r = 0; r < 5; ++r)
                for (int c = 0; c <= r; ++c) M[r * 5 + c] = lane_tree(&pb[0][0], 21, e++);
        }
        double ev[3];
        oracle_sym3_eigenvalues(cov, ev);
        double spread = ev[2];
        if (spread <= 0.0 || ev[1] <= 1e-12 * spread) {
            out[k].flags = flags | RT3D_FLAG_DEGENERATE;
            continue;
        }
        sphere_t fit = fit_sphere(M, mean);
        double p[3] = {pt->x, pt->y, pt->z}, proj[3];
        if (!fit.valid || !project_sphere(&fit, prm->sphere_degeneracy_eps, p, proj)) {
            out[k].flags = flags | RT3D_FLAG_DEGENERATE;
            continue;
        }
        out[k].x = proj[0];
        out[k].y = proj[1];
        out[k].z = proj[2];
    }
    free(nb);
    free(q);
    free(w);
    sidx_free(&idx);
    return 0;
}

typedef struct dist_id {
    double d2;
    uint32_t id;
} dist_id;
static int cmp_dist_id(const void* a, const void* b) {
    const dist_id* x = (const dist_id*)a;
    const dist_id* y = (const dist_id*)b;
    if (x->d2 != y->d2) return x->d2 < y->d2 ? -1 : 1;
    return (x->id > y->id) - (x->id < y->id);
}

/* knn_intensity_filter, denoise.hpp:223-237 (+ query_knn, spatial_index.hpp:51-62) */
int oracle_knn_intensity_filter(const rt3d_point* cloud, uint64_t n, int k,
                                const rt3d_point* index_cloud, uint64_t n_index, double cell,
                                double radius, rt3d_point* out) {
    if (k < 1 || radius <= 0.0 || cell <= 0.0) return -1;
    if (radius > cell * (1.0 + 1e-12) && n > 0) return -1;
    sidx_t idx;
    sidx_build(&idx, index_cloud, n_index, cell);
    memmove(out, cloud, sizeof(rt3d_point) * n);
    uint32_t* nb = NULL;
    uint64_t cap = 0;
    dist_id* ranked = NULL;
    uint64_t rcap = 0;
    double* r_new = (double*)malloc(sizeof(double) * (n ? n : 1));
    for (uint64_t q = 0; q < n; ++q) {
        const rt3d_point* pt = &cloud[q];
        r_new[q] = pt->intensity;
        uint64_t cnt = sidx_query(&idx, pt->x, pt->y, pt->z, radius, &nb, &cap);
        if (cnt > rcap) {
            rcap = cnt;
            ranked = (dist_id*)realloc(ranked, sizeof(dist_id) * rcap);
        }
        for (uint64_t m = 0; m < cnt; ++m) {
            const rt3d_point* o = &index_cloud[nb[m]];
            ranked[m].d2 = sqdist(o->x, o->y, o->z, pt->x, pt->y, pt->z);
            ranked[m].id = nb[m];
        }
        qsort(ranked, cnt, sizeof(dist_id), cmp_dist_id);
        uint64_t keep = (uint64_t)k < cnt ? (uint64_t)k : cnt;
        if (keep == 0) continue;
        double acc = 0.0;
        for (uint64_t m = 0; m < keep; ++m) acc += index_cloud[ranked[m].id].intensity;
        r_new[q] = acc / (double)keep;
    }
    for (uint64_t q = 0; q < n; ++q) out[q].intensity = r_new[q];
    free(r_new);
    free(nb);
    free(ranked);
    sidx_free(&idx);
    return 0;
}

/* prune, denoise.hpp:241-248 */
uint64_t oracle_prune(const rt3d_point* cloud, uint64_t n, double r_min, rt3d_point* out) {
    uint64_t m = 0;
    for (uint64_t k = 0; k < n; ++k)
        if (cloud[k].intensity >= r_min) out[m++] = cloud[k];
    return m;
}

/* ------------------------------------------------------------------------ */
/* FFT low-pass, denoise.hpp:254-319 (direct DFT stands in for FFTW)         */
/* ------------------------------------------------------------------------ */
static double lowpass_mask(double rho, double cutoff) {
    if (cutoff >= 1.0) return 1.0;
    double w = std_min(0.2 * cutoff, 1.0 - cutoff);
    double lo = cutoff - w;
    if (rho <= lo) return 1.0;
    if (rho >= cutoff) return 0.0;
    return 0.5 * (1.0 + cos(M_PI * (rho - lo) / w));
}

/* unnormalised 1-D DFT along a strided line; sign -1 forward, +1 backward */
static void dft_line(const double* re, const double* im, int n, int stride, int sign, double* ore,
                     double* oim, const double* cs, const double* sn) {
    for (int k = 0; k < n; ++k) {
        double ar = 0.0, ai = 0.0;
        for (int x = 0; x < n; ++x) {
            int ph = (int)(((long long)k * x) % n);
            double c = cs[ph], s = sign * sn[ph];
            double xr = re[(size_t)x * stride], xi = im[(size_t)x * stride];
            ar += xr * c - xi * s;
            ai += xr * s + xi * c;
        }
        ore[(size_t)k * stride] = ar;
        oim[(size_t)k * stride] = ai;
    }
}

static void dft2(double* re, double* im, int nr, int nc, int sign) {
    size_t total = (size_t)nr * nc;
    double* tr = (double*)malloc(sizeof(double) * total);
    double* ti = (double*)malloc(sizeof(double) * total);
    int nmax = nr > nc ? nr : nc;
    double* cs = (double*)malloc(sizeof(double) * nmax);
    double* sn = (double*)malloc(sizeof(double) * nmax);
    for (int k = 0; k < nc; ++k) {
        cs[k] = cos(2.0 * M_PI * k / nc);
        sn[k] = sin(2.0 * M_PI * k / nc);
    }
    for (int a = 0; a < nr; ++a)
        dft_line(re + (size_t)a * nc, im + (size_t)a * nc, nc, 1, sign, tr + (size_t)a * nc,
                 ti + (size_t)a * nc, cs, sn);
    for (int k = 0; k < nr; ++k) {
        cs[k] = cos(2.0 * M_PI * k / nr);
        sn[k] = sin(2.0 * M_PI * k / nr);
    }
    for (int b = 0; b < nc; ++b) dft_line(tr + b, ti + b, nr, nc, sign, re + b, im + b, cs, sn);
    free(tr);
    free(ti);
    free(cs);
    free(sn);
}

int oracle_fft_lowpass_filter(const double* img, int nr, int nc, double cutoff,
                              int clamp_nonneg, double* out) {
    if (cutoff <= 0.0 || cutoff > 1.0) return -1;
    if (nr < 2 || nc < 2) return -1;
    size_t total = (size_t)nr * nc;
    double* re = (double*)malloc(sizeof(double) * total);
    double* im = (double*)calloc(total, sizeof(double));
    for (size_t k = 0; k < total; ++k) re[k] = img[k];
    dft2(re, im, nr, nc, -1);
    const double fmax_r = (double)(nr / 2) / nr;
    const double fmax_c = (double)(nc / 2) / nc;
    const double rho_max = sqrt(fmax_r * fmax_r + fmax_c * fmax_c);
    for (int a = 0; a < nr; ++a) {
        int far = (a <= nr / 2) ? a : a - nr;
        double fr = (double)far / nr;
        for (int b = 0; b < nc; ++b) {
            int fac = (b <= nc / 2) ? b : b - nc;
            double fc = (double)fac / nc;
            double rho = sqrt(fr * fr + fc * fc) / rho_max;
            double mval = lowpass_mask(rho, cutoff);
            re[(size_t)a * nc + b] *= mval;
            im[(size_t)a * nc + b] *= mval;
        }
    }
    dft2(re, im, nr, nc, +1);
    for (size_t k = 0; k < total; ++k) {
        double v = re[k] / (double)total;
        out[k] = clamp_nonneg ? std_max(0.0, v) : v;
    }
    free(re);
    free(im);
    return 0;
}

/* ------------------------------------------------------------------------ */
/* PALM, reconstruct.hpp:251-435                                             */
/* ------------------------------------------------------------------------ */
static int cfg_validate(const rt3d_recon_config* c) {
    if (c->max_iters < 1 || c->stop_tol < 0.0) return -1;
    if (c->backtrack_beta <= 0.0 || c->backtrack_beta >= 1.0) return -1;
    if (c->knn_k < 1 || c->r_min < 0.0) return -1;
    if (c->apss.kernel_radius <= 0.0 || c->apss.min_neighbors < 4 ||
        c->apss.sphere_degeneracy_eps < 0.0)
        return -1;
    if (c->init.max_returns < 1 || c->init.min_separation < 1 || c->init.peak_threshold < 0.0)
        return -1;
    return 0;
}

/* precondition lambda, reconstruct.hpp:312-317 */
static void precondition(double* dir, const double* curv, uint64_t n) {
    double cmax = 0.0;
    for (uint64_t k = 0; k < n; ++k) cmax = std_max(cmax, curv[k]);
    double floor_ = 1e-3 * cmax + 1e-30;
    for (uint64_t k = 0; k < n; ++k) dir[k] /= (curv[k] + floor_);
}

enum { BLK_T = 0, BLK_R = 1, BLK_B = 2 };

static void apply_block(state_t* st, int blk, double a, const double* before, const double* dir,
                        uint64_t n, double t_limit) {
    if (blk == BLK_T) {
        for (uint64_t k = 0; k < n; ++k) {
            rt3d_point* pt = &st->pts[k];
            pt->t = std_clamp(before[k] - a * dir[k], 0.0, t_limit);
            pt->z = pt->t * st->sensor->bres;
        }
    } else if (blk == BLK_R) {
        for (uint64_t k = 0; k < n; ++k) st->pts[k].intensity = std_max(0.0, before[k] - a * dir[k]);
    } else {
        for (uint64_t k = 0; k < n; ++k) st->bg[k] = std_max(0.0, before[k] - a * dir[k]);
    }
}
static void restore_block(state_t* st, int blk, const double* before, uint64_t n) {
    if (blk == BLK_T) {
        for (uint64_t k = 0; k < n; ++k) {
            rt3d_point* pt = &st->pts[k];
            pt->t = before[k];
            pt->z = pt->t * st->sensor->bres;
        }
    } else if (blk == BLK_R) {
        for (uint64_t k = 0; k < n; ++k) st->pts[k].intensity = before[k];
    } else {
        for (uint64_t k = 0; k < n; ++k) st->bg[k] = before[k];
    }
}

/* safeguarded_step, reconstruct.hpp:274-292 */
static double safeguarded_step(double* alpha, double beta, double nll_current, state_t* st,
                               const rt3d_cube* cube, int blk, const double* before,
                               const double* dir, uint64_t n, double t_limit, int* backtracks) {
    if (*alpha <= 0.0) {
        *alpha = 0.0;
        return nll_current;
    }
    for (int attempt = 0; attempt < kMaxBacktracks; ++attempt) {
        apply_block(st, blk, *alpha, before, dir, n, t_limit);
        double candidate = state_nll(st, cube);
        if (candidate <= nll_current) return candidate;
        restore_block(st, blk, before, n);
        *alpha *= beta;
        ++*backtracks;
    }
    *alpha = 0.0;
    return nll_current;
}

static int palm_impl(const rt3d_cube* cube, const rt3d_recon_config* cfg, state_t* st,
                     rt3d_step_diag* diag) {
    const sensor_t* sn = st->sensor;
    size_t n_pix = (size_t)sn->rows * sn->cols;
    memset(diag, 0, sizeof(*diag));
    diag->points_before = st->n;
    double current = state_nll(st, cube);
    diag->nll_before = current;
    const double t_limit = (double)cube->n_bins * (1.0 - 1e-12);
    uint64_t cap = st->n;
    double* dir = (double*)malloc(sizeof(double) * (cap > n_pix ? cap : n_pix) + 8);
    double* before = (double*)malloc(sizeof(double) * (cap > n_pix ? cap : n_pix) + 8);
    double* c1 = (double*)malloc(sizeof(double) * (cap ? cap : 1));
    double* c2 = (double*)malloc(sizeof(double) * (cap ? cap : 1));
    double* c3 = (double*)malloc(sizeof(double) * n_pix);
    uint8_t* oog = (uint8_t*)malloc(cap ? cap : 1);

    /* ---- depth block ---- */
    if (st->n > 0) {
        uint64_t n = st->n;
        state_grad_depth(st, cube, dir, oog);
        for (uint64_t k = 0; k < n; ++k)
            if (oog[k]) st->pts[k].flags |= RT3D_FLAG_OUT_OF_GATE;
        double alpha = cfg->step_t;
        if (cfg->step_t_auto) {
            state_curvatures(st, cube, c1, c2, c3);
            precondition(dir, c1, n);
            alpha = 1.0;
        }
        for (uint64_t k = 0; k < n; ++k) before[k] = st->pts[k].t;
        current = safeguarded_step(&alpha, cfg->backtrack_beta, current, st, cube, BLK_T, before,
                                   dir, n, t_limit, &diag->depth.backtracks);
        diag->depth.step_used = alpha;
        diag->depth.nll_after_grad = current;

        rt3d_point* proj = (rt3d_point*)malloc(sizeof(rt3d_point) * n);
        oracle_apss_project(st->pts, n, &cfg->apss, st->pts, n, cfg->apss.kernel_radius, proj);
        for (uint64_t k = 0; k < n; ++k) {
            rt3d_point* pt = &proj[k];
            pt->t = std_clamp(pt->z / sn->bres, 0.0, t_limit);
            world_from_lidar(pt->fi, pt->fj, pt->t, sn, &pt->x, &pt->y, &pt->z);
        }
        memcpy(st->pts, proj, sizeof(rt3d_point) * n);
        free(proj);
        state_refresh(st);
        current = state_nll(st, cube);
        diag->depth.nll_after_denoise = current;
    } else {
        diag->depth.nll_after_grad = diag->depth.nll_after_denoise = current;
    }

    /* ---- intensity block ---- */
    if (st->n > 0) {
        uint64_t n = st->n;
        state_grad_intensity(st, cube, dir);
        double alpha = cfg->step_r;
        if (cfg->step_r_auto) {
            state_curvatures(st, cube, c1, c2, c3);
            precondition(dir, c2, n);
            alpha = 1.0;
        }
        for (uint64_t k = 0; k < n; ++k) before[k] = st->pts[k].intensity;
        current = safeguarded_step(&alpha, cfg->backtrack_beta, current, st, cube, BLK_R, before,
                                   dir, n, t_limit, &diag->intensity.backtracks);
        diag->intensity.step_used = alpha;
        diag->intensity.nll_after_grad = current;

        rt3d_point* tmp = (rt3d_point*)malloc(sizeof(rt3d_point) * n);
        oracle_knn_intensity_filter(st->pts, n, cfg->knn_k, st->pts, n, cfg->apss.kernel_radius,
                                    cfg->apss.kernel_radius, tmp);
        st->n = oracle_prune(tmp, n, cfg->r_min, st->pts);
        free(tmp);
        state_refresh(st);
        current = state_nll(st, cube);
        diag->intensity.nll_after_denoise = current;
    } else {
        diag->intensity.nll_after_grad = diag->intensity.nll_after_denoise = current;
    }

    /* ---- background block ---- */
    {
        state_grad_background(st, cube, dir);
        double alpha = cfg->step_b;
        if (cfg->step_b_auto) {
            state_curvatures(st, cube, c1, c2, c3);
            precondition(dir, c3, n_pix);
            alpha = 1.0;
        }
        for (size_t k = 0; k < n_pix; ++k) before[k] = st->bg[k];
        current = safeguarded_step(&alpha, cfg->backtrack_beta, current, st, cube, BLK_B, before,
                                   dir, n_pix, t_limit, &diag->background.backtracks);
        diag->background.step_used = alpha;
        diag->background.nll_after_grad = current;
        if (cfg->background_mode == 1) {
            double* tmp = (double*)malloc(sizeof(double) * n_pix);
            oracle_fft_lowpass_filter(st->bg, sn->rows, sn->cols, cfg->fft_cutoff, 1, tmp);
            memcpy(st->bg, tmp, sizeof(double) * n_pix);
            free(tmp);
        }
        for (size_t k = 0; k < n_pix; ++k)
            st->bg[k] = (st->bg[k] < kBackgroundFloor) ? kBackgroundFloor : st->bg[k];
        current = state_nll(st, cube);
        diag->background.nll_after_denoise = current;
    }
    diag->nll_after = current;
    diag->points_after = st->n;
    free(dir);
    free(before);
    free(c1);
    free(c2);
    free(c3);
    free(oog);
    return 0;
}

int oracle_palm_step(const rt3d_cube* cube, const rt3d_sensor* sensor,
                     const rt3d_recon_config* cfg, rt3d_point* points, uint64_t* n,
                     double* background, rt3d_step_diag* diag) {
    if (cfg_validate(cfg)) return -1;
    sensor_t sn;
    sensor_make(&sn, sensor);
    state_t st;
    if (state_make(&st, &sn, points, *n, background, *n)) {
        state_free(&st);
        sensor_free(&sn);
        return -1;
    }
    int rc = palm_impl(cube, cfg, &st, diag);
    *n = st.n;
    state_free(&st);
    sensor_free(&sn);
    return rc;
}

int oracle_reconstruct(const rt3d_cube* cube, const rt3d_sensor* sensor,
                       const rt3d_recon_config* cfg, rt3d_point* points, uint64_t* n_points,
                       double* background, double* nll_trace, rt3d_step_diag* steps,
                       int* iterations) {
    if (cfg_validate(cfg)) return -1;
    sensor_t sn;
    sensor_make(&sn, sensor);
    uint64_t n = 0;
    int rc = init_impl(cube, &sn, &cfg->init, points, &n, background);
    if (rc) {
        sensor_free(&sn);
        return rc;
    }
    state_t st;
    state_make(&st, &sn, points, n, background, n);
    double init_nll = state_nll(&st, cube);
    nll_trace[0] = init_nll;
    int iters = 0;
    double previous = init_nll;
    for (int it = 0; it < cfg->max_iters; ++it) {
        palm_impl(cube, cfg, &st, &steps[it]);
        nll_trace[it + 1] = steps[it].nll_after;
        ++iters;
        double rel = fabs(previous - steps[it].nll_after) / std_max(1.0, fabs(previous));
        previous = steps[it].nll_after;
        if (rel < cfg->stop_tol) break;
    }
    *n_points = st.n;
    *iterations = iters;
    state_free(&st);
    sensor_free(&sn);
    return 0;
}

/* baseline_xcorr, eval.hpp:91-126 */
int oracle_baseline_xcorr(const rt3d_cube* cube, const rt3d_sensor* sensor, rt3d_point* points,
                          uint64_t* n_points) {
    if (sensor->n_rows != cube->n_rows || sensor->n_cols != cube->n_cols ||
        sensor->n_bins != cube->n_bins)
        return -1;
    sensor_t sn;
    sensor_make(&sn, sensor);
    size_t n_pix = (size_t)cube->n_rows * cube->n_cols;
    uint64_t np = 0;
    for (size_t p = 0; p < n_pix; ++p) {
        int i = (int)p / sn.cols, j = (int)p % sn.cols;
        double g = effective_gain(&sn, p);
        if (g == 0.0) continue;
        uint64_t eb = cube->offsets[p], ee = cube->offsets[p + 1];
        if (eb == ee) continue;
        const irf_t* irf = sensor_irf(&sn, p);
        rt3d_peak pk;
        int npk = mf_peaks(cube->events + eb, ee - eb, irf, cube->n_bins, 1, 0.0, 1, &pk);
        if (npk == 0) continue;
        double irf_mass = irf_mass_in_gate(irf, pk.t, cube->n_bins);
        if (irf_mass <= 0.0) continue;
        rt3d_point* pt = &points[np++];
        memset(pt, 0, sizeof(*pt));
        pt->i = i;
        pt->j = j;
        pt->fi = i * sn.s + sn.s / 2;
        pt->fj = j * sn.s + sn.s / 2;
        pt->t = pk.t;
        double coarse_pitch = sn.pitch * sn.s;
        pt->x = (i + 0.5) * coarse_pitch;
        pt->y = (j + 0.5) * coarse_pitch;
        pt->z = pk.t * sn.bres;
        pt->intensity = pk.mass / (g * irf_mass);
    }
    *n_points = np;
    sensor_free(&sn);
    return 0;
}

/* ---- evaluate (eval.hpp:33-87) ----------------------------------------
   Points go into transverse columns (floor(x/pitch), floor(y/pitch))
   (eval.hpp:39-43); columns are visited in (cx, cy) order like the
   reference's std::map (:44-48, :54).  Inside a column every (est, truth)
   pair within tau is a candidate (:60-65); candidates are taken greedily in
   (err, truth, est) order, each point at most once (:66-79).  The depth and
   intensity sums run in that same order. */
typedef struct {
    int64_t cx, cy;
    uint32_t id; /* est ids first, then n_est + truth id */
} ev_item;

static int ev_item_cmp(const void* a, const void* b) {
    const ev_item* p = (const ev_item*)a;
    const ev_item* q = (const ev_item*)b;
    if (p->cx != q->cx) return p->cx < q->cx ? -1 : 1;
    if (p->cy != q->cy) return p->cy < q->cy ? -1 : 1;
    return p->id < q->id ? -1 : (p->id > q->id);
}

typedef struct {
    double err;
    uint32_t e, t;
} ev_pair;

static int ev_pair_cmp(const void* a, const void* b) {
    const ev_pair* p = (const ev_pair*)a;
    const ev_pair* q = (const ev_pair*)b;
    if (p->err != q->err) return p->err < q->err ? -1 : 1;
    if (p->t != q->t) return p->t < q->t ? -1 : 1;
    return p->e < q->e ? -1 : (p->e > q->e);
}

int oracle_evaluate(const rt3d_point* est, uint64_t n_est, const rt3d_point* truth, uint64_t n_truth,
                    double tau, double pitch, double* out7) {
    if (tau <= 0.0 || pitch <= 0.0) return 1;
    const uint64_t n = n_est + n_truth;
    ev_item* it = (ev_item*)malloc((n ? n : 1) * sizeof *it);
    for (uint64_t q = 0; q < n; ++q) {
        const rt3d_point* p = q < n_est ? &est[q] : &truth[q - n_est];
        it[q].cx = (int64_t)floor(p->x / pitch);
        it[q].cy = (int64_t)floor(p->y / pitch);
        it[q].id = (uint32_t)q;
    }
    qsort(it, n, sizeof *it, ev_item_cmp);
    uint8_t* e_used = (uint8_t*)calloc(n_est ? n_est : 1, 1);
    uint8_t* t_used = (uint8_t*)calloc(n_truth ? n_truth : 1, 1);
    double sq_depth = 0.0, abs_intensity = 0.0;
    uint64_t matched = 0;
    for (uint64_t a = 0; a < n;) {
        uint64_t b = a, ne = 0;
        while (b < n && it[b].cx == it[a].cx && it[b].cy == it[a].cy) {
            ne += it[b].id < n_est;
            ++b;
        }
        const uint64_t nt = (b - a) - ne;
        ev_pair* pr = (ev_pair*)malloc((ne * nt ? ne * nt : 1) * sizeof *pr);
        uint64_t np = 0;
        for (uint64_t i = a; i < a + ne; ++i)
            for (uint64_t j = a + ne; j < b; ++j) {
                const uint32_t e = it[i].id, t = it[j].id - (uint32_t)n_est;
                const double err = fabs(est[e].z - truth[t].z);
                if (err <= tau) {
                    pr[np].err = err;
                    pr[np].e = e;
                    pr[np].t = t;
                    ++np;
                }
            }
        qsort(pr, np, sizeof *pr, ev_pair_cmp);
        for (uint64_t k = 0; k < np; ++k) {
            if (e_used[pr[k].e] || t_used[pr[k].t]) continue;
            e_used[pr[k].e] = t_used[pr[k].t] = 1;
            ++matched;
            sq_depth += pr[k].err * pr[k].err;
            abs_intensity += fabs(est[pr[k].e].intensity - truth[pr[k].t].intensity);
        }
        free(pr);
        a = b;
    }
    free(it);
    free(e_used);
    free(t_used);
    out7[0] = n_truth ? (double)matched / (double)n_truth : 1.0;
    out7[1] = n_est ? (double)(n_est - matched) / (double)n_est : 0.0;
    out7[2] = matched ? sqrt(sq_depth / (double)matched) : 0.0;
    out7[3] = matched ? abs_intensity / (double)matched : 0.0;
    out7[4] = (double)n_truth;
    out7[5] = (double)n_est;
    out7[6] = (double)matched;
    return 0;
}
