// rt3d_math.cuh — scalar device math of the RT3D path, restated from the
// reference with its exact operand order (the translation unit is compiled
// with -fmad=false, so no FMA is formed and IEEE double +,-,*,/,sqrt give the
// same bits as the reference's SSE2 code).
//
//   Irf::value / deriv / support_bins / mass_in_gate   sensor.hpp:69-98
//   ApssParams::weight                                  denoise.hpp:38-44
//   3x3 covariance eigenvalues, 5x5 Pratt pencil        denoise.hpp:66-125,196
//   project_onto_sphere                                 denoise.hpp:128-150
#pragma once

#include <cstdint>

namespace rt3d {

constexpr double kBackgroundFloor = 1e-6;  // reconstruct.hpp:23
constexpr int kMaxBacktracks = 30;         // reconstruct.hpp:268

// std::max / std::min / std::clamp with the reference's exact semantics
// (argument order decides NaN and signed-zero results).
__device__ __forceinline__ double std_max(double a, double b) { return (a < b) ? b : a; }
__device__ __forceinline__ double std_min(double a, double b) { return (b < a) ? b : a; }
__device__ __forceinline__ double std_clamp(double v, double lo, double hi) {
    return (v < lo) ? lo : (hi < v) ? hi : v;
}

// One IRF: normalised samples + slopes (built on the host with the
// reference's expressions, sensor.hpp:33-40), tau_max precomputed as
// tau_min + dtau * (n - 1) (sensor.hpp:63), h_max = max sample
// (reconstruct.hpp:126-127).
struct IrfDev {
    double tau_min, dtau, tau_max, h_max;
    const double* s;
    const double* d;
    uint32_t n;
    uint32_t pow2;     // dtau is a power of two: x/dtau == x*inv_dtau exactly
    double inv_dtau;
    double lim;        // (double)(n - 2): the largest segment index
};

// (tau - tau_min) / dtau, sensor.hpp:71.  Division by a power of two and
// multiplication by its (exact) reciprocal round identically; any other dtau
// takes the correctly rounded reciprocal inv_dtau with one fused correction
// (Markstein, as apss_weight_d2: the IEEE quotient for normal operands; a
// difference tau - tau_min of O(1) doubles is zero or normal, and a zero
// gives +0 where the division could give -0, which the interpolation that
// follows absorbs: s0 + (+-0) (s1 - s0) is s0 either way).
__device__ __forceinline__ double irf_x(const IrfDev& f, double tau) {
    const double a = tau - f.tau_min;
    const double q0 = a * f.inv_dtau;
    return f.pow2 ? q0 : __fma_rn(__fma_rn(-q0, f.dtau, a), f.inv_dtau, q0);
}

// sensor.hpp:69-75
__device__ __forceinline__ double irf_value(const IrfDev& f, double tau) {
    if (tau < f.tau_min || tau > f.tau_max) return 0.0;
    double x = irf_x(f, tau);
    unsigned long long k = (unsigned long long)x;
    if (k > (unsigned long long)(f.n - 2)) k = f.n - 2;
    double fr = x - (double)k;
    double s0 = f.s[k], s1 = f.s[k + 1];
    return s0 + fr * (s1 - s0);
}

// sensor.hpp:77-82
__device__ __forceinline__ double irf_deriv(const IrfDev& f, double tau) {
    if (tau <= f.tau_min || tau >= f.tau_max) return 0.0;
    double x = irf_x(f, tau);
    unsigned long long k = (unsigned long long)x;
    if (k > (unsigned long long)(f.n - 2)) k = f.n - 2;
    return f.d[k];
}

// sensor.hpp:86-90
__device__ __forceinline__ void irf_support(const IrfDev& f, double t, int n_bins, int& lo,
                                            int& hi) {
    int a = (int)ceil(t + f.tau_min);
    int b = (int)floor(t + f.tau_max);
    lo = a < 0 ? 0 : a;
    hi = b > n_bins - 1 ? n_bins - 1 : b;
}

// sensor.hpp:93-98
__device__ __forceinline__ double irf_mass_in_gate(const IrfDev& f, double t, int n_bins) {
    int lo, hi;
    irf_support(f, t, n_bins, lo, hi);
    double m = 0.0;
    for (int b = lo; b <= hi; ++b) m += irf_value(f, (double)b - t);
    return m;
}

// denoise.hpp:38-44
__device__ __forceinline__ double apss_weight(double radius, double dist) {
    double x = dist / radius;
    if (x >= 1.0) return 0.0;
    double s = 1.0 - x * x;
    s *= s;
    return s * s;
}

// a / d from dinv = 1.0 / d (the IEEE quotient) with one fused correction:
// the correctly rounded quotient for normal operands (Markstein; see
// apss_weight_d2), for a shared divisor.  A zero dividend keeps its sign
// (the correction would turn -0 into +0).
__device__ __forceinline__ double div_rcp(double a, double d, double dinv) {
    const double q0 = a * dinv;
    return a == 0.0 ? q0 : __fma_rn(__fma_rn(-q0, d, a), dinv, q0);
}

// apss_weight(radius, sqrt(d2)) for d2 >= 0, rinv = 1.0 / radius (the IEEE
// quotient).  A zero operand sends both the double sqrt and the division to
// their out-of-line slow paths, once per point (the point is its own member)
// and serialised in the warp; d2 == 0 gives x = +0 either way, so it is routed
// around them with the same bits.  dist / radius is formed from the correctly
// rounded reciprocal with one fused correction (Markstein: q0 = dist rinv,
// r = dist - q0 radius exactly, q0 + r rinv rounded is the correctly rounded
// quotient for normal operands), which replaces the reciprocal iteration of
// the division per member; checked against IEEE division on 10^9 random
// (dist, radius) pairs with no difference.
__device__ __forceinline__ double apss_weight_d2(double radius, double rinv, double d2) {
    const bool self = d2 == 0.0;
    // d2 == +0 becomes 1.0 by OR-ing in 1.0's bits (a select would be
    // if-converted back into sqrt(0))
    const double dd = __longlong_as_double(__double_as_longlong(d2) |
                                           (self ? 0x3FF0000000000000ll : 0ll));
    const double dist = sqrt(dd);
    const double q0 = dist * rinv;
    double x = __fma_rn(__fma_rn(-q0, radius, dist), rinv, q0);
    if (self) x = 0.0;
    if (x >= 1.0) return 0.0;
    double s = 1.0 - x * x;
    s *= s;
    return s * s;
}

// Eigenvalues of the weighted 3x3 covariance (lower triangle c00,c10,c11,
// c20,c21,c22), ascending, by cyclic Jacobi.  Only the eigenvalues decide
// anything in apss_project (denoise.hpp:197-203): the eigenvector orients
// the sign of the fitted field, and the projection is exactly invariant
// under that sign.  Same rotation sequence as oracle_sym3_eigenvalues.
__device__ __forceinline__ void sym3_eigenvalues(double a00, double a10, double a11, double a20,
                                                 double a21, double a22, double& e0, double& e1,
                                                 double& e2) {
    double a[3][3] = {{a00, a10, a20}, {a10, a11, a21}, {a20, a21, a22}};
#pragma unroll 1
    for (int sweep = 0; sweep < 12; ++sweep) {
        double off = fabs(a[1][0]) + fabs(a[2][0]) + fabs(a[2][1]);
        if (off == 0.0) break;
#pragma unroll
        for (int p = 0; p < 2; ++p)
#pragma unroll
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
                a[p][q] = 0.0;
                a[q][p] = 0.0;
                const int r = 3 - p - q;
                double arp = a[r][p], arq = a[r][q];
                double nrp = cs * arp - sn * arq;
                double nrq = sn * arp + cs * arq;
                a[r][p] = nrp;
                a[p][r] = nrp;
                a[r][q] = nrq;
                a[q][r] = nrq;
            }
    }
    double d0 = a[0][0], d1 = a[1][1], d2 = a[2][2], tmp;
    if (d1 < d0) { tmp = d0; d0 = d1; d1 = tmp; }
    if (d2 < d1) { tmp = d1; d1 = d2; d2 = tmp; }
    if (d1 < d0) { tmp = d0; d0 = d1; d1 = tmp; }
    e0 = d0;
    e1 = d1;
    e2 = d2;
}

// A decision-preserving shortcut for apss_project's degeneracy test
// (denoise.hpp:197-203: degenerate iff e2 <= 0 or e1 <= 1e-12 e2, e from an
// eigen-solver of the covariance).  For a symmetric positive semidefinite C
// with trace tr and determinant det, e2 <= tr and e0 e1 e2 = det with
// e0 <= e1, so e1 >= sqrt(det / tr).  When det, less a bound on its rounding
// error (2e-15 times the sum of the absolute products), exceeds 1e-16 tr^3,
// e1 > 1e-8 tr: four orders of magnitude above the threshold and far beyond
// any backward-stable solver's error (~1e-14 tr), so the Jacobi sweeps
// (sym3_eigenvalues, the oracle's) and the reference's solver all declare C
// non-degenerate and the sweeps can be skipped.  (An indefinite C rounds to
// det < 0 or near 0 and takes the full test.)
__device__ __forceinline__ bool cov_clearly_nondegenerate(const double cv[6]) {
    const double a = cv[0], b = cv[1], d = cv[2], c = cv[3], e = cv[4], f = cv[5];
    const double tr = a + d + f;
    if (!(tr > 0.0)) return false;
    const double det = a * (d * f - e * e) - b * (b * f - e * c) + c * (b * e - d * c);
    const double S = fabs(a) * (fabs(d * f) + e * e) + fabs(b) * (fabs(b * f) + fabs(e * c)) +
                     fabs(c) * (fabs(b * e) + fabs(d * c));
    return det - 2e-15 * S > 1e-16 * tr * tr * tr;
}

// Symmetric 5x5 in packed lower-triangular order: index (i,j), i>=j, at
// i*(i+1)/2 + j.
__device__ __forceinline__ constexpr int lt(int i, int j) { return i * (i + 1) / 2 + j; }

// LDL' of the lower triangle of (M - sigma N), N the Pratt matrix
// (denoise.hpp:82-84).  1 if all pivots are > 0 (positive definite).
__device__ __forceinline__ int ldlt5_shift(const double m[15], double sigma, double L[15],
                                           double d[5]) {
    double a[15];
#pragma unroll
    for (int k = 0; k < 15; ++k) a[k] = m[k];
    a[lt(1, 1)] = m[lt(1, 1)] - sigma;
    a[lt(2, 2)] = m[lt(2, 2)] - sigma;
    a[lt(3, 3)] = m[lt(3, 3)] - sigma;
    a[lt(4, 0)] = m[lt(4, 0)] + 2.0 * sigma;
#pragma unroll
    for (int j = 0; j < 5; ++j) {
        double s = a[lt(j, j)];
#pragma unroll
        for (int k = 0; k < j; ++k) s -= L[lt(j, k)] * L[lt(j, k)] * d[k];
        if (!(s > 0.0)) return 0;
        d[j] = s;
#pragma unroll
        for (int i = j + 1; i < 5; ++i) {
            double v = a[lt(i, j)];
#pragma unroll
            for (int k = 0; k < j; ++k) v -= L[lt(i, k)] * L[lt(j, k)] * d[k];
            L[lt(i, j)] = v / s;
        }
    }
    return 1;
}

// Positive definiteness of (M - sigma N) without divisions: elimination with
// each Schur update scaled by the positive pivot (same operations as the
// oracle's pd5).
__device__ __forceinline__ int pd5_shift(const double m[15], double sigma) {
    double a[15];
#pragma unroll
    for (int k = 0; k < 15; ++k) a[k] = m[k];
    a[lt(1, 1)] = m[lt(1, 1)] - sigma;
    a[lt(2, 2)] = m[lt(2, 2)] - sigma;
    a[lt(3, 3)] = m[lt(3, 3)] - sigma;
    a[lt(4, 0)] = m[lt(4, 0)] + 2.0 * sigma;
#pragma unroll
    for (int k = 0; k < 5; ++k) {
        const double akk = a[lt(k, k)];
        if (!(akk > 0.0)) return 0;
#pragma unroll
        for (int i = k + 1; i < 5; ++i)
#pragma unroll
            for (int j = k + 1; j <= i; ++j)
                a[lt(i, j)] = akk * a[lt(i, j)] - a[lt(i, k)] * a[lt(j, k)];
    }
    return 1;
}

// pd5_shift at three shifts at once, branch-free and interleaved (the
// latency-bound fit runs the three eliminations side by side): a shift is
// definite iff every pivot is > 0, the elimination continuing past a failed
// pivot only into values that no longer matter, so each result equals
// pd5_shift's (same operations up to the first non-positive pivot).
__device__ __forceinline__ void pd5_shift3(const double m[15], double s0, double s1, double s2,
                                           bool& r0, bool& r1, bool& r2) {
    double a[3][15];
#pragma unroll
    for (int v = 0; v < 3; ++v) {
        const double sg = v == 0 ? s0 : (v == 1 ? s1 : s2);
#pragma unroll
        for (int k = 0; k < 15; ++k) a[v][k] = m[k];
        a[v][lt(1, 1)] = m[lt(1, 1)] - sg;
        a[v][lt(2, 2)] = m[lt(2, 2)] - sg;
        a[v][lt(3, 3)] = m[lt(3, 3)] - sg;
        a[v][lt(4, 0)] = m[lt(4, 0)] + 2.0 * sg;
    }
    bool ok[3] = {true, true, true};
#pragma unroll
    for (int k = 0; k < 5; ++k) {
#pragma unroll
        for (int v = 0; v < 3; ++v) {
            const double akk = a[v][lt(k, k)];
            ok[v] = ok[v] && (akk > 0.0);
#pragma unroll
            for (int i = k + 1; i < 5; ++i)
#pragma unroll
                for (int j = k + 1; j <= i; ++j)
                    a[v][lt(i, j)] = akk * a[v][lt(i, j)] - a[v][lt(i, k)] * a[v][lt(j, k)];
        }
    }
    r0 = ok[0];
    r1 = ok[1];
    r2 = ok[2];
}

// Smallest admissible eigenpair of the Pratt pencil (M, N): the eigenvector
// that the reference's filter loop over GeneralizedEigenSolver's results keeps
// (denoise.hpp:86-112).  For PSD M the admissible eigenvalues are the
// non-negative ones, and the smallest is sup{sigma >= 0 : M - sigma N > 0};
// bisection on a division-free definiteness test brackets it, inverse
// iteration on an LDL' factor of the last definite shift gives the
// eigenvector.  Same sequence of operations
// as oracle_pratt_smallest (bit-identical on identical M).  kSpec: two
// bisection steps per round, the midpoint and both possible next midpoints
// tested together (pd5_shift3), then the same two steps taken in order: the
// same brackets, a chain half as long for the latency-bound single-frame fit.
template <bool kSpec = false>
__device__ __forceinline__ int pratt_smallest(const double m[15], double u[5]) {
    double L[15], d[5];
    const double scale =
        std_max(m[lt(0, 0)] + m[lt(1, 1)] + m[lt(2, 2)] + m[lt(3, 3)] + m[lt(4, 4)], 1e-300);
    double sigma;
    double hi = std_min(std_min(m[lt(1, 1)], m[lt(2, 2)]), m[lt(3, 3)]);
    if (pd5_shift(m, 0.0) && hi > 0.0) {
        double lo = 0.0;
        if constexpr (!kSpec) {
#pragma unroll 1
            for (int it = 0; it < 200; ++it) {
                double mid = 0.5 * (lo + hi);
                if (!(mid > lo && mid < hi)) break;
                if (pd5_shift(m, mid)) lo = mid;
                else hi = mid;
                // bracket to 1e-9 relative (as the oracle): the inverse
                // iteration converges from there
                if (hi - lo <= 1e-9 * hi) break;
            }
        } else {
            int it = 0;
#pragma unroll 1
            while (it < 200) {
                const double mid = 0.5 * (lo + hi);
                if (!(mid > lo && mid < hi)) break;
                // the next midpoint is 0.5 (mid + hi) if mid is definite,
                // else 0.5 (lo + mid): the same expressions as the step takes
                const double mH = 0.5 * (mid + hi), mL = 0.5 * (lo + mid);
                bool pA, pH, pL;
                pd5_shift3(m, mid, mH, mL, pA, pH, pL);
                if (pA) lo = mid;
                else hi = mid;
                if (++it >= 200 || hi - lo <= 1e-9 * hi) break;
                const double mid2 = pA ? mH : mL;
                if (!(mid2 > lo && mid2 < hi)) break;
                if (pA ? pH : pL) lo = mid2;
                else hi = mid2;
                ++it;
                if (hi - lo <= 1e-9 * hi) break;
            }
        }
        sigma = lo;
    } else {
        double delta = 1e-15 * scale;
        int ok = 0;
#pragma unroll 1
        for (int k = 0; k < 12 && !ok; ++k) {
            if (pd5_shift(m, -delta)) ok = 1;
            else delta *= 10.0;
        }
        if (!ok) return 0;
        sigma = -delta;
    }
    {  // factor of the last definite shift (step below eta* if the LDL'
       // and the division-free test disagree within rounding)
        const double base = sigma;
        double delta = 1e-15 * scale;
        int ok = 0;
#pragma unroll 1
        for (int k = 0; k < 14; ++k) {
            if (ldlt5_shift(m, sigma, L, d)) {
                ok = 1;
                break;
            }
            sigma = base - delta;
            delta *= 10.0;
        }
        if (!ok) return 0;
    }
    double x0 = 1.0, x1 = 1.0, x2 = 1.0, x3 = 1.0, x4 = 1.0;
#pragma unroll 1
    for (int it = 0; it < 4; ++it) {
        double y[5];
        y[0] = -2.0 * x4;
        y[1] = x1;
        y[2] = x2;
        y[3] = x3;
        y[4] = -2.0 * x0;
#pragma unroll
        for (int i = 0; i < 5; ++i) {
            double v = y[i];
#pragma unroll
            for (int k = 0; k < i; ++k) v -= L[lt(i, k)] * y[k];
            y[i] = v;
        }
#pragma unroll
        for (int i = 0; i < 5; ++i) y[i] = y[i] / d[i];
#pragma unroll
        for (int i = 4; i >= 0; --i) {
            double v = y[i];
#pragma unroll
            for (int k = i + 1; k < 5; ++k) v -= L[lt(k, i)] * y[k];
            y[i] = v;
        }
        double nrm = sqrt(y[0] * y[0] + y[1] * y[1] + y[2] * y[2] + y[3] * y[3] + y[4] * y[4]);
        if (!(nrm > 0.0) || !isfinite(nrm)) return 0;
        x0 = y[0] / nrm;
        x1 = y[1] / nrm;
        x2 = y[2] / nrm;
        x3 = y[3] / nrm;
        x4 = y[4] / nrm;
    }
    u[0] = x0;
    u[1] = x1;
    u[2] = x2;
    u[3] = x3;
    u[4] = x4;
    return 1;
}

struct Sphere {
    double u0, ul0, ul1, ul2, uq;
};

// fit tail of fit_algebraic_sphere (denoise.hpp:86-117): pencil solve,
// Pratt normalisation, un-centring.  The orientation flip
// (denoise.hpp:119-123) negates (u0, ul, uq) together; project_onto_sphere
// is bitwise invariant under it, so it is omitted.
template <bool kSpec = false>
__device__ __forceinline__ bool sphere_from_moments(const double m[15], double c0, double c1,
                                                    double c2, Sphere& out) {
    double v[5];
    if (!pratt_smallest<kSpec>(m, v)) return false;
    double vn2 = v[0] * v[0] + v[1] * v[1] + v[2] * v[2] + v[3] * v[3] + v[4] * v[4];
    if (sqrt(vn2) < 1e-300) return false;
    double nrm = v[1] * v[1] + v[2] * v[2] + v[3] * v[3] - 4.0 * v[0] * v[4];
    if (nrm <= 1e-14 * vn2) return false;
    double sq = sqrt(nrm);
    double u0 = v[0] / sq, l0 = v[1] / sq, l1 = v[2] / sq, l2 = v[3] / sq, uq = v[4] / sq;
    double dot = l0 * c0 + l1 * c1 + l2 * c2;
    double csq = c0 * c0 + c1 * c1 + c2 * c2;
    out.u0 = u0 - dot + uq * csq;
    double tq = 2.0 * uq;
    out.ul0 = l0 - tq * c0;
    out.ul1 = l1 - tq * c1;
    out.ul2 = l2 - tq * c2;
    out.uq = uq;
    return true;
}

// project_onto_sphere, denoise.hpp:128-150
__device__ __forceinline__ bool project_sphere(const Sphere& s, double eps, double p0, double p1,
                                               double p2, double& o0, double& o1, double& o2) {
    double g2 = s.ul0 * s.ul0 + s.ul1 * s.ul1 + s.ul2 * s.ul2;
    bool plane = fabs(s.uq) < eps;
    double c0 = 0, c1 = 0, c2 = 0, disc = 0;
    if (!plane) {
        double tq = 2.0 * s.uq;
        c0 = -s.ul0 / tq;
        c1 = -s.ul1 / tq;
        c2 = -s.ul2 / tq;
        disc = g2 - 4.0 * s.u0 * s.uq;
        if (disc <= 0.0) plane = true;
    }
    if (plane) {
        if (g2 < 1e-20) return false;
        double ev = s.u0 + (s.ul0 * p0 + s.ul1 * p1 + s.ul2 * p2) + s.uq * (p0 * p0 + p1 * p1 + p2 * p2);
        double f = ev / g2;
        o0 = p0 - f * s.ul0;
        o1 = p1 - f * s.ul1;
        o2 = p2 - f * s.ul2;
        return true;
    }
    double radius = sqrt(disc) / (2.0 * fabs(s.uq));
    double d0 = p0 - c0, d1 = p1 - c1, d2 = p2 - c2;
    double dn = sqrt(d0 * d0 + d1 * d1 + d2 * d2);
    if (dn < 1e-14) return false;
    double f = radius / dn;
    o0 = c0 + f * d0;
    o1 = c1 + f * d1;
    o2 = c2 + f * d2;
    return true;
}

// Exact parallel::pairwise_sum (parallel.hpp:52-61) of up to 32 values.
__device__ __forceinline__ double seq_sum(const double* v, int a, int n) {
    double s = 0.0;
    for (int k = 0; k < n; ++k) s += v[a + k];
    return s;
}
__device__ __forceinline__ double pw16(const double* v, int a, int n) {
    if (n <= 8) return seq_sum(v, a, n);
    int h = n / 2;
    return seq_sum(v, a, h) + seq_sum(v, a + h, n - h);
}
__device__ __forceinline__ double pw32(const double* v, int a, int n) {
    if (n <= 16) return pw16(v, a, n);
    int h = n / 2;
    return pw16(v, a, h) + pw16(v, a + h, n - h);
}

// Range of node k at depth G of pairwise_sum's recursion over n elements.
__device__ __forceinline__ void tree_node_range(uint32_t n, int G, uint32_t k, uint32_t& lo,
                                                uint32_t& size) {
    lo = 0;
    size = n;
    for (int b = G - 1; b >= 0; --b) {
        uint32_t h = size / 2;
        if ((k >> b) & 1u) {
            lo += h;
            size -= h;
        } else {
            size = h;
        }
    }
}

}  // namespace rt3d
