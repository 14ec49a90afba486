// TEST-ONLY stand-in for the FFTW3 calls in denoise.hpp:278-306
// (fftw_plan_dft_2d / fftw_execute / fftw_destroy_plan, unnormalised, FFTW
// sign convention).  FFTW is not installed in this image; this exists only so
// that oracle/Makefile can compile the reference headers unchanged.  The
// transform is a direct separable DFT with exactly reduced twiddle phases.
#pragma once

#include <cmath>
#include <complex>
#include <vector>

typedef double fftw_complex[2];
#define FFTW_FORWARD (-1)
#define FFTW_BACKWARD (+1)
#define FFTW_ESTIMATE (1U << 6)

struct fftw_plan_s {
    int nr, nc, sign;
    fftw_complex* in;
    fftw_complex* out;
};
typedef fftw_plan_s* fftw_plan;

inline fftw_plan fftw_plan_dft_2d(int nr, int nc, fftw_complex* in, fftw_complex* out, int sign,
                                  unsigned) {
    return new fftw_plan_s{nr, nc, sign, in, out};
}

inline void fftw_execute(const fftw_plan p) {
    const int nr = p->nr, nc = p->nc;
    const double pi = 3.14159265358979323846;
    std::vector<std::complex<double>> a(static_cast<size_t>(nr) * nc), b(a.size());
    for (size_t k = 0; k < a.size(); ++k) a[k] = {p->in[k][0], p->in[k][1]};
    // along columns of each row
    for (int r = 0; r < nr; ++r)
        for (int k = 0; k < nc; ++k) {
            std::complex<double> acc = 0.0;
            for (int x = 0; x < nc; ++x) {
                long long ph = (static_cast<long long>(k) * x) % nc;
                double ang = p->sign * 2.0 * pi * static_cast<double>(ph) / nc;
                acc += a[static_cast<size_t>(r) * nc + x] * std::complex<double>(std::cos(ang), std::sin(ang));
            }
            b[static_cast<size_t>(r) * nc + k] = acc;
        }
    // along rows of each column
    for (int c = 0; c < nc; ++c)
        for (int k = 0; k < nr; ++k) {
            std::complex<double> acc = 0.0;
            for (int x = 0; x < nr; ++x) {
                long long ph = (static_cast<long long>(k) * x) % nr;
                double ang = p->sign * 2.0 * pi * static_cast<double>(ph) / nr;
                acc += b[static_cast<size_t>(x) * nc + c] * std::complex<double>(std::cos(ang), std::sin(ang));
            }
            a[static_cast<size_t>(k) * nc + c] = acc;
        }
    for (size_t k = 0; k < a.size(); ++k) {
        p->out[k][0] = a[k].real();
        p->out[k][1] = a[k].imag();
    }
}

inline void fftw_destroy_plan(fftw_plan p) { delete p; }
