// Forward simulator photon sampling on the device: simulate_cube's per-pixel
// loop (simulate.hpp:181-205) with rate_profile (likelihood.hpp:80-95) and
// CounterRng::next_poisson (rng.hpp:11-98).
//
// The reference's RNG is already counter-based, keyed by (seed, pixel, bin,
// stream), so every (pixel, bin) sample is independent of every other and of
// the thread layout: one warp per pixel, one lane per bin in 32-bin chunks.
// The rate at a bin is accumulated in the reference's order (background,
// then the pixel's truth points in cloud order, each g*r*h) with
// -fmad=false, so lambda is bit-identical; the samplers use libdevice's
// exp/log/lgamma where the reference uses glibc's (both within 1 ulp), so a
// sample can differ only where a uniform lands within an ulp of a decision
// boundary (tests/test_sim.py measures the agreement).
//
// Two passes over the same samples (they are recomputed, not stored): count
// the active bins per pixel, exclusive-scan into the CSR offsets, write (the
// write pass stops at a pixel's last event).  The RNG key chain and the
// background's exp(-lambda) are hoisted per pixel.
#include <cub/cub.cuh>

#include "rt3d_sim.cuh"

namespace rt3d {
namespace {

constexpr uint64_t kGamma = 0x9E3779B97F4A7C15ull;

__device__ __forceinline__ uint64_t mix64(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

// CounterRng (rng.hpp:11-40).  The constructor's chain
//   base = mix(mix(mix(mix(a+G) ^ mix(b+2G)) ^ mix(c+3G)) ^ mix(d+5G))
// is evaluated in pieces: the seed and pixel terms once per pixel, the bin
// term once per bin for both streams; the values are the same.
struct Crng {
    uint64_t base, counter;
    __device__ explicit Crng(uint64_t b) : base(b), counter(0) {}
    __device__ uint64_t next_u64() { return mix64(base + (++counter) * kGamma); }
    __device__ double next_unit() {
        return ((double)(next_u64() >> 11) + 0.5) * 0x1.0p-53;
    }
    // rng.hpp:52-61 (limit = exp(-lambda), hoisted by the caller when lambda
    // is the same for every bin of a pixel)
    __device__ uint32_t inversion(double limit) {
        uint32_t k = 0;
        double p = 1.0;
        do {
            ++k;
            p *= next_unit();
        } while (p > limit);
        return k - 1;
    }
    // PTRD, rng.hpp:63-96
    __device__ uint32_t ptrd(double lambda) {
        const double slam = sqrt(lambda);
        const double loglam = log(lambda);
        const double b = 0.931 + 2.53 * slam;
        const double a = -0.059 + 0.02483 * b;
        const double inv_alpha = 1.1239 + 1.1328 / (b - 3.4);
        const double vr = 0.9277 - 3.6224 / (b - 2.0);
        for (;;) {
            double u;
            double v = next_unit();
            if (v <= 0.86 * vr) {
                u = v / vr - 0.43;
                return (uint32_t)floor((2.0 * a / (0.5 - fabs(u)) + b) * u + lambda + 0.445);
            }
            if (v >= vr) {
                u = next_unit() - 0.5;
            } else {
                u = v / vr - 0.93;
                u = (u < 0 ? -0.5 : 0.5) - u;
                v = next_unit() * vr;
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
    __device__ uint32_t poisson(double lambda, double limit) {
        if (!(lambda > 0.0)) return 0;
        if (lambda < 10.0) return inversion(limit);
        return ptrd(lambda);
    }
};

// Per-pixel constants of the sampler.
struct PixelRng {
    uint64_t base_px;  // mix(mix(seed+G) ^ mix(p+2G))
    uint64_t m1, m2;   // mix(1+5G), mix(2+5G): the stream terms
    double lam_bg, limit_bg;
};

__device__ __forceinline__ PixelRng pixel_rng(const SimArgs& a, uint32_t p, double g) {
    PixelRng r;
    r.base_px = mix64(mix64(a.seed + kGamma) ^ mix64((uint64_t)p + 2 * kGamma));
    r.m1 = mix64(1 + 5 * kGamma);
    r.m2 = mix64(2 + 5 * kGamma);
    r.lam_bg = g * a.background[p];
    r.limit_bg = exp(-r.lam_bg);
    return r;
}

// One lane's bin: {signal, background} photons (simulate.hpp:190-201).
__device__ __forceinline__ uint2 sample_bin(const SimArgs& a, const IrfDev& f, const PixelRng& R,
                                            uint32_t p, double g, int t, uint32_t k0,
                                            uint32_t k1) {
    const double lam_bg = R.lam_bg;
    double lam = lam_bg;
    for (uint32_t k = k0; k < k1; ++k) {
        const uint32_t q = __ldg(&a.bpts[k]);
        const double tp = __ldg(&a.pt_t[q]);
        int lo, hi;
        irf_support(f, tp, a.bins, lo, hi);
        if (t >= lo && t <= hi) lam += g * __ldg(&a.pt_r[q]) * irf_value(f, (double)t - tp);
    }
    const double d = lam - lam_bg;
    const double lam_sig = d > 0.0 ? d : 0.0;
    uint32_t zs = 0, zb = 0;
    const uint64_t h = mix64(R.base_px ^ mix64((uint64_t)t + 3 * kGamma));
    if (lam_sig > 0.0) zs = Crng(mix64(h ^ R.m1)).poisson(lam_sig, lam_sig < 10.0 ? exp(-lam_sig) : 0.0);
    if (lam_bg > 0.0) zb = Crng(mix64(h ^ R.m2)).poisson(lam_bg, R.limit_bg);
    return make_uint2(zs, zb);
}

template <bool WRITE>
__global__ void __launch_bounds__(256) sim_kernel(SimArgs a, uint32_t* counts,
                                                  unsigned long long* photons,
                                                  const uint32_t* off, uint2* events) {
    const uint32_t npix = (uint32_t)a.rows * (uint32_t)a.cols;
    const uint32_t p = blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32;
    const int lane = threadIdx.x & 31;
    unsigned long long sig = 0, bgp = 0;
    if (p < npix) {
        const double g = a.dead[p] ? 0.0 : a.gain[p];  // effective_gain, sensor.hpp:166-168
        uint32_t n = 0;
        if (g != 0.0) {
            const IrfDev& f = a.irf_of_pix ? a.irfs[a.irf_of_pix[p]] : a.irfs[0];
            const uint32_t k0 = a.boff[p], k1 = a.boff[p + 1];
            uint32_t base = WRITE ? off[p] : 0;
            const uint32_t end = WRITE ? off[p + 1] : 0;
            if (WRITE && end == base) return;  // no events: nothing to write
            const PixelRng R = pixel_rng(a, p, g);
            for (int t0 = 0; t0 < a.bins; t0 += 32) {
                const int t = t0 + lane;
                uint2 z = make_uint2(0, 0);
                if (t < a.bins) z = sample_bin(a, f, R, p, g, t, k0, k1);
                const uint32_t tot = z.x + z.y;
                const unsigned m = __ballot_sync(0xffffffffu, tot > 0);
                if (WRITE) {
                    if (tot > 0)
                        events[base + __popc(m & ((1u << lane) - 1))] = make_uint2((uint32_t)t, tot);
                    base += __popc(m);
                    if (base == end) break;  // the pixel's last event is written
                } else {
                    n += __popc(m);
                    sig += z.x;
                    bgp += z.y;
                }
            }
        }
        if (!WRITE && lane == 0) counts[p] = n;
    }
    if (!WRITE) {
        for (int o = 16; o > 0; o >>= 1) {
            sig += __shfl_xor_sync(0xffffffffu, sig, o);
            bgp += __shfl_xor_sync(0xffffffffu, bgp, o);
        }
        if (lane == 0 && (sig | bgp)) {  // integer atomics: order-independent
            atomicAdd(&photons[0], sig);
            atomicAdd(&photons[1], bgp);
        }
    }
}

}  // namespace

cudaError_t sim_count(const SimArgs& a, uint32_t* counts, uint32_t* off,
                      unsigned long long* photons, void* scratch, size_t* scratch_bytes,
                      cudaStream_t stream) {
    const uint32_t npix = (uint32_t)a.rows * (uint32_t)a.cols;
    if (!scratch) {
        return cub::DeviceScan::ExclusiveSum(nullptr, *scratch_bytes, counts, off, npix + 1,
                                             stream);
    }
    cudaError_t e = cudaMemsetAsync(photons, 0, 16, stream);
    if (e) return e;
    if ((e = cudaMemsetAsync(counts + npix, 0, 4, stream))) return e;
    const uint32_t wpb = 8;
    sim_kernel<false><<<(npix + wpb - 1) / wpb, wpb * 32, 0, stream>>>(a, counts, photons,
                                                                       nullptr, nullptr);
    if ((e = cudaGetLastError())) return e;
    return cub::DeviceScan::ExclusiveSum(scratch, *scratch_bytes, counts, off, npix + 1, stream);
}

cudaError_t sim_write(const SimArgs& a, const uint32_t* off, uint2* events, cudaStream_t stream) {
    const uint32_t npix = (uint32_t)a.rows * (uint32_t)a.cols;
    const uint32_t wpb = 8;
    sim_kernel<true><<<(npix + wpb - 1) / wpb, wpb * 32, 0, stream>>>(a, nullptr, nullptr, off,
                                                                      events);
    return cudaGetLastError();
}

}  // namespace rt3d
