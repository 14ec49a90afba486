// Interface between rt3d.cu (session, C ABI) and rt3d_sim.cu (the forward
// simulator's photon sampling).  Kept separate so the
// sampling kernels rebuild without recompiling the reconstruction kernels.
#pragma once
#include <cuda_runtime.h>

#include <cstdint>

#include "rt3d_math.cuh"

namespace rt3d {

struct SimArgs {
    const IrfDev* irfs;         // one, or one per pixel
    const uint32_t* irf_of_pix; // nullptr: shared IRF
    const double* gain;         // f64[npix]
    const uint8_t* dead;        // u8[npix]
    const double* background;   // f64[npix], the true background rate per bin
    const uint32_t* boff;       // truth buckets: CSR by coarse pixel, cloud order
    const uint32_t* bpts;
    const double* pt_t;         // truth depth (bins), indexed by cloud index
    const double* pt_r;         // truth intensity (already scaled)
    int rows, cols, bins;
    uint64_t seed;
};

// Sample the cube on `stream`: per-pixel event counts, their exclusive scan
// into `off` (u32[npix+1]), then the events (uint2{bin,count}[off[npix]]),
// which are written into a buffer the caller sizes after reading off[npix]
// (`events` == nullptr on the first call).  `photons` receives
// {signal, background} totals.  Returns a cudaError_t.
cudaError_t sim_count(const SimArgs& a, uint32_t* counts, uint32_t* off,
                      unsigned long long* photons, void* scratch, size_t* scratch_bytes,
                      cudaStream_t stream);
cudaError_t sim_write(const SimArgs& a, const uint32_t* off, uint2* events, cudaStream_t stream);

}  // namespace rt3d
