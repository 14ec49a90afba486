// rt3d_stage_g32.cu — stage kernels with 32 lanes per pixel in the likelihood
// sweeps (see rt3d_stage.cuh).
#include "rt3d_stage.cuh"

namespace rt3d {

StageFn stage_fn_g32(int st) {
    static const StageFn tab[kNumStages] = {
        stage_kernel<ST_FIRST, 32>, stage_kernel<ST_DEPTH, 32>, stage_kernel<ST_INTENSITY, 32>,
        stage_kernel<ST_TAIL, 32>, stage_kernel<ST_ITER, 32>};
    return tab[st];
}

}  // namespace rt3d
