// rt3d_stage_g4.cu — stage kernels with 4 lanes per pixel in the likelihood
// sweeps (see rt3d_stage.cuh).
#include "rt3d_stage.cuh"

namespace rt3d {

StageFn stage_fn_g4(int st) {
    static const StageFn tab[kNumStages] = {
        stage_kernel<ST_FIRST, 4>, stage_kernel<ST_DEPTH, 4>, stage_kernel<ST_INTENSITY, 4>,
        stage_kernel<ST_TAIL, 4>, stage_kernel<ST_ITER, 4>};
    return tab[st];
}

}  // namespace rt3d
