// rt3d_stage_g3.cu — stage kernels with 3 lanes per pixel in the likelihood
// sweeps (see rt3d_stage.cuh).
#include "rt3d_stage.cuh"

namespace rt3d {

StageFn stage_fn_g3(int st) {
    static const StageFn tab[kNumStages] = {
        stage_kernel<ST_FIRST, 3>, stage_kernel<ST_DEPTH, 3>, stage_kernel<ST_INTENSITY, 3>,
        stage_kernel<ST_TAIL, 3>, stage_kernel<ST_ITER, 3>};
    return tab[st];
}

}  // namespace rt3d
