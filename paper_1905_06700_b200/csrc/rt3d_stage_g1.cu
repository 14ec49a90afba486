// rt3d_stage_g1.cu — stage kernels with a thread per pixel in the likelihood
// sweeps (large dense arrays; see rt3d_stage.cuh, sweep_node_thread).  The
// one-launch iteration (ST_ITER) is not built for this configuration.
#include "rt3d_stage.cuh"

namespace rt3d {

StageFn stage_fn_g1(int st) {
    static const StageFn tab[kNumStages] = {
        stage_kernel<ST_FIRST, 1>, stage_kernel<ST_DEPTH, 1>, stage_kernel<ST_INTENSITY, 1>,
        stage_kernel<ST_TAIL, 1>, nullptr};
    return tab[st];
}

}  // namespace rt3d
