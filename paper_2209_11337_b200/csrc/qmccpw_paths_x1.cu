// qmccpw_paths_x1.cu -- path kernels with X1 conditioning (Newton threshold; the
// lookback's upper envelope), QMC only.
#include "qmccpw_paths.cuh"

namespace qmccpw {

cudaError_t launch_paths_x1(const PathArgs& args, int construction, cudaStream_t st, int* smem_out) {
    const bool ow = args.owen != 0;
    if (construction == kStd)
        return ow ? launch_paths_t<kStd, kX1, kQmc, true>(args, st, smem_out)
                  : launch_paths_t<kStd, kX1, kQmc, false>(args, st, smem_out);
    if (construction == kBB)
        return ow ? launch_paths_t<kBB, kX1, kQmc, true>(args, st, smem_out)
                  : launch_paths_t<kBB, kX1, kQmc, false>(args, st, smem_out);
    return ow ? launch_paths_t<kPca, kX1, kQmc, true>(args, st, smem_out)
              : launch_paths_t<kPca, kX1, kQmc, false>(args, st, smem_out);
}

}  // namespace qmccpw
