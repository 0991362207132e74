// qmccpw_paths_x1.cu -- path kernels with X1 conditioning (Newton threshold; the
// lookback's upper envelope), QMC only.
#ifndef QMCCPW_X1_EXP256
#define QMCCPW_X1_EXP256 1  // measured: PCA-X1 87.2 -> 85.1 ms, BB-X1 87.3 -> 85.3
#endif
#ifndef QMCCPW_EXP256
#define QMCCPW_EXP256 QMCCPW_X1_EXP256  // 256-entry exp table through L1 (qmccpw_math.cuh)
#endif
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
