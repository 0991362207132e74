// qmccpw_pca_x1_lb.cu -- PCA paths on DMMA tiles, X1 conditioning with a lookback option: the
// warp's c_j are staged in shared memory and each lane walks its path's upper envelope.
#ifndef QMCCPW_X1_EXP256
#define QMCCPW_X1_EXP256 1  // measured: PCA-X1 87.2 -> 85.1 ms, BB-X1 87.3 -> 85.3
#endif
#ifndef QMCCPW_EXP256
#define QMCCPW_EXP256 QMCCPW_X1_EXP256  // 256-entry exp table through L1 (qmccpw_math.cuh)
#endif
#include "qmccpw_pca.cuh"

namespace qmccpw {

cudaError_t launch_pca_x1_lb(const PathArgs& args, cudaStream_t st, bool* handled) {
    return args.owen ? launch_pca<kX1, true, true>(args, st, handled) : launch_pca<kX1, false, true>(args, st, handled);
}

}  // namespace qmccpw
