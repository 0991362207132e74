// qmccpw_pca_x1_owen.cu -- PCA paths on DMMA tiles, X1 conditioning, Owen-scrambled points.
#ifndef QMCCPW_X1_EXP256
#define QMCCPW_X1_EXP256 1  // measured: PCA-X1 87.2 -> 85.1 ms, BB-X1 87.3 -> 85.3
#endif
#ifndef QMCCPW_EXP256
#define QMCCPW_EXP256 QMCCPW_X1_EXP256  // 256-entry exp table through L1 (qmccpw_math.cuh)
#endif
#include "qmccpw_pca.cuh"

namespace qmccpw {

cudaError_t launch_pca_x1_owen(const PathArgs& args, cudaStream_t st, bool* handled) {
    return launch_pca<kX1, true>(args, st, handled);
}

}  // namespace qmccpw
