// qmccpw_pca_x1_owen.cu -- PCA paths on DMMA tiles, X1 conditioning, Owen-scrambled points.
#include "qmccpw_pca.cuh"

namespace qmccpw {

cudaError_t launch_pca_x1_owen(const PathArgs& args, cudaStream_t st, bool* handled) {
    return launch_pca<kX1, true>(args, st, handled);
}

}  // namespace qmccpw
