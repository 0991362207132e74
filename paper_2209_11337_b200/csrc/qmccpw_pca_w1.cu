// qmccpw_pca_w1.cu -- PCA paths on DMMA tiles, W1 conditioning (d <= 128).
// exp / log tables in shared memory (see qmccpw_math.cuh)?
#ifndef QMCCPW_PCA_W1_SMEM_TABLES
#define QMCCPW_PCA_W1_SMEM_TABLES 1
#endif
#define QMCCPW_SMEM_TABLES QMCCPW_PCA_W1_SMEM_TABLES
#define QMCCPW_LOG1P_FACTORED 1  // (qmccpw_math.cuh fast_log)
#ifndef QMCCPW_EXP256
#define QMCCPW_EXP256 1  // (qmccpw_math.cuh fast_exp: 256-entry table, degree 4)
#endif
#ifndef QMCCPW_ICDF_SHIFTED_LOG
#define QMCCPW_ICDF_SHIFTED_LOG 1  // (qmccpw_math.cuh normal_from_u32_xn)
#endif
#ifndef QMCCPW_ICDF_SHIFTED_X2
#define QMCCPW_ICDF_SHIFTED_X2 1  // the paired normals too
#endif
#include "qmccpw_pca.cuh"

namespace qmccpw {

cudaError_t launch_pca_w1(const PathArgs& args, cudaStream_t st, bool* handled) {
    return args.owen ? launch_pca<kW1, true>(args, st, handled) : launch_pca<kW1, false>(args, st, handled);
}

}  // namespace qmccpw
