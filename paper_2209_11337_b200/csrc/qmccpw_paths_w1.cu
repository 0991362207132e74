// qmccpw_paths_w1.cu -- path kernels with W1 conditioning (all methods) and the
// launch_paths dispatcher (X1 kernels: qmccpw_paths_x1.cu; PCA on DMMA: qmccpw_pca_*.cu).
#define QMCCPW_SMEM_TABLES 1  // exp / log tables in shared memory (see qmccpw_math.cuh)
#define QMCCPW_LOG1P_FACTORED 1  // (qmccpw_math.cuh fast_log)
#ifndef QMCCPW_EXP256
#define QMCCPW_EXP256 1  // (qmccpw_math.cuh fast_exp: 256-entry table, degree 4)
#endif
#ifndef QMCCPW_ICDF_SHIFTED_LOG
#define QMCCPW_ICDF_SHIFTED_LOG 1  // (qmccpw_math.cuh normal_from_u32_xn)
#endif
#include "qmccpw_paths.cuh"

#ifndef QMCCPW_BB_X1_MMA
#define QMCCPW_BB_X1_MMA 1
#endif
#ifndef QMCCPW_STD_X1_MMA
#define QMCCPW_STD_X1_MMA 0  // measured slower: C4 STD-X1 57.9 ms on the path kernel, 66.2 on the quad kernel
#endif

namespace qmccpw {

cudaError_t launch_paths(const PathArgs& args, int construction, int conditioning, int method, cudaStream_t st,
                         int* smem_out) {
    if (method == kLr) return launch_paths_t<kStd, kW1, kLr, false>(args, st, smem_out);
    if (method == kMc) return construction == kBB ? launch_paths_t<kBB, kW1, kMc, false>(args, st, smem_out)
                                                  : launch_paths_t<kStd, kW1, kMc, false>(args, st, smem_out);
    if (method == kMcAv) return construction == kBB ? launch_paths_t<kBB, kW1, kMcAv, false>(args, st, smem_out)
                                                    : launch_paths_t<kStd, kW1, kMcAv, false>(args, st, smem_out);
    if (method == kQmc && (construction == kPca ||
                           (conditioning == kX1 && !args.has_lookback &&
                            ((construction == kBB && QMCCPW_BB_X1_MMA) || (construction == kStd && QMCCPW_STD_X1_MMA))))) {
        // fragment-native tensor-core path for d <= 128 (BB-X1: the bridge's matrix, qmccpw_api.cu)
        bool handled = false;
        cudaError_t e = conditioning == kW1 ? launch_pca_w1(args, st, &handled) : launch_pca_x1(args, st, &handled);
        if (handled) return e;
    }
    if (conditioning == kX1) return launch_paths_x1(args, construction, st, smem_out);
    const bool ow = args.owen != 0;
    if (construction == kStd)
        return ow ? launch_paths_t<kStd, kW1, kQmc, true>(args, st, smem_out)
                  : launch_paths_t<kStd, kW1, kQmc, false>(args, st, smem_out);
    if (construction == kBB)
        return ow ? launch_paths_t<kBB, kW1, kQmc, true>(args, st, smem_out)
                  : launch_paths_t<kBB, kW1, kQmc, false>(args, st, smem_out);
    return ow ? launch_paths_t<kPca, kW1, kQmc, true>(args, st, smem_out)
              : launch_paths_t<kPca, kW1, kQmc, false>(args, st, smem_out);
}

}  // namespace qmccpw
