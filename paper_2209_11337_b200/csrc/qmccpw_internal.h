// qmccpw_internal.h -- structures shared by the host API (qmccpw_api.cu) and
// the sm_100a kernels (qmccpw_kernels.cu).  Not part of the public ABI.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace qmccpw {

constexpr int kMaxOpt = 3;            // options fused on one path per launch
constexpr int kCellPoints = 4096;     // points of one replicate per cell (block)
constexpr int kMaxDimGpu = 256;       // largest d the kernels support
constexpr int kNewtonIt = 2;          // X1 threshold: at least 2 Halley updates, then up to kNewtonMax
constexpr int kNewtonMax = 8;
// Halley's iteration converges cubically: once an update is below kHalleyTol (relative),
// the error it leaves is ~C |du|^3 << 1e-16, so that update is the last (predictive stop)
constexpr double kHalleyTol = 1e-6;

// ---- QMCCPW_CHECKED builds (scripts/checked_build.py -> libqmccpw_checked.so): device-side
// bounds asserts at the computed shared- and global-memory indices of the hot path, a memcheck
// substitute (compute-sanitizer is closed on the GPU pool).  A failed check executes __trap(),
// so the launch fails with cudaErrorLaunchFailure and the call returns QMCCPW_ECUDA.  In the
// production build the macros expand to nothing.
#ifndef QMCCPW_CHECKED
#define QMCCPW_CHECKED 0
#endif
#if QMCCPW_CHECKED && defined(__CUDA_ARCH__)
// [p, p + n) must lie inside the block's dynamic shared memory window
__device__ __forceinline__ void qmccpw_chk_dsmem(const void* p, size_t n) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    uint32_t dyn;
    asm volatile("mov.u32 %0, %%dynamic_smem_size;" : "=r"(dyn));
    const unsigned char* c = static_cast<const unsigned char*>(p);
    if (c < smem_raw || c + n > smem_raw + dyn) __trap();
}
#define QMCCPW_CHECK(cond) \
    do {                   \
        if (!(cond)) __trap(); \
    } while (0)
#define QMCCPW_CHK_SMEM(ptr) qmccpw_chk_dsmem((ptr), sizeof(*(ptr)))
#else
#define QMCCPW_CHECK(cond) \
    do {                   \
    } while (0)
#define QMCCPW_CHK_SMEM(ptr) \
    do {                     \
    } while (0)
#endif

enum Construction { kStd = 0, kBB = 1, kPca = 2 };
enum Conditioning { kW1 = 0, kX1 = 1 };
enum Method { kQmc = 0, kLr = 1, kMc = 2, kMcAv = 3 };
enum OptType { kArith = 0, kBinary = 1, kLookback = 2 };

// Everything one launch of the path kernel needs, passed BY VALUE as the
// kernel argument (no per-call host->device copy).
struct PathArgs {
    // geometry
    int d;
    int n_opt;
    int tpb_log2;            // threads per block = 2^tpb_log2
    int dim_begin;           // first Sobol' dimension consumed (1 when x_1 is not needed)
    uint64_t n_points;       // points per replicate
    uint64_t point_offset;   // first Sobol' index
    uint32_t n_reps;
    uint32_t rep_base;       // global index of local replicate 0 (LR counters; hooks)
    uint32_t cells_per_rep;
    uint64_t cell_begin;     // first global cell of this launch
    uint64_t cell_end;
    // market (shared by all options of the launch)
    double S0, r, sigma, T;
    double omega;            // r - sigma^2/2 (reading 1)
    double t1;               // T/d
    double sqrt_t1;          // sqrt(T/d) = sqrt(dt)
    double s;                // sigma sqrt(t1)
    double inv_s;            // 1/s
    double inv_sigma;
    double inv_S0;           // 1/S0
    double inv_d;            // 1/d
    double S0_inv_d;         // S0/d (the W1 sums are kept without S0)
    double2 wt[kMaxDimGpu];  // (omega t, sigma t) at t = j dt = t_{j+1} - t_1, j < d (W1Acc)
    double Dfac;             // e^{-rT}
    double Afac;             // e^{r(t1 - T)}
    double lnS0;
    double sqrtT;
    double bb_b[16];         // b_k = sqrt(T / 2^{k+1}), k = 1..m (index k)
    int bb_m;
    uint8_t bb_seq[kMaxDimGpu + 2];  // Sobol' dimension of the i-th normal consumed by the time-order
                                     // bridge (Alg. 4's consumption order), padded by repetition
    // options
    int has_lookback;        // track S~_max / argmax (lookback present)
    int tail_leader[kMaxOpt];  // first option with the same strike and statistic (shares psi etc.)
    int x1_need_arith[kMaxOpt];  // X1: some option of this leader's strike group is arithmetic
    int type[kMaxOpt];
    double K[kMaxOpt];
    double lnK[kMaxOpt];
    double lndK[kMaxOpt];    // ln(d K)
    double piv[kMaxOpt][4];  // pivots p_{o,q}
    // X1
    double mean_a;           // (1/d) sum_j a_j
    // tables (device pointers)
    const uint32_t* vscr;    // [n_reps][d][32] scrambled direction numbers
    const uint32_t* shift;   // [n_reps][d]
    const double* M;         // [M_ld][M_ld] path matrix (PCA), zero-padded to a multiple of 8
    const double* Mf;        // the same in pca_kernel's B-fragment order (launch_mma_bfrag); W1: rows minus row 0
    int M_ld;
    const double* a;         // [d] first column a_j of the path matrix (X1)
    const double* inv_sa;    // [d] 1/(sigma a_j)   (X1)
    // LR
    uint64_t seed;
    // outputs
    double* partials;        // [cell][partial_doubles_per_cell]
    int partial_stride;      // doubles per cell = n_opt*8 + 3
    // parity hook: per-path values out[(point index within range)][4] (NULL in production)
    double* path_out;
    int hook_option;         // option index whose values go to path_out
    int owen;                // 1: nested (Owen) scrambling, shift[] holds the per-dimension seeds
    int x1_lin;              // X1: a_j is linear in j (STD: constant, BB: t_j / sqrt(T)), d >= 2
};

// ---- portfolio (C5): up to kMaxPortfolio options in up to kMaxFamilies (sigma, T) families
// sharing S0, r, d; PCA-W1 on the tensor cores (d <= 128).
constexpr int kMaxPortfolio = 1024;
constexpr int kMaxFamilies = 8;

struct PortfolioOption {  // device table, one per option, ordered by type (see launch_portfolio_plan)
    int type;
    int family;
    int slot;      // the option's index in the call (its partial-row slot)
    int pad;
    double K, lnK;
    double piv[4];
};

struct Family {            // market constants of one (sigma, T) family
    double sigma, T, omega, t1, sqrt_t1, s, inv_s, inv_sigma, Dfac, Afac, sqrtT;
};

struct PortfolioArgs {
    int d, n_opt, n_fam, tpb_log2, M_ld;
    uint64_t n_points, point_offset;
    uint32_t n_reps, rep_base, cells_per_rep;
    uint64_t cell_begin, cell_end;
    double S0, r, lnS0;
    int has_lookback;
    Family fam[kMaxFamilies];
    const PortfolioOption* opts;  // [n_opt] device
    const uint32_t* vscr;
    const uint32_t* shift;
    const double* M;               // PCA of T = 1, [M_ld][M_ld]
    double* partials;
    int partial_stride;            // 8 n_opt + 3
    double* path_out;              // hook: [point][n_opt][4] or NULL
    int owen;                      // 1: nested (Owen) scrambling (see PathArgs)
};

cudaError_t launch_portfolio(const PortfolioArgs& args, cudaStream_t st);

// Launchers (qmccpw_kernels.cu).  All return cudaError_t of the launch.
cudaError_t launch_randomization(const uint32_t* d_base_v, const uint32_t* d_base_shift, int d, uint32_t n_reps,
                                 uint32_t rep_base, uint64_t seed, int mode, uint32_t* d_vscr, uint32_t* d_shift,
                                 cudaStream_t st);
cudaError_t launch_path_matrix(int construction, int d, int ld, double T, double sigma, double* d_M, double* d_a,
                               double* d_inv_sa, cudaStream_t st);
cudaError_t launch_mma_bfrag(const double* d_M, int ld, bool shift_row0, double* d_Mf, cudaStream_t st);
cudaError_t launch_gpca_rotate(double* d_M, int ld, int d, double T, double omega, double sigma, double* d_a,
                               double* d_inv_sa, cudaStream_t st);
cudaError_t launch_paths_x1(const PathArgs& args, int construction, cudaStream_t st, int* smem_out);
cudaError_t launch_pca_w1(const PathArgs& args, cudaStream_t st, bool* handled);  // handled = false: d not tiled
cudaError_t launch_pca_x1(const PathArgs& args, cudaStream_t st, bool* handled);
cudaError_t launch_paths(const PathArgs& args, int construction, int conditioning, int method, cudaStream_t st,
                         int* smem_bytes_out);
cudaError_t launch_reduce_cells(const double* d_partials, int stride, uint32_t rep_begin, uint32_t rep_end,
                                uint32_t cells_per_rep, double* d_rep_sums, cudaStream_t st);
cudaError_t launch_sobol_hook(const uint32_t* d_vscr, const uint32_t* d_shift, int d, uint32_t dim_begin,
                              uint32_t dim_end, uint64_t k_begin, uint64_t k_end, int owen, uint32_t* d_out,
                              cudaStream_t st);
cudaError_t launch_normals_hook(const uint32_t* d_vscr, const uint32_t* d_shift, int d, uint64_t k_begin,
                                uint64_t k_end, int method, uint64_t seed, uint32_t rep, int owen, double* d_out,
                                cudaStream_t st);

uint64_t& launch_counter();  // thread-local count of kernel launches

}  // namespace qmccpw
