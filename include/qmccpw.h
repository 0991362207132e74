/*
 * qmccpw.h -- C ABI of the B200-native QMC-CPW hot path (arXiv 2209.11337).
 *
 * The library (paper_2209_11337_b200/libqmccpw.so) estimates the price and the
 * delta, vega and gamma of arithmetic Asian, binary Asian and fixed-strike
 * lookback calls by the Quasi-Monte Carlo conditional pathwise method of
 * PAPER.md Sec. 3.4 and Sec. 4.5, in FP64, on one
 * sm_100a GPU per call.  Citations "P:<n>" are lines of PAPER.md; readings of
 * silent or garbled passages are numbered as in DESIGN.md / SURVEY.md 8(c).
 *
 * Conventions for every function:
 *   - No C++ exception crosses the ABI; every function returns an int status
 *     (QMCCPW_OK or a negative QMCCPW_E* code) and, on failure, leaves a
 *     message for qmccpw_last_error().  Output buffers are written only on
 *     success.
 *   - Pointers named h_* / out are HOST memory owned by the caller; pointers
 *     named d_* are DEVICE memory (on cfg->device) owned by the caller.  The
 *     library owns only its cached device tables and scratch, freed by
 *     qmccpw_release().
 *   - Calls are synchronous: they return after results are on the host.  If
 *     cfg->stream is non-NULL the work is enqueued on that cudaStream_t and the
 *     call synchronises it before returning (qmccpw_partials excepted: it only
 *     enqueues).
 *   - The output bits are a function of the inputs only: launch geometry and
 *     the number of GPUs sharing the cells do not change them (Sec. 8(e)).
 *   - One in-flight call per (device, stream).  The per-call tables, library
 *     partials and pinned staging are keyed by (device, stream), so calls on
 *     different streams -- of one device or of several, from one host thread
 *     or several -- never share scratch: a qmccpw_partials still running on
 *     stream A is not disturbed by a call on stream B.  Calls on one stream
 *     are ordered by the stream.
 *   - There is no CPU fallback: without a usable sm_100a device every compute
 *     entry point returns QMCCPW_ECUDA.
 */
#ifndef QMCCPW_H
#define QMCCPW_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- status codes ----------------------------------------------------- */
enum {
    QMCCPW_OK = 0,
    QMCCPW_EINVAL = -1,       /* invalid argument (domain error, NULL pointer, range) */
    QMCCPW_EUNSUPPORTED = -2, /* valid but unsupported combination */
    QMCCPW_ECUDA = -3,        /* CUDA runtime / driver failure or no sm_100a device */
    QMCCPW_ENOMEM = -4        /* device or host allocation failed */
};

/* ---- enumerations ----------------------------------------------------- */
typedef enum {
    QMCCPW_ARITH_ASIAN_CALL = 0,  /* payoff e^{-rT}(S_A - K)^+ */
    QMCCPW_BINARY_ASIAN_CALL = 1, /* payoff e^{-rT} 1{S_A > K} */
    QMCCPW_LOOKBACK_CALL = 2      /* payoff e^{-rT}(max_j S(t_j) - K)^+ */
} qmccpw_option;

typedef enum {
    QMCCPW_STD = 0, /* standard recursion, Alg. 3 */
    QMCCPW_BB = 1,  /* Brownian bridge, Alg. 4; d must be 2^m */
    QMCCPW_PCA = 2, /* principal components of min(t_i,t_j) */
    QMCCPW_GPCA = 3 /* gradient-aligned PCA (reading 28): the PCA basis rotated by
                       a Householder reflection so that x_1 carries the whole gradient of the arithmetic
                       average at W = 0 (first column C s / sqrt(s^T C s), s_j = e^{omega t_j}); one market
                       per call (not for portfolios), same kernels and cost as PCA */
} qmccpw_construction;

typedef enum {
    QMCCPW_COND_W1 = 0, /* condition on W(t_1): the paper's variable separation */
    QMCCPW_COND_X1 = 1  /* condition on the first coordinate x_1 of the path matrix (north star):
                           arithmetic / binary threshold by Newton's method; lookback by the
                           closed-form threshold and its upper envelope */
} qmccpw_conditioning;

typedef enum {
    QMCCPW_QMC_CPW = 0,  /* randomised Sobol' + conditional pathwise estimators;
                            STD = the paper's QMC-CPW, BB = QMC+BB-CPW */
    QMCCPW_LR_MC = 1,    /* Monte Carlo likelihood-ratio baseline, P:604-629 (STD path only) */
    QMCCPW_MC_CPW = 2,   /* pseudo-random (Philox) normals + CPW estimators; STD/BB, W1 */
    QMCCPW_MC_AV_CPW = 3 /* MC-CPW with antithetic pairs x, -x averaged; STD/BB, W1;
                            n_points counts pairs */
} qmccpw_method;

typedef enum {
    QMCCPW_RAND_LMS_SHIFT = 0,     /* per-replicate left-matrix scramble + digital shift (reading 10) */
    QMCCPW_RAND_SHIFT = 1,         /* per-replicate digital shift only */
    QMCCPW_RAND_CURAND_COMPAT = 2, /* cuRAND QUASI_SCRAMBLED_SOBOL32; identical for every replicate */
    QMCCPW_RAND_NONE = 3,          /* plain Sobol' (cuRAND QUASI_SOBOL32) */
    QMCCPW_RAND_OWEN = 4           /* nested uniform (Owen) scrambling of every coordinate, per-replicate
                                      per-dimension seeds (reading 27): a hash-drawn
                                      random permutation tree (Laine-Karras / Burley 2020) on top of plain
                                      Sobol', so each replicate is an Owen-scrambled (t, m, s)-net */
} qmccpw_randomization;

/* ---- parameter blocks ------------------------------------------------- */
/* Market and contract.  Monitoring dates t_j = j T / d, j = 1..d.
 * S0, K, sigma, T finite and > 0; r finite; 1 <= d <= 256 on the GPU. */
typedef struct {
    double S0, K, r, sigma, T;
    int32_t d;
} qmccpw_params;

/* Method configuration.  NULL -> defaults: QMC_CPW, BB if d is a power of
 * two else STD, W1, LMS_SHIFT, seed 2209113370, point_offset 0, device =
 * the current device, stream = NULL (the legacy default stream). */
typedef struct {
    int32_t method, construction, conditioning, randomization;
    uint64_t seed;         /* keys the Philox4x32-10 randomisation / LR normals */
    uint64_t point_offset; /* first Sobol' index k; points k = offset + i, i < n_points */
    int32_t device;        /* CUDA device ordinal, or -1 for the current device */
    void* stream;          /* cudaStream_t or NULL */
} qmccpw_config;

/* Result for one option.  Index q: [0] price G, [1] delta, [2] vega, [3] gamma.
 *   mean[q]       C = (1/L) sum_l C_l, C_l the mean over the n_points of replicate l
 *   se[q]         sqrt(sum_l (C_l - C)^2 / (L (L-1)))             (NaN when L = 1)
 *   sigma_run[q]  sqrt(sum_l (C_l - C)^2 / L), the paper's error (NaN when L = 1)
 *   within_var[q] mean over l of the variance of the per-path values in replicate l */
typedef struct {
    double mean[4], se[4], sigma_run[4], within_var[4];
    uint64_t n_points;
    uint32_t n_replicates;
    uint64_t newton_unconverged; /* X1 paths whose threshold iteration (Halley) had not converged
                                    after 8 updates: last update > 1e-6 relative (expect 0) */
    uint64_t argmax_near_ties;   /* lookback paths with two S~(t_j) within 1e-12 in log (expect 0) */
} qmccpw_result;

/* ---- core entry points ------------------------------------------------ */
/* One option.  n_points >= 1 Sobol' points per replicate (point_offset +
 * n_points <= 2^32), n_replicates in [1, 2^24).
 * EINVAL: non-finite / non-positive S0, K, sigma, T; non-finite r; d outside
 *   [1, 1024]; n_points = 0 or beyond the Sobol32 period; n_replicates = 0;
 *   NULL p or out.
 * EUNSUPPORTED: BB with d != 2^m (Alg. 4 is defined for 2^m steps);
 *   LR_MC with a construction other than STD;
 *   MC_CPW / MC_AV_CPW with PCA, GPCA or X1;
 *   d > 256 on the GPU. */
int qmccpw_price_greeks(int32_t option, const qmccpw_params* p, uint64_t n_points, uint32_t n_replicates,
                        const qmccpw_config* cfg, qmccpw_result* out);

/* n_options options priced on the SAME points in one pass (one path feeds all
 * of them, SURVEY.md 8(a5) "option fusion").  options[i], p[i] for i <
 * n_options; out[i] receives option i.  All p[i] share S0, r and d.
 *  - 1..3 options that also share sigma and T (may differ in K): the fused
 *    path kernel, any method / construction / conditioning;
 *  - otherwise (up to 1024 options in up to 8 (sigma, T) families; the C5
 *    portfolio): the portfolio kernel, QMC-CPW with PCA + W1 only and d <= 128
 *    (padded to 8, 16, 32, 64 or 128); W(T) = sqrt(T) W(1) and the S~
 *    statistics are shared per family, the tails run per option.
 * EUNSUPPORTED for other combinations. */
int qmccpw_price_greeks_batch(const int32_t* options, const qmccpw_params* p, int32_t n_options,
                              uint64_t n_points, uint32_t n_replicates, const qmccpw_config* cfg,
                              qmccpw_result* out);

/* ---- multi-GPU building blocks (the caller owns the process group) ------
 * The work is split into cells: cell c = (replicate l, block b of 4096
 * consecutive point indices), c = l * cells_per_replicate + b.  Each cell's
 * partial is partial_doubles_per_cell doubles:
 *   [o][q][0] = sum over its points of (f - pivot_{o,q}),
 *   [o][q][1] = sum of (f - pivot_{o,q})^2, then 3 counters
 *   (newton_unconverged, argmax_near_ties, points evaluated) stored as exact
 *   doubles.  partial_doubles_per_cell = 8 n_options + 3.
 * Pivots are the d = 1 Black-Scholes values of each output. */
int qmccpw_cell_count(const qmccpw_params* p, int32_t n_options, uint64_t n_points, uint32_t n_replicates,
                      const qmccpw_config* cfg, uint64_t* n_cells, uint64_t* partial_doubles_per_cell);

/* Enqueue the cells [cell_begin, cell_end) on cfg->stream, writing their
 * partials into d_partials + cell * partial_doubles_per_cell (device memory
 * of n_cells * partial_doubles_per_cell doubles, caller-owned).  Cells outside
 * the range are not touched, so a zero-initialised buffer summed across ranks
 * (one all-reduce) is exact. */
int qmccpw_partials(const int32_t* options, const qmccpw_params* p, int32_t n_options, uint64_t n_points,
                    uint32_t n_replicates, const qmccpw_config* cfg, uint64_t cell_begin, uint64_t cell_end,
                    double* d_partials);

/* Reduce the cells of replicates [rep_begin, rep_end) of d_partials (fixed,
 * sequential cell order) into rows rep of d_rep_sums (device, caller-owned,
 * n_replicates * partial_doubles_per_cell doubles); other rows untouched.
 * Enqueue only (cfg->stream).  Ranks owning disjoint replicate ranges can
 * all-reduce zero-initialised d_rep_sums exactly; a replicate whose cells are
 * split between ranks (each rank's other cells zero in its d_partials) sums to
 * the two partial sums (deterministic, equal to rounding). */
int qmccpw_replicate_sums(const double* d_partials, const qmccpw_params* p, int32_t n_options, uint64_t n_points,
                          uint32_t n_replicates, const qmccpw_config* cfg, uint32_t rep_begin, uint32_t rep_end,
                          double* d_rep_sums);

/* Host-only finalisation (no device work): replicate sums h_rep_sums
 * [n_replicates][partial_doubles_per_cell] (host memory) -> out[n_options]
 * (P:643-652).  EINVAL if any replicate's point counter differs from
 * n_points (a rank's or a cell range's contribution is missing). */
int qmccpw_finalize(const double* h_rep_sums, const int32_t* options, const qmccpw_params* p, int32_t n_options,
                    uint64_t n_points, uint32_t n_replicates, const qmccpw_config* cfg, qmccpw_result* out);

/* Reduce device partials of ALL cells (fixed cell order) and finalise into
 * out[n_options].  d_partials is device memory as filled above. */
int qmccpw_finalize_device(const double* d_partials, const int32_t* options, const qmccpw_params* p,
                           int32_t n_options, uint64_t n_points, uint32_t n_replicates, const qmccpw_config* cfg,
                           qmccpw_result* out);

/* ---- parity hooks (small ranges; results in host memory) -------------- */
/* Sobol' integers y(replicate, j, k) for j in [dim_begin, dim_end), k in
 * [k_begin, k_end) (absolute indices, k_end <= 2^32), out[(j-dim_begin)*(k_end-k_begin) + (k-k_begin)].
 * Gray-code order, point 0 included. */
int qmccpw_sobol_u32(uint32_t replicate, uint32_t dim_begin, uint32_t dim_end, uint64_t k_begin, uint64_t k_end,
                     const qmccpw_config* cfg, uint32_t* out);
/* Standard normals x[(k-k_begin)*d + j] = Phi^{-1}((y+1/2) 2^-32) of the QMC
 * path (or of the Philox LR path when cfg->method == QMCCPW_LR_MC). */
int qmccpw_normals(uint32_t replicate, int32_t d, uint64_t k_begin, uint64_t k_end, const qmccpw_config* cfg,
                   double* out);
/* Per-path estimator values out[(k-k_begin)*4 + q] computed by the production
 * kernel's device code for points k in [k_begin, k_end) of one replicate. */
int qmccpw_path_values(int32_t option, const qmccpw_params* p, uint32_t replicate, uint64_t k_begin,
                       uint64_t k_end, const qmccpw_config* cfg, double* out);

/* ---- measurement -------------------------------------------------------- */
/* FP64 roof microbenchmarks on `device`: DFMA TFLOP/s at
 * full occupancy (independent chains), dependent-DFMA latency in SM cycles,
 * FP64 tensor-core (mma.sync m8n8k4, SASS DMMA) TFLOP/s, and the SM clock in
 * MHz measured during the DFMA run (clock64 cycles / %globaltimer ns of one block's span), so
 * that dfma_tflops / (2 x 148 x 64 x clock) is the per-clock fraction of the
 * FP64 pipe's peak.  Outputs are host pointers. */
int qmccpw_fp64_roof(int32_t device, double* dfma_tflops, double* dfma_latency_cycles, double* dmma_tflops,
                     double* sm_clock_mhz);

/* Per-path values of a portfolio call (the C5 portfolio kernel):
 * out[((k-k_begin)*n_options + o)*4 + q]. */
int qmccpw_portfolio_path_values(const int32_t* options, const qmccpw_params* p, int32_t n_options,
                                 uint32_t replicate, uint64_t k_begin, uint64_t k_end, const qmccpw_config* cfg,
                                 double* out);

/* ---- housekeeping ----------------------------------------------------- */
const char* qmccpw_last_error(void); /* thread-local; valid until the next call on this thread */
void qmccpw_release(int32_t device);  /* frees cached device tables/scratch (-1: all devices) */
/* number of the library's kernel launches issued by this thread since the
 * last reset (bench.py's gpu_launches evidence) */
uint64_t qmccpw_launch_count(int32_t reset);

#ifdef __cplusplus
}
#endif
#endif
