/*
 * qmccpw_oracle.h -- plain, slow, obviously-correct CPU oracle for QMC-CPW
 * (arXiv 2209.11337).
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load this library.  The
 * product path (paper_2209_11337_b200/, libqmccpw.so) never includes, links or
 * calls anything under oracle/, and this file shares no code, header, table or
 * constant generator with it.
 *
 * Every function follows PAPER.md (cited as P:<line>) step by step in FP64;
 * readings of silent or garbled passages are listed in DESIGN.md ("Readings")
 * and SURVEY.md Sec. 8(c).
 */
#ifndef QMCCPW_ORACLE_H
#define QMCCPW_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* option types; 100/101 are TEST-ONLY geometric products used by
 * the closed-form pin of SURVEY.md B3 */
enum { OR_ARITH = 0, OR_BINARY = 1, OR_LOOKBACK = 2, OR_GEOM_CALL = 100, OR_GEOM_DIGITAL = 101 };
/* OR_GPCA (row f3, reading 28): the PCA basis rotated by a Householder reflection so
 * that x_1 carries the whole gradient of the arithmetic average at the origin */
enum { OR_STD = 0, OR_BB = 1, OR_PCA = 2, OR_GPCA = 3 };
enum { OR_COND_W1 = 0, OR_COND_X1 = 1 };
/* methods compared in the paper: QMC-CPW (with the construction of the
 * config: STD = the paper's QMC-CPW, BB = QMC+BB-CPW), LR+MC, MC-CPW and
 * MC+AV-CPW (pseudo-random normals, antithetic pairs averaged) */
enum { OR_QMC_CPW = 0, OR_LR_MC = 1, OR_MC_CPW = 2, OR_MC_AV_CPW = 3 };
/* randomisation of the Sobol' points: per-replicate left-matrix scramble +
 * digital shift, shift only, none (plain Sobol'), or nested (Owen) scrambling
 * of every coordinate (reading 27) */
enum { OR_RAND_LMS_SHIFT = 0, OR_RAND_SHIFT = 1, OR_RAND_NONE = 3, OR_RAND_OWEN = 4 };

typedef struct {
    double S0, r, sigma, T;
    int32_t d;
} or_market;

typedef struct {
    int32_t type;
    double K;
} or_option;

typedef struct {
    int32_t method, construction, conditioning, randomization;
    uint64_t seed, point_offset;
} or_config;

typedef struct {
    double mean[4], se[4], sigma_run[4], within_var[4]; /* price, delta, vega, gamma */
    uint64_t n_points;
    uint32_t n_replicates;
    uint64_t argmax_near_ties;
    double mean_abs[4]; /* mean over all N L paths of |f|: the scale of SURVEY.md 8(c)'s means tolerance
                           1e-9 max(|C|, mean|f|); a statistic of the run, not an estimator output */
} or_result;

/* O1: load Joe-Kuo parameters (file format "d s a m_1..m_s"); returns #dims or <0 */
int or_load_joe_kuo(const char* path);
/* O1: expanded direction numbers v[j*32+b], j < d (dimension 0 = identity) */
int or_direction_numbers(int32_t d, uint32_t* v);
/* O1: the recurrence of P:166 for arbitrary (s, a, m_1..m_s): m_out[0..count) = m_1..m_count */
int or_expand_recurrence(int32_t s, int32_t a, const uint32_t* m_init, int32_t count, uint64_t* m_out);
/* primitive polynomial of 0-based dimension j >= 1: degree s and Joe-Kuo a */
int or_polynomial(int32_t j, int32_t* s, int32_t* a);

/* O2: Philox4x32-10 (Salmon et al. 2011) */
void or_philox4x32_10(const uint32_t ctr[4], const uint32_t key[2], uint32_t out[4]);
/* O2: randomised direction numbers v'[j*32+b] and shifts c[j] for replicate rep */
int or_randomization(uint64_t seed, uint32_t rep, int32_t d, int32_t randomization,
                     uint32_t* vscr, uint32_t* shift);

/* O2b: nested uniform (Owen) scramble of one 32-bit coordinate with a per-(replicate,
 * dimension) seed: digit i of the result (MSB first) is digit i of y flipped by a
 * function of the seed and digits 0..i-1 only (reading 27) */
uint32_t or_owen_scramble(uint32_t y, uint32_t seed);

/* O3: Sobol' integers y(rep, j, k) = c ^ XOR_{b in gray(k)} v'_b (direct formula),
 * out[(j-dim_begin)*(k_end-k_begin) + (k-k_begin)] */
int or_sobol_u32(uint32_t rep, uint32_t dim_begin, uint32_t dim_end, uint64_t k_begin, uint64_t k_end,
                 const or_config* cfg, uint32_t* out);
/* O3 with caller-supplied direction numbers and shifts (for the libcurand pin) */
int or_sobol_from_vectors(const uint32_t* v, const uint32_t* shift, uint32_t dim_begin, uint32_t dim_end,
                          uint64_t k_begin, uint64_t k_end, uint32_t* out);

/* O4: inverse normal CDF (AS241 + one Newton step) and the lattice map */
double or_inv_normal_cdf(double u);
double or_normal_from_u32(uint32_t y);
/* normals x[(k-k_begin)*d + j] of the QMC path (Sobol' dim j -> x_{j+1}) */
int or_normals(uint32_t rep, int32_t d, uint64_t k_begin, uint64_t k_end, const or_config* cfg, double* out);
/* normals of the LR+MC path (Philox, domain tag 0x02) */
int or_lr_normals(uint32_t rep, int32_t d, uint64_t k_begin, uint64_t k_end, uint64_t seed, double* out);

/* O5: path matrix M (row-major M[j*d+k]) of a construction, and W = construct(x) */
int or_path_matrix(int32_t construction, int32_t d, double T, double* M);
int or_construct(int32_t construction, int32_t d, double T, const double* x, double* W);
/* O5b: the GPCA path matrix of a market (it depends on omega = r - sigma^2/2 through the gradient) */
int or_path_matrix_gpca(const or_market* mk, double* M);

/* O6-O9: per-path estimator values for explicit normals x[d]; out[4] = G, delta, vega, gamma */
int or_estimate(const or_option* opt, const or_market* mk, int32_t method, int32_t construction,
                int32_t conditioning, const double* x, double* out);
/* per-path values over points k of replicate rep; out[(k-k_begin)*4 + q] */
int or_path_values(const or_option* opt, const or_market* mk, const or_config* cfg, uint32_t rep,
                   uint64_t k_begin, uint64_t k_end, double* out);
/* pivots p_{o,q}: the d = 1 Black-Scholes values of each output (Sec. 8(a8)) */
int or_pivots(const or_option* opt, const or_market* mk, double* p4);

/* O10: full run; out[n_opt]; rep_means optional [L][n_opt][4] replicate means C_l */
int or_price_greeks(const or_option* opts, int32_t n_opt, const or_market* mk, uint64_t n_points,
                    uint32_t n_replicates, const or_config* cfg, int32_t n_threads, or_result* out,
                    double* rep_means);

/* O10: replicate summary */
int or_summarize(const double* C_l, int32_t L, double* mean, double* se, double* sigma_run);

const char* or_last_error(void);

#ifdef __cplusplus
}
#endif
#endif
