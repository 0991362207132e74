/*
 * qmccpw_oracle.c -- plain CPU oracle for the QMC-CPW hot path (arXiv 2209.11337).
 *
 * TEST INFRASTRUCTURE ONLY: see qmccpw_oracle.h.  No blocking, no fusion, no
 * reordering beyond what the paper's definitions and algorithms state.  FP64
 * throughout, -O2, no -ffast-math.  Independent of the CUDA path: it shares
 * no code, header, table or constant generator with paper_2209_11337_b200/.
 *
 * Steps, each citing PAPER.md as P:<line>:
 *   O1 direction numbers      P:153-175 (recurrence P:166, identity dim P:147)
 *   O2 randomisation          P:179-181, P:440  (LMS + digital shift, Philox)
 *   O3 Sobol' integers        P:125-151 (XOR form P:147-151), Gray-code order
 *   O4 uniform -> normal      AS241 (Wichura 1988) + one Newton step
 *   O5 path construction      STD Alg. 3; BB Alg. 4;
 *                             PCA of the Brownian covariance
 *   O6 separated path         P:338-373 (S~(t_j), W~)
 *   O7 threshold              W1: psi_d of P:393 ; X1: bisection on the
 *                             monotone average map (north star)
 *   O8 estimators             P:396-414, P:538-602 (readings in DESIGN.md)
 *   O9 LR+MC baseline
 *   O10 statistics
 *
 * Parity pins for every function are in tests/test_oracle_*.py.
 */
#include "qmccpw_oracle.h"

#include <float.h>
#include <math.h>
#include <pthread.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#define OR_MAX_DIM 1024

static __thread char g_err[256];
static int set_err(int code, const char* msg) {
    snprintf(g_err, sizeof g_err, "%s", msg);
    return code;
}
const char* or_last_error(void) { return g_err; }

/* ------------------------------------------------------------------------ */
/* O1  Direction numbers                                         */
/* ------------------------------------------------------------------------ */
static int g_ndims = 0;                 /* dimensions available incl. dim 0 */
static int g_s[OR_MAX_DIM], g_a[OR_MAX_DIM];
static uint32_t g_minit[OR_MAX_DIM][32];

int or_load_joe_kuo(const char* path) {
    FILE* f = fopen(path, "r");
    if (!f) return set_err(-1, "cannot open Joe-Kuo file");
    char line[1024];
    int n = 1; /* dimension 0 (Joe-Kuo d = 1) is the identity */
    g_s[0] = 0;
    g_a[0] = 0;
    if (!fgets(line, sizeof line, f)) { fclose(f); return set_err(-1, "empty Joe-Kuo file"); }
    while (n < OR_MAX_DIM && fgets(line, sizeof line, f)) {
        char* p = line;
        int dim, s, a, used;
        if (sscanf(p, "%d %d %d%n", &dim, &s, &a, &used) != 3) break;
        p += used;
        if (dim != n + 1 || s < 1 || s > 31) { fclose(f); return set_err(-1, "bad Joe-Kuo row"); }
        g_s[n] = s;
        g_a[n] = a;
        for (int i = 0; i < s; i++) {
            unsigned m;
            if (sscanf(p, "%u%n", &m, &used) != 1) { fclose(f); return set_err(-1, "short Joe-Kuo row"); }
            p += used;
            g_minit[n][i] = m;
        }
        n++;
    }
    fclose(f);
    g_ndims = n;
    return n;
}

int or_polynomial(int32_t j, int32_t* s, int32_t* a) {
    if (j < 1 || j >= g_ndims) return set_err(-1, "dimension out of range");
    *s = g_s[j];
    *a = g_a[j];
    return 0;
}

/* m_k for k = 1..32 of 0-based dimension j by the recurrence of P:166:
 *   m_k = 2c_1 m_{k-1} ^ 2^2 c_2 m_{k-2} ^ ... ^ 2^{s-1} c_{s-1} m_{k-s+1} ^ 2^s m_{k-s} ^ m_{k-s}
 * with c_i = bit (s-1-i) of a; then g_k = m_k / 2^k, i.e. v_b = m_{b+1} << (31-b). */
int or_expand_recurrence(int32_t s, int32_t a, const uint32_t* m_init, int32_t count, uint64_t* m_out) {
    uint64_t m[65]; /* 1-based */
    if (s < 1 || s > 31 || count < 1 || count > 64) return set_err(-1, "bad recurrence arguments");
    for (int k = 1; k <= s && k <= count; k++) m[k] = m_init[k - 1];
    for (int k = s + 1; k <= count; k++) {
        uint64_t mk = (m[k - s] << s) ^ m[k - s];
        for (int i = 1; i <= s - 1; i++) {
            int c_i = (a >> (s - 1 - i)) & 1;
            if (c_i) mk ^= m[k - i] << i;
        }
        m[k] = mk;
    }
    for (int k = 1; k <= count; k++) m_out[k - 1] = m[k];
    return 0;
}

static void direction_numbers_dim(int j, uint32_t v[32]) {
    uint64_t m[33]; /* 1-based */
    if (j == 0) {   /* identity generator matrix: van der Corput */
        for (int b = 0; b < 32; b++) v[b] = 1u << (31 - b);
        return;
    }
    or_expand_recurrence(g_s[j], g_a[j], g_minit[j], 32, m + 1);
    for (int b = 0; b < 32; b++) v[b] = (uint32_t)(m[b + 1] << (31 - b));
}

int or_direction_numbers(int32_t d, uint32_t* v) {
    if (d < 1 || d > g_ndims) return set_err(-1, "d out of range of the loaded table");
    for (int j = 0; j < d; j++) direction_numbers_dim(j, v + 32 * j);
    return 0;
}

/* ------------------------------------------------------------------------ */
/* O2  Randomisation: Philox4x32-10 -> per-replicate LMS + digital shift     */
/* ------------------------------------------------------------------------ */
void or_philox4x32_10(const uint32_t ctr[4], const uint32_t key[2], uint32_t out[4]) {
    uint32_t c0 = ctr[0], c1 = ctr[1], c2 = ctr[2], c3 = ctr[3];
    uint32_t k0 = key[0], k1 = key[1];
    for (int round = 0; round < 10; round++) {
        if (round > 0) {
            k0 += 0x9E3779B9u; /* Weyl key schedule */
            k1 += 0xBB67AE85u;
        }
        uint64_t p0 = (uint64_t)0xD2511F53u * c0;
        uint64_t p1 = (uint64_t)0xCD9E8D57u * c2;
        uint32_t hi0 = (uint32_t)(p0 >> 32), lo0 = (uint32_t)p0;
        uint32_t hi1 = (uint32_t)(p1 >> 32), lo1 = (uint32_t)p1;
        uint32_t n0 = hi1 ^ c1 ^ k0;
        uint32_t n1 = lo1;
        uint32_t n2 = hi0 ^ c3 ^ k1;
        uint32_t n3 = lo0;
        c0 = n0; c1 = n1; c2 = n2; c3 = n3;
    }
    out[0] = c0; out[1] = c1; out[2] = c2; out[3] = c3;
}

static int parity32(uint32_t x) {
    int p = 0;
    while (x) { p ^= 1; x &= x - 1; }
    return p;
}

/* O2b  Nested uniform scrambling (Owen 1995; P:179-181 names it).
 * Reading 27: the random permutations of Owen's tree are drawn by a hash, the
 * Laine-Karras construction with Burley's constants (JCGT 9(4), 2020): on the
 * bit-reversed coordinate r (r's bit i = y's digit i, MSB first),
 *     r <- r + seed;  r <- r XOR (r * C_m) for the four constants C_m;
 * then reversed back.  Addition carries and products with even constants only
 * move information from lower to higher bits of r, so digit i of the output is
 * digit i of y XOR a function of (seed, digits 0..i-1): a nested scramble.
 * Written out digit by digit, without machine multiplication, so that it reads
 * against that definition (the pins in tests/test_oracle_owen.py check the
 * nesting, bijectivity and net properties it must have). */
static uint32_t reverse32(uint32_t y) {
    uint32_t r = 0;
    for (int i = 0; i < 32; i++) r |= ((y >> i) & 1u) << (31 - i);
    return r;
}
static uint32_t mul_mod32(uint32_t a, uint32_t c) { /* a * c mod 2^32 as a sum of shifted copies */
    uint32_t s = 0;
    for (int b = 0; b < 32; b++)
        if ((c >> b) & 1u) s += a << b;
    return s;
}
uint32_t or_owen_scramble(uint32_t y, uint32_t seed) {
    static const uint32_t C[4] = {0x6c50b47cu, 0xb82f1e52u, 0xc7afe638u, 0x8d22f6e6u};
    uint32_t r = reverse32(y);
    r += seed;
    for (int m = 0; m < 4; m++) r ^= mul_mod32(r, C[m]);
    return reverse32(r);
}

/* Randomisation of dimension j in replicate rep (reading 10):
 * 32 Philox words from counters (j, w, 0, (rep<<8)|0x01), w = 0..7, key = seed.
 * word 0 -> digital shift; word i -> row i of a lower-triangular (MSB-first)
 * unit-diagonal matrix L over GF(2) (Matousek's left matrix scramble).
 * Scrambled direction number v'_b = L v_b, output digit i = parity(row_i & v). */
int or_randomization(uint64_t seed, uint32_t rep, int32_t d, int32_t randomization, uint32_t* vscr,
                     uint32_t* shift) {
    if (d < 1 || d > g_ndims) return set_err(-1, "d out of range");
    if (rep >= (1u << 24)) return set_err(-1, "replicate index >= 2^24");
    const uint32_t key[2] = {(uint32_t)seed, (uint32_t)(seed >> 32)};
    for (int j = 0; j < d; j++) {
        uint32_t v[32], w[32], rows[32];
        direction_numbers_dim(j, v);
        for (uint32_t blk = 0; blk < 8; blk++) {
            uint32_t ctr[4] = {(uint32_t)j, blk, 0u, (rep << 8) | 0x01u};
            or_philox4x32_10(ctr, key, w + 4 * blk);
        }
        for (int i = 0; i < 32; i++) {
            if (randomization == OR_RAND_LMS_SHIFT && i > 0)
                rows[i] = (1u << (31 - i)) | (w[i] & (~0u << (32 - i)));
            else
                rows[i] = 1u << (31 - i); /* identity row */
        }
        for (int b = 0; b < 32; b++) {
            uint32_t out = 0;
            for (int i = 0; i < 32; i++) out |= (uint32_t)parity32(rows[i] & v[b]) << (31 - i);
            vscr[32 * j + b] = out;
        }
        /* OWEN: plain direction numbers; word 0 is the dimension's scramble seed */
        shift[j] = (randomization == OR_RAND_NONE) ? 0u : w[0];
    }
    return 0;
}

/* coordinate j of point k under the config's randomisation: for OWEN the shift
 * slot c holds the scramble seed and the plain Sobol' integer is scrambled */
static uint32_t sobol_direct(const uint32_t* v32, uint32_t shift, uint64_t k);
static uint32_t sobol_point(const uint32_t* v32, uint32_t c, uint64_t k, int32_t randomization) {
    if (randomization == OR_RAND_OWEN) return or_owen_scramble(sobol_direct(v32, 0u, k), c);
    return sobol_direct(v32, c, k);
}

/* ------------------------------------------------------------------------ */
/* O3  Sobol' integers, direct formula in Gray-code order */
/* ------------------------------------------------------------------------ */
static uint32_t sobol_direct(const uint32_t* v32, uint32_t shift, uint64_t k) {
    uint32_t g = (uint32_t)(k ^ (k >> 1)); /* Gray code of the point index */
    uint32_t y = shift;
    for (int b = 0; b < 32; b++)
        if ((g >> b) & 1u) y ^= v32[b];
    return y;
}

int or_sobol_from_vectors(const uint32_t* v, const uint32_t* shift, uint32_t dim_begin, uint32_t dim_end,
                          uint64_t k_begin, uint64_t k_end, uint32_t* out) {
    if (dim_end < dim_begin || k_end < k_begin || k_end > (1ull << 32)) return set_err(-1, "bad range");
    uint64_t nk = k_end - k_begin;
    for (uint32_t j = dim_begin; j < dim_end; j++)
        for (uint64_t k = k_begin; k < k_end; k++)
            out[(uint64_t)(j - dim_begin) * nk + (k - k_begin)] = sobol_direct(v + 32 * j, shift[j], k);
    return 0;
}

int or_sobol_u32(uint32_t rep, uint32_t dim_begin, uint32_t dim_end, uint64_t k_begin, uint64_t k_end,
                 const or_config* cfg, uint32_t* out) {
    if (dim_end > (uint32_t)g_ndims || dim_end < dim_begin) return set_err(-1, "bad dimension range");
    uint32_t* v = malloc(sizeof(uint32_t) * 32 * (dim_end ? dim_end : 1));
    uint32_t* c = malloc(sizeof(uint32_t) * (dim_end ? dim_end : 1));
    int rc = 0;
    if (dim_end > 0) rc = or_randomization(cfg->seed, rep, (int32_t)dim_end, cfg->randomization, v, c);
    if (rc == 0) {
        uint64_t nk = k_end - k_begin;
        for (uint32_t j = dim_begin; j < dim_end; j++)
            for (uint64_t k = k_begin; k < k_end; k++)
                out[(uint64_t)(j - dim_begin) * nk + (k - k_begin)] = sobol_point(v + 32 * j, c[j], k, cfg->randomization);
    }
    free(v);
    free(c);
    return rc;
}

/* ------------------------------------------------------------------------ */
/* O4  Inverse normal CDF                                                    */
/* ------------------------------------------------------------------------ */
static double Phi(double x) { return 0.5 * erfc(-x * M_SQRT1_2); }     /* normal CDF */
static double Phibar(double x) { return 0.5 * erfc(x * M_SQRT1_2); }   /* 1 - Phi(x) */
static double phi(double x) { return exp(-0.5 * x * x) / sqrt(2.0 * M_PI); }

/* Wichura, AS241 PPND16 (Applied Statistics 37, 1988), then one Newton step
 * x <- x - (Phi(x) - p)/phi(x).  The upper half is mirrored (1 - p is exact
 * there) and, in AS241's central region, the residual Phi(x) - p is formed as
 * erf(x/sqrt2)/2 - (p - 1/2) so that the Newton step keeps relative accuracy
 * near p = 1/2 (Phi(x) - p via erfc would cancel there). */
double or_inv_normal_cdf(double p) {
    if (!(p > 0.0 && p < 1.0)) return NAN;
    if (p > 0.5) return -or_inv_normal_cdf(1.0 - p);
    double q = p - 0.5, r, val, res;
    if (fabs(q) <= 0.425) {
        r = 0.180625 - q * q;
        val = q * (((((((r * 2509.0809287301226727 + 33430.575583588128105) * r + 67265.770927008700853) * r +
                        45921.953931549871457) * r + 13731.693765509461125) * r + 1971.5909503065514427) * r +
                     133.14166789178437745) * r + 3.387132872796366608) /
              (((((((r * 5226.495278852545925 + 28729.085735721942674) * r + 39307.89580009271061) * r +
                   21213.794301586595867) * r + 5394.1960214247511077) * r + 687.1870074920579083) * r +
                42.313330701600911252) * r + 1.0);
        res = 0.5 * erf(val * M_SQRT1_2) - q;
    } else {
        r = sqrt(-log(p)); /* p < 1/2 here */
        if (r <= 5.0) {
            r -= 1.6;
            val = (((((((r * 7.7454501427834140764e-4 + 0.0227238449892691845833) * r + 0.24178072517745061177) * r +
                       1.27045825245236838258) * r + 3.64784832476320460504) * r + 5.7694972214606914055) * r +
                    4.6303378461565452959) * r + 1.42343711074968357734) /
                  (((((((r * 1.05075007164441684324e-9 + 5.475938084995344946e-4) * r + 0.0151986665636164571966) * r +
                       0.14810397642748007459) * r + 0.68976733498510000455) * r + 1.6763848301838038494) * r +
                    2.05319162663775882187) * r + 1.0);
        } else {
            r -= 5.0;
            val = (((((((r * 2.01033439929228813265e-7 + 2.71155556874348757815e-5) * r + 0.0012426609473880784386) * r +
                       0.026532189526576123093) * r + 0.29656057182850489123) * r + 1.7848265399172913358) * r +
                    5.4637849111641143699) * r + 6.6579046435011037772) /
                  (((((((r * 2.04426310338993978564e-15 + 1.4215117583164458887e-7) * r + 1.8463183175100546818e-5) * r +
                       7.868691311456132591e-4) * r + 0.0148753612908506148525) * r + 0.13692988092273580531) * r +
                    0.59983220655588793769) * r + 1.0);
        }
        val = -val; /* q < 0 */
        res = Phi(val) - p;
    }
    return val - res / phi(val);
}

/* u = (y + 1/2) 2^-32 (cuRAND's lattice convention); evaluated on the lower
 * half and mirrored so that x(2^32-1-y) = -x(y) exactly. */
double or_normal_from_u32(uint32_t y) {
    if (y >= 0x80000000u) return -or_inv_normal_cdf(((double)(0xFFFFFFFFu - y) + 0.5) * 0x1p-32);
    return or_inv_normal_cdf(((double)y + 0.5) * 0x1p-32);
}

int or_normals(uint32_t rep, int32_t d, uint64_t k_begin, uint64_t k_end, const or_config* cfg, double* out) {
    if (d < 1 || d > g_ndims) return set_err(-1, "d out of range");
    uint32_t* v = malloc(sizeof(uint32_t) * 32 * d);
    uint32_t* c = malloc(sizeof(uint32_t) * d);
    int rc = or_randomization(cfg->seed, rep, d, cfg->randomization, v, c);
    if (rc == 0)
        for (uint64_t k = k_begin; k < k_end; k++)
            for (int j = 0; j < d; j++)
                out[(k - k_begin) * d + j] = or_normal_from_u32(sobol_point(v + 32 * j, c[j], k, cfg->randomization));
    free(v);
    free(c);
    return rc;
}

/* LR+MC normals: Philox counter (k_lo, k_hi, j/4, (rep<<8)|0x02), word j%4 */
static double lr_normal(uint64_t seed, uint32_t rep, uint64_t k, int j) {
    const uint32_t key[2] = {(uint32_t)seed, (uint32_t)(seed >> 32)};
    uint32_t ctr[4] = {(uint32_t)k, (uint32_t)(k >> 32), (uint32_t)(j / 4), (rep << 8) | 0x02u}, w[4];
    or_philox4x32_10(ctr, key, w);
    return or_normal_from_u32(w[j % 4]);
}

int or_lr_normals(uint32_t rep, int32_t d, uint64_t k_begin, uint64_t k_end, uint64_t seed, double* out) {
    for (uint64_t k = k_begin; k < k_end; k++)
        for (int j = 0; j < d; j++) out[(k - k_begin) * d + j] = lr_normal(seed, rep, k, j);
    return 0;
}

/* ------------------------------------------------------------------------ */
/* O5  Path construction W = construct(x), W_j = W(t_j), t_j = j T / d        */
/* ------------------------------------------------------------------------ */
static int is_pow2(int d) { return d > 0 && (d & (d - 1)) == 0; }

/* Alg. 3 (reading 6): W(t_1) = sqrt(dt) x_1, W(t_j) = W(t_{j-1}) + sqrt(dt) x_j */
static void construct_std(int d, double T, const double* x, double* W) {
    double sdt = sqrt(T / d), acc = 0.0;
    for (int j = 0; j < d; j++) {
        acc += sdt * x[j];
        W[j] = acc;
    }
}

/* Alg. 4 literally, with the terminal scaled by sqrt(T) and
 * b_k = sqrt(T / 2^{k+1}) (reading 9); increments, then their prefix sum. */
static void construct_bb(int d, double T, const double* x, double* W) {
    double* path = malloc(sizeof(double) * d);
    int idx = 0;
    path[0] = sqrt(T) * x[idx]; /* terminal value first */
    for (int k = 1; (1 << k) <= d; k++) {
        int i = (1 << k) - 1;
        double b = sqrt(T / (double)(1ull << (k + 1)));
        for (int j = (1 << (k - 1)) - 1; j >= 0; j--) {
            idx++;
            double z = x[idx];
            double a = 0.5 * path[j];
            path[i] = a - b * z;
            i--;
            path[i] = a + b * z;
            i--;
        }
    }
    double acc = 0.0;
    for (int j = 0; j < d; j++) {
        acc += path[j];
        W[j] = acc;
    }
    free(path);
}

/* PCA of C_ij = min(t_i, t_j) in closed form:
 * theta_k = (2k-1) pi / (2d+1), lambda_k = dt / (4 sin^2(theta_k/2)),
 * v_k(j) = sqrt(4/(2d+1)) sin(j theta_k), M_jk = sqrt(lambda_k) v_k(j), j,k = 1..d. */
static void pca_matrix(int d, double T, double* M) {
    double dt = T / d;
    for (int k = 1; k <= d; k++) {
        double theta = (2.0 * k - 1.0) * M_PI / (2.0 * d + 1.0);
        double sh = sin(0.5 * theta);
        double lambda = dt / (4.0 * sh * sh);
        for (int j = 1; j <= d; j++) M[(j - 1) * d + (k - 1)] = sqrt(lambda) * sqrt(4.0 / (2.0 * d + 1.0)) * sin(j * theta);
    }
}

int or_construct(int32_t construction, int32_t d, double T, const double* x, double* W) {
    if (d < 1) return set_err(-1, "d < 1");
    if (construction == OR_STD) {
        construct_std(d, T, x, W);
    } else if (construction == OR_BB) {
        if (!is_pow2(d)) return set_err(-2, "Brownian bridge needs d = 2^m (Alg. 4)");
        construct_bb(d, T, x, W);
    } else if (construction == OR_PCA) {
        double* M = malloc(sizeof(double) * d * d);
        pca_matrix(d, T, M);
        for (int j = 0; j < d; j++) {
            double s = 0.0;
            for (int k = 0; k < d; k++) s += M[j * d + k] * x[k];
            W[j] = s;
        }
        free(M);
    } else if (construction == OR_GPCA) {
        return set_err(-1, "GPCA depends on the market: use or_path_matrix_gpca");
    } else {
        return set_err(-1, "unknown construction");
    }
    return 0;
}

/* O5b GPCA (P:883, P:904-906 name it, reading 28).  The
 * gradient of the arithmetic average A = (1/d) sum_j S0 exp(omega t_j + sigma W_j)
 * at W = 0 is proportional to s_j = exp(omega t_j).  With the PCA matrix M (M M^T
 * = C), q = M^T s / |M^T s| and the Householder reflection H = I - 2 v v^T/(v^T v),
 * v = e_1 - q (H e_1 = q, H orthogonal), the GPCA matrix is M H: still M H (M H)^T
 * = C, and (M H)^T s = H q |M^T s| = e_1 |M^T s|, so the linear part of the average
 * depends on x_1 alone.  Its first column is C s / sqrt(s^T C s) > 0. */
static void gpca_matrix(int d, double T, double omega, double* M) {
    double* s = malloc(sizeof(double) * d);
    double* v = malloc(sizeof(double) * d);
    pca_matrix(d, T, M);
    for (int j = 0; j < d; j++) s[j] = exp(omega * (j + 1) * (T / d));
    double norm2 = 0.0;
    for (int k = 0; k < d; k++) {
        double qk = 0.0; /* (M^T s)_k */
        for (int j = 0; j < d; j++) qk += M[j * d + k] * s[j];
        v[k] = qk;
        norm2 += qk * qk;
    }
    double norm = sqrt(norm2), vv = 0.0;
    for (int k = 0; k < d; k++) {
        v[k] = (k == 0 ? 1.0 : 0.0) - v[k] / norm; /* v = e_1 - q */
        vv += v[k] * v[k];
    }
    if (vv > 0.0) {
        for (int j = 0; j < d; j++) {
            double u = 0.0; /* (M v)_j */
            for (int k = 0; k < d; k++) u += M[j * d + k] * v[k];
            for (int k = 0; k < d; k++) M[j * d + k] -= 2.0 * u * v[k] / vv;
        }
    }
    free(s);
    free(v);
}

int or_path_matrix_gpca(const or_market* mk, double* M) {
    if (mk->d < 1 || mk->d > OR_MAX_DIM) return set_err(-1, "d out of range");
    gpca_matrix(mk->d, mk->T, mk->r - 0.5 * mk->sigma * mk->sigma, M);
    return 0;
}

/* the path matrix a config needs for a market */
static int path_matrix_mk(int32_t construction, const or_market* mk, double* M);

/* M[:,k] = construct(e_k): the path matrix of any of the three constructions */
int or_path_matrix(int32_t construction, int32_t d, double T, double* M) {
    if (construction == OR_PCA) {
        pca_matrix(d, T, M);
        return 0;
    }
    double* e = calloc(d, sizeof(double));
    double* col = malloc(sizeof(double) * d);
    int rc = 0;
    for (int k = 0; k < d && rc == 0; k++) {
        e[k] = 1.0;
        rc = or_construct(construction, d, T, e, col);
        for (int j = 0; j < d; j++) M[j * d + k] = col[j];
        e[k] = 0.0;
    }
    free(e);
    free(col);
    return rc;
}

static int path_matrix_mk(int32_t construction, const or_market* mk, double* M) {
    if (construction == OR_GPCA) return or_path_matrix_gpca(mk, M);
    return or_path_matrix(construction, mk->d, mk->T, M);
}

/* ------------------------------------------------------------------------ */
/* O6-O8  Conditional pathwise estimators                                    */
/* ------------------------------------------------------------------------ */
typedef struct {
    double S0, K, r, sigma, T, omega, t1, s, D, A;
    int d;
} mkt_t;

static void mkt_fill(mkt_t* m, const or_market* mk, double K) {
    m->S0 = mk->S0; m->K = K; m->r = mk->r; m->sigma = mk->sigma; m->T = mk->T; m->d = mk->d;
    m->omega = mk->r - 0.5 * mk->sigma * mk->sigma;    /* reading 1: omega = r - sigma^2/2 */
    m->t1 = mk->T / mk->d;                              /* t_1 = dt = T/d */
    m->s = mk->sigma * sqrt(m->t1);                     /* sigma sqrt(t_1) */
    m->D = exp(-mk->r * mk->T);                         /* e^{-rT} */
    m->A = exp(mk->r * (m->t1 - mk->T));                /* e^{r(t_1 - T)} */
}

/* "call-like" smoothed payoff with statistic stat and vega inner term I
 * (arithmetic P:560-576; lookback P:584-600 with the 1/d removed, reading 3) */
static void cpw_call(const mkt_t* m, double stat, double I, double* out) {
    double psi = (log(m->K) - log(stat) - m->omega * m->t1) / m->s; /* P:393 / P:586 */
    out[0] = m->A * stat * Phibar(psi - m->s) - m->D * m->K * Phibar(psi);
    out[1] = m->A * (stat / m->S0) * Phibar(psi - m->s);
    out[2] = m->A * Phibar(psi - m->s) * I + m->K * m->D * phi(psi) * sqrt(m->t1);
    out[3] = m->K * m->D / (m->S0 * m->S0 * m->s) * phi(psi);
}

/* binary Asian (P:401, P:412, P:544, P:550 read as dG/dsigma, reading 4) */
static void cpw_binary(const mkt_t* m, double stat, double I, double* out) {
    double psi = (log(m->K) - log(stat) - m->omega * m->t1) / m->s;
    out[0] = m->D * Phibar(psi);
    out[1] = m->D / (m->S0 * m->s) * phi(psi);
    out[2] = m->D * phi(psi) * (I / (m->s * stat) + psi / m->sigma - sqrt(m->t1));
    out[3] = m->D / (m->S0 * m->S0 * m->s) * phi(psi) * (psi / m->s - 1.0);
}

static double log_mean_tie_tol = 1e-12;

/* W1 mode (the paper's Sec. 3.4.1): condition on W(t_1) */
static int estimate_w1(int type, const mkt_t* m, const double* W, double* out, int* near_tie) {
    int d = m->d;
    double sumS = 0.0, sumI = 0.0, sumLog = 0.0, sumWt = 0.0;
    double Smax = -1.0, Imax = 0.0, emax = -INFINITY;
    for (int j = 1; j <= d; j++) {
        double tj = (double)j * m->T / d;
        double Wt = W[j - 1] - W[0];                              /* W~(t_j - t_1) */
        double e = m->omega * (tj - m->t1) + m->sigma * Wt;
        double St = m->S0 * exp(e);                               /* S~(t_j) */
        sumS += St;
        sumI += St * (Wt - m->sigma * (tj - m->t1));              /* vega inner sum */
        sumLog += log(m->S0) + e;
        sumWt += Wt - m->sigma * (tj - m->t1);
        if (St > Smax) {                                          /* lowest argmax (reading 20) */
            Smax = St;
            Imax = St * (Wt - m->sigma * (tj - m->t1));
            emax = e;
        }
    }
    if (near_tie) {
        int ties = 0;
        for (int j = 1; j <= d; j++) {
            double tj = (double)j * m->T / d;
            double e = m->omega * (tj - m->t1) + m->sigma * (W[j - 1] - W[0]);
            if (fabs(e - emax) < log_mean_tie_tol) ties++;
        }
        *near_tie = ties > 1;
    }
    double SA = sumS / d, IA = sumI / d;
    switch (type) {
    case OR_ARITH: cpw_call(m, SA, IA, out); break;
    case OR_BINARY: cpw_binary(m, SA, IA, out); break;
    case OR_LOOKBACK: cpw_call(m, Smax, Imax, out); break;
    case OR_GEOM_CALL:
    case OR_GEOM_DIGITAL: {
        double SG = exp(sumLog / d), IG = SG * (sumWt / d);
        if (type == OR_GEOM_CALL) cpw_call(m, SG, IG, out);
        else cpw_binary(m, SG, IG, out);
        break;
    }
    default: return set_err(-1, "unknown option type");
    }
    return 0;
}

/* X1 mode (north star): condition on x_1 of the full
 * path matrix.  S(t_j) = exp(c_j + sigma a_j x_1), c_j = ln S0 + omega t_j +
 * sigma R_j, a_j = M_j1, R_j = sum_{k>=2} M_jk x_k.  Threshold u* solves
 * sum_j exp(c_j + sigma a_j u) = d K by plain bisection (reading 19). */
static int estimate_x1(int type, const mkt_t* m, const double* M, const double* x, double* out) {
    int d = m->d;
    double *a = malloc(sizeof(double) * d), *R = malloc(sizeof(double) * d), *c = malloc(sizeof(double) * d);
    double lnK = log(m->K), lndK = log(d * m->K);
    double lo = INFINITY, hi = INFINITY;
    for (int j = 0; j < d; j++) {
        double tj = (double)(j + 1) * m->T / d;
        a[j] = M[j * d + 0];
        double Rj = 0.0;
        for (int k = 1; k < d; k++) Rj += M[j * d + k] * x[k];
        R[j] = Rj;
        c[j] = log(m->S0) + m->omega * tj + m->sigma * Rj;
        if (!(a[j] > 0.0)) { free(a); free(R); free(c); return set_err(-2, "X1 needs a_j > 0"); }
        double l = (lnK - c[j]) / (m->sigma * a[j]), h = (lndK - c[j]) / (m->sigma * a[j]);
        if (l < lo) lo = l;
        if (h < hi) hi = h;
    }
    /* h(lo) <= 0 <= h(hi); bisect until the bracket is ~1 ulp of max(1,|u|) */
    for (int it = 0; it < 2000; it++) {
        double mid = 0.5 * (lo + hi);
        if (!(mid > lo && mid < hi)) break;
        double scale = fmax(1.0, fmax(fabs(lo), fabs(hi)));
        if (hi - lo <= 0x1p-53 * scale) break;
        double sum = 0.0;
        for (int j = 0; j < d; j++) sum += exp(c[j] + m->sigma * a[j] * mid);
        if (sum - d * m->K > 0.0) hi = mid;
        else lo = mid;
    }
    double u = 0.5 * (lo + hi);
    double Dst = 0.0, Qst = 0.0, Vst = 0.0, sumW = 0.0, sumWv = 0.0;
    for (int j = 0; j < d; j++) {
        double tj = (double)(j + 1) * m->T / d;
        double Ej = exp(c[j] + m->sigma * a[j] * u);               /* E*_j */
        Dst += a[j] * Ej;
        Qst += a[j] * a[j] * Ej;
        Vst += Ej * (R[j] - m->sigma * tj + a[j] * u);
        double wj = exp(c[j] + 0.5 * m->sigma * m->sigma * a[j] * a[j]);
        double Pj = Phi(m->sigma * a[j] - u);
        sumW += wj * Pj;
        sumWv += wj * (R[j] - m->sigma * tj + m->sigma * a[j] * a[j]) * Pj;
    }
    double D = m->D, S0 = m->S0, K = m->K, sg = m->sigma;
    if (type == OR_ARITH) {
        out[0] = D * (sumW / d - K * Phibar(u));
        out[1] = D * sumW / (d * S0);
        out[2] = D * (sumWv / d + phi(u) * Dst / d);
        out[3] = D * d * K * K * phi(u) / (S0 * S0 * sg * Dst);
    } else if (type == OR_BINARY) {
        double up = -d * K / (S0 * sg * Dst); /* u' = du* / dS0 */
        out[0] = D * Phibar(u);
        out[1] = D * phi(u) * d * K / (S0 * sg * Dst);
        out[2] = D * phi(u) * Vst / (sg * Dst);
        out[3] = D * (d * K / sg) * phi(u) / (S0 * Dst) * (-u * up - 2.0 / S0 - sg * up * Qst / Dst);
    } else {
        free(a); free(R); free(c);
        return set_err(-2, "X1 conditioning: unsupported option type");
    }
    free(a); free(R); free(c);
    return 0;
}

/* Lookback under X1.  With lines
 * l_j(u) = c_j + b_j u, b_j = sigma a_j, max_j S(t_j) = exp(L(u)), L = max_j l_j:
 * {L > ln K} = {u > u*}, u* = min_j (ln K - c_j)/b_j.  Line j is the maximum on
 * [lo_j, hi_j]: lo_j = max over lines i of smaller slope of their crossing
 * x_ij = (c_i - c_j)/(b_j - b_i), hi_j = min over lines of larger slope; an
 * equal-slope line with a larger intercept (or the same one and a lower index)
 * hides j.  Then, on [max(lo_j, u*), hi_j]:
 *   G     = D [ sum_j w_j (Phibar(lo - b_j) - Phibar(hi - b_j)) - K Phibar(u*) ],
 *           w_j = exp(c_j + b_j^2/2)
 *   delta = (G + D K Phibar(u*)) / S0                      (all c_j shift by ln S0)
 *   gamma = D K phi(u*) / (S0^2 b_{j0}),  j0 the line that crosses ln K at u*
 *   vega  = D sum_j w_j [ (R_j - sigma t_j + sigma a_j^2)(Phibar(lo - b_j) - Phibar(hi - b_j))
 *                         + a_j (phi(lo - b_j) - phi(hi - b_j)) ]
 * (the envelope is continuous, so breakpoint motion contributes nothing). */
static int estimate_x1_lookback(const mkt_t* m, const double* M, const double* x, double* out) {
    int d = m->d;
    double *b = malloc(sizeof(double) * d), *c = malloc(sizeof(double) * d), *R = malloc(sizeof(double) * d);
    double lnK = log(m->K), u_star = INFINITY;
    int j0 = 0;
    for (int j = 0; j < d; j++) {
        double tj = (double)(j + 1) * m->T / d, Rj = 0.0;
        for (int k = 1; k < d; k++) Rj += M[j * d + k] * x[k];
        R[j] = Rj;
        c[j] = log(m->S0) + m->omega * tj + m->sigma * Rj;
        b[j] = m->sigma * M[j * d + 0];
        if (!(b[j] > 0.0)) { free(b); free(c); free(R); return set_err(-2, "X1 needs a_j > 0"); }
        double uj = (lnK - c[j]) / b[j];
        if (uj < u_star) { u_star = uj; j0 = j; }
    }
    double J = 0.0, V = 0.0;
    for (int j = 0; j < d; j++) {
        double lo = u_star, hi = INFINITY;
        int hidden = 0;
        for (int i = 0; i < d && !hidden; i++) {
            if (i == j) continue;
            if (b[i] < b[j]) lo = fmax(lo, (c[i] - c[j]) / (b[j] - b[i]));
            else if (b[i] > b[j]) hi = fmin(hi, (c[i] - c[j]) / (b[j] - b[i]));
            else if (c[i] > c[j] || (c[i] == c[j] && i < j)) hidden = 1;
        }
        if (hidden || !(lo < hi)) continue;
        double tj = (double)(j + 1) * m->T / d, aj = b[j] / m->sigma;
        double w = exp(c[j] + 0.5 * b[j] * b[j]);
        double dP = Phibar(lo - b[j]) - (isinf(hi) ? 0.0 : Phibar(hi - b[j]));
        double dphi = phi(lo - b[j]) - (isinf(hi) ? 0.0 : phi(hi - b[j]));
        J += w * dP;
        V += w * ((R[j] - m->sigma * tj + m->sigma * aj * aj) * dP + aj * dphi);
    }
    double D = m->D, K = m->K, S0 = m->S0;
    out[0] = D * (J - K * Phibar(u_star));
    out[1] = D * J / S0;
    out[2] = D * V;
    out[3] = D * K * phi(u_star) / (S0 * S0 * b[j0]);
    free(b); free(c); free(R);
    return 0;
}

/* O9  LR+MC: STD path of full prices, payoff x score */
static int estimate_lr(int type, const mkt_t* m, const double* x, double* out) {
    int d = m->d;
    double sdt = sqrt(m->t1), W = 0.0, sumS = 0.0, Smax = -1.0, vscore = 0.0;
    for (int j = 1; j <= d; j++) {
        double tj = (double)j * m->T / d;
        W += sdt * x[j - 1];
        double S = m->S0 * exp(m->omega * tj + m->sigma * W);
        sumS += S;
        if (S > Smax) Smax = S;
        vscore += (x[j - 1] * x[j - 1] - 1.0) / m->sigma - x[j - 1] * sqrt(m->t1);
    }
    double SA = sumS / d, f;
    switch (type) {
    case OR_ARITH: f = m->D * fmax(SA - m->K, 0.0); break;
    case OR_BINARY: f = (SA > m->K) ? m->D : 0.0; break;
    case OR_LOOKBACK: f = m->D * fmax(Smax - m->K, 0.0); break;
    default: return set_err(-1, "LR supports the three paper options only");
    }
    double Z1 = x[0], S0 = m->S0, sg = m->sigma, t1 = m->t1;
    out[0] = f;
    out[1] = f * Z1 / (S0 * sg * sqrt(t1));
    out[2] = f * vscore;
    out[3] = f * ((Z1 * Z1 - 1.0) / (S0 * S0 * sg * sg * t1) - Z1 / (S0 * S0 * sg * sqrt(t1)));
    return 0;
}

static int estimate_impl(const or_option* opt, const or_market* mk, int method, int construction, int conditioning,
                         const double* M, const double* x, double* out, int* near_tie) {
    mkt_t m;
    mkt_fill(&m, mk, opt->K);
    if (near_tie) *near_tie = 0;
    if (method == OR_LR_MC) return estimate_lr(opt->type, &m, x, out);
    if (method == OR_MC_AV_CPW) {
        /* the estimate from the path of x and from its antithetic path -x, combined */
        double* xm = malloc(sizeof(double) * mk->d);
        double o1[4], o2[4];
        int t1 = 0, t2 = 0;
        for (int j = 0; j < mk->d; j++) xm[j] = -x[j];
        int rc = estimate_impl(opt, mk, OR_QMC_CPW, construction, conditioning, M, x, o1, near_tie ? &t1 : NULL);
        if (rc == 0) rc = estimate_impl(opt, mk, OR_QMC_CPW, construction, conditioning, M, xm, o2, near_tie ? &t2 : NULL);
        for (int q = 0; q < 4; q++) out[q] = 0.5 * (o1[q] + o2[q]);
        if (near_tie) *near_tie = t1 + t2;
        free(xm);
        return rc;
    }
    if (conditioning == OR_COND_X1)
        return opt->type == OR_LOOKBACK ? estimate_x1_lookback(&m, M, x, out) : estimate_x1(opt->type, &m, M, x, out);
    double* W = malloc(sizeof(double) * mk->d);
    int rc = 0;
    if (construction == OR_GPCA || (construction == OR_PCA && M != NULL)) {
        /* W = M x with the call's path matrix (GPCA; PCA: the same pca_matrix that
         * or_construct would rebuild for every path, built once per call) */
        for (int j = 0; j < mk->d; j++) {
            double acc = 0.0;
            for (int k = 0; k < mk->d; k++) acc += M[j * mk->d + k] * x[k];
            W[j] = acc;
        }
    } else {
        rc = or_construct(construction, mk->d, mk->T, x, W);
    }
    if (rc == 0) rc = estimate_w1(opt->type, &m, W, out, opt->type == OR_LOOKBACK ? near_tie : NULL);
    free(W);
    return rc;
}

static int validate(const or_option* opt, const or_market* mk, int method, int construction, int conditioning) {
    if (!(mk->S0 > 0) || !(mk->sigma > 0) || !(mk->T > 0) || !isfinite(mk->r) || !isfinite(mk->S0) ||
        !isfinite(mk->sigma) || !isfinite(mk->T))
        return set_err(-1, "invalid market parameters");
    if (!(opt->K > 0) || !isfinite(opt->K)) return set_err(-1, "invalid strike");
    if (mk->d < 1 || mk->d > OR_MAX_DIM) return set_err(-1, "d out of range");
    if (construction == OR_BB && !is_pow2(mk->d)) return set_err(-2, "BB needs d = 2^m");
    if (method == OR_LR_MC && construction != OR_STD) return set_err(-2, "LR+MC uses the STD path");
    if (construction < OR_STD || construction > OR_GPCA) return set_err(-1, "unknown construction");
    if ((method == OR_MC_CPW || method == OR_MC_AV_CPW) && (construction >= OR_PCA || conditioning != OR_COND_W1))
        return set_err(-2, "MC-CPW / MC+AV-CPW: STD or BB construction, W1 conditioning");
    if (method < 0 || method > 3) return set_err(-1, "unknown method");
    if (method == OR_QMC_CPW && conditioning == OR_COND_X1 && opt->type != OR_ARITH && opt->type != OR_BINARY &&
        opt->type != OR_LOOKBACK)
        return set_err(-2, "X1 conditioning supports the three paper options only");
    return 0;
}

int or_estimate(const or_option* opt, const or_market* mk, int32_t method, int32_t construction,
                int32_t conditioning, const double* x, double* out) {
    int rc = validate(opt, mk, method, construction, conditioning);
    if (rc) return rc;
    double* M = NULL;
    if (method == OR_QMC_CPW && (conditioning == OR_COND_X1 || construction >= OR_PCA)) {
        M = malloc(sizeof(double) * mk->d * mk->d);
        path_matrix_mk(construction, mk, M);
    }
    rc = estimate_impl(opt, mk, method, construction, conditioning, M, x, out, NULL);
    free(M);
    return rc;
}

int or_path_values(const or_option* opt, const or_market* mk, const or_config* cfg, uint32_t rep,
                   uint64_t k_begin, uint64_t k_end, double* out) {
    int rc = validate(opt, mk, cfg->method, cfg->construction, cfg->conditioning);
    if (rc) return rc;
    if (mk->d > g_ndims) return set_err(-1, "d beyond the loaded direction table");
    int d = mk->d;
    double* x = malloc(sizeof(double) * d);
    double* M = NULL;
    if (cfg->method == OR_QMC_CPW && (cfg->conditioning == OR_COND_X1 || cfg->construction >= OR_PCA)) {
        M = malloc(sizeof(double) * d * d);
        path_matrix_mk(cfg->construction, mk, M);
    }
    for (uint64_t k = k_begin; k < k_end && rc == 0; k++) {
        if (cfg->method != OR_QMC_CPW) rc = or_lr_normals(rep, d, k, k + 1, cfg->seed, x);
        else rc = or_normals(rep, d, k, k + 1, cfg, x);
        if (rc == 0) rc = estimate_impl(opt, mk, cfg->method, cfg->construction, cfg->conditioning, M, x,
                                        out + 4 * (k - k_begin), NULL);
    }
    free(x);
    free(M);
    return rc;
}

/* ------------------------------------------------------------------------ */
/* O10  Statistics                                               */
/* ------------------------------------------------------------------------ */
/* Black-Scholes d = 1 values used as pivots (a call, or a cash-or-nothing digital) */
int or_pivots(const or_option* opt, const or_market* mk, double* p) {
    double S0 = mk->S0, K = opt->K, r = mk->r, sg = mk->sigma, T = mk->T, D = exp(-r * T);
    double sT = sg * sqrt(T);
    double d1 = (log(S0 / K) + (r + 0.5 * sg * sg) * T) / sT, d2 = d1 - sT;
    if (opt->type == OR_BINARY || opt->type == OR_GEOM_DIGITAL) {
        p[0] = D * Phi(d2);
        p[1] = D * phi(d2) / (S0 * sT);
        p[2] = -D * phi(d2) * d1 / sg;
        p[3] = -D * phi(d2) * d1 / (S0 * S0 * sg * sg * T);
    } else {
        p[0] = S0 * Phi(d1) - K * D * Phi(d2);
        p[1] = Phi(d1);
        p[2] = S0 * phi(d1) * sqrt(T);
        p[3] = phi(d1) / (S0 * sT);
    }
    return 0;
}

/* C = (1/L) sum_l C_l ; sigma = sqrt((1/L) sum_l (C - C_l)^2) (divisor L);
 * plus the standard error of C, sqrt(sum (C_l - C)^2 / (L (L-1))).  L < 2 -> NaN. */
int or_summarize(const double* C_l, int32_t L, double* mean, double* se, double* sigma_run) {
    if (L < 1) return set_err(-1, "L < 1");
    double sum = 0.0, dev2 = 0.0;
    for (int l = 0; l < L; l++) sum += C_l[l];
    double C = sum / L;
    for (int l = 0; l < L; l++) dev2 += (C - C_l[l]) * (C - C_l[l]);
    *mean = C;
    *sigma_run = L > 1 ? sqrt(dev2 / L) : NAN;
    *se = L > 1 ? sqrt(dev2 / ((double)L * (L - 1))) : NAN;
    return 0;
}

typedef struct { double s, c; } neum_t; /* Neumaier compensated sum */
static void neum_add(neum_t* a, double x) {
    double t = a->s + x;
    if (fabs(a->s) >= fabs(x)) a->c += (a->s - t) + x;
    else a->c += (x - t) + a->s;
    a->s = t;
}
static double neum_val(const neum_t* a) { return a->s + a->c; }

typedef struct {
    const or_option* opts;
    int n_opt;
    const or_market* mk;
    const or_config* cfg;
    uint64_t N;
    uint32_t L;
    const double* M;
    const double* piv;     /* [n_opt][4] */
    double* S1;            /* [L][n_opt][4] */
    double* S2;            /* [L][n_opt][4] */
    double* SA;            /* [L][n_opt][4] sum of |f| (the 8(c) tolerance scale) */
    uint64_t* ties;        /* [L] */
    int next;
    int rc;
    pthread_mutex_t mu;
} job_t;

static void* worker(void* arg) {
    job_t* jb = (job_t*)arg;
    int d = jb->mk->d, n_opt = jb->n_opt;
    double* x = malloc(sizeof(double) * d);
    uint32_t* v = malloc(sizeof(uint32_t) * 32 * d);
    uint32_t* c = malloc(sizeof(uint32_t) * d);
    neum_t* acc1 = malloc(sizeof(neum_t) * n_opt * 4);
    neum_t* acc2 = malloc(sizeof(neum_t) * n_opt * 4);
    neum_t* acca = malloc(sizeof(neum_t) * n_opt * 4);
    for (;;) {
        int rep = __atomic_fetch_add(&jb->next, 1, __ATOMIC_SEQ_CST);
        if (rep >= (int)jb->L) break;
        int rc = 0;
        if (jb->cfg->method == OR_QMC_CPW)
            rc = or_randomization(jb->cfg->seed, (uint32_t)rep, d, jb->cfg->randomization, v, c);
        memset(acc1, 0, sizeof(neum_t) * n_opt * 4);
        memset(acc2, 0, sizeof(neum_t) * n_opt * 4);
        memset(acca, 0, sizeof(neum_t) * n_opt * 4);
        uint64_t ties = 0;
        for (uint64_t i = 0; i < jb->N && rc == 0; i++) {
            uint64_t k = jb->cfg->point_offset + i;
            if (jb->cfg->method != OR_QMC_CPW) {
                for (int j = 0; j < d; j++) x[j] = lr_normal(jb->cfg->seed, (uint32_t)rep, k, j);
            } else {
                for (int j = 0; j < d; j++)
                    x[j] = or_normal_from_u32(sobol_point(v + 32 * j, c[j], k, jb->cfg->randomization));
            }
            for (int o = 0; o < n_opt && rc == 0; o++) {
                double f[4];
                int tie = 0;
                rc = estimate_impl(&jb->opts[o], jb->mk, jb->cfg->method, jb->cfg->construction,
                                   jb->cfg->conditioning, jb->M, x, f, &tie);
                ties += (uint64_t)tie;
                for (int q = 0; q < 4; q++) {
                    double y = f[q] - jb->piv[o * 4 + q];
                    neum_add(&acc1[o * 4 + q], y);
                    neum_add(&acc2[o * 4 + q], y * y);
                    neum_add(&acca[o * 4 + q], fabs(f[q]));
                }
            }
        }
        for (int i = 0; i < n_opt * 4; i++) {
            jb->S1[(size_t)rep * n_opt * 4 + i] = neum_val(&acc1[i]);
            jb->S2[(size_t)rep * n_opt * 4 + i] = neum_val(&acc2[i]);
            jb->SA[(size_t)rep * n_opt * 4 + i] = neum_val(&acca[i]);
        }
        jb->ties[rep] = ties;
        if (rc) {
            pthread_mutex_lock(&jb->mu);
            jb->rc = rc;
            pthread_mutex_unlock(&jb->mu);
        }
    }
    free(x); free(v); free(c); free(acc1); free(acc2); free(acca);
    return NULL;
}

int or_price_greeks(const or_option* opts, int32_t n_opt, const or_market* mk, uint64_t n_points,
                    uint32_t n_replicates, const or_config* cfg, int32_t n_threads, or_result* out,
                    double* rep_means) {
    if (!opts || !mk || !cfg || !out || n_opt < 1) return set_err(-1, "null argument");
    if (n_points == 0 || n_replicates == 0) return set_err(-1, "n_points and n_replicates must be > 0");
    if (cfg->point_offset + n_points > (1ull << 32)) return set_err(-1, "beyond the Sobol32 period");
    if (mk->d > g_ndims) return set_err(-1, "d beyond the loaded direction table");
    for (int o = 0; o < n_opt; o++) {
        int rc = validate(&opts[o], mk, cfg->method, cfg->construction, cfg->conditioning);
        if (rc) return rc;
    }
    int d = mk->d, L = (int)n_replicates;
    job_t jb;
    memset(&jb, 0, sizeof jb);
    jb.opts = opts; jb.n_opt = n_opt; jb.mk = mk; jb.cfg = cfg; jb.N = n_points; jb.L = n_replicates;
    double* M = NULL;
    if (cfg->method == OR_QMC_CPW && (cfg->conditioning == OR_COND_X1 || cfg->construction >= OR_PCA)) {
        M = malloc(sizeof(double) * d * d);
        path_matrix_mk(cfg->construction, mk, M);
    }
    jb.M = M;
    double* piv = malloc(sizeof(double) * n_opt * 4);
    for (int o = 0; o < n_opt; o++) or_pivots(&opts[o], mk, piv + 4 * o);
    jb.piv = piv;
    jb.S1 = malloc(sizeof(double) * L * n_opt * 4);
    jb.S2 = malloc(sizeof(double) * L * n_opt * 4);
    jb.SA = malloc(sizeof(double) * L * n_opt * 4);
    jb.ties = calloc(L, sizeof(uint64_t));
    pthread_mutex_init(&jb.mu, NULL);
    if (n_threads < 1) n_threads = 1;
    if (n_threads > L) n_threads = L;
    pthread_t* th = malloc(sizeof(pthread_t) * n_threads);
    for (int t = 0; t < n_threads; t++) pthread_create(&th[t], NULL, worker, &jb);
    for (int t = 0; t < n_threads; t++) pthread_join(th[t], NULL);
    int rc = jb.rc;
    if (rc == 0) {
        double N = (double)n_points;
        for (int o = 0; o < n_opt; o++) {
            or_result* res = &out[o];
            memset(res, 0, sizeof *res);
            res->n_points = n_points;
            res->n_replicates = n_replicates;
            for (int l = 0; l < L; l++) res->argmax_near_ties += jb.ties[l];
            for (int q = 0; q < 4; q++) {
                double p = piv[o * 4 + q], sumV = 0.0, sumA = 0.0;
                double* Cl = malloc(sizeof(double) * L);
                for (int l = 0; l < L; l++) {
                    double s1 = jb.S1[(size_t)l * n_opt * 4 + o * 4 + q], s2 = jb.S2[(size_t)l * n_opt * 4 + o * 4 + q];
                    Cl[l] = p + s1 / N;                            /* C_P^(l) */
                    if (rep_means) rep_means[(size_t)l * n_opt * 4 + o * 4 + q] = Cl[l];
                    sumV += s2 / N - (s1 / N) * (s1 / N);          /* within-replicate variance */
                    sumA += jb.SA[(size_t)l * n_opt * 4 + o * 4 + q] / N;
                }
                or_summarize(Cl, L, &res->mean[q], &res->se[q], &res->sigma_run[q]);
                free(Cl);
                res->within_var[q] = sumV / L;
                res->mean_abs[q] = sumA / L;
            }
        }
    }
    free(th); free(piv); free(jb.S1); free(jb.S2); free(jb.SA); free(jb.ties); free(M);
    pthread_mutex_destroy(&jb.mu);
    return rc;
}
