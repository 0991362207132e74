// qmccpw_math.cuh -- FP64 device math for the QMC-CPW kernels (sm_100a).
//
// The hot path is FP64-pipe / issue-slot bound, so the
// special functions on it are written for a minimal instruction count:
// every polynomial coefficient and constant lives in __constant__ memory, so
// DFMA takes it as a constant-bank operand instead of two UMOVs per 64-bit
// literal (CUDA's normcdfinv/exp spent ~6.6k UMOVs per path, v0 profile).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

// polynomial degrees of the function kernels (see the selections below).  The generated
// header keeps only the selected fits in the constant bank (QMCCPW_COEFF_GUARDS; measured
// on one B200 against emitting every fit: C5 73.4 -> 68.0 ms, PCA-X1 111.8 -> 108.5, BB-W1
// 27.6 -> 27.5)
#ifndef QMCCPW_COEFF_GUARDS
#define QMCCPW_COEFF_GUARDS 1
#endif
#ifndef QMCCPW_ICDF_DEG
#define QMCCPW_ICDF_DEG 22
#endif
#ifndef QMCCPW_MILLS_DEG
#define QMCCPW_MILLS_DEG 23
#endif
#ifndef QMCCPW_LOGEXP_LO
#define QMCCPW_LOGEXP_LO 1
#endif
#include "qmccpw_coeffs.cuh"

namespace qmccpw {

struct MathConst {
    double log2e, shift, ln2_hi, ln2_lo, one, two, half, minus_half, w_split, inv_sqrt_2pi, inv_sqrt2, p32, p33,
        four, pdf_floor, mills_c, mills_2c, exp_floor, e64_inv_ln2, e64_ln2_hi, e64_ln2_lo;
};
__constant__ MathConst MC = {
    1.4426950408889634074,        // log2(e)
    6755399441055744.0,           // 1.5 * 2^52 (round-to-integer shifter)
    6.93147180369123816490e-01,   // ln2 high part (low 32 bits zero: n*ln2_hi exact)
    1.90821492927058770002e-10,   // ln2 low part
    1.0, 2.0, 0.5, -0.5,
    6.25,                         // central / tail split of the inverse normal (w = -ln(1 - z^2))
    0.398942280401432677939946059934,  // 1/sqrt(2 pi)
    0.707106781186547524400844362105,  // 1/sqrt(2)
    0x1p-32, 0x1p-33, 4.0, -700.0, 3.0, 6.0, 700.0,
    EXP64_INV_LN2, EXP64_LN2_HI, EXP64_LN2_LO};

// degrees of the exp and log1p kernels (fit_device_polys.py): exp(r), |r| <= ln2/128,
// degree 6 (3.4e-21) or 5 (2.2e-18 relative); (log1p(r) - r)/r^2, |r| <= 2^-7, degree 5
// or 4 (5.2e-13 relative, i.e. <= 1.6e-17 absolute in log1p(r))
// degree of the Mills-ratio polynomial: 27 (6.2e-17) or 23 (5.3e-17, the same rounding floor)
constexpr int kMillsDeg = QMCCPW_MILLS_DEG;
#if QMCCPW_MILLS_DEG == 27
#define MILLS_P MILLS_H
#elif QMCCPW_MILLS_DEG == 23
#define MILLS_P MILLS_H_D23
#else
#error "QMCCPW_MILLS_DEG must be 23 or 27"
#endif
#if QMCCPW_LOGEXP_LO
constexpr int kExpDeg = 5, kLogDeg = 4;
#define EXP_P EXP64_POLY_D5
#define LOG_P LOG1P_L_D4
#else
constexpr int kExpDeg = 6, kLogDeg = 5;
#define EXP_P EXP64_POLY
#define LOG_P LOG1P_L
#endif

// Philox4x32-10 (Salmon et al., SC'11): 10 rounds of two 32x32->64 products,
// Weyl key schedule.  c = counter in, output out (in place).
__device__ __forceinline__ void philox4x32_10(uint32_t c[4], uint32_t k0, uint32_t k1) {
#pragma unroll
    for (int r = 0; r < 10; ++r) {
        const uint32_t lo0 = 0xD2511F53u * c[0], hi0 = __umulhi(0xD2511F53u, c[0]);
        const uint32_t lo1 = 0xCD9E8D57u * c[2], hi1 = __umulhi(0xCD9E8D57u, c[2]);
        const uint32_t n0 = hi1 ^ c[1] ^ k0, n2 = hi0 ^ c[3] ^ k1;
        c[0] = n0;
        c[1] = lo1;
        c[2] = n2;
        c[3] = lo0;
        k0 += 0x9E3779B9u;
        k1 += 0xBB67AE85u;
    }
}

// The exp and log tables (1.5 KB) can be staged per block in shared memory by
// math_tables_load (every kernel that uses fast_exp / fast_log calls it before its first
// barrier): 32-bit shared addressing instead of 64-bit global address arithmetic.
// Per translation unit (QMCCPW_SMEM_TABLES, set before the include): measured faster for
// the W1 kernels (STD-W1 -3.8 %, BB-W1 -0.7 %), slower for PCA-X1 (+1.5 %) and the C5
// portfolio (+2.2 %), which read the tables through L1 instead.
#ifndef QMCCPW_SMEM_TABLES
#define QMCCPW_SMEM_TABLES 0
#endif
// QMCCPW_EXP256 (W1 units, with the shared tables): exp from a 256-entry 2^(j/256) table and a
// degree-4 polynomial on |r| <= ln2/512 -- the same 2.4e-18 fit error as the 64-entry table's
// degree 5, one DFMA fewer per exponential; 2 KB of shared memory instead of 0.5 KB
#ifndef QMCCPW_EXP256
#define QMCCPW_EXP256 0
#endif
#define QMCCPW_EXP256_ON (QMCCPW_EXP256 && QMCCPW_SMEM_TABLES)
// (units without the shared tables read the 256-entry table through L1: QMCCPW_EXP256_L1)
#define QMCCPW_EXP256_L1 (QMCCPW_EXP256 && !QMCCPW_SMEM_TABLES)
#if QMCCPW_SMEM_TABLES
__shared__ double2 s_log_tab[64];
#if QMCCPW_EXP256_ON
__shared__ double s_exp_tab[256];
#else
__shared__ double s_exp_tab[64];
#endif
#define QMCCPW_LOG_TAB(i) s_log_tab[i]
#define QMCCPW_EXP_TAB(i) s_exp_tab[i]
#else
#define QMCCPW_LOG_TAB(i) __ldg(reinterpret_cast<const double2*>(LOG_TAB) + (i))
#if QMCCPW_EXP256_L1
#define QMCCPW_EXP_TAB(i) __ldg(EXP_TAB256 + (i))
#else
#define QMCCPW_EXP_TAB(i) __ldg(EXP_TAB + (i))
#endif
#endif
#if QMCCPW_EXP256_ON || QMCCPW_EXP256_L1
constexpr int kExpBits = 8, kExpDegK = 4;
#define EXP_PK EXP256_POLY_D4
#define EXP_INV_LN2K (4.0 * EXP64_INV_LN2)   // 256/ln2 (exact power-of-two scalings of the
#define EXP_LN2_HIK (0.25 * EXP64_LN2_HI)    // 64-entry table's constants)
#define EXP_LN2_LOK (0.25 * EXP64_LN2_LO)
#else
constexpr int kExpBits = 6, kExpDegK = kExpDeg;
#define EXP_PK EXP_P
#define EXP_INV_LN2K MC.e64_inv_ln2
#define EXP_LN2_HIK MC.e64_ln2_hi
#define EXP_LN2_LOK MC.e64_ln2_lo
#endif
constexpr int kExpMask = (1 << kExpBits) - 1;
// QMCCPW_ICDF_SHIFTED_LOG (W1 units, with the shared tables): the normals' logarithm returns
// ln t + 3.125 directly -- a second table (1/c_i, ln c_i + 3.125) -- so the central polynomial's
// variable v = -ln t - 3.125 is its negation (free in the DFMA) and the tail test w >= 6.25 is the
// integer test hi(ln t + 3.125) >= hi(-3.125) on the sign-magnitude word (no DADD, no DSETP)
#ifndef QMCCPW_ICDF_SHIFTED_LOG
#define QMCCPW_ICDF_SHIFTED_LOG 0
#endif
#if QMCCPW_SMEM_TABLES && QMCCPW_ICDF_SHIFTED_LOG
__shared__ double2 s_log_tab_c[64];
#endif
__device__ __forceinline__ void math_tables_load(int tid, int nthreads) {
#if QMCCPW_SMEM_TABLES
#if QMCCPW_EXP256_ON
    for (int i = tid; i < 256; i += nthreads) s_exp_tab[i] = __ldg(EXP_TAB256 + i);
#endif
    for (int i = tid; i < 64; i += nthreads) {
        s_log_tab[i] = __ldg(reinterpret_cast<const double2*>(LOG_TAB) + i);
#if !QMCCPW_EXP256_ON
        s_exp_tab[i] = __ldg(EXP_TAB + i);
#endif
#if QMCCPW_ICDF_SHIFTED_LOG
        const double2 c = __ldg(reinterpret_cast<const double2*>(LOG_TAB) + i);
        s_log_tab_c[i] = make_double2(c.x, c.y + 3.125);
#endif
    }
#else
    (void)tid;
    (void)nthreads;
#endif
}

// exp(x) for |x| < 700 (all arguments on this path are bounded far inside):
// x = (64 k + j) ln2/64 + r, |r| <= ln2/128, e^x = 2^k 2^(j/64) e^r with 2^(j/64)
// from a 64-entry table (512 B, staged in shared memory) and e^r by a degree-6
// polynomial (rel. error 3.4e-21 before rounding); 2^k added to the exponent field.
// 7 coefficients instead of 13: ~40 % fewer FP64 operations than a |r| <= ln2/2 form.
__device__ __forceinline__ double fast_exp(double x) {
    const double t = fma(x, EXP_INV_LN2K, MC.shift);
    const int ni = __double2loint(t);
    const double n = t - MC.shift;
    double r = fma(n, -EXP_LN2_HIK, x);
    r = fma(n, -EXP_LN2_LOK, r);
    const double T = QMCCPW_EXP_TAB(ni & kExpMask);
    double p = EXP_PK[kExpDegK];
#pragma unroll
    for (int j = kExpDegK - 1; j >= 0; --j) p = fma(p, r, EXP_PK[j]);
    p *= T;
    return __hiloint2double(__double2hiint(p) + ((ni >> kExpBits) << 20), __double2loint(p));
}

// 1/y for y in [1, 4): FP64 MUFU seed + two Newton steps
__device__ __forceinline__ double rcp_newton(double y) {
    double r;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(y));
    double e = fma(-y, r, MC.one);
    r = fma(r, e, r);
    e = fma(-y, r, MC.one);
    return fma(r, e, r);
}

// ln(t) for normal t > 0 by table lookup: t = 2^k m, m in [1, 2), i = top 6 mantissa
// bits, ln t = k ln2 + ln c_i + log1p(r), r = fma(m, 1/c_i, -1) (|r| <= 2^-7, one
// rounding), log1p(r) = r + r^2 L(r).  QMCCPW_LOG1P_FACTORED (set by the W1 units): r (1 + r L(r))
// added to ln c_i in one fma, two FP64 operations for r + r^2 L + ln c_i instead of three and one
// rounding fewer (A/B: W1 modes -0.6 %, but C5 +2 % -- its constant-bank layout; off elsewhere).
// ~10 FP64 ops and no MUFU against ~22 + a MUFU
// for the atanh form; the 1 KB table is staged in shared memory (math_tables_load).
#ifndef QMCCPW_LOG1P_FACTORED
#define QMCCPW_LOG1P_FACTORED 0
#endif
#if QMCCPW_LOG1P_FACTORED
#define LOG1P_PLUS(r, p, c) fma((r), fma((r), (p), MC.one), (c))
#else
#define LOG1P_PLUS(r, p, c) (fma((r) * (r), (p), (r)) + (c))
#endif
__device__ __forceinline__ void fast_log_x2(double ta, double tb, double& la, double& lb) {
    const int ha = __double2hiint(ta), hb = __double2hiint(tb);
    const double ma = __hiloint2double((ha & 0x000FFFFF) | 0x3FF00000, __double2loint(ta));
    const double mb = __hiloint2double((hb & 0x000FFFFF) | 0x3FF00000, __double2loint(tb));
    const double ka = (double)((ha >> 20) - 1023), kb = (double)((hb >> 20) - 1023);
    const double2 ca = QMCCPW_LOG_TAB((ha >> 14) & 63);
    const double2 cb = QMCCPW_LOG_TAB((hb >> 14) & 63);
    const double ra = fma(ma, ca.x, -MC.one), rb = fma(mb, cb.x, -MC.one);
    double pa = LOG_P[kLogDeg], pb = LOG_P[kLogDeg];
#pragma unroll
    for (int j = kLogDeg - 1; j >= 0; --j) {
        pa = fma(pa, ra, LOG_P[j]);
        pb = fma(pb, rb, LOG_P[j]);
    }
    const double sa = LOG1P_PLUS(ra, pa, ca.y), sb = LOG1P_PLUS(rb, pb, cb.y);
    la = fma(ka, MC.ln2_hi, fma(ka, MC.ln2_lo, sa));
    lb = fma(kb, MC.ln2_hi, fma(kb, MC.ln2_lo, sb));
}

__device__ __forceinline__ double fast_log(double t) {
    const int h = __double2hiint(t);
    const double m = __hiloint2double((h & 0x000FFFFF) | 0x3FF00000, __double2loint(t));
    const double k = (double)((h >> 20) - 1023);
    const double2 c = QMCCPW_LOG_TAB((h >> 14) & 63);
    const double r = fma(m, c.x, -MC.one);
    double p = LOG_P[kLogDeg];
#pragma unroll
    for (int j = kLogDeg - 1; j >= 0; --j) p = fma(p, r, LOG_P[j]);
    return fma(k, MC.ln2_hi, fma(k, MC.ln2_lo, LOG1P_PLUS(r, p, c.y)));
}

// degree of the central Phi^{-1} polynomial (fit_device_polys.py: max rel. error of the
// double-rounded polynomial 4.3e-17 at 24, 1.7e-16 at 23, 3.3e-16 at 22)
constexpr int kIcdfDeg = QMCCPW_ICDF_DEG;
#if QMCCPW_ICDF_DEG == 24
#define ICDF_C ICDF_CENTRAL
#elif QMCCPW_ICDF_DEG == 23
#define ICDF_C ICDF_CENTRAL_D23
#elif QMCCPW_ICDF_DEG == 22
#define ICDF_C ICDF_CENTRAL_D22
#else
#error "QMCCPW_ICDF_DEG must be 22, 23 or 24"
#endif

// z = 2u - 1 for the lower-half lattice word yl < 2^31, u = (yl + 1/2) 2^-32, in one FP64 add:
// (2 yl + 1) 2^-32 - 1 with the odd integer 2 yl + 1 < 2^32 converted exactly, scaled by an
// exponent decrement, and no constant register; the result is exact (z = -(2^32 - 2 yl - 1) 2^-32 has 32 significant bits), and so
// is 1 - z^2 = 4u(1 - u) before its one rounding: fma(-z, z, 1) is bit-identical to the former
// (4u)(1 - u) with 4u and 1 - u exact (three FP64 operations fewer per normal)
__device__ __forceinline__ double z_from_lower(uint32_t yl) {
    const double o = (double)(2u * yl + 1u);  // >= 1: the 2^-32 scale is an exponent decrement
    return __hiloint2double(__double2hiint(o) - (32 << 20), __double2loint(o)) - 1.0;
}

// -r when the lattice point is in the upper half (y >= 2^31), else r: the sign bit of y moved into
// r's sign bit (one integer op; the select form cost a DADD negation and two FSELs)
__device__ __forceinline__ double mirror_upper(double r, uint32_t y) {
    return __hiloint2double(__double2hiint(r) ^ (int)(y & 0x80000000u), __double2loint(r));
}

// (a3) lattice point -> standard normal, Phi^{-1}((y + 1/2) 2^-32).
// Lower half (y < 2^31) evaluated, upper half mirrored (exact symmetry).
// Giles' variable w = -ln(1 - z^2) = -ln(4u(1-u)), z = 2u - 1 (exact):
// Phi^{-1}(u) = z P(w); the central polynomial covers u > 4.8e-4, so ~97% of
// warps never enter the tail branch.
__device__ __forceinline__ double normal_from_u32(uint32_t y) {
    const bool upper = (y >> 31) != 0u;
    const uint32_t yl = upper ? ~y : y;
    const double z = z_from_lower(yl);
    const double t = fma(-z, z, 1.0);  // = 4u(1 - u) exactly before rounding (see z_from_lower)
    const double w = -fast_log(t);
    double p;
    if (w < MC.w_split) {
        const double v = w - ICDF_CENTRAL_CENTER;
        p = ICDF_C[kIcdfDeg];
#pragma unroll
        for (int j = kIcdfDeg - 1; j >= 0; --j) p = fma(p, v, ICDF_C[j]);
    } else {
        const double v = sqrt(w) - ICDF_TAIL_CENTER;
        p = ICDF_TAIL[24];
#pragma unroll
        for (int j = 23; j >= 0; --j) p = fma(p, v, ICDF_TAIL[j]);
    }
    return mirror_upper(z * p, y);
}

// phi(x); flushes to 0 below e^-700 (|x| > 37.4), where fast_exp's exponent
// arithmetic would leave the normal range (the oracle's value there is < 1e-305)
// ---- paired versions: two independent evaluations interleaved, so every
// coefficient loaded into a uniform register feeds two DFMAs and the two Horner
// chains hide each other's latency ------------------------------------------
__device__ __forceinline__ void fast_exp_x2(double xa, double xb, double& ra, double& rb) {
    const double ta = fma(xa, EXP_INV_LN2K, MC.shift), tb = fma(xb, EXP_INV_LN2K, MC.shift);
    const int na = __double2loint(ta), nb = __double2loint(tb);
    const double Ta = QMCCPW_EXP_TAB(na & kExpMask), Tb = QMCCPW_EXP_TAB(nb & kExpMask);
    const double fa = ta - MC.shift, fb = tb - MC.shift;
    double qa = fma(fa, -EXP_LN2_HIK, xa), qb = fma(fb, -EXP_LN2_HIK, xb);
    qa = fma(fa, -EXP_LN2_LOK, qa);
    qb = fma(fb, -EXP_LN2_LOK, qb);
    double pa = EXP_PK[kExpDegK], pb = EXP_PK[kExpDegK];
#pragma unroll
    for (int j = kExpDegK - 1; j >= 0; --j) {
        pa = fma(pa, qa, EXP_PK[j]);
        pb = fma(pb, qb, EXP_PK[j]);
    }
    pa *= Ta;
    pb *= Tb;
    ra = __hiloint2double(__double2hiint(pa) + ((na >> kExpBits) << 20), __double2loint(pa));
    rb = __hiloint2double(__double2hiint(pb) + ((nb >> kExpBits) << 20), __double2loint(pb));
}

// four exponentials with interleaved Horner chains (one coefficient load per four DFMAs)
__device__ __forceinline__ void fast_exp_x4(const double (&x)[4], double (&r)[4]) {
    double t[4], f[4], q[4], T[4], p[4];
    int n[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        t[i] = fma(x[i], EXP_INV_LN2K, MC.shift);
        n[i] = __double2loint(t[i]);
        T[i] = QMCCPW_EXP_TAB(n[i] & kExpMask);
        f[i] = t[i] - MC.shift;
        q[i] = fma(f[i], -EXP_LN2_HIK, x[i]);
    }
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        q[i] = fma(f[i], -EXP_LN2_LOK, q[i]);
        p[i] = EXP_PK[kExpDegK];
    }
#pragma unroll
    for (int j = kExpDegK - 1; j >= 0; --j)
#pragma unroll
        for (int i = 0; i < 4; ++i) p[i] = fma(p[i], q[i], EXP_PK[j]);
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        p[i] *= T[i];
        r[i] = __hiloint2double(__double2hiint(p[i]) + ((n[i] >> kExpBits) << 20), __double2loint(p[i]));
    }
}

static __device__ __noinline__ double icdf_tail_poly(double w) {
    const double v = sqrt(w) - ICDF_TAIL_CENTER;
    double p = ICDF_TAIL[24];
#pragma unroll
    for (int j = 23; j >= 0; --j) p = fma(p, v, ICDF_TAIL[j]);
    return p;
}

// two lattice points -> two standard normals (same arithmetic as normal_from_u32)
#ifndef QMCCPW_ICDF_SHIFTED_X2
#define QMCCPW_ICDF_SHIFTED_X2 0
#endif
#if !(QMCCPW_SMEM_TABLES && QMCCPW_ICDF_SHIFTED_LOG && QMCCPW_ICDF_SHIFTED_X2)  // (else: the xn<2> form, below)
__device__ __forceinline__ void normal_from_u32_x2(uint32_t ya, uint32_t yb, double& xa, double& xb) {
    const bool upa = (ya >> 31) != 0u, upb = (yb >> 31) != 0u;
    const uint32_t la = upa ? ~ya : ya, lb = upb ? ~yb : yb;
    const double za = z_from_lower(la), zb = z_from_lower(lb);
    const double ta = fma(-za, za, 1.0), tb = fma(-zb, zb, 1.0);
    double wa, wb;
    fast_log_x2(ta, tb, wa, wb);
    wa = -wa;
    wb = -wb;
    const double va = wa - ICDF_CENTRAL_CENTER, vb = wb - ICDF_CENTRAL_CENTER;
    double pa = ICDF_C[kIcdfDeg], pb = ICDF_C[kIcdfDeg];
#pragma unroll
    for (int j = kIcdfDeg - 1; j >= 0; --j) {
        pa = fma(pa, va, ICDF_C[j]);
        pb = fma(pb, vb, ICDF_C[j]);
    }
    if (wa >= MC.w_split) pa = icdf_tail_poly(wa);  // u < 4.8e-4: rare, divergent
    if (wb >= MC.w_split) pb = icdf_tail_poly(wb);
    const double ra = za * pa, rb = zb * pb;
    xa = mirror_upper(ra, ya);
    xb = mirror_upper(rb, yb);
}
#endif

// one lattice point -> one normal, out of line: for the bridge's rare data-dependent levels
// (the terminal and the levels c >= 3 of each group's first descent), so that their copies
// of the polynomial do not sit in the hot loop's instruction stream
static __device__ __noinline__ double normal_from_u32_call(uint32_t y) { return normal_from_u32(y); }

// ln t for N arguments at once (same arithmetic as fast_log / fast_log_x2)
// SHIFTED (QMCCPW_ICDF_SHIFTED_LOG): l = ln t + 3.125
template <int N, bool SHIFTED = false>
__device__ __forceinline__ void fast_log_xn(const double (&t)[N], double (&l)[N]) {
    double m[N], k[N], r[N], p[N];
    double2 c[N];
#pragma unroll
    for (int i = 0; i < N; ++i) {
        const int h = __double2hiint(t[i]);
        m[i] = __hiloint2double((h & 0x000FFFFF) | 0x3FF00000, __double2loint(t[i]));
        k[i] = (double)((h >> 20) - 1023);
#if QMCCPW_SMEM_TABLES && QMCCPW_ICDF_SHIFTED_LOG
        c[i] = SHIFTED ? s_log_tab_c[(h >> 14) & 63] : QMCCPW_LOG_TAB((h >> 14) & 63);
#else
        c[i] = QMCCPW_LOG_TAB((h >> 14) & 63);
#endif
        r[i] = fma(m[i], c[i].x, -MC.one);
        p[i] = LOG_P[kLogDeg];
    }
#pragma unroll
    for (int j = kLogDeg - 1; j >= 0; --j)
#pragma unroll
        for (int i = 0; i < N; ++i) p[i] = fma(p[i], r[i], LOG_P[j]);
#pragma unroll
    for (int i = 0; i < N; ++i) {
        const double s = LOG1P_PLUS(r[i], p[i], c[i].y);
        l[i] = fma(k[i], MC.ln2_hi, fma(k[i], MC.ln2_lo, s));
    }
}

// N lattice points -> N standard normals (same arithmetic as normal_from_u32): N interleaved
// Horner chains, so each coefficient loaded into a uniform register feeds N DFMAs
template <int N>
__device__ __forceinline__ void normal_from_u32_xn(const uint32_t (&y)[N], double (&x)[N]) {
    bool up[N];
    double z[N], t[N], w[N], v[N], p[N];
#pragma unroll
    for (int i = 0; i < N; ++i) {
        up[i] = (y[i] >> 31) != 0u;
        const uint32_t l = up[i] ? ~y[i] : y[i];
        z[i] = z_from_lower(l);
        t[i] = fma(-z[i], z[i], 1.0);
    }
#if QMCCPW_SMEM_TABLES && QMCCPW_ICDF_SHIFTED_LOG
    fast_log_xn<N, true>(t, w);  // w = ln t + 3.125 = -(v)
#pragma unroll
    for (int i = 0; i < N; ++i) {
        v[i] = -w[i];
        p[i] = ICDF_C[kIcdfDeg];
    }
#pragma unroll
    for (int j = kIcdfDeg - 1; j >= 0; --j)
#pragma unroll
        for (int i = 0; i < N; ++i) p[i] = fma(p[i], v[i], ICDF_C[j]);
#pragma unroll
    for (int i = 0; i < N; ++i) {
        // -ln t >= 6.25  <=>  ln t + 3.125 <= -3.125: the high word of a negative double grows
        // with its magnitude, and -3.125's low word is zero
        if ((uint32_t)__double2hiint(w[i]) >= 0xC0090000u) p[i] = icdf_tail_poly(3.125 - w[i]);
        x[i] = mirror_upper(z[i] * p[i], y[i]);
    }
#else
    fast_log_xn<N>(t, w);
#pragma unroll
    for (int i = 0; i < N; ++i) {
        w[i] = -w[i];
        v[i] = w[i] - ICDF_CENTRAL_CENTER;
        p[i] = ICDF_C[kIcdfDeg];
    }
#pragma unroll
    for (int j = kIcdfDeg - 1; j >= 0; --j)
#pragma unroll
        for (int i = 0; i < N; ++i) p[i] = fma(p[i], v[i], ICDF_C[j]);
#pragma unroll
    for (int i = 0; i < N; ++i) {
        if (w[i] >= MC.w_split) p[i] = icdf_tail_poly(w[i]);  // u < 4.8e-4: rare, divergent
        x[i] = mirror_upper(z[i] * p[i], y[i]);
    }
#endif
}
#if QMCCPW_SMEM_TABLES && QMCCPW_ICDF_SHIFTED_LOG && QMCCPW_ICDF_SHIFTED_X2
// (per unit: the PCA-W1 kernel gains with it, STD-W1 loses 7 % -- measured)
__device__ __forceinline__ void normal_from_u32_x2(uint32_t ya, uint32_t yb, double& xa, double& xb) {
    const uint32_t y[2] = {ya, yb};
    double x[2];
    normal_from_u32_xn<2>(y, x);
    xa = x[0];
    xb = x[1];
}
#endif
// four lattice points -> four standard normals: each coefficient loaded into a uniform register
// feeds four DFMAs (half the constant-load instructions per normal of the paired form)
__device__ __forceinline__ void normal_from_u32_x4(const uint32_t (&y)[4], double (&x)[4]) {
    normal_from_u32_xn<4>(y, x);
}

__device__ __forceinline__ double normal_pdf(double x) {
    const double a = MC.minus_half * x * x;
    return a > MC.pdf_floor ? MC.inv_sqrt_2pi * fast_exp(a) : 0.0;
}
// Phibar(x) = 1 - Phi(x) and phi(x) together, for two arguments.  Phibar(|x|) =
// phi(|x|) R(|x|), R the Mills ratio: h(t) = (|x| + 3) R, t = (|x| - 3)/(|x| + 3),
// polynomial fitted on |x| <= 40 (rel. 6e-17); x^2 is split exactly (hi + lo)
// so phi keeps full relative accuracy in the tails.  For x < 0, 1 - Phibar(|x|)
// with Phibar(|x|) <= 1/2: no cancellation (reading 22: never 1 - Phi(psi)).
__device__ __forceinline__ void phibar_phi_x2(double xa, double xb, double& Qa, double& Qb, double& pha,
                                              double& phb) {
    const double aa = fabs(xa), ab = fabs(xb);
    const double ra = rcp_newton(aa + MC.mills_c), rb = rcp_newton(ab + MC.mills_c);
    const double ta = fma(-MC.mills_2c, ra, MC.one) - MILLS_H_CENTER, tb = fma(-MC.mills_2c, rb, MC.one) - MILLS_H_CENTER;
    double ha = MILLS_P[kMillsDeg], hb = MILLS_P[kMillsDeg];
#pragma unroll
    for (int j = kMillsDeg - 1; j >= 0; --j) {
        ha = fma(ha, ta, MILLS_P[j]);
        hb = fma(hb, tb, MILLS_P[j]);
    }
    const double sa = aa * aa, sb = ab * ab;
    const double la = fma(aa, aa, -sa), lb = fma(ab, ab, -sb);
    double ea, eb;
    fast_exp_x2(MC.minus_half * sa, MC.minus_half * sb, ea, eb);
    pha = (sa < MC.exp_floor * MC.two) ? MC.inv_sqrt_2pi * ea * fma(MC.minus_half, la, MC.one) : 0.0;
    phb = (sb < MC.exp_floor * MC.two) ? MC.inv_sqrt_2pi * eb * fma(MC.minus_half, lb, MC.one) : 0.0;
    const double qa = pha * (ha * ra), qb = phb * (hb * rb);
    Qa = xa >= 0.0 ? qa : MC.one - qa;
    Qb = xb >= 0.0 ? qb : MC.one - qb;
}
// The Mills ratio R(|x|) = Phibar(|x|) / phi(|x|) alone, for two arguments: the polynomial
// part of phibar_phi_x2, same arithmetic (Phibar(|x|) = phi(|x|) R(|x|) there).  The X1
// arithmetic sums use it with w_j phi(u - sigma a_j) = phi(u) E_j (qmccpw_device.cuh x1_solve).
__device__ __forceinline__ void mills_x2(double xa, double xb, double& Ra, double& Rb) {
    const double aa = fabs(xa), ab = fabs(xb);
    const double ra = rcp_newton(aa + MC.mills_c), rb = rcp_newton(ab + MC.mills_c);
    const double ta = fma(-MC.mills_2c, ra, MC.one) - MILLS_H_CENTER, tb = fma(-MC.mills_2c, rb, MC.one) - MILLS_H_CENTER;
    double ha = MILLS_P[kMillsDeg], hb = MILLS_P[kMillsDeg];
#pragma unroll
    for (int j = kMillsDeg - 1; j >= 0; --j) {
        ha = fma(ha, ta, MILLS_P[j]);
        hb = fma(hb, tb, MILLS_P[j]);
    }
    Ra = ha * ra;
    Rb = hb * rb;
}

// The same for four arguments (two options of the C5 portfolio's phase B): four
// independent Horner chains per coefficient load.
__device__ __forceinline__ void phibar_phi_x4(const double (&x)[4], double (&Q)[4], double (&ph)[4]) {
    double a[4], r[4], t[4], h[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        a[i] = fabs(x[i]);
        r[i] = rcp_newton(a[i] + MC.mills_c);
        t[i] = fma(-MC.mills_2c, r[i], MC.one) - MILLS_H_CENTER;
        h[i] = MILLS_P[kMillsDeg];
    }
#pragma unroll
    for (int j = kMillsDeg - 1; j >= 0; --j)
#pragma unroll
        for (int i = 0; i < 4; ++i) h[i] = fma(h[i], t[i], MILLS_P[j]);
    double sq[4], lo[4], e[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        sq[i] = a[i] * a[i];
        lo[i] = fma(a[i], a[i], -sq[i]);
    }
    fast_exp_x2(MC.minus_half * sq[0], MC.minus_half * sq[1], e[0], e[1]);
    fast_exp_x2(MC.minus_half * sq[2], MC.minus_half * sq[3], e[2], e[3]);
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        ph[i] = (sq[i] < MC.exp_floor * MC.two) ? MC.inv_sqrt_2pi * e[i] * fma(MC.minus_half, lo[i], MC.one) : 0.0;
        const double q = ph[i] * (h[i] * r[i]);
        Q[i] = x[i] >= 0.0 ? q : MC.one - q;
    }
}

// The Mills ratio R(|x|) for four arguments (four Horner chains per coefficient load), and
// phi for two: the two halves of phibar_phi_x4, same arithmetic.  The C5 portfolio's phase B
// combines them with A S~ phi(psi - s) = D K phi(psi), so one phi serves both Phibar's.
__device__ __forceinline__ void mills_x4(const double (&x)[4], double (&R)[4]) {
    double a[4], r[4], t[4], h[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        a[i] = fabs(x[i]);
        r[i] = rcp_newton(a[i] + MC.mills_c);
        t[i] = fma(-MC.mills_2c, r[i], MC.one) - MILLS_H_CENTER;
        h[i] = MILLS_P[kMillsDeg];
    }
#pragma unroll
    for (int j = kMillsDeg - 1; j >= 0; --j)
#pragma unroll
        for (int i = 0; i < 4; ++i) h[i] = fma(h[i], t[i], MILLS_P[j]);
#pragma unroll
    for (int i = 0; i < 4; ++i) R[i] = h[i] * r[i];
}
__device__ __forceinline__ void phi_x2(double xa, double xb, double& pa, double& pb) {
    const double aa = fabs(xa), ab = fabs(xb);
    const double sa = aa * aa, sb = ab * ab;
    const double la = fma(aa, aa, -sa), lb = fma(ab, ab, -sb);
    double ea, eb;
    fast_exp_x2(MC.minus_half * sa, MC.minus_half * sb, ea, eb);
    pa = (sa < MC.exp_floor * MC.two) ? MC.inv_sqrt_2pi * ea * fma(MC.minus_half, la, MC.one) : 0.0;
    pb = (sb < MC.exp_floor * MC.two) ? MC.inv_sqrt_2pi * eb * fma(MC.minus_half, lb, MC.one) : 0.0;
}

__device__ __forceinline__ double normal_sf(double x) {
    double Q, Q2, ph, ph2;
    phibar_phi_x2(x, x, Q, Q2, ph, ph2);
    return Q;
}
__device__ __forceinline__ double normal_cdf(double x) { return normal_sf(-x); }

}  // namespace qmccpw
