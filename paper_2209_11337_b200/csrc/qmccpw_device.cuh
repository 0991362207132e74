// qmccpw_device.cuh -- device building blocks shared by the sm_100a kernels of the
// QMC-CPW hot path (arXiv 2209.11337): stateless Sobol' tables, the W1 accumulators,
// the option tails, X1 threshold solvers, the LR path and the block reductions.
//
// One thread carries one path at a time through the whole pipeline in FP64
// ("each thread will be responsible for the simulation of one
// path"), but nothing is materialised in HBM: Sobol' integers come from two
// per-block shared-memory tables, the normals are consumed as they are produced,
// the Brownian bridge is generated in time order from a log2(d)-deep stack, and
// each block reduces its cell of 4096 points to one row of partial sums.  The
// paper instead materialises normals and the bridge in global memory and names
// that round trip as its 4x slowdown.
//
// Device code here is independent of oracle/: it is written from the paper
// and SURVEY.md Sec. 8(a); tests compare the two on the same points.
#pragma once
#include <cuda_runtime.h>
#include <math_constants.h>
#include <stdint.h>

#include "qmccpw_internal.h"
#include "qmccpw_math.cuh"

namespace qmccpw {

// ---------------------------------------------------------------------------
// (a2) Sobol' integers without per-thread state.  A block of 2^p threads visits
// the points k = K0 + tid + a 2^p (a = 0, 1, ...).  With k = A 2^p + tau and
// tau = 32 w + l (l the lane slot), the Gray code g(k) = k ^ (k >> 1) splits as
//   g(k) = (g(A) << p) ^ ((A & 1) << (p-1)) ^ g(l) ^ ((w & 1) << 4) ^ (g(w) << 5)
// (P:147-151 XOR form), so y_j(k) = HW_j(A, w) ^ G_j(l) with
//   G_j(l)    = XOR_{b in g(l)} v'_{j,b}                       (per block,  [d][32])
//   HW_j(A,w) = c_j ^ XOR_{b in g(A)} v'_{j,p+b} ^ (A&1) v'_{j,p-1}
//               ^ (w&1) v'_{j,4} ^ XOR_{b in g(w)} v'_{j,5+b}      (per point iteration)
// Threads of a block share A up to +1 (first index not 2^p-aligned), so HW is
// built for A and A+1 (f = 0, 1).  Per dimension a thread does two
// shared-memory loads and one XOR; nothing is stored per thread.
// ---------------------------------------------------------------------------
// (a2, row f4) nested uniform (Owen) scramble of one coordinate: on the bit-reversed
// integer (digit i of y -> bit i), add the dimension's seed and apply four
// xor-multiplies by even constants (Laine-Karras hash, Burley's constants): carries
// and even products only move information towards higher bits, so output digit i is
// input digit i flipped by a function of (seed, digits 0..i-1).  BREV + 4 IMAD + 4 LOP3.
__device__ __forceinline__ uint32_t owen_scramble(uint32_t y, uint32_t seed) {
    uint32_t r = __brev(y) + seed;
    r ^= r * 0x6c50b47cu;
    r ^= r * 0xb82f1e52u;
    r ^= r * 0xc7afe638u;
    r ^= r * 0x8d22f6e6u;
    return __brev(r);
}

struct SobolBlock {
    const uint32_t* G;   // smem [d][32]
    const uint32_t* HW;  // smem, current buffer [2][nw][d]
    int d, nw;
    int lane_t, w_t, f_t;
    const uint32_t* os = nullptr;  // Owen seeds [d] (smem) or nullptr (LMS / shift / plain: folded into HW)
    __device__ __forceinline__ uint32_t get(int j) const {
        QMCCPW_CHECK(j >= 0 && j < d && f_t >= 0 && f_t < 2 && w_t >= 0 && w_t < nw && lane_t >= 0 && lane_t < 32);
        QMCCPW_CHK_SMEM(&HW[(f_t * nw + w_t) * d + j]);
        QMCCPW_CHK_SMEM(&G[j * 32 + lane_t]);
        const uint32_t y = HW[(f_t * nw + w_t) * d + j] ^ G[j * 32 + lane_t];
        return os != nullptr ? owen_scramble(y, os[j]) : y;
    }
};

__device__ __forceinline__ void sobol_build_g(const uint32_t* vt, int d, uint32_t* G, int tid, int tpb) {
    for (int idx = tid; idx < d * 32; idx += tpb) {
        const int j = idx >> 5, l = idx & 31;
        const int g = l ^ (l >> 1);
        uint32_t y = 0;
#pragma unroll
        for (int b = 0; b < 5; ++b)
            if ((g >> b) & 1) y ^= vt[j * 32 + b];
        QMCCPW_CHK_SMEM(&G[idx]);
        G[idx] = y;
    }
}

// The same table built incrementally.  HW_j(A, w) = B_j(A) ^ WP_j(w) with
//   B_j(A) = c_j ^ XOR_{b in g(A)} v'_{j,p+b} ^ (A&1) v'_{j,p-1},  WP_j(w) = (w&1) v'_{j,4} ^ XOR_{b in g(w)} v'_{j,5+b},
// and the Gray code of A+1 differs from that of A in bit ctz(A+1) only, so
//   B_j(A+1) = B_j(A) ^ v'_{j,p+ctz(A+1)} ^ v'_{j,p-1}:
// one XOR pair per dimension per step instead of a popcount loop.  B_j(A+1) of this step
// is B_j(A) of the next one; BS [d] keeps it (owned by the thread of dimension j, so no
// extra barrier).  first: build B_j(A) directly.
__device__ __forceinline__ uint32_t sobol_base_step(const uint32_t* v, int p, uint64_t A1) {
    const int c = __ffsll((long long)A1) - 1;  // A1 >= 1
    uint32_t r = v[p - 1];
    if (p + c < 32) r ^= v[p + c];
    return r;
}
__device__ __forceinline__ void sobol_build_hw_inc(const uint32_t* vt, const uint32_t* sh, int d, int j0, int p, int nw,
                                                   uint64_t A, bool first, uint32_t* BS, uint32_t* HW, int tid,
                                                   int tpb) {
    for (int j = tid; j < d; j += tpb) {
        if (j < j0) continue;
        const uint32_t* v = vt + j * 32;
        uint32_t b0;
        if (first) {
            b0 = sh != nullptr ? sh[j] : 0u;
            if (A & 1) b0 ^= v[p - 1];
            uint32_t gA = (uint32_t)(A ^ (A >> 1)) & ((p >= 32) ? 0u : (0xFFFFFFFFu >> p));
            while (gA) {
                b0 ^= v[p + __ffs(gA) - 1];
                gA &= gA - 1;
            }
        } else {
            b0 = BS[j];
        }
        const uint32_t b1 = b0 ^ sobol_base_step(v, p, A + 1);
        QMCCPW_CHK_SMEM(&BS[j]);
        BS[j] = b1;
        const uint32_t v4 = v[4], v5 = v[5], v6 = v[6];
        for (int w = 0; w < nw; ++w) {
            const int gw = w ^ (w >> 1);
            const uint32_t wp = ((w & 1) ? v4 : 0u) ^ ((gw & 1) ? v5 : 0u) ^ ((gw & 2) ? v6 : 0u);
            QMCCPW_CHK_SMEM(&HW[(nw + w) * d + j]);
            HW[w * d + j] = b0 ^ wp;
            HW[(nw + w) * d + j] = b1 ^ wp;
        }
    }
}

__device__ __forceinline__ void sobol_build_hw(const uint32_t* vt, const uint32_t* sh, int d, int j0, int p, int nw,
                                               uint64_t A0, uint32_t* HW, int tid, int tpb) {
    const int n = 2 * nw * d;
    for (int idx = tid; idx < n; idx += tpb) {
        const int j = idx % d, rest = idx / d;
        if (j < j0) continue;
        const int w = rest % nw, f = rest / nw;
        const uint64_t A = A0 + (uint64_t)f;
        const uint32_t* v = vt + j * 32;
        uint32_t y = sh != nullptr ? sh[j] : 0u;  // nullptr: unshifted (Owen: sh holds the seeds)
        if (A & 1) y ^= v[p - 1];
        if (w & 1) y ^= v[4];
        const int gw = w ^ (w >> 1);
        if (gw & 1) y ^= v[5];
        if (gw & 2) y ^= v[6];
        uint32_t gA = (uint32_t)(A ^ (A >> 1)) & ((p >= 32) ? 0u : (0xFFFFFFFFu >> p));
        while (gA) {
            const int b = __ffs(gA) - 1;
            y ^= v[p + b];
            gA &= gA - 1;
        }
        HW[idx] = y;
    }
}

// ---------------------------------------------------------------------------
// (a5) W1-mode accumulators over the separated path S~(t_j):
// S~_A, I_A (vega inner sum), and the lookback's S~_max with the
// lowest argmax j* and I_max = S~_{j*}(W~_{j*} - sigma(t_{j*} - t_1))
// (P:599 with the 1/d removed, reading 3).  Near-ties are tracked with the
// runner-up exponent.
// ---------------------------------------------------------------------------
// (MC-CPW / MC+AV-CPW / LR+MC normals, drawn in paths_kernel and lr_path: Philox4x32-10,
// counter (k_lo, k_hi, j/4, (rep<<8)|0x02), word j%4 -- the paper's PSEUDO generator.)
// QMCCPW_TRACK_FLAG: the near-tie test of the lookback's argmax kept as a flag ("the runner-up
// is within 1e-12 of the running maximum", reset when a new maximum clears the old one by
// 1e-12) instead of the runner-up value itself: the same decision (both compare the same
// difference of two doubles), two instructions and one register pair less per date
#ifndef QMCCPW_TRACK_FLAG
#define QMCCPW_TRACK_FLAG 1
#endif
struct W1Acc {
    double sumS, sumI, emax, esec, ymax;
    bool tie;
    __device__ __forceinline__ void reset() {
        sumS = 0.0; sumI = 0.0; emax = -CUDART_INF; esec = -CUDART_INF; ymax = 0.0;
        tie = false;
    }
    // lookback: lowest argmax of e_j (= argmax of S~_j) and the runner-up exponent,
    // with plain compare-selects (no NaN-aware fmax/fmin: e is always finite)
    __device__ __forceinline__ void track(double e, double y) {
#if QMCCPW_TRACK_FLAG
        const double dd = e - emax;  // -inf - (-inf) never happens: emax starts at -inf, e is finite
        const bool gt = dd > 0.0;
        const bool near = fabs(dd) < 1e-12;
        tie = gt ? near : (tie || near);
        ymax = gt ? y : ymax;
        emax = gt ? e : emax;
#else
        const bool gt = e > emax;
        const double cand = gt ? emax : e;
        esec = cand > esec ? cand : esec;
        ymax = gt ? y : ymax;
        emax = gt ? e : emax;
#endif
    }
    // a near-tie of the argmax (reading 20): the runner-up within 1e-12 of the maximum in log
    __device__ __forceinline__ bool near_tie() const {
#if QMCCPW_TRACK_FLAG
        return tie;
#else
        return emax - esec < 1e-12;
#endif
    }
    // set from a (max, runner-up) pair reduced elsewhere (the PCA quad reduction)
    __device__ __forceinline__ void set_max(double em, double es, double ym) {
        emax = em;
        esec = es;
        ymax = ym;
        tie = em - es < 1e-12;
    }
    // date index j (0-based, t_{j+1} - t_1 = j dt), Wt = W~(t_{j+1} - t_1); P.wt[j] = (omega j dt,
    // sigma j dt), read from the constant bank (j is warp-uniform in every caller).  The sums are
    // kept without the factor S0 (S~_j = S0 X_j): sumS = sum_j X_j, sumI = sum_j X_j y_j; the
    // tail scales by S0/d.
    __device__ __forceinline__ void push(const PathArgs& P, int j, double Wt) {
        const double2 c = P.wt[j];
        const double e = fma(P.sigma, Wt, c.x);
        const double X = fast_exp(e);
        const double y = Wt - c.y;
        sumS += X;
        sumI = fma(X, y, sumI);
        if (P.has_lookback) track(e, y);
    }
    // dates j and j+1 together (paired exp)
    __device__ __forceinline__ void push2(const PathArgs& P, int j, double Wa, double Wb) {
        const double2 ca = P.wt[j], cb = P.wt[j + 1];
        const double ea = fma(P.sigma, Wa, ca.x), eb = fma(P.sigma, Wb, cb.x);
        double Xa, Xb;
        fast_exp_x2(ea, eb, Xa, Xb);
        const double ya = Wa - ca.y, yb = Wb - cb.y;
        sumS += Xa;
        sumI = fma(Xa, ya, sumI);
        sumS += Xb;
        sumI = fma(Xb, yb, sumI);
        if (P.has_lookback) {
            track(ea, ya);
            track(eb, yb);
        }
    }
    // S~_max and I_max = S~_{j*} (W~_{j*} - sigma (t_{j*} - t_1)), rebuilt once per path
    __device__ __forceinline__ double smax(const PathArgs& P) const { return P.S0 * fast_exp(emax); }
};

// Two-slot FIFO of standard normals drawn in a fixed dimension order, two
// lattice points per refill (normal_from_u32_x2): the construction loops
// consume one normal at a time while the special functions run paired.
struct NormalFifo {
    double x0, x1;
    int have;
    __device__ __forceinline__ void reset() { have = 0; }
    template <class DimAt>
    __device__ __forceinline__ double next(const SobolBlock& sob, DimAt dim_at) {
        if (have == 0) {
            // the partner of the last normal of an odd count (BB-X1: d - 1 normals; d = 1) would be
            // table row d, past the [d] rows: clamp it (its value is never consumed).  Found by the
            // QMCCPW_CHECKED build (tests/test_memory_safety.py)
            const int j1 = dim_at(1);
            normal_from_u32_x2(sob.get(dim_at(0)), sob.get(j1 < sob.d ? j1 : sob.d - 1), x0, x1);
            have = 2;
        }
        const double r = (have == 2) ? x0 : x1;
        --have;
        return r;
    }
};

// P.wt in shared memory, for callers whose date index varies across the warp (the PCA quad
// layout): tt[j] = (omega t, sigma t) at t = j dt, j < d (t = t_{j+1} - t_1)
__device__ __forceinline__ void date_table_fill(const PathArgs& P, double2* tt, int tid, int tpb) {
    for (int j = tid; j < P.d; j += tpb) {
        QMCCPW_CHK_SMEM(&tt[j]);
        tt[j] = P.wt[j];
    }
}

// (a6)+(a7) W1 threshold psi_d and the closed-form smoothed
// payoff and Greeks (readings 1-5), all options of the
// launch at once.  Options with the same strike and statistic (the arithmetic
// and binary Asians of C4) share psi, phi(psi), Phibar(psi), Phibar(psi - s):
// P.tail_leader[o] names the first such option.
// sink(o, f4) receives option o's four values (price, delta, vega, gamma) as soon as they
// are formed, so a caller that reduces them at once keeps nothing per option live.
// Divisions: 1/S0 and 1/d come precomputed; I/stat is y_max for the maximum statistic
// (I_max = S_max y_max) and sumI/sumS for the average (the 1/d cancels); ln S_max =
// ln S0 + e_max needs no logarithm.
template <class Sink>
__device__ __forceinline__ void tail_w1_each(const PathArgs& P, const W1Acc& acc, Sink&& sink) {
    const double SA = acc.sumS * P.S0_inv_d, IA = acc.sumI * P.S0_inv_d;  // sums without S0 (W1Acc)
    const double Smax = P.has_lookback ? acc.smax(P) : SA;
    const double Imax = Smax * acc.ymax;
    const double lnSA = fast_log(SA);
    const double lnSmax = P.lnS0 + acc.emax;
    double psi[kMaxOpt], Q0[kMaxOpt], Q1[kMaxOpt], ph[kMaxOpt];
    const double D = P.Dfac, iS0 = P.inv_S0;
#pragma unroll
    for (int o = 0; o < kMaxOpt; ++o) {
        if (o >= P.n_opt) break;
        const bool lb = P.type[o] == kLookback;
        const int ld = P.tail_leader[o];
        if (ld == o) {
            psi[o] = (P.lnK[o] - (lb ? lnSmax : lnSA) - P.omega * P.t1) * P.inv_s;
            double phs;
            phibar_phi_x2(psi[o], psi[o] - P.s, Q0[o], Q1[o], ph[o], phs);
        } else {
            // leader index ld < o (so ld is 0 or 1), resolved with selects between constant
            // indices: an index expression here put these arrays in local memory
            psi[o] = ld == 0 ? psi[0] : psi[1];
            Q0[o] = ld == 0 ? Q0[0] : Q0[1];
            Q1[o] = ld == 0 ? Q1[0] : Q1[1];
            ph[o] = ld == 0 ? ph[0] : ph[1];
        }
        const double stat = lb ? Smax : SA;
        const double K = P.K[o];
        double f4[4];
        if (P.type[o] == kBinary) {
            const double rat = lb ? acc.ymax : acc.sumI / acc.sumS;  // I / stat
            const double Dph = D * ph[o];
            f4[0] = D * Q0[o];
            f4[1] = Dph * P.inv_s * iS0;
            f4[2] = Dph * (rat * P.inv_s + psi[o] * P.inv_sigma - P.sqrt_t1);
            f4[3] = Dph * P.inv_s * (iS0 * iS0) * (psi[o] * P.inv_s - 1.0);
        } else {
            const double I = lb ? Imax : IA;
            f4[0] = P.Afac * stat * Q1[o] - D * K * Q0[o];
            f4[1] = P.Afac * (stat * iS0) * Q1[o];
            f4[2] = P.Afac * Q1[o] * I + K * D * ph[o] * P.sqrt_t1;
            f4[3] = K * D * ph[o] * P.inv_s * (iS0 * iS0);
        }
        sink(o, f4);
    }
}
__device__ __forceinline__ void tail_w1_all(const PathArgs& P, const W1Acc& acc, double f[kMaxOpt][4]) {
    tail_w1_each(P, acc, [&](int o, const double (&f4)[4]) {
#pragma unroll
        for (int q = 0; q < 4; ++q) f[o][q] = f4[q];
    });
}
// (a6)+(a7) X1 mode: u* solves sum_j exp(c_j + sigma a_j u) = dK
// by Newton from the AM-GM start, warp-uniform iteration count, clamped to the
// bracket; then the conditional payoff and Greeks.  cb = per-thread c_j column.
struct X1Sums {
    double u, Dst, Qst, Vst, sumW, sumWv;
};

// X1 threshold step for f(u) = ln S(u) - ln(dK), S(u) = sum_j e^{c_j + sigma a_j u}:
// f' = sigma m1, f'' = sigma^2 (m2 - m1^2), m1 = SA/S, m2 = SAA/S.  Halley's update
// du = (f/f') / (1 - f f''/(2 f'^2)), the Newton step when the correction is large (far from
// the root); f is convex-increasing in u for a_j > 0, so both steps move toward the root.
__device__ __forceinline__ double halley_step(double h, double S, double SA, double SAA, double sg) {
    const double invS = 1.0 / S;
    const double m1 = SA * invS, m2 = SAA * invS;
    const double newton = h / (sg * m1);
    const double corr = 0.5 * h * (m2 - m1 * m1) / (m1 * m1);
    return fabs(corr) < 0.5 ? newton / (1.0 - corr) : newton;
}

__device__ __forceinline__ X1Sums x1_solve(const PathArgs& P, int o, bool arith, const double* cb, int stride,
                                           unsigned& unconverged) {
    const int d = P.d;
    const double lnK = P.lnK[o], lndK = P.lndK[o], sg = P.sigma;
    double u_lo = CUDART_INF, u_hi = CUDART_INF, sumc = 0.0;
    for (int j = 0; j < d; ++j) {
        const double cj = cb[j * stride];
        const double isa = P.inv_sa[j];
        u_lo = fmin(u_lo, (lnK - cj) * isa);
        u_hi = fmin(u_hi, (lndK - cj) * isa);
        sumc += cj;
    }
    double u = fmin(u_hi, (lnK - sumc / d) / (sg * P.mean_a));
    bool conv = false;
    if (P.a[0] == P.a[d - 1]) {
        // equal slopes (STD): S(u) = e^{sigma a u} sum_j e^{c_j}, so the threshold is closed-form,
        // u* = (ln(d K) - ln sum_j e^{c_j}) / (sigma a) -- no iteration
        // ... and every final sum factors through S = sum_j e^{c_j}, S_R = sum e^{c_j} R_j and
        // S_t = sum e^{c_j} t_j (E_j = g e^{c_j}, g = e^{sigma a u}; w_j = h e^{c_j}, h = e^{sigma^2 a^2/2};
        // one common Phibar(u - sigma a)): one pass of exponentials for threshold and payoff
        double S = 0.0, SR = 0.0, St = 0.0;
        int j = 0;
#pragma unroll 1
        for (; j + 1 < d; j += 2) {
            const double ca = cb[j * stride], cbb = cb[(j + 1) * stride];
            const double ta = (double)(j + 1) * P.t1, tb = (double)(j + 2) * P.t1;
            double Ea, Eb;
            fast_exp_x2(ca, cbb, Ea, Eb);
            S += Ea;
            SR = fma(Ea, (ca - P.lnS0 - P.omega * ta) * P.inv_sigma, SR);
            St = fma(Ea, ta, St);
            S += Eb;
            SR = fma(Eb, (cbb - P.lnS0 - P.omega * tb) * P.inv_sigma, SR);
            St = fma(Eb, tb, St);
        }
        if (j < d) {
            const double ca = cb[j * stride], ta = (double)(j + 1) * P.t1;
            const double Ea = fast_exp(ca);
            S += Ea;
            SR = fma(Ea, (ca - P.lnS0 - P.omega * ta) * P.inv_sigma, SR);
            St = fma(Ea, ta, St);
        }
        const double a = P.a[0];
        u = fmin((lndK - fast_log(S)) / (sg * a), u_hi);
        double g, h;
        fast_exp_x2(sg * a * u, 0.5 * sg * sg * a * a, g, h);
        double sumW = 0.0, sumWv = 0.0;
        if (arith) {
            double Pf, Q2, p1, p2;
            phibar_phi_x2(u - sg * a, u - sg * a, Pf, Q2, p1, p2);
            sumW = h * Pf * S;
            sumWv = h * Pf * (SR - sg * St + sg * a * a * S);
        }
        return X1Sums{u, a * g * S, a * a * g * S, g * (SR - sg * St + a * u * S), sumW, sumWv};
    } else
    for (int it = 0; it < kNewtonMax; ++it) {
        double S = 0.0, SA = 0.0, SAA = 0.0;
        int j = 0;
#pragma unroll 1
        for (; j + 1 < d; j += 2) {
            const double aa = P.a[j], ab = P.a[j + 1];
            double Ea, Eb;
            fast_exp_x2(fma(sg * aa, u, cb[j * stride]), fma(sg * ab, u, cb[(j + 1) * stride]), Ea, Eb);
            S += Ea;
            SA = fma(aa, Ea, SA);
            SAA = fma(aa * aa, Ea, SAA);
            S += Eb;
            SA = fma(ab, Eb, SA);
            SAA = fma(ab * ab, Eb, SAA);
        }
        if (j < d) {
            const double aj = P.a[j];
            const double E = fast_exp(fma(sg * aj, u, cb[j * stride]));
            S += E;
            SA = fma(aj, E, SA);
            SAA = fma(aj * aj, E, SAA);
        }
        const double du = halley_step(fast_log(S) - lndK, S, SA, SAA, sg);
        conv = fabs(du) <= kHalleyTol * fmax(1.0, fabs(u));
        u = fmin(fmax(u - du, u_lo), u_hi);
        if (it + 1 >= kNewtonIt && __all_sync(__activemask(), conv)) break;
    }
    unconverged += conv ? 0u : 1u;
    double Dst = 0.0, Qst = 0.0, Vst = 0.0, sumW = 0.0, sumWv = 0.0;
    // equal slopes (STD: a_j = sqrt(dt)): Phibar(u - sigma a_j) is one number for every date
    const bool flat = arith && P.a[0] == P.a[d - 1];
    double Pflat = 1.0;
    if (flat) {
        double Q2, p1, p2;
        phibar_phi_x2(u - sg * P.a[0], u - sg * P.a[0], Pflat, Q2, p1, p2);
    }
    // a_j linear in j (STD, BB): w_j = e^{c_j + sigma^2 a_j^2 / 2} = E_j q_j with
    // q_j = e^{kappa_j}, kappa_j = sigma a_j (sigma a_j / 2 - u) quadratic in j, so q_j follows
    // by two products per date (ratio rho_j = q_{j+1}/q_j, rho_{j+1} = rho_j e^{(sigma da)^2})
    const bool lin = arith && P.x1_lin;
    // w_j Phibar(x_j), x_j = u - sigma a_j, without a per-date phi: w_j phi(x_j) = phi(u) E_j, so it
    // is phi(u) E_j R(x_j) for x_j >= 0 and w_j - phi(u) E_j R(-x_j) below (R the Mills ratio)
    double phu = 0.0;
    if (arith && !flat) {
        double Qu_, Q2_, ph2_;
        phibar_phi_x2(u, u, Qu_, Q2_, phu, ph2_);
    }
    double qa = 0.0, rho = 0.0, g = 0.0;
    if (lin) {
        const double a0 = P.a[0], a1 = P.a[1], sda = sg * (a1 - a0);
        const double k0 = sg * a0 * fma(0.5 * sg, a0, -u), k1 = sg * a1 * fma(0.5 * sg, a1, -u);
        fast_exp_x2(k0, k1 - k0, qa, rho);
        g = fast_exp(sda * sda);
    }
#pragma unroll 1
    for (int j = 0; j < d; j += 2) {
        const int jb = (j + 1 < d) ? j + 1 : j;
        const double wgt = (j + 1 < d) ? 1.0 : 0.0;  // odd d: the duplicate pair member counts 0
        const double aa = P.a[j], ab = P.a[jb], ca = cb[j * stride], cbb = cb[jb * stride];
        const double ta = (double)(j + 1) * P.t1, tb = (double)(jb + 1) * P.t1;
        const double Ra = (ca - P.lnS0 - P.omega * ta) * P.inv_sigma, Rb = (cbb - P.lnS0 - P.omega * tb) * P.inv_sigma;
        double Ea, Eb;
        fast_exp_x2(fma(sg * aa, u, ca), fma(sg * ab, u, cbb), Ea, Eb);
        Eb *= wgt;
        Dst = fma(aa, Ea, Dst);
        Qst = fma(aa * aa, Ea, Qst);
        Vst = fma(Ea, Ra - sg * ta + aa * u, Vst);
        Dst = fma(ab, Eb, Dst);
        Qst = fma(ab * ab, Eb, Qst);
        Vst = fma(Eb, Rb - sg * tb + ab * u, Vst);
        if (arith) {
            double wa, wb;
            if (lin) {
                const double qb = qa * rho;
                wa = Ea * qa;
                wb = Eb * qb;
                rho *= g;
                qa = qb * rho;
                rho *= g;
            } else {
                fast_exp_x2(fma(0.5 * sg * sg * aa, aa, ca), fma(0.5 * sg * sg * ab, ab, cbb), wa, wb);
            }
            wb *= wgt;
            double WPa = wa, WPb = wb;  // flat: the common Phibar(u - sigma a) is applied after the loop
            if (!flat) {  // Phi(sigma a - u) = Phibar(u - sigma a)
                const double xa = u - sg * aa, xb = u - sg * ab;
                double Ma, Mb;
                mills_x2(xa, xb, Ma, Mb);
                const double ga = phu * Ea * Ma, gb = phu * Eb * Mb;  // Eb, wb carry the odd-d weight
                WPa = xa >= 0.0 ? ga : wa - ga;
                WPb = xb >= 0.0 ? gb : wb - gb;
            }
            sumW += WPa;
            sumWv = fma(Ra - sg * ta + sg * aa * aa, WPa, sumWv);
            sumW += WPb;
            sumWv = fma(Rb - sg * tb + sg * ab * ab, WPb, sumWv);
        }
    }
    if (flat) {
        sumW *= Pflat;
        sumWv *= Pflat;
    }
    return X1Sums{u, Dst, Qst, Vst, sumW, sumWv};
}

// outputs of option o from the shared sums of its strike
__device__ __forceinline__ void x1_outputs(const PathArgs& P, int o, const X1Sums& x, double f[4]) {
    const double D = P.Dfac, S0 = P.S0, K = P.K[o], dd = (double)P.d, sg = P.sigma, u = x.u;
    const double Dst = x.Dst, Qst = x.Qst, Vst = x.Vst, sumW = x.sumW, sumWv = x.sumWv;
    const bool arith = P.type[o] == kArith;
    double ph, Qu, Q2, ph2;
    phibar_phi_x2(u, u, Qu, Q2, ph, ph2);
    if (arith) {
        f[0] = D * (sumW / dd - K * Qu);
        f[1] = D * sumW / (dd * S0);
        f[2] = D * (sumWv / dd + ph * Dst / dd);
        f[3] = D * dd * K * K * ph / (S0 * S0 * sg * Dst);
    } else {
        const double up = -dd * K / (S0 * sg * Dst);
        f[0] = D * Qu;
        f[1] = D * ph * dd * K / (S0 * sg * Dst);
        f[2] = D * ph * Vst / (sg * Dst);
        f[3] = D * (dd * K / sg) * ph / (S0 * Dst) * (-u * up - 2.0 / S0 - sg * up * Qst / Dst);
    }
}

// Lookback under X1 (next-row f1).  Lines l_j(u) = c_j + b_j u,
// b_j = sigma a_j; u* = min_j (ln K - c_j)/b_j in closed form; G integrates
// exp(max_j l_j(u)) phi(u) over [u*, inf), walking the upper envelope from u*:
// on each segment the next breakpoint is the first steeper line to overtake.
// (Slopes and hull in shared memory measured slower: bank conflicts of the divergent per-lane
// reads, and 9 KB more per block cost the PCA variant an occupancy step.)
__device__ __forceinline__ void x1_lookback(const PathArgs& P, int o, const double* cb, int stride, double f[4]) {
    const int d = P.d;
    const double sg = P.sigma, lnK = P.lnK[o];
    double ustar = CUDART_INF;
    int j0 = 0;
    for (int j = 0; j < d; ++j) {
        const double uj = (lnK - cb[j * stride]) * __ldg(P.inv_sa + j);
        if (uj < ustar) {
            ustar = uj;
            j0 = j;
        }
    }
    // The upper envelope of the lines c_j + b_j u, b_j = sigma a_j, by the monotone
    // convex-hull pass (O(d), no divisions): every construction has a_j nondecreasing in
    // j (STD: equal; BB: t_j/sqrt(T); PCA / GPCA: positive increasing first column), so
    // lines arrive by slope; a line is dropped when the next one overtakes it no later
    // than it overtakes its predecessor.  Equal slopes keep the higher line.  Only u >= u*
    // matters: there line j0 is the highest (c_j + b_j u* <= c_j + b_j u_j = ln K), and a
    // flatter line below it stays below, so the pass starts at j0.
    uint8_t hull[kMaxDimGpu];  // line indices (d <= 256)
    int top = 0;
    if (__ldg(P.a) == __ldg(P.a + d - 1)) {  // STD: all slopes equal -> the single highest line (lowest j on ties)
        int best = 0;
        for (int j = 1; j < d; ++j) best = cb[j * stride] > cb[best * stride] ? j : best;
        hull[0] = (uint8_t)best;
        top = 1;
    } else {
        // the top two hull lines (T = top, S = second) stay in registers; a pop reloads S
        double bT = 0.0, cT = 0.0, bS = 0.0, cS = 0.0;
        for (int j = j0; j < d; ++j) {
            const double b3 = sg * __ldg(P.a + j), c3 = cb[j * stride];
            if (top > 0 && bT == b3) {
                if (c3 <= cT) continue;
                --top;  // same slope, higher line: replaces the top
                bT = bS;
                cT = cS;
                if (top >= 2) {
                    const int l = hull[top - 2];
                    bS = sg * __ldg(P.a + l);
                    cS = cb[l * stride];
                }
            }
            // T is never the maximum iff x(S, new) <= x(S, T), x(p, q) = (c_p - c_q) / (b_q - b_p)
            while (top >= 2 && (cS - c3) * (bT - bS) <= (cS - cT) * (b3 - bS)) {
                --top;
                bT = bS;
                cT = cS;
                if (top >= 2) {
                    const int l = hull[top - 2];
                    bS = sg * __ldg(P.a + l);
                    cS = cb[l * stride];
                }
            }
            QMCCPW_CHECK(top < kMaxDimGpu);
            hull[top++] = (uint8_t)j;
            bS = bT;
            cS = cT;
            bT = b3;
            cT = c3;
        }
    }
    // the envelope segment that contains u*: on a breakpoint tie the steeper line (it
    // dominates just after)
    int k = 0;
    while (k + 1 < top) {
        const int l1 = hull[k], l2 = hull[k + 1];
        const double x = (cb[l1 * stride] - cb[l2 * stride]) / (sg * (__ldg(P.a + l2) - __ldg(P.a + l1)));
        if (x > ustar) break;
        ++k;
    }
    double J = 0.0, V = 0.0, lo = ustar;
    for (; k < top; ++k) {
        const int act = hull[k];
        const double bact = sg * __ldg(P.a + act), cact = cb[act * stride];
        const int nxt = (k + 1 < top) ? hull[k + 1] : -1;
        double hi = CUDART_INF;
        if (nxt >= 0) hi = (cact - cb[nxt * stride]) / (sg * __ldg(P.a + nxt) - bact);
        hi = fmax(hi, lo);
        const double aa = bact / sg;
        const double tj = (double)(act + 1) * P.t1;
        const double Rj = (cact - P.lnS0 - P.omega * tj) * P.inv_sigma;
        const double w = fast_exp(fma(0.5 * bact, bact, cact));
        double Qlo, Qhi, plo, phi_hi;
        phibar_phi_x2(lo - bact, (nxt < 0) ? 0.0 : hi - bact, Qlo, Qhi, plo, phi_hi);
        if (nxt < 0) {
            Qhi = 0.0;
            phi_hi = 0.0;
        }
        J = fma(w, Qlo - Qhi, J);
        V = fma(w, (Rj - sg * tj + sg * aa * aa) * (Qlo - Qhi) + aa * (plo - phi_hi), V);
        lo = hi;
    }
    const double D = P.Dfac, S0 = P.S0, K = P.K[o];
    double Qu, Q2, ph, ph2;
    phibar_phi_x2(ustar, ustar, Qu, Q2, ph, ph2);
    f[0] = D * (J - K * Qu);
    f[1] = D * J / S0;
    f[2] = D * V;
    f[3] = D * K * ph / (S0 * S0 * sg * __ldg(P.a + j0));
}

// sum / min over the four lanes of a quad (lanes 4q .. 4q + 3)
__device__ __forceinline__ double quad_sum(double v) {
    v += __shfl_xor_sync(0xffffffffu, v, 1);
    return v + __shfl_xor_sync(0xffffffffu, v, 2);
}
__device__ __forceinline__ double quad_min(double v) {
    v = fmin(v, __shfl_xor_sync(0xffffffffu, v, 1));
    return fmin(v, __shfl_xor_sync(0xffffffffu, v, 2));
}

// Lookback under X1 over a quad (the PCA kernel's layout: lane r4 holds the path's lines
// j = 8 jt + 2 r4 + e, e = 0, 1, at slot v = 2 jt + e; cq(v, lane_r4) returns c_j of slot v held
// by quad lane lane_r4).  The same envelope integral as x1_lookback, built by gift wrapping
// instead of a per-lane hull: from j0 = argmin_j u_j (the top line at u*), the next segment's
// line is the steeper line that overtakes the active one first, x(act, k) = (c_act - c_k) /
// (b_k - b_act) minimal (ties: the steeper), found by the four lanes over their 16 lines each
// and a quad reduction; division-free comparisons (b_k > b_act).  Slopes strictly increase
// with j for BB, PCA and GPCA; equal slopes (STD) leave the single highest line.
template <int NV, class CQ>
__device__ __forceinline__ void x1_lookback_quad(const PathArgs& P, int o, int r4, CQ cq, double f[4]) {
    const int d = P.d;
    const double sg = P.sigma, lnK = P.lnK[o];
    // u* and j0 (lowest j among the minima)
    double ust = CUDART_INF;
    int j0 = 0x7fffffff;
#pragma unroll 1
    for (int v = 0; v < NV; ++v) {
        const int j = 8 * (v >> 1) + 2 * r4 + (v & 1);
        if (j < d) {
            const double uj = (lnK - cq(v, r4)) * __ldg(P.inv_sa + j);
            if (uj < ust || (uj == ust && j < j0)) {
                ust = uj;
                j0 = j;
            }
        }
    }
#pragma unroll
    for (int off = 1; off <= 2; off <<= 1) {
        const double pu = __shfl_xor_sync(0xffffffffu, ust, off);
        const int pj = __shfl_xor_sync(0xffffffffu, j0, off);
        if (pu < ust || (pu == ust && pj < j0)) {
            ust = pu;
            j0 = pj;
        }
    }
    auto cj = [&](int j) { return cq(2 * (j >> 3) + (j & 1), (j & 7) >> 1); };
    double J = 0.0, V = 0.0;
    int act = j0;
    double lo = ust;
    const bool flat = __ldg(P.a) == __ldg(P.a + d - 1);
    if (flat) {  // STD: all slopes equal -> the single highest line (lowest j on ties), from u*
        double cb = -CUDART_INF;
        int jb = 0x7fffffff;
#pragma unroll 1
        for (int v = 0; v < NV; ++v) {
            const int j = 8 * (v >> 1) + 2 * r4 + (v & 1);
            if (j < d) {
                const double c = cq(v, r4);
                if (c > cb || (c == cb && j < jb)) {
                    cb = c;
                    jb = j;
                }
            }
        }
#pragma unroll
        for (int off = 1; off <= 2; off <<= 1) {
            const double pc = __shfl_xor_sync(0xffffffffu, cb, off);
            const int pj = __shfl_xor_sync(0xffffffffu, jb, off);
            if (pc > cb || (pc == cb && pj < jb)) {
                cb = pc;
                jb = pj;
            }
        }
        act = jb;
    }
    // the quads of a warp finish after different segment counts, and the loop shuffles with a
    // full mask: it runs until every quad is done (warp-uniform exit), finished quads idle
    // the quads of a warp finish after different segment counts, and the loop shuffles with a
    // full mask: it runs until every quad is done (warp-uniform exit), finished quads idle.
    // (Dealing the segment integrals round-robin over the quad measured slower: 192.4 -> 198.1
    // ms for C4 PCA-X1 with the lookback, register pressure.)
    bool done = false;
#pragma unroll 1
    for (;;) {
        if (!__any_sync(0xffffffffu, !done)) break;
        const double ca = cj(act), ba = sg * __ldg(P.a + act);
        // my best overtaking line: smallest x = N / D (D > 0), ties to the larger j
        double Nb = 0.0, Db = 0.0;
        int kb = -1;
        if (!flat) {
            // my lines are j(v) = 8 (v >> 1) + 2 r4 + (v & 1), increasing in v: start at the first
            // one beyond act (act only grows, so the scans shrink along the walk)
            const int rel = act + 1 - 2 * r4;  // smallest j - 2 r4 wanted
            int v = rel <= 0 ? 0 : 2 * (rel >> 3) + ((rel & 7) == 0 ? 0 : ((rel & 7) == 1 ? 1 : 2));
#pragma unroll 1
            for (; v < NV; ++v) {
                const int j = 8 * (v >> 1) + 2 * r4 + (v & 1);
                if (j > act && j < d) {
                    const double D = sg * __ldg(P.a + j) - ba;
                    if (D > 0.0) {
                        const double N = ca - cq(v, r4);
                        const double lhs = N * Db, rhs = Nb * D;
                        if (kb < 0 || lhs < rhs || (lhs == rhs && j > kb)) {
                            Nb = N;
                            Db = D;
                            kb = j;
                        }
                    }
                }
            }
        }
#pragma unroll
        for (int off = 1; off <= 2; off <<= 1) {
            const double pN = __shfl_xor_sync(0xffffffffu, Nb, off);
            const double pD = __shfl_xor_sync(0xffffffffu, Db, off);
            const int pk = __shfl_xor_sync(0xffffffffu, kb, off);
            if (pk >= 0) {
                const double lhs = pN * Db, rhs = Nb * pD;
                if (kb < 0 || lhs < rhs || (lhs == rhs && pk > kb)) {
                    Nb = pN;
                    Db = pD;
                    kb = pk;
                }
            }
        }
        if (done) continue;
        double hi = kb >= 0 ? Nb / Db : CUDART_INF;
        hi = fmax(hi, lo);
        const double aa = ba / sg;
        const double tj = (double)(act + 1) * P.t1;
        const double Rj = (ca - P.lnS0 - P.omega * tj) * P.inv_sigma;
        const double w = fast_exp(fma(0.5 * ba, ba, ca));
        double Qlo, Qhi, plo, phi_hi;
        phibar_phi_x2(lo - ba, (kb < 0) ? 0.0 : hi - ba, Qlo, Qhi, plo, phi_hi);
        if (kb < 0) {
            Qhi = 0.0;
            phi_hi = 0.0;
        }
        J = fma(w, Qlo - Qhi, J);
        V = fma(w, (Rj - sg * tj + sg * aa * aa) * (Qlo - Qhi) + aa * (plo - phi_hi), V);
        if (kb < 0) {
            done = true;
        } else {
            act = kb;
            lo = hi;
        }
    }
    const double D = P.Dfac, S0 = P.S0, K = P.K[o];
    double Qu, Q2, ph, ph2;
    phibar_phi_x2(ust, ust, Qu, Q2, ph, ph2);
    f[0] = D * (J - K * Qu);
    f[1] = D * J / S0;
    f[2] = D * V;
    f[3] = D * K * ph / (S0 * S0 * sg * __ldg(P.a + j0));
}

// STD-X1 streamed (equal slopes a_j = a): every strike's threshold, the arithmetic / binary sums
// and the lookback's single top line follow from S = sum e^{c_j}, S_R = sum e^{c_j} R_j,
// S_t = sum e^{c_j} t_j and the highest c_j (lowest j on ties), all accumulated while the path is
// generated -- no per-date storage (the one-pass algebra of x1_solve's equal-slope branch; the
// lookback's envelope is the single top line, x1_lookback's equal-slope branch)
struct X1Stream {
    double S, SR, St, cmax;
    int jmax;
    __device__ __forceinline__ void reset() {
        S = 0.0; SR = 0.0; St = 0.0; cmax = -CUDART_INF; jmax = 0;
    }
    // date j (0-based): c = c_j, t = t_j = (j + 1) t_1, E = e^{c_j}
    __device__ __forceinline__ void push(const PathArgs& P, int j, double c, double t, double E) {
        S += E;
        SR = fma(E, (c - P.lnS0 - P.omega * t) * P.inv_sigma, SR);
        St = fma(E, t, St);
        if (c > cmax) {
            cmax = c;
            jmax = j;
        }
    }
};
__device__ __forceinline__ void tail_x1_stream(const PathArgs& P, const X1Stream& st, double f[kMaxOpt][4]) {
    const double sg = P.sigma, a = __ldg(P.a), isa = __ldg(P.inv_sa);
    const double lnS = fast_log(st.S);
    double h, hd;
    fast_exp_x2(0.5 * sg * sg * a * a, 0.0, h, hd);
#pragma unroll 1
    for (int o = 0; o < P.n_opt; ++o) {
        if (P.type[o] == kLookback) {
            // envelope = line jmax from u* = (ln K - c_max) / (sigma a) on
            const double ustar = (P.lnK[o] - st.cmax) * isa;
            const double bact = sg * a, cact = st.cmax, aa = bact / sg;
            const double tj = (double)(st.jmax + 1) * P.t1;
            const double Rj = (cact - P.lnS0 - P.omega * tj) * P.inv_sigma;
            const double w = fast_exp(fma(0.5 * bact, bact, cact));
            double Qlo, Qhi, plo, phi_hi;
            phibar_phi_x2(ustar - bact, 0.0, Qlo, Qhi, plo, phi_hi);
            const double J = w * Qlo;
            const double V = w * ((Rj - sg * tj + sg * aa * aa) * Qlo + aa * plo);
            const double D = P.Dfac, S0 = P.S0, K = P.K[o];
            double Qu, Q2, ph, ph2;
            phibar_phi_x2(ustar, ustar, Qu, Q2, ph, ph2);
            double fl[4] = {D * (J - K * Qu), D * J / S0, D * V, D * K * ph / (S0 * S0 * sg * a)};
#pragma unroll
            for (int o3 = 0; o3 < kMaxOpt; ++o3)
                if (o3 == o)
#pragma unroll
                    for (int qq = 0; qq < 4; ++qq) f[o3][qq] = fl[qq];
            continue;
        }
        if (P.tail_leader[o] != o) continue;
        const double u_hi = (P.lndK[o] - st.cmax) * isa;
        const double u = fmin((P.lndK[o] - lnS) / (sg * a), u_hi);
        const double g = fast_exp(sg * a * u);
        double sumW = 0.0, sumWv = 0.0;
        if (P.x1_need_arith[o]) {
            double Pf, Q2, p1, p2;
            phibar_phi_x2(u - sg * a, u - sg * a, Pf, Q2, p1, p2);
            sumW = h * Pf * st.S;
            sumWv = h * Pf * (st.SR - sg * st.St + sg * a * a * st.S);
        }
        const X1Sums xs{u, a * g * st.S, a * a * g * st.S, g * (st.SR - sg * st.St + a * u * st.S), sumW, sumWv};
#pragma unroll
        for (int o2 = 0; o2 < kMaxOpt; ++o2)
            if (o2 < P.n_opt && P.tail_leader[o2] == o) x1_outputs(P, o2, xs, f[o2]);
    }
}

// all options of the launch: one Newton solve (and one set of E*-sums) per distinct strike
__device__ __forceinline__ void tail_x1_all(const PathArgs& P, const double* cb, int stride, double f[kMaxOpt][4],
                                            unsigned& unconverged) {
    X1Sums xs[kMaxOpt];
#pragma unroll
    for (int o = 0; o < kMaxOpt; ++o) {
        if (o >= P.n_opt) break;
        if (P.type[o] == kLookback) {
            x1_lookback(P, o, cb, stride, f[o]);
            xs[o] = X1Sums{0, 0, 0, 0, 0, 0};
            continue;
        }
        const int ld = P.tail_leader[o];
        if (ld == o) {
            xs[o] = x1_solve(P, o, P.x1_need_arith[o] != 0, cb, stride, unconverged);
        } else {
            xs[o] = ld == 0 ? xs[0] : xs[1];
        }
        x1_outputs(P, o, xs[o], f[o]);
    }
}

// (a9) LR+MC: Philox normals (counter (k_lo, k_hi, j/4, (rep<<8)|0x02)),
// STD path of full prices, payoff x score.
__device__ __forceinline__ void lr_path(const PathArgs& P, uint32_t rep, uint64_t k, double f[kMaxOpt][4]) {
    const int d = P.d;
    double W = 0.0, sumS = 0.0, Smax = 0.0, vscore = 0.0, Z1 = 0.0;
    for (int jq = 0; jq < d; jq += 4) {
        uint32_t c[4] = {(uint32_t)k, (uint32_t)(k >> 32), (uint32_t)(jq >> 2), (rep << 8) | 0x02u};
        philox4x32_10(c, (uint32_t)P.seed, (uint32_t)(P.seed >> 32));
        double xs[4];
        normal_from_u32_x2(c[0], c[1], xs[0], xs[1]);
        if (jq + 2 < d) normal_from_u32_x2(c[2], c[3], xs[2], xs[3]);
#pragma unroll
        for (int w = 0; w < 4; ++w) {
            const int j = jq + w;
            if (j < d) {
                const double x = xs[w];
                if (j == 0) Z1 = x;
                W = fma(P.sqrt_t1, x, W);
                const double S = P.S0 * fast_exp(fma(P.sigma, W, P.omega * (double)(j + 1) * P.t1));
                sumS += S;
                Smax = fmax(Smax, S);
                vscore += (x * x - 1.0) * P.inv_sigma - x * P.sqrt_t1;
            }
        }
    }
    const double SA = sumS / d, S0 = P.S0, sg = P.sigma, t1 = P.t1;
    const double sd = Z1 / (S0 * sg * P.sqrt_t1);
    const double sgm = (Z1 * Z1 - 1.0) / (S0 * S0 * sg * sg * t1) - Z1 / (S0 * S0 * sg * P.sqrt_t1);
#pragma unroll
    for (int o = 0; o < kMaxOpt; ++o) {
        if (o >= P.n_opt) break;
        double pay;
        if (P.type[o] == kArith) pay = P.Dfac * fmax(SA - P.K[o], 0.0);
        else if (P.type[o] == kBinary) pay = (SA > P.K[o]) ? P.Dfac : 0.0;
        else pay = P.Dfac * fmax(Smax - P.K[o], 0.0);
        f[o][0] = pay;
        f[o][1] = pay * sd;
        f[o][2] = pay * vscore;
        f[o][3] = pay * sgm;
    }
}

// ---------------------------------------------------------------------------
// The fused path kernel: one block = one cell (replicate, 4096 points).
// ---------------------------------------------------------------------------
// (a8) per-iteration warp reduction of the centred sums of option o (8 slots: S1, S2
// per Greek, slot 2q + {0,1}, the partials layout): a reduce-scatter that halves
// the slot set at xor 16, 8, 4 (each lane sends the half it drops), then a butterfly
// over xor 2, 1; lanes 4s..4s+3 end with the warp total of slot s = lane >> 2, and
// lane 4s adds it to the warp's running sums wacc[o*8 + s] in shared memory (no
// per-thread accumulators, nothing live in registers across paths).
__device__ __forceinline__ void warp_slot_sums_one(const double (&f4)[4], const double (&piv)[4], bool valid, int lane,
                                                   double* wacc8) {
    double v[8];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        const double y = valid ? f4[q] - piv[q] : 0.0;
        v[2 * q] = y;
        v[2 * q + 1] = y * y;
    }
#pragma unroll
    for (int half = 4; half > 0; half >>= 1) {
        const bool up = (lane & (half * 4)) != 0;
#pragma unroll
        for (int j = 0; j < half; ++j) {
            const double send = up ? v[j] : v[j + half];
            const double keep = up ? v[j + half] : v[j];
            v[j] = keep + __shfl_xor_sync(0xffffffffu, send, half * 4);
        }
    }
    v[0] += __shfl_xor_sync(0xffffffffu, v[0], 2);
    v[0] += __shfl_xor_sync(0xffffffffu, v[0], 1);
    if ((lane & 3) == 0) wacc8[lane >> 2] += v[0];
}
// skip_lookback: leave the lookback options' slots alone (their values arrive separately)
__device__ __forceinline__ void warp_slot_sums(const double (&f)[kMaxOpt][4], const PathArgs& P, bool valid,
                                               int lane, double* wacc, bool skip_lookback = false) {
#pragma unroll
    for (int o = 0; o < kMaxOpt; ++o) {
        if (o >= P.n_opt) break;  // warp-uniform
        if (skip_lookback && P.type[o] == kLookback) continue;
        QMCCPW_CHECK(o * 8 + 7 < 32);
        warp_slot_sums_one(f[o], P.piv[o], valid, lane, wacc + o * 8);
    }
}

// the W1 tail reduced on the fly: option o's values go straight into the warp's slot sums
// (and to the per-path hook), so no [option][Greek] array is held (it was kept in local
// memory by the path kernels: 85 local loads/stores per path in BB-W1)
__device__ __forceinline__ void tail_w1_reduce(const PathArgs& P, const W1Acc& acc, bool valid, int lane,
                                               double* wacc, uint64_t i) {
    tail_w1_each(P, acc, [&](int o, const double (&f4)[4]) {
        if (P.path_out != nullptr && valid && o == P.hook_option)
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                QMCCPW_CHECK(i < P.n_points);
                P.path_out[i * 4 + q] = f4[q];
            }
        warp_slot_sums_one(f4, P.piv[o], valid, lane, wacc + o * 8);
    });
}

// per-thread (S1, S2) double2 accumulators in smem: cheaper in issue slots than the warp
// reduction, so kernels with smem to spare (pca_kernel, register-limited) use it; the
// path kernel, at its smem limit, uses warp_slot_sums (measured: BB-W1 -8%, PCA-W1 +4%)
__device__ __forceinline__ void thread_acc2(const double (&f)[kMaxOpt][4], const PathArgs& P, bool valid,
                                            double2* acc2, int tpb, int tid) {
    if (!valid) return;
#pragma unroll
    for (int o = 0; o < kMaxOpt; ++o) {
        if (o >= P.n_opt) break;
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const double y = f[o][q] - P.piv[o][q];
            double2* a = acc2 + (size_t)(o * 4 + q) * tpb + tid;
            QMCCPW_CHK_SMEM(a);
            double2 t = *a;
            t.x += y;
            t.y = fma(y, y, t.y);
            *a = t;
        }
    }
}
__device__ __forceinline__ void acc2_to_wacc(const PathArgs& P, const double2* acc2, double* wacc, int tpb, int tid) {
    const int lane = tid & 31;
    for (int v = 0; v < P.n_opt * 8; ++v) {
        const double2 t = acc2[(size_t)(v >> 1) * tpb + tid];
        double s1 = (v & 1) ? t.y : t.x;
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) s1 += __shfl_xor_sync(0xffffffffu, s1, off);
        if (lane == 0) wacc[(tid >> 5) * 32 + v] = s1;
    }
}

// (a8) fixed-shape reduction of a block's accumulators into its cell's partials:
// warp butterfly, then the warps in order (deterministic for a given block size).
__device__ __forceinline__ void block_epilogue(const PathArgs& P, const double* accs, const double* wacc, double* red,
                                               int n_acc, int tpb, int tid, uint64_t cell, unsigned unconverged,
                                               unsigned ties, unsigned npts) {
    const int lane = tid & 31, warp = tid >> 5, nwarps = tpb >> 5;
    const int n_out = P.partial_stride;
    __syncthreads();  // red aliases the Sobol' tables
    if (accs == nullptr) {  // per-warp sums (warp_slot_sums)
        QMCCPW_CHECK(n_acc + 3 <= 32 && warp < 4);
        if (lane < n_acc) red[warp * 32 + lane] = wacc[warp * 32 + lane];
    } else {
        for (int v = 0; v < n_acc; ++v) {
            double s1 = accs[v * tpb + tid];
#pragma unroll
            for (int off = 16; off > 0; off >>= 1) s1 += __shfl_xor_sync(0xffffffffu, s1, off);
            if (lane == 0) red[warp * 32 + v] = s1;
        }
    }
    unsigned uc = unconverged, tc = ties, nc = npts;
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
        uc += __shfl_xor_sync(0xffffffffu, uc, off);
        tc += __shfl_xor_sync(0xffffffffu, tc, off);
        nc += __shfl_xor_sync(0xffffffffu, nc, off);
    }
    if (lane == 0) {
        QMCCPW_CHK_SMEM(&red[warp * 32 + P.n_opt * 8 + 2]);
        red[warp * 32 + P.n_opt * 8 + 0] = (double)uc;
        red[warp * 32 + P.n_opt * 8 + 1] = (double)tc;
        red[warp * 32 + P.n_opt * 8 + 2] = (double)nc;  // points this cell evaluated (completeness check)
    }
    __syncthreads();
    if (tid < n_out) {
        double s = 0.0;
        for (int w = 0; w < nwarps; ++w) s += red[w * 32 + tid];
        QMCCPW_CHECK(cell >= P.cell_begin && cell < P.cell_end);
        P.partials[(size_t)cell * n_out + tid] = s;
    }
}


}  // namespace qmccpw
