// qmccpw_kernels.cu -- sm_100a kernels of the QMC-CPW hot path (arXiv 2209.11337).
//
// One thread carries one path at a time through the whole pipeline in FP64
// ("each thread will be responsible for the simulation of one
// path"), but nothing is materialised in HBM: Sobol' integers live in
// per-thread shared-memory state advanced by the Gray-code stride rule, the
// normals are consumed as they are produced, the Brownian bridge is generated
// in time order from a log2(d)-deep stack, and each block reduces its cell of
// 4096 points to one row of partial sums.  The paper instead materialises
// normals and the bridge in global memory and names that round trip as its
// 4x slowdown.
//
// Device code here is independent of oracle/: it is written from the paper
// and SURVEY.md Sec. 8(a); tests compare the two on the same points.

#include <cuda_runtime.h>
#include <math_constants.h>
#include <stdint.h>

#include "qmccpw_internal.h"
#include "qmccpw_math.cuh"

namespace qmccpw {

uint64_t& launch_counter() {
    static thread_local uint64_t n = 0;
    return n;
}

// ---------------------------------------------------------------------------
// (a1) randomisation tables on the device: per (replicate, dimension) a
// Matousek left-matrix scramble L (unit lower-triangular in MSB-first digit
// order) and a digital shift, both from Philox4x32-10 keyed by the seed with
// counter (j, w, 0, (rep<<8)|0x01).  v'_b = L v_b is formed column-wise:
// v' = XOR over the set digits t of v of column t of L.
// ---------------------------------------------------------------------------
__global__ void randomization_kernel(const uint32_t* __restrict__ base_v, const uint32_t* __restrict__ base_shift,
                                     int d, uint32_t n_reps, uint32_t rep_base, uint32_t key0, uint32_t key1, int mode,
                                     uint32_t* __restrict__ vscr, uint32_t* __restrict__ shift) {
    const uint64_t gid = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const uint64_t total = (uint64_t)n_reps * d * 32;
    if (gid >= total) return;
    const int b = (int)(gid & 31);
    const uint64_t rj = gid >> 5;
    const int j = (int)(rj % d);
    const uint32_t rep = rep_base + (uint32_t)(rj / d);
    const uint32_t v = base_v[j * 32 + b];
    if (mode == 2) {  // tables used as given (cuRAND-compatible / plain)
        vscr[gid] = v;
        if (b == 0) shift[rj] = base_shift[j];
        return;
    }
    uint32_t w[32];
#pragma unroll
    for (uint32_t blk = 0; blk < 8; ++blk) {
        uint32_t c[4] = {(uint32_t)j, blk, 0u, (rep << 8) | 0x01u};
        philox4x32_10(c, key0, key1);
        w[4 * blk + 0] = c[0];
        w[4 * blk + 1] = c[1];
        w[4 * blk + 2] = c[2];
        w[4 * blk + 3] = c[3];
    }
    if (b == 0) shift[rj] = w[0];  // modes 0, 1: digital shift; mode 3 (Owen): the dimension's scramble seed
    if (mode == 1 || mode == 3) {  // shift only / Owen: plain direction numbers
        vscr[gid] = v;
        return;
    }
    uint32_t out = 0;
    for (int t = 0; t < 32; ++t) {           // digit t <-> bit 31-t
        if (!((v >> (31 - t)) & 1u)) continue;
        uint32_t col = 1u << (31 - t);       // unit diagonal
        for (int i = t + 1; i < 32; ++i)     // row i has random digits 0..i-1 (bits 31..32-i)
            col |= ((w[i] >> (31 - t)) & 1u) << (31 - i);
        out ^= col;
    }
    vscr[gid] = out;
}

cudaError_t launch_randomization(const uint32_t* d_base_v, const uint32_t* d_base_shift, int d, uint32_t n_reps,
                                 uint32_t rep_base, uint64_t seed, int mode, uint32_t* d_vscr, uint32_t* d_shift,
                                 cudaStream_t st) {
    const uint64_t total = (uint64_t)n_reps * d * 32;
    const int tpb = 256;
    const unsigned grid = (unsigned)((total + tpb - 1) / tpb);
    randomization_kernel<<<grid, tpb, 0, st>>>(d_base_v, d_base_shift, d, n_reps, rep_base, (uint32_t)seed,
                                               (uint32_t)(seed >> 32), mode, d_vscr, d_shift);
    ++launch_counter();
    return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// (a1) path-matrix tables.  PCA of C = [min(t_i,t_j)] in closed form:
// theta_k = (2k-1) pi/(2d+1), lambda_k = dt/(4 sin^2(theta_k/2)),
// M_jk = sqrt(lambda_k) sqrt(4/(2d+1)) sin(j theta_k) (1-based), evaluated
// with sinpi on exactly reduced rational arguments.  a_j = M_j1 for every
// construction (STD: sqrt(dt); BB: t_j/sqrt(T)).
// ---------------------------------------------------------------------------
__global__ void path_matrix_kernel(int construction, int d, int ld, double T, double sigma, double* __restrict__ M,
                                   double* __restrict__ a, double* __restrict__ inv_sa) {
    const int idx = blockIdx.x * blockDim.x + threadIdx.x;
    const double dt = T / d;
    const long long den = 2LL * d + 1;
    if (construction == kPca && M != nullptr && idx < ld * ld && (idx / ld >= d || idx % ld >= d)) {
        M[idx] = 0.0;  // zero padding to the mma tile multiple
    } else if (construction == kPca && M != nullptr && idx < ld * ld) {
        const int j = idx / ld + 1, k = idx % ld + 1;
        const double sh = sinpi((double)(2 * k - 1) / (double)(2 * den));        // sin(theta_k / 2)
        const long long num = ((long long)j * (2 * k - 1)) % (2 * den);           // j theta_k / pi mod 2
        const double s = sinpi((double)num / (double)den);
        M[idx] = sqrt(dt / (4.0 * sh * sh)) * sqrt(4.0 / (double)den) * s;
    }
    if (idx < d) {
        const int j = idx + 1;
        double aj;
        if (construction == kStd) {
            aj = sqrt(dt);
        } else if (construction == kBB) {
            aj = (double)j * dt / sqrt(T);
        } else {
            const double sh = sinpi(1.0 / (double)(2 * den));
            const long long num = (long long)j % (2 * den);
            aj = sqrt(dt / (4.0 * sh * sh)) * sqrt(4.0 / (double)den) * sinpi((double)num / (double)den);
        }
        a[idx] = aj;
        inv_sa[idx] = 1.0 / (sigma * aj);
    }
}

cudaError_t launch_path_matrix(int construction, int d, int ld, double T, double sigma, double* d_M, double* d_a,
                               double* d_inv_sa, cudaStream_t st) {
    const int n = (construction == kPca && d_M) ? (ld * ld > d ? ld * ld : d) : d;
    const int tpb = 256;
    path_matrix_kernel<<<(n + tpb - 1) / tpb, tpb, 0, st>>>(construction, d, ld, T, sigma, d_M, d_a, d_inv_sa);
    ++launch_counter();
    return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// (a1, row f3) GPCA: rotate the PCA matrix in place, M <- M H, by the Householder
// reflection H = I - 2 v v^T / (v^T v), v = e_1 - q, q = M^T s / |M^T s|, s_j =
// exp(omega t_j) (the arithmetic average's gradient at W = 0): H e_1 = q, so the
// new first column is C s / sqrt(s^T C s) and M^T s is parallel to e_1.  One
// block; then a_j = M_j1 and 1/(sigma a_j) for X1.  Runs once per call.
// ---------------------------------------------------------------------------
__global__ void gpca_rotate_kernel(double* __restrict__ M, int ld, int d, double dt, double omega, double sigma,
                                   double* __restrict__ a, double* __restrict__ inv_sa) {
    extern __shared__ double gsm[];
    double* sv = gsm;       // s_j, then v_k
    double* u = gsm + d;    // (M^T s)_k, then (M v)_j
    __shared__ double red[32];
    const int tid = threadIdx.x, nt = blockDim.x;
    for (int j = tid; j < d; j += nt) sv[j] = exp(omega * (double)(j + 1) * dt);
    __syncthreads();
    for (int k = tid; k < d; k += nt) {
        double w = 0.0;
        for (int j = 0; j < d; ++j) w = fma(M[(size_t)j * ld + k], sv[j], w);
        u[k] = w;
    }
    __syncthreads();
    auto block_sum = [&](double x) {  // deterministic: warp butterflies, then warps in order
        for (int off = 16; off > 0; off >>= 1) x += __shfl_xor_sync(0xffffffffu, x, off);
        if ((tid & 31) == 0) red[tid >> 5] = x;
        __syncthreads();
        double t = 0.0;
        for (int w = 0; w < (nt + 31) / 32; ++w) t += red[w];
        __syncthreads();
        return t;
    };
    double part = 0.0;
    for (int k = tid; k < d; k += nt) part = fma(u[k], u[k], part);
    const double norm = sqrt(block_sum(part));
    part = 0.0;
    for (int k = tid; k < d; k += nt) {
        const double vk = (k == 0 ? 1.0 : 0.0) - u[k] / norm;
        sv[k] = vk;
        part = fma(vk, vk, part);
    }
    const double vv = block_sum(part);  // its barriers also publish sv
    if (vv > 0.0) {
        for (int j = tid; j < d; j += nt) {
            double w = 0.0;
            for (int k = 0; k < d; ++k) w = fma(M[(size_t)j * ld + k], sv[k], w);
            u[j] = w;
        }
        __syncthreads();
        const double c = 2.0 / vv;
        for (int idx = tid; idx < d * d; idx += nt) {
            const int j = idx / d, k = idx % d;
            M[(size_t)j * ld + k] -= c * u[j] * sv[k];
        }
        __syncthreads();
    }
    for (int j = tid; j < d; j += nt) {
        const double aj = M[(size_t)j * ld];
        a[j] = aj;
        inv_sa[j] = 1.0 / (sigma * aj);
    }
}

cudaError_t launch_gpca_rotate(double* d_M, int ld, int d, double T, double omega, double sigma, double* d_a,
                               double* d_inv_sa, cudaStream_t st) {
    gpca_rotate_kernel<<<1, 256, (size_t)2 * d * sizeof(double), st>>>(d_M, ld, d, T / d, omega, sigma, d_a, d_inv_sa);
    ++launch_counter();
    return cudaGetLastError();
}

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
        G[idx] = y;
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
// MC-CPW / MC+AV-CPW / LR+MC normals: Philox4x32-10, counter (k_lo, k_hi, j/4,
// (rep<<8)|0x02), word j%4 (the paper's PSEUDO generator).
__device__ __forceinline__ uint32_t pick4(const uint32_t c[4], int w) {
    return w == 0 ? c[0] : (w == 1 ? c[1] : (w == 2 ? c[2] : c[3]));
}
__device__ __forceinline__ void mc_normal_pair(const PathArgs& P, uint32_t rep, uint64_t k, int ja, int jb, double& xa,
                                               double& xb) {
    uint32_t ca[4] = {(uint32_t)k, (uint32_t)(k >> 32), (uint32_t)(ja >> 2), (rep << 8) | 0x02u};
    philox4x32_10(ca, (uint32_t)P.seed, (uint32_t)(P.seed >> 32));
    const uint32_t ya = pick4(ca, ja & 3);
    uint32_t yb;
    if ((jb >> 2) == (ja >> 2)) {
        yb = pick4(ca, jb & 3);
    } else {
        uint32_t cb[4] = {(uint32_t)k, (uint32_t)(k >> 32), (uint32_t)(jb >> 2), (rep << 8) | 0x02u};
        philox4x32_10(cb, (uint32_t)P.seed, (uint32_t)(P.seed >> 32));
        yb = pick4(cb, jb & 3);
    }
    normal_from_u32_x2(ya, yb, xa, xb);
}

struct W1Acc {
    double sumS, sumI, emax, esec, ymax;
    __device__ __forceinline__ void reset() {
        sumS = 0.0; sumI = 0.0; emax = -CUDART_INF; esec = -CUDART_INF; ymax = 0.0;
    }
    // lookback: lowest argmax of e_j (= argmax of S~_j) and the runner-up exponent,
    // with plain compare-selects (no NaN-aware fmax/fmin: e is always finite)
    __device__ __forceinline__ void track(double e, double y) {
        const bool gt = e > emax;
        const double cand = gt ? emax : e;
        esec = cand > esec ? cand : esec;
        ymax = gt ? y : ymax;
        emax = gt ? e : emax;
    }
    // date index j (0-based, t_{j+1} - t_1 = j dt), Wt = W~(t_{j+1} - t_1)
    __device__ __forceinline__ void push(const PathArgs& P, int j, double Wt) {
        const double tt = (double)j * P.t1;
        const double e = fma(P.sigma, Wt, P.omega * tt);
        const double St = P.S0 * fast_exp(e);
        const double y = fma(-P.sigma, tt, Wt);
        sumS += St;
        sumI = fma(St, y, sumI);
        if (P.has_lookback) track(e, y);
    }
    // dates j and j+1 together (paired exp)
    __device__ __forceinline__ void push2(const PathArgs& P, int j, double Wa, double Wb) {
        const double ta = (double)j * P.t1, tb = ta + P.t1;
        const double ea = fma(P.sigma, Wa, P.omega * ta), eb = fma(P.sigma, Wb, P.omega * tb);
        double Xa, Xb;
        fast_exp_x2(ea, eb, Xa, Xb);
        const double Sa = P.S0 * Xa, Sb = P.S0 * Xb;
        const double ya = fma(-P.sigma, ta, Wa), yb = fma(-P.sigma, tb, Wb);
        sumS += Sa;
        sumI = fma(Sa, ya, sumI);
        sumS += Sb;
        sumI = fma(Sb, yb, sumI);
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
            normal_from_u32_x2(sob.get(dim_at(0)), sob.get(dim_at(1)), x0, x1);
            have = 2;
        }
        const double r = (have == 2) ? x0 : x1;
        --have;
        return r;
    }
    // same, with an arbitrary pair drawer draw(dim_a, dim_b, x_a, x_b)
    template <class Draw, class DimAt>
    __device__ __forceinline__ double next_from(Draw draw, DimAt dim_at) {
        if (have == 0) {
            draw(dim_at(0), dim_at(1), x0, x1);
            have = 2;
        }
        const double r = (have == 2) ? x0 : x1;
        --have;
        return r;
    }
};

// (a6)+(a7) W1 threshold psi_d and the closed-form smoothed
// payoff and Greeks (readings 1-5), all options of the
// launch at once.  Options with the same strike and statistic (the arithmetic
// and binary Asians of C4) share psi, phi(psi), Phibar(psi), Phibar(psi - s):
// P.tail_leader[o] names the first such option.
__device__ __forceinline__ void tail_w1_all(const PathArgs& P, const W1Acc& acc, double f[kMaxOpt][4]) {
    const double inv_d = 1.0 / (double)P.d;
    const double SA = acc.sumS * inv_d, IA = acc.sumI * inv_d;
    const double Smax = P.has_lookback ? acc.smax(P) : SA;
    const double Imax = Smax * acc.ymax;
    double lnSA, lnSmax;
    fast_log_x2(SA, Smax, lnSA, lnSmax);
    double psi[kMaxOpt], Q0[kMaxOpt], Q1[kMaxOpt], ph[kMaxOpt];
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
            // leader index ld < o, resolved with selects (no dynamic register indexing)
            psi[o] = ld == 0 ? psi[0] : psi[ld == 1 ? 1 : 0];
            Q0[o] = ld == 0 ? Q0[0] : Q0[ld == 1 ? 1 : 0];
            Q1[o] = ld == 0 ? Q1[0] : Q1[ld == 1 ? 1 : 0];
            ph[o] = ld == 0 ? ph[0] : ph[ld == 1 ? 1 : 0];
        }
        const double stat = lb ? Smax : SA;
        const double I = lb ? Imax : IA;
        const double K = P.K[o], D = P.Dfac, S0 = P.S0;
        if (P.type[o] == kBinary) {
            f[o][0] = D * Q0[o];
            f[o][1] = D * ph[o] * P.inv_s / S0;
            f[o][2] = D * ph[o] * (I * P.inv_s / stat + psi[o] * P.inv_sigma - P.sqrt_t1);
            f[o][3] = D * ph[o] * P.inv_s / (S0 * S0) * (psi[o] * P.inv_s - 1.0);
        } else {
            f[o][0] = P.Afac * stat * Q1[o] - D * K * Q0[o];
            f[o][1] = P.Afac * (stat / S0) * Q1[o];
            f[o][2] = P.Afac * Q1[o] * I + K * D * ph[o] * P.sqrt_t1;
            f[o][3] = K * D * ph[o] * P.inv_s / (S0 * S0);
        }
    }
}

// (a6)+(a7) X1 mode: u* solves sum_j exp(c_j + sigma a_j u) = dK
// by Newton from the AM-GM start, warp-uniform iteration count, clamped to the
// bracket; then the conditional payoff and Greeks.  cb = per-thread c_j column.
struct X1Sums {
    double u, Dst, Qst, Vst, sumW, sumWv;
};

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
    for (int it = 0; it < kNewtonMax; ++it) {
        double S = 0.0, SA = 0.0;
        int j = 0;
#pragma unroll 1
        for (; j + 1 < d; j += 2) {
            const double aa = P.a[j], ab = P.a[j + 1];
            double Ea, Eb;
            fast_exp_x2(fma(sg * aa, u, cb[j * stride]), fma(sg * ab, u, cb[(j + 1) * stride]), Ea, Eb);
            S += Ea;
            SA = fma(aa, Ea, SA);
            S += Eb;
            SA = fma(ab, Eb, SA);
        }
        if (j < d) {
            const double aj = P.a[j];
            const double E = fast_exp(fma(sg * aj, u, cb[j * stride]));
            S += E;
            SA = fma(aj, E, SA);
        }
        const double h = fast_log(S) - lndK;
        const double du = h * S / (sg * SA);
        conv = fabs(du) <= 1e-13 * fmax(1.0, fabs(u));
        u = fmin(fmax(u - du, u_lo), u_hi);
        if (it + 1 >= kNewtonIt && __all_sync(__activemask(), conv)) break;
    }
    unconverged += conv ? 0u : 1u;
    double Dst = 0.0, Qst = 0.0, Vst = 0.0, sumW = 0.0, sumWv = 0.0;
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
            double wa, wb, Pa, Pb, pa, pb;
            fast_exp_x2(fma(0.5 * sg * sg * aa, aa, ca), fma(0.5 * sg * sg * ab, ab, cbb), wa, wb);
            phibar_phi_x2(u - sg * aa, u - sg * ab, Pa, Pb, pa, pb);  // Phi(sigma a - u) = Phibar(u - sigma a)
            wb *= wgt;
            sumW = fma(wa, Pa, sumW);
            sumWv = fma(wa * (Ra - sg * ta + sg * aa * aa), Pa, sumWv);
            sumW = fma(wb, Pb, sumW);
            sumWv = fma(wb * (Rb - sg * tb + sg * ab * ab), Pb, sumWv);
        }
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
__device__ __forceinline__ void x1_lookback(const PathArgs& P, int o, const double* cb, int stride, double f[4]) {
    const int d = P.d;
    const double sg = P.sigma, lnK = P.lnK[o];
    double ustar = CUDART_INF;
    int j0 = 0;
    for (int j = 0; j < d; ++j) {
        const double uj = (lnK - cb[j * stride]) * P.inv_sa[j];
        if (uj < ustar) {
            ustar = uj;
            j0 = j;
        }
    }
    // active line at u*: the maximum there; on ties the steeper one (it dominates just after)
    int act = 0;
    double best = -CUDART_INF, bact = 0.0;
    for (int j = 0; j < d; ++j) {
        const double bj = sg * __ldg(P.a + j);
        const double v = fma(bj, ustar, cb[j * stride]);
        if (v > best || (v == best && bj > bact)) {
            best = v;
            act = j;
            bact = bj;
        }
    }
    double J = 0.0, V = 0.0, lo = ustar;
    for (int seg = 0; seg < d; ++seg) {
        const double cact = cb[act * stride];
        double hi = CUDART_INF, bn = 0.0;
        int nxt = -1;
        for (int i = 0; i < d; ++i) {
            const double bi = sg * __ldg(P.a + i);
            if (bi > bact) {
                const double x = (cact - cb[i * stride]) / (bi - bact);
                if (x < hi || (x == hi && bi > bn)) {
                    hi = x;
                    nxt = i;
                    bn = bi;
                }
            }
        }
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
        if (nxt < 0) break;
        lo = hi;
        act = nxt;
        bact = bn;
    }
    const double D = P.Dfac, S0 = P.S0, K = P.K[o];
    double Qu, Q2, ph, ph2;
    phibar_phi_x2(ustar, ustar, Qu, Q2, ph, ph2);
    f[0] = D * (J - K * Qu);
    f[1] = D * J / S0;
    f[2] = D * V;
    f[3] = D * K * ph / (S0 * S0 * sg * __ldg(P.a + j0));
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
            xs[o] = ld == 0 ? xs[0] : xs[ld == 1 ? 1 : 0];
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
__device__ __forceinline__ void warp_slot_sums(const double (&f)[kMaxOpt][4], const PathArgs& P, bool valid,
                                               int lane, double* wacc) {
#pragma unroll
    for (int o = 0; o < kMaxOpt; ++o) {
        if (o >= P.n_opt) break;  // warp-uniform
        double v[8];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const double y = valid ? f[o][q] - P.piv[o][q] : 0.0;
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
        if ((lane & 3) == 0) wacc[o * 8 + (lane >> 2)] += v[0];
    }
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
        red[warp * 32 + P.n_opt * 8 + 0] = (double)uc;
        red[warp * 32 + P.n_opt * 8 + 1] = (double)tc;
        red[warp * 32 + P.n_opt * 8 + 2] = (double)nc;  // points this cell evaluated (completeness check)
    }
    __syncthreads();
    if (tid < n_out) {
        double s = 0.0;
        for (int w = 0; w < nwarps; ++w) s += red[w * 32 + tid];
        P.partials[(size_t)cell * n_out + tid] = s;
    }
}

#ifndef QMCCPW_BB_MINB
#define QMCCPW_BB_MINB 8
#endif
#ifndef QMCCPW_STD_MINB
#define QMCCPW_STD_MINB 6
#endif
// resident blocks per SM the register allocator must allow (128 threads each); 0 = ptxas'
// own choice.  Measured on C4 (ms/step): BB-W1 34.3 (ptxas, 96 regs) / 33.8 (7) / 33.4
// (8: 64 regs, a few spills to L1); STD-W1 33.1 (4) / 31.9 (5) / 31.2 (6)
template <int CONSTR, int COND, int METHOD>
constexpr int paths_min_blocks() {
    return (COND == kW1 && METHOD == kQmc) ? (CONSTR == kBB ? QMCCPW_BB_MINB : CONSTR == kStd ? QMCCPW_STD_MINB : 0) : 0;
}
template <int CONSTR, int COND, int METHOD>
__global__ void __launch_bounds__(128, paths_min_blocks<CONSTR, COND, METHOD>())
    paths_kernel(const PathArgs P) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int tpb_log2 = P.tpb_log2;
    const int tpb = 1 << tpb_log2;
    const int tid = threadIdx.x;
    const int d = P.d;
    const uint64_t cell = P.cell_begin + blockIdx.x;
    const uint32_t rep_local = (uint32_t)(cell / P.cells_per_rep);
    const uint64_t blk = cell % P.cells_per_rep;
    const uint64_t i0 = blk * (uint64_t)kCellPoints;
    const int ppt = kCellPoints >> tpb_log2;
    constexpr bool kNeedBuf = (METHOD == kQmc) && (CONSTR == kPca || COND == kX1);
    constexpr bool kTwoBuf = (METHOD == kQmc) && (CONSTR == kPca && COND == kX1);
    constexpr bool kWarpMma = (METHOD == kQmc) && (CONSTR == kPca && COND == kW1);

    // shared memory carve-up (8-byte aligned first):
    //   buf0, buf1 [d][tpb] | vt [d][32] | sh [d] | G [d][32] | pad | HW [2][2][nw][d] (>= 1 KB)
    // the reduction scratch red [4 warps][32] aliases HW after the point loop; the
    // centred sums live in one register per lane (warp_slot_sums).
    const int nw = tpb >> 5;
    const int n_acc = P.n_opt * 8;
    const int lane = tid & 31;
    double* buf0 = reinterpret_cast<double*>(smem_raw);
    double* buf1 = buf0 + (kWarpMma ? (size_t)P.M_ld * (tpb + 8) : (kNeedBuf ? (size_t)d * tpb : 0));
    uint32_t* vt = reinterpret_cast<uint32_t*>(buf1 + (kTwoBuf ? (size_t)d * tpb : 0));
    uint32_t* sh = vt + (METHOD == kQmc ? (size_t)d * 32 : 0);
    uint32_t* G = sh + (METHOD == kQmc ? d : 0);
    uint32_t* HW = G + (METHOD == kQmc ? (size_t)d * 32 : 0);
    HW += ((uintptr_t)HW & 7) ? 1 : 0;
    double* red = reinterpret_cast<double*>(HW);
    const int hw_size = 2 * nw * d;

    const uint64_t K0 = P.point_offset + i0;
    const uint64_t Ab = K0 >> tpb_log2;
    const uint64_t kt = K0 + (uint64_t)tid;
    SobolBlock sob{G, HW, d, nw, (int)(kt & 31), (int)((kt >> 5) & (uint64_t)(nw - 1)), (int)((kt >> tpb_log2) - Ab),
                   P.owen ? sh : nullptr};
    if (METHOD == kQmc) {
        const uint32_t* src = P.vscr + (size_t)rep_local * d * 32;
        for (int idx = tid; idx < d * 32; idx += tpb) vt[idx] = src[idx];
        for (int idx = tid; idx < d; idx += tpb) sh[idx] = P.shift[(size_t)rep_local * d + idx];
        __syncthreads();
        sobol_build_g(vt, d, G, tid, tpb);
    }
    __shared__ double wacc[4 * 32];  // per-warp centred sums (tpb <= 128)
    wacc[tid] = 0.0;
    __syncwarp();
    if (kWarpMma)  // zero X rows d..dp-1 (the padded K of the mma tiles)
        for (int r = d; r < P.M_ld; ++r) buf0[(size_t)r * (tpb + 8) + tid] = 0.0;
    unsigned unconverged = 0, ties = 0, npts = 0;

    for (int a = 0; a < ppt; ++a) {
        if (i0 + ((uint64_t)a << tpb_log2) >= P.n_points) break;  // block-uniform: ragged last cell
        if (METHOD == kQmc) {
            uint32_t* HWb = HW + (a & 1) * hw_size;  // double-buffered: one barrier per iteration
            sobol_build_hw(vt, P.owen ? nullptr : sh, d, P.dim_begin, tpb_log2, nw, Ab + (uint64_t)a, HWb, tid, tpb);
            __syncthreads();
            sob.HW = HWb;
        }
        const uint64_t i = i0 + tid + ((uint64_t)a << tpb_log2);
        // every lane runs (the warp reduction and the mma.sync tiles need the whole warp);
        // lanes past N in a ragged last iteration evaluate a real lattice point whose
        // result and counters are dropped
        const bool valid = i < P.n_points;
        const unsigned unconverged0 = unconverged, ties0 = ties;
        npts += valid ? 1u : 0u;
        const uint64_t k = P.point_offset + i;
        double f[kMaxOpt][4];

        if (METHOD == kLr) {
            lr_path(P, P.rep_base + rep_local, k, f);
        } else if (METHOD == kMc || METHOD == kMcAv) {
            // MC-CPW and MC+AV-CPW: pseudo-random normals through the
            // same W1 estimator; the antithetic path of -x has W~ -> -W~ (the constructions
            // are linear), so one traversal feeds both accumulators.
            const uint32_t rep = P.rep_base + rep_local;
            W1Acc w1, w1m;
            w1.reset();
            w1m.reset();
            if (CONSTR == kStd) {
                double Wt = 0.0;
                w1.push(P, 0, 0.0);
                if (METHOD == kMcAv) w1m.push(P, 0, 0.0);
#pragma unroll 1
                for (int jq = 0; jq < d; jq += 4) {
                    uint32_t c[4] = {(uint32_t)k, (uint32_t)(k >> 32), (uint32_t)(jq >> 2), (rep << 8) | 0x02u};
                    philox4x32_10(c, (uint32_t)P.seed, (uint32_t)(P.seed >> 32));
                    double xs[4];
                    normal_from_u32_x2(c[0], c[1], xs[0], xs[1]);
                    normal_from_u32_x2(c[2], c[3], xs[2], xs[3]);
#pragma unroll
                    for (int w = 0; w < 4; ++w) {
                        const int j = jq + w;
                        if (j >= 1 && j < d) {
                            Wt = fma(P.sqrt_t1, xs[w], Wt);
                            w1.push(P, j, Wt);
                            if (METHOD == kMcAv) w1m.push(P, j, -Wt);
                        }
                    }
                }
            } else {
                NormalFifo fifo;
                fifo.reset();
                int pos = 0;
                auto dim_at = [&](int o) { return (int)P.bb_seq[pos + o]; };
                auto draw = [&](int da, int db, double& xa, double& xb) { mc_normal_pair(P, rep, k, da, db, xa, xb); };
                double stW[12];
                int sp = 0;
                stW[0] = P.sqrtT * fifo.next_from(draw, dim_at);
                pos += 2;
                double Wl = 0.0, W1 = 0.0, Wpend = 0.0;
                const int m = P.bb_m;
#pragma unroll 1
                for (int j = 1; j <= d; ++j) {
                    const int e = (j == 1) ? m : (__ffs(j - 1) - 1);
                    double Wj;
                    if (e == 0) {
                        Wj = stW[sp];
                        --sp;
                    } else {
                        double Wr = stW[sp];
#pragma unroll 1
                        for (int c = e - 1; c >= 0; --c) {
                            const bool refill = fifo.have == 0;
                            const double x = fifo.next_from(draw, dim_at);
                            pos += refill ? 2 : 0;
                            const double Wm = fma(P.bb_b[m - c], x, 0.5 * (Wl + Wr));
                            if (c > 0) stW[++sp] = Wm;
                            Wr = Wm;
                        }
                        Wj = Wr;
                    }
                    if (j == 1) W1 = Wj;
                    if (j & 1) {
                        Wpend = Wj - W1;
                    } else {
                        w1.push2(P, j - 2, Wpend, Wj - W1);
                        if (METHOD == kMcAv) w1m.push2(P, j - 2, -Wpend, -(Wj - W1));
                    }
                    Wl = Wj;
                }
                if (d & 1) {
                    w1.push(P, d - 1, Wpend);
                    if (METHOD == kMcAv) w1m.push(P, d - 1, -Wpend);
                }
            }
            if (P.has_lookback && w1.emax - w1.esec < 1e-12) ++ties;
            tail_w1_all(P, w1, f);
            if (METHOD == kMcAv) {
                if (P.has_lookback && w1m.emax - w1m.esec < 1e-12) ++ties;
                double fm[kMaxOpt][4];
                tail_w1_all(P, w1m, fm);
#pragma unroll
                for (int o = 0; o < kMaxOpt; ++o)
#pragma unroll
                    for (int qq = 0; qq < 4; ++qq) f[o][qq] = 0.5 * (f[o][qq] + fm[o][qq]);
            }
        } else if (COND == kW1) {
            W1Acc w1;
            w1.reset();
            if (CONSTR == kStd) {
                // Alg. 3: W~ accumulates sqrt(dt) x_j for j >= 2; x_1 cancels in
                // W - W(t_1).  Normals and exps two dates at a time.
                double Wt = 0.0;
                w1.push(P, 0, 0.0);
                int j = 1;
#pragma unroll 1
                for (; j + 1 < d; j += 2) {
                    double xa, xb;
                    normal_from_u32_x2(sob.get(j), sob.get(j + 1), xa, xb);
                    const double Wa = fma(P.sqrt_t1, xa, Wt);
                    Wt = fma(P.sqrt_t1, xb, Wa);
                    w1.push2(P, j, Wa, Wt);
                }
                if (j < d) {
                    Wt = fma(P.sqrt_t1, normal_from_u32(sob.get(j)), Wt);
                    w1.push(P, j, Wt);
                }
            } else if (CONSTR == kBB) {
                // Alg. 4 generated in time order, two dates per step.  At odd
                // j = 2p+1 the bridge descends e = 1 + ctz(p) levels (e = m at p = 0) from the
                // interval (t_{j-1}, t_{j-1+2^e}]: midpoint mid = j-1+2^c (c = e-1..0) sits at
                // level m-c, consumes the next Sobol' dimension of Alg. 4's order (bb_seq, built
                // on the host), W(mid) = (W(l) + W(r))/2 + b_{m-c} x, and is pushed for c > 0.
                // W(t_j) is the c = 0 midpoint; W(t_{j+1}) is then exactly the stack top.
                NormalFifo fifo;
                fifo.reset();
                int pos = 0;
                auto dim_at = [&](int o) { return (int)P.bb_seq[pos + o]; };
                double stW[12];
                int sp = 0;
                stW[0] = P.sqrtT * fifo.next(sob, dim_at);
                pos += 2;
                const int m = P.bb_m;
                if (d == 1) {
                    w1.push(P, 0, 0.0);
                } else {
                    double Wl = 0.0, W1 = 0.0;
#pragma unroll 1
                    for (int pp = 0; pp < (d >> 1); ++pp) {
                        const int e = (pp == 0) ? m : __ffs(pp);  // 1 + ctz(pp)
                        double Wr = stW[sp];
#pragma unroll 1
                        for (int c = e - 1; c >= 0; --c) {
                            const bool refill = fifo.have == 0;
                            const double x = fifo.next(sob, dim_at);
                            pos += refill ? 2 : 0;
                            const double Wm = fma(P.bb_b[m - c], x, 0.5 * (Wl + Wr));
                            if (c > 0) stW[++sp] = Wm;
                            Wr = Wm;
                        }
                        const double Wodd = Wr, Weven = stW[sp];
                        --sp;
                        if (pp == 0) W1 = Wodd;
                        w1.push2(P, 2 * pp, Wodd - W1, Weven - W1);
                        Wl = Weven;
                    }
                }
            } else {
                // PCA: W = X M^T, the one dense contraction, on the FP64 tensor
                // cores.  Each thread writes its path's normals as a column of X (shared
                // memory, row stride tpb + 8 doubles: the 4 k-rows of an A fragment fall on
                // disjoint bank halves); each warp then runs mma.sync.m8n8k4.f64 (SASS DMMA)
                // over its 32 paths x dp times: A = X[k][path] (8 paths x 4 k), B = M[j][k]
                // (4 k x 8 j, from L1), D = 8 paths x 8 j.  Lane (q = lane/4, r = lane%4) ends
                // up holding W for paths 8 rt + q (rt = 0..3) at times jt + 2r + {0,1}; it
                // accumulates those paths' S~ statistics, the quad reduces them, and the
                // owning lane takes them over for the tail.
                const int XS = tpb + 8;
                const int dp = P.M_ld;
                double* xc = buf0 + tid;
                int kk = 0;
#pragma unroll 1
                for (; kk + 1 < d; kk += 2) {
                    double xa, xc2;
                    normal_from_u32_x2(sob.get(kk), sob.get(kk + 1), xa, xc2);
                    xc[kk * XS] = xa;
                    xc[(kk + 1) * XS] = xc2;
                }
                if (kk < d) xc[kk * XS] = normal_from_u32(sob.get(kk));
                __syncwarp();
                const int lane = tid & 31, q = lane >> 2, r4 = lane & 3;
                const double* Xw = buf0 + (tid & ~31);
                double sS[4], sI[4], em[4], es[4], ym[4], W1r[4];
                int jm[4];
#pragma unroll
                for (int rt = 0; rt < 4; ++rt) {
                    sS[rt] = 0.0; sI[rt] = 0.0; em[rt] = -CUDART_INF; es[rt] = -CUDART_INF; ym[rt] = 0.0;
                    jm[rt] = 0x7fffffff; W1r[rt] = 0.0;
                }
#pragma unroll 1
                for (int jt = 0; jt < dp; jt += 8) {
                    double acc[4][2];
#pragma unroll
                    for (int rt = 0; rt < 4; ++rt) acc[rt][0] = acc[rt][1] = 0.0;
                    const double* Mrow = P.M + (size_t)(jt + q) * dp + r4;
                    const double* Xk = Xw + (size_t)r4 * XS + q;
#pragma unroll 2
                    for (int kt = 0; kt < dp; kt += 4) {
                        const double bfrag = __ldg(Mrow + kt);
                        const double* Xr = Xk + (size_t)kt * XS;
#pragma unroll
                        for (int rt = 0; rt < 4; ++rt) {
                            const double afrag = Xr[8 * rt];
                            asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                                         : "+d"(acc[rt][0]), "+d"(acc[rt][1])
                                         : "d"(afrag), "d"(bfrag));
                        }
                    }
                    if (jt == 0) {
#pragma unroll
                        for (int rt = 0; rt < 4; ++rt) W1r[rt] = __shfl_sync(0xffffffffu, acc[rt][0], lane & ~3);
                    }
                    const int j0 = jt + 2 * r4;
#pragma unroll
                    for (int rt = 0; rt < 4; ++rt) {
                        const double Wa = acc[rt][0] - W1r[rt], Wb = acc[rt][1] - W1r[rt];
                        const double ta = (double)j0 * P.t1, tb = ta + P.t1;
                        const double ea = fma(P.sigma, Wa, P.omega * ta), eb = fma(P.sigma, Wb, P.omega * tb);
                        double Xa, Xb;
                        fast_exp_x2(ea, eb, Xa, Xb);
                        const double va = (j0 < d) ? 1.0 : 0.0, vb = (j0 + 1 < d) ? 1.0 : 0.0;
                        const double Sa = P.S0 * Xa * va, Sb = P.S0 * Xb * vb;
                        const double ya = fma(-P.sigma, ta, Wa), yb = fma(-P.sigma, tb, Wb);
                        sS[rt] += Sa;
                        sI[rt] = fma(Sa, ya, sI[rt]);
                        sS[rt] += Sb;
                        sI[rt] = fma(Sb, yb, sI[rt]);
                        if (P.has_lookback) {
                            const double eav = (j0 < d) ? ea : -CUDART_INF, ebv = (j0 + 1 < d) ? eb : -CUDART_INF;
                            // lowest index wins ties (j0 < j0 + 1 < later tiles)
                            bool gt = eav > em[rt];
                            es[rt] = fmax(es[rt], gt ? em[rt] : eav);
                            ym[rt] = gt ? ya : ym[rt];
                            jm[rt] = gt ? j0 : jm[rt];
                            em[rt] = gt ? eav : em[rt];
                            gt = ebv > em[rt];
                            es[rt] = fmax(es[rt], gt ? em[rt] : ebv);
                            ym[rt] = gt ? yb : ym[rt];
                            jm[rt] = gt ? j0 + 1 : jm[rt];
                            em[rt] = gt ? ebv : em[rt];
                        }
                    }
                }
                __syncwarp();  // X may be overwritten by the next point only after every lane's mma
                // quad reduction (lanes 4q..4q+3 hold disjoint j's of the same paths)
#pragma unroll
                for (int rt = 0; rt < 4; ++rt) {
#pragma unroll
                    for (int off = 1; off <= 2; off <<= 1) {
                        sS[rt] += __shfl_xor_sync(0xffffffffu, sS[rt], off);
                        sI[rt] += __shfl_xor_sync(0xffffffffu, sI[rt], off);
                        if (P.has_lookback) {
                            const double pe = __shfl_xor_sync(0xffffffffu, em[rt], off);
                            const double pes = __shfl_xor_sync(0xffffffffu, es[rt], off);
                            const double py = __shfl_xor_sync(0xffffffffu, ym[rt], off);
                            const int pj = __shfl_xor_sync(0xffffffffu, jm[rt], off);
                            const bool take = pe > em[rt] || (pe == em[rt] && pj < jm[rt]);
                            es[rt] = fmax(fmax(es[rt], pes), fmin(em[rt], pe));
                            em[rt] = take ? pe : em[rt];
                            ym[rt] = take ? py : ym[rt];
                            jm[rt] = take ? pj : jm[rt];
                        }
                    }
                }
                // hand path 8 rt + q's statistics to its owner lane (lane = 8 rt + q)
                const int src = 4 * (lane & 7), mine = lane >> 3;
#pragma unroll
                for (int rt = 0; rt < 4; ++rt) {
                    const double a0 = __shfl_sync(0xffffffffu, sS[rt], src);
                    const double a1 = __shfl_sync(0xffffffffu, sI[rt], src);
                    const double a2 = __shfl_sync(0xffffffffu, em[rt], src);
                    const double a3 = __shfl_sync(0xffffffffu, es[rt], src);
                    const double a4 = __shfl_sync(0xffffffffu, ym[rt], src);
                    if (rt == mine) {
                        w1.sumS = a0;
                        w1.sumI = a1;
                        w1.emax = a2;
                        w1.esec = a3;
                        w1.ymax = a4;
                    }
                }
            }
            if (P.has_lookback && w1.emax - w1.esec < 1e-12) ++ties;
            tail_w1_all(P, w1, f);
        } else {
            // X1: c_j = ln S0 + omega t_j + sigma R_j, R = M x with x_1 := 0
            double* cb = (CONSTR == kPca ? buf1 : buf0) + tid;
            if (CONSTR == kStd) {
                double R = 0.0;
                cb[0] = P.lnS0 + P.omega * P.t1;
                int j = 1;
#pragma unroll 1
                for (; j + 1 < d; j += 2) {
                    double xa, xb2;
                    normal_from_u32_x2(sob.get(j), sob.get(j + 1), xa, xb2);
                    R = fma(P.sqrt_t1, xa, R);
                    cb[j * tpb] = P.lnS0 + P.omega * (double)(j + 1) * P.t1 + P.sigma * R;
                    R = fma(P.sqrt_t1, xb2, R);
                    cb[(j + 1) * tpb] = P.lnS0 + P.omega * (double)(j + 2) * P.t1 + P.sigma * R;
                }
                if (j < d) {
                    R = fma(P.sqrt_t1, normal_from_u32(sob.get(j)), R);
                    cb[j * tpb] = P.lnS0 + P.omega * (double)(j + 1) * P.t1 + P.sigma * R;
                }
            } else if (CONSTR == kBB) {
                // same time-order bridge with the terminal loading of x_1 removed (R = M x, x_1 := 0);
                // normals in Alg. 4 order from bb_seq[1..]
                NormalFifo fifo;
                fifo.reset();
                int pos = 1;
                auto dim_at = [&](int o) { return (int)P.bb_seq[pos + o]; };
                double stW[12];
                int sp = 0;
                stW[0] = 0.0;
                double Wl = 0.0;
                const int m = P.bb_m;
#pragma unroll 1
                for (int j = 1; j <= d; ++j) {
                    const int e = (j == 1) ? m : (__ffs(j - 1) - 1);
                    double Rj;
                    if (e == 0) {
                        Rj = stW[sp];
                        --sp;
                    } else {
                        double Wr = stW[sp];
#pragma unroll 1
                        for (int c = e - 1; c >= 0; --c) {
                            const bool refill = fifo.have == 0;
                            const double x = fifo.next(sob, dim_at);
                            pos += refill ? 2 : 0;
                            const double Wm = fma(P.bb_b[m - c], x, 0.5 * (Wl + Wr));
                            if (c > 0) stW[++sp] = Wm;
                            Wr = Wm;
                        }
                        Rj = Wr;
                    }
                    cb[(j - 1) * tpb] = P.lnS0 + P.omega * (double)j * P.t1 + P.sigma * Rj;
                    Wl = Rj;
                }
            } else {
                double* xb = buf0 + tid;
                int kk = 1;
#pragma unroll 1
                for (; kk + 1 < d; kk += 2) {
                    double xa, xc;
                    normal_from_u32_x2(sob.get(kk), sob.get(kk + 1), xa, xc);
                    xb[kk * tpb] = xa;
                    xb[(kk + 1) * tpb] = xc;
                }
                if (kk < d) xb[kk * tpb] = normal_from_u32(sob.get(kk));
                int j = 0;
#pragma unroll 1
                for (; j + 1 < d; j += 2) {
                    const double* Ma = P.M + (size_t)j * P.M_ld;
                    const double* Mb = Ma + P.M_ld;
                    double Ra = 0.0, Rb = 0.0;
#pragma unroll 4
                    for (int q = 1; q < d; ++q) {
                        const double xq = xb[q * tpb];
                        Ra = fma(__ldg(Ma + q), xq, Ra);
                        Rb = fma(__ldg(Mb + q), xq, Rb);
                    }
                    cb[j * tpb] = P.lnS0 + P.omega * (double)(j + 1) * P.t1 + P.sigma * Ra;
                    cb[(j + 1) * tpb] = P.lnS0 + P.omega * (double)(j + 2) * P.t1 + P.sigma * Rb;
                }
                if (j < d) {
                    const double* Ma = P.M + (size_t)j * P.M_ld;
                    double Ra = 0.0;
                    for (int q = 1; q < d; ++q) Ra = fma(__ldg(Ma + q), xb[q * tpb], Ra);
                    cb[j * tpb] = P.lnS0 + P.omega * (double)(j + 1) * P.t1 + P.sigma * Ra;
                }
            }
            tail_x1_all(P, cb, tpb, f, unconverged);
        }

        if (!valid) {
            unconverged = unconverged0;
            ties = ties0;
        }
        if (P.path_out != nullptr && valid) {
#pragma unroll
            for (int o = 0; o < kMaxOpt; ++o)
                if (o == P.hook_option)
                    for (int q = 0; q < 4; ++q) P.path_out[i * 4 + q] = f[o][q];
        }
        warp_slot_sums(f, P, valid, lane, wacc + (tid >> 5) * 32);
        (void)k;
    }

    block_epilogue(P, nullptr, wacc, red, n_acc, tpb, tid, cell, unconverged, ties, npts);
}


// ---------------------------------------------------------------------------
// PCA on the FP64 tensor cores, fragment-native (no per-path shared memory).
//
// W = X M^T (or R = X M[:,1:]^T for X1) is the one dense contraction of the
// path.  A warp works on its 32 points as 4 row tiles of 8 paths.
// Lane (q = lane/4, r = lane%4) draws, for path 8 rt + q, exactly the normals
// of its m8n8k4 A fragments -- x[path][4 f + r], f = 0..KF-1 -- straight from
// the block's Sobol' tables (any lane can form any path's y_j), so X never goes
// through shared memory.  mma.sync.m8n8k4.f64 (SASS DMMA) against B = M[j][k]
// (L1) leaves lane (q, r) with W(t_j) of its path at j = 8 jt + 2 r + {0, 1}.
//  * W1: the quad accumulates the S~ statistics of its path from those
//    values, reduces them, and the owning lane runs the option tails.
//  * X1: c_j stays in the quad's registers; Newton's sums over j are
//    quad-reduced, so the threshold is solved by the 4 lanes together.
// ---------------------------------------------------------------------------
__device__ __forceinline__ double quad_sum(double v) {
    v += __shfl_xor_sync(0xffffffffu, v, 1);
    return v + __shfl_xor_sync(0xffffffffu, v, 2);
}
__device__ __forceinline__ double quad_min(double v) {
    v = fmin(v, __shfl_xor_sync(0xffffffffu, v, 1));
    return fmin(v, __shfl_xor_sync(0xffffffffu, v, 2));
}

#ifndef QMCCPW_PCA_W1_MINB
#define QMCCPW_PCA_W1_MINB 4
#endif
#ifndef QMCCPW_PCA_X1_MINB
#define QMCCPW_PCA_X1_MINB 5
#endif
// d <= 64: shared memory allows 5 blocks/SM, so cap registers to match (measured on C4:
// PCA-W1 72.4 -> 69.4 ms, PCA-X1 175 -> 165 ms); larger d is smem-limited anyway
template <int COND, int KF>
constexpr int pca_min_blocks() {
    return KF > 16 ? 0 : (COND == kW1 ? QMCCPW_PCA_W1_MINB : QMCCPW_PCA_X1_MINB);
}
template <int COND, int KF>
__global__ void __launch_bounds__(128, pca_min_blocks<COND, KF>()) pca_kernel(const PathArgs P) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    constexpr int DP = 4 * KF;  // padded dimension (multiple of 8)
    constexpr int JT = DP / 8;  // column tiles of 8 dates
    const int tpb_log2 = P.tpb_log2, tpb = 1 << tpb_log2, tid = threadIdx.x, d = P.d;
    const int lane = tid & 31, q = lane >> 2, r4 = lane & 3, wbase = tid & ~31;
    const uint64_t cell = P.cell_begin + blockIdx.x;
    const uint32_t rep_local = (uint32_t)(cell / P.cells_per_rep);
    const uint64_t blk = cell % P.cells_per_rep;
    const uint64_t i0 = blk * (uint64_t)kCellPoints;
    const int ppt = kCellPoints >> tpb_log2;
    const int nw = tpb >> 5;
    const int n_acc = P.n_opt * 8;
    // per-path accumulators in smem: X1 as scalars (one quad lane per path), W1 as (S1, S2) pairs
    double* accs = reinterpret_cast<double*>(smem_raw);
    double2* acc2 = reinterpret_cast<double2*>(smem_raw);
    uint32_t* vt = reinterpret_cast<uint32_t*>(accs + (size_t)n_acc * tpb);
    uint32_t* sh = vt + (size_t)d * 32;
    uint32_t* G = sh + d;
    uint32_t* HW = G + (size_t)d * 32;
    HW += ((uintptr_t)HW & 7) ? 1 : 0;
    double* red = reinterpret_cast<double*>(HW);
    const int hw_size = 2 * nw * d;
    const uint64_t K0 = P.point_offset + i0;
    const uint64_t Ab = K0 >> tpb_log2;
    {
        const uint32_t* src = P.vscr + (size_t)rep_local * d * 32;
        for (int idx = tid; idx < d * 32; idx += tpb) vt[idx] = src[idx];
        for (int idx = tid; idx < d; idx += tpb) sh[idx] = P.shift[(size_t)rep_local * d + idx];
        __syncthreads();
        sobol_build_g(vt, d, G, tid, tpb);
    }
    for (int v = 0; v < n_acc; ++v) accs[v * tpb + tid] = 0.0;
    __shared__ double wacc[4 * 32];  // per-warp centred sums (tpb <= 128)
    wacc[tid] = 0.0;
    __syncwarp();
    unsigned unconverged = 0, ties = 0, npts = 0;
    const double sg = P.sigma;

    for (int a = 0; a < ppt; ++a) {
        if (i0 + ((uint64_t)a << tpb_log2) >= P.n_points) break;  // block-uniform
        uint32_t* HWb = HW + (a & 1) * hw_size;
        sobol_build_hw(vt, P.owen ? nullptr : sh, d, 0, tpb_log2, nw, Ab + (uint64_t)a, HWb, tid, tpb);
        __syncthreads();
        // W1: statistics of this lane's own path, handed over by its quad after each row tile
        W1Acc w1own;
        w1own.reset();
#pragma unroll 1
        for (int rt = 0; rt < 4; ++rt) {
            const int tp = wbase + 8 * rt + q;  // block slot of this quad's path
            const uint64_t kp0 = K0 + (uint64_t)tp;
            const uint64_t ip = i0 + (uint64_t)tp + ((uint64_t)a << tpb_log2);
            const bool valid = ip < P.n_points;
            const SobolBlock sp{G, HWb, d, nw, (int)(kp0 & 31), (int)((kp0 >> 5) & (uint64_t)(nw - 1)),
                                (int)((kp0 >> tpb_log2) - Ab), P.owen ? sh : nullptr};
            // A fragments: x[path][4 f + r4]
            double afr[KF];
#pragma unroll
            for (int f = 0; f < KF; f += 2) {
                const int ja = 4 * f + r4, jb = 4 * (f + 1) + r4;
                double xa, xb;
                normal_from_u32_x2(sp.get(ja < d ? ja : d - 1), sp.get(jb < d ? jb : d - 1), xa, xb);
                afr[f] = (ja < d && !(COND == kX1 && ja == 0)) ? xa : 0.0;
                afr[f + 1] = (jb < d && !(COND == kX1 && jb == 0)) ? xb : 0.0;
            }
            double cv[2 * JT];  // W(t_j) (W1) or c_j (X1) at j = 8 jt + 2 r4 + e
            double W1v = 0.0;
#pragma unroll
            for (int jt = 0; jt < JT; ++jt) {
                double acc0 = 0.0, acc1 = 0.0;
                const double* Mrow = P.M + (size_t)(8 * jt + q) * DP + r4;
#pragma unroll
                for (int f = 0; f < KF; ++f) {
                    const double bfrag = __ldg(Mrow + 4 * f);
                    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                                 : "+d"(acc0), "+d"(acc1)
                                 : "d"(afr[f]), "d"(bfrag));
                }
                cv[2 * jt] = acc0;
                cv[2 * jt + 1] = acc1;
            }
            if (COND == kW1) {
                W1v = __shfl_sync(0xffffffffu, cv[0], lane & ~3);  // W(t_1) of this path
                double sS = 0.0, sI = 0.0, em = -CUDART_INF, es = -CUDART_INF, ym = 0.0;
#pragma unroll
                for (int jt = 0; jt < JT; ++jt) {
                    const int j0 = 8 * jt + 2 * r4;
                    const double Wa = cv[2 * jt] - W1v, Wb = cv[2 * jt + 1] - W1v;
                    const double ta = (double)j0 * P.t1, tb = ta + P.t1;
                    const double ea = fma(sg, Wa, P.omega * ta), eb = fma(sg, Wb, P.omega * tb);
                    double Xa, Xb;
                    fast_exp_x2(ea, eb, Xa, Xb);
                    const double Sa = (j0 < d) ? P.S0 * Xa : 0.0, Sb = (j0 + 1 < d) ? P.S0 * Xb : 0.0;
                    const double ya = fma(-sg, ta, Wa), yb = fma(-sg, tb, Wb);
                    sS += Sa;
                    sI = fma(Sa, ya, sI);
                    sS += Sb;
                    sI = fma(Sb, yb, sI);
                    if (P.has_lookback) {
                        const double eav = (j0 < d) ? ea : -CUDART_INF, ebv = (j0 + 1 < d) ? eb : -CUDART_INF;
                        bool gt = eav > em;
                        es = fmax(es, gt ? em : eav);
                        ym = gt ? ya : ym;
                        em = gt ? eav : em;
                        gt = ebv > em;
                        es = fmax(es, gt ? em : ebv);
                        ym = gt ? yb : ym;
                        em = gt ? ebv : em;
                    }
                }
                // quad reduction (the 4 lanes hold disjoint dates of the same path)
                sS = quad_sum(sS);
                sI = quad_sum(sI);
                if (P.has_lookback) {
#pragma unroll
                    for (int off = 1; off <= 2; off <<= 1) {
                        const double pe = __shfl_xor_sync(0xffffffffu, em, off);
                        const double pes = __shfl_xor_sync(0xffffffffu, es, off);
                        const double py = __shfl_xor_sync(0xffffffffu, ym, off);
                        const bool take = pe > em;  // an exact tie is a near-tie either way
                        es = fmax(fmax(es, pes), fmin(em, pe));
                        em = take ? pe : em;
                        ym = take ? py : ym;
                    }
                }
                // owner of path 8 rt + q is lane 8 rt + q: it reads lane 4 (its q) of this row tile
                const int src = 4 * (lane & 7);
                const double a0 = __shfl_sync(0xffffffffu, sS, src);
                const double a1 = __shfl_sync(0xffffffffu, sI, src);
                const double a2 = __shfl_sync(0xffffffffu, em, src);
                const double a3 = __shfl_sync(0xffffffffu, es, src);
                const double a4 = __shfl_sync(0xffffffffu, ym, src);
                if ((lane >> 3) == rt) {
                    w1own.sumS = a0;
                    w1own.sumI = a1;
                    w1own.emax = a2;
                    w1own.esec = a3;
                    w1own.ymax = a4;
                }
            } else {
                // X1: c_j = ln S0 + omega t_j + sigma R_j, then one Newton solve per strike group
#pragma unroll
                for (int jt = 0; jt < JT; ++jt) {
                    const int j0 = 8 * jt + 2 * r4;
                    cv[2 * jt] = fma(sg, cv[2 * jt], fma(P.omega, (double)(j0 + 1) * P.t1, P.lnS0));
                    cv[2 * jt + 1] = fma(sg, cv[2 * jt + 1], fma(P.omega, (double)(j0 + 2) * P.t1, P.lnS0));
                }
                double f[kMaxOpt][4];
#pragma unroll
                for (int o = 0; o < kMaxOpt; ++o) {
                    if (o >= P.n_opt) break;
                    if (P.tail_leader[o] != o) continue;
                    const double lnK = P.lnK[o], lndK = P.lndK[o];
                    // bracket [min_j (lnK - c_j)/(sigma a_j), min_j (ln dK - c_j)/(sigma a_j)] and mean c
                    double ulo = CUDART_INF, uhi = CUDART_INF, sumc = 0.0;
#pragma unroll
                    for (int v = 0; v < 2 * JT; ++v) {
                        const int j = 8 * (v >> 1) + 2 * r4 + (v & 1);
                        if (j < d) {
                            const double isa = __ldg(P.inv_sa + j);
                            ulo = fmin(ulo, (lnK - cv[v]) * isa);
                            uhi = fmin(uhi, (lndK - cv[v]) * isa);
                            sumc += cv[v];
                        }
                    }
                    ulo = quad_min(ulo);
                    uhi = quad_min(uhi);
                    sumc = quad_sum(sumc);
                    double u = fmin(uhi, (lnK - sumc / d) / (sg * P.mean_a));
                    bool conv = false;
#pragma unroll 1
                    for (int it = 0; it < kNewtonMax; ++it) {
                        double S = 0.0, SA = 0.0;
#pragma unroll
                        for (int jt = 0; jt < JT; ++jt) {
                            const int j0 = 8 * jt + 2 * r4;
                            const double aa = (j0 < d) ? __ldg(P.a + j0) : 0.0;
                            const double ab = (j0 + 1 < d) ? __ldg(P.a + j0 + 1) : 0.0;
                            double Ea, Eb;
                            fast_exp_x2(fma(sg * aa, u, cv[2 * jt]), fma(sg * ab, u, cv[2 * jt + 1]), Ea, Eb);
                            Ea = (j0 < d) ? Ea : 0.0;
                            Eb = (j0 + 1 < d) ? Eb : 0.0;
                            S += Ea;
                            SA = fma(aa, Ea, SA);
                            S += Eb;
                            SA = fma(ab, Eb, SA);
                        }
                        S = quad_sum(S);
                        SA = quad_sum(SA);
                        const double h = fast_log(S) - lndK;
                        const double du = h * S / (sg * SA);
                        conv = !valid || fabs(du) <= 1e-13 * fmax(1.0, fabs(u));
                        u = fmin(fmax(u - du, ulo), uhi);
                        if (it + 1 >= kNewtonIt && __all_sync(0xffffffffu, conv)) break;
                    }
                    if (r4 == 0 && valid && !conv) ++unconverged;
                    double Dst = 0.0, Qst = 0.0, Vst = 0.0, sumW = 0.0, sumWv = 0.0;
                    const bool need_arith = P.x1_need_arith[o] != 0;
#pragma unroll
                    for (int jt = 0; jt < JT; ++jt) {
                        const int j0 = 8 * jt + 2 * r4;
                        const double aa = (j0 < d) ? __ldg(P.a + j0) : 0.0;
                        const double ab = (j0 + 1 < d) ? __ldg(P.a + j0 + 1) : 0.0;
                        const double ta = (double)(j0 + 1) * P.t1, tb = ta + P.t1;
                        const double ca = cv[2 * jt], cb2 = cv[2 * jt + 1];
                        const double Ra = (ca - P.lnS0 - P.omega * ta) * P.inv_sigma;
                        const double Rb = (cb2 - P.lnS0 - P.omega * tb) * P.inv_sigma;
                        double Ea, Eb;
                        fast_exp_x2(fma(sg * aa, u, ca), fma(sg * ab, u, cb2), Ea, Eb);
                        Ea = (j0 < d) ? Ea : 0.0;
                        Eb = (j0 + 1 < d) ? Eb : 0.0;
                        Dst = fma(aa, Ea, Dst);
                        Qst = fma(aa * aa, Ea, Qst);
                        Vst = fma(Ea, Ra - sg * ta + aa * u, Vst);
                        Dst = fma(ab, Eb, Dst);
                        Qst = fma(ab * ab, Eb, Qst);
                        Vst = fma(Eb, Rb - sg * tb + ab * u, Vst);
                        if (need_arith) {
                            double wa, wb, Pa, Pb, pa, pb;
                            fast_exp_x2(fma(0.5 * sg * sg * aa, aa, ca), fma(0.5 * sg * sg * ab, ab, cb2), wa, wb);
                            phibar_phi_x2(u - sg * aa, u - sg * ab, Pa, Pb, pa, pb);
                            wa = (j0 < d) ? wa : 0.0;
                            wb = (j0 + 1 < d) ? wb : 0.0;
                            sumW = fma(wa, Pa, sumW);
                            sumWv = fma(wa * (Ra - sg * ta + sg * aa * aa), Pa, sumWv);
                            sumW = fma(wb, Pb, sumW);
                            sumWv = fma(wb * (Rb - sg * tb + sg * ab * ab), Pb, sumWv);
                        }
                    }
                    const X1Sums xs{u, quad_sum(Dst), quad_sum(Qst), quad_sum(Vst), quad_sum(sumW), quad_sum(sumWv)};
#pragma unroll
                    for (int o2 = 0; o2 < kMaxOpt; ++o2)
                        if (o2 < P.n_opt && P.tail_leader[o2] == o) x1_outputs(P, o2, xs, f[o2]);
                }
                if (r4 == 0 && valid) {  // one lane per path records it
                    ++npts;
                    if (P.path_out != nullptr) {
#pragma unroll
                        for (int o = 0; o < kMaxOpt; ++o)
                            if (o == P.hook_option)
                                for (int qq = 0; qq < 4; ++qq) P.path_out[ip * 4 + qq] = f[o][qq];
                    }
#pragma unroll
                    for (int o = 0; o < kMaxOpt; ++o) {
                        if (o < P.n_opt) {
#pragma unroll
                            for (int qq = 0; qq < 4; ++qq) {
                                const double y = f[o][qq] - P.piv[o][qq];
                                double* a1 = accs + (size_t)(o * 8 + qq * 2) * tpb + tp;
                                a1[0] += y;
                                a1[tpb] = fma(y, y, a1[tpb]);
                            }
                        }
                    }
                }
            }
        }
        if (COND == kW1) {
            const W1Acc& w1 = w1own;
            const uint64_t i = i0 + tid + ((uint64_t)a << tpb_log2);
            const bool valid = i < P.n_points;  // all lanes run: the warp reduction needs them
            npts += valid ? 1u : 0u;
            if (valid && P.has_lookback && w1.emax - w1.esec < 1e-12) ++ties;
            double f[kMaxOpt][4];
            tail_w1_all(P, w1, f);
            if (P.path_out != nullptr && valid) {
#pragma unroll
                for (int o = 0; o < kMaxOpt; ++o)
                    if (o == P.hook_option)
                        for (int qq = 0; qq < 4; ++qq) P.path_out[i * 4 + qq] = f[o][qq];
            }
            thread_acc2(f, P, valid, acc2, tpb, tid);
        }
    }
    if (COND == kW1) acc2_to_wacc(P, acc2, wacc, tpb, tid);
    block_epilogue(P, COND == kX1 ? accs : nullptr, wacc, red, n_acc, tpb, tid, cell, unconverged, ties, npts);
}

static size_t pca_smem_bytes(const PathArgs& a) {
    const size_t tpb = (size_t)1 << a.tpb_log2, nw = tpb / 32;
    size_t b = (size_t)a.n_opt * 8 * tpb * sizeof(double);
    b += ((size_t)a.d * 32 * 2 + a.d) * sizeof(uint32_t) + 4;
    const size_t hw = 2 * 2 * nw * a.d * sizeof(uint32_t), red = 4 * 32 * sizeof(double);
    return b + (hw > red ? hw : red);
}

template <int K, int KF>
static cudaError_t launch_pca_t(const PathArgs& args_in, cudaStream_t st) {
    static thread_local int set_for[64] = {0};
    int dev = 0;
    cudaGetDevice(&dev);
    if (set_for[dev & 63] == 0) {
        cudaError_t e = cudaFuncSetAttribute(pca_kernel<K, KF>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
        if (e != cudaSuccess) return e;
        set_for[dev & 63] = 1;
    }
    PathArgs args = args_in;
    int best_lg = -1, best_warps = -1;
    for (int lg = 7; lg >= 5; --lg) {
        args.tpb_log2 = lg;
        const size_t smem = pca_smem_bytes(args);
        if (smem > 200 * 1024) continue;
        int nb = 0;
        if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, pca_kernel<K, KF>, 1 << lg, smem) != cudaSuccess) continue;
        if (nb * (1 << lg) / 32 > best_warps) {
            best_warps = nb * (1 << lg) / 32;
            best_lg = lg;
        }
    }
    if (best_lg < 0) return cudaErrorInvalidConfiguration;
    args.tpb_log2 = best_lg;
    const uint64_t nblocks = args.cell_end - args.cell_begin;
    if (nblocks == 0) return cudaSuccess;
    pca_kernel<K, KF><<<(unsigned)nblocks, 1 << best_lg, pca_smem_bytes(args), st>>>(args);
    ++launch_counter();
    return cudaGetLastError();
}

template <int K>
static cudaError_t launch_pca(const PathArgs& args, cudaStream_t st, bool* handled) {
    *handled = true;
    switch (args.M_ld) {
    case 8: return launch_pca_t<K, 2>(args, st);
    case 16: return launch_pca_t<K, 4>(args, st);
    case 24: return launch_pca_t<K, 6>(args, st);
    case 32: return launch_pca_t<K, 8>(args, st);
    case 40: return launch_pca_t<K, 10>(args, st);
    case 48: return launch_pca_t<K, 12>(args, st);
    case 56: return launch_pca_t<K, 14>(args, st);
    case 64: return launch_pca_t<K, 16>(args, st);
    case 96: return launch_pca_t<K, 24>(args, st);
    case 128: return launch_pca_t<K, 32>(args, st);
    default: *handled = false; return cudaSuccess;
    }
}


// ---------------------------------------------------------------------------
// C5 portfolio kernel: many options on shared points.
//  Phase A (per point): the fragment-native PCA contraction gives W(t_j) for
//    T = 1 once; every (sigma, T) family rescales it (M(T) = sqrt(T) M(1)) and
//    accumulates its S~ statistics (S~_A, I_A, S~_max, I_max), quad-reduced and
//    staged in shared memory.  Exps: families x d per point, shared by all
//    options of a family.
//  Phase B: thread t owns options t, t + tpb, ...; for each it runs only the
//    per-option tail (psi, Phibar, phi, four outputs)
//    over the block's staged points, accumulating in registers.
// ---------------------------------------------------------------------------
constexpr int kStatW = 7;  // staged per (point, family): SA, lnSA, IA, Smax, lnSmax, Imax, near-tie flag

template <int KF>
__global__ void __launch_bounds__(128) portfolio_kernel(const PortfolioArgs P) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    constexpr int DP = 4 * KF;
    constexpr int JT = DP / 8;
    const int tpb_log2 = P.tpb_log2, tpb = 1 << tpb_log2, tid = threadIdx.x, d = P.d;
    const int lane = tid & 31, q = lane >> 2, r4 = lane & 3, wbase = tid & ~31;
    const int nfam = P.n_fam, nopt = P.n_opt;
    const uint64_t cell = P.cell_begin + blockIdx.x;
    const uint32_t rep_local = (uint32_t)(cell / P.cells_per_rep);
    const uint64_t blk = cell % P.cells_per_rep;
    const uint64_t i0 = blk * (uint64_t)kCellPoints;
    const int ppt = kCellPoints >> tpb_log2;
    const int nw = tpb >> 5;
    // smem: acc [8][nopt] | stats [tpb][nfam][kStatW] | vt | sh | G | HW
    double* accs = reinterpret_cast<double*>(smem_raw);
    double* stats = accs + (size_t)8 * nopt;
    uint32_t* vt = reinterpret_cast<uint32_t*>(stats + (size_t)tpb * nfam * kStatW);
    uint32_t* sh = vt + (size_t)d * 32;
    uint32_t* G = sh + d;
    uint32_t* HW = G + (size_t)d * 32;
    HW += ((uintptr_t)HW & 7) ? 1 : 0;
    double* red = reinterpret_cast<double*>(HW);
    const int hw_size = 2 * nw * d;
    const uint64_t K0 = P.point_offset + i0;
    const uint64_t Ab = K0 >> tpb_log2;
    {
        const uint32_t* src = P.vscr + (size_t)rep_local * d * 32;
        for (int idx = tid; idx < d * 32; idx += tpb) vt[idx] = src[idx];
        for (int idx = tid; idx < d; idx += tpb) sh[idx] = P.shift[(size_t)rep_local * d + idx];
        for (int idx = tid; idx < 8 * nopt; idx += tpb) accs[idx] = 0.0;
        __syncthreads();
        sobol_build_g(vt, d, G, tid, tpb);
    }
    unsigned ties = 0, npts = 0;

    for (int a = 0; a < ppt; ++a) {
        if (i0 + ((uint64_t)a << tpb_log2) >= P.n_points) break;  // block-uniform
        uint32_t* HWb = HW + (a & 1) * hw_size;
        sobol_build_hw(vt, P.owen ? nullptr : sh, d, 0, tpb_log2, nw, Ab + (uint64_t)a, HWb, tid, tpb);
        __syncthreads();  // also: every thread has left phase B of the previous point
        // ---- phase A -------------------------------------------------------
#pragma unroll 1
        for (int rt = 0; rt < 4; ++rt) {
            const int tp = wbase + 8 * rt + q;
            const uint64_t kp0 = K0 + (uint64_t)tp;
            const SobolBlock sp{G, HWb, d, nw, (int)(kp0 & 31), (int)((kp0 >> 5) & (uint64_t)(nw - 1)),
                                (int)((kp0 >> tpb_log2) - Ab), P.owen ? sh : nullptr};
            double afr[KF];
#pragma unroll
            for (int f = 0; f < KF; f += 2) {
                const int ja = 4 * f + r4, jb = 4 * (f + 1) + r4;
                double xa, xb;
                normal_from_u32_x2(sp.get(ja < d ? ja : d - 1), sp.get(jb < d ? jb : d - 1), xa, xb);
                afr[f] = ja < d ? xa : 0.0;
                afr[f + 1] = jb < d ? xb : 0.0;
            }
            double cv[2 * JT];
#pragma unroll
            for (int jt = 0; jt < JT; ++jt) {
                double acc0 = 0.0, acc1 = 0.0;
                const double* Mrow = P.M + (size_t)(8 * jt + q) * DP + r4;
#pragma unroll
                for (int f = 0; f < KF; ++f) {
                    const double bfrag = __ldg(Mrow + 4 * f);
                    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                                 : "+d"(acc0), "+d"(acc1)
                                 : "d"(afr[f]), "d"(bfrag));
                }
                cv[2 * jt] = acc0;
                cv[2 * jt + 1] = acc1;
            }
            const double W1v = __shfl_sync(0xffffffffu, cv[0], lane & ~3);
#pragma unroll
            for (int v = 0; v < 2 * JT; ++v) cv[v] -= W1v;  // W~(t_j - t_1) for T = 1
#pragma unroll 1
            for (int fi = 0; fi < nfam; ++fi) {
                const Family& F = P.fam[fi];
                const double sgT = F.sigma * F.sqrtT;  // W~ scales by sqrt(T)
                double sS = 0.0, sI = 0.0, em = -CUDART_INF, es = -CUDART_INF, ym = 0.0;
#pragma unroll
                for (int jt = 0; jt < JT; ++jt) {
                    const int j0 = 8 * jt + 2 * r4;
                    const double ta = (double)j0 * F.t1, tb = ta + F.t1;
                    const double Wa = F.sqrtT * cv[2 * jt], Wb = F.sqrtT * cv[2 * jt + 1];
                    const double ea = fma(sgT, cv[2 * jt], F.omega * ta), eb = fma(sgT, cv[2 * jt + 1], F.omega * tb);
                    double Xa, Xb;
                    fast_exp_x2(ea, eb, Xa, Xb);
                    const double Sa = (j0 < d) ? P.S0 * Xa : 0.0, Sb = (j0 + 1 < d) ? P.S0 * Xb : 0.0;
                    const double ya = fma(-F.sigma, ta, Wa), yb = fma(-F.sigma, tb, Wb);
                    sS += Sa;
                    sI = fma(Sa, ya, sI);
                    sS += Sb;
                    sI = fma(Sb, yb, sI);
                    if (P.has_lookback) {
                        const double eav = (j0 < d) ? ea : -CUDART_INF, ebv = (j0 + 1 < d) ? eb : -CUDART_INF;
                        bool gt = eav > em;
                        es = fmax(es, gt ? em : eav);
                        ym = gt ? ya : ym;
                        em = gt ? eav : em;
                        gt = ebv > em;
                        es = fmax(es, gt ? em : ebv);
                        ym = gt ? yb : ym;
                        em = gt ? ebv : em;
                    }
                }
                sS = quad_sum(sS);
                sI = quad_sum(sI);
                if (P.has_lookback) {
#pragma unroll
                    for (int off = 1; off <= 2; off <<= 1) {
                        const double pe = __shfl_xor_sync(0xffffffffu, em, off);
                        const double pes = __shfl_xor_sync(0xffffffffu, es, off);
                        const double py = __shfl_xor_sync(0xffffffffu, ym, off);
                        const bool take = pe > em;
                        es = fmax(fmax(es, pes), fmin(em, pe));
                        em = take ? pe : em;
                        ym = take ? py : ym;
                    }
                }
                if (r4 == 0) {
                    const double SA = sS / (double)d, Smax = P.has_lookback ? P.S0 * fast_exp(em) : SA;
                    double lnSA, lnSmax;
                    fast_log_x2(SA, Smax, lnSA, lnSmax);
                    double* st = stats + ((size_t)tp * nfam + fi) * kStatW;
                    st[0] = SA;
                    st[1] = lnSA;
                    st[2] = sI / (double)d;
                    st[3] = Smax;
                    st[4] = lnSmax;
                    st[5] = Smax * ym;
                    st[6] = (P.has_lookback && em - es < 1e-12) ? 1.0 : 0.0;
                }
            }
        }
        __syncthreads();
        // ---- phase B -------------------------------------------------------
        const uint64_t ib = i0 + ((uint64_t)a << tpb_log2);
        const int np = (int)((P.n_points - ib) < (uint64_t)tpb ? (P.n_points - ib) : (uint64_t)tpb);
        if (tid < np) ++npts;
#pragma unroll 1
        for (int o = tid; o < nopt; o += tpb) {
            const PortfolioOption op = P.opts[o];
            const Family& F = P.fam[op.family];
            const bool lb = op.type == kLookback, bin = op.type == kBinary;
            const double K = op.K, D = F.Dfac, S0 = P.S0;
            double s1[4] = {0, 0, 0, 0}, s2[4] = {0, 0, 0, 0};
#pragma unroll 1
            for (int pth = 0; pth < np; ++pth) {
                const double* st = stats + ((size_t)pth * nfam + op.family) * kStatW;
                const double stat = lb ? st[3] : st[0];
                const double lnst = lb ? st[4] : st[1];
                const double I = lb ? st[5] : st[2];
                if (lb && st[6] != 0.0) ++ties;
                const double psi = (op.lnK - lnst - F.omega * F.t1) * F.inv_s;
                double Q0, Q1, ph, phs;
                phibar_phi_x2(psi, psi - F.s, Q0, Q1, ph, phs);
                double f[4];
                if (bin) {
                    f[0] = D * Q0;
                    f[1] = D * ph * F.inv_s / S0;
                    f[2] = D * ph * (I * F.inv_s / stat + psi * F.inv_sigma - F.sqrt_t1);
                    f[3] = D * ph * F.inv_s / (S0 * S0) * (psi * F.inv_s - 1.0);
                } else {
                    f[0] = F.Afac * stat * Q1 - D * K * Q0;
                    f[1] = F.Afac * (stat / S0) * Q1;
                    f[2] = F.Afac * Q1 * I + K * D * ph * F.sqrt_t1;
                    f[3] = K * D * ph * F.inv_s / (S0 * S0);
                }
                if (P.path_out != nullptr)
                    for (int qq = 0; qq < 4; ++qq) P.path_out[((ib + pth) * nopt + o) * 4 + qq] = f[qq];
#pragma unroll
                for (int qq = 0; qq < 4; ++qq) {
                    const double y = f[qq] - op.piv[qq];
                    s1[qq] += y;
                    s2[qq] = fma(y, y, s2[qq]);
                }
            }
#pragma unroll
            for (int qq = 0; qq < 4; ++qq) {
                accs[(2 * qq) * nopt + o] += s1[qq];
                accs[(2 * qq + 1) * nopt + o] += s2[qq];
            }
        }
    }
    // ---- epilogue: options are owned by single threads; counters reduced -----
    __syncthreads();
    const int stride = P.partial_stride;
    for (int o = tid; o < nopt; o += tpb)
#pragma unroll
        for (int v = 0; v < 8; ++v) P.partials[(size_t)cell * stride + o * 8 + v] = accs[v * nopt + o];
    unsigned tc = ties, nc = npts;
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
        tc += __shfl_xor_sync(0xffffffffu, tc, off);
        nc += __shfl_xor_sync(0xffffffffu, nc, off);
    }
    if (lane == 0) {
        red[(tid >> 5) * 2 + 0] = (double)tc;
        red[(tid >> 5) * 2 + 1] = (double)nc;
    }
    __syncthreads();
    if (tid == 0) {
        double t = 0.0, n = 0.0;
        for (int w = 0; w < nw; ++w) {
            t += red[w * 2];
            n += red[w * 2 + 1];
        }
        P.partials[(size_t)cell * stride + nopt * 8 + 0] = 0.0;  // Newton: not used (W1)
        P.partials[(size_t)cell * stride + nopt * 8 + 1] = t;
        P.partials[(size_t)cell * stride + nopt * 8 + 2] = n;
    }
}

static size_t portfolio_smem_bytes(const PortfolioArgs& a) {
    const size_t tpb = (size_t)1 << a.tpb_log2, nw = tpb / 32;
    size_t b = (size_t)8 * a.n_opt * sizeof(double) + tpb * a.n_fam * kStatW * sizeof(double);
    b += ((size_t)a.d * 32 * 2 + a.d) * sizeof(uint32_t) + 4;
    const size_t hw = 2 * 2 * nw * a.d * sizeof(uint32_t), red = 4 * 32 * sizeof(double);
    return b + (hw > red ? hw : red);
}

template <int KF>
static cudaError_t launch_portfolio_t(const PortfolioArgs& args_in, cudaStream_t st) {
    static thread_local int set_for[64] = {0};
    int dev = 0;
    cudaGetDevice(&dev);
    if (set_for[dev & 63] == 0) {
        cudaError_t e = cudaFuncSetAttribute(portfolio_kernel<KF>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
        if (e != cudaSuccess) return e;
        set_for[dev & 63] = 1;
    }
    PortfolioArgs args = args_in;
    args.tpb_log2 = 7;  // 128 threads: 4 warps of 32 points, options strided over the block
    const size_t smem = portfolio_smem_bytes(args);
    if (smem > 200 * 1024) return cudaErrorInvalidConfiguration;
    const uint64_t nblocks = args.cell_end - args.cell_begin;
    if (nblocks == 0) return cudaSuccess;
    portfolio_kernel<KF><<<(unsigned)nblocks, 128, smem, st>>>(args);
    ++launch_counter();
    return cudaGetLastError();
}

cudaError_t launch_portfolio(const PortfolioArgs& args, cudaStream_t st) {
    switch (args.M_ld) {
    case 8: return launch_portfolio_t<2>(args, st);
    case 16: return launch_portfolio_t<4>(args, st);
    case 32: return launch_portfolio_t<8>(args, st);
    case 64: return launch_portfolio_t<16>(args, st);
    case 128: return launch_portfolio_t<32>(args, st);
    default: return cudaErrorInvalidValue;
    }
}

static size_t path_smem_bytes(const PathArgs& a, int constr, int cond, int method) {
    const size_t tpb = (size_t)1 << a.tpb_log2, nw = tpb / 32;
    const bool need_buf = method == kQmc && (constr == kPca || cond == kX1);
    const bool two_buf = method == kQmc && constr == kPca && cond == kX1;
    size_t b = 0;
    if (method == kQmc && constr == kPca && cond == kW1) b += (size_t)a.M_ld * (tpb + 8) * sizeof(double);
    else if (need_buf) b += (size_t)a.d * tpb * sizeof(double);
    if (two_buf) b += (size_t)a.d * tpb * sizeof(double);
    size_t hw = 0;
    if (method == kQmc) {
        b += ((size_t)a.d * 32 * 2 + a.d) * sizeof(uint32_t) + 4;  // vt, sh, G, alignment pad
        hw = 2 * 2 * nw * a.d * sizeof(uint32_t);
    }
    const size_t red = 4 * 32 * sizeof(double);
    return b + (hw > red ? hw : red);
}

template <int C, int K, int M>
static cudaError_t launch_paths_t(const PathArgs& args_in, cudaStream_t st, int* smem_out) {
    // raise the dynamic-smem limit once per device (not on every call: it is a driver round trip)
    static thread_local int set_for[64] = {0};
    int dev = 0;
    cudaGetDevice(&dev);
    if (set_for[dev & 63] == 0) {
        cudaError_t e = cudaFuncSetAttribute(paths_kernel<C, K, M>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             200 * 1024);
        if (e != cudaSuccess) return e;
        set_for[dev & 63] = 1;
    }
    // block size: the candidate (128, 64, 32 threads) with the most resident warps per SM
    // (registers and shared memory both counted by the occupancy calculator); a deterministic
    // function of (mode, d, n_opt), so results stay independent of the GPU count.
    PathArgs args = args_in;
    int best_lg = -1, best_warps = -1;
    for (int lg = 7; lg >= 5; --lg) {
        args.tpb_log2 = lg;
        const size_t smem = path_smem_bytes(args, C, K, M);
        if (smem > 200 * 1024) continue;
        int nb = 0;
        if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, paths_kernel<C, K, M>, 1 << lg, smem) != cudaSuccess)
            continue;
        const int warps = nb * (1 << lg) / 32;
        if (warps > best_warps) {
            best_warps = warps;
            best_lg = lg;
        }
    }
    if (best_lg < 0) return cudaErrorInvalidConfiguration;
    args.tpb_log2 = best_lg;
    const size_t smem = path_smem_bytes(args, C, K, M);
    if (smem_out) *smem_out = (int)smem;
    const uint64_t nblocks = args.cell_end - args.cell_begin;
    if (nblocks == 0) return cudaSuccess;
    paths_kernel<C, K, M><<<(unsigned)nblocks, 1 << args.tpb_log2, smem, st>>>(args);
    ++launch_counter();
    return cudaGetLastError();
}

cudaError_t launch_paths(const PathArgs& args, int construction, int conditioning, int method, cudaStream_t st,
                         int* smem_out) {
    if (method == kLr) return launch_paths_t<kStd, kW1, kLr>(args, st, smem_out);
    if (method == kMc) return construction == kBB ? launch_paths_t<kBB, kW1, kMc>(args, st, smem_out)
                                                  : launch_paths_t<kStd, kW1, kMc>(args, st, smem_out);
    if (method == kMcAv) return construction == kBB ? launch_paths_t<kBB, kW1, kMcAv>(args, st, smem_out)
                                                    : launch_paths_t<kStd, kW1, kMcAv>(args, st, smem_out);
    if (construction == kPca && method == kQmc && !(conditioning == kX1 && args.has_lookback)) {
        // fragment-native tensor-core path for d <= 128 (the X1 lookback walks its envelope per thread)
        bool handled = false;
        cudaError_t e = conditioning == kW1 ? launch_pca<kW1>(args, st, &handled) : launch_pca<kX1>(args, st, &handled);
        if (handled) return e;
    }
    if (conditioning == kW1) {
        if (construction == kStd) return launch_paths_t<kStd, kW1, kQmc>(args, st, smem_out);
        if (construction == kBB) return launch_paths_t<kBB, kW1, kQmc>(args, st, smem_out);
        return launch_paths_t<kPca, kW1, kQmc>(args, st, smem_out);
    }
    if (construction == kStd) return launch_paths_t<kStd, kX1, kQmc>(args, st, smem_out);
    if (construction == kBB) return launch_paths_t<kBB, kX1, kQmc>(args, st, smem_out);
    return launch_paths_t<kPca, kX1, kQmc>(args, st, smem_out);
}

// ---------------------------------------------------------------------------
// (a8) per-replicate reduction over cells, fixed sequential order (so that a
// multi-GPU all-reduced partial buffer reduces to identical bits).
// ---------------------------------------------------------------------------
__global__ void reduce_cells_kernel(const double* __restrict__ partials, int stride, uint32_t rep_begin,
                                    uint32_t cells_per_rep, double* __restrict__ rep_sums) {
    const uint32_t rep = rep_begin + blockIdx.x;
    for (int t = threadIdx.x; t < stride; t += blockDim.x) {  // rows can be long (portfolio: 8 n_opt + 3)
        const double* p = partials + (size_t)rep * cells_per_rep * stride + t;
        double s = 0.0;
        for (uint32_t c = 0; c < cells_per_rep; ++c) s += p[(size_t)c * stride];
        rep_sums[(size_t)rep * stride + t] = s;
    }
}

cudaError_t launch_reduce_cells(const double* d_partials, int stride, uint32_t rep_begin, uint32_t rep_end,
                                uint32_t cells_per_rep, double* d_rep_sums, cudaStream_t st) {
    if (rep_end <= rep_begin) return cudaSuccess;
    const int threads = stride <= 32 ? 32 : 256;
    reduce_cells_kernel<<<rep_end - rep_begin, threads, 0, st>>>(d_partials, stride, rep_begin, cells_per_rep,
                                                                 d_rep_sums);
    ++launch_counter();
    return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// Parity hooks: the same SobolBlock / normal code the path kernel runs.
// One block of 128 threads walks 4096 points of [k_begin, k_end) like a cell.
// ---------------------------------------------------------------------------
struct HookSmem {
    uint32_t *vt, *sh, *G, *HW;
};
__device__ __forceinline__ HookSmem hook_setup(unsigned char* raw, const uint32_t* vscr, const uint32_t* shift, int d,
                                               int tid, int tpb) {
    HookSmem h;
    h.vt = reinterpret_cast<uint32_t*>(raw);
    h.sh = h.vt + (size_t)d * 32;
    h.G = h.sh + d;
    h.HW = h.G + (size_t)d * 32;
    for (int idx = tid; idx < d * 32; idx += tpb) h.vt[idx] = vscr[idx];
    for (int idx = tid; idx < d; idx += tpb) h.sh[idx] = shift[idx];
    __syncthreads();
    sobol_build_g(h.vt, d, h.G, tid, tpb);
    return h;
}

__global__ void sobol_hook_kernel(const uint32_t* __restrict__ vscr, const uint32_t* __restrict__ shift, int d,
                                  uint32_t dim_begin, uint32_t dim_end, uint64_t k_begin, uint64_t k_end, int owen,
                                  uint32_t* __restrict__ out) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int tpb_log2 = 7, tpb = 128, tid = threadIdx.x, nw = 4;
    HookSmem h = hook_setup(smem_raw, vscr, shift, d, tid, tpb);
    const uint64_t nk = k_end - k_begin;
    const uint64_t K0 = k_begin + (uint64_t)blockIdx.x * kCellPoints;
    const uint64_t Ab = K0 >> tpb_log2, kt = K0 + tid;
    SobolBlock sob{h.G, h.HW, d, nw, (int)(kt & 31), (int)((kt >> 5) & 3), (int)((kt >> tpb_log2) - Ab),
                   owen ? h.sh : nullptr};
    for (int a = 0; a < kCellPoints / tpb; ++a) {
        if (K0 + ((uint64_t)a << tpb_log2) >= k_end) break;
        uint32_t* HWb = h.HW + (a & 1) * 2 * nw * d;
        sobol_build_hw(h.vt, owen ? nullptr : h.sh, d, 0, tpb_log2, nw, Ab + (uint64_t)a, HWb, tid, tpb);
        __syncthreads();
        sob.HW = HWb;
        const uint64_t k = K0 + tid + ((uint64_t)a << tpb_log2);
        if (k >= k_end) continue;
        for (uint32_t j = dim_begin; j < dim_end; ++j) out[(size_t)(j - dim_begin) * nk + (k - k_begin)] = sob.get(j);
    }
}

__global__ void normals_hook_kernel(const uint32_t* __restrict__ vscr, const uint32_t* __restrict__ shift, int d,
                                    uint64_t k_begin, uint64_t k_end, int method, uint64_t seed, uint32_t rep,
                                    int owen, double* __restrict__ out) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int tpb_log2 = 7, tpb = 128, tid = threadIdx.x, nw = 4;
    const uint64_t K0 = k_begin + (uint64_t)blockIdx.x * kCellPoints;
    if (method != kQmc) {  // LR+MC, MC-CPW, MC+AV-CPW: the Philox stream
        for (int a = 0; a < kCellPoints / tpb; ++a) {
            const uint64_t k = K0 + tid + ((uint64_t)a << tpb_log2);
            if (k >= k_end) break;
            for (int jq = 0; jq < d; jq += 4) {
                uint32_t c[4] = {(uint32_t)k, (uint32_t)(k >> 32), (uint32_t)(jq >> 2), (rep << 8) | 0x02u};
                philox4x32_10(c, (uint32_t)seed, (uint32_t)(seed >> 32));
                double xs[4];
                normal_from_u32_x2(c[0], c[1], xs[0], xs[1]);
                normal_from_u32_x2(c[2], c[3], xs[2], xs[3]);
                for (int w = 0; w < 4 && jq + w < d; ++w) out[(k - k_begin) * d + jq + w] = xs[w];
            }
        }
        return;
    }
    HookSmem h = hook_setup(smem_raw, vscr, shift, d, tid, tpb);
    const uint64_t Ab = K0 >> tpb_log2, kt = K0 + tid;
    SobolBlock sob{h.G, h.HW, d, nw, (int)(kt & 31), (int)((kt >> 5) & 3), (int)((kt >> tpb_log2) - Ab),
                   owen ? h.sh : nullptr};
    for (int a = 0; a < kCellPoints / tpb; ++a) {
        if (K0 + ((uint64_t)a << tpb_log2) >= k_end) break;
        uint32_t* HWb = h.HW + (a & 1) * 2 * nw * d;
        sobol_build_hw(h.vt, owen ? nullptr : h.sh, d, 0, tpb_log2, nw, Ab + (uint64_t)a, HWb, tid, tpb);
        __syncthreads();
        sob.HW = HWb;
        const uint64_t k = K0 + tid + ((uint64_t)a << tpb_log2);
        if (k >= k_end) continue;
        int j = 0;
        for (; j + 1 < d; j += 2) {
            double xa, xb;
            normal_from_u32_x2(sob.get(j), sob.get(j + 1), xa, xb);
            out[(k - k_begin) * d + j] = xa;
            out[(k - k_begin) * d + j + 1] = xb;
        }
        if (j < d) out[(k - k_begin) * d + j] = normal_from_u32(sob.get(j));
    }
}

cudaError_t launch_sobol_hook(const uint32_t* d_vscr, const uint32_t* d_shift, int d, uint32_t dim_begin,
                              uint32_t dim_end, uint64_t k_begin, uint64_t k_end, int owen, uint32_t* d_out,
                              cudaStream_t st) {
    const uint64_t nk = k_end - k_begin;
    const unsigned grid = (unsigned)((nk + kCellPoints - 1) / kCellPoints);
    const size_t smem = ((size_t)d * 64 + d + 2 * 2 * 4 * d) * 4;
    cudaError_t e = cudaFuncSetAttribute(sobol_hook_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    sobol_hook_kernel<<<grid, 128, smem, st>>>(d_vscr, d_shift, d, dim_begin, dim_end, k_begin, k_end, owen, d_out);
    ++launch_counter();
    return cudaGetLastError();
}

cudaError_t launch_normals_hook(const uint32_t* d_vscr, const uint32_t* d_shift, int d, uint64_t k_begin,
                                uint64_t k_end, int method, uint64_t seed, uint32_t rep, int owen, double* d_out,
                                cudaStream_t st) {
    const uint64_t nk = k_end - k_begin;
    const unsigned grid = (unsigned)((nk + kCellPoints - 1) / kCellPoints);
    const size_t smem = method != kQmc ? 0 : ((size_t)d * 64 + d + 2 * 2 * 4 * d) * 4;
    cudaError_t e =
        cudaFuncSetAttribute(normals_hook_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    normals_hook_kernel<<<grid, 128, smem, st>>>(d_vscr, d_shift, d, k_begin, k_end, method, seed, rep, owen, d_out);
    ++launch_counter();
    return cudaGetLastError();
}

}  // namespace qmccpw
