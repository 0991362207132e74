// qmccpw_portfolio.cu -- the C5 portfolio kernel (1024 options on shared paths).
#ifndef QMCCPW_PF_EXP256
#define QMCCPW_PF_EXP256 1  // measured: C5 61.95 -> 61.73 ms
#endif
#ifndef QMCCPW_EXP256
#define QMCCPW_EXP256 QMCCPW_PF_EXP256  // 256-entry exp table through L1 (qmccpw_math.cuh)
#endif
#include "qmccpw_device.cuh"

namespace qmccpw {

// ---------------------------------------------------------------------------
// C5 portfolio kernel: many options on shared points.
//  Phase A (per point): the fragment-native PCA contraction gives W(t_j) for
//    T = 1 once; every (sigma, T) family rescales it (M(T) = sqrt(T) M(1)) and
//    accumulates its S~ statistics (S~_A, I_A, S~_max, I_max), quad-reduced and
//    staged in shared memory.  Exps: families x d per point, shared by all
//    options of a family.
//  Phase B: thread t owns options t, t + tpb, ...; it runs two of them at a time
//    (independent chains for ILP) through the per-option tail (psi, Phibar, phi,
//    four outputs) over the block's staged points, with
//    per-option constants instead of divisions, accumulating in registers and
//    then into the cell's partial row in global memory (read-modify-write by the
//    owning thread only: deterministic, and no 64 KB of per-option smem, so two
//    blocks fit per SM).
// ---------------------------------------------------------------------------
constexpr int kStatW = 8;  // staged per (point, family): SA, lnSA, IA, IA/SA, Smax, lnSmax, Imax/Smax, near-tie flag

template <int KF, bool OWEN>
__global__ void __launch_bounds__(128, 3) portfolio_kernel(const PortfolioArgs P) {  // 3 blocks: 72.5 KB smem each
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
    // smem: stats [tpb/2][nfam][kStatW] | vt | sh | G | HW
    double* stats = reinterpret_cast<double*>(smem_raw);  // [tpb/2 slots][nfam][kStatW]
    double* prow = P.partials + (size_t)cell * P.partial_stride;  // this cell's row: [nopt][8] + 3 counters
    const double inv_d = 1.0 / (double)d;
    uint32_t* vt = reinterpret_cast<uint32_t*>(stats + (size_t)(tpb / 2) * nfam * kStatW);
    uint32_t* sh = vt + (size_t)d * 32;
    uint32_t* G = sh + d;
    uint32_t* HW = G + (size_t)d * 32;
    HW += ((uintptr_t)HW & 7) ? 1 : 0;
    double* red = reinterpret_cast<double*>(HW);
    const int hw_size = 2 * nw * d;
    const uint64_t K0 = P.point_offset + i0;
    const uint64_t Ab = K0 >> tpb_log2;
    {
        math_tables_load(tid, tpb);
        const uint32_t* src = P.vscr + (size_t)rep_local * d * 32;
        QMCCPW_CHECK(rep_local < P.n_reps && cell < P.cell_end);
        for (int idx = tid; idx < d * 32; idx += tpb) {
            QMCCPW_CHK_SMEM(&vt[idx]);
            vt[idx] = src[idx];
        }
        for (int idx = tid; idx < d; idx += tpb) {
            QMCCPW_CHK_SMEM(&sh[idx]);
            sh[idx] = P.shift[(size_t)rep_local * d + idx];
        }
        for (int o = tid; o < nopt; o += tpb)  // zeroed by the thread that will own the option
#pragma unroll
            for (int v = 0; v < 8; ++v) prow[o * 8 + v] = 0.0;
        __syncthreads();
        sobol_build_g(vt, d, G, tid, tpb);
    }
    unsigned ties = 0, npts = 0;

    for (int a = 0; a < ppt; ++a) {
        if (i0 + ((uint64_t)a << tpb_log2) >= P.n_points) break;  // block-uniform
        uint32_t* HWb = HW + (a & 1) * hw_size;
        sobol_build_hw(vt, OWEN ? nullptr : sh, d, 0, tpb_log2, nw, Ab + (uint64_t)a, HWb, tid, tpb);  // (the incremental build measured slower here: 72.6 vs 77.9 ms)
        __syncthreads();  // also: every thread has left phase B of the previous point
        const uint64_t ib = i0 + ((uint64_t)a << tpb_log2);
        const int np = (int)((P.n_points - ib) < (uint64_t)tpb ? (P.n_points - ib) : (uint64_t)tpb);
        if (tid < np) ++npts;
        // two halves of 64 points (row tiles 0-1, then 2-3 of every warp): half the staged
        // statistics, so three blocks fit per SM
#pragma unroll 1
        for (int half = 0; half < 2; ++half) {
        // ---- phase A -------------------------------------------------------
#pragma unroll 1
        for (int rt = 2 * half; rt < 2 * half + 2; ++rt) {
            const int tp = wbase + 8 * rt + q;
            const int slot = (wbase >> 1) + 8 * (rt - 2 * half) + q;  // 16 per warp per half
            const uint64_t kp0 = K0 + (uint64_t)tp;
            const SobolBlock sp{G, HWb, d, nw, (int)(kp0 & 31), (int)((kp0 >> 5) & (uint64_t)(nw - 1)),
                                (int)((kp0 >> tpb_log2) - Ab), OWEN ? sh : nullptr};
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
                    const double SA = sS * inv_d, Smax = P.has_lookback ? P.S0 * fast_exp(em) : SA;
                    double lnSA, lnSmax;
                    fast_log_x2(SA, Smax, lnSA, lnSmax);
                    double* st = stats + ((size_t)slot * nfam + fi) * kStatW;
                    QMCCPW_CHK_SMEM(&st[7]);
                    st[0] = SA;
                    st[1] = lnSA;
                    st[2] = sI * inv_d;
                    st[3] = sI / sS;  // I_A / S~_A (binary vega)
                    st[4] = Smax;
                    st[5] = lnSmax;
                    st[6] = ym;  // I_max / S~_max (lookback vega)
                    st[7] = (P.has_lookback && em - es < 1e-12) ? 1.0 : 0.0;
                }
            }
        }
        __syncthreads();
        // ---- phase B -------------------------------------------------------
        // per-option constants (P:396-414, P:544-600 with the divisions hoisted).  Calls
        // (arithmetic, lookback) use A S~ phi(psi - s) = D K phi(psi) (psi = (ln K - ln S~ -
        // omega t_1)/s, omega + sigma^2/2 = r), so A S~ Phibar(psi - s) is D K phi(psi) R(psi - s)
        // for psi >= s and A S~ - D K phi(psi) R(s - psi) below, R the Mills ratio: one phi per
        // option and point instead of two; vega takes I/S~ from the staged statistics.  The
        // binary call needs Phibar(psi) alone.  The option table is ordered by type, so a warp
        // runs one type (one Mills pair for two binaries, four otherwise).
        struct OptC {
            const double* st;  // stats of the option's family, point 0
            int lb, bin, slot;
            double c_lnK, c_s, inv_s, K, D, DK, Afac, sqrt_t1, inv_sigma, inv_S0, c1, c3;
            double piv[4];
        };
        auto load_opt = [&](int o, OptC& c) {
            const PortfolioOption op = P.opts[o];
            const Family& F = P.fam[op.family];
            const double inv_S0 = 1.0 / P.S0;
            c.st = stats + (size_t)op.family * kStatW;
            c.lb = op.type == kLookback;
            c.bin = op.type == kBinary;
            c.slot = op.slot;
            c.c_lnK = op.lnK - F.omega * F.t1;
            c.c_s = F.s;
            c.inv_s = F.inv_s;
            c.K = op.K;
            c.D = F.Dfac;
            c.DK = F.Dfac * op.K;
            c.Afac = F.Afac;
            c.sqrt_t1 = F.sqrt_t1;
            c.inv_sigma = F.inv_sigma;
            c.inv_S0 = inv_S0;
            c.c1 = F.Dfac * F.inv_s * inv_S0;                                                // binary delta factor
            c.c3 = (c.bin ? F.Dfac : op.K * F.Dfac) * F.inv_s * inv_S0 * inv_S0;            // gamma factor
            for (int qq = 0; qq < 4; ++qq) c.piv[qq] = op.piv[qq];
        };
        // one point of one option: R0 = R(|psi|), R1 = R(|psi - s|), ph = phi(psi)
        auto tail = [&](const OptC& c, const double* st, double psi, double R0, double R1, double ph, double f[4]) {
            const double q0 = ph * R0;
            const double Q0 = psi >= 0.0 ? q0 : MC.one - q0;
            if (c.bin) {
                f[0] = c.D * Q0;
                f[1] = c.c1 * ph;
                f[2] = c.D * ph * (st[3] * c.inv_s + psi * c.inv_sigma - c.sqrt_t1);
                f[3] = c.c3 * ph * (psi * c.inv_s - 1.0);
            } else {
                const double stat = c.lb ? st[4] : st[0], IoS = c.lb ? st[6] : st[3];  // I / S~
                const double g1 = c.DK * ph * R1;
                const double AQ1S = (psi - c.c_s >= 0.0) ? g1 : c.Afac * stat - g1;  // A S~ Phibar(psi - s)
                f[0] = AQ1S - c.DK * Q0;
                f[1] = AQ1S * c.inv_S0;
                f[2] = AQ1S * IoS + c.K * c.D * ph * c.sqrt_t1;
                f[3] = c.c3 * ph;
            }
        };
        const int fstride = nfam * kStatW;  // stats stride between points
#pragma unroll 1
        for (int o = tid; o < nopt; o += 2 * tpb) {
            const int o2 = o + tpb;
            const bool two = o2 < nopt;
            OptC A, B;
            load_opt(o, A);
            load_opt(two ? o2 : o, B);
            const bool bins = A.bin && B.bin;
            double s1a[4] = {0, 0, 0, 0}, s2a[4] = {0, 0, 0, 0}, s1b[4] = {0, 0, 0, 0}, s2b[4] = {0, 0, 0, 0};
#pragma unroll 1
            for (int sl = 0; sl < 64; ++sl) {
                const int pth = 32 * (sl >> 4) + 8 * (2 * half + ((sl >> 3) & 1)) + (sl & 7);  // block slot
                if (pth >= np) continue;  // ragged last iteration (block-uniform)
                const double* sa = A.st + (size_t)sl * fstride;
                const double* sb = B.st + (size_t)sl * fstride;
                if (A.lb && sa[7] != 0.0) ++ties;
                if (two && B.lb && sb[7] != 0.0) ++ties;
                const double psia = (A.c_lnK - (A.lb ? sa[5] : sa[1])) * A.inv_s;
                const double psib = (B.c_lnK - (B.lb ? sb[5] : sb[1])) * B.inv_s;
                double R[4];
                if (bins) {
                    mills_x2(psia, psib, R[0], R[2]);
                    R[1] = R[3] = 0.0;
                } else {
                    const double xq[4] = {psia, psia - A.c_s, psib, psib - B.c_s};
                    mills_x4(xq, R);
                }
                double pha, phb;
                phi_x2(psia, psib, pha, phb);
                double fa[4], fb[4];
                tail(A, sa, psia, R[0], R[1], pha, fa);
                tail(B, sb, psib, R[2], R[3], phb, fb);
                if (P.path_out != nullptr) {
#pragma unroll
                    for (int qq = 0; qq < 4; ++qq) P.path_out[((ib + pth) * nopt + A.slot) * 4 + qq] = fa[qq];
                    if (two)
#pragma unroll
                        for (int qq = 0; qq < 4; ++qq) P.path_out[((ib + pth) * nopt + B.slot) * 4 + qq] = fb[qq];
                }
#pragma unroll
                for (int qq = 0; qq < 4; ++qq) {
                    const double ya = fa[qq] - A.piv[qq], yb = fb[qq] - B.piv[qq];
                    s1a[qq] += ya;
                    s2a[qq] = fma(ya, ya, s2a[qq]);
                    s1b[qq] += yb;
                    s2b[qq] = fma(yb, yb, s2b[qq]);
                }
            }
#pragma unroll
            for (int qq = 0; qq < 4; ++qq) {
                prow[A.slot * 8 + 2 * qq] += s1a[qq];
                prow[A.slot * 8 + 2 * qq + 1] += s2a[qq];
            }
            if (two) {
#pragma unroll
                for (int qq = 0; qq < 4; ++qq) {
                    prow[B.slot * 8 + 2 * qq] += s1b[qq];
                    prow[B.slot * 8 + 2 * qq + 1] += s2b[qq];
                }
            }
        }
        __syncthreads();  // phase B done before the next half's phase A overwrites the stats
        }  // half
    }
    // ---- epilogue: option sums are already in the row; counters reduced -----
    __syncthreads();
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
        prow[nopt * 8 + 0] = 0.0;  // Newton: not used (W1)
        prow[nopt * 8 + 1] = t;
        prow[nopt * 8 + 2] = n;
    }
}

static size_t portfolio_smem_bytes(const PortfolioArgs& a) {
    const size_t tpb = (size_t)1 << a.tpb_log2, nw = tpb / 32;
    size_t b = (tpb / 2) * a.n_fam * kStatW * sizeof(double);  // one half (64 points) staged at a time
    b += ((size_t)a.d * 32 * 2 + a.d) * sizeof(uint32_t) + 4;
    const size_t hw = 2 * 2 * nw * a.d * sizeof(uint32_t), red = 4 * 32 * sizeof(double);
    return b + (hw > red ? hw : red);
}

template <int KF, bool OW>
static cudaError_t launch_portfolio_t(const PortfolioArgs& args_in, cudaStream_t st) {
    static thread_local int set_for[64] = {0};
    int dev = 0;
    cudaGetDevice(&dev);
    if (set_for[dev & 63] == 0) {
        cudaError_t e = cudaFuncSetAttribute(portfolio_kernel<KF, OW>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
        if (e != cudaSuccess) return e;
        set_for[dev & 63] = 1;
    }
    PortfolioArgs args = args_in;
    args.tpb_log2 = 7;  // 128 threads: 4 warps of 32 points, options strided over the block
    const size_t smem = portfolio_smem_bytes(args);
    if (smem > 200 * 1024) return cudaErrorInvalidConfiguration;
    const uint64_t nblocks = args.cell_end - args.cell_begin;
    if (nblocks == 0) return cudaSuccess;
    portfolio_kernel<KF, OW><<<(unsigned)nblocks, 128, smem, st>>>(args);
    ++launch_counter();
    return cudaGetLastError();
}

cudaError_t launch_portfolio(const PortfolioArgs& args, cudaStream_t st) {
    switch (args.M_ld) {
    case 8: return args.owen ? launch_portfolio_t<2, true>(args, st) : launch_portfolio_t<2, false>(args, st);
    case 16: return args.owen ? launch_portfolio_t<4, true>(args, st) : launch_portfolio_t<4, false>(args, st);
    case 32: return args.owen ? launch_portfolio_t<8, true>(args, st) : launch_portfolio_t<8, false>(args, st);
    case 64: return args.owen ? launch_portfolio_t<16, true>(args, st) : launch_portfolio_t<16, false>(args, st);
    case 128: return args.owen ? launch_portfolio_t<32, true>(args, st) : launch_portfolio_t<32, false>(args, st);
    default: return cudaErrorInvalidValue;
    }
}

}  // namespace qmccpw
