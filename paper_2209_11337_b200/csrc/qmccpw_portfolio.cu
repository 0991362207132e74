// qmccpw_portfolio.cu -- the C5 portfolio kernel (1024 options on shared paths).
#include "qmccpw_device.cuh"

namespace qmccpw {

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

template <int KF, bool OWEN>
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
        sobol_build_hw(vt, OWEN ? nullptr : sh, d, 0, tpb_log2, nw, Ab + (uint64_t)a, HWb, tid, tpb);
        __syncthreads();  // also: every thread has left phase B of the previous point
        // ---- phase A -------------------------------------------------------
#pragma unroll 1
        for (int rt = 0; rt < 4; ++rt) {
            const int tp = wbase + 8 * rt + q;
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
