// qmccpw_pca.cuh -- PCA paths on the FP64 tensor cores (fragment-native DMMA) and
// its launcher templates; instantiated by qmccpw_pca_w1.cu and qmccpw_pca_x1.cu.
#pragma once
#include "qmccpw_device.cuh"

namespace qmccpw {

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
#ifndef QMCCPW_PCA_W1_MINB
#define QMCCPW_PCA_W1_MINB 8
#endif
// W1: per-warp reduce-scatter of the centred sums (warp_slot_sums, no per-thread smem
// accumulators: 24.6 KB less shared memory per block at 3 options) instead of the per-thread
// (S1, S2) pairs, so more blocks fit.  A/B on one B200, C4 PCA-W1 (ms/step): per-thread pairs
// at 4 blocks/SM 50.63; warp sums at 4 / 5 / 6 / 7 / 8 blocks/SM 50.50 / 47.34 / 46.87 / 46.63
// / 46.54 (8: 64 registers, 344 B of spills to L1) -- profiles/r02/ab_*
#ifndef QMCCPW_PCA_WARPSUM
#define QMCCPW_PCA_WARPSUM 1
#endif
#ifndef QMCCPW_LB_QUAD
#define QMCCPW_LB_QUAD 1
#endif
// quad-walk lookback kernel: A/B on one B200, C4 PCA-X1 with the lookback (ms/step): per-lane
// hull 202.0; quad walk at 3 / 4 / 5 blocks/SM 230.5 / 207.0 / 192.8 (scans from the first line
// beyond the active one)
#ifndef QMCCPW_LB_MINB
#define QMCCPW_LB_MINB 5
#endif
// A/B on one B200, C4 PCA-X1 / BB-X1 (ms/step): rolled 91.5 / 91.5; unrolled by 2 90.5 / 90.5;
// by 4 95.7 / 96.1
#ifndef QMCCPW_LB_UNROLL
#define QMCCPW_LB_UNROLL 1
#endif
#ifndef QMCCPW_X1_UNROLL
#define QMCCPW_X1_UNROLL 2
#endif
#ifndef QMCCPW_PCA_X1_SMEMC
#define QMCCPW_PCA_X1_SMEMC 1
#endif
#ifndef QMCCPW_PCA_X1_MINB
#define QMCCPW_PCA_X1_MINB 5
#endif
// d <= 64: shared memory allows 5 blocks/SM, so cap registers to match (measured on C4:
// PCA-W1 72.4 -> 69.4 ms, PCA-X1 175 -> 165 ms); larger d is smem-limited anyway
// (with a lookback the [d][32] per-warp staging allows 2 blocks/SM at d = 64: registers are free)
template <int COND, int KF, bool LB>
constexpr int pca_min_blocks() {
    return KF > 16 ? 0
                   : (LB ? (QMCCPW_LB_QUAD ? QMCCPW_LB_MINB : 2) : (COND == kW1 ? QMCCPW_PCA_W1_MINB : QMCCPW_PCA_X1_MINB));
}
// byte offset of the X1 lookback staging: accs [n_acc][tpb] | vt, sh, G (+ pad) | HW / red
// W1 only: the date table (date_table_fill) first.  Not for X1: its 1 KB took PCA-X1 past the
// 196 KiB shared-memory carveout at 5 blocks/SM (228 KiB: L1 hit rate 94 -> 76 %, PCA-X1
// 87.8 -> 90.7 ms, the lookback 193 -> 203.5 ms)
__host__ __device__ __forceinline__ size_t pca_date_table_bytes(bool w1, int d) { return w1 ? (size_t)d * 16 : 0; }
// QMCCPW_PCA_VT_GLOBAL: the replicate's scrambled direction numbers are read where they are
// (global memory, L1) instead of a [d][32] shared copy: they are touched only by the table
// builds (sobol_build_g once, ~4 words per dimension per 128 points in sobol_build_hw_inc), and
// the 8 KB per block moves the PCA kernels to a smaller shared-memory carveout (more L1 for M)
#ifndef QMCCPW_PCA_VT_GLOBAL
#define QMCCPW_PCA_VT_GLOBAL 1
#endif
__host__ __device__ __forceinline__ size_t pca_stage_offset(int n_acc, int d, int tpb, bool w1) {
    const size_t nw = (size_t)tpb / 32;
    size_t b = pca_date_table_bytes(w1, d);
    b += (size_t)n_acc * tpb * sizeof(double);
    b += ((size_t)d * 32 * (QMCCPW_PCA_VT_GLOBAL ? 1 : 2) + d) * sizeof(uint32_t) + 4;
    const size_t hw = (2 * 2 * nw * d + d) * sizeof(uint32_t), red = 4 * 32 * sizeof(double);
    b += hw > red ? hw : red;
    return (b + 7) & ~(size_t)7;
}
// (X1 lookback with the per-lane hull: slopes and hulls in shared memory measured slower --
// 215.5 -> 234.1 / 300.3 ms -- bank conflicts of divergent reads and an occupancy step; removed.)
// LB (X1 only): the launch has a lookback option (staging + per-lane envelope walk)
template <int COND, int KF, bool OWEN, bool LB>
__global__ void __launch_bounds__(128, pca_min_blocks<COND, KF, LB>()) pca_kernel(const PathArgs P) {
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
    // X1 without a lookback (QMCCPW_PCA_X1_SMEMC): the lane's c_j go to shared memory after the
    // contraction and the per-strike passes loop over them rolled (small code, 32 registers
    // freed); the centred sums are warp-reduced like W1's
    // X1 lookback by a quad-cooperative envelope walk (QMCCPW_LB_QUAD, x1_lookback_quad): the
    // c_j stay in the quad layout (shared memory, as kSmemC), no per-warp [d][32] staging
    constexpr bool kLbQuad = COND == kX1 && LB && QMCCPW_LB_QUAD && QMCCPW_PCA_X1_SMEMC;
    constexpr bool kSmemC = COND == kX1 && (!LB || kLbQuad) && QMCCPW_PCA_X1_SMEMC;
    constexpr int kXU = kSmemC ? (LB ? QMCCPW_LB_UNROLL : QMCCPW_X1_UNROLL) : 2 * JT;  // unroll of the X1 per-date loops
    constexpr bool kWarpSum = (COND == kW1 && QMCCPW_PCA_WARPSUM) || kSmemC;
    const int n_acc_smem = kWarpSum ? 0 : n_acc;  // smem accumulator rows
    // per-path accumulators in smem: X1 as scalars (one quad lane per path), W1 as (S1, S2) pairs
    double2* tt = reinterpret_cast<double2*>(smem_raw);  // [d] date table (omega t, sigma t)
    double* accs = reinterpret_cast<double*>(smem_raw + pca_date_table_bytes(COND == kW1, d));
    double2* acc2 = reinterpret_cast<double2*>(accs);
#if QMCCPW_PCA_VT_GLOBAL
    const uint32_t* vt = P.vscr + (size_t)rep_local * d * 32;
    uint32_t* sh = reinterpret_cast<uint32_t*>(accs + (size_t)n_acc_smem * tpb);
#else
    uint32_t* vt = reinterpret_cast<uint32_t*>(accs + (size_t)n_acc_smem * tpb);
    uint32_t* sh = vt + (size_t)d * 32;
#endif
    uint32_t* G = sh + d;
    uint32_t* HW = G + (size_t)d * 32;
    HW += ((uintptr_t)HW & 7) ? 1 : 0;
    double* red = reinterpret_cast<double*>(HW);
    const int hw_size = 2 * nw * d;
    uint32_t* BS = HW + 2 * hw_size;  // [d] incremental Gray bases (sobol_build_hw_inc)
    // X1 with a lookback: c_j of the warp's 32 paths staged [d][32] per warp, so that each lane
    // walks the upper envelope of its own path (the quad layout holds a path over 4 lanes)
    double* stage_base = reinterpret_cast<double*>(smem_raw + pca_stage_offset(n_acc_smem, d, tpb, COND == kW1));
    double* stage = stage_base + (size_t)(tid >> 5) * d * 32;
    double* cst = stage_base + tid;  // kSmemC: c_j of this lane at [v][tpb], v < 2 JT
    const uint64_t K0 = P.point_offset + i0;
    const uint64_t Ab = K0 >> tpb_log2;
    {
        math_tables_load(tid, tpb);
        if (COND == kW1) date_table_fill(P, tt, tid, tpb);
        QMCCPW_CHECK(rep_local < P.n_reps && cell < P.cell_end);
#if !QMCCPW_PCA_VT_GLOBAL
        const uint32_t* src = P.vscr + (size_t)rep_local * d * 32;
        for (int idx = tid; idx < d * 32; idx += tpb) {
            QMCCPW_CHK_SMEM(&vt[idx]);
            vt[idx] = src[idx];
        }
#endif
        for (int idx = tid; idx < d; idx += tpb) {
            QMCCPW_CHK_SMEM(&sh[idx]);
            sh[idx] = P.shift[(size_t)rep_local * d + idx];
        }
        __syncthreads();
        sobol_build_g(vt, d, G, tid, tpb);
    }
    for (int v = 0; v < n_acc_smem; ++v) {
        QMCCPW_CHK_SMEM(&accs[v * tpb + tid]);
        accs[v * tpb + tid] = 0.0;
    }
    __shared__ double wacc[4 * 32];  // per-warp centred sums (tpb <= 128)
    wacc[tid] = 0.0;
    __syncwarp();
    unsigned unconverged = 0, ties = 0, npts = 0;
    const double sg = P.sigma;

    for (int a = 0; a < ppt; ++a) {
        if (i0 + ((uint64_t)a << tpb_log2) >= P.n_points) break;  // block-uniform
        uint32_t* HWb = HW + (a & 1) * hw_size;
        sobol_build_hw_inc(vt, OWEN ? nullptr : sh, d, 0, tpb_log2, nw, Ab + (uint64_t)a, a == 0, BS, HWb, tid, tpb);
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
                                (int)((kp0 >> tpb_log2) - Ab), OWEN ? sh : nullptr};
            // k-steps f (pairs) outer, not unrolled: each step draws this lane's two A
            // elements (four k-steps per iteration with four-way normals measured slower:
            // C4 PCA-W1 46.4 -> 50.7 ms at 8 blocks/SM, 47.2 at 6;
            // elements x[path][4 f + r4] and feeds them to all JT column tiles at once, so
            // the code holds one normal pair and 2 JT DMMAs instead of KF/2 pairs and KF JT
            // (the unrolled form was instruction-fetch bound); same k order, same bits.
            double cv[2 * JT];  // W(t_j) (W1) or c_j (X1) at j = 8 jt + 2 r4 + e
#pragma unroll
            for (int v = 0; v < 2 * JT; ++v) cv[v] = 0.0;
#pragma unroll 1
            for (int f = 0; f < KF; f += 2) {
                const int ja = 4 * f + r4, jb = 4 * (f + 1) + r4;
                double xa, xb;
                normal_from_u32_x2(sp.get(ja < d ? ja : d - 1), sp.get(jb < d ? jb : d - 1), xa, xb);
                const double a0 = (ja < d && !(COND == kX1 && ja == 0)) ? xa : 0.0;
                const double a1 = (jb < d && !(COND == kX1 && jb == 0)) ? xb : 0.0;
#pragma unroll
                for (int jt = 0; jt < JT; ++jt) {
                    // M[8 jt + q][r4 + 4 f] and [.. + 4 (f + 1)], adjacent in the fragment order
                    // (the lookback kernel keeps the two row-major loads: 194.5 vs 193.1 ms)
                    double b0, b1;
                    if (!LB) {
                        const double2 bb = __ldg(reinterpret_cast<const double2*>(P.Mf) +
                                                 ((size_t)(8 * jt + q) * (DP / 8) + (f >> 1)) * 4 + r4);
                        b0 = bb.x;
                        b1 = bb.y;
                    } else {
                        const double* Mrow = P.M + (size_t)(8 * jt + q) * DP + r4 + 4 * f;
                        b0 = __ldg(Mrow);
                        b1 = __ldg(Mrow + 4);
                    }
                    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                                 : "+d"(cv[2 * jt]), "+d"(cv[2 * jt + 1])
                                 : "d"(a0), "d"(b0));
                    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                                 : "+d"(cv[2 * jt]), "+d"(cv[2 * jt + 1])
                                 : "d"(a1), "d"(b1));
                }
            }
            if (COND == kW1) {
                // Mf's rows are M's minus row 0 (launch_mma_bfrag): cv holds W~(t_j) = W(t_j) - W(t_1)
                double sS = 0.0, sI = 0.0, em = -CUDART_INF, es = -CUDART_INF, ym = 0.0;
#pragma unroll
                for (int jt = 0; jt < JT; ++jt) {
                    const int j0 = 8 * jt + 2 * r4;
                    const double Wa = cv[2 * jt], Wb = cv[2 * jt + 1];
                    // (omega t, sigma t) of dates j0, j0 + 1 (rows past d read date 0: masked below)
                    const double2 ca = tt[j0 < d ? j0 : 0], cb = tt[j0 + 1 < d ? j0 + 1 : 0];
                    const double ea = fma(sg, Wa, ca.x), eb = fma(sg, Wb, cb.x);
                    double Xa, Xb;
                    fast_exp_x2(ea, eb, Xa, Xb);
                    const double Sa = (j0 < d) ? Xa : 0.0, Sb = (j0 + 1 < d) ? Xb : 0.0;  // W1Acc: sums without S0
                    const double ya = Wa - ca.y, yb = Wb - cb.y;
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
                    w1own.set_max(a2, a3, a4);
                }
            } else {
                // X1: c_j = ln S0 + omega t_j + sigma R_j, then one Newton solve per strike group
#pragma unroll
                for (int jt = 0; jt < JT; ++jt) {
                    const int j0 = 8 * jt + 2 * r4;
                    cv[2 * jt] = fma(sg, cv[2 * jt], fma(P.omega, (double)(j0 + 1) * P.t1, P.lnS0));
                    cv[2 * jt + 1] = fma(sg, cv[2 * jt + 1], fma(P.omega, (double)(j0 + 2) * P.t1, P.lnS0));
                }
                if (kSmemC) {
#pragma unroll
                    for (int v = 0; v < 2 * JT; ++v) {
                        QMCCPW_CHK_SMEM(&cst[(size_t)v * tpb]);
                        cst[(size_t)v * tpb] = cv[v];
                    }
                }
#define CV(v) (kSmemC ? cst[(size_t)(v) * tpb] : cv[(v)])
                if (LB && !kLbQuad) {
                    double* sw = stage + 8 * rt + q;
                    constexpr int SS = 32;
#pragma unroll
                    for (int jt = 0; jt < JT; ++jt) {
                        const int j0 = 8 * jt + 2 * r4;
                        if (j0 < d) QMCCPW_CHK_SMEM(&sw[j0 * SS]);
                        if (j0 < d) sw[j0 * SS] = cv[2 * jt];
                        if (j0 + 1 < d) sw[(j0 + 1) * SS] = cv[2 * jt + 1];
                    }
                }
                double f[kMaxOpt][4];
                // one Newton solve per strike group, not unrolled over the options: the
                // body is large and the instruction cache is the limiter (ncu: 41 % of
                // stalls were no_instructions with three unrolled copies)
#pragma unroll 1
                for (int o = 0; o < kMaxOpt; ++o) {
                    if (o >= P.n_opt) break;
                    if (P.tail_leader[o] != o || P.type[o] == kLookback) continue;
                    const double lnK = P.lnK[o], lndK = P.lndK[o];
                    // bracket [min_j (lnK - c_j)/(sigma a_j), min_j (ln dK - c_j)/(sigma a_j)] and mean c
                    double ulo = CUDART_INF, uhi = CUDART_INF, sumc = 0.0;
#pragma unroll kXU
                    for (int v = 0; v < 2 * JT; ++v) {
                        const int j = 8 * (v >> 1) + 2 * r4 + (v & 1);
                        if (j < d) {
                            const double isa = __ldg(P.inv_sa + j);
                            const double cvv = CV(v);
                            ulo = fmin(ulo, (lnK - cvv) * isa);
                            uhi = fmin(uhi, (lndK - cvv) * isa);
                            sumc += cvv;
                        }
                    }
                    ulo = quad_min(ulo);
                    uhi = quad_min(uhi);
                    sumc = quad_sum(sumc);
                    double u = fmin(uhi, (lnK - sumc / d) / (sg * P.mean_a));
                    bool conv = false;
                    const bool need_arith = P.x1_need_arith[o] != 0;
#pragma unroll 1
                    for (int it = 0; it < kNewtonMax; ++it) {
                        double S = 0.0, SA = 0.0, SAA = 0.0;
#pragma unroll kXU
                        for (int jt = 0; jt < JT; ++jt) {
                            const int j0 = 8 * jt + 2 * r4;
                            const double aa = (j0 < d) ? __ldg(P.a + j0) : 0.0;
                            const double ab = (j0 + 1 < d) ? __ldg(P.a + j0 + 1) : 0.0;
                            double Ea, Eb;
                            fast_exp_x2(fma(sg * aa, u, CV(2 * jt)), fma(sg * ab, u, CV(2 * jt + 1)), Ea, Eb);
                            Ea = (j0 < d) ? Ea : 0.0;
                            Eb = (j0 + 1 < d) ? Eb : 0.0;
                            S += Ea;
                            SA = fma(aa, Ea, SA);
                            SAA = fma(aa * aa, Ea, SAA);
                            S += Eb;
                            SA = fma(ab, Eb, SA);
                            SAA = fma(ab * ab, Eb, SAA);
                        }
                        S = quad_sum(S);
                        SA = quad_sum(SA);
                        SAA = quad_sum(SAA);
                        const double du = halley_step(fast_log(S) - lndK, S, SA, SAA, sg);
                        conv = !valid || fabs(du) <= kHalleyTol * fmax(1.0, fabs(u));
                        u = fmin(fmax(u - du, ulo), uhi);
                        if (it + 1 >= kNewtonIt && __all_sync(0xffffffffu, conv)) break;
                    }
                    if (r4 == 0 && valid && !conv) ++unconverged;
                    double Dst = 0.0, Qst = 0.0, Vst = 0.0, sumW = 0.0, sumWv = 0.0;
                    // arithmetic sums: w_j Phibar(x_j), x_j = u - sigma a_j, without a per-date phi:
                    // w_j phi(x_j) = phi(u) E_j, so it is phi(u) E_j R(x_j) for x_j >= 0 and
                    // w_j - phi(u) E_j R(-x_j) below (R the Mills ratio)
                    double phu = 0.0;
                    if (need_arith) {
                        double Qu_, Q2_, ph2_;
                        phibar_phi_x2(u, u, Qu_, Q2_, phu, ph2_);
                    }
#pragma unroll kXU
                    for (int jt = 0; jt < JT; ++jt) {
                        const int j0 = 8 * jt + 2 * r4;
                        const double aa = (j0 < d) ? __ldg(P.a + j0) : 0.0;
                        const double ab = (j0 + 1 < d) ? __ldg(P.a + j0 + 1) : 0.0;
                        const double ta = (double)(j0 + 1) * P.t1, tb = ta + P.t1;
                        const double ca = CV(2 * jt), cb2 = CV(2 * jt + 1);
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
                            double wa, wb, Ma, Mb;
                            fast_exp_x2(fma(0.5 * sg * sg * aa, aa, ca), fma(0.5 * sg * sg * ab, ab, cb2), wa, wb);
                            const double xa = u - sg * aa, xb = u - sg * ab;
                            mills_x2(xa, xb, Ma, Mb);
                            const double ga = phu * Ea * Ma, gb = phu * Eb * Mb;  // Ea, Eb are 0 past d
                            const double WPa = (j0 < d) ? (xa >= 0.0 ? ga : wa - ga) : 0.0;
                            const double WPb = (j0 + 1 < d) ? (xb >= 0.0 ? gb : wb - gb) : 0.0;
                            sumW += WPa;
                            sumWv = fma(Ra - sg * ta + sg * aa * aa, WPa, sumWv);
                            sumW += WPb;
                            sumWv = fma(Rb - sg * tb + sg * ab * ab, WPb, sumWv);
                        }
                    }
                    const X1Sums xs{u, quad_sum(Dst), quad_sum(Qst), quad_sum(Vst), quad_sum(sumW), quad_sum(sumWv)};
#pragma unroll
                    for (int o2 = 0; o2 < kMaxOpt; ++o2)
                        if (o2 < P.n_opt && P.tail_leader[o2] == o) x1_outputs(P, o2, xs, f[o2]);
                }
                if (kLbQuad) {
                    const double* cbase = stage_base + (tid & ~3);
                    auto cq = [&](int v, int L) { return cbase[(size_t)v * tpb + L]; };
#pragma unroll 1
                    for (int o = 0; o < kMaxOpt; ++o) {
                        if (o >= P.n_opt) break;
                        if (P.type[o] != kLookback) continue;
                        double fl[4];
                        x1_lookback_quad<2 * JT>(P, o, r4, cq, fl);
                        // f[o] = fl through selects (no dynamic register indexing)
#pragma unroll
                        for (int o3 = 0; o3 < kMaxOpt; ++o3)
                            if (o3 == o)
#pragma unroll
                                for (int qq = 0; qq < 4; ++qq) f[o3][qq] = fl[qq];
                    }
                }
                if (r4 == 0 && valid) {  // one lane per path records it
                    ++npts;
                    if (P.path_out != nullptr) {
#pragma unroll
                        for (int o = 0; o < kMaxOpt; ++o)
                            if (o == P.hook_option && (kLbQuad || P.type[o] != kLookback))
                                for (int qq = 0; qq < 4; ++qq) P.path_out[ip * 4 + qq] = f[o][qq];
                    }
                    if (!kSmemC) {
#pragma unroll
                        for (int o = 0; o < kMaxOpt; ++o) {
                            if (o < P.n_opt && P.type[o] != kLookback) {
#pragma unroll
                                for (int qq = 0; qq < 4; ++qq) {
                                    const double y = f[o][qq] - P.piv[o][qq];
                                    double* a1 = accs + (size_t)(o * 8 + qq * 2) * tpb + tp;
                                    QMCCPW_CHK_SMEM(&a1[tpb]);
                                    a1[0] += y;
                                    a1[tpb] = fma(y, y, a1[tpb]);
                                }
                            }
                        }
                    }
                }
                // the quad's four lanes hold the same f: lane r4 = 0 contributes each path once
                if (kSmemC)
                    warp_slot_sums(f, P, valid && r4 == 0, lane, wacc + (tid >> 5) * 32,
                                   /*skip_lookback=*/LB && !kLbQuad);
            }
        }
#undef CV
        if (COND == kX1 && LB && !kLbQuad) {
            // lookback options: lane L walks the envelope of path wbase + L from the staged c_j
            __syncwarp();
            const int tp = wbase + lane;
            const uint64_t ip = i0 + (uint64_t)tp + ((uint64_t)a << tpb_log2);
            const bool valid = ip < P.n_points;
#pragma unroll 1
            for (int o = 0; o < P.n_opt; ++o) {
                if (P.type[o] != kLookback) continue;
                double fl[4];
                x1_lookback(P, o, stage + lane, 32, fl);
                if (valid && P.path_out != nullptr && o == P.hook_option)
                    for (int qq = 0; qq < 4; ++qq) P.path_out[ip * 4 + qq] = fl[qq];
                if (valid) {
#pragma unroll
                    for (int qq = 0; qq < 4; ++qq) {
                        const double y = fl[qq] - P.piv[o][qq];
                        double* a1 = accs + (size_t)(o * 8 + qq * 2) * tpb + tp;
                        a1[0] += y;
                        a1[tpb] = fma(y, y, a1[tpb]);
                    }
                }
            }
            __syncwarp();  // the next batch overwrites the staging
        }
        if (COND == kW1) {
            const W1Acc& w1 = w1own;
            const uint64_t i = i0 + tid + ((uint64_t)a << tpb_log2);
            const bool valid = i < P.n_points;  // all lanes run: the warp reduction needs them
            npts += valid ? 1u : 0u;
            if (valid && P.has_lookback && w1.near_tie()) ++ties;
            if (kWarpSum) {
                tail_w1_reduce(P, w1, valid, lane, wacc + (tid >> 5) * 32, i);
            } else {
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
    }
    if (COND == kW1 && !kWarpSum) acc2_to_wacc(P, acc2, wacc, tpb, tid);
    block_epilogue(P, (COND == kX1 && !kWarpSum) ? accs : nullptr, wacc, red, n_acc, tpb, tid, cell, unconverged, ties,
                   npts);
}

static size_t pca_smem_bytes(const PathArgs& a, bool lb, int cond) {
    const size_t tpb = (size_t)1 << a.tpb_log2;
    const bool lbquad = cond == kX1 && lb && QMCCPW_LB_QUAD && QMCCPW_PCA_X1_SMEMC;
    const bool smemc = cond == kX1 && (!lb || lbquad) && QMCCPW_PCA_X1_SMEMC;
    lb = lb && !lbquad;  // no per-warp staging
    const bool warpsum = (cond == kW1 && QMCCPW_PCA_WARPSUM) || smemc;
    size_t b = pca_stage_offset(warpsum ? 0 : a.n_opt * 8, a.d, (int)tpb, cond == kW1);
    if (smemc) b += (size_t)(a.M_ld / 4) * tpb * sizeof(double);  // c_j [2 JT][tpb]
    if (lb) b += tpb * a.d * sizeof(double);  // [nw][d][32] staging
    return b;
}

template <int K, int KF, bool OW, bool LB>
static cudaError_t launch_pca_t(const PathArgs& args_in, cudaStream_t st) {
    static thread_local int set_for[64] = {0};
    int dev = 0;
    cudaGetDevice(&dev);
    if (set_for[dev & 63] == 0) {
        cudaError_t e = cudaFuncSetAttribute(pca_kernel<K, KF, OW, LB>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
        if (e != cudaSuccess) return e;
        set_for[dev & 63] = 1;
    }
    PathArgs args = args_in;
    int best_lg = -1, best_warps = -1;
    for (int lg = 7; lg >= 5; --lg) {
        args.tpb_log2 = lg;
        const size_t smem = pca_smem_bytes(args, LB, K);
        if (smem > 200 * 1024) continue;
        int nb = 0;
        if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, pca_kernel<K, KF, OW, LB>, 1 << lg, smem) != cudaSuccess) continue;
        if (nb * (1 << lg) / 32 > best_warps) {
            best_warps = nb * (1 << lg) / 32;
            best_lg = lg;
        }
    }
    if (best_lg < 0) return cudaErrorInvalidConfiguration;
    args.tpb_log2 = best_lg;
    const uint64_t nblocks = args.cell_end - args.cell_begin;
    if (nblocks == 0) return cudaSuccess;
    pca_kernel<K, KF, OW, LB><<<(unsigned)nblocks, 1 << best_lg, pca_smem_bytes(args, LB, K), st>>>(args);
    ++launch_counter();
    return cudaGetLastError();
}

template <int K, bool OW, bool LB = false>
static cudaError_t launch_pca(const PathArgs& args, cudaStream_t st, bool* handled) {
    *handled = true;
    switch (args.M_ld) {
    case 8: return launch_pca_t<K, 2, OW, LB>(args, st);
    case 16: return launch_pca_t<K, 4, OW, LB>(args, st);
    case 24: return launch_pca_t<K, 6, OW, LB>(args, st);
    case 32: return launch_pca_t<K, 8, OW, LB>(args, st);
    case 40: return launch_pca_t<K, 10, OW, LB>(args, st);
    case 48: return launch_pca_t<K, 12, OW, LB>(args, st);
    case 56: return launch_pca_t<K, 14, OW, LB>(args, st);
    case 64: return launch_pca_t<K, 16, OW, LB>(args, st);
    case 96: return launch_pca_t<K, 24, OW, LB>(args, st);
    case 128: return launch_pca_t<K, 32, OW, LB>(args, st);
    default: *handled = false; return cudaSuccess;
    }
}


}  // namespace qmccpw
