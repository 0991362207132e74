// qmccpw_paths.cuh -- the fused path kernel (STD / BB / PCA-fallback x W1 / X1 x
// QMC / LR / MC / MC+AV) and its launcher template; instantiated by
// qmccpw_paths_w1.cu and qmccpw_paths_x1.cu (separate translation units so the
// build compiles them in parallel).
#pragma once
#include "qmccpw_device.cuh"

namespace qmccpw {

#ifndef QMCCPW_STD_X4
#define QMCCPW_STD_X4 1
#endif
#ifndef QMCCPW_BB_SHIFT_W1
#define QMCCPW_BB_SHIFT_W1 1
#endif
#ifndef QMCCPW_BB_MINB
#define QMCCPW_BB_MINB 8
#endif
#ifndef QMCCPW_STD_MINB
#define QMCCPW_STD_MINB 7
#endif
// resident blocks per SM the register allocator must allow (128 threads each); 0 = ptxas'
// own choice.  Measured on C4 (ms/step): BB-W1 34.3 (ptxas, 96 regs) / 33.8 (7) / 33.4
// (8: 64 regs, a few spills to L1); STD-W1 33.1 (4) / 31.9 (5) / 31.2 (6); v11: 27.20 (6) / 27.03 (7) / 27.4 (8)
// MC+AV-CPW with the bridge: 140 registers uncapped at v18 (3 blocks/SM; 46.2 -> 51.5 ms
// against v17), so it is capped at 4 blocks
// BB-W1 (QMC) at d >= 8: the eight-dates-per-group bridge (static expression tree for the last
// seven normals of each group, four-way normals); 0: the pairwise bridge with the normal FIFO.
// A/B on one B200, C4 BB-W1 (ms/step): pairwise 27.94; grouped at 8 / 7 / 6 blocks/SM
// 26.33 / 26.57 / 26.66
#ifndef QMCCPW_BB_GROUPED
#define QMCCPW_BB_GROUPED 1
#endif
// (grouped bridge at d = 64 with the terminal and group 0's dynamic levels as one four-way
// batch measured slower: 25.60 -> 26.42 ms, spills; removed)
// STD-X1 streamed through one pass (X1Stream, no per-date storage)
#ifndef QMCCPW_STD_X1_STREAM
#define QMCCPW_STD_X1_STREAM 1
#endif
// A/B on one B200, C4 STD-X1 (ms/step, arithmetic + binary / with the lookback): per-date columns
// 45.0 / 53.6; streamed at 4 / 6 / 8 blocks/SM 27.6 / 28.4, 27.9 / 28.7, 28.3 / 29.2
#ifndef QMCCPW_STDX1_MINB
#define QMCCPW_STDX1_MINB 4
#endif
// grouped bridge: exps of four dates at once (push4) and the rare single normals out of line
// A/B on one B200, C4 BB-W1 (ms/step): neither 26.43, push4 26.90, out-of-line single normals
// 26.07, both 26.40
// the seven static normals of a group as 4 + 3 interleaved chains (two coefficient streams)
// instead of 4 + 2 + 1 (three)
#ifndef QMCCPW_BB_X3
#define QMCCPW_BB_X3 1
#endif
#ifndef QMCCPW_BB_PUSH4
#define QMCCPW_BB_PUSH4 0
#endif
#ifndef QMCCPW_BB_N1CALL
#define QMCCPW_BB_N1CALL 1
#endif
#if QMCCPW_BB_N1CALL
#define NORMAL1 normal_from_u32_call
#else
#define NORMAL1 normal_from_u32
#endif
#ifndef QMCCPW_BBAV_MINB
#define QMCCPW_BBAV_MINB 4
#endif
template <int CONSTR, int COND, int METHOD>
constexpr int paths_min_blocks() {
    return (COND == kW1 && METHOD == kQmc) ? (CONSTR == kBB ? QMCCPW_BB_MINB : CONSTR == kStd ? QMCCPW_STD_MINB : 0)
           : (COND == kX1 && METHOD == kQmc && CONSTR == kStd && QMCCPW_STD_X1_STREAM) ? QMCCPW_STDX1_MINB
           : (COND == kW1 && METHOD == kMcAv && CONSTR == kBB) ? QMCCPW_BBAV_MINB
                                                                : 0;
}
// OWEN: nested scrambling of the Sobol' coordinates (row f4) -- a template flag so
// that the other randomisations pay nothing for it (measured 0.5-4 % as a runtime test)
template <int CONSTR, int COND, int METHOD, bool OWEN>
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
    // STD-X1 streams its sums (X1Stream): no per-date c_j columns
    constexpr bool kStdStream = (METHOD == kQmc) && CONSTR == kStd && COND == kX1 && QMCCPW_STD_X1_STREAM;
    constexpr bool kNeedBuf = (METHOD == kQmc) && (CONSTR == kPca || COND == kX1) && !kStdStream;
    constexpr bool kTwoBuf = (METHOD == kQmc) && (CONSTR == kPca && COND == kX1);
    // QMC W1 reduces each option's values as the tail forms them (tail_w1_reduce)
    constexpr bool kFusedTail = (METHOD == kQmc) && COND == kW1;
    // X tile [M_ld][tpb + 8] in buf0 for the DMMA contraction: PCA-W1 always, PCA-X1 up to
    // d = 128 (beyond, the X tile and the c_j columns do not both fit: per-thread matvec)
    const bool kMmaX = (METHOD == kQmc) && CONSTR == kPca && (COND == kW1 || P.M_ld <= 128);

    // shared memory carve-up (8-byte aligned first):
    //   buf0, buf1 [d][tpb] | vt [d][32] | sh [d] | G [d][32] | pad | HW [2][2][nw][d] (>= 1 KB)
    // the reduction scratch red [4 warps][32] aliases HW after the point loop; the
    // centred sums live in one register per lane (warp_slot_sums).
    const int nw = tpb >> 5;
    const int n_acc = P.n_opt * 8;
    const int lane = tid & 31;
    double* buf0 = reinterpret_cast<double*>(smem_raw);
    double* buf1 = buf0 + (kMmaX ? (size_t)P.M_ld * (tpb + 8) : (kNeedBuf ? (size_t)d * tpb : 0));
    uint32_t* vt = reinterpret_cast<uint32_t*>(buf1 + (kTwoBuf ? (size_t)d * tpb : 0));
    uint32_t* sh = vt + (METHOD == kQmc ? (size_t)d * 32 : 0);
    uint32_t* G = sh + (METHOD == kQmc ? d : 0);
    uint32_t* HW = G + (METHOD == kQmc ? (size_t)d * 32 : 0);
    HW += ((uintptr_t)HW & 7) ? 1 : 0;
    double* red = reinterpret_cast<double*>(HW);
    const int hw_size = 2 * nw * d;
    uint32_t* BS = HW + 2 * hw_size;  // [d] incremental Gray bases (sobol_build_hw_inc)

    const uint64_t K0 = P.point_offset + i0;
    const uint64_t Ab = K0 >> tpb_log2;
    const uint64_t kt = K0 + (uint64_t)tid;
    SobolBlock sob{G, HW, d, nw, (int)(kt & 31), (int)((kt >> 5) & (uint64_t)(nw - 1)), (int)((kt >> tpb_log2) - Ab),
                   OWEN ? sh : nullptr};
    // BB stages the replicate's tables in the bridge's consumption order (row i =
    // Sobol' dimension bb_seq[i]), so the i-th normal reads row i: no per-normal
    // dimension lookup
    constexpr bool kPerm = (CONSTR == kBB && METHOD == kQmc);
    math_tables_load(tid, tpb);
    if (METHOD != kQmc) __syncthreads();  // QMC: the barrier below publishes the tables
    if (METHOD == kQmc) {
        const uint32_t* src = P.vscr + (size_t)rep_local * d * 32;
        QMCCPW_CHECK(rep_local < P.n_reps && cell < P.cell_end);
        for (int idx = tid; idx < d * 32; idx += tpb) {
            QMCCPW_CHK_SMEM(&vt[idx]);
            QMCCPW_CHECK(!kPerm || P.bb_seq[idx >> 5] < d);
            vt[idx] = src[kPerm ? (int)P.bb_seq[idx >> 5] * 32 + (idx & 31) : idx];
        }
        for (int idx = tid; idx < d; idx += tpb) {
            QMCCPW_CHK_SMEM(&sh[idx]);
            sh[idx] = P.shift[(size_t)rep_local * d + (kPerm ? P.bb_seq[idx] : idx)];
        }
        __syncthreads();
        sobol_build_g(vt, d, G, tid, tpb);
    }
    __shared__ double wacc[4 * 32];  // per-warp centred sums (tpb <= 128)
    wacc[tid] = 0.0;
    __syncwarp();
    if (kMmaX) {  // zero X rows d..dp-1 (the padded K of the mma tiles); X1: also row 0 (x_1 := 0)
        for (int r = d; r < P.M_ld; ++r) buf0[(size_t)r * (tpb + 8) + tid] = 0.0;
        if (COND == kX1) buf0[tid] = 0.0;
    }
    unsigned unconverged = 0, ties = 0, npts = 0;

    for (int a = 0; a < ppt; ++a) {
        if (i0 + ((uint64_t)a << tpb_log2) >= P.n_points) break;  // block-uniform: ragged last cell
        if (METHOD == kQmc) {
            uint32_t* HWb = HW + (a & 1) * hw_size;  // double-buffered: one barrier per iteration
            sobol_build_hw_inc(vt, OWEN ? nullptr : sh, d, P.dim_begin, tpb_log2, nw, Ab + (uint64_t)a, a == 0, BS, HWb, tid,
                               tpb);
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
                // the path's d normals in Sobol'-dimension order first (one Philox block per 4
                // dimensions), then the bridge reads them in its consumption order (bb_seq):
                // d/4 Philox calls instead of ~1.7 per pair of consumed normals
                double xs[kMaxDimGpu];
#pragma unroll 1
                for (int jq = 0; jq < d; jq += 4) {
                    uint32_t c[4] = {(uint32_t)k, (uint32_t)(k >> 32), (uint32_t)(jq >> 2), (rep << 8) | 0x02u};
                    philox4x32_10(c, (uint32_t)P.seed, (uint32_t)(P.seed >> 32));
                    double x4[4];
                    normal_from_u32_x2(c[0], c[1], x4[0], x4[1]);
                    normal_from_u32_x2(c[2], c[3], x4[2], x4[3]);
#pragma unroll
                    for (int w = 0; w < 4; ++w)
                        if (jq + w < d) xs[jq + w] = x4[w];
                }
                int pos = 0;
                double stW[12];
                int sp = 0;
                stW[0] = P.sqrtT * xs[P.bb_seq[pos++]];
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
                            const double x = xs[P.bb_seq[pos++]];
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
            if (P.has_lookback && w1.near_tie()) ++ties;
            tail_w1_all(P, w1, f);
            if (METHOD == kMcAv) {
                if (P.has_lookback && w1m.near_tie()) ++ties;
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
#if QMCCPW_STD_X4
                // four dates per step: the normals as four interleaved chains (as BB-W1's groups)
#pragma unroll 1
                for (; j + 3 < d; j += 4) {
                    const uint32_t y4[4] = {sob.get(j), sob.get(j + 1), sob.get(j + 2), sob.get(j + 3)};
                    double x4[4];
                    normal_from_u32_x4(y4, x4);
                    const double Wa = fma(P.sqrt_t1, x4[0], Wt);
                    const double Wb = fma(P.sqrt_t1, x4[1], Wa);
                    const double Wc = fma(P.sqrt_t1, x4[2], Wb);
                    Wt = fma(P.sqrt_t1, x4[3], Wc);
                    w1.push2(P, j, Wa, Wb);
                    w1.push2(P, j + 2, Wc, Wt);
                }
#endif
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
            } else if (CONSTR == kBB && QMCCPW_BB_GROUPED && d >= 8) {
                // Alg. 4 in time order, eight dates per group g (pairs 4g..4g+3 of the
                // pairwise form below).  Pair 4g descends e0 = 3 + ctz(g) levels (e0 = m at
                // g = 0); pairs 4g+1, 4g+2, 4g+3 descend 1, 2, 1.  So only levels c >= 3 of the
                // first descent are data-dependent: they go through the stack (pushed for c > 3;
                // the c = 3 midpoint is the group's right end R = W(8g+8), or R is popped when
                // e0 = 3), and the last seven normals of the group -- levels 2, 1, 0 of pair 4g,
                // then 1, 2, 1 normals -- are consecutive in Alg. 4's order and feed a fixed
                // expression tree with no stack traffic, no FIFO and no branches.  Every W is
                // the same fma / 0.5 (l + r) expression as in the pairwise form (same bits).
                const int m = P.bb_m;
                const double b0 = P.bb_b[m], b1 = P.bb_b[m - 1], b2 = P.bb_b[m - 2];
                double stW[12];
                int sp = 0;
                int pos = 0;
                stW[0] = P.sqrtT * NORMAL1(sob.get(pos++));  // terminal: W(T) = sqrt(T) x_0
                double Wl = 0.0, W1 = 0.0;
                (void)W1;
#pragma unroll 1
                for (int g = 0; g < (d >> 3); ++g) {
                    const int e0 = (g == 0) ? m : 2 + __ffs(g);
                    double R;
                    if (e0 == 3) {
                        R = stW[sp];
                        --sp;
                    } else {
                        double Wr = stW[sp];
#pragma unroll 1
                        for (int c = e0 - 1; c >= 3; --c) {
                            const double Wm = fma(P.bb_b[m - c], NORMAL1(sob.get(pos++)), 0.5 * (Wl + Wr));
                            if (c > 3) stW[++sp] = Wm;
                            Wr = Wm;
                        }
                        R = Wr;
                    }
                    QMCCPW_CHECK(sp >= -1 && sp < 12 && pos + 7 <= d);
                    uint32_t y4[4] = {sob.get(pos), sob.get(pos + 1), sob.get(pos + 2), sob.get(pos + 3)};
                    double x[7];
                    double x4[4];
                    normal_from_u32_x4(y4, x4);
#if QMCCPW_BB_X3
                    {  // the last three as three interleaved chains (one coefficient stream)
                        const uint32_t y3[3] = {sob.get(pos + 4), sob.get(pos + 5), sob.get(pos + 6)};
                        double x3[3];
                        normal_from_u32_xn<3>(y3, x3);
                        x[4] = x3[0];
                        x[5] = x3[1];
                        x[6] = x3[2];
                    }
#else
                    normal_from_u32_x2(sob.get(pos + 4), sob.get(pos + 5), x[4], x[5]);
                    x[6] = normal_from_u32(sob.get(pos + 6));
#endif
                    pos += 7;
#if QMCCPW_BB_SHIFT_W1
                    double M4 = fma(b2, x4[0], 0.5 * (Wl + R));   // W(8g+4)
                    double M2 = fma(b1, x4[1], 0.5 * (Wl + M4));  // W(8g+2)
                    double Wa = fma(b0, x4[2], 0.5 * (Wl + M2));  // W(8g+1)
                    // once W(t_1) is known (group 0), every live value -- the group's M4, M2, R and
                    // the stack -- is shifted by it; the bridge is linear, so all later midpoints
                    // come out as W~ = W - W(t_1) and W1's increments need no per-date subtraction
                    const double shift = (g == 0) ? Wa : 0.0;
                    if (g == 0) {
#pragma unroll 1
                        for (int i = 0; i <= sp; ++i) stW[i] -= shift;
                    }
                    M4 -= shift;
                    M2 -= shift;
                    R -= shift;
                    Wa -= shift;
                    const double W3 = fma(b0, x4[3], 0.5 * (M2 + M4));
                    const double W6 = fma(b1, x[4], 0.5 * (M4 + R));
                    const double W5 = fma(b0, x[5], 0.5 * (M4 + W6));
                    const double W7 = fma(b0, x[6], 0.5 * (W6 + R));
                    w1.push2(P, 8 * g, Wa, M2);
                    w1.push2(P, 8 * g + 2, W3, M4);
                    w1.push2(P, 8 * g + 4, W5, W6);
                    w1.push2(P, 8 * g + 6, W7, R);
#else
                    const double M4 = fma(b2, x4[0], 0.5 * (Wl + R));   // W(8g+4)
                    const double M2 = fma(b1, x4[1], 0.5 * (Wl + M4));  // W(8g+2)
                    const double Wa = fma(b0, x4[2], 0.5 * (Wl + M2));  // W(8g+1)
                    if (g == 0) W1 = Wa;
                    const double W3 = fma(b0, x4[3], 0.5 * (M2 + M4));
                    const double W6 = fma(b1, x[4], 0.5 * (M4 + R));
                    const double W5 = fma(b0, x[5], 0.5 * (M4 + W6));
                    const double W7 = fma(b0, x[6], 0.5 * (W6 + R));
                    w1.push2(P, 8 * g, Wa - W1, M2 - W1);
                    w1.push2(P, 8 * g + 2, W3 - W1, M4 - W1);
                    w1.push2(P, 8 * g + 4, W5 - W1, W6 - W1);
                    w1.push2(P, 8 * g + 6, W7 - W1, R - W1);
#endif
                    Wl = R;
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
                auto dim_at = [&](int o) { return pos + o; };  // tables are in consumption order (kPerm)
                double stW[12];
                int sp = 0;
                stW[0] = P.sqrtT * fifo.next(sob, dim_at);
                pos += 2;
                const int m = P.bb_m;
                if (d == 1) {
                    w1.push(P, 0, 0.0);
                } else {
                    double Wl = 0.0, W1 = 0.0;
                    // e = 1 (half of the steps) and e = 2 (a quarter) in straight-line code:
                    // no stack store, no loop, the two finest b's in registers
                    const double bm = P.bb_b[m], bm1 = P.bb_b[m > 1 ? m - 1 : m];
                    auto next_x = [&]() {
                        const bool refill = fifo.have == 0;
                        const double x = fifo.next(sob, dim_at);
                        pos += refill ? 2 : 0;
                        return x;
                    };
#pragma unroll 1
                    for (int pp = 0; pp < (d >> 1); ++pp) {
                        const int e = (pp == 0) ? m : __ffs(pp);  // 1 + ctz(pp)
                        const double top = stW[sp];
                        double Wodd, Weven;
                        if (e == 1) {
                            Wodd = fma(bm, next_x(), 0.5 * (Wl + top));
                            Weven = top;
                            --sp;
                        } else if (e == 2) {  // push + pop of the level m-1 midpoint cancel
                            Weven = fma(bm1, next_x(), 0.5 * (Wl + top));
                            Wodd = fma(bm, next_x(), 0.5 * (Wl + Weven));
                        } else {
                            double Wr = top;
#pragma unroll 1
                            for (int c = e - 1; c >= 0; --c) {
                                const double Wm = fma(P.bb_b[m - c], next_x(), 0.5 * (Wl + Wr));
                                if (c > 0) stW[++sp] = Wm;
                                Wr = Wm;
                            }
                            Wodd = Wr;
                            Weven = stW[sp];
                            --sp;
                        }
                        if (pp == 0) W1 = Wodd;
                        QMCCPW_CHECK(sp >= -1 && sp < 12 && pos <= d + 2);
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
                    QMCCPW_CHK_SMEM(&xc[(kk + 1) * XS]);
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
                        const double Sa = Xa * va, Sb = Xb * vb;  // W1Acc: sums without S0
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
                        w1.set_max(a2, a3, a4);
                    }
                }
            }
            if (P.has_lookback && w1.near_tie()) ++ties;
            tail_w1_reduce(P, w1, valid, lane, wacc + (tid >> 5) * 32, i);  // kFusedTail
        } else {
            // X1: c_j = ln S0 + omega t_j + sigma R_j, R = M x with x_1 := 0
            double* cb = (CONSTR == kPca ? buf1 : buf0) + tid;
            if (kStdStream) {
                X1Stream xst;
                xst.reset();
                double R = 0.0;
                {
                    const double c0 = P.lnS0 + P.omega * P.t1, t0 = P.t1;
                    xst.push(P, 0, c0, t0, fast_exp(c0));
                }
                int j = 1;
#pragma unroll 1
                for (; j + 1 < d; j += 2) {
                    double xa, xb2;
                    normal_from_u32_x2(sob.get(j), sob.get(j + 1), xa, xb2);
                    R = fma(P.sqrt_t1, xa, R);
                    const double ca = P.lnS0 + P.omega * (double)(j + 1) * P.t1 + P.sigma * R;
                    R = fma(P.sqrt_t1, xb2, R);
                    const double cb2 = P.lnS0 + P.omega * (double)(j + 2) * P.t1 + P.sigma * R;
                    double Ea, Eb;
                    fast_exp_x2(ca, cb2, Ea, Eb);
                    xst.push(P, j, ca, (double)(j + 1) * P.t1, Ea);
                    xst.push(P, j + 1, cb2, (double)(j + 2) * P.t1, Eb);
                }
                if (j < d) {
                    R = fma(P.sqrt_t1, normal_from_u32(sob.get(j)), R);
                    const double c = P.lnS0 + P.omega * (double)(j + 1) * P.t1 + P.sigma * R;
                    xst.push(P, j, c, (double)(j + 1) * P.t1, fast_exp(c));
                }
                tail_x1_stream(P, xst, f);
            } else if (CONSTR == kStd) {
                double R = 0.0;
                cb[0] = P.lnS0 + P.omega * P.t1;
                int j = 1;
#pragma unroll 1
                for (; j + 1 < d; j += 2) {
                    double xa, xb2;
                    normal_from_u32_x2(sob.get(j), sob.get(j + 1), xa, xb2);
                    R = fma(P.sqrt_t1, xa, R);
                    QMCCPW_CHK_SMEM(&cb[(j + 1) * tpb]);
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
                auto dim_at = [&](int o) { return pos + o; };  // tables in consumption order (kPerm)
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
                    QMCCPW_CHK_SMEM(&cb[(j - 1) * tpb]);
                    QMCCPW_CHECK(sp >= -1 && sp < 12 && pos <= d + 1);  // the last date pops the bottom
                    cb[(j - 1) * tpb] = P.lnS0 + P.omega * (double)j * P.t1 + P.sigma * Rj;
                    Wl = Rj;
                }
            } else if (!kMmaX) {
                // PCA, d > 128: per-thread R = M x (x_1 := 0) from shared memory
                double* xb = buf0 + tid;
                int kk = 1;
#pragma unroll 1
                for (; kk + 1 < d; kk += 2) {
                    double xa, xc;
                    normal_from_u32_x2(sob.get(kk), sob.get(kk + 1), xa, xc);
                    QMCCPW_CHK_SMEM(&xb[(kk + 1) * tpb]);
                    xb[kk * tpb] = xa;
                    xb[(kk + 1) * tpb] = xc;
                }
                if (kk < d) xb[kk * tpb] = normal_from_u32(sob.get(kk));
#pragma unroll 1
                for (int j = 0; j < d; ++j) {
                    const double* Ma = P.M + (size_t)j * P.M_ld;
                    double Ra = 0.0;
#pragma unroll 4
                    for (int q2 = 1; q2 < d; ++q2) Ra = fma(__ldg(Ma + q2), xb[q2 * tpb], Ra);
                    QMCCPW_CHK_SMEM(&cb[j * tpb]);
                    cb[j * tpb] = P.lnS0 + P.omega * (double)(j + 1) * P.t1 + P.sigma * Ra;
                }
            } else {
                // PCA: R = X M^T (x_1 := 0) on the FP64 tensor cores, as in the W1 branch:
                // X[k][path] in shared memory (row stride tpb + 8), mma.sync.m8n8k4.f64 over
                // the warp's 32 paths, and each lane writes its tile's c_j into the owning
                // threads' columns of cb
                const int XS = tpb + 8, dp = P.M_ld;
                double* xcol = buf0 + tid;
                int kk = 1;
#pragma unroll 1
                for (; kk + 1 < d; kk += 2) {
                    double xa, xc;
                    normal_from_u32_x2(sob.get(kk), sob.get(kk + 1), xa, xc);
                    xcol[kk * XS] = xa;
                    xcol[(kk + 1) * XS] = xc;
                }
                if (kk < d) xcol[kk * XS] = normal_from_u32(sob.get(kk));
                __syncwarp();
                const int q = lane >> 2, r4 = lane & 3, wbase = tid & ~31;
                const double* Xk = buf0 + wbase + (size_t)r4 * XS + q;
#pragma unroll 1
                for (int jt = 0; jt < dp; jt += 8) {
                    double acc[4][2];
#pragma unroll
                    for (int rt = 0; rt < 4; ++rt) acc[rt][0] = acc[rt][1] = 0.0;
                    const double* Mrow = P.M + (size_t)(jt + q) * dp + r4;
#pragma unroll 2
                    for (int kt = 0; kt < dp; kt += 4) {
                        const double bfrag = __ldg(Mrow + kt);
                        const double* Xr = Xk + (size_t)kt * XS;
#pragma unroll
                        for (int rt = 0; rt < 4; ++rt)
                            asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                                         : "+d"(acc[rt][0]), "+d"(acc[rt][1])
                                         : "d"(Xr[8 * rt]), "d"(bfrag));
                    }
                    const int j0 = jt + 2 * r4;  // lane (q, r4) holds R at dates j0, j0 + 1 of paths 8 rt + q
#pragma unroll
                    for (int rt = 0; rt < 4; ++rt) {
                        double* col = buf1 + wbase + 8 * rt + q;
                        if (j0 < d) QMCCPW_CHK_SMEM(&col[(size_t)j0 * tpb]);
                        if (j0 < d) col[(size_t)j0 * tpb] = P.lnS0 + P.omega * (double)(j0 + 1) * P.t1 + P.sigma * acc[rt][0];
                        if (j0 + 1 < d)
                            col[(size_t)(j0 + 1) * tpb] = P.lnS0 + P.omega * (double)(j0 + 2) * P.t1 + P.sigma * acc[rt][1];
                    }
                }
                __syncwarp();

            }
            if (!kStdStream) tail_x1_all(P, cb, tpb, f, unconverged);
        }

        if (!valid) {
            unconverged = unconverged0;
            ties = ties0;
        }
        if (!kFusedTail) {
            if (P.path_out != nullptr && valid) {
#pragma unroll
                for (int o = 0; o < kMaxOpt; ++o)
                    if (o == P.hook_option)
#pragma unroll
                        for (int q = 0; q < 4; ++q) {
                            QMCCPW_CHECK(i < P.n_points);
                            P.path_out[i * 4 + q] = f[o][q];
                        }
            }
            warp_slot_sums(f, P, valid, lane, wacc + (tid >> 5) * 32);
        }
        (void)k;
    }

    block_epilogue(P, nullptr, wacc, red, n_acc, tpb, tid, cell, unconverged, ties, npts);
}


static size_t path_smem_bytes(const PathArgs& a, int constr, int cond, int method) {
    const size_t tpb = (size_t)1 << a.tpb_log2, nw = tpb / 32;
    const bool need_buf = method == kQmc && (constr == kPca || cond == kX1) &&
                          !(constr == kStd && cond == kX1 && QMCCPW_STD_X1_STREAM);
    const bool two_buf = method == kQmc && constr == kPca && cond == kX1;
    size_t b = 0;
    if (method == kQmc && constr == kPca && (cond == kW1 || a.M_ld <= 128))
        b += (size_t)a.M_ld * (tpb + 8) * sizeof(double);  // X tile (DMMA)
    else if (need_buf) b += (size_t)a.d * tpb * sizeof(double);
    if (two_buf) b += (size_t)a.d * tpb * sizeof(double);
    size_t hw = 0;
    if (method == kQmc) {
        b += ((size_t)a.d * 32 * 2 + a.d) * sizeof(uint32_t) + 4;  // vt, sh, G, alignment pad
        hw = (2 * 2 * nw * a.d + a.d) * sizeof(uint32_t);
    }
    const size_t red = 4 * 32 * sizeof(double);
    return b + (hw > red ? hw : red);
}

template <int C, int K, int M, bool OW>
static cudaError_t launch_paths_t(const PathArgs& args_in, cudaStream_t st, int* smem_out) {
    // raise the dynamic-smem limit once per device (not on every call: it is a driver round trip)
    static thread_local int set_for[64] = {0};
    int dev = 0;
    cudaGetDevice(&dev);
    if (set_for[dev & 63] == 0) {
        cudaError_t e = cudaFuncSetAttribute(paths_kernel<C, K, M, OW>, cudaFuncAttributeMaxDynamicSharedMemorySize,
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
        if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, paths_kernel<C, K, M, OW>, 1 << lg, smem) != cudaSuccess)
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
    paths_kernel<C, K, M, OW><<<(unsigned)nblocks, 1 << args.tpb_log2, smem, st>>>(args);
    ++launch_counter();
    return cudaGetLastError();
}

}  // namespace qmccpw
