// qmccpw_kernels.cu -- table kernels (randomisation, path matrix, GPCA rotation),
// the cell reduction and the parity hooks of the QMC-CPW hot path (arXiv 2209.11337).
// The path kernels are in qmccpw_paths*.cu / qmccpw_pca*.cu / qmccpw_portfolio.cu.
//
// Device code here is independent of oracle/: it is written from the paper
// and SURVEY.md Sec. 8(a); tests compare the two on the same points.

#include "qmccpw_device.cuh"

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
    if (construction == kStd && M != nullptr && idx < ld * ld) {
        // Alg. 3 as a matrix: W(t_j) = sqrt(dt) (x_1 + ... + x_j), Sobol' dimension k -> x_{k+1}
        const int j = idx / ld + 1, k = idx % ld;
        M[idx] = (j <= d && k < j) ? sqrt(dt) : 0.0;
    }
    if (construction == kBB && M != nullptr && idx < ld * ld) {
        // Alg. 4 as a matrix (the Levy-Ciesielski form of the bridge): Sobol' dimension 0 is the
        // terminal, W_j gains t_j / sqrt(T) x_0; dimension k >= 1 is the midpoint of interval
        // jj = 2^lev - 1 - k at level lev (2^lev <= 2k + 1 < 2^(lev+1)), mid = (2 jj + 1) 2^c,
        // c = m - lev, and W_j gains b_lev x_k times the hat max(0, 1 - |j - mid| / 2^c)
        const int j = idx / ld + 1, k = idx % ld;
        double v = 0.0;
        if (j <= d && k < d) {
            if (k == 0) {
                v = (double)j * dt / sqrt(T);
            } else {
                int m = 0;
                while ((1 << m) < d) ++m;
                int lev = 0;
                while ((2 << lev) <= k) ++lev;  // 2^lev <= k < 2^(lev+1)
                ++lev;                            // levels are 1-based: dimension 1 is level 1
                const int jj = (1 << lev) - 1 - k, c = m - lev;
                const int mid = (2 * jj + 1) << c, half = 1 << c;
                const int dist = j > mid ? j - mid : mid - j;
                if (dist < half) v = sqrt(T / ldexp(1.0, lev + 1)) * (1.0 - (double)dist / (double)half);
            }
        }
        M[idx] = v;
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

// M (row-major [ld][ld]) in the order pca_kernel reads its m8n8k4 B fragments: lane (q, r4)
// of a warp needs M[row][r4 + 4 f] and M[row][r4 + 4 (f + 1)] for each even k-step f, so
// Mf[((row * ld/8) + f/2) * 8 + 2 r4 + e] = M[row][r4 + 4 (f + e)]: one 16-byte load per
// pair of k-steps instead of two 8-byte loads.  shift_row0 (W1): every row minus row 0, so the
// contraction yields W~(t_j) = W(t_j) - W(t_1) directly (W1's increments) and the
// kernel needs no per-date subtraction.
__global__ void mma_bfrag_kernel(const double* __restrict__ M, int ld, int shift_row0, double* __restrict__ Mf) {
    const int idx = blockIdx.x * blockDim.x + threadIdx.x;
    if (idx >= ld * ld) return;
    const int row = idx / ld, rem = idx % ld;
    const int fp = rem >> 3, r4 = (rem & 7) >> 1, e = rem & 1;
    const int col = r4 + 4 * (2 * fp + e);
    Mf[idx] = M[(size_t)row * ld + col] - (shift_row0 ? M[col] : 0.0);
}

cudaError_t launch_mma_bfrag(const double* d_M, int ld, bool shift_row0, double* d_Mf, cudaStream_t st) {
    const int n = ld * ld, tpb = 256;
    mma_bfrag_kernel<<<(n + tpb - 1) / tpb, tpb, 0, st>>>(d_M, ld, shift_row0 ? 1 : 0, d_Mf);
    ++launch_counter();
    return cudaGetLastError();
}

cudaError_t launch_path_matrix(int construction, int d, int ld, double T, double sigma, double* d_M, double* d_a,
                               double* d_inv_sa, cudaStream_t st) {
    const int n = d_M ? (ld * ld > d ? ld * ld : d) : d;
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
        sobol_build_hw_inc(h.vt, owen ? nullptr : h.sh, d, 0, tpb_log2, nw, Ab + (uint64_t)a, a == 0,
                           h.HW + 4 * nw * d, HWb, tid, tpb);  // the path kernels' incremental build
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
    math_tables_load(tid, tpb);
    __syncthreads();
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
        sobol_build_hw_inc(h.vt, owen ? nullptr : h.sh, d, 0, tpb_log2, nw, Ab + (uint64_t)a, a == 0,
                           h.HW + 4 * nw * d, HWb, tid, tpb);  // the path kernels' incremental build
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
    const size_t smem = ((size_t)d * 64 + d + 2 * 2 * 4 * d + d) * 4;
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
    const size_t smem = method != kQmc ? 0 : ((size_t)d * 64 + d + 2 * 2 * 4 * d + d) * 4;
    cudaError_t e =
        cudaFuncSetAttribute(normals_hook_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    normals_hook_kernel<<<grid, 128, smem, st>>>(d_vscr, d_shift, d, k_begin, k_end, method, seed, rep, owen, d_out);
    ++launch_counter();
    return cudaGetLastError();
}

}  // namespace qmccpw
