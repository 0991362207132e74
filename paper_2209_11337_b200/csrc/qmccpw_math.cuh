// qmccpw_math.cuh -- FP64 device math for the QMC-CPW kernels (sm_100a).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace qmccpw {

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

// (a3) lattice point -> standard normal.  u = (y + 1/2) 2^-32 is exact in
// FP64; the upper half is mirrored, x(2^32-1-y) = -x(y), so the lattice
// symmetry is exact.  The inverse CDF itself is CUDA's normcdfinv.
__device__ __forceinline__ double normal_from_u32(uint32_t y) {
    const bool upper = (y >> 31) != 0u;
    const uint32_t yl = upper ? ~y : y;
    const double u = fma((double)yl, 0x1p-32, 0x1p-33);
    const double x = normcdfinv(u);
    return upper ? -x : x;
}

__device__ __forceinline__ double normal_pdf(double x) {
    return 0.398942280401432677939946059934 * exp(-0.5 * x * x);
}
// Phibar(x) = 1 - Phi(x) = erfc(x/sqrt2)/2, never formed as 1 - Phi (reading 22)
__device__ __forceinline__ double normal_sf(double x) { return 0.5 * erfc(x * 0.707106781186547524400844362105); }
__device__ __forceinline__ double normal_cdf(double x) { return 0.5 * erfc(-x * 0.707106781186547524400844362105); }

}  // namespace qmccpw
