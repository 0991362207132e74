// fp64_mix_bench.cu -- does the FP64 tensor core (DMMA) share the FP64 datapath with DFMA on
// sm_100a?  Times DFMA alone, DMMA alone and both interleaved in one kernel; if they share it,
// the mixed kernel's combined FMA rate equals the single-pipe peak, else it approaches the sum.
// Build + run (on a B200): nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/mix fp64_mix_bench.cu && /tmp/mix
#include <cstdio>
#include <cuda_runtime.h>

template <int NF, int NM>
__global__ void mix(double* out, int iters, double a, double b) {
    double x[8];
    for (int i = 0; i < 8; ++i) x[i] = threadIdx.x * 1e-3 + i;
    double c[4][2] = {{0, 0}, {0, 0}, {0, 0}, {0, 0}};
    double fa = threadIdx.x * 1e-3, fb = 1.0 - fa;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int r = 0; r < NF; ++r)
#pragma unroll
            for (int i = 0; i < 8; ++i) x[i] = fma(x[i], a, b);
#pragma unroll
        for (int r = 0; r < NM; ++r)
#pragma unroll
            for (int i = 0; i < 4; ++i)
                asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                             : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(fa), "d"(fb));
    }
    double s = 0;
    for (int i = 0; i < 8; ++i) s += x[i];
    for (int i = 0; i < 4; ++i) s += c[i][0] + c[i][1];
    if (s == 1234.5) out[0] = s;
}

template <int NF, int NM>
void run(const char* name, int sms) {
    double* d;
    cudaMalloc(&d, 8);
    const int blocks = sms * 4, tpb = 256, iters = 1 << 14;
    mix<NF, NM><<<blocks, tpb>>>(d, 64, 0.999, 1e-7);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    mix<NF, NM><<<blocks, tpb>>>(d, iters, 0.999, 1e-7);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    const double thr = (double)blocks * tpb, warps = thr / 32;
    const double dfma = thr * iters * NF * 8, dmma_fma = warps * iters * NM * 4 * 256.0;
    printf("%-28s %8.3f ms  DFMA %6.2f TFLOP/s  DMMA %6.2f TFLOP/s  total %6.2f TFLOP/s\n", name, ms,
           2 * dfma / ms / 1e9, 2 * dmma_fma / ms / 1e9, 2 * (dfma + dmma_fma) / ms / 1e9);
    cudaFree(d);
}

// DFMA-only variants: chain count, operands from registers (b loaded per thread) or constants
template <int ILP, bool REG>
__global__ void dfma_only(double* out, int iters, double a, double b) {
    double x[ILP];
    for (int i = 0; i < ILP; ++i) x[i] = threadIdx.x * 1e-3 + i;
    double ra = a + threadIdx.x * 1e-12, rb = b + threadIdx.x * 1e-15;
#pragma unroll 2
    for (int it = 0; it < iters; ++it)
#pragma unroll
        for (int i = 0; i < ILP; ++i) x[i] = REG ? fma(x[i], ra, rb) : fma(x[i], a, b);
    double s = 0;
    for (int i = 0; i < ILP; ++i) s += x[i];
    if (s == 1234.5) out[0] = s;
}
template <int ILP, bool REG>
void run_only(const char* name, int sms, int bps, int tpb) {
    double* d;
    cudaMalloc(&d, 8);
    const int blocks = sms * bps, iters = (1 << 17) / ILP;
    dfma_only<ILP, REG><<<blocks, tpb>>>(d, 64, 0.999, 1e-7);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    dfma_only<ILP, REG><<<blocks, tpb>>>(d, iters, 0.999, 1e-7);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    printf("%-40s %8.3f ms  DFMA %6.2f TFLOP/s\n", name, ms, 2.0 * blocks * tpb * (double)iters * ILP / ms / 1e9);
    cudaFree(d);
}

int main() {
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    run<4, 0>("DFMA only (32/iter)", sms);
    run<0, 1>("DMMA only (4/iter)", sms);
    run<4, 1>("DFMA 32 + DMMA 4 per iter", sms);
    run<2, 1>("DFMA 16 + DMMA 4 per iter", sms);
    run<4, 2>("DFMA 32 + DMMA 8 per iter", sms);
    run_only<8, false>("DFMA ILP8 const operands 4x256", sms, 4, 256);
    run_only<8, true>("DFMA ILP8 register operands 4x256", sms, 4, 256);
    run_only<16, true>("DFMA ILP16 register operands 4x256", sms, 4, 256);
    run_only<4, true>("DFMA ILP4 register operands 8x256", sms, 8, 256);
    run_only<8, true>("DFMA ILP8 register operands 2x512", sms, 2, 512);
    run_only<8, true>("DFMA ILP8 register operands 8x128", sms, 8, 128);
    return 0;
}
