// qmccpw_microbench.cu -- FP64 roof microbenchmarks on sm_100a.
//
// Measures the denominators of the roofline the path kernel is reported
// against: DFMA lane-throughput at full occupancy (independent chains), the
// dependent-DFMA latency (one chain, one warp), and FP64 tensor-core (DMMA
// m8n8k4) throughput.  Timed with CUDA events on the given stream.
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/qmccpw.h"
#include "qmccpw_internal.h"

namespace qmccpw {

// ILP independent chains per thread, the iteration loop unrolled 4x so that loop overhead is
// ~1 instruction per 32 DFMAs; block 0 / thread 0 records clock64() and %globaltimer at both
// ends, so the caller gets the SM clock the run actually saw (cycles / ns of the same span)
template <int ILP>
__global__ void dfma_throughput_kernel(double* out, int iters, double a, double b, long long* cycles) {
    double x[ILP];
#pragma unroll
    for (int i = 0; i < ILP; ++i) x[i] = (double)(threadIdx.x + i) * 1e-3;
    long long g0;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g0));
    const long long t0 = clock64();
#pragma unroll 4
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < ILP; ++i) x[i] = fma(x[i], a, b);
    }
    const long long t1 = clock64();
    long long g1;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g1));
    double s = 0.0;
#pragma unroll
    for (int i = 0; i < ILP; ++i) s += x[i];
    if (s == 12345.678) out[blockIdx.x] = s;  // keep the chains alive
    if (blockIdx.x == 0 && threadIdx.x == 0 && cycles) {
        cycles[0] = t1 - t0;  // SM cycles and nanoseconds of the same span: the clock it ran at
        cycles[1] = g1 - g0;
    }
}

__global__ void dfma_latency_kernel(double* out, int iters, double a, double b, long long* cycles) {
    double x = threadIdx.x * 1e-3;
    const long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
        x = fma(x, a, b);
        x = fma(x, a, b);
        x = fma(x, a, b);
        x = fma(x, a, b);
    }
    const long long t1 = clock64();
    if (threadIdx.x == 0) *cycles = t1 - t0;
    if (x == 12345.678) out[0] = x;
}

__global__ void dmma_throughput_kernel(double* out, int iters) {
    double a = threadIdx.x * 1e-3, b = 1.0 - threadIdx.x * 1e-3;
    double c0[2] = {0, 0}, c1[2] = {0, 0}, c2[2] = {0, 0}, c3[2] = {0, 0};
    for (int it = 0; it < iters; ++it) {
        asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                     : "+d"(c0[0]), "+d"(c0[1]) : "d"(a), "d"(b));
        asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                     : "+d"(c1[0]), "+d"(c1[1]) : "d"(a), "d"(b));
        asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                     : "+d"(c2[0]), "+d"(c2[1]) : "d"(a), "d"(b));
        asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                     : "+d"(c3[0]), "+d"(c3[1]) : "d"(a), "d"(b));
    }
    const double s = c0[0] + c0[1] + c1[0] + c1[1] + c2[0] + c2[1] + c3[0] + c3[1];
    if (s == 12345.678) out[blockIdx.x] = s;
}

}  // namespace qmccpw

using namespace qmccpw;

extern "C" int qmccpw_fp64_roof(int32_t device, double* dfma_tflops, double* dfma_latency_cycles,
                                double* dmma_tflops, double* sm_clock_mhz) {
    if (!dfma_tflops || !dfma_latency_cycles || !dmma_tflops || !sm_clock_mhz) return QMCCPW_EINVAL;
    if (cudaSetDevice(device) != cudaSuccess) return QMCCPW_ECUDA;
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
    double* d_out = nullptr;
    long long* d_cyc = nullptr;
    if (cudaMalloc(&d_out, 1 << 20) != cudaSuccess) return QMCCPW_ENOMEM;
    cudaMalloc(&d_cyc, 2 * sizeof(long long));
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    float ms = 0.f;
    // DFMA: 8 independent chains per thread, 4 blocks x 256 threads per SM (32 warps), long
    // enough (~0.2 s) that launch and tail effects are < 0.1 %
    const int iters = 1 << 16, blocks = sms * 4, tpb = 256;
    dfma_throughput_kernel<8><<<blocks, tpb>>>(d_out, 1024, 0.999999, 1e-7, nullptr);  // warm-up
    cudaEventRecord(e0);
    dfma_throughput_kernel<8><<<blocks, tpb>>>(d_out, iters, 0.999999, 1e-7, d_cyc);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    *dfma_tflops = 2.0 * 8.0 * iters * (double)blocks * tpb / (ms * 1e-3) / 1e12;
    long long span[2] = {0, 1};
    cudaMemcpy(span, d_cyc, sizeof span, cudaMemcpyDeviceToHost);
    *sm_clock_mhz = span[1] > 0 ? (double)span[0] / (double)span[1] * 1e3 : 0.0;  // cycles per ns -> MHz
    launch_counter() += 2;
    // latency: one warp, one dependent chain
    dfma_latency_kernel<<<1, 32>>>(d_out, 4096, 0.999999, 1e-7, d_cyc);
    long long cyc = 0;
    cudaMemcpy(&cyc, d_cyc, sizeof cyc, cudaMemcpyDeviceToHost);
    *dfma_latency_cycles = (double)cyc / (4.0 * 4096);
    launch_counter() += 1;
    // clock under a long DFMA load: elapsed SM cycles vs time
    // DMMA m8n8k4: 256 FMA = 512 FLOP per warp instruction, 4 independent accumulators
    const int diters = 2048, dblocks = sms * 8, dtpb = 256;
    dmma_throughput_kernel<<<dblocks, dtpb>>>(d_out, 16);
    cudaEventRecord(e0);
    dmma_throughput_kernel<<<dblocks, dtpb>>>(d_out, diters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    *dmma_tflops = 512.0 * 4.0 * diters * (double)dblocks * (dtpb / 32) / (ms * 1e-3) / 1e12;
    launch_counter() += 2;
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    cudaFree(d_out);
    cudaFree(d_cyc);
    return cudaGetLastError() == cudaSuccess ? QMCCPW_OK : QMCCPW_ECUDA;
}
