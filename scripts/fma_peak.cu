// FMA throughput microbenchmark (scalar FP32 FFMA, packed FP32x2 FFMA2, FP64
// DFMA): the compute ceilings the pair kernels are held against in DESIGN.md.
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o build/fma_peak scripts/fma_peak.cu
#include <cstdio>
#include <cuda_runtime.h>

constexpr int kChains = 8, kIters = 4096;

__global__ void k_f32(float *out, float a, float b) {
    float x[kChains];
#pragma unroll
    for (int c = 0; c < kChains; ++c) x[c] = threadIdx.x + c;
    for (int i = 0; i < kIters; ++i)
#pragma unroll
        for (int c = 0; c < kChains; ++c) x[c] = fmaf(x[c], a, b);
    float s = 0.f;
#pragma unroll
    for (int c = 0; c < kChains; ++c) s += x[c];
    if (s == 1.2345f) out[0] = s;
}

__global__ void k_f32x2(float *out, float a, float b) {
    unsigned long long x[kChains];
    const unsigned long long av = (unsigned long long)__float_as_uint(a) |
                                  ((unsigned long long)__float_as_uint(a) << 32);
    const unsigned long long bv = (unsigned long long)__float_as_uint(b) |
                                  ((unsigned long long)__float_as_uint(b) << 32);
#pragma unroll
    for (int c = 0; c < kChains; ++c) x[c] = (unsigned long long)(threadIdx.x + c) * 0x100000001ull;
    for (int i = 0; i < kIters; ++i)
#pragma unroll
        for (int c = 0; c < kChains; ++c)
            asm volatile("fma.rn.f32x2 %0, %0, %1, %2;" : "+l"(x[c]) : "l"(av), "l"(bv));
    unsigned long long s = 0;
#pragma unroll
    for (int c = 0; c < kChains; ++c) s ^= x[c];
    if (s == 12345ull) out[0] = 1.f;
}

__global__ void k_f64(double *out, double a, double b) {
    double x[kChains];
#pragma unroll
    for (int c = 0; c < kChains; ++c) x[c] = threadIdx.x + c;
    for (int i = 0; i < kIters; ++i)
#pragma unroll
        for (int c = 0; c < kChains; ++c) x[c] = fma(x[c], a, b);
    double s = 0.0;
#pragma unroll
    for (int c = 0; c < kChains; ++c) s += x[c];
    if (s == 1.2345) out[0] = s;
}

template <class F>
static double best_ms(F launch) {
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    launch();
    cudaDeviceSynchronize();
    float best = 1e30f;
    for (int r = 0; r < 10; ++r) {
        cudaEventRecord(e0);
        launch();
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        best = ms < best ? ms : best;
    }
    return best;
}

int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const int blocks = sms * 8, threads = 256;
    float *fo;
    double *dout;
    cudaMalloc(&fo, 16);
    cudaMalloc(&dout, 16);
    const double fmas = (double)blocks * threads * kIters * kChains;
    const double t32 = best_ms([&] { k_f32<<<blocks, threads>>>(fo, 0.999f, 0.001f); });
    const double t2 = best_ms([&] { k_f32x2<<<blocks, threads>>>(fo, 0.999f, 0.001f); });
    const double t64 = best_ms([&] { k_f64<<<blocks, threads>>>(dout, 0.999, 0.001); });
    printf("{\"sms\": %d, \"fp32_ffma_tflops\": %.1f, \"fp32x2_ffma2_tflops\": %.1f, "
           "\"fp64_dfma_tflops\": %.1f, \"how\": \"%d CTAs x %d threads x %d iters x %d "
           "independent chains, best of 10, 2 flop per FMA (x2 per FFMA2)\"}\n",
           sms, 2 * fmas / t32 * 1e-9, 4 * fmas / t2 * 1e-9, 2 * fmas / t64 * 1e-9, blocks,
           threads, kIters, kChains);
    return cudaGetLastError() != cudaSuccess;
}
