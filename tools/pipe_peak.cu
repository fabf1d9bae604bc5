// Pipe throughput microbenchmark (B200): DFMA (FP64 pipe), FFMA (FMA pipe) and
// MUFU.EX2 issue rates, many independent chains per thread, full device.
// Output: one JSON line (ops/s, per-SM ops/clk at the measured clock).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/pipe_peak tools/pipe_peak.cu
#include <cstdio>
#include <cuda_runtime.h>

constexpr int kChains = 8, kIters = 4096;

__global__ void dfma_kernel(double* out, double a, double b) {
    double x[kChains];
#pragma unroll
    for (int c = 0; c < kChains; ++c) x[c] = threadIdx.x * 1e-3 + c;
    for (int i = 0; i < kIters; ++i)
#pragma unroll
        for (int c = 0; c < kChains; ++c) x[c] = fma(x[c], a, b);
    double s = 0;
#pragma unroll
    for (int c = 0; c < kChains; ++c) s += x[c];
    if (s == 12345.0) out[0] = s;
}

__global__ void ffma_kernel(float* out, float a, float b) {
    float x[kChains];
#pragma unroll
    for (int c = 0; c < kChains; ++c) x[c] = threadIdx.x * 1e-3f + c;
    for (int i = 0; i < kIters; ++i)
#pragma unroll
        for (int c = 0; c < kChains; ++c) x[c] = fmaf(x[c], a, b);
    float s = 0;
#pragma unroll
    for (int c = 0; c < kChains; ++c) s += x[c];
    if (s == 12345.0f) out[0] = s;
}

__global__ void ex2_kernel(float* out) {
    float x[kChains];
#pragma unroll
    for (int c = 0; c < kChains; ++c) x[c] = -1e-3f * (threadIdx.x + c);
    for (int i = 0; i < kIters; ++i)
#pragma unroll
        for (int c = 0; c < kChains; ++c) asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(x[c]));
    float s = 0;
#pragma unroll
    for (int c = 0; c < kChains; ++c) s += x[c];
    if (s == 12345.0f) out[0] = s;
}

template <class F>
double rate(F launch, double ops) {
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    launch();
    cudaDeviceSynchronize();
    float best = 1e30f;
    for (int r = 0; r < 5; ++r) {
        cudaEventRecord(a);
        launch();
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        if (ms < best) best = ms;
    }
    return ops / (best * 1e-3);
}

int main() {
    cudaDeviceProp p;
    cudaGetDeviceProperties(&p, 0);
    int clk_khz = 0;
    cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, 0);
    const int sms = p.multiProcessorCount, blocks = sms * 8, threads = 256;
    const double ops = (double)blocks * threads * kIters * kChains;
    double* d;
    cudaMalloc(&d, 64);
    const double r64 = rate([&] { dfma_kernel<<<blocks, threads>>>(d, 0.999999, 1e-7); }, ops);
    const double r32 = rate([&] { ffma_kernel<<<blocks, threads>>>((float*)d, 0.999f, 1e-4f); }, ops);
    const double rex = rate([&] { ex2_kernel<<<blocks, threads>>>((float*)d); }, ops);
    const double hz = clk_khz * 1e3;
    printf("{\"sms\": %d, \"clock_mhz_attr\": %.0f, \"dfma_per_s\": %.4e, \"ffma_per_s\": %.4e, "
           "\"ex2_per_s\": %.4e, \"dfma_per_sm_clk\": %.2f, \"ffma_per_sm_clk\": %.2f, "
           "\"ex2_per_sm_clk\": %.2f}\n",
           sms, hz / 1e6, r64, r32, rex, r64 / sms / hz, r32 / sms / hz, rex / sms / hz);
    return 0;
}
