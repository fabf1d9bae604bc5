// atomic_peak.cu -- R_atom: the float64 atomic (RED) throughput of a B200 at the
// address spreads the raster kernel produces (SURVEY.md §8(d) asks for it; it
// is not in MEASURED_PEAKS.json).  Standalone measurement tool, not product code.
//
// Patterns (one float64 atomicAdd per active lane per iteration, return value
// unused -> RED.E.ADD.F64):
//   rand32   32 active lanes, independent uniformly random addresses
//   rand16   16 active lanes (the raster's grouped path fires <= 16 per warp)
//   coal     32 lanes, one contiguous 256 B segment per warp instruction
//   f32      rand32 with float32 (the north star's fp32 N x L alternative)
//   fixed_pair_rand16  the deterministic accumulator's add: two u64 REDs into the
//            (hi, lo) words of one 16-byte entry, 16 random lanes (entry adds/s,
//            over the doubled accumulator size of the same config)
// over accumulators of 16 MB (C2: E=2 x 1 M float64), 256 MB (C3) and
// 1.5 GB (C4: E=64 x 3 M).  CUDA events, best of 5 after a warm-up.
//
// build + run (GPU box): nvcc -gencode arch=compute_100a,code=sm_100a -O3 \
//   -o /tmp/atomic_peak tools/atomic_peak.cu && /tmp/atomic_peak > profiles/r1_atomic_peak.json
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

#define CK(x)                                                                   \
    do {                                                                        \
        cudaError_t e_ = (x);                                                   \
        if (e_ != cudaSuccess) {                                                \
            fprintf(stderr, "%s: %s\n", #x, cudaGetErrorString(e_));            \
            exit(1);                                                            \
        }                                                                       \
    } while (0)

__device__ __forceinline__ unsigned long long mix(unsigned long long x) {
    x ^= x >> 33;
    x *= 0xff51afd7ed558ccdull;
    x ^= x >> 33;
    x *= 0xc4ceb9fe1a85ec53ull;
    x ^= x >> 33;
    return x;
}

enum Pattern { kRand32 = 0, kRand16 = 1, kCoal = 2 };

template <typename T, int kPattern>
__global__ void __launch_bounds__(256) red_kernel(T* acc, unsigned long long n, int iters,
                                                  unsigned long long seed) {
    const unsigned long long t = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x;
    const int lane = threadIdx.x & 31;
    const unsigned long long warp = t >> 5, nwarps = (gridDim.x * (unsigned long long)blockDim.x) >> 5;
    unsigned long long h = mix(t ^ seed);
    for (int i = 0; i < iters; ++i) {
        unsigned long long idx;
        if (kPattern == kCoal) {
            idx = (((warp + (unsigned long long)i * nwarps) * 32ull) + lane) % n;
        } else {
            h = mix(h + 0x9e3779b97f4a7c15ull);
            idx = h % n;
        }
        if (kPattern != kRand16 || lane < 16) atomicAdd(acc + idx, (T)1);
    }
}

// The deterministic accumulator's add (FS_ACC_FIXED): two uint64 REDs into the
// (hi, lo) words of one 16-byte entry, 16 random lanes per warp instruction.
__global__ void __launch_bounds__(256) fixed_pair_kernel(unsigned long long* acc,
                                                         unsigned long long n_entries, int iters,
                                                         unsigned long long seed) {
    const unsigned long long t = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x;
    const int lane = threadIdx.x & 31;
    unsigned long long h = mix(t ^ seed);
    for (int i = 0; i < iters; ++i) {
        h = mix(h + 0x9e3779b97f4a7c15ull);
        unsigned long long* p = acc + 2 * (h % n_entries);
        if (lane < 16) {
            asm volatile("red.global.add.u64 [%0], %1;" ::"l"(p), "l"(h >> 40) : "memory");
            asm volatile("red.global.add.u64 [%0], %1;" ::"l"(p + 1), "l"(h & 0xffffffffull)
                         : "memory");
        }
    }
}

static double run_fixed(unsigned long long* acc, unsigned long long n_entries) {
    const int blocks = 148 * 8, threads = 256, iters = 256;
    cudaEvent_t a, b;
    CK(cudaEventCreate(&a));
    CK(cudaEventCreate(&b));
    fixed_pair_kernel<<<blocks, threads>>>(acc, n_entries, iters, 1);
    CK(cudaDeviceSynchronize());
    float best = 1e30f;
    for (int r = 0; r < 5; ++r) {
        CK(cudaEventRecord(a));
        fixed_pair_kernel<<<blocks, threads>>>(acc, n_entries, iters, 2 + r);
        CK(cudaEventRecord(b));
        CK(cudaEventSynchronize(b));
        float ms;
        CK(cudaEventElapsedTime(&ms, a, b));
        if (ms < best) best = ms;
    }
    CK(cudaEventDestroy(a));
    CK(cudaEventDestroy(b));
    return (double)blocks * threads / 32 * 16 * iters / (best * 1e-3);  // entry adds per second
}

template <typename T, int kPattern>
static double run(T* acc, unsigned long long n, int lanes) {
    const int blocks = 148 * 8, threads = 256, iters = 256;
    cudaEvent_t a, b;
    CK(cudaEventCreate(&a));
    CK(cudaEventCreate(&b));
    red_kernel<T, kPattern><<<blocks, threads>>>(acc, n, iters, 1);
    CK(cudaDeviceSynchronize());
    float best = 1e30f;
    for (int r = 0; r < 5; ++r) {
        CK(cudaEventRecord(a));
        red_kernel<T, kPattern><<<blocks, threads>>>(acc, n, iters, 2 + r);
        CK(cudaEventRecord(b));
        CK(cudaEventSynchronize(b));
        float ms;
        CK(cudaEventElapsedTime(&ms, a, b));
        if (ms < best) best = ms;
    }
    CK(cudaEventDestroy(a));
    CK(cudaEventDestroy(b));
    const double ops = (double)blocks * threads / 32 * lanes * iters;
    return ops / (best * 1e-3);  // atomics per second
}

int main() {
    cudaDeviceProp p;
    CK(cudaGetDeviceProperties(&p, 0));
    int clk_khz = 0;
    CK(cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, 0));
    const unsigned long long sizes[3] = {16ull << 20, 256ull << 20, 1536ull << 20};
    // the fixed-point accumulator of the same configs is twice as large (16 B per entry)
    const unsigned long long fixed_sizes[3] = {32ull << 20, 512ull << 20, 3072ull << 20};
    const char* names[3] = {"16MB_C2", "256MB_C3", "1536MB_C4"};
    void* buf;
    CK(cudaMalloc(&buf, fixed_sizes[2]));
    CK(cudaMemset(buf, 0, fixed_sizes[2]));
    printf("{\n \"device\": \"%s\", \"sms\": %d, \"sm_clock_mhz_nominal\": %d,\n", p.name,
           p.multiProcessorCount, clk_khz / 1000);
    printf(" \"how\": \"tools/atomic_peak.cu: %d blocks x 256 threads x 256 iterations of atomicAdd "
           "(RED, result unused), best of 5, CUDA events\",\n",
           148 * 8);
    printf(" \"unit\": \"G atomics/s\",\n \"results\": {\n");
    for (int s = 0; s < 3; ++s) {
        const unsigned long long n64 = sizes[s] / 8, n32 = sizes[s] / 4;
        const double r32 = run<double, kRand32>((double*)buf, n64, 32);
        const double r16 = run<double, kRand16>((double*)buf, n64, 16);
        const double rc = run<double, kCoal>((double*)buf, n64, 32);
        const double rf = run<float, kRand32>((float*)buf, n32, 32);
        const double rx = run_fixed((unsigned long long*)buf, fixed_sizes[s] / 16);
        printf("  \"%s\": {\"f64_rand32\": %.2f, \"f64_rand16\": %.2f, \"f64_coalesced\": %.2f, "
               "\"f32_rand32\": %.2f, \"fixed_pair_rand16\": %.2f}%s\n",
               names[s], r32 * 1e-9, r16 * 1e-9, rc * 1e-9, rf * 1e-9, rx * 1e-9, s < 2 ? "," : "");
    }
    printf(" }\n}\n");
    CK(cudaFree(buf));
    return 0;
}
