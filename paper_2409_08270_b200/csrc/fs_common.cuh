// fs_common.cuh -- shared device types and helpers for the FlashSplat B200 label solver.
//
// Numerics contract: every quantity that feeds a
// discrete decision of the reference (cull, radius, tile range, depth order,
// alpha floor, transmittance floor) or a contribution weight is computed in
// float64 with the reference's operation order and without FMA contraction
// (explicit __d*_rn intrinsics or -fmad=false).  float32 is only used for a
// conservative pre-screen that rejects samples whose alpha is certainly
// below the floor.
#pragma once

#include <cstdint>
#include <cstdio>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

// Device-side bounds / invariant checks, compiled in only for the checked build
// (make checked -> _lib_checked/, FS_LIB=checked): compute-sanitizer is not
// available on the GPU pool, so the shared-memory and global indices the
// kernels compute are asserted instead and the GPU test-suite is run against
// that build.  A failed check prints its location and traps.
#ifdef FS_CHECKS
#define FS_CHECK(cond)                                                                     \
    do {                                                                                   \
        if (!(cond)) {                                                                     \
            printf("FS_CHECK failed %s:%d: %s (block %d thread %d)\n", __FILE__, __LINE__, \
                   #cond, (int)blockIdx.x, (int)threadIdx.x);                              \
            __trap();                                                                      \
        }                                                                                  \
    } while (0)
#else
#define FS_CHECK(cond) \
    do {               \
    } while (0)
#endif

namespace fs {

constexpr int kTile = 16;             // rasterizer.py:31
constexpr int kTilePixels = kTile * kTile;
constexpr double kDilation = 0.3;     // scene.py:25
constexpr double kAlphaClamp = 0.99;  // scene.py:26
constexpr double kDegenerateDet = 1e-12;  // scene.py:27

// Per-view camera, passed by value to kernels (scene.py:164-203).
struct Camera {
    int32_t width, height;
    double fx, fy, cx, cy;
    double w2c[16];
    double near_clip;
};

// float32 screen record of one projected Gaussian (32 B, one per scene slot).
// cut: power threshold below which alpha < alpha_floor for sure;
// hxy: half extents (hx, hy) of the alpha-floor ellipse, pixel units, inflated
//      and rounded UP to float16 (rec_hx / rec_hy: exact float32 values, the
//      same ones for the binning's tile cull and the raster's strip test);
// oid: the Gaussian's input id (accumulator row, channel row) -- scenes are
//      stored in spatial order (fs_order.cu), so it differs from the slot.
struct __align__(16) Rec32 {
    float mx, my, a, b, c, cut;
    unsigned int hxy, oid;
};
__device__ __forceinline__ unsigned int pack_hxy(float hx, float hy) {
    const __half2 h = __halves2half2(__float2half_ru(hx), __float2half_ru(hy));
    return *reinterpret_cast<const unsigned int*>(&h);
}
__device__ __forceinline__ float rec_hx(const Rec32& s) {
    return __half2float(__ushort_as_half((unsigned short)(s.hxy & 0xffffu)));
}
__device__ __forceinline__ float rec_hy(const Rec32& s) {
    return __half2float(__ushort_as_half((unsigned short)(s.hxy >> 16)));
}

// float64 record used for the exact contribution (48 B, one per gid).
struct __align__(16) Rec64 {
    double mx, my, a, b, c, o;
};

// Per-view device counters (reset at the start of every view).
struct ViewCounters {
    unsigned long long key_or;   // OR of visible depth keys
    unsigned long long key_nand; // OR of the complemented keys (= ~AND): all-zero is the empty state
    unsigned int n_emitted;      // visible after all culls (scene.py:311)
    unsigned int n_behind;
    unsigned int n_degenerate;
    unsigned int n_offscreen;
    unsigned int n_instances;    // (tile, gaussian) pairs emitted
    unsigned int n_valid;        // n_instances, or 0 when it overflowed the buffers
    unsigned int overflow;       // instances exceeded capacity -> view skipped
    unsigned int max_label;      // largest out-of-range mask label (>= E) seen by the raster kernel, else 0
    unsigned long long tile_steps;   // list entries walked by the raster kernel
    unsigned long long exact_evals;  // float64 alpha evaluations
    unsigned long long atomics;      // global accumulator atomics issued
};

// Device-side projection export for the stage-level API (scene.py:252-312).
struct ProjectExport {
    uint8_t* alive;
    double* mean2d;  // N x 2
    double* conic;   // N x 3
    double* depth;   // N
    int64_t* radius; // N
    const uint8_t* member;  // N, input, nullable: only members are binned (render subsets,
                            // project_scene(member_mask=...), scene.py:346-350)
    const unsigned int* perm;  // nullable: scene slot p holds input Gaussian perm[p]
                               // (fs_order.cu); exports and member are by input id
};

__host__ __device__ inline int tiles_x_of(int w) { return (w + kTile - 1) / kTile; }
__host__ __device__ inline int tiles_y_of(int h) { return (h + kTile - 1) / kTile; }

// Order-preserving map of a float64 to uint64 (valid for all non-NaN values).
__device__ __forceinline__ unsigned long long f64_sort_key(double z) {
    unsigned long long b = static_cast<unsigned long long>(__double_as_longlong(z));
    return (b >> 63) ? ~b : (b | 0x8000000000000000ull);
}

// Packed inclusive tile rectangle: tx0 | tx1 << 16 | ty0 << 32 | ty1 << 48.
// Empty rectangles (tx0 > tx1 or ty0 > ty1) are stored as 0xFFFF... -> count 0.
__device__ __forceinline__ unsigned int rect_count(unsigned long long r) {
    if (r == ~0ull) return 0u;
    unsigned int tx0 = r & 0xFFFF, tx1 = (r >> 16) & 0xFFFF;
    unsigned int ty0 = (r >> 32) & 0xFFFF, ty1 = (r >> 48) & 0xFFFF;
    return (tx1 - tx0 + 1) * (ty1 - ty0 + 1);
}

// Records a CUDA failure as the thread's last error; returns FS_ECUDA.
int set_cuda_error(cudaError_t e, const char* expr, const char* file, int line);

}  // namespace fs

#define FS_CUDA_CHECK(expr)                                                    \
    do {                                                                       \
        cudaError_t _e = (expr);                                               \
        if (_e != cudaSuccess) return fs::set_cuda_error(_e, #expr, __FILE__, __LINE__); \
    } while (0)
