// fs_order.cu -- spatial order of the resident scene.
//
// The resident scene is stored along a Morton (Z-order) curve of the Gaussian
// means instead of in input order: slot p holds input Gaussian perm[p].  Every
// per-view kernel then sees spatially coherent neighbours -- a block of the
// binning's emit kernel scatters its instances into a few tile buckets (runs
// of coalesced stores instead of one 32-B sector per 4-B id), and the raster's
// record gathers hit fewer DRAM pages.  Results do not depend on the order:
// tile lists are sorted by (depth, input id) (the tie id is perm[p]), the
// accumulator rows, exports and caller-side per-Gaussian arrays stay indexed by
// the input id, and the fixed-point sums commute.  Measured upper bound (host
// permutation of the synthetic scenes, tools/morton_probe.py): C2 -2%, C4 -10%.
//
// The order is a stable radix sort of 30-bit Morton codes (10 bits per axis
// over the means' bounding box), so it is deterministic: equal codes keep input
// order.  One-time cost per scene (fs_set_scene / fs_set_scene_ply).
#include <cub/device/device_radix_sort.cuh>

#include "fs_common.cuh"
#include "fs_kernels.cuh"

namespace fs {

namespace {

struct MeanSource {
    const double* aos;   // N x 3 float64 (fs_set_scene), or
    const float* verts;  // PLY records (fs_set_scene_ply)
    int stride, ox, oy, oz;
    __device__ __forceinline__ void get(int i, double& x, double& y, double& z) const {
        if (aos) {
            x = aos[3 * (size_t)i];
            y = aos[3 * (size_t)i + 1];
            z = aos[3 * (size_t)i + 2];
        } else {
            const float* r = verts + (size_t)i * stride;
            x = r[ox];
            y = r[oy];
            z = r[oz];
        }
    }
};

// order-preserving double <-> uint64 (finite values), for 64-bit atomicMin/Max
__device__ __forceinline__ unsigned long long ord_of(double v) {
    const unsigned long long b = (unsigned long long)__double_as_longlong(v);
    return (b >> 63) ? ~b : (b | 0x8000000000000000ull);
}
__device__ __forceinline__ double val_of(unsigned long long u) {
    return __longlong_as_double((long long)((u >> 63) ? (u & 0x7fffffffffffffffull) : ~u));
}

__device__ __forceinline__ unsigned long long warp_min64(unsigned long long v) {
#pragma unroll
    for (int o = 16; o; o >>= 1) {
        const unsigned long long w = __shfl_xor_sync(0xffffffffu, v, o);
        v = w < v ? w : v;
    }
    return v;
}
__device__ __forceinline__ unsigned long long warp_max64(unsigned long long v) {
#pragma unroll
    for (int o = 16; o; o >>= 1) {
        const unsigned long long w = __shfl_xor_sync(0xffffffffu, v, o);
        v = w > v ? w : v;
    }
    return v;
}

// box[0..2] = min, box[3..5] = max of the finite mean coordinates (order-mapped)
__global__ void bbox_kernel(int n, MeanSource src, unsigned long long* __restrict__ box) {
    unsigned long long lo[3] = {~0ull, ~0ull, ~0ull}, hi[3] = {0ull, 0ull, 0ull};
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        double c[3];
        src.get(i, c[0], c[1], c[2]);
#pragma unroll
        for (int a = 0; a < 3; ++a) {
            if (!isfinite(c[a])) continue;
            const unsigned long long u = ord_of(c[a]);
            lo[a] = u < lo[a] ? u : lo[a];
            hi[a] = u > hi[a] ? u : hi[a];
        }
    }
#pragma unroll
    for (int a = 0; a < 3; ++a) {
        lo[a] = warp_min64(lo[a]);
        hi[a] = warp_max64(hi[a]);
        if ((threadIdx.x & 31) == 0) {
            atomicMin(&box[a], lo[a]);
            atomicMax(&box[3 + a], hi[a]);
        }
    }
}

__global__ void bbox_init_kernel(unsigned long long* box) {
    if (threadIdx.x < 6) box[threadIdx.x] = threadIdx.x < 3 ? ~0ull : 0ull;
}

#ifndef FS_MORTON_BITS
#define FS_MORTON_BITS 10  // per axis (<= 10: 30-bit codes)
#endif
constexpr int kBits = FS_MORTON_BITS;
constexpr double kCells = (double)((1 << kBits) - 1);

// 10 bits -> every third bit of 30
__device__ __forceinline__ unsigned int spread3(unsigned int x) {
    x &= 0x3ffu;
    x = (x | (x << 16)) & 0x030000ffu;
    x = (x | (x << 8)) & 0x0300f00fu;
    x = (x | (x << 4)) & 0x030c30c3u;
    x = (x | (x << 2)) & 0x09249249u;
    return x;
}

__global__ void morton_kernel(int n, MeanSource src, const unsigned long long* __restrict__ box,
                              unsigned int* __restrict__ code, unsigned int* __restrict__ idx) {
    double lo[3], scale[3];
#pragma unroll
    for (int a = 0; a < 3; ++a) {
        const bool any = box[a] <= box[3 + a];
        lo[a] = any ? val_of(box[a]) : 0.0;
        const double ext = any ? val_of(box[3 + a]) - lo[a] : 0.0;
        scale[a] = ext > 0.0 ? kCells / ext : 0.0;
    }
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        double c[3];
        src.get(i, c[0], c[1], c[2]);
        unsigned int q[3];
#pragma unroll
        for (int a = 0; a < 3; ++a) {
            const double t = (c[a] - lo[a]) * scale[a];  // NaN / inf clamp below
            q[a] = t >= kCells ? (unsigned int)kCells : (t > 0.0 ? (unsigned int)t : 0u);
        }
        code[i] = spread3(q[0]) | (spread3(q[1]) << 1) | (spread3(q[2]) << 2);
        idx[i] = (unsigned int)i;
    }
}

size_t align256(size_t x) { return (x + 255) & ~(size_t)255; }

size_t cub_temp_bytes(int n) {
    size_t temp = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, temp, (unsigned int*)nullptr, (unsigned int*)nullptr,
                                    (unsigned int*)nullptr, (unsigned int*)nullptr, n, 0,
                                    3 * kBits);
    return temp;
}

// Scratch carved from one caller-owned device buffer (grow-only in the context):
// per-call cudaMallocAsync / cudaFreeAsync here stalled whole solves for up to
// 0.8 s now and then (pool trimming), so nothing is allocated per call.
cudaError_t order_from(int n, MeanSource src, unsigned int* perm, void* scratch,
                       size_t scratch_bytes, int num_sms, cudaStream_t st) {
    if (n <= 0) return cudaSuccess;
    const size_t n4 = align256(4 * (size_t)n), temp_bytes = cub_temp_bytes(n);
    if (scratch_bytes < 256 + 3 * n4 + temp_bytes) return cudaErrorInvalidValue;
    char* p = static_cast<char*>(scratch);
    auto* box = reinterpret_cast<unsigned long long*>(p);
    auto* code = reinterpret_cast<unsigned int*>(p + 256);
    auto* code_sorted = reinterpret_cast<unsigned int*>(p + 256 + n4);
    auto* idx = reinterpret_cast<unsigned int*>(p + 256 + 2 * n4);
    void* temp = p + 256 + 3 * n4;
    size_t tb = temp_bytes;
    bbox_init_kernel<<<1, 32, 0, st>>>(box);
    int grid = (n + 255) / 256;
    if (grid > num_sms * 8) grid = num_sms * 8;
    bbox_kernel<<<grid, 256, 0, st>>>(n, src, box);
    morton_kernel<<<grid, 256, 0, st>>>(n, src, box, code, idx);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    return cub::DeviceRadixSort::SortPairs(temp, tb, code, code_sorted, idx, perm, n, 0, 3 * kBits,
                                           st);
}

}  // namespace

size_t scene_order_scratch_bytes(int n) {
    return n <= 0 ? 0 : 256 + 3 * align256(4 * (size_t)n) + cub_temp_bytes(n);
}

cudaError_t launch_scene_order(int n, const double* means_aos, unsigned int* perm, void* scratch,
                               size_t scratch_bytes, int num_sms, cudaStream_t st) {
    MeanSource src{means_aos, nullptr, 0, 0, 0, 0};
    return order_from(n, src, perm, scratch, scratch_bytes, num_sms, st);
}

cudaError_t launch_scene_order_ply(int n, const float* verts, int stride, const PlyOffsets& off,
                                   unsigned int* perm, void* scratch, size_t scratch_bytes,
                                   int num_sms, cudaStream_t st) {
    MeanSource src{nullptr, verts, stride, off.k[0], off.k[1], off.k[2]};
    return order_from(n, src, perm, scratch, scratch_bytes, num_sms, st);
}

}  // namespace fs
