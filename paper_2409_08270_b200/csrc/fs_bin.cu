// fs_bin.cu -- K2b/K2d: tile binning on the device (reference rasterizer.py:72-113).
//
// Input: all N Gaussians sorted by (depth, gid) (fs_sort.cu), each with its
// inclusive tile rectangle from the projection kernel.  Output: per-tile
// ranges into an instance array whose gids are, within every tile, in
// (depth, gid) order -- exactly TileBinning.tile_lists.
//
//   emit_reduce  per-block instance counts over contiguous rank chunks
//   emit_scan    one block: exclusive scan of the block counts, total, overflow
//   emit_write   block-local scan + write (tile, gid) in rank order
//   tile sort    stable LSD radix over the tile-id bits (fs_sort.cu)
//   tile_ranges  tile_start[t] = first instance of tile t
#include "fs_common.cuh"
#include "fs_kernels.cuh"

namespace fs {

namespace {

constexpr int kBinThreads = 256;

__device__ __forceinline__ void rank_chunk(unsigned int n, int b, int g, unsigned int& lo,
                                           unsigned int& hi) {
    unsigned int chunk = (n + g - 1) / g;
    chunk = (chunk + 255u) & ~255u;
    lo = min((unsigned long long)n, (unsigned long long)chunk * b);
    hi = min((unsigned long long)n, (unsigned long long)chunk * (b + 1));
}

__device__ __forceinline__ unsigned int block_sum(unsigned int v, unsigned int* s_warp) {
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    __syncthreads();
    if (lane == 0) s_warp[warp] = v;
    __syncthreads();
    unsigned int t = 0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += s_warp[w];
    return t;
}

// exclusive block scan; returns exclusive prefix, *total = block total
__device__ __forceinline__ unsigned int block_exclusive_scan(unsigned int v, unsigned int* s_warp,
                                                             unsigned int* total) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    unsigned int x = v;
    for (int o = 1; o < 32; o <<= 1) {
        unsigned int y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    __syncthreads();
    if (lane == 31) s_warp[warp] = x;
    __syncthreads();
    unsigned int base = 0, tot = 0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) {
        unsigned int s = s_warp[w];
        if (w < warp) base += s;
        tot += s;
    }
    *total = tot;
    return base + x - v;
}

__global__ void __launch_bounds__(kBinThreads) emit_reduce_kernel(
    int n, const unsigned int* __restrict__ v0, const unsigned int* __restrict__ v1,
    const unsigned long long* __restrict__ depth_oa, const unsigned long long* __restrict__ rect,
    unsigned int* __restrict__ block_sums) {
    __shared__ unsigned int s_warp[kBinThreads / 32];
    const unsigned int* gids = pass_parity(depth_oa[0] ^ depth_oa[1], 8) ? v1 : v0;
    unsigned int lo, hi;
    rank_chunk((unsigned)n, blockIdx.x, gridDim.x, lo, hi);
    unsigned int s = 0;
    for (unsigned int r = lo + threadIdx.x; r < hi; r += kBinThreads) s += rect_count(rect[gids[r]]);
    s = block_sum(s, s_warp);
    if (threadIdx.x == 0) block_sums[blockIdx.x] = s;
}

__global__ void __launch_bounds__(1024) emit_scan_kernel(unsigned int* __restrict__ block_sums,
                                                          int g, unsigned int capacity,
                                                          ViewCounters* __restrict__ vc) {
    __shared__ unsigned long long s[1024];
    unsigned long long v = threadIdx.x < (unsigned)g ? block_sums[threadIdx.x] : 0ull;
    s[threadIdx.x] = v;
    __syncthreads();
    for (int off = 1; off < 1024; off <<= 1) {
        unsigned long long y = threadIdx.x >= (unsigned)off ? s[threadIdx.x - off] : 0ull;
        __syncthreads();
        s[threadIdx.x] += y;
        __syncthreads();
    }
    if (threadIdx.x < (unsigned)g) block_sums[threadIdx.x] = (unsigned int)(s[threadIdx.x] - v);
    if (threadIdx.x == 1023) {
        unsigned long long total = s[1023];
        bool over = total > capacity;
        vc->n_instances = total > 0xFFFFFFFFull ? 0xFFFFFFFFu : (unsigned int)total;
        vc->overflow = over ? 1u : 0u;
        vc->n_valid = over ? 0u : (unsigned int)total;
    }
}

__global__ void __launch_bounds__(kBinThreads) emit_write_kernel(
    int n, int tiles_x, const unsigned int* __restrict__ v0, const unsigned int* __restrict__ v1,
    const unsigned long long* __restrict__ depth_oa, const unsigned long long* __restrict__ rect,
    const unsigned int* __restrict__ block_offsets, unsigned int* __restrict__ ikeys,
    unsigned int* __restrict__ ivals, const ViewCounters* __restrict__ vc) {
    if (vc->overflow) return;
    __shared__ unsigned int s_warp[kBinThreads / 32];
    const unsigned int* gids = pass_parity(depth_oa[0] ^ depth_oa[1], 8) ? v1 : v0;
    unsigned int lo, hi;
    rank_chunk((unsigned)n, blockIdx.x, gridDim.x, lo, hi);
    unsigned int running = block_offsets[blockIdx.x];
    for (unsigned int base = lo; base < hi; base += kBinThreads) {
        unsigned int r = base + threadIdx.x;
        unsigned int gid = 0, cnt = 0;
        unsigned long long rc = ~0ull;
        if (r < hi) {
            gid = gids[r];
            rc = rect[gid];
            cnt = rect_count(rc);
        }
        unsigned int total;
        unsigned int pos = running + block_exclusive_scan(cnt, s_warp, &total);
        if (cnt) {
            unsigned int tx0 = rc & 0xFFFF, tx1 = (rc >> 16) & 0xFFFF;
            unsigned int ty0 = (rc >> 32) & 0xFFFF, ty1 = (rc >> 48) & 0xFFFF;
            for (unsigned int ty = ty0; ty <= ty1; ++ty)
                for (unsigned int tx = tx0; tx <= tx1; ++tx) {
                    ikeys[pos] = ty * (unsigned)tiles_x + tx;
                    ivals[pos] = gid;
                    ++pos;
                }
        }
        running += total;
    }
}

__global__ void tile_ranges_kernel(int ntiles, int tile_passes, const unsigned int* __restrict__ k0,
                                   const unsigned int* __restrict__ k1,
                                   const unsigned long long* __restrict__ tile_oa,
                                   unsigned int* __restrict__ tile_start,
                                   const ViewCounters* __restrict__ vc) {
    const unsigned int n = vc->n_valid;
    const unsigned int* keys = pass_parity(tile_oa[0] ^ tile_oa[1], tile_passes) ? k1 : k0;
    const unsigned int stride = gridDim.x * blockDim.x;
    const unsigned int tid = blockIdx.x * blockDim.x + threadIdx.x;
    if (n == 0) {
        for (unsigned int t = tid; t <= (unsigned)ntiles; t += stride) tile_start[t] = 0;
        return;
    }
    for (unsigned int i = tid; i < n; i += stride) {
        unsigned int k = keys[i];
        int prev = i ? (int)keys[i - 1] : -1;
        for (int t = prev + 1; t <= (int)k; ++t) tile_start[t] = i;
        if (i == n - 1)
            for (int t = (int)k + 1; t <= ntiles; ++t) tile_start[t] = n;
    }
}


// ---- binning of an explicit splat list (TileBinning over ProjectedGaussian) ----

__device__ __forceinline__ void block_or_and(unsigned long long o, unsigned long long a,
                                             unsigned long long* dst) {
    for (int off = 16; off > 0; off >>= 1) {
        o |= __shfl_xor_sync(0xffffffffu, o, off);
        a &= __shfl_xor_sync(0xffffffffu, a, off);
    }
    if ((threadIdx.x & 31) == 0) {
        atomicOr(dst, o);
        atomicAnd(dst + 1, a);
    }
}

// keys = gaussian index (secondary sort key), vals = list position, rect per position
__global__ void splat_index_kernel(int k, const long long* __restrict__ index,
                                   const double* __restrict__ mean2d,
                                   const long long* __restrict__ radius, int width, int height,
                                   unsigned long long* __restrict__ keys,
                                   unsigned int* __restrict__ vals,
                                   unsigned long long* __restrict__ rect,
                                   unsigned long long* __restrict__ oa) {
    const int tx_n = tiles_x_of(width), ty_n = tiles_y_of(height);
    const int stride = gridDim.x * blockDim.x;
    const int iters = (k + stride - 1) / stride;
    unsigned long long o = 0, a = ~0ull;
    for (int it = 0; it < iters; ++it) {
        int i = it * stride + blockIdx.x * blockDim.x + threadIdx.x;
        if (i < k) {
            unsigned long long key = (unsigned long long)index[i] ^ 0x8000000000000000ull;
            keys[i] = key;
            vals[i] = (unsigned)i;
            o |= key;
            a &= key;
            double mx = mean2d[2 * i], my = mean2d[2 * i + 1], r = (double)radius[i];
            double fx0 = floor((mx - r) / kTile), fx1 = floor((mx + r) / kTile);
            double fy0 = floor((my - r) / kTile), fy1 = floor((my + r) / kTile);
            int tx0 = fx0 < 0.0 ? 0 : (fx0 > tx_n ? tx_n : (int)fx0);
            int tx1 = fx1 > tx_n - 1 ? tx_n - 1 : (fx1 < -1.0 ? -1 : (int)fx1);
            int ty0 = fy0 < 0.0 ? 0 : (fy0 > ty_n ? ty_n : (int)fy0);
            int ty1 = fy1 > ty_n - 1 ? ty_n - 1 : (fy1 < -1.0 ? -1 : (int)fy1);
            rect[i] = (tx0 <= tx1 && ty0 <= ty1)
                          ? ((unsigned long long)tx0 | ((unsigned long long)tx1 << 16) |
                             ((unsigned long long)ty0 << 32) | ((unsigned long long)ty1 << 48))
                          : ~0ull;
        }
    }
    block_or_and(o, a, oa);
}

// depth keys in index order (input of the stable depth sort)
__global__ void splat_depth_kernel(int k, const double* __restrict__ depth,
                                   unsigned long long* __restrict__ k0,
                                   unsigned int* __restrict__ v0, unsigned long long* __restrict__ k1,
                                   unsigned int* __restrict__ v1,
                                   const unsigned long long* __restrict__ idx_oa,
                                   ViewCounters* __restrict__ vc) {
    const bool p = pass_parity(idx_oa[0] ^ idx_oa[1], 8);
    const unsigned int* src = p ? v1 : v0;
    const int stride = gridDim.x * blockDim.x;
    const int iters = (k + stride - 1) / stride;
    unsigned long long o = 0, a = ~0ull;
    for (int it = 0; it < iters; ++it) {
        int i = it * stride + blockIdx.x * blockDim.x + threadIdx.x;
        unsigned int pos = 0;
        if (i < k) pos = src[i];
        __syncthreads();  // in-place when p == 0: everyone read before anyone writes
        if (i < k) {
            unsigned long long key = f64_sort_key(depth[pos]);
            k0[i] = key;
            v0[i] = pos;
            o |= key;
            a &= key;
        }
    }
    block_or_and(o, a, &vc->key_or);
}

}  // namespace

void launch_bin(int n, int ntiles, int tiles_x, int tile_passes, const BinBuffers& b,
                ViewCounters* vc, int num_sms, cudaStream_t st) {
    const int g = sort_grid(num_sms);
    emit_reduce_kernel<<<g, kBinThreads, 0, st>>>(n, b.dvals[0], b.dvals[1], b.depth_or_and, b.rect,
                                                  b.block_sums);
    emit_scan_kernel<<<1, 1024, 0, st>>>(b.block_sums, g, b.capacity, vc);
    emit_write_kernel<<<g, kBinThreads, 0, st>>>(n, tiles_x, b.dvals[0], b.dvals[1], b.depth_or_and,
                                                 b.rect, b.block_sums, b.ikeys[0], b.ivals[0], vc);
    launch_radix_sort<unsigned int>(b.ikeys[0], b.ivals[0], b.ikeys[1], b.ivals[1], &vc->n_valid, 0u,
                                    b.tile_or_and, tile_passes, b.hist, num_sms, st);
    tile_ranges_kernel<<<num_sms * 4, 256, 0, st>>>(ntiles, tile_passes, b.ikeys[0], b.ikeys[1],
                                                    b.tile_or_and, b.tile_start, vc);
}

void launch_bin_splats_keys(int k, const long long* index, const double* mean2d,
                            const long long* radius, const double* depth, int width, int height,
                            unsigned long long* dk0, unsigned int* dv0, unsigned long long* dk1,
                            unsigned int* dv1, unsigned long long* rect, unsigned long long* idx_oa,
                            unsigned int* hist, ViewCounters* vc, int num_sms, cudaStream_t st) {
    if (k <= 0) return;
    int grid = min((k + 255) / 256, num_sms * 8);
    splat_index_kernel<<<grid, 256, 0, st>>>(k, index, mean2d, radius, width, height, dk0, dv0, rect,
                                             idx_oa);
    launch_radix_sort<unsigned long long>(dk0, dv0, dk1, dv1, nullptr, (unsigned)k, idx_oa, 8, hist,
                                          num_sms, st);
    splat_depth_kernel<<<grid, 256, 0, st>>>(k, depth, dk0, dv0, dk1, dv1, idx_oa, vc);
}

}  // namespace fs
