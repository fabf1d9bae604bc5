// fs_bin.cu -- K2: tile binning on the device (reference rasterizer.py:72-113).
//
// TileBinning appends every visible splat, in (depth, index) order, to every
// tile its inclusive radius box covers.  Here the work splits in two:
//
//   binning   (this file) -- per-tile buckets of gids in arbitrary order:
//     bin_count   per-block tile histogram over a contiguous gid range (shared
//                 memory atomics), written to a tile-major count matrix;
//     scan        exclusive scan of the count matrix -> per-(tile, block)
//                 write offsets, tile_start, instance total, overflow flag;
//     bin_emit    every block re-walks its gid range and places instances
//                 (32-bit primary depth key << 32 | gid) with shared-memory
//                 cursors (no global atomics);
//   ordering  (fs_tilesort.cuh) -- each tile's bucket is sorted in shared
//             memory by the primary key, ties resolved by (float64 key, id).
//
// No global sort of N depth keys or of the (tile, splat) instances is needed.
#include <algorithm>

#include "fs_common.cuh"
#include "fs_kernels.cuh"
#include "fs_tilesort.cuh"

namespace fs {

namespace {

constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;
constexpr int kBinThreads = 1024;  // count / emit: latency-bound gid walks, full occupancy

__device__ __forceinline__ void gid_range(int n, int b, int g, int& lo, int& hi) {
    const long long per = ((long long)n + g - 1) / g;
    lo = (int)min((long long)n, per * b);
    hi = (int)min((long long)n, per * (b + 1));
}

// Primary key: the 32 highest bits in which the view's depth keys differ.
__device__ __forceinline__ int primary_shift(const unsigned long long* oa) {
    const unsigned long long vary = oa[0] ^ oa[1];
    const int hb = vary ? 63 - __clzll((long long)vary) : 0;
    return hb > 31 ? hb - 31 : 0;
}

// per-block tile histogram of a contiguous gid range -> count[t * g + b]
__global__ void __launch_bounds__(kBinThreads) bin_count_kernel(BinBuffers b, int ntiles,
                                                             int tiles_x) {
    extern __shared__ unsigned int s_hist[];
    for (int t = threadIdx.x; t < ntiles; t += kBinThreads) s_hist[t] = 0;
    __syncthreads();
    int lo, hi;
    gid_range(b.n, blockIdx.x, gridDim.x, lo, hi);
    for (int g = lo + threadIdx.x; g < hi; g += kBinThreads) count_rect_tiles(b.rect[g], tiles_x, s_hist);
    __syncthreads();
    for (int t = threadIdx.x; t < ntiles; t += kBinThreads)
        b.count_bt[(size_t)t * gridDim.x + blockIdx.x] = s_hist[t];
}

// exclusive scan of v over the block (blockDim == kThreads); *total = block sum
__device__ __forceinline__ unsigned int block_scan(unsigned int v, unsigned int* s_w,
                                                   unsigned int* total) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    unsigned int x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const unsigned int y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) s_w[warp] = x;
    __syncthreads();
    unsigned int base = 0, tot = 0;
#pragma unroll
    for (int w = 0; w < kWarps; ++w) {
        base += w < warp ? s_w[w] : 0u;
        tot += s_w[w];
    }
    __syncthreads();
    *total = tot;
    return base + x - v;
}

// 3-kernel exclusive scan of the tile-major (tile, block) count matrix
__global__ void __launch_bounds__(kThreads) scan_reduce_kernel(const unsigned int* __restrict__ a,
                                                               long long m,
                                                               unsigned int* __restrict__ partial) {
    __shared__ unsigned int s_w[kWarps];
    const long long per = (m + gridDim.x - 1) / gridDim.x;
    const long long lo = min(m, per * blockIdx.x), hi = min(m, lo + per);
    unsigned int s = 0;
    for (long long i = lo + threadIdx.x; i < hi; i += kThreads) s += a[i];
    unsigned int tot;
    block_scan(s, s_w, &tot);
    if (threadIdx.x == 0) partial[blockIdx.x] = tot;
}

__global__ void __launch_bounds__(1024) scan_partials_kernel(unsigned int* __restrict__ partial,
                                                             int g, unsigned int capacity,
                                                             ViewCounters* __restrict__ vc) {
    __shared__ unsigned long long s[1024];
    const unsigned long long v = threadIdx.x < (unsigned)g ? partial[threadIdx.x] : 0ull;
    s[threadIdx.x] = v;
    __syncthreads();
    for (int off = 1; off < 1024; off <<= 1) {
        const unsigned long long y = threadIdx.x >= (unsigned)off ? s[threadIdx.x - off] : 0ull;
        __syncthreads();
        s[threadIdx.x] += y;
        __syncthreads();
    }
    if (threadIdx.x < (unsigned)g) partial[threadIdx.x] = (unsigned int)(s[threadIdx.x] - v);
    if (threadIdx.x == 1023) {
        const unsigned long long total = s[1023];
        const bool over = total > capacity;
        vc->n_instances = total > 0xFFFFFFFFull ? 0xFFFFFFFFu : (unsigned int)total;
        vc->overflow = over ? 1u : 0u;
        vc->n_valid = over ? 0u : (unsigned int)total;
    }
}

__global__ void __launch_bounds__(kThreads) scan_apply_kernel(unsigned int* __restrict__ a,
                                                              long long m, int g_blocks,
                                                              const unsigned int* __restrict__ partial,
                                                              int ntiles,
                                                              unsigned int* __restrict__ tile_start,
                                                              const ViewCounters* __restrict__ vc) {
    __shared__ unsigned int s_w[kWarps];
    const long long per = (m + gridDim.x - 1) / gridDim.x;
    const long long lo = min(m, per * blockIdx.x), hi = min(m, lo + per);
    // each thread scans a contiguous sub-segment
    const long long sub = (hi - lo + kThreads - 1) / kThreads;
    const long long s0 = min(hi, lo + sub * threadIdx.x), s1 = min(hi, s0 + sub);
    unsigned int sum = 0;
    for (long long i = s0; i < s1; ++i) sum += a[i];
    unsigned int tot;
    unsigned int run = partial[blockIdx.x] + block_scan(sum, s_w, &tot);
    for (long long i = s0; i < s1; ++i) {
        const unsigned int c = a[i];
        a[i] = run;
        if (i % g_blocks == 0) tile_start[i / g_blocks] = run;
        run += c;
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) tile_start[ntiles] = vc->n_valid;
}

// per-block: cursors from the scanned matrix, then shared-memory atomics place
// every instance of the block's gid range
__global__ void __launch_bounds__(kBinThreads) bin_emit_kernel(BinBuffers b, int ntiles, int tiles_x,
                                                            const ViewCounters* __restrict__ vc) {
    if (vc->overflow) return;
    extern __shared__ unsigned int s_cur[];
    for (int t = threadIdx.x; t < ntiles; t += kBinThreads)
        s_cur[t] = b.count_bt[(size_t)t * gridDim.x + blockIdx.x];
    __syncthreads();
    const int shift = primary_shift(b.key_oa);
    const unsigned long long z = b.key_oa[1];
    int lo, hi;
    gid_range(b.n, blockIdx.x, gridDim.x, lo, hi);
    for (int g = lo + threadIdx.x; g < hi; g += kBinThreads) {
        const unsigned long long rc = b.rect[g];
        if (rc == ~0ull) continue;
        unsigned long long key = b.k64[g];
        if (key == ~0ull) key = z;
        // instance = (32-bit primary depth key, gid)
        const unsigned long long e = ((key >> shift) << 32) | (unsigned int)g;
        const unsigned int tx0 = rc & 0xFFFF, tx1 = (rc >> 16) & 0xFFFF;
        const unsigned int ty0 = (rc >> 32) & 0xFFFF, ty1 = (rc >> 48) & 0xFFFF;
        for (unsigned int ty = ty0; ty <= ty1; ++ty)
            for (unsigned int tx = tx0; tx <= tx1; ++tx)
                b.inst[atomicAdd(&s_cur[ty * (unsigned)tiles_x + tx], 1u)] = e;
    }
}

__global__ void __launch_bounds__(kThreads) tile_sort_kernel(TileSortArgs t) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int tile = blockIdx.x;
    if (t.vc->overflow) return;
    const unsigned int begin = t.tile_start[tile], end = t.tile_start[tile + 1];
    if (begin >= end) return;
    sort_tile_list(t.inst + begin, sorted_view(t.inst, begin), t.scratch64 + 2ull * begin, end - begin,
                   t.keys, smem_raw, t.cap);
}

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

// explicit splat list: rect + depth key per list position, key OR/AND
__global__ void splat_keys_kernel(int k, const double* __restrict__ mean2d,
                                  const long long* __restrict__ radius,
                                  const double* __restrict__ depth, int width, int height,
                                  unsigned long long* __restrict__ rect,
                                  unsigned long long* __restrict__ k64,
                                  ViewCounters* __restrict__ vc) {
    const int tx_n = tiles_x_of(width), ty_n = tiles_y_of(height);
    const int stride = gridDim.x * blockDim.x;
    const int iters = (k + stride - 1) / stride;
    unsigned long long o = 0, a = ~0ull;
    for (int it = 0; it < iters; ++it) {
        const int i = it * stride + blockIdx.x * blockDim.x + threadIdx.x;
        if (i < k) {
            rect[i] = tile_rect(mean2d[2 * i], mean2d[2 * i + 1], (double)radius[i], tx_n, ty_n);
            const unsigned long long key = f64_sort_key(depth[i]);
            k64[i] = key;
            o |= key;
            a &= key;
        }
    }
    block_or_and(o, a, &vc->key_or);
}

}  // namespace

int bin_blocks(int num_sms) { return 2 * num_sms; }
int bin_scan_blocks(int num_sms) { return 4 * num_sms; }

cudaError_t bin_configure() {
    cudaError_t e = cudaFuncSetAttribute(bin_count_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)(kMaxTiles * sizeof(unsigned int)));
    if (e != cudaSuccess) return e;
    return cudaFuncSetAttribute(bin_emit_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                (int)(kMaxTiles * sizeof(unsigned int)));
}

void launch_bin(int ntiles, int tiles_x, const BinBuffers& b, ViewCounters* vc, int num_sms,
                cudaStream_t st) {
    const int g = bin_blocks(num_sms), g2 = bin_scan_blocks(num_sms);
    const size_t smem = sizeof(unsigned int) * (size_t)ntiles;
    const long long m = (long long)ntiles * g;
    bin_count_kernel<<<g, kBinThreads, smem, st>>>(b, ntiles, tiles_x);
    scan_reduce_kernel<<<g2, kThreads, 0, st>>>(b.count_bt, m, b.partial);
    scan_partials_kernel<<<1, 1024, 0, st>>>(b.partial, g2, b.capacity, vc);
    scan_apply_kernel<<<g2, kThreads, 0, st>>>(b.count_bt, m, g, b.partial, ntiles, b.tile_start, vc);
    bin_emit_kernel<<<g, kBinThreads, smem, st>>>(b, ntiles, tiles_x, vc);
}

size_t tile_sort_smem_bytes(unsigned int cap) {
    // packed (key, gid) entries, digit counters, misc, 16-bit entry indices
    return 8 * (size_t)cap + sizeof(unsigned int) * (2048 + 64) + 2 * (size_t)cap;
}

cudaError_t tile_sort_configure(unsigned int cap) {
    return cudaFuncSetAttribute(tile_sort_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                (int)tile_sort_smem_bytes(cap));
}

void launch_tile_sort(int ntiles, const TileSortArgs& t, cudaStream_t st) {
    if (ntiles <= 0) return;
    tile_sort_kernel<<<ntiles, kThreads, tile_sort_smem_bytes(t.cap), st>>>(t);
}

void launch_splat_keys(int k, const double* mean2d, const long long* radius, const double* depth,
                       int width, int height, unsigned long long* rect, unsigned long long* k64,
                       ViewCounters* vc, int num_sms, cudaStream_t st) {
    if (k <= 0) return;
    const int grid = std::min((k + 255) / 256, num_sms * 8);
    splat_keys_kernel<<<grid, 256, 0, st>>>(k, mean2d, radius, depth, width, height, rect, k64, vc);
}

}  // namespace fs
