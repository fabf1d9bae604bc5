// fs_bin.cu -- K2: tile binning on the device (reference rasterizer.py:72-113).
//
// TileBinning appends every visible splat, in (depth, index) order, to every
// tile its inclusive radius box covers.  Here the work splits in two:
//
//   binning   (this file) -- per-tile buckets of gids in arbitrary order:
//     bin_count   per-block tile histogram over a contiguous gid range (shared
//                 memory atomics), written to a tile-major count matrix;
//     tile_scan   one warp per tile scans the tile's row of the count matrix
//                 -> per-(tile, block) offsets inside the bucket, bucket length;
//     tile_start  one CTA: bucket starts, instance total, overflow flag, and
//                 the raster launch order (longest buckets first);
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
#ifndef FS_BIN_THREADS
#define FS_BIN_THREADS 1024
#endif
constexpr int kBinThreads = FS_BIN_THREADS;  // count / emit: latency-bound gid walks
constexpr int kUnroll = 4;         // gids per thread with their loads issued together

__device__ __forceinline__ void gid_range(int n, int b, int g, int& lo, int& hi) {
    const long long per = ((long long)n + g - 1) / g;
    lo = (int)min((long long)n, per * b);
    hi = (int)min((long long)n, per * (b + 1));
}

// Primary key: the 32 highest bits in which the view's depth keys differ.
__device__ __forceinline__ int primary_shift(const unsigned long long* oa) {
    const unsigned long long vary = oa[0] ^ ~oa[1];  // OR ^ AND
    const int hb = vary ? 63 - __clzll((long long)vary) : 0;
    return hb > 31 ? hb - 31 : 0;
}

// The rectangle rc clipped to the tile rows [ty_lo, ty_hi) of a band; false if empty.
template <bool kBanded>
__device__ __forceinline__ bool band_rows(unsigned long long rc, int ty_lo, int ty_hi,
                                          unsigned int& ty0, unsigned int& ty1) {
    if (rc == ~0ull) return false;
    ty0 = (unsigned int)((rc >> 32) & 0xFFFF);
    ty1 = (unsigned int)((rc >> 48) & 0xFFFF);
    if (!kBanded) return true;  // one band: every row of the image
    ty0 = max(ty0, (unsigned int)ty_lo);
    ty1 = min(ty1, (unsigned int)(ty_hi - 1));
    return ty0 <= ty1;
}

// per-block tile histogram of a contiguous gid range -> count[t * g + b], for the
// tile rows [ty_lo, ty_hi) (one band: the whole image unless it has more than
// kMaxTiles tiles, whose histograms would not fit shared memory)
template <bool kBanded>
__global__ void __launch_bounds__(kBinThreads) bin_count_kernel(BinBuffers b, int ntiles,
                                                             int tiles_x, int ty_lo, int ty_hi) {
    extern __shared__ unsigned int s_hist[];
    const int t_lo = ty_lo * tiles_x, nband = min(ntiles, ty_hi * tiles_x) - t_lo;
    for (int t = threadIdx.x; t < nband; t += kBinThreads) s_hist[t] = 0;
    __syncthreads();
    int lo, hi;
    gid_range(b.n, blockIdx.x, gridDim.x, lo, hi);
    // kUnroll independent loads in flight per thread (the walk is latency-bound)
    for (int g0 = lo + threadIdx.x; g0 < hi; g0 += kUnroll * kBinThreads) {
        unsigned long long rc[kUnroll];
#pragma unroll
        for (int j = 0; j < kUnroll; ++j) {
            const int g = g0 + j * kBinThreads;
            rc[j] = g < hi ? b.rect[g] : ~0ull;
        }
#pragma unroll
        for (int j = 0; j < kUnroll; ++j) {
            unsigned int ty0, ty1;
            if (!band_rows<kBanded>(rc[j], ty_lo, ty_hi, ty0, ty1)) continue;
            const unsigned int tx0 = rc[j] & 0xFFFF, tx1 = (rc[j] >> 16) & 0xFFFF;
            for (unsigned int ty = ty0; ty <= ty1; ++ty)
                for (unsigned int tx = tx0; tx <= tx1; ++tx)
                    atomicAdd(&s_hist[ty * (unsigned)tiles_x + tx - t_lo], 1u);
        }
    }
    __syncthreads();
    for (int t = threadIdx.x; t < nband; t += kBinThreads)
        b.count_bt[(size_t)(t + t_lo) * gridDim.x + blockIdx.x] = s_hist[t];
}

// per tile (one warp each): exclusive scan of the tile's row of the count
// matrix in place -> offsets of the blocks' runs inside the bucket; the row
// sum is the bucket length
__global__ void __launch_bounds__(kThreads) tile_scan_kernel(unsigned int* __restrict__ count_bt,
                                                             int ntiles, int g,
                                                             unsigned int* __restrict__ tile_total) {
    const int t = (int)((blockIdx.x * kThreads + threadIdx.x) >> 5), lane = threadIdx.x & 31;
    if (t >= ntiles) return;
    unsigned int* row = count_bt + (size_t)t * g;
    unsigned int carry = 0;
    for (int i0 = 0; i0 < g; i0 += 32) {
        const int i = i0 + lane;
        const unsigned int v = i < g ? row[i] : 0u;
        unsigned int x = v;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const unsigned int y = __shfl_up_sync(0xffffffffu, x, o);
            if (lane >= o) x += y;
        }
        if (i < g) row[i] = carry + x - v;
        carry += __shfl_sync(0xffffffffu, x, 31);
    }
    if (lane == 0) tile_total[t] = carry;
}

// One CTA: bucket starts (exclusive scan of the bucket lengths), the instance
// total / overflow flag, and the raster launch order -- tiles by decreasing
// bucket length (counting sort on length / 8), so the long tiles start in the
// first wave and the short ones fill the tail.
__global__ void __launch_bounds__(1024) tile_start_kernel(const unsigned int* __restrict__ total,
                                                          int ntiles, unsigned int capacity,
                                                          ViewCounters* __restrict__ vc,
                                                          unsigned int* __restrict__ tile_start,
                                                          unsigned int* __restrict__ order) {
    __shared__ unsigned long long s_w[32];
    __shared__ unsigned int hist[1024];
    __shared__ unsigned int h_w[32];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int per = (ntiles + 1023) / 1024;
    const int t0 = min(ntiles, tid * per), t1 = min(ntiles, t0 + per);
    unsigned long long sum = 0;
    for (int t = t0; t < t1; ++t) sum += total[t];
    unsigned long long x = sum;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const unsigned long long y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) s_w[warp] = x;
    hist[tid] = 0;
    __syncthreads();
    if (warp == 0) {
        const unsigned long long w = s_w[lane];
        unsigned long long z = w;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const unsigned long long y = __shfl_up_sync(0xffffffffu, z, o);
            if (lane >= o) z += y;
        }
        s_w[lane] = z - w;
    }
    __syncthreads();
    unsigned long long run = s_w[warp] + x - sum;
    for (int t = t0; t < t1; ++t) {
        const unsigned int n = total[t];
        tile_start[t] = (unsigned int)run;
        run += n;
        atomicAdd(&hist[1023u - min(n >> 3, 1023u)], 1u);
    }
    if (tid == 1023) {  // run == grand total
        const bool over = run > capacity;
        vc->n_instances = run > 0xFFFFFFFFull ? 0xFFFFFFFFu : (unsigned int)run;
        vc->overflow = over ? 1u : 0u;
        vc->n_valid = over ? 0u : (unsigned int)run;
        tile_start[ntiles] = over ? 0u : (unsigned int)run;
    }
    __syncthreads();
    const unsigned int v = hist[tid];
    unsigned int hx = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const unsigned int y = __shfl_up_sync(0xffffffffu, hx, o);
        if (lane >= o) hx += y;
    }
    if (lane == 31) h_w[warp] = hx;
    __syncthreads();
    if (warp == 0) {
        const unsigned int w = h_w[lane];
        unsigned int z = w;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const unsigned int y = __shfl_up_sync(0xffffffffu, z, o);
            if (lane >= o) z += y;
        }
        h_w[lane] = z - w;
    }
    __syncthreads();
    hist[tid] = h_w[warp] + hx - v;
    __syncthreads();
    for (int t = t0; t < t1; ++t)
        order[atomicAdd(&hist[1023u - min(total[t] >> 3, 1023u)], 1u)] = (unsigned int)t;
}

// per-block: cursors = bucket start + the block's offset inside the bucket,
// then shared-memory atomics place every instance of the block's gid range
template <bool kBanded>
__global__ void __launch_bounds__(kBinThreads) bin_emit_kernel(BinBuffers b, int ntiles, int tiles_x,
                                                            const ViewCounters* __restrict__ vc,
                                                            int ty_lo, int ty_hi) {
    if (vc->overflow) return;
    extern __shared__ unsigned int s_cur[];
    const int t_lo = ty_lo * tiles_x, nband = min(ntiles, ty_hi * tiles_x) - t_lo;
    for (int t = threadIdx.x; t < nband; t += kBinThreads)
        s_cur[t] = b.tile_start[t + t_lo] + b.count_bt[(size_t)(t + t_lo) * gridDim.x + blockIdx.x];
    __syncthreads();
    const int shift = primary_shift(b.key_oa);
    const unsigned long long z = ~b.key_oa[1];  // AND of the visible keys
    int lo, hi;
    gid_range(b.n, blockIdx.x, gridDim.x, lo, hi);
    for (int g0 = lo + threadIdx.x; g0 < hi; g0 += kUnroll * kBinThreads) {
        unsigned long long rc[kUnroll], key[kUnroll];
#pragma unroll
        for (int j = 0; j < kUnroll; ++j) {  // all loads first: kUnroll in flight
            const int g = g0 + j * kBinThreads;
            rc[j] = g < hi ? b.rect[g] : ~0ull;
            key[j] = g < hi ? b.k64[g] : 0ull;
        }
#pragma unroll
        for (int j = 0; j < kUnroll; ++j) {
            const unsigned long long r = rc[j];
            if (r == ~0ull) continue;
            const unsigned long long k = key[j] == ~0ull ? z : key[j];
            // instance = (32-bit primary depth key, gid)
            const unsigned long long e = ((k >> shift) << 32) | (unsigned int)(g0 + j * kBinThreads);
            unsigned int ty0, ty1;
            if (!band_rows<kBanded>(r, ty_lo, ty_hi, ty0, ty1)) continue;
            const unsigned int tx0 = r & 0xFFFF, tx1 = (r >> 16) & 0xFFFF;
            FS_CHECK(tx1 < (unsigned)tiles_x && ty1 * (unsigned)tiles_x + tx1 < (unsigned)ntiles);
            for (unsigned int ty = ty0; ty <= ty1; ++ty)
                for (unsigned int tx = tx0; tx <= tx1; ++tx) {
                    const unsigned int t = ty * (unsigned)tiles_x + tx;
                    const unsigned int at = atomicAdd(&s_cur[t - t_lo], 1u);
                    FS_CHECK(at < b.tile_start[t + 1] && at < b.capacity);
                    b.inst[at] = e;
                }
        }
    }
}

__global__ void __launch_bounds__(kThreads) tile_sort_kernel(TileSortArgs t) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int tile = blockIdx.x;
    if (t.vc->overflow) return;
    const unsigned int begin = t.tile_start[tile], end = t.tile_start[tile + 1];
    if (begin >= end) return;
    sort_tile_list(t.inst + begin, sorted_view(t.inst, begin), t.scratch64 + 2ull * begin, end - begin,
                   t.keys, smem_raw, t.cap,
                   8 * ((size_t)t.cap + 2) + sizeof(unsigned int) * (2048 + 64) + 2 * (size_t)t.cap);
}

__device__ __forceinline__ void block_or_and(unsigned long long o, unsigned long long a,
                                             unsigned long long* dst) {
    for (int off = 16; off > 0; off >>= 1) {
        o |= __shfl_xor_sync(0xffffffffu, o, off);
        a &= __shfl_xor_sync(0xffffffffu, a, off);
    }
    if ((threadIdx.x & 31) == 0) {
        atomicOr(dst, o);
        atomicOr(dst + 1, ~a);
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

// Most binning blocks a launch uses (the count matrix is sized for it): two
// 1 024-thread blocks per SM when the binning has the GPU to itself.
int bin_blocks(int num_sms) { return 2 * num_sms; }

// Blocks for a binning that runs beside other streams' raster launches (the
// accumulate view loop): a third of the SMs.  Fewer, longer blocks leave the
// raster CTAs of the other views their SMs and shrink the count matrix the
// scan walks -- C2 solve 70.0 -> 67.1 ms, C4 310 -> 303 ms against 2 per SM
// (37-49 blocks best; 18 or fewer starve the binning).
#ifndef FS_BIN_OVL_NUM
#define FS_BIN_OVL_NUM 1
#endif
#ifndef FS_BIN_OVL_DEN
#define FS_BIN_OVL_DEN 3
#endif
int bin_blocks_overlapped(int num_sms) {
    return std::max(1, num_sms * FS_BIN_OVL_NUM / FS_BIN_OVL_DEN);
}

cudaError_t bin_configure() {
    const int bytes = (int)(kMaxTiles * sizeof(unsigned int));
    cudaError_t e;
    if ((e = cudaFuncSetAttribute(bin_count_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes)) ||
        (e = cudaFuncSetAttribute(bin_count_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes)) ||
        (e = cudaFuncSetAttribute(bin_emit_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes)))
        return e;
    return cudaFuncSetAttribute(bin_emit_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
}

void launch_bin(int ntiles, int tiles_x, const BinBuffers& b, ViewCounters* vc, int num_sms,
                cudaStream_t st, int blocks) {
    const int g = blocks > 0 ? std::min(blocks, bin_blocks(num_sms)) : bin_blocks(num_sms);
    // tile-row bands whose per-block histograms fit shared memory (one band for
    // every image up to kMaxTiles tiles)
    const int ty_n = (ntiles + tiles_x - 1) / tiles_x;
    const int band = std::max(1, kMaxTiles / tiles_x);
    const size_t smem = sizeof(unsigned int) * (size_t)std::min(ntiles, band * tiles_x);
    const bool banded = band < ty_n;
    for (int y = 0; y < ty_n; y += band) {
        if (banded)
            bin_count_kernel<true><<<g, kBinThreads, smem, st>>>(b, ntiles, tiles_x, y, std::min(ty_n, y + band));
        else
            bin_count_kernel<false><<<g, kBinThreads, smem, st>>>(b, ntiles, tiles_x, 0, ty_n);
    }
    tile_scan_kernel<<<(ntiles + kWarps - 1) / kWarps, kThreads, 0, st>>>(b.count_bt, ntiles, g,
                                                                         b.tile_total);
    tile_start_kernel<<<1, 1024, 0, st>>>(b.tile_total, ntiles, b.capacity, vc, b.tile_start,
                                          b.tile_order);
    for (int y = 0; y < ty_n; y += band) {
        if (banded)
            bin_emit_kernel<true><<<g, kBinThreads, smem, st>>>(b, ntiles, tiles_x, vc, y, std::min(ty_n, y + band));
        else
            bin_emit_kernel<false><<<g, kBinThreads, smem, st>>>(b, ntiles, tiles_x, vc, 0, ty_n);
    }
}

size_t tile_sort_smem_bytes(unsigned int cap) {
    // packed (key, gid) entries, digit counters, misc, 16-bit entry indices
    return 8 * ((size_t)cap + 2) + sizeof(unsigned int) * (2048 + 64) + 2 * (size_t)cap;
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
