// fs_bin.cu -- K2b-K2d: tile binning on the device (reference rasterizer.py:72-113).
//
// Input: all N Gaussians sorted by (depth, gid) by the depth radix sort
// (fs_sort.cu) -- the position of a Gaussian in that order is its depth
// rank -- plus each Gaussian's inclusive tile rectangle and the per-tile
// instance counts, both produced by the projection kernel.
//
//   tile_scan    one block: exclusive scan of the tile counts -> tile_start,
//                per-tile write cursors, instance total, overflow flag;
//   emit_ranks   one thread per depth rank: append the rank to the bucket of
//                every tile its rectangle covers (atomic cursor, any order);
//   sort_tile    one CTA per tile (inside the raster kernel, or standalone for
//                the binning API): sort the bucket's ranks in shared memory
//                (stable LSD radix, 8-bit digits, digits constant over the
//                tile skipped), map rank -> gid.  Ranks are unique, so the
//                result is exactly TileBinning.tile_lists' (depth, gid)
//                order.  Buckets longer than the shared-memory capacity are
//                sorted in chunks and merged through global memory.
// Sorting each tile's short bucket in shared memory replaces a global radix
// sort of all (tile, rank) instances.
#include <algorithm>

#include "fs_common.cuh"
#include "fs_kernels.cuh"
#include "fs_tilesort.cuh"

namespace fs {

namespace {

constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;

__device__ __forceinline__ void rank_range(int n, int b, int g, int& lo, int& hi) {
    const long long per = ((long long)n + g - 1) / g;
    lo = (int)min((long long)n, per * b);
    hi = (int)min((long long)n, per * (b + 1));
}

// per-block tile histogram of a contiguous range of depth ranks -> count[t * g + b]
__global__ void __launch_bounds__(kThreads) bin_count_kernel(
    int n, int ntiles, int tiles_x, const unsigned int* __restrict__ v0,
    const unsigned int* __restrict__ v1, const SortState* __restrict__ dst,
    const unsigned long long* __restrict__ rect, unsigned int* __restrict__ count_bt) {
    extern __shared__ unsigned int s_hist[];
    for (int t = threadIdx.x; t < ntiles; t += kThreads) s_hist[t] = 0;
    __syncthreads();
    const unsigned int* gids = sort_result_parity(dst) ? v1 : v0;
    int lo, hi;
    rank_range(n, blockIdx.x, gridDim.x, lo, hi);
    for (int r = lo + threadIdx.x; r < hi; r += kThreads) count_rect_tiles(rect[gids[r]], tiles_x, s_hist);
    __syncthreads();
    for (int t = threadIdx.x; t < ntiles; t += kThreads) count_bt[(size_t)t * gridDim.x + blockIdx.x] = s_hist[t];
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
// every instance of the block's rank range (buckets: block segments in rank
// order; order inside a segment is restored by the per-tile sort)
__global__ void __launch_bounds__(kThreads) bin_emit_kernel(
    int n, int ntiles, int tiles_x, const unsigned int* __restrict__ v0,
    const unsigned int* __restrict__ v1, const SortState* __restrict__ dst,
    const unsigned long long* __restrict__ rect, const unsigned int* __restrict__ off_bt,
    unsigned int* __restrict__ inst, const ViewCounters* __restrict__ vc) {
    if (vc->overflow) return;
    extern __shared__ unsigned int s_cur[];
    for (int t = threadIdx.x; t < ntiles; t += kThreads) s_cur[t] = off_bt[(size_t)t * gridDim.x + blockIdx.x];
    __syncthreads();
    const unsigned int* gids = sort_result_parity(dst) ? v1 : v0;
    int lo, hi;
    rank_range(n, blockIdx.x, gridDim.x, lo, hi);
    for (int r = lo + threadIdx.x; r < hi; r += kThreads) {
        const unsigned long long rc = rect[gids[r]];
        if (rc == ~0ull) continue;
        const unsigned int tx0 = rc & 0xFFFF, tx1 = (rc >> 16) & 0xFFFF;
        const unsigned int ty0 = (rc >> 32) & 0xFFFF, ty1 = (rc >> 48) & 0xFFFF;
        for (unsigned int ty = ty0; ty <= ty1; ++ty)
            for (unsigned int tx = tx0; tx <= tx1; ++tx)
                inst[atomicAdd(&s_cur[ty * (unsigned)tiles_x + tx], 1u)] = (unsigned int)r;
    }
}

__global__ void __launch_bounds__(kThreads) tile_sort_kernel(TileSortArgs t) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int tile = blockIdx.x;
    if (t.vc->overflow) return;
    const unsigned int begin = t.tile_start[tile], end = t.tile_start[tile + 1];
    if (begin >= end) return;
    sort_tile_list(t.inst + begin, t.scratch + begin, end - begin, resolve_keys(t),
                   reinterpret_cast<unsigned int*>(smem_raw), t.cap);
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

// keys = gaussian index (secondary sort key), vals = list position, rect +
// tile counts per position
__global__ void splat_index_kernel(int k, const long long* __restrict__ index,
                                   const double* __restrict__ mean2d,
                                   const long long* __restrict__ radius, int width, int height,
                                   unsigned long long* __restrict__ keys,
                                   unsigned int* __restrict__ vals,
                                   unsigned long long* __restrict__ rect,
                                   unsigned int* __restrict__ tile_count,
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
            const unsigned long long rc =
                tile_rect(mean2d[2 * i], mean2d[2 * i + 1], (double)radius[i], tx_n, ty_n);
            rect[i] = rc;
        }
    }
    block_or_and(o, a, oa);
}

// 64-bit depth key per list position (the index sort's result gives the
// stable input order of the depth sort)
__global__ void splat_depth_kernel(int k, const double* __restrict__ depth,
                                   unsigned long long* __restrict__ k64,
                                   ViewCounters* __restrict__ vc) {
    const int stride = gridDim.x * blockDim.x;
    const int iters = (k + stride - 1) / stride;
    unsigned long long o = 0, a = ~0ull;
    for (int it = 0; it < iters; ++it) {
        int i = it * stride + blockIdx.x * blockDim.x + threadIdx.x;
        if (i < k) {
            const unsigned long long key = f64_sort_key(depth[i]);
            k64[i] = key;
            o |= key;
            a &= key;
        }
    }
    block_or_and(o, a, &vc->key_or);
}

__global__ void primary_keys_kernel(int n, const unsigned long long* __restrict__ k64,
                                    const unsigned long long* __restrict__ oa64,
                                    const unsigned int* order0, const unsigned int* order1,
                                    const SortState* __restrict__ order_state,
                                    unsigned int* __restrict__ pk, unsigned int* vals,
                                    unsigned long long* __restrict__ pk_oa) {
    const unsigned int* order = order_state ? (sort_result_parity(order_state) ? order1 : order0)
                                            : order0;
    const unsigned long long o = oa64[0], z = oa64[1];
    const unsigned long long vary = o ^ z;
    const int hb = vary ? 63 - __clzll((long long)vary) : 0;
    const int shift = hb > 31 ? hb - 31 : 0;
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        pk_oa[0] = (unsigned int)(o >> shift);
        pk_oa[1] = (unsigned int)(z >> shift);
    }
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        const unsigned int g = order ? order[i] : (unsigned int)i;
        unsigned long long key = k64[g];
        if (key == ~0ull) key = z;  // invisible: never widens the varying digits
        pk[i] = (unsigned int)(key >> shift);
        vals[i] = g;
    }
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

void launch_bin(int n, int ntiles, int tiles_x, const BinBuffers& b, ViewCounters* vc,
                int num_sms, cudaStream_t st) {
    const int g = bin_blocks(num_sms), g2 = bin_scan_blocks(num_sms);
    const size_t smem = sizeof(unsigned int) * (size_t)ntiles;
    const long long m = (long long)ntiles * g;
    bin_count_kernel<<<g, kThreads, smem, st>>>(n, ntiles, tiles_x, b.sorted_gid[0], b.sorted_gid[1],
                                                b.depth_state, b.rect, b.count_bt);
    scan_reduce_kernel<<<g2, kThreads, 0, st>>>(b.count_bt, m, b.partial);
    scan_partials_kernel<<<1, 1024, 0, st>>>(b.partial, g2, b.capacity, vc);
    scan_apply_kernel<<<g2, kThreads, 0, st>>>(b.count_bt, m, g, b.partial, ntiles, b.tile_start, vc);
    bin_emit_kernel<<<g, kThreads, smem, st>>>(n, ntiles, tiles_x, b.sorted_gid[0], b.sorted_gid[1],
                                               b.depth_state, b.rect, b.count_bt, b.inst, vc);
}

size_t tile_sort_smem_bytes(unsigned int cap) {
    return sizeof(unsigned int) * (2 * (size_t)cap + kWarps * 256 + 64);
}

cudaError_t tile_sort_configure(unsigned int cap) {
    return cudaFuncSetAttribute(tile_sort_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                (int)tile_sort_smem_bytes(cap));
}

void launch_tile_sort(int ntiles, const TileSortArgs& t, cudaStream_t st) {
    if (ntiles <= 0) return;
    tile_sort_kernel<<<ntiles, kThreads, tile_sort_smem_bytes(t.cap), st>>>(t);
}

void launch_bin_splats_keys(int k, const long long* index, const double* mean2d,
                            const long long* radius, const double* depth, int width, int height,
                            unsigned long long* dk0, unsigned int* dv0, unsigned long long* dk1,
                            unsigned int* dv1, unsigned long long* rect, unsigned long long* k64,
                            unsigned long long* idx_oa, SortState* idx_state,
                            unsigned long long* idx_status, ViewCounters* vc, int num_sms,
                            cudaStream_t st) {
    if (k <= 0) return;
    int grid = std::min((k + 255) / 256, num_sms * 8);
    splat_index_kernel<<<grid, 256, 0, st>>>(k, index, mean2d, radius, width, height, dk0, dv0, rect,
                                             nullptr, idx_oa);
    launch_radix_sort<unsigned long long>(dk0, dv0, dk1, dv1, nullptr, (unsigned)k, idx_oa, nullptr,
                                          8, idx_state, idx_status, num_sms, st);
    splat_depth_kernel<<<grid, 256, 0, st>>>(k, depth, k64, vc);
}

void launch_primary_keys(int n, const unsigned long long* k64, const unsigned long long* oa64,
                         const unsigned int* order0, const unsigned int* order1,
                         const SortState* order_state, unsigned int* pk, unsigned int* vals,
                         unsigned long long* pk_oa, int num_sms, cudaStream_t st) {
    const int grid = std::max(1, std::min((n + 255) / 256, num_sms * 8));
    primary_keys_kernel<<<grid, 256, 0, st>>>(n, k64, oa64, order0, order1, order_state, pk, vals,
                                              pk_oa);
}

}  // namespace fs
