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

__global__ void __launch_bounds__(1024) tile_scan_kernel(int ntiles,
                                                          const unsigned int* __restrict__ count,
                                                          unsigned int* __restrict__ start,
                                                          unsigned int* __restrict__ cursor,
                                                          unsigned int capacity,
                                                          ViewCounters* __restrict__ vc) {
    __shared__ unsigned long long s[1024];
    const int per = (ntiles + 1023) / 1024;
    const int lo = min(ntiles, (int)threadIdx.x * per), hi = min(ntiles, lo + per);
    unsigned long long sum = 0;
    for (int t = lo; t < hi; ++t) sum += count[t];
    s[threadIdx.x] = sum;
    __syncthreads();
    for (int off = 1; off < 1024; off <<= 1) {
        const unsigned long long y = threadIdx.x >= (unsigned)off ? s[threadIdx.x - off] : 0ull;
        __syncthreads();
        s[threadIdx.x] += y;
        __syncthreads();
    }
    unsigned long long run = s[threadIdx.x] - sum;
    const unsigned long long total = s[1023];
    const bool over = total > capacity;
    for (int t = lo; t < hi; ++t) {
        const unsigned int r = over ? 0u : (unsigned int)run;
        start[t] = r;
        cursor[t] = r;
        run += count[t];
    }
    if (threadIdx.x == 1023) {
        start[ntiles] = over ? 0u : (unsigned int)total;
        vc->n_instances = total > 0xFFFFFFFFull ? 0xFFFFFFFFu : (unsigned int)total;
        vc->overflow = over ? 1u : 0u;
        vc->n_valid = over ? 0u : (unsigned int)total;
    }
}

__global__ void __launch_bounds__(kThreads) emit_ranks_kernel(
    int n, int tiles_x, const unsigned int* __restrict__ v0, const unsigned int* __restrict__ v1,
    const SortState* __restrict__ dst, const unsigned long long* __restrict__ rect,
    unsigned int* __restrict__ cursor, unsigned int* __restrict__ inst,
    const ViewCounters* __restrict__ vc) {
    if (vc->overflow) return;
    const unsigned int* gids = sort_result_parity(dst) ? v1 : v0;
    for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < n; r += gridDim.x * blockDim.x) {
        const unsigned long long rc = rect[gids[r]];
        if (rc == ~0ull) continue;
        const unsigned int tx0 = rc & 0xFFFF, tx1 = (rc >> 16) & 0xFFFF;
        const unsigned int ty0 = (rc >> 32) & 0xFFFF, ty1 = (rc >> 48) & 0xFFFF;
        for (unsigned int ty = ty0; ty <= ty1; ++ty)
            for (unsigned int tx = tx0; tx <= tx1; ++tx) {
                const unsigned int pos = atomicAdd(&cursor[ty * (unsigned)tiles_x + tx], 1u);
                inst[pos] = (unsigned int)r;
            }
    }
}

__global__ void __launch_bounds__(kThreads) tile_sort_kernel(TileSortArgs t) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int tile = blockIdx.x;
    if (t.vc->overflow) return;
    const unsigned int begin = t.tile_start[tile], end = t.tile_start[tile + 1];
    if (begin >= end) return;
    const unsigned int* sg = sort_result_parity(t.depth_state) ? t.sorted_gid[1] : t.sorted_gid[0];
    sort_tile_list(t.inst + begin, t.scratch + begin, end - begin, sg, t.rank_bits,
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
            count_rect_tiles(rc, tx_n, tile_count);
        }
    }
    block_or_and(o, a, oa);
}

// depth keys in index order (input of the stable depth sort)
__global__ void splat_depth_kernel(int k, const double* __restrict__ depth,
                                   unsigned long long* __restrict__ k0,
                                   unsigned int* __restrict__ v0, unsigned long long* __restrict__ k1,
                                   unsigned int* __restrict__ v1,
                                   const SortState* __restrict__ ist,
                                   ViewCounters* __restrict__ vc) {
    const bool p = sort_result_parity(ist);
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

void launch_bin(int n, int ntiles, int tiles_x, const BinBuffers& b, ViewCounters* vc,
                int num_sms, cudaStream_t st) {
    tile_scan_kernel<<<1, 1024, 0, st>>>(ntiles, b.tile_count, b.tile_start, b.tile_cursor,
                                         b.capacity, vc);
    const int grid = std::max(1, std::min((n + kThreads - 1) / kThreads, num_sms * 8));
    emit_ranks_kernel<<<grid, kThreads, 0, st>>>(n, tiles_x, b.sorted_gid[0], b.sorted_gid[1],
                                                 b.depth_state, b.rect, b.tile_cursor, b.inst, vc);
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
                            unsigned int* dv1, unsigned long long* rect, unsigned int* tile_count,
                            unsigned long long* idx_oa, SortState* idx_state,
                            unsigned long long* idx_status, ViewCounters* vc, int num_sms,
                            cudaStream_t st) {
    if (k <= 0) return;
    int grid = std::min((k + 255) / 256, num_sms * 8);
    splat_index_kernel<<<grid, 256, 0, st>>>(k, index, mean2d, radius, width, height, dk0, dv0, rect,
                                             tile_count, idx_oa);
    launch_radix_sort<unsigned long long>(dk0, dv0, dk1, dv1, nullptr, (unsigned)k, idx_oa, nullptr,
                                          8, idx_state, idx_status, num_sms, st);
    splat_depth_kernel<<<grid, 256, 0, st>>>(k, depth, dk0, dv0, dk1, dv1, idx_state, vc);
}

}  // namespace fs
