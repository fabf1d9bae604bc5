// fs_tilesort.cuh -- per-tile sort of a bucket of depth ranks (shared by the
// raster kernel prologue, fs_raster.cu, and the standalone tile_sort_kernel
// of the binning API, fs_bin.cu).  See fs_bin.cu for the pipeline.
#pragma once

#include "fs_common.cuh"
#include "fs_kernels.cuh"

namespace fs {
namespace tilesort {

constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;

// ---------------------------------------------------------------------------
// Per-tile sort of a bucket of depth ranks (device function shared by the
// raster kernel's prologue and tile_sort_kernel).  256 threads.  `smem` holds
// at least 2*cap + kWarps*256 + 64 words.  On return list[0..n) holds gids in
// (depth, gid) order.
// ---------------------------------------------------------------------------

// exclusive scan over 256 values held one per thread (blockDim == 256)
static __device__ __forceinline__ unsigned int block_excl_scan256(unsigned int v, unsigned int* s_w) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    unsigned int x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const unsigned int y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) s_w[warp] = x;
    __syncthreads();
    unsigned int base = 0;
#pragma unroll
    for (int w = 0; w < kWarps; ++w) base += w < warp ? s_w[w] : 0u;
    __syncthreads();
    return base + x - v;
}

// stable LSD radix sort of n <= cap keys in shared memory; returns the buffer
// holding the result (a or b)
static __device__ unsigned int* smem_radix_sort(unsigned int* a, unsigned int* b, unsigned int n,
                                         int bits, unsigned int* whist, unsigned int* s_misc) {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const unsigned int lt_mask = (1u << lane) - 1u;
    // digits that vary over this tile
    unsigned int o = 0, z = 0xFFFFFFFFu;
    for (unsigned int i = threadIdx.x; i < n; i += kThreads) {
        o |= a[i];
        z &= a[i];
    }
    o = __reduce_or_sync(0xffffffffu, o);
    z = __reduce_and_sync(0xffffffffu, z);
    if (lane == 0) {
        s_misc[warp] = o;
        s_misc[kWarps + warp] = z;
    }
    __syncthreads();
    unsigned int vary = 0, allz = 0xFFFFFFFFu;
#pragma unroll
    for (int w = 0; w < kWarps; ++w) {
        vary |= s_misc[w];
        allz &= s_misc[kWarps + w];
    }
    vary ^= allz;
    __syncthreads();
    // each warp owns a contiguous slice (keeps the scatter stable)
    const unsigned int per = ((n + kWarps - 1) / kWarps + 31u) & ~31u;
    const unsigned int lo = min(n, per * warp), hi = min(n, lo + per);
    for (int shift = 0; shift < bits; shift += 8) {
        if (!((vary >> shift) & 0xFFu)) continue;
        for (int i = threadIdx.x; i < kWarps * 256; i += kThreads) whist[i] = 0;
        __syncthreads();
        for (unsigned int base = lo; base < hi; base += 32) {
            const unsigned int idx = base + lane;
            const bool valid = idx < hi;
            const unsigned int d = valid ? (a[idx] >> shift) & 0xFFu : 0u;
            const unsigned int peers = __match_any_sync(0xffffffffu, valid ? d : 256u + lane);
            if (valid && lane == 31 - __clz(peers)) whist[warp * 256 + d] += __popc(peers);
            __syncwarp();
        }
        __syncthreads();
        // digit-major, warp-minor exclusive offsets
        {
            const int d = threadIdx.x;
            unsigned int run = 0;
#pragma unroll
            for (int w = 0; w < kWarps; ++w) {
                const unsigned int c = whist[w * 256 + d];
                whist[w * 256 + d] = run;
                run += c;
            }
            const unsigned int base = block_excl_scan256(run, s_misc);
#pragma unroll
            for (int w = 0; w < kWarps; ++w) whist[w * 256 + d] += base;
        }
        __syncthreads();
        for (unsigned int base = lo; base < hi; base += 32) {
            const unsigned int idx = base + lane;
            const bool valid = idx < hi;
            const unsigned int key = valid ? a[idx] : 0u;
            const unsigned int d = (key >> shift) & 0xFFu;
            const unsigned int peers = __match_any_sync(0xffffffffu, valid ? d : 256u + lane);
            const unsigned int off = valid ? whist[warp * 256 + d] : 0u;
            __syncwarp();
            if (valid) {
                b[off + __popc(peers & lt_mask)] = key;
                if (lane == 31 - __clz(peers)) whist[warp * 256 + d] = off + __popc(peers);
            }
            __syncwarp();
        }
        __syncthreads();
        unsigned int* t = a;
        a = b;
        b = t;
    }
    return a;
}

// merge sorted src[lo, mid) and src[mid, hi) into dst[lo, hi) with the whole block
static __device__ void block_merge(const unsigned int* src, unsigned int* dst, unsigned int lo,
                            unsigned int mid, unsigned int hi) {
    const unsigned int na = mid - lo, nb = hi - mid, total = na + nb;
    const unsigned int per = (total + kThreads - 1) / kThreads;
    const unsigned int d0 = min(total, per * threadIdx.x), d1 = min(total, d0 + per);
    if (d0 >= d1) return;
    const unsigned int* A = src + lo;
    const unsigned int* B = src + mid;
    // merge path: i elements of A and d0 - i of B precede output position d0
    unsigned int l = d0 > nb ? d0 - nb : 0u, r = min(d0, na);
    while (l < r) {
        const unsigned int m = (l + r) >> 1;
        if (A[m] <= B[d0 - m - 1]) l = m + 1;
        else r = m;
    }
    unsigned int i = l, j = d0 - l;
    for (unsigned int k = d0; k < d1; ++k) {
        const bool take_a = j >= nb || (i < na && A[i] <= B[j]);
        dst[lo + k] = take_a ? A[i++] : B[j++];
    }
}

// Entries whose 32-bit primary depth keys tie are re-ordered by the full
// 64-bit key (stable, so gid order survives among exact ties).  `rk` holds
// depth ranks (sorted), `pk` their primary keys; runs of equal pk are
// contiguous because ranks are ordered by pk.  Runs are tiny in practice.
static __device__ void fix_primary_ties(unsigned int* rk, const unsigned int* pk, unsigned int n,
                                        const unsigned int* __restrict__ sorted_gid,
                                        const unsigned long long* __restrict__ k64) {
    for (unsigned int i = threadIdx.x; i + 1 < n; i += kThreads) {
        if (pk[i + 1] != pk[i] || (i > 0 && pk[i - 1] == pk[i])) continue;  // not a run start
        unsigned int j = i + 1;
        while (j + 1 < n && pk[j + 1] == pk[i]) ++j;
        // insertion sort rk[i..j] by k64[gid] (stable)
        for (unsigned int x = i + 1; x <= j; ++x) {
            const unsigned int r = rk[x];
            const unsigned long long key = k64[sorted_gid[r]];
            unsigned int y = x;
            while (y > i && k64[sorted_gid[rk[y - 1]]] > key) {
                rk[y] = rk[y - 1];
                --y;
            }
            rk[y] = r;
        }
    }
}

static __device__ __noinline__ void sort_tile_list(unsigned int* list, unsigned int* scratch,
                                                   unsigned int n, const TileSortKeys& K,
                                                   unsigned int* smem, unsigned int cap) {
    unsigned int* a = smem;
    unsigned int* b = smem + cap;
    unsigned int* whist = smem + 2 * cap;
    unsigned int* misc = whist + kWarps * 256;
    if (n <= cap) {
        for (unsigned int i = threadIdx.x; i < n; i += kThreads) a[i] = list[i];
        __syncthreads();
        unsigned int* res = smem_radix_sort(a, b, n, K.rank_bits, whist, misc);
        unsigned int* pk = res == a ? b : a;
        for (unsigned int i = threadIdx.x; i < n; i += kThreads) pk[i] = K.pkey[res[i]];
        __syncthreads();
        fix_primary_ties(res, pk, n, K.sorted_gid, K.k64);
        __syncthreads();
        for (unsigned int i = threadIdx.x; i < n; i += kThreads) list[i] = K.sorted_gid[res[i]];
        __syncthreads();
        return;
    }
    // long bucket: sort chunks of cap in shared memory, then merge through global memory
    for (unsigned int c0 = 0; c0 < n; c0 += cap) {
        const unsigned int m = min(cap, n - c0);
        for (unsigned int i = threadIdx.x; i < m; i += kThreads) a[i] = list[c0 + i];
        __syncthreads();
        const unsigned int* res = smem_radix_sort(a, b, m, K.rank_bits, whist, misc);
        for (unsigned int i = threadIdx.x; i < m; i += kThreads) list[c0 + i] = res[i];
        __syncthreads();
    }
    unsigned int* src = list;
    unsigned int* dst = scratch;
    for (unsigned int width = cap; width < n; width *= 2) {
        for (unsigned int lo = 0; lo < n; lo += 2 * width) {
            const unsigned int mid = min(n, lo + width), hi = min(n, lo + 2 * width);
            block_merge(src, dst, lo, mid, hi);
        }
        __threadfence_block();
        __syncthreads();
        unsigned int* t = src;
        src = dst;
        dst = t;
    }
    // primary keys of the merged list go to the other global buffer
    for (unsigned int i = threadIdx.x; i < n; i += kThreads) dst[i] = K.pkey[src[i]];
    __threadfence_block();
    __syncthreads();
    fix_primary_ties(src, dst, n, K.sorted_gid, K.k64);
    __threadfence_block();
    __syncthreads();
    for (unsigned int i = threadIdx.x; i < n; i += kThreads) list[i] = K.sorted_gid[src[i]];
    __syncthreads();
}

}  // namespace tilesort
using tilesort::sort_tile_list;
}  // namespace fs
