// fs_tilesort.cuh -- per-tile depth ordering of a tile's bucket (shared by the
// raster kernel prologue, fs_raster.cu, and the standalone tile_sort_kernel
// of the binning API, fs_bin.cu).
//
// A bucket holds the gids whose tile rectangle covers the tile, in arbitrary
// order.  The reference order is np.lexsort((index, depth)) with float64 depth
// (rasterizer.py:91).  Per tile:
//   0. the bucket comes into shared memory by one TMA bulk copy;
//   1. single-pass counting sort (shared memory, 2048 buckets) of
//      (primary << 32 | gid) by an 11-bit digit that is monotone in the 32-bit
//      primary key (= the 32 highest bits in which the view's float64 depth
//      keys differ) over the bucket's own key range;
//   2. entries sharing a digit are ranked within their digit run by the full
//      order (primary key, full 64-bit depth key, tie id) -- tie id = gid for
//      scenes, the splat's gaussian_index for explicit splat lists -- each
//      thread ranking its own entries, so runs cost no serial passes.
// Buckets longer than `cap` keep only their primary keys in shared memory
// (up to ~7 300 entries in the raster kernel's 52 KB); longer ones are sorted
// in chunks and merged through global memory.  The result is exactly the
// reference's tile list.
#pragma once

#include "fs_common.cuh"
#include "fs_kernels.cuh"

namespace fs {
namespace tilesort {

constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;

static __device__ __forceinline__ unsigned int pk_of(unsigned long long e) {
    return (unsigned int)(e >> 32);
}

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

// merge sorted src[lo, mid) and src[mid, hi) into dst[lo, hi) by primary key
static __device__ void block_merge(const unsigned long long* src, unsigned long long* dst,
                                   unsigned int lo, unsigned int mid, unsigned int hi) {
    const unsigned int na = mid - lo, nb = hi - mid, total = na + nb;
    const unsigned int per = (total + kThreads - 1) / kThreads;
    const unsigned int d0 = min(total, per * threadIdx.x), d1 = min(total, d0 + per);
    if (d0 >= d1) return;
    const unsigned long long* A = src + lo;
    const unsigned long long* B = src + mid;
    unsigned int l = d0 > nb ? d0 - nb : 0u, r = min(d0, na);
    while (l < r) {  // merge path
        const unsigned int m = (l + r) >> 1;
        if (pk_of(A[m]) <= pk_of(B[d0 - m - 1])) l = m + 1;
        else r = m;
    }
    unsigned int i = l, j = d0 - l;
    for (unsigned int k = d0; k < d1; ++k) {
        const bool take_a = j >= nb || (i < na && pk_of(A[i]) <= pk_of(B[j]));
        dst[lo + k] = take_a ? A[i++] : B[j++];
    }
}

// full order of an entry: (64-bit depth key, tie id)
static __device__ __forceinline__ bool entry_less(unsigned long long x, unsigned long long y,
                                                  const TileSortKeys K) {
    const unsigned int gx = (unsigned int)x, gy = (unsigned int)y;
    const unsigned long long kx = K.k64[gx], ky = K.k64[gy];
    if (kx != ky) return kx < ky;
    const unsigned int tx = K.tie ? K.tie[gx] : gx, ty = K.tie ? K.tie[gy] : gy;
    return tx < ty;
}

// Re-order runs of equal primary key by (k64, tie).  `e` is sorted by
// primary key; `flag` (n bytes) is scratch.
static __device__ void fix_primary_ties(unsigned long long* e, unsigned int n,
                                        const TileSortKeys K, unsigned char* flag) {
    // inversion check of each adjacent equal-key pair, in parallel
    for (unsigned int i = threadIdx.x; i + 1 < n; i += kThreads)
        flag[i] = (pk_of(e[i]) == pk_of(e[i + 1]) && entry_less(e[i + 1], e[i], K)) ? 1 : 0;
    __syncthreads();
    for (unsigned int i = threadIdx.x; i + 1 < n; i += kThreads) {
        if (pk_of(e[i + 1]) != pk_of(e[i]) || (i > 0 && pk_of(e[i - 1]) == pk_of(e[i]))) continue;
        unsigned int j = i + 1;
        bool inverted = flag[i] != 0;
        while (j + 1 < n && pk_of(e[j + 1]) == pk_of(e[i])) {
            inverted |= flag[j] != 0;
            ++j;
        }
        if (!inverted) continue;
        for (unsigned int x = i + 1; x <= j; ++x) {  // insertion sort of the run (stable)
            const unsigned long long v = e[x];
            unsigned int y = x;
            while (y > i && entry_less(v, e[y - 1], K)) {
                e[y] = e[y - 1];
                --y;
            }
            e[y] = v;
        }
    }
}

// ---- single-pass counting sort (the n <= cap path) ----
// Entries are bucketed by an 11-bit digit that is monotone in the primary key
// over this bucket's own key range; digit ties are then ordered by the full
// (primary, 64-bit depth, id) order.  Not stable -- it does not need to be,
// every tie is resolved by the full order afterwards.
struct DigitMap {
    unsigned int lo, shift;
};

static __device__ __forceinline__ unsigned int digit_of(unsigned int pk, DigitMap m) {
    return (pk - m.lo) >> m.shift;
}


// a[0, n) -> b[0, n): indices into a, grouped by digit (unordered within a
// digit); hist[d] is left at the end offset of digit d.
template <class PK>
static __device__ void smem_count_sort(PK pk, unsigned short* b, unsigned int n,
                                       unsigned int* hist, unsigned int* s_misc, DigitMap* map) {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    unsigned int lo = 0xFFFFFFFFu, hi = 0;
    for (unsigned int i = threadIdx.x; i < n; i += kThreads) {
        const unsigned int k = pk(i);
        lo = min(lo, k);
        hi = max(hi, k);
    }
    lo = __reduce_min_sync(0xffffffffu, lo);
    hi = __reduce_max_sync(0xffffffffu, hi);
    if (lane == 0) {
        s_misc[warp] = lo;
        s_misc[kWarps + warp] = hi;
    }
    for (int i = threadIdx.x; i < 2048; i += kThreads) hist[i] = 0;
    __syncthreads();
#pragma unroll
    for (int w = 0; w < kWarps; ++w) {
        lo = min(lo, s_misc[w]);
        hi = max(hi, s_misc[kWarps + w]);
    }
    const unsigned int range = hi - lo;
    const int bits = range ? 32 - __clz(range) : 0;
    const DigitMap m{lo, bits > 11 ? (unsigned int)(bits - 11) : 0u};
    *map = m;
    for (unsigned int i = threadIdx.x; i < n; i += kThreads) atomicAdd(&hist[digit_of(pk(i), m)], 1u);
    __syncthreads();
    unsigned int c[8], sum = 0;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
        c[j] = hist[threadIdx.x * 8 + j];
        sum += c[j];
    }
    unsigned int run = block_excl_scan256(sum, s_misc);
#pragma unroll
    for (int j = 0; j < 8; ++j) {
        hist[threadIdx.x * 8 + j] = run;
        run += c[j];
    }
    __syncthreads();
    for (unsigned int i = threadIdx.x; i < n; i += kThreads) {
        const unsigned int d = digit_of(pk(i), m);
        FS_CHECK(d < 2048u);
        const unsigned int at = atomicAdd(&hist[d], 1u);
        FS_CHECK(at < n);
        b[at] = (unsigned short)i;
    }
    __syncthreads();
}

// Places every entry of the digit-sorted e[0, n) at its final position:
// entries alone in their digit stay, entries of a digit run of length r are
// ranked within the run by the full order (r comparisons each, all threads in
// parallel).  hist[d] = end offset of digit d (as left by smem_count_sort).
// store(pos, entry) receives every entry exactly once.
template <class PK, class Entry, class Store>
static __device__ __forceinline__ void place_digit_runs(PK pk, Entry entry, const unsigned short* idx,
                                                        unsigned int n, const unsigned int* hist,
                                                        DigitMap m, const TileSortKeys K,
                                                        Store store) {
    for (unsigned int p = threadIdx.x; p < n; p += kThreads) {
        const unsigned int i = idx[p];
        const unsigned int key = pk(i);
        const unsigned int d = digit_of(key, m);
        const unsigned int s = d ? hist[d - 1] : 0u, t = hist[d];
        unsigned int pos = p;
        if (t - s > 1u) {
            pos = s;
            for (unsigned int q = s; q < t; ++q) {
                if (q == p) continue;  // (itself: equal keys would take the slow path)
                const unsigned int j = idx[q], kj = pk(j);
                // primary key first; only equal primaries consult the full entries
                pos += (kj != key ? kj < key : entry_less(entry(j), entry(i), K)) ? 1u : 0u;
            }
        }
        FS_CHECK(pos < n && i < n);
        store(pos, i);
    }
}

// ---- TMA bulk copy of a bucket into shared memory (cp.async.bulk + mbarrier) ----
static __device__ __forceinline__ unsigned int smem_addr(const void* p) {
    return (unsigned int)__cvta_generic_to_shared(p);
}

// Copies in[0, n) (8-byte entries) into shared memory with one bulk-copy
// instruction issued by thread 0 and completed on an mbarrier; returns where
// in[0] landed.  The copy starts at the 16-byte aligned address at or below
// `in` (one extra leading entry when `in` is 8 mod 16) and is rounded up to a
// multiple of 16 bytes, so the global buffer carries 2 entries of slack and
// `region` has room for n + 2 entries.  Every thread returns after the data
// has arrived.
static __device__ unsigned long long* bulk_load_bucket(const unsigned long long* in, unsigned int n,
                                                       unsigned long long* region,
                                                       unsigned long long* bar) {
    const unsigned int head = (unsigned int)((reinterpret_cast<uintptr_t>(in) >> 3) & 1u);
    const unsigned int bytes = ((n + head) * 8u + 15u) & ~15u;
    const unsigned int b = smem_addr(bar);
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(b));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"(bytes)
                     : "memory");
        asm volatile(
            "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
            ::"r"(smem_addr(region)), "l"(in - head), "r"(bytes), "r"(b)
            : "memory");
    }
    __syncthreads();  // the barrier is initialised before anyone waits on it
    unsigned int done = 0;
    while (!done)
        asm volatile(
            "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n"
            " selp.u32 %0, 1, 0, p;\n}"
            : "=r"(done)
            : "r"(b)
            : "memory");
    __syncthreads();
    if (threadIdx.x == 0) asm volatile("mbarrier.inval.shared::cta.b64 [%0];" ::"r"(b) : "memory");
    return region + head;
}

// Sorts the instances in[0, n) into the reference order and writes their gids
// to out[0, n) (out may alias in: every read precedes the first write).
// smem: at least tile_sort_smem_bytes(cap) bytes; scratch64: 2n entries of
// global scratch.
static __device__ __noinline__ void sort_tile_list(const unsigned long long* in, unsigned int* out,
                                                   unsigned long long* scratch64, unsigned int n,
                                                   const TileSortKeys K, unsigned char* smem,
                                                   unsigned int cap, size_t smem_bytes) {
    unsigned long long* region = reinterpret_cast<unsigned long long*>(smem);  // cap + 2 entries
    unsigned long long* a = region;
    unsigned int* whist = reinterpret_cast<unsigned int*>(region + cap + 2);
    unsigned int* misc = whist + 2048;
    unsigned short* b = reinterpret_cast<unsigned short*>(misc + 64);
    unsigned long long* bar = reinterpret_cast<unsigned long long*>(misc + 62);
    FS_CHECK(reinterpret_cast<unsigned char*>(b + cap) <= smem + smem_bytes);
    if (n <= cap) {
        a = bulk_load_bucket(in, n, region, bar);  // TMA: global bucket -> shared memory
        const unsigned long long* sa = a;
        auto pk = [sa](unsigned int i) { return pk_of(sa[i]); };
        auto entry = [sa](unsigned int i) { return sa[i]; };
        DigitMap m;
        smem_count_sort(pk, b, n, whist, misc, &m);
        place_digit_runs(pk, entry, b, n, whist, m, K,
                         [&](unsigned int pos, unsigned int i) { out[pos] = (unsigned int)sa[i]; });
        __syncthreads();
        return;
    }
    // medium bucket: only the 32-bit primary keys (+ 16-bit indices) in shared
    // memory, which holds up to `cap2` entries; gids come from the global bucket,
    // the ordered gids pass through the (global) scratch
    const unsigned int cap2 = (unsigned int)((smem_bytes - 4u * (2048 + 64)) / 6u);
    if (n <= cap2) {
        unsigned int* hist2 = reinterpret_cast<unsigned int*>(smem);
        unsigned int* misc2 = hist2 + 2048;
        unsigned int* pks = misc2 + 64;
        unsigned short* idx2 = reinterpret_cast<unsigned short*>(pks + cap2);
        FS_CHECK(reinterpret_cast<unsigned char*>(idx2 + n) <= smem + smem_bytes);
        for (unsigned int i = threadIdx.x; i < n; i += kThreads) pks[i] = pk_of(in[i]);
        __syncthreads();
        auto pk = [pks](unsigned int i) { return pks[i]; };
        auto entry = [in](unsigned int i) { return in[i]; };
        unsigned int* tmp = reinterpret_cast<unsigned int*>(scratch64);
        DigitMap m;
        smem_count_sort(pk, idx2, n, hist2, misc2, &m);
        place_digit_runs(pk, entry, idx2, n, hist2, m, K,
                         [&](unsigned int pos, unsigned int i) { tmp[pos] = (unsigned int)in[i]; });
        __syncthreads();  // every read of `in` is done before `out` (aliasing it) is written
        for (unsigned int i = threadIdx.x; i < n; i += kThreads) out[i] = tmp[i];
        __syncthreads();
        return;
    }
    // long bucket: sort chunks in shared memory, merge through global memory
    unsigned long long* g0 = scratch64;
    unsigned long long* g1 = scratch64 + n;
    for (unsigned int c0 = 0; c0 < n; c0 += cap) {
        const unsigned int m = min(cap, n - c0);
        for (unsigned int i = threadIdx.x; i < m; i += kThreads) a[i] = in[c0 + i];
        __syncthreads();
        const unsigned long long* sa = a;
        auto pk = [sa](unsigned int i) { return pk_of(sa[i]); };
        auto entry = [sa](unsigned int i) { return sa[i]; };
        DigitMap dm;
        smem_count_sort(pk, b, m, whist, misc, &dm);
        unsigned long long* dst = g0 + c0;  // chunk fully ordered
        place_digit_runs(pk, entry, b, m, whist, dm, K,
                         [&](unsigned int pos, unsigned int i) { dst[pos] = sa[i]; });
        __syncthreads();
    }
    unsigned long long* src = g0;
    unsigned long long* dst = g1;
    for (unsigned int width = cap; width < n; width *= 2) {
        for (unsigned int lo = 0; lo < n; lo += 2 * width) {
            const unsigned int mid = min(n, lo + width), hi = min(n, lo + 2 * width);
            block_merge(src, dst, lo, mid, hi);
        }
        __syncthreads();
        unsigned long long* t = src;
        src = dst;
        dst = t;
    }
    // tie fix-up flags for the long list live in the other global buffer
    fix_primary_ties(src, n, K, reinterpret_cast<unsigned char*>(dst));
    __syncthreads();
    for (unsigned int i = threadIdx.x; i < n; i += kThreads) out[i] = (unsigned int)src[i];
    __syncthreads();
}

}  // namespace tilesort
using tilesort::sort_tile_list;
}  // namespace fs
