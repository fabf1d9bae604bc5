// fs_sort.cu -- stable LSD radix sort with device-resident counts (K2a / K2c).
//
// Used per view:
//   * depth sort: 64-bit order-preserving float64 depth keys, values = gid.
//     Input is in gid order, so stability breaks depth ties by index exactly
//     like np.lexsort((indices, depths)) (rasterizer.py:91).
//   * tile sort: 32-bit tile ids, values = gid, input in depth-rank order, so
//     every tile's list comes out depth-ordered (rasterizer.py:92-99).
//
// Onesweep structure (one kernel per digit pass):
//   hist   one read of all keys -> 256-bin histograms of every digit position
//          (positions known constant from the key OR/AND are skipped);
//   scan   one block: exclusive scan of each position's histogram, the mask
//          of passes that actually permute (no bin holds all keys), a new
//          epoch for the look-back status words, tile counters reset;
//   pass   per 2048-key tile (ids claimed in launch order with an atomic):
//          warp-level stable ranking with match_any, tile digit counts
//          published as (epoch, AGGREGATE, count), decoupled look-back over
//          earlier tiles to the first (epoch, INCLUSIVE, prefix), scatter.
// Counts come from device memory and grids from capacities, so a whole view
// needs no host round trip.  Ping-pong parity = number of permuting passes
// before the current one; consumers read it from SortState::active.
#include <algorithm>

#include "fs_common.cuh"
#include "fs_kernels.cuh"

namespace fs {

namespace {

constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;
constexpr int kItems = 8;                       // keys per lane per tile
constexpr int kTileKeys = kThreads * kItems;    // 2048 keys per sub-tile
constexpr int kSub = 4;                         // sub-tiles per block tile
constexpr int kBlockKeys = kSub * kTileKeys;    // 8192 keys per look-back tile
constexpr int kWindow = 8;                      // look-back window (tiles per round trip)
constexpr unsigned long long kFlagAgg = 1ull << 32;
constexpr unsigned long long kFlagInc = 2ull << 32;

// Status words carry their own payload (flag + count), so relaxed gpu-scope
// accesses suffice: no other memory is published through them.  (acquire
// loads compile to an L1 invalidate per load -- CCTL.IVALL -- which made the
// look-back 3x slower.)
__device__ __forceinline__ unsigned long long ld_status(const unsigned long long* p) {
    unsigned long long v;
    asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}

__device__ __forceinline__ void st_status(unsigned long long* p, unsigned long long v) {
    asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

template <typename K>
__device__ __forceinline__ K fix_key(K k, const unsigned long long* sub) {
    // invisible entries carry the all-ones sentinel; give them the AND of the
    // valid keys so they never widen the set of permuting digits
    return (sub && k == (K)~(K)0) ? (K)sub[0] : k;
}

__device__ __forceinline__ unsigned int load_n(const unsigned int* d_n, unsigned int n_fixed) {
    return d_n ? *d_n : n_fixed;
}

// digits that may vary: from the key OR/AND when known, else all
__device__ __forceinline__ bool digit_may_vary(const unsigned long long* oa, int p) {
    return oa ? ((((oa[0] ^ oa[1]) >> (8 * p)) & 0xFFull) != 0ull) : true;
}

template <typename K>
__global__ void __launch_bounds__(kThreads) hist_kernel(const K* __restrict__ keys,
                                                        const unsigned int* __restrict__ d_n,
                                                        unsigned int n_fixed, int passes,
                                                        const unsigned long long* __restrict__ oa,
                                                        const unsigned long long* __restrict__ sub,
                                                        SortState* __restrict__ st) {
    __shared__ unsigned int s_hist[8][256];
    for (int i = threadIdx.x; i < 8 * 256; i += kThreads) (&s_hist[0][0])[i] = 0;
    __syncthreads();
    const unsigned int n = load_n(d_n, n_fixed);
    bool vary[8];
#pragma unroll
    for (int p = 0; p < 8; ++p) vary[p] = p < passes && digit_may_vary(oa, p);
    const int lane = threadIdx.x & 31;
    const unsigned int stride = gridDim.x * kThreads;
    const unsigned int iters = (n + stride - 1) / stride;
    for (unsigned int it = 0; it < iters; ++it) {
        const unsigned int i = it * stride + blockIdx.x * kThreads + threadIdx.x;
        const bool valid = i < n;
        const K k = valid ? fix_key<K>(keys[i], sub) : (K)0;
#pragma unroll
        for (int p = 0; p < 8; ++p) {
            if (!vary[p]) continue;
            const unsigned int d = (unsigned int)((k >> (8 * p)) & 0xFF);
            const unsigned int peers = __match_any_sync(0xffffffffu, valid ? d : 256u + lane);
            if (valid && lane == 31 - __clz(peers)) atomicAdd(&s_hist[p][d], __popc(peers));
        }
    }
    __syncthreads();
    for (int p = 0; p < passes; ++p) {
        if (!vary[p]) continue;
        const int d = threadIdx.x;
        if (s_hist[p][d]) atomicAdd(&st->offsets[p][d], s_hist[p][d]);
    }
}

// one block of 256 threads
__global__ void __launch_bounds__(256) scan_kernel(const unsigned int* __restrict__ d_n,
                                                   unsigned int n_fixed, int passes,
                                                   const unsigned long long* __restrict__ oa,
                                                   SortState* __restrict__ st) {
    __shared__ unsigned int s[256];
    __shared__ int s_full;
    const unsigned int n = load_n(d_n, n_fixed);
    const int d = threadIdx.x;
    unsigned int active = 0;
    for (int p = 0; p < passes; ++p) {
        const unsigned int c = digit_may_vary(oa, p) ? st->offsets[p][d] : (d == 0 ? n : 0u);
        if (d == 0) s_full = 0;
        __syncthreads();
        if (c == n) s_full = 1;  // every key in one bin: the pass is the identity
        s[d] = c;
        __syncthreads();
        for (int off = 1; off < 256; off <<= 1) {  // inclusive Hillis-Steele scan
            const unsigned int y = d >= off ? s[d - off] : 0u;
            __syncthreads();
            s[d] += y;
            __syncthreads();
        }
        st->offsets[p][d] = s[d] - c;
        if (!s_full) active |= 1u << p;
        __syncthreads();
    }
    if (d < 8) st->tile_counter[d] = 0;
    if (d == 0) {
        st->active = n > 1 ? active : 0u;
        st->epoch = st->epoch + 1;
    }
}

template <typename K>
__global__ void __launch_bounds__(kThreads, 2) pass_kernel(
    K* k0, unsigned int* v0, K* k1, unsigned int* v1, const unsigned int* __restrict__ d_n,
    unsigned int n_fixed, int pass, const unsigned long long* __restrict__ sub,
    SortState* __restrict__ st, unsigned long long* __restrict__ status /* tiles x 256 */) {
    const unsigned int active = st->active;
    if (!((active >> pass) & 1u)) return;
    const unsigned int n = load_n(d_n, n_fixed);
    __shared__ unsigned int s_tile;
    __shared__ unsigned short s_cnt[kSub][kWarps][256];  // per (sub-tile, warp) digit counts
    __shared__ unsigned char s_rank[kBlockKeys];          // rank inside the (sub, warp, digit) group
    __shared__ unsigned int s_base[256];
    if (threadIdx.x == 0) s_tile = atomicAdd(&st->tile_counter[pass], 1u);
    for (int i = threadIdx.x; i < kSub * kWarps * 256 / 2; i += kThreads)
        reinterpret_cast<unsigned int*>(&s_cnt[0][0][0])[i] = 0u;
    __syncthreads();
    const unsigned int tile = s_tile;
    const unsigned int base = tile * kBlockKeys;
    if (base >= n) return;
    const bool flip = __popc(active & ((1u << pass) - 1u)) & 1;
    const K* src_k = flip ? k1 : k0;
    const unsigned int* src_v = flip ? v1 : v0;
    K* dst_k = flip ? k0 : k1;
    unsigned int* dst_v = flip ? v0 : v1;
    // status tag unique per (sort call, pass): passes of one sort share the buffer
    const unsigned int epoch = (st->epoch * 8u + (unsigned)pass) & 0x3FFFFFFFu;
    const int shift = 8 * pass;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const unsigned int lt_mask = (1u << lane) - 1u;

    // phase 1: stable ranks and (sub-tile, warp) digit counts; key order inside
    // the block tile is (sub, warp, item, lane)
    for (int sb = 0; sb < kSub; ++sb) {
#pragma unroll
        for (int it = 0; it < kItems; ++it) {
            const unsigned int off = sb * kTileKeys + warp * (32 * kItems) + it * 32 + lane;
            const unsigned int idx = base + off;
            const bool valid = idx < n;
            const K key = valid ? fix_key<K>(src_k[idx], sub) : (K)0;
            const unsigned int d = (unsigned int)((key >> shift) & 0xFF);
            const unsigned int peers = __match_any_sync(0xffffffffu, valid ? d : 256u + lane);
            const unsigned int before = valid ? s_cnt[sb][warp][d] : 0u;
            __syncwarp();
            if (valid && lane == 31 - __clz(peers))
                s_cnt[sb][warp][d] = (unsigned short)(before + __popc(peers));
            __syncwarp();
            s_rank[off] = (unsigned char)(before + __popc(peers & lt_mask));
        }
    }
    __syncthreads();
    {
        // tile digit totals -> exclusive (sub, warp) prefixes; publish + look back
        const int d = threadIdx.x;
        unsigned int run = 0;
        for (int sb = 0; sb < kSub; ++sb)
#pragma unroll
            for (int w = 0; w < kWarps; ++w) {
                const unsigned int c = s_cnt[sb][w][d];
                s_cnt[sb][w][d] = (unsigned short)run;
                run += c;
            }
        unsigned long long* my = status + (size_t)tile * 256 + d;
        const unsigned long long tag = (unsigned long long)epoch << 34;
        unsigned int excl = 0;
        if (tile == 0) {
            st_status(my, tag | kFlagInc | run);
        } else {
            st_status(my, tag | kFlagAgg | run);
            // windowed look-back: kWindow independent loads in flight per step
            long long t = (long long)tile - 1;
            bool done = false;
            while (!done) {
                unsigned long long win[kWindow];
#pragma unroll
                for (int k = 0; k < kWindow; ++k)
                    win[k] = (t - k >= 0) ? ld_status(status + (size_t)(t - k) * 256 + d)
                                          : (tag | kFlagInc);  // before tile 0: prefix 0
                int k = 0;
#pragma unroll
                for (int q = 0; q < kWindow; ++q) {
                    if (done || q != k) continue;
                    const unsigned long long s = win[q];
                    if ((unsigned int)(s >> 34) != epoch || !(s & (3ull << 32))) continue;  // not ready
                    excl += (unsigned int)(s & 0xFFFFFFFFull);
                    if (s & kFlagInc) done = true;
                    ++k;
                }
                t -= k;  // resume at the first entry that was not ready
            }
            st_status(my, tag | kFlagInc | (excl + run));
        }
        s_base[d] = st->offsets[pass][d] + excl;
    }
    __syncthreads();
    // phase 2: re-read (L2-hot) and scatter
    for (int sb = 0; sb < kSub; ++sb) {
#pragma unroll
        for (int it = 0; it < kItems; ++it) {
            const unsigned int off = sb * kTileKeys + warp * (32 * kItems) + it * 32 + lane;
            const unsigned int idx = base + off;
            if (idx < n) {
                const K key = fix_key<K>(src_k[idx], sub);
                const unsigned int d = (unsigned int)((key >> shift) & 0xFF);
                const unsigned int pos = s_base[d] + s_cnt[sb][warp][d] + s_rank[off];
                dst_k[pos] = key;
                dst_v[pos] = src_v[idx];
            }
        }
    }
}

__global__ void sort_reset_kernel(SortState* st) {
    // zero the histograms before every sort (the epoch survives)
    for (int i = threadIdx.x; i < 8 * 256; i += blockDim.x) (&st->offsets[0][0])[i] = 0;
}

}  // namespace

size_t sort_status_words(unsigned int n_cap) {
    return (size_t)std::max(1u, (n_cap + kBlockKeys - 1) / kBlockKeys) * 256;
}

template <typename K>
int launch_radix_sort(K* keys0, unsigned int* vals0, K* keys1, unsigned int* vals1,
                      const unsigned int* d_n, unsigned int n_cap,
                      const unsigned long long* d_or_and, const unsigned long long* sub, int passes,
                      SortState* st, unsigned long long* status, int num_sms, cudaStream_t s) {
    sort_reset_kernel<<<1, 256, 0, s>>>(st);
    const int hist_grid = std::min<long long>(num_sms * 4, std::max<long long>(1, ((long long)n_cap + kThreads * 8 - 1) / (kThreads * 8)));
    hist_kernel<K><<<hist_grid, kThreads, 0, s>>>(keys0, d_n, n_cap, passes, d_or_and, sub, st);
    scan_kernel<<<1, 256, 0, s>>>(d_n, n_cap, passes, d_or_and, st);
    const int tiles = (int)(sort_status_words(n_cap) / 256);
    for (int p = 0; p < passes; ++p)
        pass_kernel<K><<<tiles, kThreads, 0, s>>>(keys0, vals0, keys1, vals1, d_n, n_cap, p, sub,
                                                  st, status);
    return 3 + passes;
}

template int launch_radix_sort<unsigned long long>(unsigned long long*, unsigned int*,
                                                   unsigned long long*, unsigned int*,
                                                   const unsigned int*, unsigned int,
                                                   const unsigned long long*,
                                                   const unsigned long long*, int, SortState*,
                                                   unsigned long long*, int, cudaStream_t);
template int launch_radix_sort<unsigned int>(unsigned int*, unsigned int*, unsigned int*,
                                             unsigned int*, const unsigned int*, unsigned int,
                                             const unsigned long long*, const unsigned long long*,
                                             int, SortState*, unsigned long long*, int,
                                             cudaStream_t);

}  // namespace fs
