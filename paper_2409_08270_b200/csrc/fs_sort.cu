// fs_sort.cu -- stable LSD radix sort with device-resident counts (K2a / K2c).
//
// Used twice per view:
//   * depth sort: 64-bit order-preserving float64 depth keys, values = gid.
//     Input is in gid order, so stability breaks depth ties by index exactly
//     like np.lexsort((indices, depths)) (rasterizer.py:91).
//   * tile sort: 32-bit tile ids, values = gid, input in depth-rank order, so
//     every tile's list comes out depth-ordered (rasterizer.py:92-99).
//
// Every kernel takes the element count from device memory and a fixed grid,
// so a whole view can be captured in one CUDA graph without host syncs.
// A pass whose 8-bit digit is constant over all valid keys (known from the
// device-side OR/AND of the keys) is skipped by all three of its kernels; the
// ping-pong parity is recomputed by every kernel from the same mask.
//
// Per pass: upsweep (per-block digit histogram) -> one-block exclusive scan of
// the digit-major histogram -> downsweep (stable block-local ranking with
// warp match_any, scatter).  Blocks own contiguous chunks, tiles inside a
// chunk are processed in order, warps inside a tile own consecutive 256-key
// slices: the scatter is stable.
#include "fs_common.cuh"
#include "fs_kernels.cuh"

namespace fs {

namespace {

constexpr int kSortThreads = 256;
constexpr int kSortWarps = kSortThreads / 32;
constexpr int kItemsPerWarp = 256;  // 8 iterations x 32 lanes
constexpr int kTileKeys = kSortWarps * kItemsPerWarp;

__device__ __forceinline__ unsigned int load_count(const unsigned int* d_n, unsigned int n_fixed) {
    return d_n ? *d_n : n_fixed;
}

__device__ __forceinline__ void chunk_of(unsigned int n, int b, int g, unsigned int& lo,
                                         unsigned int& hi) {
    unsigned int chunk = (n + g - 1) / g;
    chunk = (chunk + 31u) & ~31u;
    lo = min((unsigned long long)n, (unsigned long long)chunk * b);
    hi = min((unsigned long long)n, (unsigned long long)chunk * (b + 1));
}

template <typename K>
__device__ __forceinline__ K fix_key(K k, unsigned long long and_mask) {
    // invisible entries carry the all-ones sentinel; give them a key that is
    // constant in every skipped digit (they are filtered later by rect = empty)
    return k == (K)~(K)0 ? (K)and_mask : k;
}

template <typename K>
__global__ void __launch_bounds__(kSortThreads) upsweep_kernel(
    const K* __restrict__ k0, const K* __restrict__ k1, const unsigned int* __restrict__ d_n,
    unsigned int n_fixed, const unsigned long long* __restrict__ oa, int pass,
    unsigned int* __restrict__ hist) {
    const unsigned long long varying = oa[0] ^ oa[1];
    const int shift = 8 * pass;
    if (!pass_active(varying, shift)) return;
    const K* keys = pass_parity(varying, pass) ? k1 : k0;
    __shared__ unsigned int s_hist[kSortWarps][256];
    for (int i = threadIdx.x; i < kSortWarps * 256; i += kSortThreads) (&s_hist[0][0])[i] = 0;
    __syncthreads();
    unsigned int n = load_count(d_n, n_fixed), lo, hi;
    chunk_of(n, blockIdx.x, gridDim.x, lo, hi);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (unsigned int base = lo + warp * 32; base < hi; base += kSortThreads) {
        unsigned int idx = base + lane;
        bool valid = idx < hi;
        unsigned int d = 0;
        if (valid) d = (unsigned int)((fix_key<K>(keys[idx], oa[1]) >> shift) & 0xFF);
        unsigned int peers = __match_any_sync(0xffffffffu, valid ? d : 256u + lane);
        if (valid && lane == 31 - __clz(peers)) s_hist[warp][d] += __popc(peers);
        __syncwarp();
    }
    __syncthreads();
    for (int d = threadIdx.x; d < 256; d += kSortThreads) {
        unsigned int s = 0;
#pragma unroll
        for (int w = 0; w < kSortWarps; ++w) s += s_hist[w][d];
        hist[(size_t)d * gridDim.x + blockIdx.x] = s;
    }
}

// One block: exclusive scan (in place) over the digit-major histogram.
__global__ void __launch_bounds__(1024) scan_hist_kernel(unsigned int* __restrict__ hist,
                                                         int entries,
                                                         const unsigned long long* __restrict__ oa,
                                                         int pass) {
    if (oa && !pass_active(oa[0] ^ oa[1], 8 * pass)) return;
    __shared__ unsigned int s_part[1024];
    const int per = (entries + blockDim.x - 1) / blockDim.x;
    const int lo = threadIdx.x * per, hi = min(entries, lo + per);
    unsigned int sum = 0;
    for (int i = lo; i < hi; ++i) sum += hist[i];
    s_part[threadIdx.x] = sum;
    __syncthreads();
    // Hillis-Steele inclusive scan over 1024 partials
    for (int off = 1; off < (int)blockDim.x; off <<= 1) {
        unsigned int v = threadIdx.x >= (unsigned)off ? s_part[threadIdx.x - off] : 0;
        __syncthreads();
        s_part[threadIdx.x] += v;
        __syncthreads();
    }
    unsigned int run = threadIdx.x ? s_part[threadIdx.x - 1] : 0;
    for (int i = lo; i < hi; ++i) {
        unsigned int v = hist[i];
        hist[i] = run;
        run += v;
    }
}

template <typename K>
__global__ void __launch_bounds__(kSortThreads) downsweep_kernel(
    K* k0, unsigned int* v0, K* k1, unsigned int* v1, const unsigned int* __restrict__ d_n,
    unsigned int n_fixed,
    const unsigned long long* __restrict__ oa, int pass, const unsigned int* __restrict__ hist) {
    const unsigned long long varying = oa[0] ^ oa[1];
    const int shift = 8 * pass;
    if (!pass_active(varying, shift)) return;
    const bool flip = pass_parity(varying, pass);
    const K* src_k = flip ? k1 : k0;
    const unsigned int* src_v = flip ? v1 : v0;
    K* dst_k = flip ? k0 : k1;
    unsigned int* dst_v = flip ? v0 : v1;

    __shared__ unsigned int s_cnt[kSortWarps][256];
    __shared__ unsigned int s_off[256];
    unsigned int n = load_count(d_n, n_fixed), lo, hi;
    chunk_of(n, blockIdx.x, gridDim.x, lo, hi);
    for (int d = threadIdx.x; d < 256; d += kSortThreads) s_off[d] = hist[(size_t)d * gridDim.x + blockIdx.x];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const unsigned int lt_mask = (1u << lane) - 1u;
    for (unsigned int tile = lo; tile < hi; tile += kTileKeys) {
        for (int i = threadIdx.x; i < kSortWarps * 256; i += kSortThreads) (&s_cnt[0][0])[i] = 0;
        __syncthreads();
        K key[8];
        unsigned int val[8], rank[8], dig[8];
#pragma unroll
        for (int it = 0; it < 8; ++it) {
            unsigned int idx = tile + warp * kItemsPerWarp + it * 32 + lane;
            bool valid = idx < hi;
            key[it] = valid ? fix_key<K>(src_k[idx], oa[1]) : (K)0;
            val[it] = valid ? src_v[idx] : 0u;
            unsigned int d = (unsigned int)((key[it] >> shift) & 0xFF);
            dig[it] = valid ? d : 0xFFFFFFFFu;
            unsigned int peers = __match_any_sync(0xffffffffu, valid ? d : 256u + lane);
            unsigned int before = valid ? s_cnt[warp][d] : 0u;
            __syncwarp();
            if (valid && lane == 31 - __clz(peers)) s_cnt[warp][d] = before + __popc(peers);
            __syncwarp();
            rank[it] = before + __popc(peers & lt_mask);
        }
        __syncthreads();
        for (int d = threadIdx.x; d < 256; d += kSortThreads) {
            unsigned int run = s_off[d];
#pragma unroll
            for (int w = 0; w < kSortWarps; ++w) {
                unsigned int c = s_cnt[w][d];
                s_cnt[w][d] = run;
                run += c;
            }
            s_off[d] = run;
        }
        __syncthreads();
#pragma unroll
        for (int it = 0; it < 8; ++it) {
            if (dig[it] != 0xFFFFFFFFu) {
                unsigned int pos = s_cnt[warp][dig[it]] + rank[it];
                dst_k[pos] = key[it];
                dst_v[pos] = val[it];
            }
        }
        __syncthreads();
    }
}

}  // namespace

int sort_grid(int num_sms) { return 2 * num_sms; }

size_t sort_hist_entries(int num_sms) { return (size_t)256 * sort_grid(num_sms); }

template <typename K>
int launch_radix_sort(K* keys0, unsigned int* vals0, K* keys1, unsigned int* vals1,
                      const unsigned int* d_n, unsigned int n_fixed,
                      const unsigned long long* d_or_and, int passes, unsigned int* hist,
                      int num_sms, cudaStream_t st) {
    const int g = sort_grid(num_sms);
    for (int p = 0; p < passes; ++p) {
        upsweep_kernel<K><<<g, kSortThreads, 0, st>>>(keys0, keys1, d_n, n_fixed, d_or_and, p, hist);
        scan_hist_kernel<<<1, 1024, 0, st>>>(hist, 256 * g, d_or_and, p);
        downsweep_kernel<K><<<g, kSortThreads, 0, st>>>(keys0, vals0, keys1, vals1, d_n, n_fixed,
                                                        d_or_and, p, hist);
    }
    return 0;
}

template int launch_radix_sort<unsigned long long>(unsigned long long*, unsigned int*,
                                                   unsigned long long*, unsigned int*,
                                                   const unsigned int*, unsigned int,
                                                   const unsigned long long*, int, unsigned int*,
                                                   int, cudaStream_t);
template int launch_radix_sort<unsigned int>(unsigned int*, unsigned int*, unsigned int*,
                                             unsigned int*, const unsigned int*, unsigned int,
                                             const unsigned long long*, int, unsigned int*, int,
                                             cudaStream_t);

void launch_scan_hist(unsigned int* data, int entries, cudaStream_t st) {
    scan_hist_kernel<<<1, 1024, 0, st>>>(data, entries, nullptr, 0);
}

}  // namespace fs
