// fs_assign.cu -- K5 finalize (float64 accumulator -> float32 matrix,
// contributions.py:116) and K4 biased one-vs-rest argmax (solver.py:118-172).
//
// The argmax reproduces the reference's float32 sequence bit for bit:
//   total = sum_e v[e]        sequential e = 0..E-1, each add rounded   (:126)
//   observed = total > 1e-12f                                            (:127)
//   inv = 1/total (IEEE, correctly rounded), 0 where unobserved          (:128-130)
//   fg = v*inv ; rest = ((total - v) * inv) + f32(gamma)                 (:131-134)
//   win = fg > rest && observed (strict: ties stay background)          (:135-136)
// Explicit __f*_rn intrinsics forbid FMA contraction (SURVEY.md fact 4:
// contraction flips ~1% of near-tie labels).  One thread per Gaussian
// column; loads along N are coalesced across the warp.
#include "fs_common.cuh"
#include "fs_kernels.cuh"

namespace fs {

namespace {

// Exact value of a FS_ACC_FIXED entry: (hi * 2^32 + lo) * 2^-59, one rounding
// (hi + lo's carry stays below 2^53 for any reachable total).
__device__ __forceinline__ double fixed_value(unsigned long long hi, unsigned long long lo) {
    const unsigned long long h = hi + (lo >> 32);
    return __dadd_rn(__dmul_rn(__ull2double_rn(h), 0x1p-27),
                     __dmul_rn(__ull2double_rn(lo & 0xffffffffull), 0x1p-59));
}

// Entry `at` of the accumulator summed over the parts (one per GPU / shard):
// fixed-point parts add exactly as integers; float64 parts in part order.
template <bool kFixed>
__device__ __forceinline__ double part_sum(const AccParts& P, size_t at) {
    if (kFixed) {
        unsigned long long hi = 0, lo = 0;
        for (int i = 0; i < P.n; ++i) {
            const ulonglong2 w = __ldcs(reinterpret_cast<const ulonglong2*>(P.p[i]) + at);
            hi += w.x;
            lo += w.y;
        }
        return fixed_value(hi, lo);
    }
    double v = __ldcs(static_cast<const double*>(P.p[0]) + at);
    for (int i = 1; i < P.n; ++i) v = __dadd_rn(v, __ldcs(static_cast<const double*>(P.p[i]) + at));
    return v;
}

// N x E accumulator(s) (Gaussian-major) -> E x (g1 - g0) float32 (the API
// layout, row stride ld), the contributions.py:116 cast, for Gaussians
// [g0, g1).  With several parts this is the reduce half of a reduce-scatter
// fused into the cast: the parts are other GPUs' accumulators read over
// NVLink peer memory.  Small E: one thread per Gaussian (its E entries are
// contiguous; the E stores are coalesced across the warp).
template <bool kFixed>
__global__ void finalize_small_kernel(AccParts P, float* __restrict__ out, long long ld,
                                      long long g0, long long g1, int e) {
    const long long stride = (long long)gridDim.x * blockDim.x;
    for (long long g = g0 + (long long)blockIdx.x * blockDim.x + threadIdx.x; g < g1; g += stride)
        for (int l = 0; l < e; ++l)
            out[(long long)l * ld + (g - g0)] = __double2float_rn(part_sum<kFixed>(P, (size_t)g * e + l));
}

// Larger E: 32 x 32 tiles transposed through shared memory.
template <bool kFixed>
__global__ void __launch_bounds__(256) finalize_tile_kernel(AccParts P, float* __restrict__ out,
                                                            long long ld, long long g0,
                                                            long long g1, int e) {
    __shared__ float t[32][33];
    const long long gb = g0 + (long long)blockIdx.x * 32;
    const int l0 = blockIdx.y * 32, tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
    for (int r = ty; r < 32; r += 8) {
        const long long g = gb + r;
        const int l = l0 + tx;
        if (g < g1 && l < e) t[tx][r] = __double2float_rn(part_sum<kFixed>(P, (size_t)g * e + l));
    }
    __syncthreads();
    for (int r = ty; r < 32; r += 8) {
        const int l = l0 + r;
        const long long g = gb + tx;
        if (l < e && g < g1) out[(long long)l * ld + (g - g0)] = t[r][tx];
    }
}

// mode 0 = binary (E == 2, n labels), mode 1 = scene (E x n membership);
// A and out have row stride ld (a column slice of a wider matrix).
__global__ void __launch_bounds__(256) assign_kernel(const float* __restrict__ A, long long n,
                                                     long long ld, int e_count, float gamma,
                                                     int mode, uint8_t* __restrict__ out) {
    const long long stride = (long long)gridDim.x * blockDim.x;
    for (long long col = (long long)blockIdx.x * blockDim.x + threadIdx.x; col < n; col += stride) {
        float total = A[col];
        for (int e = 1; e < e_count; ++e) total = __fadd_rn(total, A[(long long)e * ld + col]);
        const bool observed = total > 1e-12f;
        const float inv = observed ? __frcp_rn(total) : 0.0f;
        bool any = false;
        for (int e = 1; e < e_count; ++e) {
            const float v = A[(long long)e * ld + col];
            const float fg = __fmul_rn(v, inv);
            const float rest = __fadd_rn(__fmul_rn(__fsub_rn(total, v), inv), gamma);
            const bool win = observed && (fg > rest);
            if (mode == 1) {
                out[(long long)e * ld + col] = win ? 1 : 0;
                any |= win;
            } else if (e == 1) {
                out[col] = win ? 1 : 0;
            }
        }
        if (mode == 1) out[col] = any ? 0 : 1;  // row 0 = complement of the union (:171)
    }
}

// Nonzero bytes per row of a rows x n uint8 matrix (Assignment.member_counts,
// solver.py:73-77): 16-byte loads, per-byte compare, block sum, one atomic per
// block and row.
__global__ void __launch_bounds__(256) row_count_kernel(const uint8_t* __restrict__ m, long long n,
                                                        unsigned long long* __restrict__ counts) {
    __shared__ unsigned int s_w[8];
    const uint8_t* row = m + (long long)blockIdx.y * n;
    const long long stride = (long long)gridDim.x * blockDim.x;
    unsigned int c = 0;
    const long long head = (16 - (long long)(reinterpret_cast<uintptr_t>(row) & 15)) & 15;
    const long long h = head < n ? head : n;
    const long long nv = (n - h) / 16;
    const uint4* v = reinterpret_cast<const uint4*>(row + h);
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < nv; i += stride) {
        const uint4 q = v[i];
        c += __popc(__vcmpne4(q.x, 0u) & 0x01010101u) + __popc(__vcmpne4(q.y, 0u) & 0x01010101u) +
             __popc(__vcmpne4(q.z, 0u) & 0x01010101u) + __popc(__vcmpne4(q.w, 0u) & 0x01010101u);
    }
    if (blockIdx.x == 0) {  // unaligned head and the tail
        for (long long i = threadIdx.x; i < h; i += blockDim.x) c += row[i] != 0;
        for (long long i = h + nv * 16 + threadIdx.x; i < n; i += blockDim.x) c += row[i] != 0;
    }
    c = __reduce_add_sync(0xffffffffu, c);
    if ((threadIdx.x & 31) == 0) s_w[threadIdx.x >> 5] = c;
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned long long t = 0;
        for (int w = 0; w < 8; ++w) t += s_w[w];
        if (t) atomicAdd(counts + blockIdx.y, t);
    }
}

}  // namespace

void launch_row_counts(const uint8_t* m, long long n, int rows, unsigned long long* counts,
                       cudaStream_t st) {
    if (n <= 0 || rows <= 0) return;
    long long bx = (n / 16 + 255) / 256;
    if (bx > 148 * 4) bx = 148 * 4;
    if (bx < 1) bx = 1;
    // one grid row per matrix row; gridDim.y is capped at 65 535 and a scene
    // assignment can have 65 536 rows (every uint16 label an object)
    for (int r0 = 0; r0 < rows; r0 += 65535) {
        const int nr = rows - r0 < 65535 ? rows - r0 : 65535;
        row_count_kernel<<<dim3((unsigned)bx, (unsigned)nr), 256, 0, st>>>(m + (long long)r0 * n, n,
                                                                          counts + r0);
    }
}

void launch_finalize(const AccParts& parts, bool fixed, long long g0, long long g1, int e,
                     float* out, long long ld, cudaStream_t st) {
    const long long n = g1 - g0;
    if (n <= 0 || e <= 0) return;
    if (e <= 8) {
        long long blocks = (n + 255) / 256;
        if (blocks > 148 * 16) blocks = 148 * 16;
        if (fixed)
            finalize_small_kernel<true><<<(int)blocks, 256, 0, st>>>(parts, out, ld, g0, g1, e);
        else
            finalize_small_kernel<false><<<(int)blocks, 256, 0, st>>>(parts, out, ld, g0, g1, e);
    } else {
        dim3 grid((unsigned)((n + 31) / 32), (unsigned)((e + 31) / 32));
        if (fixed)
            finalize_tile_kernel<true><<<grid, 256, 0, st>>>(parts, out, ld, g0, g1, e);
        else
            finalize_tile_kernel<false><<<grid, 256, 0, st>>>(parts, out, ld, g0, g1, e);
    }
}

void launch_assign(const float* A, long long n, long long ld, int e, float gamma, int mode,
                   uint8_t* out, cudaStream_t st) {
    if (n <= 0) return;
    long long blocks = (n + 255) / 256;
    if (blocks > 148 * 16) blocks = 148 * 16;
    assign_kernel<<<(int)blocks, 256, 0, st>>>(A, n, ld, e, gamma, mode, out);
}

}  // namespace fs
