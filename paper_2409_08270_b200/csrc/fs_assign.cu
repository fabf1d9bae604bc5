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

__global__ void finalize_kernel(const double* __restrict__ acc, float* __restrict__ out,
                                long long count) {
    const long long stride = (long long)gridDim.x * blockDim.x;
    long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    const long long n2 = count / 2;
    const double2* a2 = reinterpret_cast<const double2*>(acc);
    float2* o2 = reinterpret_cast<float2*>(out);
    for (long long k = i; k < n2; k += stride) {
        double2 v = a2[k];
        o2[k] = make_float2(__double2float_rn(v.x), __double2float_rn(v.y));
    }
    if (i == 0 && (count & 1)) out[count - 1] = __double2float_rn(acc[count - 1]);
}

// mode 0 = binary (E == 2, N labels), mode 1 = scene (E x N membership)
__global__ void __launch_bounds__(256) assign_kernel(const float* __restrict__ A, long long n,
                                                     int e_count, float gamma, int mode,
                                                     uint8_t* __restrict__ out) {
    const long long stride = (long long)gridDim.x * blockDim.x;
    for (long long col = (long long)blockIdx.x * blockDim.x + threadIdx.x; col < n; col += stride) {
        float total = A[col];
        for (int e = 1; e < e_count; ++e) total = __fadd_rn(total, A[(long long)e * n + col]);
        const bool observed = total > 1e-12f;
        const float inv = observed ? __frcp_rn(total) : 0.0f;
        bool any = false;
        for (int e = 1; e < e_count; ++e) {
            const float v = A[(long long)e * n + col];
            const float fg = __fmul_rn(v, inv);
            const float rest = __fadd_rn(__fmul_rn(__fsub_rn(total, v), inv), gamma);
            const bool win = observed && (fg > rest);
            if (mode == 1) {
                out[(long long)e * n + col] = win ? 1 : 0;
                any |= win;
            } else if (e == 1) {
                out[col] = win ? 1 : 0;
            }
        }
        if (mode == 1) out[col] = any ? 0 : 1;  // row 0 = complement of the union (:171)
    }
}

}  // namespace

void launch_finalize(const double* acc, float* out, long long count, cudaStream_t st) {
    if (count <= 0) return;
    long long blocks = (count / 2 + 255) / 256;
    if (blocks > 148 * 16) blocks = 148 * 16;
    if (blocks < 1) blocks = 1;
    finalize_kernel<<<(int)blocks, 256, 0, st>>>(acc, out, count);
}

void launch_assign(const float* A, long long n, int e, float gamma, int mode, uint8_t* out,
                   cudaStream_t st) {
    if (n <= 0) return;
    long long blocks = (n + 255) / 256;
    if (blocks > 148 * 16) blocks = 148 * 16;
    assign_kernel<<<(int)blocks, 256, 0, st>>>(A, n, e, gamma, mode, out);
}

}  // namespace fs
