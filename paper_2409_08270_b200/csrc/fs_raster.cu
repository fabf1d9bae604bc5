// fs_raster.cu -- K3: per-tile front-to-back compositing that scatters alpha*T
// into the E x N float64 contribution accumulator (reference
// contributions.py:119-160, the `_accumulate_view` walk).
//
// One CTA per 16x16 tile, one thread per pixel (warp w owns tile rows 2w and
// 2w+1).  The tile's depth-ordered list is streamed through shared memory in
// batches of 256 records (one coalesced gather per thread).  For every list
// entry each warp:
//   1. skips the entry if its 2x16 pixel strip misses the entry's alpha-floor
//      ellipse box (warp-uniform, no per-lane math);
//   2. evaluates a float32 power and compares it with a conservative cut --
//      lanes that certainly have alpha < alpha_floor stop here (the reference
//      gives them no weight and no transmittance update, contributions.py:148);
//   3. runs the exact float64 path on the surviving lanes: the reference's
//      expression order without FMA contraction, float64 exp, the 0.99 clamp,
//      the alpha floor, w = alpha*T, T *= (1-alpha), T floor after the update;
//   4. aggregates: label-uniform warps reduce w with shuffles and issue one
//      float64 atomic; mixed-label warps issue one atomic per contributing lane.
// The CTA stops when no pixel of the tile is active (contributions.py:158-159).
#include "fs_common.cuh"
#include "fs_kernels.cuh"

namespace fs {

namespace {

constexpr int kRasterThreads = 256;
constexpr int kBatch = 256;

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

__global__ void __launch_bounds__(kRasterThreads, 4) raster_kernel(RasterArgs a) {
    const ViewCounters* vc = a.vc;
    if (vc->overflow) return;
    const int tile = blockIdx.x;
    const unsigned int begin = a.tile_start[tile], end = a.tile_start[tile + 1];
    if (begin >= end) return;
    const unsigned int* __restrict__ gids =
        pass_parity(a.tile_or_and[0] ^ a.tile_or_and[1], a.tile_passes) ? a.inst_gid[1] : a.inst_gid[0];

    __shared__ Rec32 s_r32[kBatch];
    __shared__ Rec64 s_r64[kBatch];
    __shared__ unsigned int s_gid[kBatch];

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int x0 = (tile % a.tiles_x) * kTile, y0 = (tile / a.tiles_x) * kTile;
    const int px = x0 + (tid & 15), py = y0 + (tid >> 4);
    const bool inside = px < a.width && py < a.height;
    const unsigned int label = inside ? a.mask[(size_t)py * a.width + px] : 0u;
    // pixel centre (k + 0.5, j + 0.5): exact in both precisions
    const double pxc = (double)px + 0.5, pyc = (double)py + 0.5;
    const float pxf = (float)pxc, pyf = (float)pyc;
    // the warp's pixel-centre strip
    const float u_lo = (float)x0 + 0.5f, u_hi = (float)x0 + 15.5f;
    const float v_lo = (float)(y0 + 2 * warp) + 0.5f, v_hi = v_lo + 1.0f;

    const unsigned int inside_mask = __ballot_sync(0xffffffffu, inside);
    const int first = inside_mask ? __ffs(inside_mask) - 1 : 0;
    const unsigned int lbl0 = __shfl_sync(0xffffffffu, label, first);
    const bool uniform = __all_sync(0xffffffffu, !inside || label == lbl0);

    const double af = a.alpha_floor, tf = a.t_floor;
    const long long n_g = a.n_gaussians;
    double* __restrict__ acc = a.acc;

    double T = 1.0;
    bool active = inside;
    bool warp_live = inside_mask != 0u;
    unsigned long long steps = 0, exact = 0, atom = 0;

    for (unsigned int b = begin; b < end; b += kBatch) {
        // contributions.py:158-159 -- the whole tile terminated; also guards smem reuse
        if (__syncthreads_count(active) == 0) break;
        const unsigned int i = b + tid;
        if (i < end) {
            const unsigned int g = gids[i];
            s_gid[tid] = g;
            s_r32[tid] = a.r32[g];
            s_r64[tid] = a.r64[g];
        }
        __syncthreads();
        const int nb = min((unsigned int)kBatch, end - b);
        steps += nb;
        if (!warp_live) continue;
        for (int j = 0; j < nb; ++j) {
            const Rec32 s = s_r32[j];
            if (u_hi < s.mx - s.hx || u_lo > s.mx + s.hx || v_hi < s.my - s.hy || v_lo > s.my + s.hy)
                continue;
            const float du = pxf - s.mx, dv = pyf - s.my;
            const float p = -0.5f * (s.a * du * du + s.c * dv * dv) - s.b * du * dv;
            const bool cand = active && p >= s.cut;
            const unsigned int cand_mask = __ballot_sync(0xffffffffu, cand);
            if (!cand_mask) continue;
            exact += __popc(cand_mask);
            double w = 0.0;
            if (cand) {
                const Rec64 q = s_r64[j];
                // power = -0.5 * (a*du*du + c*dv*dv) - b*du*dv   (contributions.py:142-145)
                const double ddu = __dsub_rn(pxc, q.mx);
                const double ddv = __dsub_rn(pyc, q.my);
                const double t1 = __dmul_rn(__dmul_rn(q.a, ddu), ddu);
                const double t2 = __dmul_rn(__dmul_rn(q.c, ddv), ddv);
                const double t3 = __dmul_rn(__dmul_rn(q.b, ddu), ddv);
                const double power = __dsub_rn(__dmul_rn(-0.5, __dadd_rn(t1, t2)), t3);
                double alpha = __dmul_rn(q.o, exp(power));  // :146-147
                alpha = alpha < kAlphaClamp ? alpha : kAlphaClamp;
                const bool use = af > 0.0 ? (alpha >= af) : true;  // :148-149
                if (use) {
                    w = __dmul_rn(alpha, T);                    // :150
                    T = __dmul_rn(T, __dsub_rn(1.0, alpha));    // :155
                    if (tf > 0.0 && !(T >= tf)) active = false; // :156-157
                }
            }
            const unsigned int contrib = __ballot_sync(0xffffffffu, w > 0.0);
            if (contrib) {
                const unsigned int g = s_gid[j];
                if (uniform) {
                    const double sum = warp_sum(w);
                    if (lane == 0) atomicAdd(acc + (size_t)lbl0 * n_g + g, sum);
                    ++atom;
                } else {
                    if (w > 0.0) atomicAdd(acc + (size_t)label * n_g + g, w);
                    atom += __popc(contrib);
                }
            }
            if (tf > 0.0) {
                warp_live = __any_sync(0xffffffffu, active);
                if (!warp_live) break;
            }
        }
    }
    // per-CTA counters (one atomic each)
    __shared__ unsigned long long s_e[8], s_a[8];
    if (lane == 0) {
        s_e[warp] = exact;
        s_a[warp] = atom;
    }
    __syncthreads();
    if (tid == 0) {
        unsigned long long e = 0, at = 0;
        for (int w = 0; w < kRasterThreads / 32; ++w) {
            e += s_e[w];
            at += s_a[w];
        }
        ViewCounters* v = a.vc;
        atomicAdd(&v->tile_steps, steps);
        atomicAdd(&v->exact_evals, e);
        atomicAdd(&v->atomics, at);
    }
}

}  // namespace

void launch_raster(const RasterArgs& a, cudaStream_t st) {
    if (a.ntiles <= 0) return;
    raster_kernel<<<a.ntiles, kRasterThreads, 0, st>>>(a);
}

}  // namespace fs
