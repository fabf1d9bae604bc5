// fs_project.cu -- K0 scene setup and K1 EWA projection (reference scene.py:228-312).
//
// Compiled with -fmad=false: every float64 expression below is evaluated in
// the same operation order as the numpy code it restates, with no FMA
// contraction, so the projected means / conics / depths / radii agree with the
// reference to the last ulp except where the reference's BLAS 3x3 matmul
// orders its sums differently.
//
// Layout: the resident scene is structure-of-arrays float64 (means x/y/z,
// the six unique entries of the world covariance, opacity) so a warp reads
// 32 consecutive doubles per field (coalesced 256 B).  The covariance is
// view-independent (scene.py:245-249) and is computed once per scene.
#include "fs_common.cuh"
#include "fs_kernels.cuh"

namespace fs {

// World covariance Sigma = (R S)(R S)^T of a unit quaternion (w, x, y, z) and
// scales (scene.py:228-249) -> its six unique entries (SoA, stride n).
__device__ __forceinline__ void store_covariance(double w, double x, double y, double z, double s0,
                                                 double s1, double s2, double* __restrict__ sig,
                                                 size_t n, int i) {
    double r[9];
    r[0] = 1.0 - 2.0 * (y * y + z * z);
    r[1] = 2.0 * (x * y - w * z);
    r[2] = 2.0 * (x * z + w * y);
    r[3] = 2.0 * (x * y + w * z);
    r[4] = 1.0 - 2.0 * (x * x + z * z);
    r[5] = 2.0 * (y * z - w * x);
    r[6] = 2.0 * (x * z - w * y);
    r[7] = 2.0 * (y * z + w * x);
    r[8] = 1.0 - 2.0 * (x * x + y * y);
    double m[9];
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        m[3 * k + 0] = r[3 * k + 0] * s0;
        m[3 * k + 1] = r[3 * k + 1] * s1;
        m[3 * k + 2] = r[3 * k + 2] * s2;
    }
    // Sigma[i][j] = sum_k m[i][k] m[j][k]; symmetric bit-for-bit (same products, same order)
    auto dot = [&](int a, int b) {
        return m[3 * a + 0] * m[3 * b + 0] + m[3 * a + 1] * m[3 * b + 1] + m[3 * a + 2] * m[3 * b + 2];
    };
    sig[0 * n + i] = dot(0, 0);
    sig[1 * n + i] = dot(0, 1);
    sig[2 * n + i] = dot(0, 2);
    sig[3 * n + i] = dot(1, 1);
    sig[4 * n + i] = dot(1, 2);
    sig[5 * n + i] = dot(2, 2);
}

// K0: AoS host layout (means N x 3, unit quats N x 4, scales N x 3) -> SoA
// means + world covariance Sigma = (R S)(R S)^T (scene.py:228-249).
// Slot p of the resident arrays takes input Gaussian i = perm[p] (spatial order,
// fs_order.cu; perm == nullptr: input order).
__global__ void scene_setup_kernel(int n, const double* __restrict__ means_aos,
                                   const double* __restrict__ quats_aos,
                                   const double* __restrict__ scales_aos,
                                   const double* __restrict__ opac_in,
                                   const unsigned int* __restrict__ perm, double* __restrict__ mx,
                                   double* __restrict__ my, double* __restrict__ mz,
                                   double* __restrict__ sig /* 6 x n */,
                                   double* __restrict__ opac) {
    for (int p = blockIdx.x * blockDim.x + threadIdx.x; p < n; p += gridDim.x * blockDim.x) {
        const size_t i = perm ? perm[p] : (unsigned int)p;
        opac[p] = opac_in[i];
        mx[p] = means_aos[3 * i + 0];
        my[p] = means_aos[3 * i + 1];
        mz[p] = means_aos[3 * i + 2];
        store_covariance(quats_aos[4 * i + 0], quats_aos[4 * i + 1], quats_aos[4 * i + 2],
                         quats_aos[4 * i + 3], scales_aos[3 * i + 0], scales_aos[3 * i + 1],
                         scales_aos[3 * i + 2], sig, (size_t)n, p);
    }
}

// K0 for a splat checkpoint: the PLY's float32 vertex
// records -> the resident float64 scene, with the loader's activations and
// the scene's validation fused in (ply.py:84-98, scene.py:96-110):
//   finite check of every required property             (ply.py:84-88)
//   means = float64(x, y, z)                              (:94)
//   scales = exp(float64(scale_k))                        (:95)
//   opacity = 1 / (1 + exp(-float64(opacity)))            (:96)
//   q = float64(rot_k) / ||q||, ||q|| = sqrt(((q0^2 + q1^2) + q2^2) + q3^2)
//       (np.linalg.norm's sequential sum; scene.py:96-100)
// bad[0..3] collect (atomicMin) the first vertex with a non-finite value, a
// zero / non-finite quaternion norm, a non-positive scale and an opacity
// outside [0, 1]; the host raises the reference's error for the first
// category that fired.  off[] = float offsets within a record, in the
// reference's REQUIRED_PROPERTIES order (x y z nx ny nz f_dc_0..2 opacity
// scale_0..2 rot_0..3).
// Slot p takes vertex i = perm[p]; bad[] and params are by vertex index.
__global__ void scene_setup_ply_kernel(int n, const float* __restrict__ verts, int stride,
                                       PlyOffsets off, const unsigned int* __restrict__ perm,
                                       double* __restrict__ mx, double* __restrict__ my,
                                       double* __restrict__ mz, double* __restrict__ sig,
                                       double* __restrict__ opac,
                                       unsigned long long* __restrict__ bad,
                                       double* __restrict__ params /* nullable: n x 8 */) {
    for (int p = blockIdx.x * blockDim.x + threadIdx.x; p < n; p += gridDim.x * blockDim.x) {
        const unsigned int i = perm ? perm[p] : (unsigned int)p;
        const float* rec = verts + (size_t)i * stride;
        float v[kPlyProps];
        bool finite = true;
#pragma unroll
        for (int k = 0; k < kPlyProps; ++k) {
            v[k] = __ldg(rec + off.k[k]);
            finite &= isfinite(v[k]);
        }
        if (!finite) {
            atomicMin(&bad[0], (unsigned long long)i);
            continue;
        }
        mx[p] = (double)v[0];
        my[p] = (double)v[1];
        mz[p] = (double)v[2];
        const double s0 = exp((double)v[10]), s1 = exp((double)v[11]), s2 = exp((double)v[12]);
        const double o = 1.0 / (1.0 + exp(-(double)v[9]));
        const double q0 = (double)v[13], q1 = (double)v[14], q2 = (double)v[15], q3 = (double)v[16];
        const double norm = sqrt(((q0 * q0 + q1 * q1) + q2 * q2) + q3 * q3);
        if (!(norm > 0.0) || !isfinite(norm)) atomicMin(&bad[1], (unsigned long long)i);
        if (!(s0 > 0.0 && s1 > 0.0 && s2 > 0.0)) atomicMin(&bad[2], (unsigned long long)i);
        if (!(o >= 0.0 && o <= 1.0)) atomicMin(&bad[3], (unsigned long long)i);
        opac[p] = o;
        const double w = q0 / norm, x = q1 / norm, y = q2 / norm, z = q3 / norm;
        store_covariance(w, x, y, z, s0, s1, s2, sig, (size_t)n, p);
        if (params) {  // the activated GaussianScene parameters, for verification
            double* p = params + 8 * (size_t)i;
            p[0] = s0; p[1] = s1; p[2] = s2; p[3] = o;
            p[4] = w; p[5] = x; p[6] = y; p[7] = z;
        }
    }
}

__device__ __forceinline__ void warp_or_and(unsigned long long& o, unsigned long long& a) {
    unsigned int olo = __reduce_or_sync(0xffffffffu, (unsigned int)o);
    unsigned int ohi = __reduce_or_sync(0xffffffffu, (unsigned int)(o >> 32));
    unsigned int alo = __reduce_and_sync(0xffffffffu, (unsigned int)a);
    unsigned int ahi = __reduce_and_sync(0xffffffffu, (unsigned int)(a >> 32));
    o = ((unsigned long long)ohi << 32) | olo;
    a = ((unsigned long long)ahi << 32) | alo;
}

// float32 screen record of a splat with mean (mx, my), conic (ia, ib, ic),
// 2-D covariance diagonal (ca, cc) and opacity o.  alpha >= floor  <=>
// power >= log(floor / o)  <=>  d^T conic d <= qmax.  Screen-only quantities
// are float32: their ~1e-7 relative error is far inside the 1e-5 / 0.01 px /
// 0.02 margins, so the screen stays conservative.
__device__ __forceinline__ Rec32 screen_record(double mx, double my, double ia, double ib,
                                               double ic, double ca, double cc, double o,
                                               double alpha_floor, bool alive, unsigned int oid) {
    Rec32 s;
    s.oid = oid;
    s.mx = (float)mx;
    s.my = (float)my;
    s.a = (float)ia;
    s.b = (float)ib;
    s.c = (float)ic;
    if (alpha_floor > 0.0 && o >= alpha_floor && alive) {
        // MUFU log2 / sqrt: a few 1e-7 relative, far inside the margins below
        const float L = __logf(__fdividef((float)o, (float)alpha_floor));  // log(o / floor) >= 0
        const float qmax = 2.0f * fmaxf(L, 0.0f);
        float sx, sy;
        asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(sx) : "f"(qmax * (float)ca));
        asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(sy) : "f"(qmax * (float)cc));
        const float hx = sx * (1.0f + 1e-5f) + 0.01f;
        const float hy = sy * (1.0f + 1e-5f) + 0.01f;
        const float spread = (fabsf((float)ia) + fabsf((float)ic) + 2.0f * fabsf((float)ib)) *
                             (hx * hx + hy * hy);
        const float margin = 0.02f + 1e-6f * spread;
        s.cut = -L - margin;
        s.hxy = pack_hxy(hx, hy);  // rounded up: still conservative
    } else if (alpha_floor > 0.0) {
        s.cut = __int_as_float(0x7f800000);  // +inf: never passes
        s.hxy = pack_hxy(0.0f, 0.0f);
    } else {
        s.cut = __int_as_float(0xff800000);  // -inf: exact blend, no screen
        s.hxy = pack_hxy(INFINITY, INFINITY);
    }
    return s;
}

// Tiles of the reference rectangle rc (rasterizer.py:106-113) that can hold a
// sample with alpha >= floor.  The raster's strip test rejects a splat for the
// pixel-centre strip [u_lo, u_hi] x [v_lo, v_hi] when u_hi < mx - hx,
// u_lo > mx + hx (same in v) -- float32, these exact expressions; tile t holds
// centres 16t + 0.5 ... 16t + 15.5, so every strip of a tile outside
//   16t + 15.5 >= mx - hx  and  16t + 0.5 <= mx + hx
// is rejected and its instance is dropped here instead (the reference gives
// such samples no weight and no transmittance update, contributions.py:148).
// Exact blend (hx = +inf) keeps the rectangle.  C2: 22% fewer instances.
__device__ __forceinline__ unsigned long long floor_box_rect(unsigned long long rc, const Rec32& s) {
    const float shx = rec_hx(s), shy = rec_hy(s);
    if (rc == ~0ull || !(shx < INFINITY) || !(shy < INFINITY)) return rc;
    const float lx = s.mx - shx, hx = s.mx + shx, ly = s.my - shy, hy = s.my + shy;
    // exact in float64: float + half-integer, then a power-of-two divide
    const double bx0 = ceil(((double)lx - 15.5) / 16.0), bx1 = floor(((double)hx - 0.5) / 16.0);
    const double by0 = ceil(((double)ly - 15.5) / 16.0), by1 = floor(((double)hy - 0.5) / 16.0);
    double tx0 = (double)(rc & 0xFFFF), tx1 = (double)((rc >> 16) & 0xFFFF);
    double ty0 = (double)((rc >> 32) & 0xFFFF), ty1 = (double)((rc >> 48) & 0xFFFF);
    tx0 = fmax(tx0, bx0);
    tx1 = fmin(tx1, bx1);
    ty0 = fmax(ty0, by0);
    ty1 = fmin(ty1, by1);
    if (!(tx0 <= tx1) || !(ty0 <= ty1)) return ~0ull;
    return (unsigned long long)tx0 | ((unsigned long long)tx1 << 16) |
           ((unsigned long long)ty0 << 32) | ((unsigned long long)ty1 << 48);
}

// K1: one thread per Gaussian.  Mirrors _project_arrays (scene.py:252-312)
// and tile_range (rasterizer.py:106-113); emits the depth sort key, the tile
// rectangle and the walk records.  cull_floor > 0 additionally drops (from
// binning only) Gaussians whose opacity is below the alpha floor: they can
// never pass `alpha >= alpha_floor` (contributions.py:148), so they touch no
// pixel.  Stats keep the reference's meaning regardless.
__global__ void __launch_bounds__(256, 4) project_kernel(
    int n, const double* __restrict__ gmx, const double* __restrict__ gmy,
    const double* __restrict__ gmz, const double* __restrict__ sig,
    const double* __restrict__ opac, Camera cam, double alpha_floor, int cull_floor,
    unsigned long long* __restrict__ keys, unsigned long long* __restrict__ rect,
    Rec32* __restrict__ r32, Rec64* __restrict__ r64, ViewCounters* __restrict__ vc,
    ProjectExport ex) {
    const double* W = cam.w2c;
    const int tx_n = tiles_x_of(cam.width), ty_n = tiles_y_of(cam.height);
    __shared__ unsigned long long s_or[8], s_and[8];
    __shared__ unsigned int s_cnt[4];
    if (threadIdx.x < 4) s_cnt[threadIdx.x] = 0;
    __syncthreads();
    unsigned long long k_or = 0, k_and = ~0ull;
    unsigned int c_emit = 0, c_behind = 0, c_deg = 0, c_off = 0;
    // grid-stride, but every thread runs the same number of iterations so the
    // warp reductions below stay convergent
    const int stride = gridDim.x * blockDim.x;
    const int iters = (n + stride - 1) / stride;
    for (int it = 0; it < iters; ++it) {
        const int i = it * stride + blockIdx.x * blockDim.x + threadIdx.x;
        if (i < n) {
            // slot i holds input Gaussian ex.perm[i]: member, exports and the
            // record's oid are by input id
            const unsigned int gin = ex.perm ? ex.perm[i] : (unsigned int)i;
            double m0 = gmx[i], m1 = gmy[i], m2 = gmz[i];
            // cam = means @ rot.T + t   (scene.py:266)
            double x = (m0 * W[0] + m1 * W[1] + m2 * W[2]) + W[3];
            double y = (m0 * W[4] + m1 * W[5] + m2 * W[6]) + W[7];
            double z = (m0 * W[8] + m1 * W[9] + m2 * W[10]) + W[11];
            bool alive = z > cam.near_clip;  // :268
            if (!alive) ++c_behind;
            double zs = alive ? z : 1.0;      // :272
            double mxp = cam.fx * x / zs + cam.cx;  // :274-275
            double myp = cam.fy * y / zs + cam.cy;
            double S[9];
            S[0] = sig[i];
            S[1] = sig[(size_t)n + i];
            S[2] = sig[2 * (size_t)n + i];
            S[4] = sig[3 * (size_t)n + i];
            S[5] = sig[4 * (size_t)n + i];
            S[8] = sig[5 * (size_t)n + i];
            S[3] = S[1];
            S[6] = S[2];
            S[7] = S[5];
            // sigma_cam = rot @ sigma @ rot.T  (:278)
            double T[9], C[9];
#pragma unroll
            for (int a = 0; a < 3; ++a)
#pragma unroll
                for (int b = 0; b < 3; ++b)
                    T[3 * a + b] = W[4 * a + 0] * S[0 + b] + W[4 * a + 1] * S[3 + b] + W[4 * a + 2] * S[6 + b];
#pragma unroll
            for (int a = 0; a < 3; ++a)
#pragma unroll
                for (int b = 0; b < 3; ++b)
                    C[3 * a + b] = T[3 * a + 0] * W[4 * b + 0] + T[3 * a + 1] * W[4 * b + 1] + T[3 * a + 2] * W[4 * b + 2];
            // J (:280-284) and cov2d = J C J^T (:285)
            double j00 = cam.fx / zs, j02 = -cam.fx * x / (zs * zs);
            double j11 = cam.fy / zs, j12 = -cam.fy * y / (zs * zs);
            double js0[3], js1[3];
#pragma unroll
            for (int c = 0; c < 3; ++c) {
                js0[c] = j00 * C[0 + c] + 0.0 * C[3 + c] + j02 * C[6 + c];
                js1[c] = 0.0 * C[0 + c] + j11 * C[3 + c] + j12 * C[6 + c];
            }
            double c00 = js0[0] * j00 + js0[1] * 0.0 + js0[2] * j02;
            double c01 = js0[0] * 0.0 + js0[1] * j11 + js0[2] * j12;
            double c11 = js1[0] * 0.0 + js1[1] * j11 + js1[2] * j12;
            double a = c00 + kDilation, b = c01, c = c11 + kDilation;  // :286-288
            double det = a * c - b * b;                                // :290
            if (alive && det <= kDegenerateDet) {
                ++c_deg;
                alive = false;
            }
            double ds = det > kDegenerateDet ? det : 1.0;  // :295
            double ia = c / ds, ib = -b / ds, ic = a / ds; // :296
            double mid = 0.5 * (a + c);                     // :298-301
            double disc = sqrt(fmax(0.25 * ((a - c) * (a - c)) + b * b, 0.0));
            double lam = fmax(mid + disc, 0.0);
            double rad = ceil(3.0 * sqrt(lam));
            if (alive && ((mxp + rad < 0.0) || (mxp - rad > (double)cam.width) ||
                          (myp + rad < 0.0) || (myp - rad > (double)cam.height))) {
                ++c_off;  // :303-310
                alive = false;
            }
            double o = opac[i];
            unsigned long long key = ~0ull, rc = ~0ull;
            if (ex.member && !ex.member[gin]) alive = false;  // not in the rendered subset
            if (alive) {
                ++c_emit;
                key = f64_sort_key(z);
                k_or |= key;
                k_and &= key;
                // tile_range (rasterizer.py:106-113), inclusive floor box
                const bool transparent = cull_floor && alpha_floor > 0.0 && !(o >= alpha_floor);
                if (!transparent) rc = tile_rect(mxp, myp, rad, tx_n, ty_n);
            }
            keys[i] = key;
            const Rec32 s = screen_record(mxp, myp, ia, ib, ic, a, c, o, alpha_floor, alive, gin);
            // binning for a floored walk: only tiles the raster's strip test can accept
            if (cull_floor && alpha_floor > 0.0) rc = floor_box_rect(rc, s);
            rect[i] = rc;
            // walk records (float64 exact, float32 screen) -- only for splats that are
            // binned: culled and fully transparent ones are never read, so their 80 B
            // are not written (views that see part of the scene skip most of them)
            if (rc != ~0ull) {
                Rec64 q;
                q.mx = mxp;
                q.my = myp;
                q.a = ia;
                q.b = ib;
                q.c = ic;
                q.o = o;
                r64[i] = q;
                r32[i] = s;
            }
            if (ex.alive) {
                ex.alive[gin] = alive ? 1 : 0;
                ex.mean2d[2 * (size_t)gin] = mxp;
                ex.mean2d[2 * (size_t)gin + 1] = myp;
                ex.conic[3 * (size_t)gin] = ia;
                ex.conic[3 * (size_t)gin + 1] = ib;
                ex.conic[3 * (size_t)gin + 2] = ic;
                ex.depth[gin] = z;
                ex.radius[gin] = (int64_t)rad;
            }
        }
    }
    // block reduction of the counters and of the key OR/AND
    warp_or_and(k_or, k_and);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (lane == 0) {
        s_or[warp] = k_or;
        s_and[warp] = k_and;
    }
    atomicAdd(&s_cnt[0], c_emit);
    atomicAdd(&s_cnt[1], c_behind);
    atomicAdd(&s_cnt[2], c_deg);
    atomicAdd(&s_cnt[3], c_off);
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned long long o = 0, a = ~0ull;
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w) {
            o |= s_or[w];
            a &= s_and[w];
        }
        if (s_cnt[0]) {
            atomicOr(&vc->key_or, o);
            atomicOr(&vc->key_nand, ~a);
            atomicAdd(&vc->n_emitted, s_cnt[0]);
        }
        if (s_cnt[1]) atomicAdd(&vc->n_behind, s_cnt[1]);
        if (s_cnt[2]) atomicAdd(&vc->n_degenerate, s_cnt[2]);
        if (s_cnt[3]) atomicAdd(&vc->n_offscreen, s_cnt[3]);
    }
}

// Resets the per-view counters (first node of every view).
__global__ void view_begin_kernel(ViewCounters* vc) {
    if (threadIdx.x == 0) {
        ViewCounters z{};
        *vc = z;  // every field's empty state is zero
    }
}

void launch_view_begin(ViewCounters* vc, cudaStream_t st) { view_begin_kernel<<<1, 32, 0, st>>>(vc); }

void launch_scene_setup(int n, const double* means, const double* quats, const double* scales,
                        const double* opac_in, const unsigned int* perm, double* mx, double* my,
                        double* mz, double* sig, double* opac, cudaStream_t st) {
    if (n <= 0) return;
    int grid = (n + 255) / 256;
    if (grid > 4096) grid = 4096;
    scene_setup_kernel<<<grid, 256, 0, st>>>(n, means, quats, scales, opac_in, perm, mx, my, mz,
                                             sig, opac);
}

void launch_scene_setup_ply(int n, const float* verts, int stride, const PlyOffsets& off,
                            const unsigned int* perm, double* mx, double* my, double* mz,
                            double* sig, double* opac, unsigned long long* bad, double* params,
                            cudaStream_t st) {
    if (n <= 0) return;
    int grid = (n + 255) / 256;
    if (grid > 4096) grid = 4096;
    scene_setup_ply_kernel<<<grid, 256, 0, st>>>(n, verts, stride, off, perm, mx, my, mz, sig, opac,
                                                 bad, params);
}

void launch_project(int n, const double* mx, const double* my, const double* mz,
                    const double* sig, const double* opac, const Camera& cam, double alpha_floor,
                    int cull_floor, unsigned long long* keys, unsigned long long* rect,
                    Rec32* r32, Rec64* r64,
                    ViewCounters* vc, ProjectExport ex, int num_sms, cudaStream_t st,
                    bool reset_counters, bool overlapped) {
    if (reset_counters) view_begin_kernel<<<1, 32, 0, st>>>(vc);
    if (n <= 0) return;
    int grid = (n + 255) / 256;
    // 8 blocks per SM alone on the GPU; 4 beside other streams' rasters (the
    // accumulate loop): C2 67.6 -> 66.9 ms (2 per SM: 67.1; C4 within 0.5%)
    int cap = num_sms * (overlapped ? 4 : 8);
    if (grid > cap) grid = cap;
    project_kernel<<<grid, 256, 0, st>>>(n, mx, my, mz, sig, opac, cam, alpha_floor, cull_floor,
                                         keys, rect, r32, r64, vc, ex);
}

// Records of an explicit splat list (render_property over a caller's
// TileBinning, rasterizer.py:133-203): the float64 walk record, the float32
// screen (covariance diagonal recovered from the conic) and the depth key.
__global__ void splat_records_kernel(int k, const double* __restrict__ mean2d,
                                     const double* __restrict__ conic,
                                     const double* __restrict__ depth,
                                     const double* __restrict__ opac, double alpha_floor,
                                     Rec32* __restrict__ r32, Rec64* __restrict__ r64,
                                     unsigned long long* __restrict__ k64) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < k; i += gridDim.x * blockDim.x) {
        const double mx = mean2d[2 * i], my = mean2d[2 * i + 1];
        const double ia = conic[3 * i], ib = conic[3 * i + 1], ic = conic[3 * i + 2];
        const double o = opac[i];
        Rec64 q;
        q.mx = mx;
        q.my = my;
        q.a = ia;
        q.b = ib;
        q.c = ic;
        q.o = o;
        r64[i] = q;
        const double det = ia * ic - ib * ib;  // conic = inverse covariance
        const bool ok = det > 0.0;
        Rec32 s = screen_record(mx, my, ia, ib, ic, ok ? ic / det : 0.0, ok ? ia / det : 0.0, o,
                                alpha_floor, true, (unsigned int)i);  // oid: the splat (channel row)
        if (!ok && alpha_floor > 0.0) {  // degenerate conic: no finite screen box
            s.cut = __int_as_float(0xff800000);
            s.hxy = pack_hxy(INFINITY, INFINITY);
        }
        r32[i] = s;
        k64[i] = f64_sort_key(depth[i]);
    }
}

void launch_splat_records(int k, const double* mean2d, const double* conic, const double* depth,
                          const double* opac, double alpha_floor, Rec32* r32, Rec64* r64,
                          unsigned long long* k64, int num_sms, cudaStream_t st) {
    if (k <= 0) return;
    int grid = (k + 255) / 256;
    if (grid > num_sms * 8) grid = num_sms * 8;
    splat_records_kernel<<<grid, 256, 0, st>>>(k, mean2d, conic, depth, opac, alpha_floor, r32, r64,
                                               k64);
}

}  // namespace fs
