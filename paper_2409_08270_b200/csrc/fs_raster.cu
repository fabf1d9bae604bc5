// fs_raster.cu -- K3: per-tile front-to-back compositing that scatters alpha*T
// into the N x E (Gaussian-major) float64 contribution accumulator (reference
// contributions.py:119-160, the `_accumulate_view` walk), and -- instantiated
// with kRender -- the per-pixel compositing of render_property
// (rasterizer.py:133-203).
//
// One CTA per 16x16 tile, launched longest bucket first; prologue: the tile's
// bucket is TMA-copied into shared memory and sorted into the reference's
// (depth, id) order (fs_tilesort.cuh).  One thread per pixel; warp w owns tile
// rows 2w and 2w+1, and the eight warps walk the list independently -- no
// block barriers after the sort:
//
//   gather   32 list entries per step (software-pipelined: records one step
//            ahead, gids two ahead): each lane tests its entry's alpha-floor
//            ellipse box against the warp's 2x16 strip and solves the float32
//            quadratic for both rows (conservative margins: samples certainly
//            below alpha_floor are dropped -- the reference gives them no
//            weight and no transmittance update, contributions.py:148); hits
//            with candidate pixels go, in list order, to a per-warp ring;
//   per mini-batch of 16 hits:
//   A  their float64 records are staged in shared memory; a warp bit-matrix
//      transpose gives every lane (pixel) its 16-bit candidate mask; the
//      (splat, pixel) pairs are packed lane-major by one prefix sum;
//   A2 exact float64 alpha per pair -- reference expression order, no FMA
//      contraction, float64 exp, 0.99 clamp, 0 below the floor -- 32 pairs per
//      round on full warps (alpha does not depend on T);
//   B  every lane walks its own candidates in list order: w = alpha*T,
//      T *= (1-alpha), T floor after the update (:150-157);
//   C  warps with at most 4 distinct labels reduce w per (splat, label) with a
//      padded transpose in shared memory + a shuffle and issue one float64
//      atomic each; warps with more labels issue one atomic per contributing
//      pixel.  The accumulator is Gaussian-major (N x E): the labels of one
//      splat share its cache lines.
// A warp stops when none of its pixels is active (contributions.py:158-159:
// pixels are independent, the reference's tile-level break is an
// optimisation of the same rule).  The label range check of
// contributions.py:108-114 runs here too, for every tile.
#include <algorithm>

#include "fs_common.cuh"
#include "fs_kernels.cuh"
#include "fs_tilesort.cuh"

namespace fs {

namespace {

constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;
constexpr int kMini = 16;      // strip hits per mini-batch
constexpr int kRing = 64;       // per-warp ring of strip hits (>= kMini - 1 + 32)
constexpr int kRowStride = 33;  // doubles per padded w/alpha row (bank-conflict-free transpose)
constexpr int kMaxGroups = 4;   // label groups per warp reduced before the atomics
// A warp's pixel block: kBH rows x kBW columns of the 16 x 16 tile, lane l at
// column l % kBW, row l / kBW (bit l of a candidate mask).
#ifndef FS_BLOCK_W
#define FS_BLOCK_W 8
#endif
constexpr int kBW = FS_BLOCK_W;
constexpr int kBH = 32 / kBW;
static_assert(kBW == 8 || kBW == 16, "warp pixel blocks are 2 x 16 or 4 x 8");

struct WarpSmem {
    Rec64 rec[kMini];        // float64 records of the mini-batch's hits
    unsigned int cm[kRing];  // candidate pixels of the hit (bit = lane)
    unsigned int gid[kRing];  // scene slot of the hit (record index)
    unsigned int oid[kRing];  // its input Gaussian id (accumulator / channel row, Rec32::oid)
    unsigned short queue[kMini * 32];
    unsigned int gmask[kMaxGroups];  // the warp's label groups (fixed for the walk)
    unsigned int glab[kMaxGroups];

    double val[kMini * kRowStride];  // alpha, then w
};

struct RasterSmem {
    WarpSmem w[kWarps];
};

// The prologue's tile sort (fs_tilesort.cuh) and the walk share the same bytes;
// sorting inside the raster kernel overlaps its latency with other CTAs' walks.
constexpr size_t kSortBytes = 8 * ((size_t)kTileSortCap + 2) + 4 * (2048 + 64) + 2 * (size_t)kTileSortCap;
union RasterShared {
    RasterSmem walk;
    unsigned char sort[kSortBytes];
};
// dynamic shared memory per CTA; 4 CTAs per SM must stay resident
constexpr size_t kRasterSmem = sizeof(RasterShared);
static_assert(4 * (kRasterSmem + 1024) <= 228 * 1024, "raster needs 4 resident CTAs per SM");

// float64 add into the accumulator as a fire-and-forget RED: atomicAdd with an
// unused result still compiles to ATOMG (the L2 returns the old value); RED
// takes 7% off the C2 raster launch
__device__ __forceinline__ void red_add(double* p, double v) {
    asm volatile("red.global.add.f64 [%0], %1;" ::"l"(p), "d"(v) : "memory");
}

// Deterministic accumulator (FS_ACC_FIXED): an entry is two uint64 words
// (hi, lo) holding sum(q >> 32) and sum(q & 0xffffffff) for q = v * 2^59
// rounded to an integer (v < 32: one RED carries at most 32 pixels' weights,
// each < 1).  Integer adds commute, so the sum -- and the float32 matrix made
// from it -- is independent of the order the REDs land in, of the stream
// schedule and of how views are split over GPUs.  Resolution 2^-59 per RED.
__device__ __forceinline__ void red_fixed(unsigned long long* p, double v) {
    const unsigned long long q = __double2ull_rn(__dmul_rn(v, 0x1p59));
    asm volatile("red.global.add.u64 [%0], %1;" ::"l"(p), "l"(q >> 32) : "memory");
    asm volatile("red.global.add.u64 [%0], %1;" ::"l"(p + 1), "l"(q & 0xffffffffull) : "memory");
}

template <bool kFixed>
__device__ __forceinline__ void acc_add(double* acc, unsigned long long* acc_fx, size_t at,
                                        double v) {
    if (kFixed)
        red_fixed(acc_fx + 2 * at, v);
    else
        red_add(acc + at, v);
}

// 32 x 32 bit-matrix transpose across the warp (lane i holds row i, bit j =
// M[i][j]; on return lane j holds column j) when only rows 0..15 can be nonzero
// (a mini-batch has at most 16 hits).  The full transpose swaps off-diagonal
// blocks of halving size with five shuffles; its first stage (16-bit halves
// between lane and lane ^ 16) is done by the caller's load -- lane l < 16 brings
// row l's low half, lane l >= 16 row (l - 16)'s high half -- so four remain.
__device__ __forceinline__ unsigned int warp_transpose16x32(unsigned int x, int lane) {
    const unsigned int masks[4] = {0x00FF00FFu, 0x0F0F0F0Fu, 0x33333333u, 0x55555555u};
#pragma unroll
    for (int s = 0; s < 4; ++s) {
        const int b = 8 >> s;
        const unsigned int m = masks[s];
        const unsigned int y = __shfl_xor_sync(0xffffffffu, x, b);
        x = (lane & b) ? ((x & ~m) | ((y & ~m) >> b)) : ((x & m) | ((y & m) << b));
    }
    return x;
}

// Candidate mask of a whole kBH x kBW block (bit r * kBW + c = pixel (xb + c,
// v_lo - 0.5 + r)): per row, the pixels whose float32 power clears the
// conservative cut, from the roots of the quadratic
//   a du^2 + 2 b dv du + c dv^2 <= Q,   Q = -2 * cut
// widened by float32 rounding margins (1e-5 relative on the discriminant, 0.03 px
// + 1e-5 relative on the interval ends); the splat's per-row invariants (1/a, Q,
// det, a*Q) are computed once.  sqrt / rcp are the MUFU approximations (~1e-7
// relative, far inside the margins).
__device__ __forceinline__ unsigned int block_candidates(const Rec32& s, float v_lo, int xb) {
    if (!(s.cut > -INFINITY)) return 0xffffffffu;  // exact blend: no alpha floor
    float inv_a;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(inv_a) : "f"(s.a));
    const float Q = -2.0f * s.cut;
    const float detc = s.a * s.c - s.b * s.b;
    const float t1 = s.a * Q, at1 = fabsf(t1);
    const float base = s.mx - 0.5f, binv = s.b * inv_a;
    unsigned int cand = 0;
#pragma unroll
    for (int r = 0; r < kBH; ++r) {
        const float dv = (v_lo + (float)r) - s.my;
        const float t2 = detc * dv * dv;
        const float D = t1 - t2 + 1e-5f * (at1 + fabsf(t2)) + 1e-20f;
        if (D >= 0.0f) {
            float sq;
            asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(sq) : "f"(D));
            const float ctr = base - binv * dv;
            const float half = sq * inv_a;
            const float eps = 0.03f + 1e-5f * fabsf(ctr);
            // the same interval with rounding conversions and integer clamps; empty
            // when c1 < c0 (bounded to +-1e9 first so the block offset cannot overflow)
            const int c0 = max(__float2int_ru(fminf(ctr - half - eps, 1.0e9f)) - xb, 0);
            const int c1 = min(__float2int_rd(fmaxf(ctr + half + eps, -1.0e9f)) - xb, kBW - 1);
            if (c0 <= c1) cand |= ((2u << c1) - (1u << c0)) << (r * kBW);
        }
    }
    return cand;
}

// float64 depth of a gid from its order-preserving key (inverse of f64_sort_key)
__device__ __forceinline__ double depth_of_key(unsigned long long k) {
    return __longlong_as_double((long long)((k >> 63) ? (k & 0x7fffffffffffffffull) : ~k));
}

// kRender = false: accumulate alpha*T into the N x E float64 accumulator (contributions.py:119-160).
// kRender = true:  composite alpha, depth and an optional channel per pixel
//                  (render_property, rasterizer.py:133-203); no mask, no atomics.
// kFixed: the accumulator is FS_ACC_FIXED (two uint64 words per entry), else float64.
template <bool kRender, bool kFixed>
__global__ void __launch_bounds__(kThreads, 4) raster_kernel(RasterArgs a) {
    const ViewCounters* vc = a.vc;
    if (vc->overflow) return;
    const int tile = (int)a.tile_order[blockIdx.x];  // longest buckets first
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    // the warp's pixel block inside the tile, and this lane's pixel
    const int xb = (tile % a.tiles_x) * kTile + (warp % (kTile / kBW)) * kBW;
    const int yb = (tile / a.tiles_x) * kTile + (warp / (kTile / kBW)) * kBH;
    const int px = xb + lane % kBW, py = yb + lane / kBW;
    const bool inside = px < a.width && py < a.height;
    const unsigned int label = (!kRender && inside) ? a.mask[(size_t)py * a.width + px] : 0u;
    if (!kRender) {
        // label range check of every pixel, empty tiles included
        // (contributions.py:108-114; the host reports the first bad view)
        const unsigned int m = __reduce_max_sync(0xffffffffu, label);
        if (lane == 0 && m >= (unsigned)a.num_objects) atomicMax(&a.vc->max_label, m);
    }
    const unsigned int begin = a.sort.tile_start[tile], end = a.sort.tile_start[tile + 1];
    if (begin >= end) return;
    const unsigned int n_list = end - begin;

    extern __shared__ __align__(16) unsigned char raster_smem[];
    RasterShared& SH = *reinterpret_cast<RasterShared*>(raster_smem);
    __shared__ unsigned long long s_cnt[3];
    __shared__ unsigned int s_done;
    if (threadIdx.x < 3) s_cnt[threadIdx.x] = 0;
    if (threadIdx.x == 0) s_done = 0;  // the tile sort's barriers publish these
    RasterSmem& S = SH.walk;
    const unsigned int* __restrict__ list;
    if (kRender && a.render.lists) {
        list = a.render.lists + begin;  // caller's binning, already in reference order
        __syncthreads();
    } else {
        // prologue: the tile's bucket -> gids in the reference (depth, id) order
        unsigned int* sorted = sorted_view(a.sort.inst, begin);
        sort_tile_list(a.sort.inst + begin, sorted, a.sort.scratch64 + 2ull * begin, n_list,
                       a.sort.keys, SH.sort, a.sort.cap, kRasterSmem);
        list = sorted;
    }
    WarpSmem& W = S.w[warp];
    const unsigned int lt_mask = (1u << lane) - 1u;
    // the warp's pixel-centre strip
    const float u_lo = (float)xb + 0.5f, u_hi = u_lo + (float)(kBW - 1);
    const float v_lo = (float)yb + 0.5f, v_hi = v_lo + (float)(kBH - 1);

    // The warp's label groups (fixed for the whole walk): lanes sharing a label.
    // With at most kMaxGroups distinct labels, C reduces w per (splat, label)
    // and issues one atomic each; otherwise one atomic per contributing pixel.
    const unsigned int grp = __match_any_sync(0xffffffffu, inside ? label : 0xffffffffu);
    const unsigned int leaders = __ballot_sync(0xffffffffu, inside && lane == __ffs(grp) - 1);
    const bool grouped = __popc(leaders) <= kMaxGroups;
    // out-of-range labels (reported through max_label) never address the accumulator
    const bool lbl_ok = label < (unsigned)a.num_objects;
    // group table in shared memory: C reads it with broadcast loads instead of shuffles
    // (the shuffle unit is the raster's contended resource)
    const int n_groups = __popc(leaders);
    if (grouped && ((leaders >> lane) & 1u)) {
        const int slot = __popc(leaders & ((1u << lane) - 1u));
        W.gmask[slot] = grp;
        W.glab[slot] = label;
    }
    __syncwarp();

    const double af_eff = a.af_eff, tf_eff = a.tf_eff;
    const unsigned int n_obj = (unsigned)a.num_objects;  // accumulator row length (N x E)
    double* __restrict__ acc = a.acc;
    unsigned long long* __restrict__ acc_fx = a.acc_fixed;
    double* __restrict__ myval = W.val;

    double T = 1.0;
    bool active = inside;
    // render accumulators (rasterizer.py:168-172)
    double r_acc = 0.0, d_acc = 0.0, v_acc[3] = {0.0, 0.0, 0.0};
    const int n_ch = kRender ? a.render.channels : 0;
    unsigned long long steps = 0, exact = 0, atom = 0;
    int head = 0, cnt = 0;  // ring of strip hits

    // software pipeline: records one chunk ahead, gids two chunks ahead
    unsigned int g_next = (unsigned)lane < n_list ? list[lane] : 0u;
    Rec32 s_next;
    if ((unsigned)lane < n_list) s_next = a.r32[g_next];
    unsigned int g_next2 = (unsigned)lane + 32 < n_list ? list[lane + 32] : 0u;
    for (unsigned int c = 0; c < n_list && __any_sync(0xffffffffu, active); c += 32) {
        // ---- gather + A: 32 entries; float32 screen of the warp's two rows ----
        const unsigned int idx = c + lane;
        unsigned int g = g_next, cand = 0;
        const Rec32 s = s_next;
        if (idx + 32 < n_list) {
            s_next = a.r32[g_next2];
            g_next = g_next2;
        }
        if (idx + 64 < n_list) g_next2 = list[idx + 64];
        if (idx < n_list) {
            const float hx = rec_hx(s), hy = rec_hy(s);
            if (!(u_hi < s.mx - hx || u_lo > s.mx + hx || v_hi < s.my - hy || v_lo > s.my + hy)) {
                cand = block_candidates(s, v_lo, xb);
            }
        }
        steps += min(32u, n_list - c);
        const bool hit = cand != 0u;
        const unsigned int bal = __ballot_sync(0xffffffffu, hit);
        if (hit) {
            FS_CHECK(g < (unsigned)a.n_gaussians && cnt + __popc(bal) <= kRing);
            const int slot = (head + cnt + __popc(bal & lt_mask)) & (kRing - 1);
            W.cm[slot] = cand;
            W.gid[slot] = g;
            W.oid[slot] = s.oid;
        }
        cnt += __popc(bal);
        __syncwarp();
        const bool last = c + 32 >= n_list;
        while (cnt >= kMini || (last && cnt > 0)) {
            const int nm = min(kMini, cnt);
            const unsigned int act = __ballot_sync(0xffffffffu, active);
            if (!act) {
                cnt = 0;
                break;
            }
            // the batch's float64 records: loads in flight while the pairs are packed
            Rec64 rq;
            if (lane < nm) rq = a.r64[W.gid[(head + lane) & (kRing - 1)]];
            // this lane's candidates of the mini-batch (bit k = k-th strip hit)
            unsigned int mine = 0u;
            if ((lane & 15) < nm) {
                const unsigned int row = W.cm[(head + (lane & 15)) & (kRing - 1)];
                mine = lane < 16 ? (row & 0xFFFFu) : (row >> 16);
            }
            mine = warp_transpose16x32(mine, lane);
            if (!active) mine = 0;
            // lane-major packing of the (splat, pixel) pairs: warp prefix sum
            const unsigned int n_mine = __popc(mine);
            // n_mine <= 16 (5 bits): the prefix from one ballot per bit -- votes, not
            // shuffles (the shuffle unit is the contended resource; -1.4% raster time)
            unsigned int incl = 0, total_u = 0;
#pragma unroll
            for (int bbit = 0; bbit < 5; ++bbit) {
                const unsigned int bal = __ballot_sync(0xffffffffu, (n_mine >> bbit) & 1u);
                incl += (unsigned int)__popc(bal & (lt_mask | (1u << lane))) << bbit;
                total_u += (unsigned int)__popc(bal) << bbit;
            }
            const int total = (int)total_u;
            if (total > 0) {
                exact += total;
                // ---- A2: exact float64 alpha on packed (splat, pixel) pairs ----
                {
                    unsigned int mm = mine, q = incl - n_mine;
                    while (mm) {
                        const int k = __ffs(mm) - 1;
                        mm &= mm - 1u;
                        FS_CHECK(q < (unsigned)(kMini * 32) && k < nm);
                        W.queue[q++] = (unsigned short)((k << 5) | lane);
                    }
                }
                if (lane < nm) W.rec[lane] = rq;
                __syncwarp();
                for (int q0 = lane; q0 < total; q0 += 32) {
                    const unsigned int e = W.queue[q0];
                    const int k = e >> 5, src = e & 31;
                    FS_CHECK(k < nm && q0 < kMini * 32);
                    const Rec64 q = W.rec[k];
                    // pixel centre (k + 0.5, j + 0.5) of the source lane, exact in float64
                    const double cx = (double)(xb + src % kBW) + 0.5;
                    const double cy = (double)(yb + src / kBW) + 0.5;
                    // power = -0.5 * (a*du*du + c*dv*dv) - b*du*dv   (contributions.py:142-145)
                    const double ddu = __dsub_rn(cx, q.mx);
                    const double ddv = __dsub_rn(cy, q.my);
                    const double t1 = __dmul_rn(__dmul_rn(q.a, ddu), ddu);
                    const double t2 = __dmul_rn(__dmul_rn(q.c, ddv), ddv);
                    const double t3 = __dmul_rn(__dmul_rn(q.b, ddu), ddv);
                    const double power = __dsub_rn(__dmul_rn(-0.5, __dadd_rn(t1, t2)), t3);
                    const double alpha = __dmul_rn(q.o, exp(power));  // :146-147
                    const double ac = alpha < kAlphaClamp ? alpha : kAlphaClamp;
                    // below the floor: no weight, no transmittance update (:148-149) --
                    // exactly what alpha = 0 does in B (w = 0 * T, T * (1 - 0) = T)
                    myval[k * kRowStride + src] = ac >= af_eff ? ac : 0.0;
                }
                __syncwarp();
                // ---- B: every lane walks its own candidates in list order ----
                if (kRender || grouped) {
                    unsigned int mm = mine;
                    while (mm) {
                        const int k = __ffs(mm) - 1;
                        mm &= mm - 1u;
                        double w = 0.0;
                        if (active) {
                            const double alpha = myval[k * kRowStride + lane];  // 0: below floor
                            w = __dmul_rn(alpha, T);                     // :150
                            T = __dmul_rn(T, __dsub_rn(1.0, alpha));     // :155
                            active = !(T < tf_eff);                      // :156-157
                            if (kRender) {
                                // rasterizer.py:184-191, summed in list order per pixel
                                const unsigned int g = W.gid[(head + k) & (kRing - 1)];
                                const size_t gi = W.oid[(head + k) & (kRing - 1)];  // by input id
                                const double z = depth_of_key(a.sort.keys.k64[g]);
                                r_acc = __dadd_rn(r_acc, w);
                                d_acc = __dadd_rn(d_acc, __dmul_rn(z, w));
#pragma unroll
                                for (int ch = 0; ch < 3; ++ch)
                                    if (ch < n_ch)
                                        v_acc[ch] = __dadd_rn(
                                            v_acc[ch],
                                            __dmul_rn(w, a.render.channel[gi * n_ch + ch]));
                            }
                        }
                        myval[k * kRowStride + lane] = w;
                    }
                } else {
                    // ungrouped warp (more than kMaxGroups labels, e.g. iid masks): every
                    // contributing pixel adds its own weight, issued straight from the walk
                    unsigned int mm = active ? mine : 0u;
                    while (mm) {
                        const int k = __ffs(mm) - 1;
                        mm &= mm - 1u;
                        const double alpha = myval[k * kRowStride + lane];  // 0: below floor
                        const double w = __dmul_rn(alpha, T);              // :150
                        T = __dmul_rn(T, __dsub_rn(1.0, alpha));           // :155
                        if (w > 0.0 && lbl_ok) {
                            const unsigned int row = W.oid[(head + k) & (kRing - 1)];
                            FS_CHECK(row < (unsigned)a.n_gaussians);
                            acc_add<kFixed>(acc, acc_fx, (size_t)row * n_obj + label, w);
                            ++atom;
                        }
                        if (T < tf_eff) {                                   // :156-157
                            active = false;
                            break;
                        }
                    }
                }
                __syncwarp();
                // ---- C: aggregation + float64 atomics (ungrouped warps added in B) ----
                if (kRender) {
                    // no scatter: the pixel keeps its own sums
                } else if (grouped) {
                    // lane = (splat k, segment of kMini pixels); one pass per label group
                    const int k = lane % kMini, seg = lane / kMini;
                    const unsigned int cmk = k < nm ? W.cm[(head + k) & (kRing - 1)] & act : 0u;
                    for (int gi = 0; gi < n_groups; ++gi) {
                        const unsigned int gmask = W.gmask[gi];
                        const unsigned int gl = W.glab[gi];
                        const unsigned int bits = ((cmk & gmask) >> (seg * kMini)) & ((1u << kMini) - 1u);
                        double v = 0.0;
#pragma unroll
                        for (int t = 0; t < kMini; ++t)
                            if ((bits >> t) & 1u) v += myval[k * kRowStride + seg * kMini + t];
#pragma unroll
                        for (int o = kMini; o < 32; o <<= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
                        const bool fire = lane < kMini && k < nm && v > 0.0 && gl < (unsigned)a.num_objects;
                        if (fire) {
                            const unsigned int row = W.oid[(head + k) & (kRing - 1)];
                            FS_CHECK(row < (unsigned)a.n_gaussians);
                            acc_add<kFixed>(acc, acc_fx, (size_t)row * n_obj + gl, v);
                            ++atom;
                        }
                    }
                }
                __syncwarp();
            }
            head = (head + nm) & (kRing - 1);
            cnt -= nm;
        }
    }
    if (kRender && inside) {
        // rasterizer.py:197-203 (depth = depth_acc / rho where rho > 0)
        const size_t at = (size_t)py * a.width + px;
        a.render.alpha[at] = r_acc;
        a.render.depth[at] = r_acc > 0.0 ? __ddiv_rn(d_acc, r_acc) : 0.0;
#pragma unroll
        for (int ch = 0; ch < 3; ++ch)
            if (ch < n_ch) a.render.value[at * n_ch + ch] = v_acc[ch];
    }
    // per-CTA counters: the last warp to finish issues the global atomics (no
    // end-of-tile barrier -- warps leave as soon as their strip is done)
    atom = __reduce_add_sync(0xffffffffu, (unsigned int)atom);  // per-lane counts
    if (lane == 0) {
        atomicAdd(&s_cnt[0], exact);
        atomicAdd(&s_cnt[1], atom);
        atomicMax(&s_cnt[2], steps);
        __threadfence_block();
        if (atomicAdd(&s_done, 1u) == kWarps - 1) {
            __threadfence_block();
            ViewCounters* v = a.vc;
            atomicAdd(&v->tile_steps, atomicAdd(&s_cnt[2], 0ull));
            atomicAdd(&v->exact_evals, atomicAdd(&s_cnt[0], 0ull));
            atomicAdd(&v->atomics, atomicAdd(&s_cnt[1], 0ull));
        }
    }
}

}  // namespace

// Per device (called by fs_create after cudaSetDevice).
cudaError_t raster_configure() {
    cudaError_t e = tile_sort_configure(kTileSortCap);
    if (e != cudaSuccess) return e;
    e = cudaFuncSetAttribute(raster_kernel<false, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)kRasterSmem);
    if (e != cudaSuccess) return e;
    e = cudaFuncSetAttribute(raster_kernel<false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)kRasterSmem);
    if (e != cudaSuccess) return e;
    return cudaFuncSetAttribute(raster_kernel<true, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                (int)kRasterSmem);
}

void launch_raster(const RasterArgs& a, cudaStream_t st) {
    if (a.ntiles <= 0) return;
    if (a.acc_fixed)
        raster_kernel<false, true><<<a.ntiles, kThreads, kRasterSmem, st>>>(a);
    else
        raster_kernel<false, false><<<a.ntiles, kThreads, kRasterSmem, st>>>(a);
}

void launch_raster_render(const RasterArgs& a, cudaStream_t st) {
    if (a.ntiles <= 0) return;
    raster_kernel<true, false><<<a.ntiles, kThreads, kRasterSmem, st>>>(a);
}

}  // namespace fs
