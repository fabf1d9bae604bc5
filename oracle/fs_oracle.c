/*
 * fs_oracle.c -- CPU restatement of the FlashSplat label-solver hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  Nothing in the product package
 * (paper_2409_08270_b200/) may link, load or call this file; it is used by
 * tests/, by __graft_entry__.smoke() as the checker, and by bench.py's
 * cpu_baseline / --impl reference leg.  The product path is the CUDA library.
 *
 * Parity status: PINNED.  tests/test_oracle_golden.py checks every function
 * below against golden vectors produced by the reference package itself
 * (tests/golden/make_golden.py imports /root/reference/pkg/src/splatlift).
 *
 * Everything is float64 and evaluated in the same operation order as the
 * numpy expressions it restates (compiled with -ffp-contract=off, no
 * -ffast-math), so per-entry results agree with the reference to the last
 * few ulps; the remaining differences come from BLAS summation order in the
 * reference's 3x3 matmuls and from libm exp() vs numpy exp().
 *
 * Reference functions restated (paths relative to /root/reference/pkg/src/splatlift):
 *   quaternion_to_rotation  scene.py:228-242
 *   covariance_3d           scene.py:245-249
 *   _project_arrays         scene.py:252-312
 *   TileBinning.__init__    rasterizer.py:72-100   (order = lexsort((index, depth)))
 *   tile_range              rasterizer.py:106-113
 *   _tile_pixel_grid        rasterizer.py:123-130
 *   _accumulate_view        contributions.py:119-160
 *   accumulate_contributions contributions.py:90-116 (f64 partials summed in view order)
 *   render_property          rasterizer.py:133-203 (per-pixel compositing of a binning)
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define ORC_TILE 16
#define ORC_COV2D_DILATION 0.3 /* scene.py:25 */
#define ORC_ALPHA_CLAMP 0.99   /* scene.py:26 */
#define ORC_DEGENERATE_DET 1e-12 /* scene.py:27 */

typedef struct {
    int32_t width, height;
    double fx, fy, cx, cy;
    double w2c[16]; /* row-major world_to_camera */
    double near_clip;
} orc_camera;

/* scene.py:228-242 (w, x, y, z), quaternion assumed normalised (scene.py:99-103). */
static void quat_rot(const double *q, double r[9]) {
    double w = q[0], x = q[1], y = q[2], z = q[3];
    r[0] = 1.0 - 2.0 * (y * y + z * z);
    r[1] = 2.0 * (x * y - w * z);
    r[2] = 2.0 * (x * z + w * y);
    r[3] = 2.0 * (x * y + w * z);
    r[4] = 1.0 - 2.0 * (x * x + z * z);
    r[5] = 2.0 * (y * z - w * x);
    r[6] = 2.0 * (x * z - w * y);
    r[7] = 2.0 * (y * z + w * x);
    r[8] = 1.0 - 2.0 * (x * x + y * y);
}

/* covariance_3d, scene.py:245-249: m = R * s (column scale), Sigma = m m^T. */
static void cov3d(const double *q, const double *s, double sig[9]) {
    double r[9], m[9];
    quat_rot(q, r);
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) m[3 * i + j] = r[3 * i + j] * s[j];
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j)
            sig[3 * i + j] = m[3 * i + 0] * m[3 * j + 0] + m[3 * i + 1] * m[3 * j + 1] +
                             m[3 * i + 2] * m[3 * j + 2];
}

static void mat3_mul(const double *a, const double *b, double *out) {
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j)
            out[3 * i + j] = a[3 * i + 0] * b[0 + j] + a[3 * i + 1] * b[3 + j] + a[3 * i + 2] * b[6 + j];
}

/*
 * _project_arrays, scene.py:252-312.  Outputs are indexed by Gaussian.
 * stats: [n_input, n_emitted, n_behind, n_degenerate, n_offscreen] (scene.py:217-225).
 */
void orc_project(int64_t n, const double *means, const double *quats, const double *scales,
                 const orc_camera *cam, uint8_t *alive_out, double *mean2d, double *conic,
                 double *depth, int64_t *radius, int64_t *stats) {
    const double *W = cam->w2c;
    double rot[9] = {W[0], W[1], W[2], W[4], W[5], W[6], W[8], W[9], W[10]};
    double rotT[9] = {W[0], W[4], W[8], W[1], W[5], W[9], W[2], W[6], W[10]};
    double t[3] = {W[3], W[7], W[11]};
    int64_t n_behind = 0, n_deg = 0, n_off = 0, n_emit = 0;
    for (int64_t i = 0; i < n; ++i) {
        const double *m = means + 3 * i;
        double cam3[3];
        for (int r = 0; r < 3; ++r)
            cam3[r] = (m[0] * rot[3 * r + 0] + m[1] * rot[3 * r + 1] + m[2] * rot[3 * r + 2]) + t[r];
        double x = cam3[0], y = cam3[1], z = cam3[2];
        int alive = z > cam->near_clip; /* :268 */
        if (!alive) ++n_behind;
        double zs = alive ? z : 1.0; /* :272 */
        double mx = cam->fx * x / zs + cam->cx;
        double my = cam->fy * y / zs + cam->cy;
        double sig[9], tmp[9], sc[9];
        cov3d(quats + 4 * i, scales + 3 * i, sig);
        mat3_mul(rot, sig, tmp); /* rot @ sigma @ rot.T, :278 */
        mat3_mul(tmp, rotT, sc);
        double j00 = cam->fx / zs, j02 = -cam->fx * x / (zs * zs);
        double j11 = cam->fy / zs, j12 = -cam->fy * y / (zs * zs);
        /* cov2d = J Sc J^T with J = [[j00,0,j02],[0,j11,j12]], :280-285 */
        double js0[3], js1[3];
        for (int c = 0; c < 3; ++c) {
            js0[c] = j00 * sc[0 + c] + 0.0 * sc[3 + c] + j02 * sc[6 + c];
            js1[c] = 0.0 * sc[0 + c] + j11 * sc[3 + c] + j12 * sc[6 + c];
        }
        double c00 = js0[0] * j00 + js0[1] * 0.0 + js0[2] * j02;
        double c01 = js0[0] * 0.0 + js0[1] * j11 + js0[2] * j12;
        double c11 = js1[0] * 0.0 + js1[1] * j11 + js1[2] * j12;
        double a = c00 + ORC_COV2D_DILATION, b = c01, c = c11 + ORC_COV2D_DILATION;
        double det = a * c - b * b; /* :290 */
        if (alive && det <= ORC_DEGENERATE_DET) {
            ++n_deg;
            alive = 0;
        }
        double ds = det > ORC_DEGENERATE_DET ? det : 1.0;
        double mid = 0.5 * (a + c);
        double disc = sqrt(fmax(0.25 * ((a - c) * (a - c)) + b * b, 0.0));
        double lam = fmax(mid + disc, 0.0);
        double rad = ceil(3.0 * sqrt(lam)); /* :301 */
        if (alive && ((mx + rad < 0.0) || (mx - rad > (double)cam->width) || (my + rad < 0.0) ||
                      (my - rad > (double)cam->height))) {
            ++n_off;
            alive = 0;
        }
        if (alive) ++n_emit;
        alive_out[i] = (uint8_t)alive;
        mean2d[2 * i] = mx;
        mean2d[2 * i + 1] = my;
        conic[3 * i] = c / ds;
        conic[3 * i + 1] = -b / ds;
        conic[3 * i + 2] = a / ds;
        depth[i] = z;
        radius[i] = (int64_t)rad;
    }
    if (stats) {
        stats[0] = n;
        stats[1] = n_emit;
        stats[2] = n_behind;
        stats[3] = n_deg;
        stats[4] = n_off;
    }
}

/* tile_range, rasterizer.py:106-113 (inclusive floor box, may be empty). */
static void tile_range(double mx, double my, int64_t r, int tx_n, int ty_n, int *tx0, int *tx1,
                       int *ty0, int *ty1) {
    double rr = (double)r;
    double a = floor((mx - rr) / ORC_TILE), b = floor((mx + rr) / ORC_TILE);
    double c = floor((my - rr) / ORC_TILE), d = floor((my + rr) / ORC_TILE);
    /* clamp before the int conversion so far-off splats stay well defined */
    *tx0 = a < 0.0 ? 0 : (a > (double)tx_n ? tx_n : (int)a);
    *tx1 = b > (double)(tx_n - 1) ? tx_n - 1 : (b < -1.0 ? -1 : (int)b);
    *ty0 = c < 0.0 ? 0 : (c > (double)ty_n ? ty_n : (int)c);
    *ty1 = d > (double)(ty_n - 1) ? ty_n - 1 : (d < -1.0 ? -1 : (int)d);
}

typedef struct {
    double depth;
    int64_t idx;
} dkey;

static int dkey_cmp(const void *pa, const void *pb) {
    const dkey *a = (const dkey *)pa, *b = (const dkey *)pb;
    if (a->depth < b->depth) return -1;
    if (a->depth > b->depth) return 1;
    return (a->idx > b->idx) - (a->idx < b->idx);
}

/*
 * TileBinning.__init__, rasterizer.py:72-100.  Fills tile_offsets[ntiles+1]
 * (CSR) and, when items != NULL, the per-tile Gaussian indices ordered by
 * (depth, index).  Returns the total instance count.
 */
int64_t orc_bin(int64_t n, const uint8_t *alive, const double *mean2d, const double *depth,
                const int64_t *radius, int width, int height, int64_t *tile_offsets, int64_t *items) {
    int tx_n = (width + ORC_TILE - 1) / ORC_TILE, ty_n = (height + ORC_TILE - 1) / ORC_TILE;
    int64_t ntiles = (int64_t)tx_n * ty_n;
    int64_t k = 0;
    for (int64_t i = 0; i < n; ++i) k += alive[i] ? 1 : 0;
    dkey *order = (dkey *)malloc(sizeof(dkey) * (size_t)(k > 0 ? k : 1));
    k = 0;
    for (int64_t i = 0; i < n; ++i)
        if (alive[i]) {
            order[k].depth = depth[i];
            order[k].idx = i;
            ++k;
        }
    qsort(order, (size_t)k, sizeof(dkey), dkey_cmp);
    memset(tile_offsets, 0, sizeof(int64_t) * (size_t)(ntiles + 1));
    for (int64_t s = 0; s < k; ++s) {
        int64_t i = order[s].idx;
        int tx0, tx1, ty0, ty1;
        tile_range(mean2d[2 * i], mean2d[2 * i + 1], radius[i], tx_n, ty_n, &tx0, &tx1, &ty0, &ty1);
        for (int ty = ty0; ty <= ty1; ++ty)
            for (int tx = tx0; tx <= tx1; ++tx) tile_offsets[(int64_t)ty * tx_n + tx + 1] += 1;
    }
    for (int64_t t = 0; t < ntiles; ++t) tile_offsets[t + 1] += tile_offsets[t];
    int64_t total = tile_offsets[ntiles];
    if (items) {
        int64_t *cursor = (int64_t *)malloc(sizeof(int64_t) * (size_t)(ntiles > 0 ? ntiles : 1));
        memcpy(cursor, tile_offsets, sizeof(int64_t) * (size_t)ntiles);
        for (int64_t s = 0; s < k; ++s) {
            int64_t i = order[s].idx;
            int tx0, tx1, ty0, ty1;
            tile_range(mean2d[2 * i], mean2d[2 * i + 1], radius[i], tx_n, ty_n, &tx0, &tx1, &ty0, &ty1);
            for (int ty = ty0; ty <= ty1; ++ty)
                for (int tx = tx0; tx <= tx1; ++tx) items[cursor[(int64_t)ty * tx_n + tx]++] = i;
        }
        free(cursor);
    }
    free(order);
    return total;
}

/* Walk counters for the roofline accounting: per view. */
typedef struct {
    int64_t tile_steps;       /* list entries walked (all pixels of a tile move together) */
    int64_t lockstep_evals;   /* tile_steps x tile pixel count */
    int64_t active_evals;     /* evaluations on still-active pixels */
    int64_t contrib_pairs;    /* (pixel, gaussian) pairs with weight > 0 */
    int64_t instances;        /* binning instances */
} orc_walk_stats;

typedef struct {
    int64_t n;
    const double *means, *quats, *scales, *opac;
} orc_scene;

/*
 * _accumulate_view, contributions.py:119-160.  Adds this view's weights into
 * part (E x N row-major f64), which the caller zeroes.  touched (N bytes,
 * optional) marks columns that received a bincount.  Summation order follows
 * the reference: per (tile, splat) a bincount over the tile's pixels in
 * raster order, then part[:, gid] += bins, tiles row-major.
 */
static int accumulate_view_impl(const orc_scene *sc, const orc_camera *cam, const uint16_t *mask,
                                int E, double alpha_floor, double t_floor, double *part,
                                uint8_t *touched, orc_walk_stats *ws) {
    int64_t n = sc->n;
    uint8_t *alive = (uint8_t *)malloc((size_t)(n > 0 ? n : 1));
    double *mean2d = (double *)malloc(sizeof(double) * 2 * (size_t)(n > 0 ? n : 1));
    double *conic = (double *)malloc(sizeof(double) * 3 * (size_t)(n > 0 ? n : 1));
    double *depth = (double *)malloc(sizeof(double) * (size_t)(n > 0 ? n : 1));
    int64_t *radius = (int64_t *)malloc(sizeof(int64_t) * (size_t)(n > 0 ? n : 1));
    orc_project(n, sc->means, sc->quats, sc->scales, cam, alive, mean2d, conic, depth, radius, NULL);
    int W = cam->width, H = cam->height;
    int tx_n = (W + ORC_TILE - 1) / ORC_TILE, ty_n = (H + ORC_TILE - 1) / ORC_TILE;
    int64_t ntiles = (int64_t)tx_n * ty_n;
    int64_t *offs = (int64_t *)malloc(sizeof(int64_t) * (size_t)(ntiles + 1));
    int64_t total = orc_bin(n, alive, mean2d, depth, radius, W, H, offs, NULL);
    int64_t *items = (int64_t *)malloc(sizeof(int64_t) * (size_t)(total > 0 ? total : 1));
    orc_bin(n, alive, mean2d, depth, radius, W, H, offs, items);
    if (ws) ws->instances += total;

    double *bins = (double *)calloc((size_t)E, sizeof(double));
    int *bin_used = (int *)malloc(sizeof(int) * (size_t)E);
    double trans[ORC_TILE * ORC_TILE];
    uint8_t act[ORC_TILE * ORC_TILE];
    int lab[ORC_TILE * ORC_TILE];

    for (int ty = 0; ty < ty_n; ++ty) {
        for (int tx = 0; tx < tx_n; ++tx) {
            int64_t t = (int64_t)ty * tx_n + tx;
            int64_t beg = offs[t], end = offs[t + 1];
            if (beg == end) continue;
            int x0 = tx * ORC_TILE, y0 = ty * ORC_TILE;
            int x1 = x0 + ORC_TILE < W ? x0 + ORC_TILE : W;
            int y1 = y0 + ORC_TILE < H ? y0 + ORC_TILE : H;
            int tw = x1 - x0, th = y1 - y0, np_ = tw * th;
            for (int p = 0; p < np_; ++p) {
                trans[p] = 1.0;
                act[p] = 1;
                lab[p] = mask[(int64_t)(y0 + p / tw) * W + x0 + p % tw];
            }
            int n_active = np_;
            for (int64_t s = beg; s < end; ++s) {
                int64_t g = items[s];
                double mx = mean2d[2 * g], my = mean2d[2 * g + 1];
                double a = conic[3 * g], b = conic[3 * g + 1], c = conic[3 * g + 2];
                double o = sc->opac[g];
                int nused = 0, any = 0;
                if (ws) {
                    ws->tile_steps += 1;
                    ws->lockstep_evals += np_;
                    ws->active_evals += n_active;
                }
                for (int p = 0; p < np_; ++p) {
                    if (!act[p]) continue; /* use == False: weight 0, no update */
                    double du = ((double)(x0 + p % tw) + 0.5) - mx;
                    double dv = ((double)(y0 + p / tw) + 0.5) - my;
                    double power = -0.5 * (a * du * du + c * dv * dv) - b * du * dv; /* :145 */
                    double alpha = o * exp(power);
                    if (alpha > ORC_ALPHA_CLAMP) alpha = ORC_ALPHA_CLAMP; /* :146-147 */
                    if (alpha_floor > 0.0 && !(alpha >= alpha_floor)) continue; /* :148-149 */
                    double w = alpha * trans[p];                                 /* :150 */
                    int l = lab[p];
                    if (bins[l] == 0.0 && w > 0.0) bin_used[nused++] = l;
                    bins[l] += w;
                    if (w > 0.0) {
                        any = 1;
                        if (ws) ws->contrib_pairs += 1;
                    }
                    trans[p] = trans[p] * (1.0 - alpha); /* :155 */
                    if (t_floor > 0.0 && !(trans[p] >= t_floor)) {
                        act[p] = 0; /* :156-157 */
                        --n_active;
                    }
                }
                if (any) {
                    for (int u = 0; u < nused; ++u) {
                        int l = bin_used[u];
                        part[(int64_t)l * n + g] += bins[l];
                        bins[l] = 0.0;
                    }
                    if (touched) touched[g] = 1;
                } else {
                    for (int u = 0; u < nused; ++u) bins[bin_used[u]] = 0.0;
                }
                if (t_floor > 0.0 && n_active == 0) break; /* :158-159 */
            }
        }
    }
    free(bins);
    free(bin_used);
    free(items);
    free(offs);
    free(alive);
    free(mean2d);
    free(conic);
    free(depth);
    free(radius);
    return 0;
}

/* Single-view partial (E x N f64, zeroed by this call). */
int orc_accumulate_view(int64_t n, const double *means, const double *quats, const double *scales,
                        const double *opac, const orc_camera *cam, const uint16_t *mask, int E,
                        double alpha_floor, double t_floor, double *part, int64_t *walk_stats) {
    orc_scene sc = {n, means, quats, scales, opac};
    memset(part, 0, sizeof(double) * (size_t)E * (size_t)n);
    orc_walk_stats ws;
    memset(&ws, 0, sizeof(ws));
    int rc = accumulate_view_impl(&sc, cam, mask, E, alpha_floor, t_floor, part, NULL, &ws);
    if (walk_stats) {
        walk_stats[0] = ws.tile_steps;
        walk_stats[1] = ws.lockstep_evals;
        walk_stats[2] = ws.active_evals;
        walk_stats[3] = ws.contrib_pairs;
        walk_stats[4] = ws.instances;
    }
    return rc;
}

/* ---- accumulate_contributions (contributions.py:90-116), view-parallel ---- */

typedef struct {
    const orc_scene *sc;
    const orc_camera *cams;
    const uint16_t *const *masks;
    int n_views, E;
    double alpha_floor, t_floor;
    double *total; /* E x N f64 */
    int next_view; /* work counter */
    int merge_turn; /* next view index allowed to merge */
    pthread_mutex_t mu;
    pthread_cond_t cv;
} orc_job;

static void *worker(void *arg) {
    orc_job *job = (orc_job *)arg;
    int64_t n = job->sc->n;
    int E = job->E;
    size_t cells = (size_t)E * (size_t)n;
    double *part = (double *)calloc(cells > 0 ? cells : 1, sizeof(double));
    uint8_t *touched = (uint8_t *)calloc((size_t)(n > 0 ? n : 1), 1);
    for (;;) {
        pthread_mutex_lock(&job->mu);
        int v = job->next_view++;
        pthread_mutex_unlock(&job->mu);
        if (v >= job->n_views) break;
        accumulate_view_impl(job->sc, &job->cams[v], job->masks[v], E, job->alpha_floor,
                             job->t_floor, part, touched, NULL);
        /* total += part in view order (contributions.py:115). */
        pthread_mutex_lock(&job->mu);
        while (job->merge_turn != v) pthread_cond_wait(&job->cv, &job->mu);
        pthread_mutex_unlock(&job->mu);
        for (int64_t g = 0; g < n; ++g) {
            if (!touched[g]) continue;
            for (int e = 0; e < E; ++e) {
                size_t at = (size_t)e * (size_t)n + (size_t)g;
                job->total[at] += part[at];
                part[at] = 0.0;
            }
            touched[g] = 0;
        }
        pthread_mutex_lock(&job->mu);
        job->merge_turn = v + 1;
        pthread_cond_broadcast(&job->cv);
        pthread_mutex_unlock(&job->mu);
    }
    free(part);
    free(touched);
    return NULL;
}

/*
 * accumulate_contributions: total_f64 (E x N, zeroed by this call) receives the
 * f64 sum in view order; the caller casts to float32 as contributions.py:116.
 * n_threads <= 0 uses one thread.  Each thread holds one E x N f64 partial.
 */
int orc_accumulate(int64_t n, const double *means, const double *quats, const double *scales,
                   const double *opac, int n_views, const orc_camera *cams,
                   const uint16_t *const *masks, int E, double alpha_floor, double t_floor,
                   int n_threads, double *total) {
    orc_scene sc = {n, means, quats, scales, opac};
    memset(total, 0, sizeof(double) * (size_t)E * (size_t)n);
    if (n_threads < 1) n_threads = 1;
    if (n_threads > n_views) n_threads = n_views > 0 ? n_views : 1;
    orc_job job;
    job.sc = &sc;
    job.cams = cams;
    job.masks = masks;
    job.n_views = n_views;
    job.E = E;
    job.alpha_floor = alpha_floor;
    job.t_floor = t_floor;
    job.total = total;
    job.next_view = 0;
    job.merge_turn = 0;
    pthread_mutex_init(&job.mu, NULL);
    pthread_cond_init(&job.cv, NULL);
    pthread_t *th = (pthread_t *)malloc(sizeof(pthread_t) * (size_t)n_threads);
    for (int i = 0; i < n_threads; ++i) pthread_create(&th[i], NULL, worker, &job);
    for (int i = 0; i < n_threads; ++i) pthread_join(th[i], NULL);
    free(th);
    pthread_mutex_destroy(&job.mu);
    pthread_cond_destroy(&job.cv);
    return 0;
}

/* ---- render_property (rasterizer.py:133-203) ----
 * Splat arrays are indexed by the CSR items (positions into them); opac and
 * channel are per splat (the caller gathers scene.opacities[indices] and
 * channel[indices]).  channels: 0 (no value), 1 (scalar) or 3 (vector).
 * value (H*W*channels), rho and depth_out (H*W) are overwritten.  Per pixel,
 * every sum runs in list order exactly as the numpy tile arrays accumulate. */
int orc_render(int64_t k, const double *mean2d, const double *conic, const double *depth,
               const double *opac, const double *channel, int channels, int W, int H,
               const int64_t *offs, const int64_t *items, double alpha_floor, double t_floor,
               double *value, double *rho, double *depth_out) {
    (void)k;
    const size_t px = (size_t)W * (size_t)H;
    memset(rho, 0, sizeof(double) * px);
    memset(depth_out, 0, sizeof(double) * px);
    if (channels > 0) memset(value, 0, sizeof(double) * px * (size_t)channels);
    int tx_n = (W + ORC_TILE - 1) / ORC_TILE, ty_n = (H + ORC_TILE - 1) / ORC_TILE;
    double trans[ORC_TILE * ORC_TILE], racc[ORC_TILE * ORC_TILE], dacc[ORC_TILE * ORC_TILE];
    double vacc[ORC_TILE * ORC_TILE * 3];
    uint8_t act[ORC_TILE * ORC_TILE];
    for (int ty = 0; ty < ty_n; ++ty) {
        for (int tx = 0; tx < tx_n; ++tx) {
            int64_t t = (int64_t)ty * tx_n + tx;
            int64_t beg = offs[t], end = offs[t + 1];
            if (beg == end) continue; /* :163-164 */
            int x0 = tx * ORC_TILE, y0 = ty * ORC_TILE;
            int x1 = x0 + ORC_TILE < W ? x0 + ORC_TILE : W;
            int y1 = y0 + ORC_TILE < H ? y0 + ORC_TILE : H;
            int tw = x1 - x0, th = y1 - y0, np_ = tw * th;
            for (int p = 0; p < np_; ++p) {
                trans[p] = 1.0;
                act[p] = 1;
                racc[p] = 0.0;
                dacc[p] = 0.0;
                for (int c = 0; c < channels; ++c) vacc[p * 3 + c] = 0.0;
            }
            int n_active = np_;
            for (int64_t s = beg; s < end; ++s) {
                int64_t g = items[s];
                double mx = mean2d[2 * g], my = mean2d[2 * g + 1];
                double a = conic[3 * g], b = conic[3 * g + 1], c = conic[3 * g + 2];
                double o = opac[g], z = depth[g];
                for (int p = 0; p < np_; ++p) {
                    if (!act[p]) continue; /* use == False: weight 0 (adds nothing) */
                    double du = ((double)(x0 + p % tw) + 0.5) - mx;
                    double dv = ((double)(y0 + p / tw) + 0.5) - my;
                    double power = -0.5 * (a * du * du + c * dv * dv) - b * du * dv; /* :178 */
                    double alpha = o * exp(power);
                    if (alpha > ORC_ALPHA_CLAMP) alpha = ORC_ALPHA_CLAMP; /* :179-180 */
                    if (alpha_floor > 0.0 && !(alpha >= alpha_floor)) continue; /* :181-182 */
                    double w = alpha * trans[p];                                 /* :183 */
                    for (int ch = 0; ch < channels; ++ch)                        /* :184-189 */
                        vacc[p * 3 + ch] += w * channel[(size_t)g * channels + ch];
                    racc[p] += w;                                                /* :190 */
                    dacc[p] += z * w;                                            /* :191 */
                    trans[p] = trans[p] * (1.0 - alpha);                         /* :192 */
                    if (t_floor > 0.0 && !(trans[p] >= t_floor)) {               /* :193-194 */
                        act[p] = 0;
                        --n_active;
                    }
                }
                if (t_floor > 0.0 && n_active == 0) break; /* :195-196 */
            }
            for (int p = 0; p < np_; ++p) {
                size_t at = (size_t)(y0 + p / tw) * (size_t)W + (size_t)(x0 + p % tw);
                rho[at] = racc[p];
                depth_out[at] = racc[p] > 0.0 ? dacc[p] / racc[p] : 0.0; /* :202-203 */
                for (int ch = 0; ch < channels; ++ch) value[at * channels + ch] = vacc[p * 3 + ch];
            }
        }
    }
    return 0;
}
