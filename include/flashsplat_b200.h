/*
 * flashsplat_b200.h -- C ABI of the B200-native FlashSplat label solver.
 *
 * Plain C types only (no torch, no C++).  Every entry point replaces one
 * function of the reference package's Python hot path (paths relative to
 * /root/reference/pkg/src/splatlift); the Python mirror in
 * paper_2409_08270_b200/ keeps the reference signatures and calls these
 * through ctypes (see INTEGRATION.md for the bindings).
 *
 * Conventions
 *   - return value: FS_OK (0) or an FS_E* code; fs_last_error() returns a
 *     thread-local message for the last failing call on this thread;
 *   - float64 host arrays are C-contiguous numpy layouts (N x 3 means,
 *     N x 4 unit quaternions (w, x, y, z), N x 3 scales, N opacities);
 *   - float32 matrices are E x N row-major (ContributionMatrix.values layout,
 *     contributions.py:52-55); the accumulator of fs_accumulate is N x E
 *     (Gaussian-major; FS_ACC_FIXED or FS_ACC_F64 entries) and the finalize
 *     entry points convert between the two;
 *   - no entry point synchronises the whole device: work is ordered after the
 *     caller's stream (fs_set_stream) and complete when the call returns;
 *   - "device" pointers are CUDA device addresses on the context's device.
 */
#ifndef FLASHSPLAT_B200_H
#define FLASHSPLAT_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define FS_OK 0
#define FS_EINVAL 1   /* invalid argument (ValueError on the Python side) */
#define FS_ECUDA 2    /* CUDA runtime failure (RuntimeError) */
#define FS_ENOMEM 3   /* device or pinned allocation failed */
#define FS_ELABEL 4   /* a mask label >= num_objects (see stats->label_error_view) */

#define FS_MODE_BINARY 0
#define FS_MODE_SCENE 1

/* Accumulator kinds (N x E, Gaussian-major, device memory, caller-zeroed).
 * FS_ACC_F64:   one float64 per entry; float64 atomics, so the low bits of
 *               an entry depend on the order the adds land in.
 * FS_ACC_FIXED: two uint64 words per entry, (hi, lo) = (sum q >> 32,
 *               sum q & 0xffffffff) for q = round(w * 2^59) per add; the
 *               value is (hi * 2^32 + lo) * 2^-59.  Integer adds commute, so
 *               the result is bit-identical for any schedule, stream count or
 *               split of the views over GPUs (
 *               test_contributions.py:160-168).  16 B per entry. */
#define FS_ACC_F64 0
#define FS_ACC_FIXED 1

typedef struct fs_context fs_context;

/* Pinhole view, scene.py:164-203 (CameraView). */
typedef struct {
    int32_t width, height;
    double fx, fy, cx, cy;
    double world_to_camera[16]; /* row-major 4x4 */
    double near_clip;
} fs_camera;

/* Cull counters, scene.py:217-225 (ProjectionStats). */
typedef struct {
    int64_t n_input, n_emitted, n_behind, n_degenerate, n_offscreen;
} fs_projection_stats;

/* Totals of one fs_accumulate call (summed over views). */
typedef struct {
    int64_t views;
    int64_t view_pixels;
    int64_t emitted;          /* visible (view, gaussian) pairs */
    int64_t instances;        /* (view, tile, gaussian) binning instances */
    int64_t tile_steps;       /* list entries walked by the raster kernel */
    int64_t exact_evals;      /* float64 alpha evaluations */
    int64_t atomics;          /* accumulator adds (one RED, or two uint64 REDs for FS_ACC_FIXED) */
    int64_t retried_views;    /* views re-run after growing the instance buffers */
    int64_t launches;         /* kernels this call launched */
    int64_t label_error_view; /* first view with a label >= num_objects, or -1 */
    double gpu_ms;            /* CUDA-event time of the view loop on the device */
    /* per-stage CUDA-event times summed over views; only with fs_set_timing(ctx, 1) */
    double prep_ms;           /* projection */
    double bin_ms;            /* tile histograms, bucket offsets, instance emission */
    double raster_ms;         /* raster kernel (in-kernel bucket sort + walk + atomics) */
} fs_accumulate_stats;

const char *fs_last_error(void);
const char *fs_version(void);

/* Context = one CUDA device + streams + workspaces.  Not thread-safe: one
 * host thread per context (fs_assign is the reentrant exception). */
int fs_create(int device, int n_streams, fs_context **out);
void fs_destroy(fs_context *ctx);
int fs_device_count(int *out);

/* Device memory helpers for callers without their own allocator. */
int fs_device_alloc(fs_context *ctx, uint64_t bytes, void **out);
int fs_device_free(fs_context *ctx, void *ptr);
int fs_memset_zero(fs_context *ctx, void *dev_ptr, uint64_t bytes);
int fs_copy_to_device(fs_context *ctx, void *dst, const void *src, uint64_t bytes);
int fs_copy_to_host(fs_context *ctx, void *dst, const void *src, uint64_t bytes);
int fs_synchronize(fs_context *ctx);

/* Stream the context's entry points order themselves after (an event recorded
 * on it at entry; default NULL = the legacy default stream, which also covers
 * torch's default stream).  No entry point synchronises the whole device. */
int fs_set_stream(fs_context *ctx, void *stream);

/* Page-locked host memory (DMA at full PCIe/C2C speed) for result arrays the
 * caller hands back to numpy -- the contribution matrix and the labels. */
int fs_host_alloc(fs_context *ctx, uint64_t bytes, void **out);
int fs_host_free(fs_context *ctx, void *ptr);
/* 1 if [ptr, ptr + bytes) is page-locked host memory (fs_host_alloc or
 * cudaHostRegister): fs_set_scene and fs_accumulate DMA such inputs directly
 * instead of staging them through the library's pinned buffers. */
int fs_host_pinned(const void *ptr, uint64_t bytes);

/* Per-stage CUDA-event timing inside fs_accumulate (events on each view's
 * stream around its stages; adds ~3 event records per view). */
int fs_set_timing(fs_context *ctx, int enable);

/* Upload a GaussianScene (scene.py:71-110, arrays already validated and the
 * quaternions normalised).  Replaces the per-view f64 input handling of
 * _project_arrays (scene.py:252-278).  The resident copy is stored in spatial
 * (Morton) order for locality; every output of every entry point -- tile
 * lists, exports, accumulator rows, labels -- stays indexed by the caller's
 * Gaussian index (set FS_SCENE_ORDER=0 in the environment to keep input order). */
int fs_set_scene(fs_context *ctx, int64_t n, const double *means, const double *quats,
                 const double *scales, const double *opacities);

/* The resident scene of src (set by fs_set_scene / fs_set_scene_ply) copied
 * into dst device to device -- over NVLink when they sit on different GPUs --
 * so a multi-GPU solve reads the host scene once instead of once per GPU. */
int fs_copy_scene(fs_context *dst, const fs_context *src);

/* load_scene_ply (ply.py:63-106) + GaussianScene (scene.py:71-110) on the
 * device: verts is the checkpoint's binary_little_endian
 * vertex block as stored in the file -- n records of stride_floats float32 --
 * and offsets[17] the float offsets of x y z nx ny nz f_dc_0..2 opacity
 * scale_0..2 rot_0..3 (the reference's REQUIRED_PROPERTIES order, ply.py:17-23)
 * within a record.  One upload, then one kernel applies the activations
 * (exp scales, logistic opacity, quaternion normalisation) and builds the
 * resident scene.  bad[4] receives the first vertex with a non-finite required
 * value, a zero quaternion norm, a non-positive scale and an opacity outside
 * [0, 1] (-1: none); FS_EINVAL if any (the scene is then not resident).
 * params (optional, n x 8 float64 host) receives the activated parameters
 * (scale_0..2, opacity, normalised w x y z) for verification. */
int fs_set_scene_ply(fs_context *ctx, int64_t n, const void *verts, int stride_floats,
                     const int32_t *offsets, int64_t *bad, double *params);

/* _project_arrays (scene.py:252-312) over the resident scene; host outputs
 * indexed by Gaussian (any may be NULL except alive). */
int fs_project(fs_context *ctx, const fs_camera *cam, uint8_t *alive, double *mean2d,
               double *conic, double *depth, int64_t *radius, fs_projection_stats *stats);

/* TileBinning.__init__ (rasterizer.py:72-100): tile_offsets[ntiles + 1] CSR
 * offsets and items[] Gaussian ids, each tile ordered by (depth, id).
 * items may be NULL to query *n_items. */
int fs_bin(fs_context *ctx, const fs_camera *cam, int64_t *tile_offsets, int64_t *items,
           int64_t items_capacity, int64_t *n_items);

/* TileBinning(view, projected) for an explicit splat list (rasterizer.py:72-100,
 * e.g. hand-built ProjectedGaussian lists): k splats with mean2d (k x 2),
 * depth, radius and gaussian index; items[] are positions in the list,
 * ordered per tile by (depth, gaussian index) like np.lexsort((indices, depths)). */
int fs_bin_splats(fs_context *ctx, int64_t k, const double *mean2d, const double *depth,
                  const int64_t *radius, const int64_t *index, int width, int height,
                  int64_t *tile_offsets, int64_t *items, int64_t items_capacity,
                  int64_t *n_items);

/* accumulate_contributions (contributions.py:90-116) / _accumulate_view
 * (contributions.py:119-160) for n_views views: adds every view's alpha*T
 * mass into acc (N x E, Gaussian-major so one splat's labels share cache
 * lines, of acc_kind, DEVICE pointer, caller-zeroed).  masks[v] is an H x W
 * uint16 label grid, host or device (masks_on_device).  A label >= num_objects
 * returns FS_ELABEL with stats->label_error_view = the first such view
 * (contributions.py:108-114). */
int fs_accumulate(fs_context *ctx, int n_views, const fs_camera *cams,
                  const uint16_t *const *masks, int masks_on_device, int num_objects,
                  double alpha_floor, double transmittance_floor, int acc_kind, void *acc,
                  fs_accumulate_stats *stats);

/* The same over several contexts (one per GPU, the same scene uploaded to
 * each) from ONE process: one host thread per context pops views from a
 * shared queue whenever one of its streams frees up (dynamic load balance;
 * contributions.py:103-116 -- A is additive over views) and accumulates into
 * accs[i] on context i's device.  Host masks only.  view_ctx (optional,
 * n_views) receives the context that ran each view.  With FS_ACC_FIXED the
 * summed result does not depend on which GPU ran which view. */
int fs_accumulate_multi(fs_context *const *ctxs, int n_ctx, int n_views, const fs_camera *cams,
                        const uint16_t *const *masks, int num_objects, double alpha_floor,
                        double transmittance_floor, int acc_kind, void *const *accs,
                        int32_t *view_ctx, fs_accumulate_stats *stats);

/* ContributionMatrix(total.astype(float32)) (contributions.py:116): the N x E
 * device accumulator -> E x N float32 (the reference's layout), written to
 * host (out_on_device = 0) or device memory. */
int fs_finalize(fs_context *ctx, int acc_kind, const void *acc, int64_t n, int num_objects,
                float *out, int out_on_device);

/* Reduce + cast of the Gaussian slice [g0, g1): the sum of n_parts N x E
 * accumulators (device pointers -- other GPUs' through peer memory, see
 * fs_enable_peer_access; part rows start at Gaussian part_g0, e.g. the output
 * of a reduce-scatter) -> float32 E x (g1 - g0) at out with row stride ld
 * (out = element (0, g0) of the caller's matrix; host or device). */
int fs_reduce_finalize(fs_context *ctx, int acc_kind, const void *const *parts, int n_parts,
                       int64_t part_g0, int64_t n, int num_objects, int64_t g0, int64_t g1,
                       float *out, int64_t ld, int out_on_device);

/* Peer access from ctx's device to peer_device (NVLink P2P loads). */
int fs_enable_peer_access(fs_context *ctx, int peer_device);

/* After fs_accumulate_multi: context i reduces column slice i of A over all
 * contexts' accumulators (peer-memory loads -- the reduce half of a
 * reduce-scatter fused into the cast; staged copies when P2P is unavailable),
 * casts it, runs the biased argmax on it (mode FS_MODE_BINARY / FS_MODE_SCENE,
 * or -1 for none; solver.py:118-172) and copies both straight into the host
 * outputs: out E x N float32, labels N (binary) or E x N (scene) uint8. */
int fs_finalize_multi(fs_context *const *ctxs, int n_ctx, int acc_kind, void *const *accs,
                      int64_t n, int num_objects, float *out, float gamma, int mode,
                      uint8_t *labels);

/* _one_vs_rest_wins + assign_binary / assign_scene (solver.py:118-172).
 * A is E x N float32; out is N (binary) or E x N (scene) uint8.  Host or
 * device pointers (on_device).  Reentrant: runs on the calling thread's
 * default stream with stream-ordered scratch and touches no context state
 * (ctx only selects the device; NULL = current device), so it can run from
 * many threads, also while fs_accumulate runs on the same context. */
int fs_assign(fs_context *ctx, const float *A, int64_t n, int num_objects, float gamma, int mode,
              uint8_t *out, int on_device);

/* Assignment.member_counts (solver.py:73-77): nonzero bytes per row of a
 * rows x n uint8 DEVICE matrix (the labels or the membership fs_assign left
 * on the device) -> counts[rows] on the host. */
int fs_member_counts(fs_context *ctx, const uint8_t *m, int64_t n, int rows, int64_t *counts);

/* ---- novel-view rendering ---- */

/* render_view / render_subset_alpha_depth (rasterizer.py:206-234) over the
 * resident scene: project (members only when member != NULL, N bytes,
 * scene.py:346-350), bin, and composite front to back per pixel
 * (render_property, rasterizer.py:133-203).  Host outputs: alpha and depth
 * H x W float64 (depth = blended depth / alpha, 0 where alpha == 0); with
 * channels 1 or 3, channel is N x channels float64 and value H x W x channels. */
int fs_render(fs_context *ctx, const fs_camera *cam, const uint8_t *member, double alpha_floor,
              double transmittance_floor, const double *channel, int channels, double *value,
              double *alpha, double *depth);

/* render_property (rasterizer.py:133-203) over a caller's TileBinning: k
 * splats (mean2d k x 2, conic k x 3 = inv_cov (a, b, c), depth, opacity =
 * scene.opacities[indices], channel k x channels gathered the same way) and
 * per-tile lists as CSR (tile_offsets[ntiles + 1], items = splat positions in
 * the order the lists are walked). */
int fs_render_splats(fs_context *ctx, int width, int height, int64_t k, const double *mean2d,
                     const double *conic, const double *depth, const double *opacity,
                     const int64_t *tile_offsets, const int64_t *items, double alpha_floor,
                     double transmittance_floor, const double *channel, int channels,
                     double *value, double *alpha, double *depth_out);

/* render_scene_mask (maskrender.py:69-95) -- and render_binary_mask
 * (maskrender.py:45-66) as num_objects = 2 with rows (~fg, fg): membership is
 * num_objects x N uint8; every non-empty object 1.. is rendered as a subset
 * and a pixel takes the object whose alpha exceeds tau with the smallest
 * blended depth (ties: smaller id).  labels: H x W uint16 (host). */
int fs_render_mask(fs_context *ctx, const fs_camera *cam, const uint8_t *membership,
                   int num_objects, double tau, double alpha_floor, double transmittance_floor,
                   uint16_t *labels);

/* ---- mask ingestion ---- */

/* Decode one label-mask PNG held in memory (masks.py:30-40 wire format:
 * non-interlaced 8- or 16-bit grayscale, pixel value = object id) into
 * out[height * width] uint16.  out == NULL only reports the dimensions.
 * Other PNG flavours return FS_EINVAL ("unsupported ...") so the caller can
 * use a general decoder.  Host-only and thread-safe (no CUDA, no context). */
int fs_decode_mask_png(const uint8_t *data, int64_t size, uint16_t *out, int64_t out_capacity,
                       int *width, int *height);

#ifdef __cplusplus
}
#endif

#endif /* FLASHSPLAT_B200_H */
