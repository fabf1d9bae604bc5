// fs_kernels.cuh -- host-side launch wrappers and device helpers shared across
// the translation units of the FlashSplat B200 library.
#pragma once

#include "fs_common.cuh"

namespace fs {

// Inclusive tile rectangle of a splat's radius box (rasterizer.py:106-113),
// packed tx0 | tx1 << 16 | ty0 << 32 | ty1 << 48; ~0 when empty.
__device__ __forceinline__ unsigned long long tile_rect(double mx, double my, double r, int tx_n,
                                                        int ty_n) {
    const double fx0 = floor((mx - r) / kTile), fx1 = floor((mx + r) / kTile);
    const double fy0 = floor((my - r) / kTile), fy1 = floor((my + r) / kTile);
    const int tx0 = fx0 < 0.0 ? 0 : (fx0 > tx_n ? tx_n : (int)fx0);
    const int tx1 = fx1 > tx_n - 1 ? tx_n - 1 : (fx1 < -1.0 ? -1 : (int)fx1);
    const int ty0 = fy0 < 0.0 ? 0 : (fy0 > ty_n ? ty_n : (int)fy0);
    const int ty1 = fy1 > ty_n - 1 ? ty_n - 1 : (fy1 < -1.0 ? -1 : (int)fy1);
    if (tx0 > tx1 || ty0 > ty1) return ~0ull;
    return (unsigned long long)tx0 | ((unsigned long long)tx1 << 16) |
           ((unsigned long long)ty0 << 32) | ((unsigned long long)ty1 << 48);
}

// ---- fs_project.cu ----
// float offsets of the PLY vertex properties in the reference's
// REQUIRED_PROPERTIES order (ply.py:17-23)
constexpr int kPlyProps = 17;
struct PlyOffsets {
    int k[kPlyProps];
};
// perm (nullable): slot p of the resident arrays takes input Gaussian perm[p]
void launch_scene_setup_ply(int n, const float* verts, int stride, const PlyOffsets& off,
                            const unsigned int* perm, double* mx, double* my, double* mz,
                            double* sig, double* opac, unsigned long long* bad, double* params,
                            cudaStream_t st);
void launch_scene_setup(int n, const double* means, const double* quats, const double* scales,
                        const double* opac_in, const unsigned int* perm, double* mx, double* my,
                        double* mz, double* sig, double* opac, cudaStream_t st);
// ---- fs_order.cu ----
// Spatial (Morton) order of the scene: perm[p] = input id of slot p.  scratch:
// a device buffer of scene_order_scratch_bytes(n) bytes owned by the caller.
size_t scene_order_scratch_bytes(int n);
cudaError_t launch_scene_order(int n, const double* means_aos, unsigned int* perm, void* scratch,
                               size_t scratch_bytes, int num_sms, cudaStream_t st);
cudaError_t launch_scene_order_ply(int n, const float* verts, int stride, const PlyOffsets& off,
                                   unsigned int* perm, void* scratch, size_t scratch_bytes,
                                   int num_sms, cudaStream_t st);
void launch_project(int n, const double* mx, const double* my, const double* mz,
                    const double* sig, const double* opac, const Camera& cam, double alpha_floor,
                    int cull_floor, unsigned long long* keys, unsigned long long* rect,
                    Rec32* r32, Rec64* r64,
                    ViewCounters* vc, ProjectExport ex, int num_sms, cudaStream_t st,
                    bool reset_counters = true, bool overlapped = false);
void launch_view_begin(ViewCounters* vc, cudaStream_t st);
void launch_splat_records(int k, const double* mean2d, const double* conic, const double* depth,
                          const double* opac, double alpha_floor, Rec32* r32, Rec64* r64,
                          unsigned long long* k64, int num_sms, cudaStream_t st);

// ---- fs_bin.cu ----
// Per-tile buckets of instances (any order) from per-block tile histograms.
// An instance is (32-bit primary depth key << 32 | gid); the primary key is
// the 32 highest bits in which the view's float64 depth keys differ.
struct BinBuffers {
    int n;                              // Gaussians (or splats)
    const unsigned long long* rect;     // per gid
    const unsigned long long* k64;      // per gid: order-preserving float64 depth key
    const unsigned long long* key_oa;   // {OR, ~AND} of the visible depth keys
    unsigned int* count_bt;             // ntiles x bin_blocks(): counts, then offsets in the tile
    unsigned int* tile_total;           // ntiles: bucket lengths
    unsigned int* tile_start;           // ntiles + 1
    unsigned int* tile_order;           // ntiles: tiles by decreasing bucket length (raster launch order)
    unsigned long long* inst;           // capacity: instances; the tile sort leaves each
                                        // bucket's depth-ordered gids in sorted_view()
    unsigned int capacity;
};
constexpr int kMaxTiles = 49152;        // tiles per binning band (per-block histograms in smem)
int bin_blocks(int num_sms);             // most blocks a binning uses (count-matrix width)
int bin_blocks_overlapped(int num_sms);  // blocks beside other streams' rasters
cudaError_t bin_configure();
// blocks: 0 = bin_blocks(num_sms)
void launch_bin(int ntiles, int tiles_x, const BinBuffers& b, ViewCounters* vc, int num_sms,
                cudaStream_t st, int blocks = 0);

// The depth-ordered gids of the bucket starting at `begin` overwrite the first
// half of the bucket's own instance bytes.
__host__ __device__ inline unsigned int* sorted_view(unsigned long long* inst, unsigned int begin) {
    return reinterpret_cast<unsigned int*>(inst + begin);
}

// Inputs of the per-tile depth ordering (fs_tilesort.cuh).
struct TileSortKeys {
    const unsigned long long* k64;   // full depth key per gid
    const unsigned int* tie;         // tie id per gid (nullptr: the gid itself)
};
struct TileSortArgs {
    const unsigned int* tile_start;
    unsigned long long* inst;
    unsigned long long* scratch64;   // 2 x capacity entries (long buckets only)
    TileSortKeys keys;
    unsigned int cap;
    const ViewCounters* vc;
};
size_t tile_sort_smem_bytes(unsigned int cap);
cudaError_t tile_sort_configure(unsigned int cap);
void launch_tile_sort(int ntiles, const TileSortArgs& t, cudaStream_t st);

// Explicit splat list (TileBinning over ProjectedGaussian): rect, depth key
// and key OR/AND per list position.
void launch_splat_keys(int k, const double* mean2d, const long long* radius, const double* depth,
                       int width, int height, unsigned long long* rect, unsigned long long* k64,
                       ViewCounters* vc, int num_sms, cudaStream_t st);

// ---- fs_raster.cu ----
constexpr unsigned int kTileSortCap = 4368;  // bucket entries sorted in shared memory
// Novel-view compositing outputs (render_property, rasterizer.py:133-203).
struct RenderArgs {
    double* alpha;                 // H x W accumulated alpha (rho)
    double* depth;                 // H x W blended depth (0 where alpha == 0)
    double* value;                 // H x W x channels (channels > 0)
    const double* channel;         // per gid x channels
    int channels;                  // 0, 1 or 3
    const unsigned int* lists;     // caller's ordered gid lists (tile_start offsets), or
                                   // nullptr: sort the binning's buckets
};
struct RasterArgs {
    int width, height, tiles_x, ntiles;
    int num_objects;
    long long n_gaussians;
    // alpha >= af_eff and T < tf_eff reproduce the reference's floors, and their
    // absence when a floor is 0 (alpha >= 0 > -1, T >= 0 > -1): see raster_floor()
    double af_eff, tf_eff;
    const uint16_t* mask;          // H x W labels (device)
    TileSortArgs sort;             // bucket -> depth-ordered gid list (prologue)
    const Rec32* r32;
    const Rec64* r64;
    double* acc;                   // N x E float64 accumulator (Gaussian-major), or
    unsigned long long* acc_fixed; // N x E x 2 uint64 fixed-point accumulator (FS_ACC_FIXED)
    ViewCounters* vc;
    const unsigned int* tile_order;  // ntiles: launch order (tile_start_kernel)
    RenderArgs render;             // launch_raster_render only
};
cudaError_t raster_configure();
void launch_raster(const RasterArgs& a, cudaStream_t st);
void launch_raster_render(const RasterArgs& a, cudaStream_t st);

// ---- fs_assign.cu ----
// Accumulator parts summed by the finalize (local or NVLink peer pointers).
constexpr int kMaxParts = 16;
struct AccParts {
    const void* p[kMaxParts];
    int n;
};
void launch_finalize(const AccParts& parts, bool fixed, long long g0, long long g1, int e,
                     float* out, long long ld, cudaStream_t st);
void launch_assign(const float* A, long long n, long long ld, int e, float gamma, int mode,
                   uint8_t* out, cudaStream_t st);
void launch_row_counts(const uint8_t* m, long long n, int rows, unsigned long long* counts,
                       cudaStream_t st);

}  // namespace fs
