// fs_kernels.cuh -- host-side launch wrappers and device helpers shared across
// the translation units of the FlashSplat B200 library.
#pragma once

#include "fs_common.cuh"

namespace fs {

// ---- radix sort state (one per sort call site, device memory) ----
struct SortState {
    unsigned int offsets[8][256];  // per digit position: histogram, then exclusive offsets
    unsigned int tile_counter[8];  // tile ids claimed by each pass
    unsigned int active;           // bit p: pass p permutes (not the identity)
    unsigned int epoch;            // look-back status generation
};

// Which ping-pong buffer holds the sorted result (0 or 1).
__device__ __forceinline__ int sort_result_parity(const SortState* st) {
    return __popc(st->active) & 1;
}

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

// One instance per covered tile.
__device__ __forceinline__ void count_rect_tiles(unsigned long long rc, int tiles_x,
                                                 unsigned int* count) {
    if (rc == ~0ull || !count) return;
    const unsigned int tx0 = rc & 0xFFFF, tx1 = (rc >> 16) & 0xFFFF;
    const unsigned int ty0 = (rc >> 32) & 0xFFFF, ty1 = (rc >> 48) & 0xFFFF;
    for (unsigned int ty = ty0; ty <= ty1; ++ty)
        for (unsigned int tx = tx0; tx <= tx1; ++tx) atomicAdd(&count[ty * (unsigned)tiles_x + tx], 1u);
}

// ---- fs_project.cu ----
void launch_scene_setup(int n, const double* means, const double* quats, const double* scales,
                        double* mx, double* my, double* mz, double* sig, cudaStream_t st);
void launch_project(int n, const double* mx, const double* my, const double* mz,
                    const double* sig, const double* opac, const Camera& cam, double alpha_floor,
                    int cull_floor, unsigned long long* keys, unsigned int* vals,
                    unsigned long long* rect, unsigned int* tile_count, Rec32* r32, Rec64* r64,
                    ViewCounters* vc, ProjectExport ex, int num_sms, cudaStream_t st);
void launch_view_begin(ViewCounters* vc, cudaStream_t st);

// ---- fs_sort.cu ----
size_t sort_status_words(unsigned int n_cap);
// d_or_and: {OR, AND} of the valid keys (digits constant over all keys are
// skipped); sub: if non-null, keys equal to all-ones are replaced by *sub.
template <typename K>
int launch_radix_sort(K* keys0, unsigned int* vals0, K* keys1, unsigned int* vals1,
                      const unsigned int* d_n, unsigned int n_cap,
                      const unsigned long long* d_or_and, const unsigned long long* sub, int passes,
                      SortState* st, unsigned long long* status, int num_sms, cudaStream_t s);

// ---- fs_bin.cu ----
struct BinBuffers {
    const unsigned int* sorted_gid[2];  // depth sort values (ping-pong)
    const SortState* depth_state;       // which of the two holds it
    const unsigned long long* rect;     // per gid
    unsigned int* count_bt;             // ntiles x bin_blocks(): counts, then offsets
    unsigned int* partial;              // bin_scan_blocks() partial sums
    unsigned int* tile_start;           // ntiles + 1
    unsigned int* inst;                 // capacity: ranks, gids after the per-tile sort
    unsigned int capacity;
};
constexpr int kMaxTiles = 49152;        // per-block tile histograms live in shared memory
int bin_blocks(int num_sms);
int bin_scan_blocks(int num_sms);
cudaError_t bin_configure();
void launch_bin(int n, int ntiles, int tiles_x, const BinBuffers& b, ViewCounters* vc,
                int num_sms, cudaStream_t st);

struct TileSortArgs {
    const unsigned int* tile_start;
    unsigned int* inst;
    unsigned int* scratch;
    const unsigned int* sorted_gid[2];   // depth sort values (ping-pong)
    const unsigned int* sorted_pkey[2];  // depth sort 32-bit primary keys (ping-pong)
    const unsigned long long* k64;       // full 64-bit depth key per gid
    const SortState* depth_state;
    int rank_bits;
    unsigned int cap;
    const ViewCounters* vc;
};

// Resolved (device-side) view of the depth order used by the per-tile sort.
struct TileSortKeys {
    const unsigned int* sorted_gid;
    const unsigned int* pkey;
    const unsigned long long* k64;
    int rank_bits;
};
__device__ __forceinline__ TileSortKeys resolve_keys(const TileSortArgs& t) {
    const int p = sort_result_parity(t.depth_state);
    return TileSortKeys{t.sorted_gid[p], t.sorted_pkey[p], t.k64, t.rank_bits};
}

// 32-bit primary depth keys: the 32 highest varying bits of the 64-bit keys
// (from their OR/AND), written in the order given by `order` (order0, or the
// result buffer of order_state's sort; both null: gid order); pk_oa receives
// the OR/AND of the primary keys.
void launch_primary_keys(int n, const unsigned long long* k64, const unsigned long long* oa64,
                         const unsigned int* order0, const unsigned int* order1,
                         const SortState* order_state, unsigned int* pk, unsigned int* vals,
                         unsigned long long* pk_oa, int num_sms, cudaStream_t st);
size_t tile_sort_smem_bytes(unsigned int cap);
cudaError_t tile_sort_configure(unsigned int cap);
void launch_tile_sort(int ntiles, const TileSortArgs& t, cudaStream_t st);

// Binning of an explicit splat list: secondary sort by gaussian index, then
// depth keys (written to dk0/dv0 for the depth sort that follows).
void launch_bin_splats_keys(int k, const long long* index, const double* mean2d,
                            const long long* radius, const double* depth, int width, int height,
                            unsigned long long* dk0, unsigned int* dv0, unsigned long long* dk1,
                            unsigned int* dv1, unsigned long long* rect, unsigned long long* k64,
                            unsigned long long* idx_oa, SortState* idx_state,
                            unsigned long long* idx_status, ViewCounters* vc, int num_sms,
                            cudaStream_t st);

// ---- fs_raster.cu ----
constexpr unsigned int kTileSortCap = 4096;  // bucket entries sorted in shared memory
struct RasterArgs {
    int width, height, tiles_x, ntiles;
    int num_objects;
    long long n_gaussians;
    double alpha_floor, t_floor;
    const uint16_t* mask;          // H x W labels (device)
    TileSortArgs sort;             // bucket -> depth-ordered gid list (prologue)
    const Rec32* r32;
    const Rec64* r64;
    double* acc;                   // E x N float64 accumulator
    ViewCounters* vc;
};
cudaError_t raster_configure();
void launch_raster(const RasterArgs& a, cudaStream_t st);

// ---- fs_assign.cu ----
void launch_finalize(const double* acc, float* out, long long count, cudaStream_t st);
void launch_assign(const float* A, long long n, int e, float gamma, int mode, uint8_t* out,
                   cudaStream_t st);

}  // namespace fs
