// fs_kernels.cuh -- host-side launch wrappers and device helpers shared across
// the translation units of the FlashSplat B200 library.
#pragma once

#include "fs_common.cuh"

namespace fs {

// ---- radix pass bookkeeping (shared by the sort and its consumers) ----
__device__ __forceinline__ bool pass_active(unsigned long long varying, int shift) {
    return ((varying >> shift) & 0xFFull) != 0ull;
}

// Number of executed passes strictly before `pass` (parity selects the buffer).
__device__ __forceinline__ int pass_parity(unsigned long long varying, int pass) {
    int p = 0;
    for (int q = 0; q < pass; ++q) p += pass_active(varying, 8 * q) ? 1 : 0;
    return p & 1;
}

// ---- fs_project.cu ----
void launch_scene_setup(int n, const double* means, const double* quats, const double* scales,
                        double* mx, double* my, double* mz, double* sig, cudaStream_t st);
void launch_project(int n, const double* mx, const double* my, const double* mz,
                    const double* sig, const double* opac, const Camera& cam, double alpha_floor,
                    int cull_floor, unsigned long long* keys, unsigned int* vals,
                    unsigned long long* rect, Rec32* r32, Rec64* r64, ViewCounters* vc,
                    ProjectExport ex, int num_sms, cudaStream_t st);

// ---- fs_sort.cu ----
int sort_grid(int num_sms);
size_t sort_hist_entries(int num_sms);
template <typename K>
int launch_radix_sort(K* keys0, unsigned int* vals0, K* keys1, unsigned int* vals1,
                      const unsigned int* d_n, unsigned int n_fixed,
                      const unsigned long long* d_or_and, int passes, unsigned int* hist,
                      int num_sms, cudaStream_t st);
void launch_scan_hist(unsigned int* data, int entries, cudaStream_t st);

// ---- fs_bin.cu ----
// After the depth sort: emit (tile, gid) instances in depth-rank order, sort
// them by tile (stable) and build per-tile ranges.  Instances beyond
// `capacity` set vc->overflow and the view is skipped by the raster kernel.
struct BinBuffers {
    unsigned long long* dkeys[2];  // depth sort ping-pong
    unsigned int* dvals[2];
    const unsigned long long* depth_or_and;  // &vc->key_or (key_or, key_and adjacent)
    const unsigned long long* rect;
    unsigned int* block_sums;  // sort_grid entries
    unsigned int* ikeys[2];    // instance tile ids (ping-pong)
    unsigned int* ivals[2];    // instance gids (ping-pong)
    const unsigned long long* tile_or_and;  // {tile mask, 0}
    unsigned int* hist;
    unsigned int* tile_start;  // ntiles + 1
    unsigned int capacity;
};
void launch_bin(int n, int ntiles, int tiles_x, int tile_passes, const BinBuffers& b,
                ViewCounters* vc, int num_sms, cudaStream_t st);

// Binning of an explicit splat list: secondary sort by gaussian index, then
// depth keys (written to dk0/dv0 for the depth sort that follows).
void launch_bin_splats_keys(int k, const long long* index, const double* mean2d,
                            const long long* radius, const double* depth, int width, int height,
                            unsigned long long* dk0, unsigned int* dv0, unsigned long long* dk1,
                            unsigned int* dv1, unsigned long long* rect, unsigned long long* idx_oa,
                            unsigned int* hist, ViewCounters* vc, int num_sms, cudaStream_t st);
void launch_view_begin(ViewCounters* vc, cudaStream_t st);

// ---- fs_raster.cu ----
struct RasterArgs {
    int width, height, tiles_x, ntiles;
    int num_objects;
    long long n_gaussians;
    double alpha_floor, t_floor;
    const uint16_t* mask;          // H x W labels (device)
    const unsigned int* tile_start;
    const unsigned int* inst_gid[2];  // instance gid ping-pong buffers
    int tile_passes;
    const unsigned long long* tile_or_and;
    const Rec32* r32;
    const Rec64* r64;
    double* acc;                   // E x N float64 accumulator
    ViewCounters* vc;
};
void launch_raster(const RasterArgs& a, cudaStream_t st);

// ---- fs_assign.cu ----
void launch_finalize(const double* acc, float* out, long long count, cudaStream_t st);
void launch_assign(const float* A, long long n, int e, float gamma, int mode, uint8_t* out,
                   cudaStream_t st);

}  // namespace fs
