// fs_capi.cu -- host runtime and C ABI of the FlashSplat B200 label solver.
//
// One fs_context owns a CUDA device, S streams and one workspace per stream.
// fs_accumulate hands views out round-robin to the streams; each view runs
// the device pipeline
//     K1 project -> K2a per-block tile histograms -> K2b per-tile scans ->
//     K2c bucket starts + launch order -> K2d emit instances ->
//     K3 raster (in-kernel bucket sort, walk, atomics, label check)
// entirely on its stream with device-side counts (no host sync inside the
// loop).  Host masks are staged through a pinned buffer per stream and
// copied on the same stream, so the copy of view v+S overlaps the kernels of
// views v+1..v+S-1.  After the loop the per-view counters are read back
// once; views whose instance count overflowed the buffers are re-run after
// growing them (the raster kernel skips an overflowed view, so nothing was
// added for it).
#include <cuda_runtime.h>
#include <nvtx3/nvToolsExt.h>

#include <algorithm>
#include <atomic>
#include <condition_variable>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <string>
#include <mutex>
#include <set>
#include <thread>
#include <vector>

#include "flashsplat_b200.h"
#include "fs_common.cuh"
#include "fs_kernels.cuh"

namespace fs {

namespace {
thread_local std::string g_error;

int fail(int code, const char* fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof(buf), fmt, ap);
    va_end(ap);
    g_error = buf;
    return code;
}

int bits_for(unsigned int v) {  // bits needed to represent values 0..v
    int b = 0;
    while (b < 32 && (v >> b) != 0u) ++b;
    return b;
}

}  // namespace

int set_cuda_error(cudaError_t e, const char* expr, const char* file, int line) {
    return fail(FS_ECUDA, "CUDA error %s (%s) at %s:%d: %s", cudaGetErrorName(e),
                cudaGetErrorString(e), file, line, expr);
}

struct Work {
    cudaStream_t stream = nullptr;
    long long n_cap = 0;
    unsigned int inst_cap = 0;
    int ntiles_cap = 0;
    size_t mask_cap = 0;
    unsigned long long* rect = nullptr;      // per gid tile rectangle
    Rec32* r32 = nullptr;
    Rec64* r64 = nullptr;
    unsigned long long* k64 = nullptr;       // per gid order-preserving float64 depth key
    unsigned int* tie = nullptr;             // per splat tie id (fs_bin_splats only)
    unsigned long long* inst = nullptr;      // per-tile buckets of instances -> sorted gids
    unsigned long long* scratch64 = nullptr; // 2 x capacity: long-bucket merge scratch
    unsigned int* count_bt = nullptr;        // ntiles x bin_blocks
    unsigned int* tile_total = nullptr;      // bucket lengths
    unsigned int* tile_start = nullptr;
    unsigned int* tile_order = nullptr;      // raster launch order (tile_start_kernel)
    ViewCounters* vc = nullptr;
    uint16_t* mask_dev = nullptr;
    uint16_t* pinned = nullptr;
    cudaEvent_t h2d_done = nullptr;
    bool h2d_pending = false;
    cudaEvent_t done = nullptr;
    cudaEvent_t view_done = nullptr;  // last view enqueued on this stream (dynamic queue)
};

}  // namespace fs

struct fs_context {
    int device = 0;
    int num_sms = 148;
    long long n = 0;
    double* mx = nullptr;
    double* my = nullptr;
    double* mz = nullptr;
    double* sig = nullptr;
    double* opac = nullptr;
    fs::ViewCounters* view_log = nullptr;
    int view_log_cap = 0;
    std::vector<fs::Work> work;
    cudaEvent_t ev_start = nullptr, ev_stop = nullptr;
    // entry points order their streams after the caller's stream (fs_set_stream;
    // default: the legacy default stream) with this event -- no device-wide sync
    cudaStream_t caller_stream = nullptr;
    cudaEvent_t ev_caller = nullptr;
    float* fin_tmp = nullptr;     // fs_reduce_finalize: E x slice float32 (host output)
    size_t fin_tmp_cap = 0;
    uint8_t* fin_lab = nullptr;   // fs_finalize_multi: the slice's labels
    size_t fin_lab_cap = 0;
    unsigned char* fin_stage = nullptr;  // peer parts staged when P2P access is unavailable
    size_t fin_stage_cap = 0;
    float* ply_raw = nullptr;     // fs_set_scene_ply: the uploaded vertex records
    size_t ply_raw_cap = 0;
    unsigned long long* ply_bad = nullptr;  // its four first-offender slots
    bool timing = false;
    std::vector<cudaEvent_t> stage_events;  // 4 per view when timing
    // grow-only scratch reused across calls (no cudaMalloc/cudaFree per call)
    long long scene_cap = 0;
    // the resident scene is stored in spatial (Morton) order: slot p holds input
    // Gaussian perm[p] (fs_order.cu); perm_on = false keeps input order
    // (FS_SCENE_ORDER=0, for A/B measurements)
    unsigned int* perm = nullptr;
    bool perm_on = false;
    void* order_scratch = nullptr;  // Morton codes + radix-sort scratch (grow-only)
    size_t order_scratch_bytes = 0;
    double* up_opac = nullptr;    // opacity staging (permuted by the setup kernel)
    double* up_means = nullptr;   // AoS staging of the scene upload
    double* up_quats = nullptr;
    double* up_scales = nullptr;
    unsigned char* pinned_up[2] = {nullptr, nullptr};  // host->device staging ring
    cudaEvent_t pinned_free[2] = {nullptr, nullptr};
    // novel-view rendering (fs_render*): outputs, inputs, mask combine
    double* rn_f64 = nullptr;     // alpha | depth | value (H*W*(2 + C))
    size_t rn_f64_cap = 0;
    double* rn_in = nullptr;      // channel (N x C) or splat arrays
    size_t rn_in_cap = 0;
    uint8_t* rn_member = nullptr;
    size_t rn_member_cap = 0;
    unsigned int* rn_u32 = nullptr;  // caller's tile lists, launch order
    size_t rn_u32_cap = 0;
    uint16_t* rn_labels = nullptr;
    size_t rn_labels_cap = 0;
    unsigned long long* rn_rect = nullptr;  // fs_render_mask: the full scene's tile rectangles
    size_t rn_rect_cap = 0;
    unsigned long long* cnt = nullptr;      // fs_member_counts
    size_t cnt_cap = 0;
};



namespace fs {
// error reporting for the host-only translation units (fs_ingest.cpp)
int report_error(int code, const char* msg) { return fail(code, "%s", msg); }
}  // namespace fs

using fs::fail;

namespace {
// NVTX range for the duration of an entry point (header-only NVTX v3: free
// unless a profiler injects itself)
struct Range {
    explicit Range(const char* name) { nvtxRangePushA(name); }
    ~Range() { nvtxRangePop(); }
};
}  // namespace

namespace {

#define CK(expr)                                                                  \
    do {                                                                          \
        cudaError_t _e = (expr);                                                  \
        if (_e != cudaSuccess) return fs::set_cuda_error(_e, #expr, __FILE__, __LINE__); \
    } while (0)

template <typename T>
int dev_alloc(T** p, size_t count) {
    if (*p) {
        cudaFree(*p);
        cudaGetLastError();
        *p = nullptr;
    }
    if (count == 0) count = 1;
    cudaError_t e = cudaMalloc(reinterpret_cast<void**>(p), count * sizeof(T));
    if (e != cudaSuccess) {
        cudaGetLastError();
        return fail(FS_ENOMEM, "cudaMalloc of %zu bytes failed: %s", count * sizeof(T),
                    cudaGetErrorString(e));
    }
    return FS_OK;
}

constexpr size_t kUploadChunk = 8u << 20;  // pinned staging chunk (bytes; 32 MB measured slower)

// Host memcpy into pinned staging, split over a persistent pool of threads:
// one core copies ~10 GB/s, well below the DMA rate, so pageable uploads were
// memcpy-bound (and spawning threads per 8 MB chunk cost ~0.2 ms a chunk).
class CopyPool {
public:
    // 8 threads: 16 on the GPU hosts measured slower (host memory bandwidth)
    CopyPool() : parts_(std::max(1u, std::min(8u, std::thread::hardware_concurrency()))) {
        for (unsigned i = 1; i < parts_; ++i) std::thread([this, i] { worker(i); }).detach();
    }
    void copy(void* dst, const void* src, size_t bytes) {
        if (parts_ == 1 || bytes < (2u << 20)) {
            memcpy(dst, src, bytes);
            return;
        }
        std::lock_guard<std::mutex> caller(call_);  // one job at a time
        {
            std::lock_guard<std::mutex> g(m_);
            dst_ = static_cast<char*>(dst);
            src_ = static_cast<const char*>(src);
            bytes_ = bytes;
            pending_ = parts_ - 1;
            ++gen_;
        }
        cv_.notify_all();
        part(0);
        std::unique_lock<std::mutex> g(m_);
        done_.wait(g, [this] { return pending_ == 0; });
    }

private:
    void part(unsigned i) {
        const size_t per = (bytes_ + parts_ - 1) / parts_;
        const size_t off = std::min(bytes_, per * i), n = std::min(bytes_ - off, per);
        if (n) memcpy(dst_ + off, src_ + off, n);
    }
    void worker(unsigned i) {
        unsigned seen = 0;
        for (;;) {
            {
                std::unique_lock<std::mutex> g(m_);
                cv_.wait(g, [&] { return gen_ != seen; });
                seen = gen_;
            }
            part(i);
            std::lock_guard<std::mutex> g(m_);
            if (--pending_ == 0) done_.notify_one();
        }
    }
    const unsigned parts_;
    std::mutex call_, m_;
    std::condition_variable cv_, done_;
    char* dst_ = nullptr;
    const char* src_ = nullptr;
    size_t bytes_ = 0;
    unsigned pending_ = 0, gen_ = 0;
};

void parallel_memcpy(void* dst, const void* src, size_t bytes) {
    static CopyPool* pool = new CopyPool();  // never destroyed: its threads are detached
    pool->copy(dst, src, bytes);
}

// Page-locked (cudaMallocHost / cudaHostRegister) host range: the DMA engine
// reads it directly, no staging copy.
bool host_pinned(const void* p, size_t bytes) {
    if (!p || !bytes) return false;
    const void* ends[2] = {p, static_cast<const char*>(p) + bytes - 1};
    for (const void* q : ends) {
        cudaPointerAttributes at;
        if (cudaPointerGetAttributes(&at, q) != cudaSuccess) {
            cudaGetLastError();
            return false;
        }
        if (at.type != cudaMemoryTypeHost) return false;
    }
    return true;
}

// Host -> device copy.  Pinned sources are copied directly; pageable ones go
// through the context's two pinned chunks, so the host memcpy of chunk i
// overlaps the DMA of chunk i-1.
int upload(fs_context* ctx, void* dst, const void* src, size_t bytes, cudaStream_t st) {
    if (host_pinned(src, bytes)) {
        CK(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, st));
        return FS_OK;
    }
    if (!ctx->pinned_up[0]) {
        for (int k = 0; k < 2; ++k) {
            CK(cudaMallocHost(reinterpret_cast<void**>(&ctx->pinned_up[k]), kUploadChunk));
            CK(cudaEventCreateWithFlags(&ctx->pinned_free[k], cudaEventDisableTiming));
            CK(cudaEventRecord(ctx->pinned_free[k], st));
        }
    }
    const unsigned char* s = static_cast<const unsigned char*>(src);
    unsigned char* d = static_cast<unsigned char*>(dst);
    int slot = 0;
    for (size_t off = 0; off < bytes; off += kUploadChunk) {
        const size_t m = std::min(kUploadChunk, bytes - off);
        CK(cudaEventSynchronize(ctx->pinned_free[slot]));
        parallel_memcpy(ctx->pinned_up[slot], s + off, m);
        CK(cudaMemcpyAsync(d + off, ctx->pinned_up[slot], m, cudaMemcpyHostToDevice, st));
        CK(cudaEventRecord(ctx->pinned_free[slot], st));
        slot ^= 1;
    }
    return FS_OK;
}

// Blocking copy ordered on one of the context's (non-blocking) streams: unlike
// cudaMemcpy on the legacy default stream it never waits for other threads'
// work on the device (a concurrent fs_assign, an NCCL stream).
cudaError_t sync_copy(void* dst, const void* src, size_t bytes, cudaMemcpyKind kind,
                      cudaStream_t st) {
    cudaError_t e = cudaMemcpyAsync(dst, src, bytes, kind, st);
    return e == cudaSuccess ? cudaStreamSynchronize(st) : e;
}

template <typename T>
int grow(T** p, size_t* cap, size_t count) {
    if (count <= *cap && *p) return FS_OK;
    if (*p) cudaFree(*p);
    *p = nullptr;
    cudaError_t e = cudaMalloc(reinterpret_cast<void**>(p), std::max<size_t>(count, 1) * sizeof(T));
    if (e != cudaSuccess) {
        cudaGetLastError();
        *cap = 0;
        return fail(FS_ENOMEM, "cudaMalloc of %zu bytes failed", count * sizeof(T));
    }
    *cap = count;
    return FS_OK;
}

void free_work(fs::Work& w) {
    auto f = [](void* p) {
        if (p) cudaFree(p);
    };
    f(w.rect); f(w.r32); f(w.r64); f(w.k64); f(w.tie); f(w.inst); f(w.scratch64);
    f(w.count_bt); f(w.tile_total); f(w.tile_start); f(w.tile_order); f(w.vc); f(w.mask_dev);
    if (w.pinned) cudaFreeHost(w.pinned);
    if (w.h2d_done) cudaEventDestroy(w.h2d_done);
    if (w.done) cudaEventDestroy(w.done);
    if (w.view_done) cudaEventDestroy(w.view_done);
    if (w.stream) cudaStreamDestroy(w.stream);
    w = fs::Work{};
}

// Size a workspace for n Gaussians, ntiles tiles, inst instances, mask_px pixels.
int ensure_work(fs_context* ctx, fs::Work& w, long long n, int ntiles, unsigned int inst,
                size_t mask_px) {
    int rc;
    if (n > w.n_cap) {
        if ((rc = dev_alloc(&w.rect, n))) return rc;
        if ((rc = dev_alloc(&w.r32, n))) return rc;
        if ((rc = dev_alloc(&w.r64, n))) return rc;
        if ((rc = dev_alloc(&w.k64, n))) return rc;
        if ((rc = dev_alloc(&w.tie, n))) return rc;
        w.n_cap = n;
    }
    if (!w.vc) {
        if ((rc = dev_alloc(&w.vc, 1))) return rc;
    }
    if (inst > w.inst_cap) {
        if ((rc = dev_alloc(&w.inst, (size_t)inst + 2))) return rc;  // +2: bulk-copy slack
        if ((rc = dev_alloc(&w.scratch64, 2 * (size_t)inst))) return rc;
        w.inst_cap = inst;
    }
    if (ntiles > w.ntiles_cap) {
        if ((rc = dev_alloc(&w.tile_start, (size_t)ntiles + 1))) return rc;
        if ((rc = dev_alloc(&w.tile_order, (size_t)ntiles))) return rc;
        if ((rc = dev_alloc(&w.tile_total, (size_t)ntiles))) return rc;
        if ((rc = dev_alloc(&w.count_bt, (size_t)ntiles * fs::bin_blocks(ctx->num_sms)))) return rc;
        w.ntiles_cap = ntiles;
    }
    if (mask_px > w.mask_cap) {
        if ((rc = dev_alloc(&w.mask_dev, mask_px))) return rc;
        if (w.pinned) cudaFreeHost(w.pinned);
        w.pinned = nullptr;
        CK(cudaMallocHost(reinterpret_cast<void**>(&w.pinned), mask_px * sizeof(uint16_t)));
        w.mask_cap = mask_px;
    }
    return FS_OK;
}

fs::Camera to_cam(const fs_camera& c) {
    fs::Camera k;
    k.width = c.width;
    k.height = c.height;
    k.fx = c.fx;
    k.fy = c.fy;
    k.cx = c.cx;
    k.cy = c.cy;
    for (int i = 0; i < 16; ++i) k.w2c[i] = c.world_to_camera[i];
    k.near_clip = c.near_clip;
    return k;
}

int check_cam(const fs_camera& c, int idx) {
    if (c.width < 1 || c.height < 1)
        return fail(FS_EINVAL, "view %d: image dimensions must be >= 1, got %dx%d", idx, c.width,
                    c.height);
    long long tiles = (long long)fs::tiles_x_of(c.width) * fs::tiles_y_of(c.height);
    if (tiles > (1 << 24)) return fail(FS_EINVAL, "view %d: image too large (%lld tiles)", idx, tiles);
    if (fs::tiles_x_of(c.width) > fs::kMaxTiles)  // one tile row per binning band at least
        return fail(FS_EINVAL, "view %d: image too wide (%d tile columns > %d)", idx,
                    fs::tiles_x_of(c.width), fs::kMaxTiles);
    return FS_OK;
}

// vc: the view's counters (the workspace's own, or a slot of the view log)
fs::BinBuffers bin_buffers(fs::Work& w, int n, fs::ViewCounters* vc = nullptr) {
    if (!vc) vc = w.vc;
    fs::BinBuffers b;
    b.n = n;
    b.rect = w.rect;
    b.k64 = w.k64;
    b.key_oa = &vc->key_or;  // key_or, key_nand are adjacent
    b.count_bt = w.count_bt;
    b.tile_total = w.tile_total;
    b.tile_order = w.tile_order;
    b.tile_start = w.tile_start;
    b.inst = w.inst;
    b.capacity = w.inst_cap;
    return b;
}

// The resident scene's slot -> input id map, or nullptr when it is in input order.
const unsigned int* scene_perm(const fs_context* ctx) { return ctx->perm_on ? ctx->perm : nullptr; }

// Grow-only scratch of the scene-order step (no per-call device allocation).
int ensure_order_scratch(fs_context* ctx, long long n) {
    const size_t need = fs::scene_order_scratch_bytes((int)n);
    if (need <= ctx->order_scratch_bytes) return FS_OK;
    if (ctx->order_scratch) CK(cudaFree(ctx->order_scratch));
    ctx->order_scratch = nullptr;
    ctx->order_scratch_bytes = 0;
    CK(cudaMalloc(&ctx->order_scratch, need));
    ctx->order_scratch_bytes = need;
    return FS_OK;
}

// Spatial scene order (fs_order.cu) unless FS_SCENE_ORDER=0.
bool scene_order_enabled() {
    const char* e = getenv("FS_SCENE_ORDER");
    return !(e && e[0] == '0');
}

fs::TileSortArgs tile_sort_args(fs::Work& w, const unsigned int* tie = nullptr,
                                fs::ViewCounters* vc = nullptr) {
    fs::TileSortArgs t;
    t.tile_start = w.tile_start;
    t.inst = w.inst;
    t.scratch64 = w.scratch64;
    t.keys.k64 = w.k64;
    t.keys.tie = tie;
    t.cap = fs::kTileSortCap;
    t.vc = vc ? vc : w.vc;
    return t;
}

// Projection + per-tile buckets of one view on workspace w (the buckets are
// depth-ordered by the raster prologue or launch_tile_sort).
// vc == nullptr: the workspace's counters, reset first; otherwise the caller's
// zeroed slot (the accumulate loop's view log -- no reset/copy kernels per view).
// bin_blocks: binning grid (0 = the full-GPU default; the accumulate loop passes
// fewer when other streams' rasters run beside it, and the projection then
// takes a smaller grid too).
void enqueue_bin(fs_context* ctx, fs::Work& w, const fs::Camera& cam, double alpha_floor,
                 int cull_floor, fs::ProjectExport ex, cudaEvent_t after_project = nullptr,
                 fs::ViewCounters* vc = nullptr, int bin_blocks = 0) {
    const int n = (int)ctx->n;
    const int tx = fs::tiles_x_of(cam.width), ntiles = tx * fs::tiles_y_of(cam.height);
    const bool own = vc == nullptr;
    if (own) vc = w.vc;
    ex.perm = scene_perm(ctx);
    fs::launch_project(n, ctx->mx, ctx->my, ctx->mz, ctx->sig, ctx->opac, cam, alpha_floor,
                       cull_floor, w.k64, w.rect, w.r32, w.r64, vc, ex,
                       ctx->num_sms, w.stream, own, bin_blocks > 0);
    if (after_project) cudaEventRecord(after_project, w.stream);
    fs::launch_bin(ntiles, tx, bin_buffers(w, n, vc), vc, ctx->num_sms, w.stream, bin_blocks);
}

// Kernels one enqueue_view launches (for the stats' launch count).
int view_launches() { return 1 + 4 + 1; }

// One view of fs_accumulate; its counters live in `log` (zeroed by the caller).
void enqueue_view(fs_context* ctx, fs::Work& w, const fs::Camera& cam, const uint16_t* mask,
                  int num_objects, double alpha_floor, double t_floor, int acc_kind, void* acc,
                  fs::ViewCounters* log, cudaEvent_t* ev = nullptr) {
    if (ev) cudaEventRecord(ev[0], w.stream);
    const int blocks = ctx->work.size() > 1 ? fs::bin_blocks_overlapped(ctx->num_sms) : 0;
    enqueue_bin(ctx, w, cam, alpha_floor, 1, fs::ProjectExport{}, ev ? ev[1] : nullptr, log, blocks);
    if (ev) cudaEventRecord(ev[2], w.stream);
    const int tx = fs::tiles_x_of(cam.width), ntiles = tx * fs::tiles_y_of(cam.height);
    fs::RasterArgs ra{};
    ra.width = cam.width;
    ra.height = cam.height;
    ra.tiles_x = tx;
    ra.ntiles = ntiles;
    ra.num_objects = num_objects;
    ra.n_gaussians = ctx->n;
    ra.af_eff = alpha_floor > 0.0 ? alpha_floor : -1.0;  // contributions.py:148-149
    ra.tf_eff = t_floor > 0.0 ? t_floor : -1.0;          // contributions.py:156-157
    ra.mask = mask;
    // tile lists in (depth, input id) order (accumulator rows: Rec32::oid)
    ra.sort = tile_sort_args(w, scene_perm(ctx), log);
    ra.r32 = w.r32;
    ra.r64 = w.r64;
    if (acc_kind == FS_ACC_FIXED)
        ra.acc_fixed = static_cast<unsigned long long*>(acc);
    else
        ra.acc = static_cast<double*>(acc);
    ra.vc = log;
    ra.tile_order = w.tile_order;
    fs::launch_raster(ra, w.stream);
    if (ev) cudaEventRecord(ev[3], w.stream);
}

// Orders the context's streams after the caller's stream (fs_set_stream; by
// default the legacy default stream, which is where torch's default stream
// and the synchronous CUDA calls of other libraries land): work enqueued before
// the call -- zeroing an accumulator, an NCCL reduction the caller waited on --
// completes before our kernels touch it.  Unlike cudaDeviceSynchronize this does
// not wait for other threads' independent work (a concurrent fs_assign).
int order_after_caller(fs_context* ctx) {
    CK(cudaEventRecord(ctx->ev_caller, ctx->caller_stream));
    for (auto& w : ctx->work) CK(cudaStreamWaitEvent(w.stream, ctx->ev_caller, 0));
    return FS_OK;
}

unsigned int initial_inst_cap(long long n) {
    long long c = std::max<long long>(1 << 22, 4 * n);
    return (unsigned int)std::min<long long>(c, 0x7fffffffLL);
}

// ---- accumulation runtime (fs_accumulate / fs_accumulate_multi) ----

// Validated view list: sizes for the workspaces.
struct ViewPlan {
    int n_views = 0;
    int max_tiles = 1;
    size_t max_px = 1;
    long long view_px = 0;
};

int plan_views(int n_views, const fs_camera* cams, const uint16_t* const* masks, int num_objects,
               int acc_kind, ViewPlan& p) {
    if (n_views < 0 || (n_views > 0 && (!cams || !masks)))
        return fail(FS_EINVAL, "fs_accumulate: bad view arguments");
    if (num_objects < 1 || num_objects > 65536)
        return fail(FS_EINVAL, "fs_accumulate: num_objects must be in [1, 65536], got %d", num_objects);
    if (acc_kind != FS_ACC_F64 && acc_kind != FS_ACC_FIXED)
        return fail(FS_EINVAL, "bad accumulator kind %d", acc_kind);
    p.n_views = n_views;
    int rc;
    for (int v = 0; v < n_views; ++v) {
        if ((rc = check_cam(cams[v], v))) return rc;
        if (!masks[v]) return fail(FS_EINVAL, "view %d: NULL mask", v);
        p.max_tiles = std::max(p.max_tiles, fs::tiles_x_of(cams[v].width) * fs::tiles_y_of(cams[v].height));
        p.max_px = std::max(p.max_px, (size_t)cams[v].width * cams[v].height);
        p.view_px += (long long)cams[v].width * cams[v].height;
    }
    return FS_OK;
}

// One context's share of an accumulation.
struct CtxRun {
    std::vector<int> views;             // global view indices run here, in enqueue order
    std::vector<fs::ViewCounters> log;  // their counters, same order
    double gpu_ms = 0, prep_ms = 0, bin_ms = 0, raster_ms = 0;
    long long launches = 0, retried = 0;
};

// Host mask of one view -> the workspace's device mask buffer, on its stream
// (stream order keeps it behind the previous view's raster).  Page-locked
// sources are DMA'd directly; pageable ones go through the stream's pinned
// buffer, whose previous copy must have finished first.
int stage_mask(fs::Work& w, const fs_camera& cam, const uint16_t* src, const uint16_t** dev) {
    const size_t bytes = (size_t)cam.width * cam.height * sizeof(uint16_t);
    if (host_pinned(src, bytes)) {
        CK(cudaMemcpyAsync(w.mask_dev, src, bytes, cudaMemcpyHostToDevice, w.stream));
    } else {
        if (w.h2d_pending) CK(cudaEventSynchronize(w.h2d_done));
        parallel_memcpy(w.pinned, src, bytes);
        CK(cudaMemcpyAsync(w.mask_dev, w.pinned, bytes, cudaMemcpyHostToDevice, w.stream));
        CK(cudaEventRecord(w.h2d_done, w.stream));
        w.h2d_pending = true;
    }
    *dev = w.mask_dev;
    return FS_OK;
}

// Accumulates views into acc on ctx's device.  queue == nullptr: views 0..n-1
// round-robin over the context's streams, all enqueued at once.  Otherwise
// views are popped from the shared queue, at most one in flight per stream, so
// several contexts (GPUs) share the list dynamically.  Each view runs
// project -> bin -> raster on one stream with its counters in a zeroed slot of
// the view log; the log is read back once, and views whose instance count
// overflowed the buffers (the raster skipped them, nothing was added) are
// re-run after growing them.
int accumulate_on(fs_context* ctx, const ViewPlan& plan, const fs_camera* cams,
                  const uint16_t* const* masks, int masks_on_device, int num_objects,
                  double alpha_floor, double t_floor, int acc_kind, void* acc,
                  std::atomic<int>* queue, CtxRun& R) {
    Range nvtx_range("view loop (project -> bin -> raster per view)");
    CK(cudaSetDevice(ctx->device));
    int rc;
    const int n_views = plan.n_views;
    const size_t mask_px = masks_on_device ? 1 : plan.max_px;
    for (auto& w : ctx->work) {
        unsigned int cap = std::max(w.inst_cap, initial_inst_cap(ctx->n));
        if ((rc = ensure_work(ctx, w, ctx->n, plan.max_tiles, cap, mask_px))) return rc;
    }
    if (n_views > ctx->view_log_cap) {
        if ((rc = dev_alloc(&ctx->view_log, (size_t)n_views))) return rc;
        ctx->view_log_cap = n_views;
    }
    const int S = (int)ctx->work.size();
    fs::Work& w0 = ctx->work[0];
    if (ctx->timing) {
        while ((int)ctx->stage_events.size() < 4 * n_views) {
            cudaEvent_t e;
            CK(cudaEventCreate(&e));
            ctx->stage_events.push_back(e);
        }
    }
    if ((rc = order_after_caller(ctx))) return rc;
    CK(cudaMemsetAsync(ctx->view_log, 0, sizeof(fs::ViewCounters) * (size_t)n_views, w0.stream));
    CK(cudaEventRecord(ctx->ev_start, w0.stream));
    for (int s = 1; s < S; ++s) CK(cudaStreamWaitEvent(ctx->work[s].stream, ctx->ev_start, 0));
    R.views.clear();
    for (int i = 0;; ++i) {
        fs::Work& w = ctx->work[i % S];
        if (queue && i >= S) CK(cudaEventSynchronize(w.view_done));  // this stream's last view
        const int v = queue ? queue->fetch_add(1) : i;
        if (v >= n_views) break;
        const uint16_t* mask = masks[v];
        if (!masks_on_device && (rc = stage_mask(w, cams[v], masks[v], &mask))) return rc;
        enqueue_view(ctx, w, to_cam(cams[v]), mask, num_objects, alpha_floor, t_floor, acc_kind,
                     acc, ctx->view_log + i, ctx->timing ? &ctx->stage_events[4 * i] : nullptr);
        if (queue) CK(cudaEventRecord(w.view_done, w.stream));
        R.views.push_back(v);
        R.launches += view_launches();
    }
    CK(cudaGetLastError());
    for (int s = 1; s < S; ++s) {
        CK(cudaEventRecord(ctx->work[s].done, ctx->work[s].stream));
        CK(cudaStreamWaitEvent(w0.stream, ctx->work[s].done, 0));
    }
    CK(cudaEventRecord(ctx->ev_stop, w0.stream));
    CK(cudaEventSynchronize(ctx->ev_stop));
    for (auto& w : ctx->work) w.h2d_pending = false;
    float ms = 0.f;
    CK(cudaEventElapsedTime(&ms, ctx->ev_start, ctx->ev_stop));
    R.gpu_ms = ms;
    const int k = (int)R.views.size();
    if (ctx->timing) {
        for (int i = 0; i < k; ++i) {
            float a = 0, b = 0, c = 0;
            cudaEvent_t* e = &ctx->stage_events[4 * i];
            CK(cudaEventElapsedTime(&a, e[0], e[1]));
            CK(cudaEventElapsedTime(&b, e[1], e[2]));
            CK(cudaEventElapsedTime(&c, e[2], e[3]));
            R.prep_ms += a;
            R.bin_ms += b;
            R.raster_ms += c;
        }
    }
    R.log.resize(k);
    if (k) CK(sync_copy(R.log.data(), ctx->view_log, sizeof(fs::ViewCounters) * k,
                        cudaMemcpyDeviceToHost, w0.stream));
    for (int j = 0; j < k; ++j) {
        if (!R.log[j].overflow) continue;
        const int v = R.views[j];
        const unsigned int need = (unsigned int)std::min<unsigned long long>(
            0x7fffffffull, (unsigned long long)R.log[j].n_instances + R.log[j].n_instances / 4 + 1024);
        for (auto& o : ctx->work)  // later calls start with the grown capacity
            if (o.inst_cap < need && (rc = ensure_work(ctx, o, ctx->n, plan.max_tiles, need, mask_px)))
                return rc;
        const uint16_t* mask = masks[v];
        if (!masks_on_device && (rc = stage_mask(w0, cams[v], masks[v], &mask))) return rc;
        CK(cudaMemsetAsync(ctx->view_log + j, 0, sizeof(fs::ViewCounters), w0.stream));
        enqueue_view(ctx, w0, to_cam(cams[v]), mask, num_objects, alpha_floor, t_floor, acc_kind,
                     acc, ctx->view_log + j);
        CK(cudaGetLastError());
        CK(sync_copy(&R.log[j], ctx->view_log + j, sizeof(fs::ViewCounters), cudaMemcpyDeviceToHost,
                     w0.stream));
        w0.h2d_pending = false;
        if (R.log[j].overflow) return fail(FS_ENOMEM, "view %d: instance buffer overflow after retry", v);
        ++R.retried;
        R.launches += view_launches();
    }
    return FS_OK;
}

// Totals over the contexts' runs; the label range error of the first offending
// view in the caller's order (contributions.py:104-114).
int finish_stats(const CtxRun* R, int n_ctx, const ViewPlan& plan, int num_objects,
                 fs_accumulate_stats* stats) {
    long long bad_view = -1;
    unsigned int bad_label = 0;
    for (int c = 0; c < n_ctx; ++c)
        for (size_t j = 0; j < R[c].views.size(); ++j)
            if (R[c].log[j].max_label >= (unsigned)num_objects &&
                (bad_view < 0 || R[c].views[j] < bad_view)) {
                bad_view = R[c].views[j];
                bad_label = R[c].log[j].max_label;
            }
    if (stats) {
        stats->label_error_view = bad_view;
        stats->views = plan.n_views;
        stats->view_pixels = plan.view_px;
        for (int c = 0; c < n_ctx; ++c) {
            for (const auto& l : R[c].log) {
                stats->emitted += l.n_emitted;
                stats->instances += l.n_instances;
                stats->tile_steps += (int64_t)l.tile_steps;
                stats->exact_evals += (int64_t)l.exact_evals;
                stats->atomics += (int64_t)l.atomics;
            }
            stats->retried_views += R[c].retried;
            stats->launches += R[c].launches;
            stats->gpu_ms = std::max(stats->gpu_ms, R[c].gpu_ms);
            stats->prep_ms += R[c].prep_ms;
            stats->bin_ms += R[c].bin_ms;
            stats->raster_ms += R[c].raster_ms;
        }
    }
    if (bad_view >= 0)
        return fail(FS_ELABEL, "view %lld: label %u exceeds object count %d", bad_view, bad_label,
                    num_objects);
    return FS_OK;
}

// ---- finalize (fs_finalize / fs_reduce_finalize / fs_finalize_multi) ----

// Peer access dev -> peer (NVLink P2P loads from dev's kernels), enabled once.
bool enable_peer(int dev, int peer) {
    if (dev == peer) return true;
    static std::mutex m;
    static std::set<std::pair<int, int>> on;
    std::lock_guard<std::mutex> g(m);
    if (on.count({dev, peer})) return true;
    int can = 0;
    if (cudaDeviceCanAccessPeer(&can, dev, peer) != cudaSuccess || !can) {
        cudaGetLastError();
        return false;
    }
    int cur = 0;
    cudaGetDevice(&cur);
    cudaSetDevice(dev);
    cudaError_t e = cudaDeviceEnablePeerAccess(peer, 0);
    cudaSetDevice(cur);
    if (e == cudaErrorPeerAccessAlreadyEnabled) e = cudaSuccess;
    cudaGetLastError();
    if (e != cudaSuccess) return false;
    on.insert({dev, peer});
    return true;
}

// Parts of slice [g0, g1) for ctx's finalize: the other contexts' accumulators
// read in place over peer memory, or -- without P2P access -- their slice
// copied into local staging first.
int gather_parts(fs_context* ctx, fs_context* const* ctxs, int n_ctx, void* const* accs,
                 int acc_kind, int num_objects, long long g0, long long g1, fs::AccParts& P) {
    const size_t entry = acc_kind == FS_ACC_FIXED ? 16 : 8;
    const size_t row = (size_t)num_objects * entry;
    const size_t slice = (size_t)(g1 - g0) * row;
    std::vector<int> staged;
    for (int i = 0; i < n_ctx; ++i) {
        if (!accs[i]) return fail(FS_EINVAL, "fs_finalize_multi: NULL accumulator %d", i);
        if (ctxs[i]->device == ctx->device || enable_peer(ctx->device, ctxs[i]->device))
            P.p[i] = accs[i];
        else
            staged.push_back(i);
    }
    if (!staged.empty()) {
        int rc = grow(&ctx->fin_stage, &ctx->fin_stage_cap, staged.size() * slice);
        if (rc) return rc;
        for (size_t k = 0; k < staged.size(); ++k) {
            const int i = staged[k];
            unsigned char* dst = ctx->fin_stage + k * slice;
            CK(cudaMemcpyPeerAsync(dst, ctx->device,
                                   static_cast<const unsigned char*>(accs[i]) + (size_t)g0 * row,
                                   ctxs[i]->device, slice, ctx->work[0].stream));
            P.p[i] = dst - (size_t)g0 * row;  // indexed by absolute Gaussian id
        }
    }
    return FS_OK;
}

// Reduce + cast (+ biased argmax when mode >= 0) of Gaussians [g0, g1) on
// ctx's device.  out: element (0, g0) of an E-row float32 matrix with row
// stride ld (device or host); labels (host, same stride; mode >= 0 only).
int finalize_slice(fs_context* ctx, const fs::AccParts& P, int acc_kind, int num_objects,
                   long long g0, long long g1, float* out, long long ld, int out_on_device,
                   uint8_t* labels, float gamma, int mode) {
    cudaStream_t st = ctx->work[0].stream;
    const long long w = g1 - g0;
    if (mode >= 0 && (out_on_device || !labels))
        return fail(FS_EINVAL, "finalize_slice: labels need a host matrix and label buffer");
    float* dst = out;
    long long dld = ld;
    int rc;
    if (!out_on_device) {
        if ((rc = grow(&ctx->fin_tmp, &ctx->fin_tmp_cap, (size_t)num_objects * w))) return rc;
        dst = ctx->fin_tmp;
        dld = w;
    }
    fs::launch_finalize(P, acc_kind == FS_ACC_FIXED, g0, g1, num_objects, dst, dld, st);
    if (!out_on_device)
        CK(cudaMemcpy2DAsync(out, sizeof(float) * ld, dst, sizeof(float) * w, sizeof(float) * w,
                             num_objects, cudaMemcpyDeviceToHost, st));
    if (mode >= 0) {
        const int rows = mode == FS_MODE_BINARY ? 1 : num_objects;
        if ((rc = grow(&ctx->fin_lab, &ctx->fin_lab_cap, (size_t)rows * w))) return rc;
        fs::launch_assign(dst, w, dld, num_objects, gamma, mode, ctx->fin_lab, st);
        CK(cudaMemcpy2DAsync(labels, ld, ctx->fin_lab, dld, w, rows, cudaMemcpyDeviceToHost, st));
    }
    CK(cudaGetLastError());
    CK(cudaStreamSynchronize(st));
    return FS_OK;
}

}  // namespace

extern "C" {

const char* fs_last_error(void) { return fs::g_error.c_str(); }

const char* fs_version(void) { return "flashsplat-b200 0.1.0 (sm_100a)"; }

int fs_device_count(int* out) {
    int c = 0;
    cudaError_t e = cudaGetDeviceCount(&c);
    if (e != cudaSuccess) {
        cudaGetLastError();
        *out = 0;
        return fs::set_cuda_error(e, "cudaGetDeviceCount", __FILE__, __LINE__);
    }
    *out = c;
    return FS_OK;
}

int fs_create(int device, int n_streams, fs_context** out) {
    if (!out) return fail(FS_EINVAL, "fs_create: out is NULL");
    *out = nullptr;
    if (n_streams < 1) n_streams = 1;
    if (n_streams > 16) n_streams = 16;
    CK(cudaSetDevice(device));
    fs_context* ctx = new fs_context();
    ctx->device = device;
    cudaDeviceProp prop;
    cudaError_t e = cudaGetDeviceProperties(&prop, device);
    if (e != cudaSuccess) {
        delete ctx;
        return fs::set_cuda_error(e, "cudaGetDeviceProperties", __FILE__, __LINE__);
    }
    if (prop.major < 10) {
        delete ctx;
        return fail(FS_ECUDA, "device %d (%s, sm_%d%d) is not sm_100: this library is built for "
                              "B200 (sm_100a) only", device, prop.name, prop.major, prop.minor);
    }
    ctx->num_sms = prop.multiProcessorCount;
    // fs_assign's stream-ordered scratch (cudaMallocAsync) comes from the device's
    // default pool; keep freed blocks there instead of trimming them back at every
    // synchronisation -- re-mapping trimmed memory stalled calls for up to 0.8 s
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, device) == cudaSuccess) {
        unsigned long long keep = ~0ull;
        cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
    }
    e = fs::raster_configure();
    if (e == cudaSuccess) e = fs::bin_configure();
    if (e != cudaSuccess) {
        delete ctx;
        return fs::set_cuda_error(e, "raster_configure", __FILE__, __LINE__);
    }
    ctx->work.resize(n_streams);
    for (auto& w : ctx->work) {
        CK(cudaStreamCreateWithFlags(&w.stream, cudaStreamNonBlocking));
        CK(cudaEventCreateWithFlags(&w.h2d_done, cudaEventDisableTiming));
        CK(cudaEventCreateWithFlags(&w.done, cudaEventDisableTiming));
        CK(cudaEventCreateWithFlags(&w.view_done, cudaEventDisableTiming));
    }
    CK(cudaEventCreateWithFlags(&ctx->ev_caller, cudaEventDisableTiming));
    CK(cudaEventCreate(&ctx->ev_start));
    CK(cudaEventCreate(&ctx->ev_stop));
    *out = ctx;
    return FS_OK;
}

void fs_destroy(fs_context* ctx) {
    if (!ctx) return;
    cudaSetDevice(ctx->device);
    for (auto& w : ctx->work)
        if (w.stream) cudaStreamSynchronize(w.stream);
    for (auto& w : ctx->work) free_work(w);
    for (void* p : {(void*)ctx->mx, (void*)ctx->my, (void*)ctx->mz, (void*)ctx->sig,
                    (void*)ctx->opac, (void*)ctx->view_log,
                    (void*)ctx->up_means, (void*)ctx->up_quats, (void*)ctx->up_scales,
                    (void*)ctx->up_opac, (void*)ctx->perm, ctx->order_scratch,
                    (void*)ctx->rn_f64, (void*)ctx->rn_in, (void*)ctx->rn_member,
                    (void*)ctx->rn_u32, (void*)ctx->rn_labels, (void*)ctx->rn_rect,
                    (void*)ctx->cnt})
        if (p) cudaFree(p);
    for (int k = 0; k < 2; ++k) {
        if (ctx->pinned_up[k]) cudaFreeHost(ctx->pinned_up[k]);
        if (ctx->pinned_free[k]) cudaEventDestroy(ctx->pinned_free[k]);
    }
    for (cudaEvent_t e : ctx->stage_events) cudaEventDestroy(e);
    if (ctx->ev_start) cudaEventDestroy(ctx->ev_start);
    if (ctx->ev_stop) cudaEventDestroy(ctx->ev_stop);
    if (ctx->ev_caller) cudaEventDestroy(ctx->ev_caller);
    for (void* p : {(void*)ctx->fin_tmp, (void*)ctx->fin_lab, (void*)ctx->fin_stage,
                    (void*)ctx->ply_raw, (void*)ctx->ply_bad})
        if (p) cudaFree(p);
    delete ctx;
}

int fs_device_alloc(fs_context* ctx, uint64_t bytes, void** out) {
    if (!ctx || !out) return fail(FS_EINVAL, "fs_device_alloc: NULL argument");
    CK(cudaSetDevice(ctx->device));
    cudaError_t e = cudaMalloc(out, bytes ? bytes : 1);
    if (e != cudaSuccess) {
        cudaGetLastError();
        return fail(FS_ENOMEM, "cudaMalloc of %llu bytes failed", (unsigned long long)bytes);
    }
    return FS_OK;
}

int fs_device_free(fs_context* ctx, void* ptr) {
    if (!ctx) return fail(FS_EINVAL, "fs_device_free: NULL context");
    CK(cudaSetDevice(ctx->device));
    if (ptr) CK(cudaFree(ptr));
    return FS_OK;
}

int fs_memset_zero(fs_context* ctx, void* p, uint64_t bytes) {
    CK(cudaSetDevice(ctx->device));
    cudaStream_t st = ctx->work[0].stream;
    CK(cudaMemsetAsync(p, 0, bytes, st));
    CK(cudaStreamSynchronize(st));
    return FS_OK;
}

int fs_copy_to_device(fs_context* ctx, void* dst, const void* src, uint64_t bytes) {
    CK(cudaSetDevice(ctx->device));
    CK(sync_copy(dst, src, bytes, cudaMemcpyHostToDevice, ctx->work[0].stream));
    return FS_OK;
}

int fs_copy_to_host(fs_context* ctx, void* dst, const void* src, uint64_t bytes) {
    CK(cudaSetDevice(ctx->device));
    CK(sync_copy(dst, src, bytes, cudaMemcpyDeviceToHost, ctx->work[0].stream));
    return FS_OK;
}

int fs_host_alloc(fs_context* ctx, uint64_t bytes, void** out) {
    if (!ctx || !out) return fail(FS_EINVAL, "fs_host_alloc: NULL argument");
    CK(cudaSetDevice(ctx->device));
    cudaError_t e = cudaHostAlloc(out, bytes ? bytes : 1, cudaHostAllocPortable);
    if (e != cudaSuccess) {
        cudaGetLastError();
        return fail(FS_ENOMEM, "cudaHostAlloc of %llu bytes failed", (unsigned long long)bytes);
    }
    return FS_OK;
}

int fs_host_free(fs_context* ctx, void* ptr) {
    if (!ctx) return fail(FS_EINVAL, "fs_host_free: NULL context");
    if (ptr) CK(cudaFreeHost(ptr));
    return FS_OK;
}

int fs_host_pinned(const void* ptr, uint64_t bytes) { return host_pinned(ptr, bytes) ? 1 : 0; }

int fs_synchronize(fs_context* ctx) {
    CK(cudaSetDevice(ctx->device));
    for (auto& w : ctx->work) CK(cudaStreamSynchronize(w.stream));
    return FS_OK;
}

int fs_set_stream(fs_context* ctx, void* stream) {
    if (!ctx) return fail(FS_EINVAL, "fs_set_stream: NULL context");
    ctx->caller_stream = static_cast<cudaStream_t>(stream);
    return FS_OK;
}

int fs_set_timing(fs_context* ctx, int enable) {
    if (!ctx) return fail(FS_EINVAL, "fs_set_timing: NULL context");
    ctx->timing = enable != 0;
    return FS_OK;
}

int fs_copy_scene(fs_context* dst, const fs_context* src) {
    Range nvtx_range("fs_copy_scene");
    if (!dst || !src) return fail(FS_EINVAL, "fs_copy_scene: NULL context");
    if (dst == src) return FS_OK;
    const long long n = src->n;
    CK(cudaSetDevice(dst->device));
    int rc;
    if ((rc = order_after_caller(dst))) return rc;
    if (n > dst->scene_cap) {
        if ((rc = dev_alloc(&dst->mx, n)) || (rc = dev_alloc(&dst->my, n)) ||
            (rc = dev_alloc(&dst->mz, n)) || (rc = dev_alloc(&dst->sig, 6 * (size_t)n)) ||
            (rc = dev_alloc(&dst->opac, n)) || (rc = dev_alloc(&dst->up_means, 3 * (size_t)n)) ||
            (rc = dev_alloc(&dst->up_quats, 4 * (size_t)n)) ||
            (rc = dev_alloc(&dst->up_scales, 3 * (size_t)n)) ||
            (rc = dev_alloc(&dst->up_opac, (size_t)n)) || (rc = dev_alloc(&dst->perm, (size_t)n)))
            return rc;
        dst->scene_cap = n;
    }
    dst->n = 0;
    if (n > 0) {
        // the source is resident (its setup call host-synchronised); device -> device over
        // NVLink when the contexts sit on different GPUs
        cudaStream_t st = dst->work[0].stream;
        const double* s_arr[5] = {src->mx, src->my, src->mz, src->sig, src->opac};
        double* d_arr[5] = {dst->mx, dst->my, dst->mz, dst->sig, dst->opac};
        const size_t cnt[5] = {(size_t)n, (size_t)n, (size_t)n, 6 * (size_t)n, (size_t)n};
        for (int k = 0; k < 5; ++k)
            CK(cudaMemcpyPeerAsync(d_arr[k], dst->device, s_arr[k], src->device,
                                   sizeof(double) * cnt[k], st));
        if (src->perm_on)
            CK(cudaMemcpyPeerAsync(dst->perm, dst->device, src->perm, src->device,
                                   sizeof(unsigned int) * (size_t)n, st));
        CK(cudaStreamSynchronize(st));
    }
    dst->perm_on = src->perm_on;
    dst->n = n;
    return FS_OK;
}

int fs_set_scene(fs_context* ctx, int64_t n, const double* means, const double* quats,
                 const double* scales, const double* opacities) {
    Range nvtx_range("fs_set_scene");
    if (!ctx) return fail(FS_EINVAL, "fs_set_scene: NULL context");
    if (n < 0 || n > 0x7fffffffLL) return fail(FS_EINVAL, "fs_set_scene: bad Gaussian count %lld", (long long)n);
    if (n > 0 && (!means || !quats || !scales || !opacities))
        return fail(FS_EINVAL, "fs_set_scene: NULL array");
    CK(cudaSetDevice(ctx->device));
    int rc;
    if ((rc = order_after_caller(ctx))) return rc;
    if (n > ctx->scene_cap) {
        if ((rc = dev_alloc(&ctx->mx, n)) || (rc = dev_alloc(&ctx->my, n)) ||
            (rc = dev_alloc(&ctx->mz, n)) || (rc = dev_alloc(&ctx->sig, 6 * (size_t)n)) ||
            (rc = dev_alloc(&ctx->opac, n)) || (rc = dev_alloc(&ctx->up_means, 3 * (size_t)n)) ||
            (rc = dev_alloc(&ctx->up_quats, 4 * (size_t)n)) ||
            (rc = dev_alloc(&ctx->up_scales, 3 * (size_t)n)) ||
            (rc = dev_alloc(&ctx->up_opac, (size_t)n)) || (rc = dev_alloc(&ctx->perm, (size_t)n)))
            return rc;
        ctx->scene_cap = n;
    }
    ctx->n = n;
    if (n == 0) return FS_OK;
    cudaStream_t st = ctx->work[0].stream;
    if ((rc = upload(ctx, ctx->up_means, means, 24 * (size_t)n, st)) ||
        (rc = upload(ctx, ctx->up_quats, quats, 32 * (size_t)n, st)) ||
        (rc = upload(ctx, ctx->up_scales, scales, 24 * (size_t)n, st)) ||
        (rc = upload(ctx, ctx->up_opac, opacities, 8 * (size_t)n, st)))
        return rc;
    ctx->perm_on = scene_order_enabled();
    if (ctx->perm_on) {
        if ((rc = ensure_order_scratch(ctx, n))) return rc;
        CK(fs::launch_scene_order((int)n, ctx->up_means, ctx->perm, ctx->order_scratch,
                                  ctx->order_scratch_bytes, ctx->num_sms, st));
    }
    fs::launch_scene_setup((int)n, ctx->up_means, ctx->up_quats, ctx->up_scales, ctx->up_opac,
                           scene_perm(ctx), ctx->mx, ctx->my, ctx->mz, ctx->sig, ctx->opac, st);
    CK(cudaGetLastError());
    CK(cudaStreamSynchronize(st));
    return FS_OK;
}

int fs_set_scene_ply(fs_context* ctx, int64_t n, const void* verts, int stride_floats,
                     const int32_t* offsets, int64_t* bad, double* params) {
    Range nvtx_range("fs_set_scene_ply");
    if (!ctx || !offsets || !bad) return fail(FS_EINVAL, "fs_set_scene_ply: NULL argument");
    if (n < 0 || n > 0x7fffffffLL) return fail(FS_EINVAL, "fs_set_scene_ply: bad vertex count %lld", (long long)n);
    if (n > 0 && !verts) return fail(FS_EINVAL, "fs_set_scene_ply: NULL vertex block");
    fs::PlyOffsets off;
    for (int k = 0; k < fs::kPlyProps; ++k) {
        if (offsets[k] < 0 || offsets[k] >= stride_floats)
            return fail(FS_EINVAL, "fs_set_scene_ply: property offset %d outside the %d-float record",
                        offsets[k], stride_floats);
        off.k[k] = offsets[k];
    }
    for (int k = 0; k < 4; ++k) bad[k] = -1;
    CK(cudaSetDevice(ctx->device));
    int rc;
    if ((rc = order_after_caller(ctx))) return rc;
    ctx->n = 0;  // not resident until validated
    if (n > ctx->scene_cap) {
        if ((rc = dev_alloc(&ctx->mx, n)) || (rc = dev_alloc(&ctx->my, n)) ||
            (rc = dev_alloc(&ctx->mz, n)) || (rc = dev_alloc(&ctx->sig, 6 * (size_t)n)) ||
            (rc = dev_alloc(&ctx->opac, n)) || (rc = dev_alloc(&ctx->up_means, 3 * (size_t)n)) ||
            (rc = dev_alloc(&ctx->up_quats, 4 * (size_t)n)) ||
            (rc = dev_alloc(&ctx->up_scales, 3 * (size_t)n)) ||
            (rc = dev_alloc(&ctx->up_opac, (size_t)n)) || (rc = dev_alloc(&ctx->perm, (size_t)n)))
            return rc;
        ctx->scene_cap = n;
    }
    if (n == 0) return FS_OK;
    const size_t bytes = (size_t)n * stride_floats * sizeof(float);
    if ((rc = grow(&ctx->ply_raw, &ctx->ply_raw_cap, bytes / sizeof(float)))) return rc;
    if (!ctx->ply_bad && (rc = dev_alloc(&ctx->ply_bad, 4))) return rc;
    cudaStream_t st = ctx->work[0].stream;
    // the records as the file stores them: one DMA (pinned) or the staged
    // ring, no host-side column gather or activation
    if ((rc = upload(ctx, ctx->ply_raw, verts, bytes, st))) return rc;
    CK(cudaMemsetAsync(ctx->ply_bad, 0xff, 4 * sizeof(unsigned long long), st));
    double* dparams = nullptr;
    if (params) CK(cudaMallocAsync(reinterpret_cast<void**>(&dparams), 64 * (size_t)n, st));
    ctx->perm_on = scene_order_enabled();
    if (ctx->perm_on) {
        if ((rc = ensure_order_scratch(ctx, n))) return rc;
        CK(fs::launch_scene_order_ply((int)n, ctx->ply_raw, stride_floats, off, ctx->perm,
                                      ctx->order_scratch, ctx->order_scratch_bytes, ctx->num_sms,
                                      st));
    }
    fs::launch_scene_setup_ply((int)n, ctx->ply_raw, stride_floats, off, scene_perm(ctx), ctx->mx,
                               ctx->my, ctx->mz, ctx->sig, ctx->opac, ctx->ply_bad, dparams, st);
    CK(cudaGetLastError());
    if (params) {
        CK(sync_copy(params, dparams, 64 * (size_t)n, cudaMemcpyDeviceToHost, st));
        CK(cudaFreeAsync(dparams, st));
    }
    unsigned long long b[4];
    CK(sync_copy(b, ctx->ply_bad, sizeof(b), cudaMemcpyDeviceToHost, st));
    bool any = false;
    for (int k = 0; k < 4; ++k) {
        bad[k] = b[k] == ~0ull ? -1 : (int64_t)b[k];
        any |= bad[k] >= 0;
    }
    if (any)
        return fail(FS_EINVAL, "fs_set_scene_ply: invalid vertices (first non-finite %lld, "
                               "quaternion %lld, scale %lld, opacity %lld)", (long long)bad[0],
                    (long long)bad[1], (long long)bad[2], (long long)bad[3]);
    ctx->n = n;
    return FS_OK;
}

int fs_project(fs_context* ctx, const fs_camera* cam, uint8_t* alive, double* mean2d,
               double* conic, double* depth, int64_t* radius, fs_projection_stats* stats) {
    Range nvtx_range("fs_project");
    if (!ctx || !cam || !alive) return fail(FS_EINVAL, "fs_project: NULL argument");
    int rc = check_cam(*cam, 0);
    if (rc) return rc;
    CK(cudaSetDevice(ctx->device));
    fs::Work& w = ctx->work[0];
    const long long n = ctx->n;
    if ((rc = ensure_work(ctx, w, n, 1, 1, 1))) return rc;
    fs::ProjectExport ex{};
    size_t n1 = (size_t)std::max<long long>(n, 1);
    if ((rc = dev_alloc(&ex.alive, n1)) || (rc = dev_alloc(&ex.mean2d, 2 * n1)) ||
        (rc = dev_alloc(&ex.conic, 3 * n1)) || (rc = dev_alloc(&ex.depth, n1)) ||
        (rc = dev_alloc(&ex.radius, n1)))
        return rc;
    ex.perm = scene_perm(ctx);
    fs::launch_project((int)n, ctx->mx, ctx->my, ctx->mz, ctx->sig, ctx->opac, to_cam(*cam), 0.0,
                       0, w.k64, w.rect, w.r32, w.r64, w.vc, ex,
                       ctx->num_sms, w.stream);
    CK(cudaGetLastError());
    CK(cudaStreamSynchronize(w.stream));
    CK(sync_copy(alive, ex.alive, (size_t)n, cudaMemcpyDeviceToHost, w.stream));
    if (mean2d) CK(sync_copy(mean2d, ex.mean2d, 16 * (size_t)n, cudaMemcpyDeviceToHost, w.stream));
    if (conic) CK(sync_copy(conic, ex.conic, 24 * (size_t)n, cudaMemcpyDeviceToHost, w.stream));
    if (depth) CK(sync_copy(depth, ex.depth, 8 * (size_t)n, cudaMemcpyDeviceToHost, w.stream));
    if (radius) CK(sync_copy(radius, ex.radius, 8 * (size_t)n, cudaMemcpyDeviceToHost, w.stream));
    if (stats) {
        fs::ViewCounters vc;
        CK(sync_copy(&vc, w.vc, sizeof(vc), cudaMemcpyDeviceToHost, w.stream));
        stats->n_input = n;
        stats->n_emitted = vc.n_emitted;
        stats->n_behind = vc.n_behind;
        stats->n_degenerate = vc.n_degenerate;
        stats->n_offscreen = vc.n_offscreen;
    }
    cudaFree(ex.alive);
    cudaFree(ex.mean2d);
    cudaFree(ex.conic);
    cudaFree(ex.depth);
    cudaFree(ex.radius);
    return FS_OK;
}

// Copies the (sorted) tile lists of workspace w to the host as CSR.
static int copy_tile_lists(fs::Work& w, int ntiles, unsigned int n_valid, int64_t* tile_offsets,
                           int64_t* items, int64_t items_capacity, int64_t* n_items) {
    std::vector<unsigned int> starts(ntiles + 1);
    CK(sync_copy(starts.data(), w.tile_start, sizeof(unsigned int) * (ntiles + 1), cudaMemcpyDeviceToHost, w.stream));
    for (int t = 0; t <= ntiles; ++t) tile_offsets[t] = starts[t];
    *n_items = n_valid;
    if (items) {
        if (items_capacity < (int64_t)n_valid) return fail(FS_EINVAL, "fs_bin: items buffer too small");
        // bucket t's gids sit in the first half of its instance bytes (sorted_view)
        std::vector<unsigned long long> g(n_valid);
        if (n_valid) CK(sync_copy(g.data(), w.inst, sizeof(unsigned long long) * n_valid, cudaMemcpyDeviceToHost, w.stream));
        for (int t = 0; t < ntiles; ++t) {
            const unsigned int* v = fs::sorted_view(g.data(), starts[t]);
            for (unsigned int i = starts[t]; i < starts[t + 1]; ++i) items[i] = v[i - starts[t]];
        }
    }
    return FS_OK;
}

int fs_bin(fs_context* ctx, const fs_camera* cam, int64_t* tile_offsets, int64_t* items,
           int64_t items_capacity, int64_t* n_items) {
    Range nvtx_range("fs_bin");
    if (!ctx || !cam || !tile_offsets || !n_items) return fail(FS_EINVAL, "fs_bin: NULL argument");
    int rc = check_cam(*cam, 0);
    if (rc) return rc;
    CK(cudaSetDevice(ctx->device));
    fs::Work& w = ctx->work[0];
    const fs::Camera k = to_cam(*cam);
    const int ntiles = fs::tiles_x_of(k.width) * fs::tiles_y_of(k.height);
    unsigned int cap = std::max(w.inst_cap, initial_inst_cap(ctx->n));
    fs::ViewCounters vc;
    for (int attempt = 0; attempt < 2; ++attempt) {
        if ((rc = ensure_work(ctx, w, ctx->n, ntiles, cap, 1))) return rc;
        enqueue_bin(ctx, w, k, 0.0, 0, fs::ProjectExport{});
        fs::launch_tile_sort(ntiles, tile_sort_args(w, scene_perm(ctx)), w.stream);
        CK(cudaGetLastError());
        CK(cudaStreamSynchronize(w.stream));
        CK(sync_copy(&vc, w.vc, sizeof(vc), cudaMemcpyDeviceToHost, w.stream));
        if (!vc.overflow) break;
        cap = (unsigned int)std::min<unsigned long long>(0x7fffffffull, (unsigned long long)vc.n_instances + 1024);
    }
    if (vc.overflow) return fail(FS_ENOMEM, "fs_bin: instance buffer overflow");
    if ((rc = copy_tile_lists(w, ntiles, vc.n_valid, tile_offsets, items, items_capacity, n_items)))
        return rc;
    if (items && scene_perm(ctx) && vc.n_valid) {  // slots -> input ids
        std::vector<unsigned int> perm((size_t)ctx->n);
        CK(sync_copy(perm.data(), ctx->perm, sizeof(unsigned int) * perm.size(),
                     cudaMemcpyDeviceToHost, w.stream));
        for (unsigned int i = 0; i < vc.n_valid; ++i) items[i] = perm[(size_t)items[i]];
    }
    return FS_OK;
}

int fs_bin_splats(fs_context* ctx, int64_t k, const double* mean2d, const double* depth,
                  const int64_t* radius, const int64_t* index, int width, int height,
                  int64_t* tile_offsets, int64_t* items, int64_t items_capacity, int64_t* n_items) {
    if (!ctx || !tile_offsets || !n_items || (k > 0 && (!mean2d || !depth || !radius || !index)))
        return fail(FS_EINVAL, "fs_bin_splats: NULL argument");
    if (k < 0 || k > 0x7fffffffLL) return fail(FS_EINVAL, "fs_bin_splats: bad splat count");
    fs_camera c{};
    c.width = width;
    c.height = height;
    int rc = check_cam(c, 0);
    if (rc) return rc;
    CK(cudaSetDevice(ctx->device));
    fs::Work& w = ctx->work[0];
    const int tx = fs::tiles_x_of(width), ntiles = tx * fs::tiles_y_of(height);
    unsigned int cap = std::max(w.inst_cap, initial_inst_cap(k));
    std::vector<unsigned int> tie((size_t)std::max<int64_t>(k, 0));
    for (int64_t i = 0; i < k; ++i) {
        if (index[i] < 0 || index[i] > 0xffffffffLL)
            return fail(FS_EINVAL, "fs_bin_splats: gaussian_index %lld out of range", (long long)index[i]);
        tie[i] = (unsigned int)index[i];
    }
    double *d_mean = nullptr, *d_depth = nullptr;
    long long* d_rad = nullptr;
    const size_t k1 = (size_t)std::max<int64_t>(k, 1);
    if ((rc = dev_alloc(&d_mean, 2 * k1)) || (rc = dev_alloc(&d_depth, k1)) ||
        (rc = dev_alloc(&d_rad, k1)))
        return rc;
    if (k > 0) {
        CK(sync_copy(d_mean, mean2d, 16 * (size_t)k, cudaMemcpyHostToDevice, w.stream));
        CK(sync_copy(d_depth, depth, 8 * (size_t)k, cudaMemcpyHostToDevice, w.stream));
        CK(sync_copy(d_rad, radius, 8 * (size_t)k, cudaMemcpyHostToDevice, w.stream));
    }
    fs::ViewCounters vc{};
    for (int attempt = 0; attempt < 2; ++attempt) {
        if ((rc = ensure_work(ctx, w, std::max<long long>(k, 1), ntiles, cap, 1))) return rc;
        fs::launch_view_begin(w.vc, w.stream);
        if (k > 0)
            CK(cudaMemcpyAsync(w.tie, tie.data(), sizeof(unsigned int) * (size_t)k,
                               cudaMemcpyHostToDevice, w.stream));
        fs::launch_splat_keys((int)k, d_mean, d_rad, d_depth, width, height, w.rect, w.k64, w.vc,
                              ctx->num_sms, w.stream);
        fs::launch_bin(ntiles, tx, bin_buffers(w, (int)k), w.vc, ctx->num_sms, w.stream);
        fs::launch_tile_sort(ntiles, tile_sort_args(w, w.tie), w.stream);
        CK(cudaGetLastError());
        CK(cudaStreamSynchronize(w.stream));
        CK(sync_copy(&vc, w.vc, sizeof(vc), cudaMemcpyDeviceToHost, w.stream));
        if (!vc.overflow) break;
        cap = (unsigned int)std::min<unsigned long long>(0x7fffffffull, (unsigned long long)vc.n_instances + 1024);
    }
    cudaFree(d_mean);
    cudaFree(d_depth);
    cudaFree(d_rad);
    if (vc.overflow) return fail(FS_ENOMEM, "fs_bin_splats: instance buffer overflow");
    return copy_tile_lists(w, ntiles, vc.n_valid, tile_offsets, items, items_capacity, n_items);
}

int fs_accumulate(fs_context* ctx, int n_views, const fs_camera* cams, const uint16_t* const* masks,
                  int masks_on_device, int num_objects, double alpha_floor, double t_floor,
                  int acc_kind, void* acc, fs_accumulate_stats* stats) {
    Range nvtx_range("fs_accumulate");
    if (!ctx) return fail(FS_EINVAL, "fs_accumulate: NULL context");
    if (stats) {
        memset(stats, 0, sizeof(*stats));
        stats->label_error_view = -1;
    }
    int rc;
    ViewPlan plan;
    if ((rc = plan_views(n_views, cams, masks, num_objects, acc_kind, plan))) return rc;
    if (!acc && ctx->n > 0) return fail(FS_EINVAL, "fs_accumulate: NULL accumulator");
    if (n_views == 0 || ctx->n == 0) return FS_OK;
    CtxRun R;
    if ((rc = accumulate_on(ctx, plan, cams, masks, masks_on_device, num_objects, alpha_floor,
                            t_floor, acc_kind, acc, nullptr, R)))
        return rc;
    return finish_stats(&R, 1, plan, num_objects, stats);
}

int fs_accumulate_multi(fs_context* const* ctxs, int n_ctx, int n_views, const fs_camera* cams,
                        const uint16_t* const* masks, int num_objects, double alpha_floor,
                        double t_floor, int acc_kind, void* const* accs, int32_t* view_ctx,
                        fs_accumulate_stats* stats) {
    Range nvtx_range("fs_accumulate_multi");
    if (!ctxs || n_ctx < 1 || n_ctx > fs::kMaxParts || !accs)
        return fail(FS_EINVAL, "fs_accumulate_multi: need 1..%d contexts and accumulators",
                    fs::kMaxParts);
    if (stats) {
        memset(stats, 0, sizeof(*stats));
        stats->label_error_view = -1;
    }
    for (int i = 0; i < n_ctx; ++i)
        for (int j = 0; j < i; ++j)
            if (ctxs[i] == ctxs[j])
                return fail(FS_EINVAL, "fs_accumulate_multi: context %d is listed twice (one host "
                                       "thread per context: use distinct contexts)", i);
    int rc;
    ViewPlan plan;
    if ((rc = plan_views(n_views, cams, masks, num_objects, acc_kind, plan))) return rc;
    const long long n = ctxs[0]->n;
    for (int i = 0; i < n_ctx; ++i) {
        if (!ctxs[i]) return fail(FS_EINVAL, "fs_accumulate_multi: NULL context %d", i);
        if (ctxs[i]->n != n)
            return fail(FS_EINVAL, "fs_accumulate_multi: context %d holds %lld Gaussians, context 0 "
                                   "%lld (upload the same scene to every context)", i,
                        (long long)ctxs[i]->n, n);
        if (!accs[i] && n > 0) return fail(FS_EINVAL, "fs_accumulate_multi: NULL accumulator %d", i);
    }
    if (n_views == 0 || n == 0) return FS_OK;
    // dynamic queue: every host thread pops the next view when one of its
    // context's streams frees up, so faster GPUs take more views
    std::atomic<int> next(0);
    std::vector<CtxRun> R(n_ctx);
    std::vector<int> codes(n_ctx, FS_OK);
    std::vector<std::string> errs(n_ctx);
    std::vector<std::thread> threads;
    for (int i = 0; i < n_ctx; ++i)
        threads.emplace_back([&, i] {
            codes[i] = accumulate_on(ctxs[i], plan, cams, masks, 0, num_objects, alpha_floor,
                                     t_floor, acc_kind, accs[i], &next, R[i]);
            if (codes[i]) errs[i] = fs::g_error;
        });
    for (auto& t : threads) t.join();
    for (int i = 0; i < n_ctx; ++i)
        if (codes[i]) return fail(codes[i], "%s", errs[i].c_str());
    if (view_ctx)
        for (int i = 0; i < n_ctx; ++i)
            for (int v : R[i].views) view_ctx[v] = i;
    return finish_stats(R.data(), n_ctx, plan, num_objects, stats);
}

int fs_enable_peer_access(fs_context* ctx, int peer_device) {
    if (!ctx) return fail(FS_EINVAL, "fs_enable_peer_access: NULL context");
    return enable_peer(ctx->device, peer_device) ? FS_OK
                                                 : fail(FS_ECUDA, "no peer access from device %d to %d",
                                                        ctx->device, peer_device);
}

int fs_reduce_finalize(fs_context* ctx, int acc_kind, const void* const* parts, int n_parts,
                       int64_t part_g0, int64_t n, int num_objects, int64_t g0, int64_t g1,
                       float* out, int64_t ld, int out_on_device) {
    Range nvtx_range("fs_reduce_finalize");
    if (!ctx) return fail(FS_EINVAL, "fs_reduce_finalize: NULL context");
    if (acc_kind != FS_ACC_F64 && acc_kind != FS_ACC_FIXED)
        return fail(FS_EINVAL, "bad accumulator kind %d", acc_kind);
    if (n < 0 || num_objects < 0 || g0 < 0 || g1 > n || g0 > g1 || part_g0 > g0)
        return fail(FS_EINVAL, "fs_reduce_finalize: bad range");
    if (n_parts < 1 || n_parts > fs::kMaxParts || !parts)
        return fail(FS_EINVAL, "fs_reduce_finalize: need 1..%d parts", fs::kMaxParts);
    if (g1 == g0 || num_objects == 0) return FS_OK;
    if (!out) return fail(FS_EINVAL, "fs_reduce_finalize: NULL output");
    if (ld < g1 - g0) return fail(FS_EINVAL, "fs_reduce_finalize: row stride %lld < slice width %lld",
                                  (long long)ld, (long long)(g1 - g0));
    CK(cudaSetDevice(ctx->device));
    int rc;
    if ((rc = order_after_caller(ctx))) return rc;
    fs::AccParts P{};
    P.n = n_parts;
    const size_t entry = acc_kind == FS_ACC_FIXED ? 16 : 8;
    for (int i = 0; i < n_parts; ++i) {
        if (!parts[i]) return fail(FS_EINVAL, "fs_reduce_finalize: NULL part %d", i);
        // element (g, l) of a part lives at (g - part_g0) * E + l
        P.p[i] = static_cast<const unsigned char*>(parts[i]) -
                 (size_t)part_g0 * num_objects * entry;
    }
    return finalize_slice(ctx, P, acc_kind, num_objects, g0, g1, out, ld, out_on_device, nullptr,
                          0.0f, -1);
}

int fs_finalize(fs_context* ctx, int acc_kind, const void* acc, int64_t n, int num_objects,
                float* out, int out_on_device) {
    return fs_reduce_finalize(ctx, acc_kind, &acc, 1, 0, n, num_objects, 0, n, out, n,
                              out_on_device);
}

int fs_finalize_multi(fs_context* const* ctxs, int n_ctx, int acc_kind, void* const* accs,
                      int64_t n, int num_objects, float* out, float gamma, int mode,
                      uint8_t* labels) {
    Range nvtx_range("fs_finalize_multi");
    if (!ctxs || n_ctx < 1 || n_ctx > fs::kMaxParts || !accs)
        return fail(FS_EINVAL, "fs_finalize_multi: need 1..%d contexts and accumulators",
                    fs::kMaxParts);
    if (acc_kind != FS_ACC_F64 && acc_kind != FS_ACC_FIXED)
        return fail(FS_EINVAL, "bad accumulator kind %d", acc_kind);
    if (mode != -1 && mode != FS_MODE_BINARY && mode != FS_MODE_SCENE)
        return fail(FS_EINVAL, "fs_finalize_multi: bad mode %d", mode);
    if (mode == FS_MODE_BINARY && num_objects != 2)
        return fail(FS_EINVAL, "binary assignment requires E=2, got E=%d", num_objects);
    if (mode == FS_MODE_SCENE && num_objects < 2)
        return fail(FS_EINVAL, "scene assignment requires E>=2, got E=%d", num_objects);
    if (mode != -1 && !(gamma >= -1.0f && gamma <= 1.0f))
        return fail(FS_EINVAL, "gamma must lie in [-1, 1], got %g", (double)gamma);
    for (int i = 0; i < n_ctx; ++i)
        for (int j = 0; j < i; ++j)
            if (ctxs[i] == ctxs[j])
                return fail(FS_EINVAL, "fs_finalize_multi: context %d is listed twice", i);
    if (n <= 0 || num_objects <= 0) return FS_OK;
    if (!out || (mode != -1 && !labels)) return fail(FS_EINVAL, "fs_finalize_multi: NULL output");
    // Column slice i of A is reduced, cast and argmax'ed on context i, reading
    // the other contexts' accumulators over NVLink peer memory: a reduce-scatter
    // fused into the finalize, then one D2H per slice straight into the host
    // matrix (no gather: the host is the destination).
    std::vector<int> codes(n_ctx, FS_OK);
    std::vector<std::string> errs(n_ctx);
    std::vector<std::thread> threads;
    for (int i = 0; i < n_ctx; ++i)
        threads.emplace_back([&, i] {
            fs_context* ctx = ctxs[i];
            const long long base = n / n_ctx, extra = n % n_ctx;
            const long long g0 = i * base + std::min<long long>(i, extra);
            const long long g1 = g0 + base + (i < extra ? 1 : 0);
            int rc = cudaSetDevice(ctx->device) == cudaSuccess ? FS_OK : FS_ECUDA;
            if (!rc) rc = order_after_caller(ctx);
            if (!rc && g1 > g0) {
                fs::AccParts P{};
                P.n = n_ctx;
                rc = gather_parts(ctx, ctxs, n_ctx, accs, acc_kind, num_objects, g0, g1, P);
                if (!rc)
                    rc = finalize_slice(ctx, P, acc_kind, num_objects, g0, g1, out + g0, n, 0,
                                        labels ? labels + g0 : nullptr, gamma, mode);
            }
            codes[i] = rc;
            if (rc) errs[i] = fs::g_error.empty() ? "CUDA error in fs_finalize_multi" : fs::g_error;
        });
    for (auto& t : threads) t.join();
    for (int i = 0; i < n_ctx; ++i)
        if (codes[i]) return fail(codes[i], "%s", errs[i].c_str());
    return FS_OK;
}

int fs_assign(fs_context* ctx, const float* A, int64_t n, int num_objects, float gamma, int mode,
              uint8_t* out, int on_device) {
    Range nvtx_range("fs_assign");
    if ((!A || !out) && n > 0) return fail(FS_EINVAL, "fs_assign: NULL argument");
    if (mode != FS_MODE_BINARY && mode != FS_MODE_SCENE) return fail(FS_EINVAL, "fs_assign: bad mode %d", mode);
    if (mode == FS_MODE_BINARY && num_objects != 2)
        return fail(FS_EINVAL, "binary assignment requires E=2, got E=%d", num_objects);
    if (mode == FS_MODE_SCENE && num_objects < 2)
        return fail(FS_EINVAL, "scene assignment requires E>=2, got E=%d", num_objects);
    if (!(gamma >= -1.0f && gamma <= 1.0f)) return fail(FS_EINVAL, "gamma must lie in [-1, 1], got %g", (double)gamma);
    if (n <= 0) return FS_OK;
    if (ctx) CK(cudaSetDevice(ctx->device));
    // Reentrant: the calling thread's default stream and stream-ordered
    // scratch (cudaMallocAsync pools), no context state -- the service's
    // thread pool calls this concurrently, also while an accumulation runs.
    cudaStream_t st = cudaStreamPerThread;
    const size_t in_bytes = sizeof(float) * (size_t)num_objects * n;
    const size_t out_bytes = (mode == FS_MODE_BINARY ? 1 : (size_t)num_objects) * n;
    const float* dA = A;
    uint8_t* dout = out;
    void *tmpA = nullptr, *tmpO = nullptr;
    if (!on_device) {
        CK(cudaMallocAsync(&tmpA, in_bytes, st));
        CK(cudaMallocAsync(&tmpO, out_bytes, st));
        CK(cudaMemcpyAsync(tmpA, A, in_bytes, cudaMemcpyHostToDevice, st));
        dA = static_cast<const float*>(tmpA);
        dout = static_cast<uint8_t*>(tmpO);
    }
    fs::launch_assign(dA, n, n, num_objects, gamma, mode, dout, st);
    CK(cudaGetLastError());
    if (!on_device) {
        CK(cudaMemcpyAsync(out, dout, out_bytes, cudaMemcpyDeviceToHost, st));
        CK(cudaFreeAsync(tmpA, st));
        CK(cudaFreeAsync(tmpO, st));
    }
    CK(cudaStreamSynchronize(st));
    return FS_OK;
}

int fs_member_counts(fs_context* ctx, const uint8_t* m, int64_t n, int rows, int64_t* counts) {
    Range nvtx_range("fs_member_counts");
    if (!ctx || !counts || (!m && n > 0 && rows > 0)) return fail(FS_EINVAL, "fs_member_counts: NULL argument");
    if (n < 0 || rows < 0) return fail(FS_EINVAL, "fs_member_counts: bad shape");
    if (rows == 0) return FS_OK;
    CK(cudaSetDevice(ctx->device));
    int rc = grow(&ctx->cnt, &ctx->cnt_cap, (size_t)rows);
    if (rc) return rc;
    cudaStream_t st = cudaStreamPerThread;
    CK(cudaMemsetAsync(ctx->cnt, 0, sizeof(unsigned long long) * rows, st));
    fs::launch_row_counts(m, n, rows, ctx->cnt, st);
    CK(cudaGetLastError());
    CK(cudaMemcpyAsync(counts, ctx->cnt, sizeof(int64_t) * rows, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    return FS_OK;
}

}  // extern "C"

// ---------------------------------------------------------------- rendering
namespace {

// perm: the scene's slot -> input id map (scene renders), nullptr for splat lists
fs::RasterArgs render_args(fs::Work& w, int width, int height, double alpha_floor,
                           double t_floor, double* out, int channels, const double* ch_dev,
                           long long n_ids, const unsigned int* perm = nullptr) {
    const int tx = fs::tiles_x_of(width), ntiles = tx * fs::tiles_y_of(height);
    const size_t px = (size_t)width * height;
    fs::RasterArgs ra{};
    ra.width = width;
    ra.height = height;
    ra.tiles_x = tx;
    ra.ntiles = ntiles;
    ra.num_objects = 1;
    ra.n_gaussians = n_ids;  // gids index the records / channel
    ra.af_eff = alpha_floor > 0.0 ? alpha_floor : -1.0;  // rasterizer.py:181-182
    ra.tf_eff = t_floor > 0.0 ? t_floor : -1.0;          // rasterizer.py:193-194
    ra.sort = tile_sort_args(w, perm);
    ra.r32 = w.r32;
    ra.r64 = w.r64;
    ra.vc = w.vc;
    ra.tile_order = w.tile_order;
    ra.render.alpha = out;
    ra.render.depth = out + px;
    ra.render.value = channels ? out + 2 * px : nullptr;
    ra.render.channel = ch_dev;
    ra.render.channels = channels;
    return ra;
}

// render_view / render_subset_alpha_depth over the resident scene into the
// device buffer out = alpha | depth | value (zeroed here).  Re-runs the view
// with larger buckets on instance overflow.
int render_scene_device(fs_context* ctx, const fs_camera* cam, const uint8_t* member_dev,
                        double alpha_floor, double t_floor, const double* ch_dev, int channels,
                        double* out) {
    fs::Work& w = ctx->work[0];
    const int tx = fs::tiles_x_of(cam->width), ntiles = tx * fs::tiles_y_of(cam->height);
    const size_t px = (size_t)cam->width * cam->height;
    unsigned int cap = std::max(w.inst_cap, initial_inst_cap(ctx->n));
    int rc;
    for (int attempt = 0; attempt < 2; ++attempt) {
        if ((rc = ensure_work(ctx, w, std::max<long long>(ctx->n, 1), ntiles, cap, 1))) return rc;
        CK(cudaMemsetAsync(out, 0, sizeof(double) * px * (2 + (size_t)channels), w.stream));
        fs::ProjectExport ex{};
        ex.member = member_dev;
        enqueue_bin(ctx, w, to_cam(*cam), alpha_floor, 1, ex);
        fs::launch_raster_render(render_args(w, cam->width, cam->height, alpha_floor, t_floor, out,
                                             channels, ch_dev, ctx->n, scene_perm(ctx)),
                                 w.stream);
        CK(cudaGetLastError());
        fs::ViewCounters vc{};
        CK(cudaMemcpyAsync(&vc, w.vc, sizeof(vc), cudaMemcpyDeviceToHost, w.stream));
        CK(cudaStreamSynchronize(w.stream));
        if (!vc.overflow) return FS_OK;
        cap = (unsigned int)std::min<unsigned long long>(0x7fffffffull,
                                                         (unsigned long long)vc.n_instances + 1024);
    }
    return fail(FS_ENOMEM, "fs_render: instance buffer overflow");
}

// labels[p] = obj where alpha > tau and depth beats the best so far (strict <:
// ties keep the smaller object id); label 0 <=> best depth still +inf
// (maskrender.py:88-93)
__global__ void mask_combine_kernel(const double* __restrict__ alpha,
                                    const double* __restrict__ depth, long long px, double tau,
                                    unsigned int obj, uint16_t* __restrict__ labels,
                                    double* __restrict__ best) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < px;
         i += (long long)gridDim.x * blockDim.x) {
        const double d = depth[i];
        if (alpha[i] > tau && (labels[i] == 0 || d < best[i])) {
            labels[i] = (uint16_t)obj;
            best[i] = d;
        }
    }
}

// Tile rectangles of one object's members (the others are never binned, like
// project_scene(member_mask=...), scene.py:346-350).
__global__ void member_rect_kernel(const unsigned long long* __restrict__ all,
                                   const uint8_t* __restrict__ member,
                                   const unsigned int* __restrict__ perm, long long n,
                                   unsigned long long* __restrict__ rect) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x)
        rect[i] = member[perm ? perm[i] : i] ? all[i] : ~0ull;  // member is by input id
}

int check_render_cam(const fs_camera* cam) { return check_cam(*cam, 0); }

}  // namespace

extern "C" {

int fs_render(fs_context* ctx, const fs_camera* cam, const uint8_t* member, double alpha_floor,
              double transmittance_floor, const double* channel, int channels, double* value,
              double* alpha, double* depth) {
    Range nvtx_range("fs_render");
    if (!ctx || !cam || !alpha || !depth) return fail(FS_EINVAL, "fs_render: NULL argument");
    if (channels != 0 && channels != 1 && channels != 3)
        return fail(FS_EINVAL, "fs_render: channels must be 0, 1 or 3, got %d", channels);
    if (channels && (!channel || !value)) return fail(FS_EINVAL, "fs_render: NULL channel/value");
    int rc = check_render_cam(cam);
    if (rc) return rc;
    CK(cudaSetDevice(ctx->device));
    if ((rc = order_after_caller(ctx))) return rc;
    fs::Work& w = ctx->work[0];
    const size_t px = (size_t)cam->width * cam->height, n = (size_t)std::max<long long>(ctx->n, 0);
    if ((rc = grow(&ctx->rn_f64, &ctx->rn_f64_cap, px * (2 + (size_t)channels)))) return rc;
    const double* ch_dev = nullptr;
    if (channels && n) {
        if ((rc = grow(&ctx->rn_in, &ctx->rn_in_cap, n * channels))) return rc;
        if ((rc = upload(ctx, ctx->rn_in, channel, sizeof(double) * n * channels, w.stream))) return rc;
        ch_dev = ctx->rn_in;
    }
    const uint8_t* member_dev = nullptr;
    if (member && n) {
        if ((rc = grow(&ctx->rn_member, &ctx->rn_member_cap, n))) return rc;
        if ((rc = upload(ctx, ctx->rn_member, member, n, w.stream))) return rc;
        member_dev = ctx->rn_member;
    }
    if ((rc = render_scene_device(ctx, cam, member_dev, alpha_floor, transmittance_floor, ch_dev,
                                  channels, ctx->rn_f64)))
        return rc;
    CK(sync_copy(alpha, ctx->rn_f64, sizeof(double) * px, cudaMemcpyDeviceToHost, w.stream));
    CK(sync_copy(depth, ctx->rn_f64 + px, sizeof(double) * px, cudaMemcpyDeviceToHost, w.stream));
    if (channels)
        CK(sync_copy(value, ctx->rn_f64 + 2 * px, sizeof(double) * px * channels,
                      cudaMemcpyDeviceToHost, w.stream));
    return FS_OK;
}

int fs_render_splats(fs_context* ctx, int width, int height, int64_t k, const double* mean2d,
                     const double* conic, const double* depth, const double* opacity,
                     const int64_t* tile_offsets, const int64_t* items, double alpha_floor,
                     double transmittance_floor, const double* channel, int channels,
                     double* value, double* alpha, double* depth_out) {
    Range nvtx_range("fs_render_splats");
    if (!ctx || !tile_offsets || !alpha || !depth_out ||
        (k > 0 && (!mean2d || !conic || !depth || !opacity)))
        return fail(FS_EINVAL, "fs_render_splats: NULL argument");
    if (k < 0 || k > 0x7fffffffLL) return fail(FS_EINVAL, "fs_render_splats: bad splat count");
    if (channels != 0 && channels != 1 && channels != 3)
        return fail(FS_EINVAL, "fs_render_splats: channels must be 0, 1 or 3, got %d", channels);
    if (channels && k > 0 && (!channel || !value))
        return fail(FS_EINVAL, "fs_render_splats: NULL channel/value");
    fs_camera c{};
    c.width = width;
    c.height = height;
    int rc = check_render_cam(&c);
    if (rc) return rc;
    const int tx = fs::tiles_x_of(width), ntiles = tx * fs::tiles_y_of(height);
    const int64_t total = tile_offsets[ntiles];
    if (tile_offsets[0] != 0 || total < 0 || total > 0xffffffffLL)
        return fail(FS_EINVAL, "fs_render_splats: bad tile offsets");
    std::vector<unsigned int> starts(ntiles + 1), order(ntiles), lists((size_t)std::max<int64_t>(total, 1));
    for (int t = 0; t <= ntiles; ++t) {
        if (t && tile_offsets[t] < tile_offsets[t - 1])
            return fail(FS_EINVAL, "fs_render_splats: tile offsets not monotone");
        starts[t] = (unsigned int)tile_offsets[t];
    }
    for (int64_t i = 0; i < total; ++i) {
        if (!items || items[i] < 0 || items[i] >= k)
            return fail(FS_EINVAL, "fs_render_splats: item %lld out of range", (long long)i);
        lists[i] = (unsigned int)items[i];
    }
    for (int t = 0; t < ntiles; ++t) order[t] = (unsigned int)t;
    CK(cudaSetDevice(ctx->device));
    if ((rc = order_after_caller(ctx))) return rc;
    fs::Work& w = ctx->work[0];
    const size_t px = (size_t)width * height, kk = (size_t)std::max<int64_t>(k, 1);
    if ((rc = ensure_work(ctx, w, (long long)kk, ntiles, std::max(w.inst_cap, 1u), 1))) return rc;
    if ((rc = grow(&ctx->rn_f64, &ctx->rn_f64_cap, px * (2 + (size_t)channels)))) return rc;
    if ((rc = grow(&ctx->rn_in, &ctx->rn_in_cap, kk * (7 + (size_t)channels)))) return rc;
    if ((rc = grow(&ctx->rn_u32, &ctx->rn_u32_cap, lists.size() + ntiles))) return rc;
    double* d_mean = ctx->rn_in;
    double* d_conic = d_mean + 2 * kk;
    double* d_depth = d_conic + 3 * kk;
    double* d_opac = d_depth + kk;
    double* d_ch = d_opac + kk;
    cudaStream_t st = w.stream;
    if (k > 0) {
        CK(cudaMemcpyAsync(d_mean, mean2d, 16 * (size_t)k, cudaMemcpyHostToDevice, st));
        CK(cudaMemcpyAsync(d_conic, conic, 24 * (size_t)k, cudaMemcpyHostToDevice, st));
        CK(cudaMemcpyAsync(d_depth, depth, 8 * (size_t)k, cudaMemcpyHostToDevice, st));
        CK(cudaMemcpyAsync(d_opac, opacity, 8 * (size_t)k, cudaMemcpyHostToDevice, st));
        if (channels)
            CK(cudaMemcpyAsync(d_ch, channel, 8 * (size_t)k * channels, cudaMemcpyHostToDevice, st));
    }
    CK(cudaMemcpyAsync(ctx->rn_u32, lists.data(), 4 * lists.size(), cudaMemcpyHostToDevice, st));
    CK(cudaMemcpyAsync(ctx->rn_u32 + lists.size(), order.data(), 4 * (size_t)ntiles,
                       cudaMemcpyHostToDevice, st));
    CK(cudaMemcpyAsync(w.tile_start, starts.data(), 4 * (size_t)(ntiles + 1), cudaMemcpyHostToDevice,
                       st));
    CK(cudaMemsetAsync(ctx->rn_f64, 0, sizeof(double) * px * (2 + (size_t)channels), st));
    fs::launch_view_begin(w.vc, st);
    fs::launch_splat_records((int)k, d_mean, d_conic, d_depth, d_opac, alpha_floor, w.r32, w.r64,
                             w.k64, ctx->num_sms, st);
    fs::RasterArgs ra = render_args(w, width, height, alpha_floor, transmittance_floor, ctx->rn_f64,
                                    channels, channels ? d_ch : nullptr, k);
    ra.render.lists = ctx->rn_u32;
    ra.tile_order = ctx->rn_u32 + lists.size();
    fs::launch_raster_render(ra, st);
    CK(cudaGetLastError());
    CK(cudaStreamSynchronize(st));
    CK(sync_copy(alpha, ctx->rn_f64, sizeof(double) * px, cudaMemcpyDeviceToHost, st));
    CK(sync_copy(depth_out, ctx->rn_f64 + px, sizeof(double) * px, cudaMemcpyDeviceToHost, st));
    if (channels)
        CK(sync_copy(value, ctx->rn_f64 + 2 * px, sizeof(double) * px * channels,
                      cudaMemcpyDeviceToHost, st));
    return FS_OK;
}

int fs_render_mask(fs_context* ctx, const fs_camera* cam, const uint8_t* membership,
                   int num_objects, double tau, double alpha_floor, double transmittance_floor,
                   uint16_t* labels) {
    Range nvtx_range("fs_render_mask");
    if (!ctx || !cam || !labels || (!membership && ctx->n > 0))
        return fail(FS_EINVAL, "fs_render_mask: NULL argument");
    if (num_objects < 1 || num_objects > 65536)
        return fail(FS_EINVAL, "fs_render_mask: num_objects must be in [1, 65536], got %d",
                    num_objects);
    if (!(tau > 0.0 && tau < 1.0)) return fail(FS_EINVAL, "tau must lie in (0, 1), got %g", tau);
    int rc = check_render_cam(cam);
    if (rc) return rc;
    CK(cudaSetDevice(ctx->device));
    if ((rc = order_after_caller(ctx))) return rc;
    fs::Work& w = ctx->work[0];
    cudaStream_t st = w.stream;
    const size_t px = (size_t)cam->width * cam->height, n = (size_t)std::max<long long>(ctx->n, 0);
    const int tx = fs::tiles_x_of(cam->width), ntiles = tx * fs::tiles_y_of(cam->height);
    if ((rc = grow(&ctx->rn_f64, &ctx->rn_f64_cap, 3 * px))) return rc;  // alpha | depth | best
    if ((rc = grow(&ctx->rn_labels, &ctx->rn_labels_cap, px))) return rc;
    CK(cudaMemsetAsync(ctx->rn_labels, 0, sizeof(uint16_t) * px, st));
    // maskrender.py:82-83: empty objects are skipped (early-exit scan per row)
    std::vector<int> objs;
    for (int obj = 1; obj < num_objects; ++obj) {
        const uint8_t* row = membership + (size_t)obj * n;
        bool any = false;
        for (size_t i = 0; i < n && !any; ++i) any = row[i] != 0;
        if (any) objs.push_back(obj);
    }
    if (!objs.empty()) {
        if ((rc = grow(&ctx->rn_member, &ctx->rn_member_cap, (size_t)num_objects * n))) return rc;
        if ((rc = grow(&ctx->rn_rect, &ctx->rn_rect_cap, n))) return rc;
        if ((rc = upload(ctx, ctx->rn_member, membership, (size_t)num_objects * n, st))) return rc;
        // Project once and bin the whole scene once: its instance count bounds
        // every object's, so the per-object loop below runs without host syncs.
        unsigned int cap = std::max(w.inst_cap, initial_inst_cap(ctx->n));
        fs::ViewCounters vc{};
        for (int attempt = 0; attempt < 2; ++attempt) {
            if ((rc = ensure_work(ctx, w, (long long)n, ntiles, cap, 1))) return rc;
            enqueue_bin(ctx, w, to_cam(*cam), alpha_floor, 1, fs::ProjectExport{});
            CK(cudaMemcpyAsync(&vc, w.vc, sizeof(vc), cudaMemcpyDeviceToHost, st));
            CK(cudaStreamSynchronize(st));
            if (!vc.overflow) break;
            cap = (unsigned int)std::min<unsigned long long>(0x7fffffffull,
                                                             (unsigned long long)vc.n_instances + 1024);
        }
        if (vc.overflow) return fail(FS_ENOMEM, "fs_render_mask: instance buffer overflow");
        CK(cudaMemcpyAsync(ctx->rn_rect, w.rect, sizeof(unsigned long long) * n,
                           cudaMemcpyDeviceToDevice, st));
        double* best = ctx->rn_f64 + 2 * px;
        const int grid = (int)std::min<size_t>((px + 255) / 256, (size_t)ctx->num_sms * 8);
        const int ngrid = (int)std::min<size_t>((n + 255) / 256, (size_t)ctx->num_sms * 8);
        const fs::RasterArgs ra = render_args(w, cam->width, cam->height, alpha_floor,
                                              transmittance_floor, ctx->rn_f64, 0, nullptr,
                                              (long long)n, scene_perm(ctx));
        for (int obj : objs) {
            member_rect_kernel<<<std::max(ngrid, 1), 256, 0, st>>>(
                ctx->rn_rect, ctx->rn_member + (size_t)obj * n, scene_perm(ctx), (long long)n,
                w.rect);
            fs::launch_bin(ntiles, tx, bin_buffers(w, (int)n, w.vc), w.vc, ctx->num_sms, st);
            CK(cudaMemsetAsync(ctx->rn_f64, 0, sizeof(double) * 2 * px, st));
            fs::launch_raster_render(ra, st);
            mask_combine_kernel<<<std::max(grid, 1), 256, 0, st>>>(
                ctx->rn_f64, ctx->rn_f64 + px, (long long)px, tau, (unsigned int)obj,
                ctx->rn_labels, best);
            CK(cudaGetLastError());
        }
    }
    CK(cudaStreamSynchronize(st));
    CK(sync_copy(labels, ctx->rn_labels, sizeof(uint16_t) * px, cudaMemcpyDeviceToHost, st));
    return FS_OK;
}

}  // extern "C"
