/* c_abi_demo.c -- the C ABI used from plain C (no Python, no torch): one
 * Gaussian in front of a 32 x 32 camera, one mask with two labels, the
 * fixed-point accumulator, the float32 cast and the binary argmax.
 * Built and run by tests/test_gpu_capi_c.py:
 *   gcc -O2 -Iinclude tests/c_abi_demo.c -Lpaper_2409_08270_b200/_lib -lflashsplat_b200 \
 *       -Wl,-rpath,paper_2409_08270_b200/_lib -o /tmp/c_abi_demo
 * Prints "A <e> <n> <value>" lines and "label <n> <value>". */
#include <stdint.h>
#include <stdio.h>
#include <string.h>

#include "flashsplat_b200.h"

#define CHECK(call)                                                           \
    do {                                                                      \
        int rc_ = (call);                                                     \
        if (rc_ != FS_OK) {                                                   \
            fprintf(stderr, "%s failed (%d): %s\n", #call, rc_, fs_last_error()); \
            return 1;                                                         \
        }                                                                     \
    } while (0)

int main(void) {
    fs_context *ctx = NULL;
    CHECK(fs_create(0, 2, &ctx));
    /* two Gaussians: one at the view centre, one off to the right, both at z = 4 */
    const int64_t n = 2;
    double means[6] = {0.0, 0.0, 4.0, 0.6, 0.0, 4.0};
    double quats[8] = {1, 0, 0, 0, 1, 0, 0, 0};
    double scales[6] = {0.2, 0.2, 0.2, 0.1, 0.1, 0.1};
    double opac[2] = {0.8, 0.6};
    CHECK(fs_set_scene(ctx, n, means, quats, scales, opac));

    fs_camera cam;
    memset(&cam, 0, sizeof(cam));
    cam.width = 32;
    cam.height = 32;
    cam.fx = cam.fy = 40.0;
    cam.cx = cam.cy = 16.0;
    for (int i = 0; i < 4; ++i) cam.world_to_camera[5 * i] = 1.0;
    cam.near_clip = 0.01;

    static uint16_t mask[32 * 32];
    for (int y = 0; y < 32; ++y)
        for (int x = 0; x < 32; ++x) mask[y * 32 + x] = x >= 16 ? 1 : 0;  /* right half: object 1 */
    const uint16_t *masks[1] = {mask};

    const int E = 2;
    void *acc = NULL;
    CHECK(fs_device_alloc(ctx, 16 * (uint64_t)E * n, &acc));
    CHECK(fs_memset_zero(ctx, acc, 16 * (uint64_t)E * n));
    fs_accumulate_stats st;
    CHECK(fs_accumulate(ctx, 1, &cam, masks, 0, E, 1.0 / 255.0, 1e-4, FS_ACC_FIXED, acc, &st));
    float A[4];
    CHECK(fs_finalize(ctx, FS_ACC_FIXED, acc, n, E, A, 0));
    uint8_t labels[2];
    CHECK(fs_assign(ctx, A, n, E, 0.0f, FS_MODE_BINARY, labels, 0));
    for (int e = 0; e < E; ++e)
        for (int g = 0; g < n; ++g) printf("A %d %d %.9g\n", e, g, (double)A[e * n + g]);
    for (int g = 0; g < n; ++g) printf("label %d %d\n", g, labels[g]);
    printf("stats views=%lld pixels=%lld exact=%lld adds=%lld\n", (long long)st.views,
           (long long)st.view_pixels, (long long)st.exact_evals, (long long)st.atomics);
    CHECK(fs_device_free(ctx, acc));
    fs_destroy(ctx);
    return 0;
}
