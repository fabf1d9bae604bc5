// fs_ingest.cpp -- native decode of label-mask PNGs.
//
// The reference loads masks with Pillow, one file at a time
// (masks.py:30-40, cli.py:74-83).  Here the common wire format -- non-interlaced
// 8- or 16-bit grayscale PNG, pixel value = object id -- is decoded in C++
// (zlib inflate + PNG row unfiltering), so a Python thread pool calling
// fs_decode_mask_png runs truly in parallel (ctypes drops the GIL).  Any other
// PNG flavour returns FS_EINVAL with "unsupported" and the caller falls back to
// the reference-equivalent Pillow path.
#include <zlib.h>

#include <cstdarg>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <vector>

#include "flashsplat_b200.h"

namespace fs {
int report_error(int code, const char* msg);  // fs_capi.cu (thread-local fs_last_error)

static int fail(int code, const char* fmt, ...) {
    char buf[256];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof(buf), fmt, ap);
    va_end(ap);
    return report_error(code, buf);
}
}  // namespace fs

namespace {

uint32_t be32(const uint8_t* p) {
    return (uint32_t)p[0] << 24 | (uint32_t)p[1] << 16 | (uint32_t)p[2] << 8 | (uint32_t)p[3];
}

int paeth(int a, int b, int c) {
    const int p = a + b - c;
    const int pa = p > a ? p - a : a - p, pb = p > b ? p - b : b - p, pc = p > c ? p - c : c - p;
    if (pa <= pb && pa <= pc) return a;
    return pb <= pc ? b : c;
}

}  // namespace

extern "C" int fs_decode_mask_png(const uint8_t* data, int64_t size, uint16_t* out,
                                  int64_t out_capacity, int* width, int* height) {
    static const uint8_t sig[8] = {137, 80, 78, 71, 13, 10, 26, 10};
    if (!data || !width || !height) return fs::fail(FS_EINVAL, "fs_decode_mask_png: NULL argument");
    if (size < 8 || memcmp(data, sig, 8) != 0) return fs::fail(FS_EINVAL, "not a PNG file");
    int64_t pos = 8;
    uint32_t w = 0, h = 0;
    int depth = 0, ctype = -1, interlace = 0;
    std::vector<uint8_t> idat;
    bool seen_ihdr = false, seen_iend = false, seen_idat = false;
    while (pos + 12 <= size && !seen_iend) {
        const uint32_t len = be32(data + pos);
        const uint8_t* type = data + pos + 4;
        const uint8_t* body = data + pos + 8;
        if (pos + 12 + (int64_t)len > size) return fs::fail(FS_EINVAL, "truncated PNG chunk");
        // Pillow verifies the CRC of every chunk it parses before the image data
        // and rejects the file on a mismatch; decline such files so the caller's
        // Pillow path raises the reference's error instead of decoding them
        if (!seen_idat && memcmp(type, "IDAT", 4) != 0 &&
            crc32(crc32(0L, type, 4), body, len) != be32(body + len))
            return fs::fail(FS_EINVAL, "PNG chunk CRC mismatch");
        if (!memcmp(type, "IHDR", 4)) {
            if (len < 13) return fs::fail(FS_EINVAL, "bad IHDR");
            if (body[10] != 0 || body[11] != 0)
                return fs::fail(FS_EINVAL, "unsupported PNG compression / filter method");
            w = be32(body);
            h = be32(body + 4);
            depth = body[8];
            ctype = body[9];
            interlace = body[12];
            seen_ihdr = true;
        } else if (!memcmp(type, "IDAT", 4)) {
            seen_idat = true;
            idat.insert(idat.end(), body, body + len);
        } else if (!memcmp(type, "IEND", 4)) {
            seen_iend = true;
        }
        pos += 12 + (int64_t)len;
    }
    if (!seen_ihdr) return fs::fail(FS_EINVAL, "PNG without IHDR");
    if (ctype != 0 || (depth != 8 && depth != 16) || interlace != 0)
        return fs::fail(FS_EINVAL, "unsupported PNG flavour (color type %d, depth %d, interlace %d)",
                        ctype, depth, interlace);
    if (w == 0 || h == 0 || (uint64_t)w * h > (1ull << 31))
        return fs::fail(FS_EINVAL, "bad PNG dimensions %ux%u", w, h);
    *width = (int)w;
    *height = (int)h;
    if (!out) return FS_OK;  // dimension query
    if (out_capacity < (int64_t)w * h) return fs::fail(FS_EINVAL, "output buffer too small");
    const int bpp = depth / 8;
    const size_t stride = (size_t)w * bpp;
    std::vector<uint8_t> raw((stride + 1) * h);
    uLongf raw_len = (uLongf)raw.size();
    const int zr = uncompress(raw.data(), &raw_len, idat.data(), (uLong)idat.size());
    if (zr != Z_OK || raw_len != raw.size()) return fs::fail(FS_EINVAL, "corrupt PNG image data");
    std::vector<uint8_t> zero(stride, 0);
    uint8_t* base = raw.data();
    const uint8_t* prev = zero.data();
    // unfilter in place: row y's bytes follow its filter byte in `raw`
    for (uint32_t y = 0; y < h; ++y) {
        uint8_t* row = base + (size_t)y * (stride + 1);
        const int f = row[0];
        uint8_t* cur = row + 1;
        switch (f) {
            case 0:
                break;
            case 1:
                for (size_t i = bpp; i < stride; ++i) cur[i] = (uint8_t)(cur[i] + cur[i - bpp]);
                break;
            case 2:
                for (size_t i = 0; i < stride; ++i) cur[i] = (uint8_t)(cur[i] + prev[i]);
                break;
            case 3:
                for (size_t i = 0; i < (size_t)bpp; ++i) cur[i] = (uint8_t)(cur[i] + (prev[i] >> 1));
                for (size_t i = bpp; i < stride; ++i)
                    cur[i] = (uint8_t)(cur[i] + ((cur[i - bpp] + prev[i]) >> 1));
                break;
            case 4:
                for (size_t i = 0; i < (size_t)bpp; ++i) cur[i] = (uint8_t)(cur[i] + prev[i]);
                for (size_t i = bpp; i < stride; ++i)
                    cur[i] = (uint8_t)(cur[i] + paeth(cur[i - bpp], prev[i], prev[i - bpp]));
                break;
            default:
                return fs::fail(FS_EINVAL, "bad PNG filter type %d", f);
        }
        uint16_t* o = out + (size_t)y * w;
        if (bpp == 2)
            for (uint32_t x = 0; x < w; ++x) o[x] = (uint16_t)(cur[2 * x] << 8 | cur[2 * x + 1]);
        else
            for (uint32_t x = 0; x < w; ++x) o[x] = cur[x];
        prev = cur;
    }
    return FS_OK;
}
