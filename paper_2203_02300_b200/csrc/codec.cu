// codec.cu -- frame ingest / egress of SURVEY 8f rank 3 (reference
// src/codec.cpp, src/image.cpp): the float <-> 8-bit conversions on the
// device (so only bytes cross PCIe) and the PNM / PFM file formats on the
// host, byte-for-byte the reference's files.
//   quantize (codec.cpp:23-26)     -> k_quantize_u8  (clamp, lround(v*255f))
//   to_gray (image.cpp:7-15)       -> k_to_gray      (Rec. 601, float, no FMA)
//   read_pnm (codec.cpp:59-82)     -> dco_read_pnm   (header grammar, errors)
//   write_pgm/ppm (codec.cpp:211-229) -> dco_write_pnm
//   write_pfm (codec.cpp:293-309)  -> dco_write_pfm  (bottom-up rows, nodata = +inf)
#include <ctype.h>
#include <stdio.h>
#include <string.h>

#include <cmath>
#include <limits>
#include <string>
#include <vector>

#include "common.cuh"

namespace dco_gpu {
namespace {

__global__ void k_quantize_u8(const float* __restrict__ in, size_t n, uint8_t* __restrict__ out) {
    const size_t i = static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= n) return;
    float v = in[i];
    // std::clamp(v, 0, 1): NaN passes through; lround(NaN) is LONG_MIN on
    // x86-64, whose low byte is 0
    v = v < 0.0f ? 0.0f : (1.0f < v ? 1.0f : v);
    out[i] = isnan(v) ? 0 : static_cast<uint8_t>(lroundf(v * 255.0f));
}

__global__ void k_to_gray(const float* __restrict__ rgb, size_t n, float* __restrict__ gray) {
    const size_t i = static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const float r = rgb[3 * i], g = rgb[3 * i + 1], b = rgb[3 * i + 2];
    gray[i] = __fadd_rn(__fadd_rn(__fmul_rn(0.299f, r), __fmul_rn(0.587f, g)), __fmul_rn(0.114f, b));
}

struct CodecFail {
    int status;
    std::string msg;
};

[[noreturn]] void codec_fail(const std::string& path, const std::string& what, long offset) {
    throw CodecFail{DCO_CODEC, path + ": " + what + " (byte offset " + std::to_string(offset) + ")"};
}

void set_err(char* err, size_t len, const std::string& m) {
    if (err && len) {
        strncpy(err, m.c_str(), len - 1);
        err[len - 1] = 0;
    }
}

// A byte reader whose position reads -1 once it has hit the end, as the
// reference's std::ifstream::tellg() does after a failed get().
struct Reader {
    FILE* f;
    bool failed = false;
    int get() {
        const int c = fgetc(f);
        if (c == EOF) failed = true;
        return c;
    }
    long tell() const { return failed ? -1 : ftell(f); }
};

// read_pnm_int, codec.cpp:29-47: whitespace and '#' comments, digits, range cap
int pnm_int(Reader& in, const std::string& path) {
    int c = in.get();
    while (c != EOF && (isspace(c) || c == '#')) {
        if (c == '#')
            while (c != EOF && c != '\n') c = in.get();
        c = in.get();
    }
    if (c == EOF || !isdigit(c)) codec_fail(path, "malformed header", in.tell());
    long value = 0;
    while (c != EOF && isdigit(c)) {
        value = value * 10 + (c - '0');
        if (value > 1 << 30) codec_fail(path, "header value out of range", in.tell());
        c = in.get();
    }
    if (c != EOF) ungetc(c, in.f);
    return static_cast<int>(value);
}

template <typename F>
int codec_guarded(char* err, size_t len, F&& fn) {
    try {
        fn();
        set_err(err, len, "");
        return DCO_OK;
    } catch (const CodecFail& e) {
        set_err(err, len, e.msg);
        return e.status;
    }
}

}  // namespace
}  // namespace dco_gpu

using namespace dco_gpu;

extern "C" {

int dco_quantize_u8(dco_ctx* ctx, const float* in, size_t n, uint8_t* out) {
    return guarded(ctx, [&] {
        if (n == 0) return;
        k_quantize_u8<<<blocks_for(n, 256), 256, 0, ctx->stream>>>(in, n, out);
        launched(ctx, "k_quantize_u8");
    });
}

int dco_to_gray(dco_ctx* ctx, const float* rgb, int w, int h, float* gray) {
    return guarded(ctx, [&] {
        require(w >= 1 && h >= 1, "to_gray: empty image");
        const size_t n = static_cast<size_t>(w) * h;
        k_to_gray<<<blocks_for(n, 256), 256, 0, ctx->stream>>>(rgb, n, gray);
        launched(ctx, "k_to_gray");
    });
}

int dco_read_pnm(const char* path, int expect_color, uint8_t* bytes, size_t cap, int* w, int* h, char* err,
                 size_t err_len) {
    return codec_guarded(err, err_len, [&] {
        if (!path || !w || !h) throw CodecFail{DCO_INPUT, "read_pnm: null argument"};
        const std::string p(path);
        FILE* f = fopen(path, "rb");
        if (!f) throw CodecFail{DCO_CODEC, p + ": cannot open file"};
        struct Closer {
            FILE* f;
            ~Closer() { fclose(f); }
        } closer{f};
        Reader in{f};
        const int m0 = in.get(), m1 = in.get();
        if (m0 != 'P' || m1 != (expect_color ? '6' : '5')) codec_fail(p, "bad magic", 0);
        const int ww = pnm_int(in, p), hh = pnm_int(in, p), maxval = pnm_int(in, p);
        if (ww < 1 || hh < 1) codec_fail(p, "degenerate dimensions", in.tell());
        if (maxval != 255) codec_fail(p, "unsupported bit depth (maxval must be 255)", in.tell());
        *w = ww;
        *h = hh;
        const size_t n = static_cast<size_t>(ww) * hh * (expect_color ? 3 : 1);
        if (!bytes) return;  // header only
        if (cap < n) throw CodecFail{DCO_INPUT, p + ": buffer too small for the payload"};
        const int sep = in.get();
        if (sep == EOF || !isspace(sep)) codec_fail(p, "malformed header", in.tell());
        const long start = in.tell();
        const size_t got = fread(bytes, 1, n, f);
        if (got != n) codec_fail(p, "truncated payload", start + static_cast<long>(got));
    });
}

int dco_write_pnm(const char* path, const uint8_t* bytes, int w, int h, int channels, char* err, size_t err_len) {
    return codec_guarded(err, err_len, [&] {
        if (!path || !bytes || w < 1 || h < 1 || (channels != 1 && channels != 3))
            throw CodecFail{DCO_INPUT, "write_pnm: bad arguments"};
        const std::string p(path);
        FILE* f = fopen(path, "wb");
        if (!f) throw CodecFail{DCO_CODEC, p + ": cannot open file for writing"};
        const size_t n = static_cast<size_t>(w) * h * channels;
        const bool ok = fprintf(f, "P%c\n%d %d\n255\n", channels == 3 ? '6' : '5', w, h) > 0 &&
                        fwrite(bytes, 1, n, f) == n;
        const bool closed = fclose(f) == 0;
        if (!ok || !closed) throw CodecFail{DCO_CODEC, p + ": write failed"};
    });
}

int dco_write_pfm(const char* path, const float* map, int w, int h, char* err, size_t err_len) {
    return codec_guarded(err, err_len, [&] {
        if (!path || !map || w < 1 || h < 1) throw CodecFail{DCO_INPUT, "write_pfm: bad arguments"};
        const std::string p(path);
        FILE* f = fopen(path, "wb");
        if (!f) throw CodecFail{DCO_CODEC, p + ": cannot open file for writing"};
        bool ok = fprintf(f, "Pf\n%d %d\n-1.0\n", w, h) > 0;
        std::vector<float> row(w);
        for (int y = h - 1; y >= 0 && ok; --y) {  // little-endian host (x86-64 / aarch64)
            for (int x = 0; x < w; ++x) {
                const float v = map[static_cast<size_t>(y) * w + x];
                row[x] = std::isfinite(v) ? v : std::numeric_limits<float>::infinity();
            }
            ok = fwrite(row.data(), 4, w, f) == static_cast<size_t>(w);
        }
        const bool closed = fclose(f) == 0;
        if (!ok || !closed) throw CodecFail{DCO_CODEC, p + ": write failed"};
    });
}

}  // extern "C"
