// contour.cu — depth-contour extraction (reference src/contour.cpp) on sm_100a:
// polar radius + gradient amplitude, projection-confidence fusion, SAT box
// filter, global-max normalisation, 5-tap Gaussian, Sobel / NMS / depth gate
// and 8-connected hysteresis.
//
// Exactness notes:
//  * hypotf / hypot / atan2f are the glibc replicas of dco_libm.h.
//  * box_filter's summed-area table keeps the reference's sequential double
//    order: one thread per row builds the running row sums, one thread per
//    column chains them (contour.cpp:113-122).
//  * the global maxima are order-independent (max is exact), so a parallel
//    atomicMax on the IEEE bits of non-negative floats is exact.
//  * hysteresis is set-defined (components of {survives, mag >= t_low}
//    holding a pixel with mag > t_high), so union-find connected components
//    reproduce the reference's BFS exactly (contour.cpp:250-277).
#include <math.h>
#include <stdint.h>
#include <string.h>

#include "common.cuh"
#include "dco_libm.h"

namespace dco_gpu {
namespace {

constexpr double kPi = 3.141592653589793;  // std::numbers::pi

__device__ __forceinline__ float clampf(float v, float lo, float hi) {
    return (v < lo) ? lo : ((hi < v) ? hi : v);
}
// std::max(a, b) for floats: (a < b) ? b : a
__device__ __forceinline__ float stdmaxf(float a, float b) { return (a < b) ? b : a; }

// ------------------------------------------------------------ polar / amp --
// flow_to_polar, contour.cpp:10-25.
__global__ void k_polar(const float* __restrict__ u, const float* __restrict__ v, size_t n,
                        float* __restrict__ r, float* __restrict__ theta) {
    size_t i = static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= n) return;
    float uu = u[i], vv = v[i];
    r[i] = dco_hypotf(uu, vv);
    if (theta) {
        float t = dco_atan2f(vv, uu);
        if (t <= -static_cast<float>(kPi)) t = static_cast<float>(kPi);
        theta[i] = t;
    }
}

// gradient_amplitude, contour.cpp:27-42 on a radius map.
__device__ __forceinline__ float amp_at(const float* r, int w, int h, int x, int y) {
    float rc = r[static_cast<size_t>(y) * w + x];
    float gu = x + 1 < w ? r[static_cast<size_t>(y) * w + x + 1] - rc
                         : (w > 1 ? rc - r[static_cast<size_t>(y) * w + x - 1] : 0.0f);
    float gv = y + 1 < h ? r[static_cast<size_t>(y + 1) * w + x] - rc
                         : (h > 1 ? rc - r[static_cast<size_t>(y - 1) * w + x] : 0.0f);
    return stdmaxf(fabsf(gu), fabsf(gv));
}

__global__ void k_grad_amp(const float* __restrict__ r, int w, int h, float* __restrict__ amp) {
    int x = blockIdx.x * blockDim.x + threadIdx.x;
    int y = blockIdx.y * blockDim.y + threadIdx.y;
    if (x >= w || y >= h) return;
    amp[static_cast<size_t>(y) * w + x] = amp_at(r, w, h, x, y);
}

// ------------------------------------------------------------------ fusion -
// sample_component, contour.cpp:46-60.
__device__ __forceinline__ float sample_component(const float* d, int w, int h, float x, float y) {
    x = clampf(x, 0.0f, static_cast<float>(w - 1));
    y = clampf(y, 0.0f, static_cast<float>(h - 1));
    int x0 = static_cast<int>(x), y0 = static_cast<int>(y);
    int x1 = min(x0 + 1, w - 1), y1 = min(y0 + 1, h - 1);
    float fx = x - static_cast<float>(x0), fy = y - static_cast<float>(y0);
    float top = d[static_cast<size_t>(y0) * w + x0] * (1 - fx) + d[static_cast<size_t>(y0) * w + x1] * fx;
    float bot = d[static_cast<size_t>(y1) * w + x0] * (1 - fx) + d[static_cast<size_t>(y1) * w + x1] * fx;
    return top * (1 - fy) + bot * fy;
}

// projection_confidence, contour.cpp:65-78.
__device__ __forceinline__ double projection_confidence(const float* fu, const float* fv, int w, int h,
                                                        int x, int y, double k) {
    size_t i = static_cast<size_t>(y) * w + x;
    float u = fu[i], v = fv[i];
    double mag = dco_hypot(static_cast<double>(u), static_cast<double>(v));
    if (mag < 1e-3) return 0.0;
    double ex = u / mag, ey = v / mag;
    float bx = static_cast<float>(x - k * ex), by = static_cast<float>(y - k * ey);
    float fx = static_cast<float>(x + k * ex), fy = static_cast<float>(y + k * ey);
    double f0 = sample_component(fu, w, h, bx, by) * ex + sample_component(fv, w, h, bx, by) * ey;
    double f1 = sample_component(fu, w, h, fx, fy) * ex + sample_component(fv, w, h, fx, fy) * ey;
    return f1 - f0;
}

// fuse_amplitudes, contour.cpp:82-106.
__global__ void k_fuse(const float* __restrict__ pu, const float* __restrict__ pv,
                       const float* __restrict__ fu, const float* __restrict__ fv,
                       const float* __restrict__ mp, const float* __restrict__ mf, int w, int h,
                       double k, float* __restrict__ out) {
    int x = blockIdx.x * blockDim.x + threadIdx.x;
    int y = blockIdx.y * blockDim.y + threadIdx.y;
    if (x >= w || y >= h) return;
    double rp = projection_confidence(pu, pv, w, h, x, y, k);
    double rf = projection_confidence(fu, fv, w, h, x, y, k);
    size_t i = static_cast<size_t>(y) * w + x;
    float a = mp[i], b = mf[i];
    out[i] = rp > rf ? a : (rf > rp ? b : stdmaxf(a, b));
}

// Pipeline fusion of flow_to_polar + gradient_amplitude (both directions) +
// fuse_amplitudes: radii are recomputed from the flow on the fly, so the
// amplitude maps never touch HBM.
__device__ __forceinline__ float radius(const float* u, const float* v, size_t i) {
    return dco_hypotf(u[i], v[i]);
}
__device__ __forceinline__ float amp_from_flow(const float* u, const float* v, int w, int h, int x,
                                               int y) {
    size_t i = static_cast<size_t>(y) * w + x;
    float rc = radius(u, v, i);
    float gu = x + 1 < w ? radius(u, v, i + 1) - rc : (w > 1 ? rc - radius(u, v, i - 1) : 0.0f);
    float gv = y + 1 < h ? radius(u, v, i + w) - rc : (h > 1 ? rc - radius(u, v, i - w) : 0.0f);
    return stdmaxf(fabsf(gu), fabsf(gv));
}

__global__ void k_amp_fuse(const float* __restrict__ pu, const float* __restrict__ pv,
                           const float* __restrict__ fu, const float* __restrict__ fv, int w, int h,
                           double k, float* __restrict__ out) {
    int x = blockIdx.x * blockDim.x + threadIdx.x;
    int y = blockIdx.y * blockDim.y + threadIdx.y;
    if (x >= w || y >= h) return;
    double rp = projection_confidence(pu, pv, w, h, x, y, k);
    double rf = projection_confidence(fu, fv, w, h, x, y, k);
    float out_v;
    if (rp > rf)
        out_v = amp_from_flow(pu, pv, w, h, x, y);
    else if (rf > rp)
        out_v = amp_from_flow(fu, fv, w, h, x, y);
    else
        out_v = stdmaxf(amp_from_flow(pu, pv, w, h, x, y), amp_from_flow(fu, fv, w, h, x, y));
    out[static_cast<size_t>(y) * w + x] = out_v;
}

// -------------------------------------------------------------- box filter -
// box_filter, contour.cpp:108-136. Row running sums (double, sequential).
__global__ void k_box_rows(const float* __restrict__ a, int w, int h, double* __restrict__ rows) {
    // one warp per row: coalesced 32-wide loads, the running sum stays a
    // strictly sequential double chain (lane 0's order) broadcast by shuffles
    const int lane = threadIdx.x & 31;
    const int y = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    if (y >= h) return;
    const float* src = a + static_cast<size_t>(y) * w;
    double* dst = rows + static_cast<size_t>(y) * w;
    double s = 0.0;
    float nxt = lane < w ? src[lane] : 0.0f;
    for (int x0 = 0; x0 < w; x0 += 32) {
        float cur = nxt;
        nxt = (x0 + 32 + lane < w) ? src[x0 + 32 + lane] : 0.0f;
        double mine = 0.0;
        const int cnt = min(32, w - x0);
        for (int j = 0; j < cnt; ++j) {
            s += static_cast<double>(__shfl_sync(0xffffffffu, cur, j));
            if (lane == j) mine = s;
        }
        if (lane < cnt) dst[x0 + lane] = mine;
    }
}
// Column chain: sat[y+1][x+1] = sat[y][x+1] + rows[y][x]; sat is (h+1)x(w+1).
__global__ void k_box_cols(const double* __restrict__ rows, int w, int h, double* __restrict__ sat) {
    int x = blockIdx.x * blockDim.x + threadIdx.x;
    if (x > w) return;
    const size_t W1 = static_cast<size_t>(w) + 1;
    if (x == 0) {
        for (int y = 0; y <= h; ++y) sat[y * W1] = 0.0;
        return;
    }
    double s = 0.0;
    sat[x] = 0.0;
    constexpr int kPF = 16;
    double cur[kPF], nxt[kPF];
#pragma unroll
    for (int j = 0; j < kPF; ++j) cur[j] = j < h ? rows[static_cast<size_t>(j) * w + (x - 1)] : 0.0;
    for (int y0 = 0; y0 < h; y0 += kPF) {
#pragma unroll
        for (int j = 0; j < kPF; ++j) {
            int y = y0 + kPF + j;
            nxt[j] = y < h ? rows[static_cast<size_t>(y) * w + (x - 1)] : 0.0;
        }
#pragma unroll
        for (int j = 0; j < kPF; ++j) {
            if (y0 + j < h) {
                s = s + cur[j];
                sat[(y0 + j + 1) * W1 + x] = s;
            }
            cur[j] = nxt[j];
        }
    }
}
__global__ void k_box_out(const double* __restrict__ sat, int w, int h, int r, float* __restrict__ out) {
    int x = blockIdx.x * blockDim.x + threadIdx.x;
    int y = blockIdx.y * blockDim.y + threadIdx.y;
    if (x >= w || y >= h) return;
    const size_t W1 = static_cast<size_t>(w) + 1;
    int y0 = max(0, y - r), y1 = min(h - 1, y + r);
    int x0 = max(0, x - r), x1 = min(w - 1, x + r);
    double sum = sat[(y1 + 1) * W1 + (x1 + 1)] - sat[y0 * W1 + (x1 + 1)] - sat[(y1 + 1) * W1 + x0] +
                 sat[y0 * W1 + x0];
    int count = (y1 - y0 + 1) * (x1 - x0 + 1);
    out[static_cast<size_t>(y) * w + x] = static_cast<float>(sum / count);
}

// ----------------------------------------------------------- normalisation -
// Global max of the valid, positive values as IEEE bits (order-free, exact).
__global__ void k_peak(const float* __restrict__ a, size_t n, unsigned* __restrict__ peak_bits) {
    size_t i = static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    unsigned b = 0;
    if (i < n) {
        float v = a[i];
        if (isfinite(v) && v > 0.0f) b = __float_as_uint(v);
    }
    block_atomic_max(peak_bits, b);
}
// normalize_amplitude, contour.cpp:138-147.
__global__ void k_normalize(const float* __restrict__ a, size_t n, const unsigned* __restrict__ peak_bits,
                            float* __restrict__ out) {
    size_t i = static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= n) return;
    float peak = __uint_as_float(*peak_bits);
    float v = a[i];
    if (peak > 0.0f && isfinite(v)) v = v / peak;
    out[i] = v;
}

// ---------------------------------------------------------------- gaussian -
// gaussian_blur, contour.cpp:149-175: double accumulation in tap order.
struct Taps {
    double k[5];
};
__global__ void k_gauss_h(const float* __restrict__ img, int w, int h, Taps t, float* __restrict__ out) {
    int x = blockIdx.x * blockDim.x + threadIdx.x;
    int y = blockIdx.y * blockDim.y + threadIdx.y;
    if (x >= w || y >= h) return;
    const float* row = img + static_cast<size_t>(y) * w;
    double acc = 0.0;
#pragma unroll
    for (int i = -2; i <= 2; ++i) acc += t.k[i + 2] * row[min(max(x + i, 0), w - 1)];
    out[static_cast<size_t>(y) * w + x] = static_cast<float>(acc);
}
__global__ void k_gauss_v(const float* __restrict__ img, int w, int h, Taps t, float* __restrict__ out) {
    int x = blockIdx.x * blockDim.x + threadIdx.x;
    int y = blockIdx.y * blockDim.y + threadIdx.y;
    if (x >= w || y >= h) return;
    double acc = 0.0;
#pragma unroll
    for (int i = -2; i <= 2; ++i) acc += t.k[i + 2] * img[static_cast<size_t>(min(max(y + i, 0), h - 1)) * w + x];
    out[static_cast<size_t>(y) * w + x] = static_cast<float>(acc);
}

// ------------------------------------------------------------ sobel / nms --
// contour.cpp:184-200: Sobel (clamped), mag = hypotf, global peak.
__global__ void k_sobel(const float* __restrict__ b, int w, int h, float* __restrict__ gx_out,
                        float* __restrict__ gy_out, float* __restrict__ mag, unsigned* __restrict__ peak_bits) {
    int x = blockIdx.x * blockDim.x + threadIdx.x;
    int y = blockIdx.y * blockDim.y + threadIdx.y;
    unsigned pb = 0;
    if (x < w && y < h) {
        int xm = max(x - 1, 0), xp = min(x + 1, w - 1), ym = max(y - 1, 0), yp = min(y + 1, h - 1);
        const float* rm = b + static_cast<size_t>(ym) * w;
        const float* r0 = b + static_cast<size_t>(y) * w;
        const float* rp = b + static_cast<size_t>(yp) * w;
        float tl = rm[xm], t = rm[x], tr = rm[xp];
        float l = r0[xm], r = r0[xp];
        float bl = rp[xm], bb = rp[x], br = rp[xp];
        float gx = (tr + 2 * r + br) - (tl + 2 * l + bl);
        float gy = (bl + 2 * bb + br) - (tl + 2 * t + tr);
        float m = dco_hypotf(gx, gy);
        size_t i = static_cast<size_t>(y) * w + x;
        gx_out[i] = gx;
        gy_out[i] = gy;
        mag[i] = m;
        if (m > 0.0f) pb = __float_as_uint(m);  // NaN-free: inputs finite
    }
    block_atomic_max(peak_bits, pb);
}

// contour.cpp:197-203: mag /= peak (peak > 0), copied out as m_i.
__global__ void k_mag_norm(float* __restrict__ mag, size_t n, const unsigned* __restrict__ peak_bits,
                           float* __restrict__ m_i) {
    size_t i = static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= n) return;
    float peak = __uint_as_float(*peak_bits);
    float v = mag[i];
    if (peak > 0.0f) v = v / peak;
    mag[i] = v;
    m_i[i] = v;
}

// NMS (contour.cpp:205-236) + depth gate (:238-248); emits the hysteresis
// classes: 0 none, 1 candidate (survives, mag >= t_low), 2 seed (mag > t_high).
// The NMS sector of contour.cpp:217-232 depends on the float a = atan2f(gy,
// gx) only through deg(a) = ((a < 0 ? a + pi : a) * 180) / pi in double,
// which is monotone in a on each sign branch; the host finds, per branch, the
// smallest float a whose deg reaches 22.5 / 67.5 / 112.5 / 157.5, so the
// device compares a with those floats (no double math per pixel). Likewise
// m >= t_low, m > t_high and conf < t_depth (float vs double) become float
// compares against the nearest floats on the right side of the thresholds.
struct NmsThresholds {
    float pos[4], neg[4];   // sector boundaries for a >= 0 and a < 0
    float low, high, depth;  // m >= low, m > high, conf < depth
};
__global__ void k_nms_gate(const float* __restrict__ gx, const float* __restrict__ gy,
                           const float* __restrict__ mag, int w, int h, const float* __restrict__ mf,
                           int qw, int qh, const NmsThresholds th, uint8_t* __restrict__ cls) {
    int x = blockIdx.x * blockDim.x + threadIdx.x;
    int y = blockIdx.y * blockDim.y + threadIdx.y;
    if (x >= w || y >= h) return;
    size_t i = static_cast<size_t>(y) * w + x;
    float m = mag[i];
    uint8_t c = 0;
    if (m > 0.0f) {
        const float a = dco_atan2f(gy[i], gx[i]);
        int sec;
        if (isnan(a)) {
            sec = 3;  // every deg comparison false: the reference's last branch
        } else {
            const float* t = a >= 0.0f ? th.pos : th.neg;
            sec = a < t[0] ? 0 : a < t[1] ? 1 : a < t[2] ? 2 : a < t[3] ? 3 : 0;
        }
        int ax, ay, bx, by;
        if (sec == 0) {
            ax = x + 1; ay = y; bx = x - 1; by = y;
        } else if (sec == 1) {
            ax = x + 1; ay = y + 1; bx = x - 1; by = y - 1;
        } else if (sec == 2) {
            ax = x; ay = y + 1; bx = x; by = y - 1;
        } else {
            ax = x - 1; ay = y + 1; bx = x + 1; by = y - 1;
        }
        ax = min(max(ax, 0), w - 1); bx = min(max(bx, 0), w - 1);
        ay = min(max(ay, 0), h - 1); by = min(max(by, 0), h - 1);
        float n1 = mag[static_cast<size_t>(ay) * w + ax];
        float n2 = mag[static_cast<size_t>(by) * w + bx];
        bool survives = m >= n1 && m >= n2;
        if (survives) {
            int mx = min(x / 2, qw - 1), my = min(y / 2, qh - 1);
            float conf = mf[static_cast<size_t>(my) * qw + mx];
            if (!isfinite(conf) || conf < th.depth) survives = false;
        }
        if (survives && m >= th.low) c = 1;
        if (survives && m > th.high) c = 2;
    }
    cls[i] = c;
}

// Every float a in [-4, 4] (and the NaNs): the sector from the thresholds
// against the reference's double expression (tests/test_gpu_flow_contour.py).
__global__ void k_nms_check(const NmsThresholds th, unsigned long long* bad) {
    unsigned long long miss = 0;
    for (unsigned long long u = blockIdx.x * static_cast<unsigned long long>(blockDim.x) + threadIdx.x;
         u < (1ull << 32); u += static_cast<unsigned long long>(gridDim.x) * blockDim.x) {
        const float a = __uint_as_float(static_cast<unsigned>(u));
        if (!(fabsf(a) <= 4.0f) && !isnan(a)) continue;
        double angle = a;
        if (angle < 0) angle += kPi;
        const double deg = angle * 180.0 / kPi;
        const int want = (deg < 22.5 || deg >= 157.5) ? 0 : deg < 67.5 ? 1 : deg < 112.5 ? 2 : 3;
        int got;
        if (isnan(a)) {
            got = 3;
        } else {
            const float* t = a >= 0.0f ? th.pos : th.neg;
            got = a < t[0] ? 0 : a < t[1] ? 1 : a < t[2] ? 2 : a < t[3] ? 3 : 0;
        }
        miss += got != want;
    }
    if (miss) atomicAdd(bad, miss);
}

// host: deg of contour.cpp:217-219 for the float atan2 value a
double nms_deg(float a) {
    double angle = a;
    if (angle < 0) angle += kPi;
    return angle * 180.0 / kPi;
}
int32_t float_key(float f) {  // order-preserving int of a non-NaN float
    int32_t i;
    memcpy(&i, &f, 4);
    return i >= 0 ? i : static_cast<int32_t>(0x80000000u - static_cast<uint32_t>(i));
}
float key_float(int32_t k) {
    int32_t i = k >= 0 ? k : static_cast<int32_t>(0x80000000u - static_cast<uint32_t>(k));
    float f;
    memcpy(&f, &i, 4);
    return f;
}
// the smallest float a in [lo, hi] with nms_deg(a) >= b (hi's successor if none)
float nms_bound(float lo, float hi, double b) {
    int64_t l = float_key(lo), r = static_cast<int64_t>(float_key(hi)) + 1;  // answer in [l, r]
    while (l < r) {
        const int64_t mid = l + (r - l) / 2;
        if (nms_deg(key_float(static_cast<int32_t>(mid))) >= b) r = mid; else l = mid + 1;
    }
    return key_float(static_cast<int32_t>(l));
}
float f_up(double t) {  // smallest float >= t
    float f = static_cast<float>(t);
    if (static_cast<double>(f) < t) f = nextafterf(f, INFINITY);
    return f;
}
float f_down(double t) {  // largest float <= t
    float f = static_cast<float>(t);
    if (static_cast<double>(f) > t) f = nextafterf(f, -INFINITY);
    return f;
}
NmsThresholds nms_thresholds(const dco_config* cfg) {
    NmsThresholds th;
    const double b[4] = {22.5, 67.5, 112.5, 157.5};
    for (int k = 0; k < 4; ++k) {
        th.pos[k] = nms_bound(0.0f, INFINITY, b[k]);
        th.neg[k] = nms_bound(-INFINITY, -1.4e-45f, b[k]);
    }
    th.low = f_up(cfg->t_low);
    th.high = f_down(cfg->t_high);
    th.depth = f_up(cfg->t_depth);
    return th;
}

// ------------------------------------------------------------- hysteresis --
__device__ __forceinline__ int uf_find(int* parent, int a) {
    int p = parent[a];
    while (p != a) {
        int gp = parent[p];
        if (gp != p) parent[a] = gp;  // path halving (benign race: any ancestor is valid)
        a = p;
        p = parent[a];
    }
    return a;
}
__device__ __forceinline__ void uf_union(int* parent, int a, int b) {
    while (true) {
        a = uf_find(parent, a);
        b = uf_find(parent, b);
        if (a == b) return;
        if (a < b) {
            int t = a;
            a = b;
            b = t;
        }
        int old = atomicMin(&parent[a], b);
        if (old == a) return;
        a = old;
    }
}
__global__ void k_uf_init(const uint8_t* __restrict__ cls, size_t n, int* __restrict__ parent,
                          uint8_t* __restrict__ seeded) {
    size_t i = static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= n) return;
    parent[i] = static_cast<int>(i);
    seeded[i] = 0;
}
__global__ void k_uf_merge(const uint8_t* __restrict__ cls, int w, int h, int* __restrict__ parent) {
    int x = blockIdx.x * blockDim.x + threadIdx.x;
    int y = blockIdx.y * blockDim.y + threadIdx.y;
    if (x >= w || y >= h) return;
    int i = y * w + x;
    if (!cls[i]) return;
    // forward half of the 8-neighbourhood: every pair visited once
    if (x + 1 < w && cls[i + 1]) uf_union(parent, i, i + 1);
    if (y + 1 < h) {
        if (x > 0 && cls[i + w - 1]) uf_union(parent, i, i + w - 1);
        if (cls[i + w]) uf_union(parent, i, i + w);
        if (x + 1 < w && cls[i + w + 1]) uf_union(parent, i, i + w + 1);
    }
}
__global__ void k_uf_seed(const uint8_t* __restrict__ cls, size_t n, int* __restrict__ parent,
                          uint8_t* __restrict__ seeded) {
    size_t i = static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= n) return;
    if (cls[i] == 2) seeded[uf_find(parent, static_cast<int>(i))] = 1;
}
__global__ void k_uf_edges(const uint8_t* __restrict__ cls, size_t n, int* __restrict__ parent,
                           const uint8_t* __restrict__ seeded, uint8_t* __restrict__ edges) {
    size_t i = static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= n) return;
    uint8_t e = 0;
    if (cls[i]) e = seeded[uf_find(parent, static_cast<int>(i))];
    edges[i] = e;
}

inline dim3 grid2(int w, int h, dim3 b) { return dim3((w + b.x - 1) / b.x, (h + b.y - 1) / b.y); }

}  // namespace

// ===================================================================== host =

void flow_to_polar(dco_ctx* ctx, const float* u, const float* v, int w, int h, float* r, float* theta) {
    size_t n = static_cast<size_t>(w) * h;
    k_polar<<<blocks_for(n, 256), 256, 0, ctx->stream>>>(u, v, n, r, theta);
    launched(ctx, "k_polar");
}

void gradient_amplitude(dco_ctx* ctx, const float* r, int w, int h, float* amp) {
    dim3 b(32, 8);
    k_grad_amp<<<grid2(w, h, b), b, 0, ctx->stream>>>(r, w, h, amp);
    launched(ctx, "k_grad_amp");
}

void fuse_amplitudes(dco_ctx* ctx, const float* pu, const float* pv, const float* fu, const float* fv,
                     const float* mp, const float* mf, int w, int h, double k, float* out) {
    dim3 b(32, 8);
    k_fuse<<<grid2(w, h, b), b, 0, ctx->stream>>>(pu, pv, fu, fv, mp, mf, w, h, k, out);
    launched(ctx, "k_fuse");
}

// amplitude of both flows + fusion in one pass (pipeline.cpp:204-210).
void amplitude_fuse(dco_ctx* ctx, const float* pu, const float* pv, const float* fu, const float* fv,
                    int w, int h, double k, float* out) {
    dim3 b(32, 8);
    k_amp_fuse<<<grid2(w, h, b), b, 0, ctx->stream>>>(pu, pv, fu, fv, w, h, k, out);
    launched(ctx, "k_amp_fuse");
}

void box_filter(dco_ctx* ctx, const float* a, int w, int h, int radius, float* out) {
    if (radius < 1) fail(DCO_INPUT, "box_filter: radius must be >= 1");
    size_t n = static_cast<size_t>(w) * h;
    double* rows = static_cast<double*>(scratch(ctx, S_SAT, (n + (w + 1) * (h + 1) + 64) * sizeof(double)));
    double* sat = rows + n;
    k_box_rows<<<blocks_for(static_cast<size_t>(h) * 32, 256), 256, 0, ctx->stream>>>(a, w, h, rows);
    launched(ctx, "k_box_rows");
    k_box_cols<<<blocks_for(w + 1, 64), 64, 0, ctx->stream>>>(rows, w, h, sat);
    launched(ctx, "k_box_cols");
    dim3 b(32, 8);
    k_box_out<<<grid2(w, h, b), b, 0, ctx->stream>>>(sat, w, h, radius, out);
    launched(ctx, "k_box_out");
}

void normalize_amplitude(dco_ctx* ctx, const float* a, int w, int h, float* out) {
    size_t n = static_cast<size_t>(w) * h;
    unsigned* peak = static_cast<unsigned*>(scratch(ctx, S_FLAG_PEAK, 64));
    cuda_check(cudaMemsetAsync(peak, 0, sizeof(unsigned), ctx->stream), "memset");
    k_peak<<<blocks_for(n, 256), 256, 0, ctx->stream>>>(a, n, peak);
    launched(ctx, "k_peak");
    k_normalize<<<blocks_for(n, 256), 256, 0, ctx->stream>>>(a, n, peak, out);
    launched(ctx, "k_normalize");
}

void gaussian_blur(dco_ctx* ctx, const float* img, int w, int h, double sigma, float* out) {
    if (sigma <= 0.0) fail(DCO_INPUT, "gaussian_blur: sigma must be positive");
    Taps t;
    double norm = 0.0;
    for (int i = -2; i <= 2; ++i) {
        t.k[i + 2] = exp(-(i * i) / (2.0 * sigma * sigma));
        norm += t.k[i + 2];
    }
    for (double& v : t.k) v /= norm;
    size_t n = static_cast<size_t>(w) * h;
    float* tmp = static_cast<float*>(scratch(ctx, S_CONTOUR3, n * sizeof(float)));
    dim3 b(32, 8);
    k_gauss_h<<<grid2(w, h, b), b, 0, ctx->stream>>>(img, w, h, t, tmp);
    launched(ctx, "k_gauss_h");
    k_gauss_v<<<grid2(w, h, b), b, 0, ctx->stream>>>(tmp, w, h, t, out);
    launched(ctx, "k_gauss_v");
}

void extract_depth_contours_prefiltered(dco_ctx* ctx, const float* blurred, int w, int h,
                                        const float* mf, int qw, int qh, const dco_config* cfg,
                                        uint8_t* edges, float* m_i) {
    require(w >= 1 && h >= 1 && qw >= 1 && qh >= 1, "extract_depth_contours: empty input");
    size_t n = static_cast<size_t>(w) * h;
    float* gxy = static_cast<float*>(scratch(ctx, S_CONTOUR0, n * 3 * sizeof(float)));
    float* gx = gxy;
    float* gy = gxy + n;
    float* mag = gxy + 2 * n;
    uint8_t* cls = static_cast<uint8_t*>(scratch(ctx, S_CONTOUR1, n * 2));
    uint8_t* seeded = cls + n;
    int* parent = static_cast<int*>(scratch(ctx, S_LABELS, n * sizeof(int)));
    unsigned* peak = static_cast<unsigned*>(scratch(ctx, S_FLAG_PEAK, 64));
    cuda_check(cudaMemsetAsync(peak, 0, sizeof(unsigned), ctx->stream), "memset");
    dim3 b(32, 8);
    k_sobel<<<grid2(w, h, b), b, 0, ctx->stream>>>(blurred, w, h, gx, gy, mag, peak);
    launched(ctx, "k_sobel");
    k_mag_norm<<<blocks_for(n, 256), 256, 0, ctx->stream>>>(mag, n, peak, m_i);
    launched(ctx, "k_mag_norm");
    k_nms_gate<<<grid2(w, h, b), b, 0, ctx->stream>>>(gx, gy, mag, w, h, mf, qw, qh, nms_thresholds(cfg), cls);
    launched(ctx, "k_nms_gate");
    k_uf_init<<<blocks_for(n, 256), 256, 0, ctx->stream>>>(cls, n, parent, seeded);
    launched(ctx, "k_uf_init");
    k_uf_merge<<<grid2(w, h, b), b, 0, ctx->stream>>>(cls, w, h, parent);
    launched(ctx, "k_uf_merge");
    k_uf_seed<<<blocks_for(n, 256), 256, 0, ctx->stream>>>(cls, n, parent, seeded);
    launched(ctx, "k_uf_seed");
    k_uf_edges<<<blocks_for(n, 256), 256, 0, ctx->stream>>>(cls, n, parent, seeded, edges);
    launched(ctx, "k_uf_edges");
}

}  // namespace dco_gpu

using namespace dco_gpu;

extern "C" {

int dco_flow_to_polar(dco_ctx* ctx, const float* u, const float* v, int w, int h, float* r, float* theta) {
    return guarded(ctx, [&] { flow_to_polar(ctx, u, v, w, h, r, theta); });
}

int dco_gradient_amplitude(dco_ctx* ctx, const float* r, int w, int h, float* amp) {
    return guarded(ctx, [&] { gradient_amplitude(ctx, r, w, h, amp); });
}

int dco_fuse_amplitudes(dco_ctx* ctx, const float* pu, const float* pv, const float* fu, const float* fv,
                        const float* mp, const float* mf, int w, int h, const dco_config* cfg,
                        float* out) {
    return guarded(ctx, [&] { fuse_amplitudes(ctx, pu, pv, fu, fv, mp, mf, w, h, cfg->confidence_offset_k, out); });
}

int dco_box_filter(dco_ctx* ctx, const float* amp, int w, int h, int radius, float* out) {
    return guarded(ctx, [&] { box_filter(ctx, amp, w, h, radius, out); });
}

int dco_normalize_amplitude(dco_ctx* ctx, const float* amp, int w, int h, float* out) {
    return guarded(ctx, [&] { normalize_amplitude(ctx, amp, w, h, out); });
}

int dco_gaussian_blur(dco_ctx* ctx, const float* img, int w, int h, double sigma, float* out) {
    return guarded(ctx, [&] { gaussian_blur(ctx, img, w, h, sigma, out); });
}

int dco_extract_depth_contours_prefiltered(dco_ctx* ctx, const float* blurred, int w, int h,
                                           const float* mf, int qw, int qh, const dco_config* cfg,
                                           uint8_t* edges, float* m_i) {
    return guarded(ctx, [&] { extract_depth_contours_prefiltered(ctx, blurred, w, h, mf, qw, qh, cfg, edges, m_i); });
}

int dco_extract_depth_contours(dco_ctx* ctx, const float* gray, int w, int h, const float* mf, int qw,
                               int qh, const dco_config* cfg, uint8_t* edges, float* m_i) {
    return guarded(ctx, [&] {
        float* blurred = static_cast<float*>(scratch(ctx, S_CONTOUR2, static_cast<size_t>(w) * h * 4));
        gaussian_blur(ctx, gray, w, h, cfg->gauss_sigma, blurred);
        extract_depth_contours_prefiltered(ctx, blurred, w, h, mf, qw, qh, cfg, edges, m_i);
    });
}

__attribute__((visibility("default"))) int dco_debug_nms_check(unsigned long long* mismatches) {
    dco_config cfg;
    dco_config_default(&cfg);
    unsigned long long* d = nullptr;
    if (cudaMalloc(&d, 8) != cudaSuccess) return DCO_CUDA;
    cudaMemset(d, 0, 8);
    dco_gpu::k_nms_check<<<1184, 256>>>(dco_gpu::nms_thresholds(&cfg), d);
    const cudaError_t e = cudaMemcpy(mismatches, d, 8, cudaMemcpyDeviceToHost);
    cudaFree(d);
    return e == cudaSuccess ? DCO_OK : DCO_CUDA;
}

}  // extern "C"
