// stereo.cu — two-stage adaptive AD-census stereo (reference src/stereo.cpp,
// src/pyramid.cpp:5-17) as sm_100a kernels.
//
// Data layout in HBM (all row-major, the reference's own layouts so the C-ABI
// needs no transposes):
//   images          float [h][w]
//   cross arms      four u8 planes left/right/up/down [h][w]   (stereo.hpp:13-35)
//   census          u64 [h][w]                                 (stereo.hpp:40-47)
//   cost volumes    float [h][w][nd], d innermost              (stereo.hpp:50-63)
//   disparity       float [h][w], NaN = nodata                 (stereo.hpp:66-78)
//
// Parity: every kernel reproduces the reference's arithmetic order exactly;
// aggregation keeps the reference's sequential double prefix sums (one thread
// per (row, d) chain, then per (column, d) chain), so it is bit-exact by
// construction, not by luck (SURVEY §7.2 H1 option a).
#include <math.h>

#include <algorithm>

#include <map>
#include <mutex>
#include <utility>

#include "common.cuh"
#include "dco_exp_table.h"
#include "dco_libm.h"

namespace dco_gpu {

__device__ const uint64_t g_exp_table[2 * DCO_EXP_TABLE_N] = DCO_EXP_TABLE_INIT;

namespace {

// ---------------------------------------------------------------- pyramid --
// downsample_half, pyramid.cpp:5-17: ((a + b) + c) + d, times 0.25f.
__global__ void k_downsample(const float* __restrict__ img, int w, int h, float* __restrict__ out,
                             int ow, int oh) {
    int x = blockIdx.x * blockDim.x + threadIdx.x;
    int y = blockIdx.y * blockDim.y + threadIdx.y;
    if (x >= ow || y >= oh) return;
    const float* r0 = img + static_cast<size_t>(2 * y) * w + 2 * x;
    const float* r1 = r0 + w;
    float sum = r0[0] + r0[1] + r1[0] + r1[1];
    out[static_cast<size_t>(y) * ow + x] = sum * 0.25f;
}

// read_pnm (codec.cpp:80, bytes/255.0f) fused with downsample_half.
__global__ void k_ingest_gray8(const uint8_t* __restrict__ g8, int w, int h, float* __restrict__ full,
                               float* __restrict__ quarter, int qw, int qh) {
    int x = blockIdx.x * blockDim.x + threadIdx.x;
    int y = blockIdx.y * blockDim.y + threadIdx.y;
    if (x >= qw || y >= qh) return;
    size_t i0 = static_cast<size_t>(2 * y) * w + 2 * x, i1 = i0 + w;
    float a = g8[i0] / 255.0f, b = g8[i0 + 1] / 255.0f, c = g8[i1] / 255.0f, d = g8[i1 + 1] / 255.0f;
    if (full) {
        full[i0] = a;
        full[i0 + 1] = b;
        full[i1] = c;
        full[i1 + 1] = d;
    }
    if (quarter) quarter[static_cast<size_t>(y) * qw + x] = (a + b + c + d) * 0.25f;
}

// Odd trailing column/row of an odd-sized frame (not covered by the 2x2 pass).
// 128-bit variant (w % 8 == 0): a thread converts 8 x 2 bytes (two uint2
// loads), writes 2 x 2 float4 of the full image and one float4 of 4 quarter
// pixels; same arithmetic as k_ingest_gray8.
__global__ void k_ingest_gray8_v4(const uint8_t* __restrict__ g8, int w, int h, float* __restrict__ full,
                                  float* __restrict__ quarter, int qw, int qh) {
    const int x4 = blockIdx.x * blockDim.x + threadIdx.x;  // 4 quarter pixels
    const int y = blockIdx.y * blockDim.y + threadIdx.y;
    if (4 * x4 >= qw || y >= qh) return;
    const size_t i0 = static_cast<size_t>(2 * y) * w + 8 * x4, i1 = i0 + w;
    const uint2 r0 = *reinterpret_cast<const uint2*>(g8 + i0), r1 = *reinterpret_cast<const uint2*>(g8 + i1);
    float a[8], c[8];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
        a[j] = ((r0.x >> (8 * j)) & 255u) / 255.0f;
        a[4 + j] = ((r0.y >> (8 * j)) & 255u) / 255.0f;
        c[j] = ((r1.x >> (8 * j)) & 255u) / 255.0f;
        c[4 + j] = ((r1.y >> (8 * j)) & 255u) / 255.0f;
    }
    if (full) {
        float4* f0 = reinterpret_cast<float4*>(full + i0);
        float4* f1 = reinterpret_cast<float4*>(full + i1);
        f0[0] = make_float4(a[0], a[1], a[2], a[3]);
        f0[1] = make_float4(a[4], a[5], a[6], a[7]);
        f1[0] = make_float4(c[0], c[1], c[2], c[3]);
        f1[1] = make_float4(c[4], c[5], c[6], c[7]);
    }
    if (quarter) {
        float q[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) q[j] = (a[2 * j] + a[2 * j + 1] + c[2 * j] + c[2 * j + 1]) * 0.25f;
        *reinterpret_cast<float4*>(quarter + static_cast<size_t>(y) * qw + 4 * x4) = make_float4(q[0], q[1], q[2], q[3]);
    }
}
__global__ void k_ingest_gray8_tail(const uint8_t* __restrict__ g8, int w, int h,
                                    float* __restrict__ full) {
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    // indices: first the last column (if w odd), then the last row (if h odd)
    int ncol = (w & 1) ? h : 0, nrow = (h & 1) ? w : 0;
    if (i < ncol) {
        size_t p = static_cast<size_t>(i) * w + (w - 1);
        full[p] = g8[p] / 255.0f;
    } else if (i < ncol + nrow) {
        size_t p = static_cast<size_t>(h - 1) * w + (i - ncol);
        full[p] = g8[p] / 255.0f;
    }
}

// ----------------------------------------------------------- cross arms ----
// grow_arm, stereo.cpp:14-26: float |I(q) - I(p)| compared in double.
__device__ __forceinline__ int grow_arm(const float* img, int w, int h, int x, int y, int dx, int dy,
                                        int l1, int l2, double tau1, double tau2) {
    const float center = img[static_cast<size_t>(y) * w + x];
    int length = 0;
    for (int l = 1; l <= l1; ++l) {
        int qx = x + l * dx, qy = y + l * dy;
        if (qx < 0 || qy < 0 || qx >= w || qy >= h) break;
        double tau = l <= l2 ? tau1 : tau2;
        float diff = fabsf(img[static_cast<size_t>(qy) * w + qx] - center);
        if (static_cast<double>(diff) >= tau) break;
        length = l;
    }
    return length;
}

__global__ void k_cross_arms_raw(const float* __restrict__ img, int w, int h, int l1, int l2,
                                 double tau1, double tau2, uint8_t* __restrict__ raw) {
    int x = blockIdx.x * blockDim.x + threadIdx.x;
    int y = blockIdx.y * blockDim.y + threadIdx.y;
    if (x >= w || y >= h) return;
    size_t n = static_cast<size_t>(w) * h, i = static_cast<size_t>(y) * w + x;
    raw[i] = static_cast<uint8_t>(grow_arm(img, w, h, x, y, -1, 0, l1, l2, tau1, tau2));
    raw[n + i] = static_cast<uint8_t>(grow_arm(img, w, h, x, y, 1, 0, l1, l2, tau1, tau2));
    raw[2 * n + i] = static_cast<uint8_t>(grow_arm(img, w, h, x, y, 0, -1, l1, l2, tau1, tau2));
    raw[3 * n + i] = static_cast<uint8_t>(grow_arm(img, w, h, x, y, 0, 1, l1, l2, tau1, tau2));
}

// The same arms with float compares: for a float diff and a double tau,
// (double)diff >= tau  <=>  diff >= tf, tf the smallest float >= tau (host,
// arm_threshold), so no conversion or FP64 compare per step; the loop splits
// at l2 instead of selecting tau per step, and walks a pointer.
__device__ __forceinline__ int grow_arm_f(const float* p, long long step, float center, int lim, int l2, float t1,
                                          float t2) {
    int l = 0;
    const int n1 = min(lim, l2);
    while (l < n1) {
        p += step;
        if (fabsf(*p - center) >= t1) return l;
        ++l;
    }
    while (l < lim) {
        p += step;
        if (fabsf(*p - center) >= t2) return l;
        ++l;
    }
    return l;
}
__global__ void k_cross_arms_f(const float* __restrict__ img, int w, int h, int l1, int l2, float t1, float t2,
                               uint8_t* __restrict__ raw) {
    const int x = blockIdx.x * blockDim.x + threadIdx.x;
    const int y = blockIdx.y * blockDim.y + threadIdx.y;
    if (x >= w || y >= h) return;
    const size_t n = static_cast<size_t>(w) * h, i = static_cast<size_t>(y) * w + x;
    const float* p = img + i;
    const float c = *p;
    raw[i] = static_cast<uint8_t>(grow_arm_f(p, -1, c, min(l1, x), l2, t1, t2));
    raw[n + i] = static_cast<uint8_t>(grow_arm_f(p, 1, c, min(l1, w - 1 - x), l2, t1, t2));
    raw[2 * n + i] = static_cast<uint8_t>(grow_arm_f(p, -static_cast<long long>(w), c, min(l1, y), l2, t1, t2));
    raw[3 * n + i] = static_cast<uint8_t>(grow_arm_f(p, w, c, min(l1, h - 1 - y), l2, t1, t2));
}

// smooth_arm_channel, stereo.cpp:30-48: 3x3 clamped median (5th order
// statistic), clamped back to the raw reach. blockIdx.z = channel.
__global__ void k_arm_median(const uint8_t* __restrict__ raw, int w, int h, uint8_t* __restrict__ a0,
                             uint8_t* __restrict__ a1, uint8_t* __restrict__ a2,
                             uint8_t* __restrict__ a3) {
    int x = blockIdx.x * blockDim.x + threadIdx.x;
    int y = blockIdx.y * blockDim.y + threadIdx.y;
    int ch = blockIdx.z;
    if (x >= w || y >= h) return;
    const uint8_t* src = raw + static_cast<size_t>(ch) * w * h;
    int v[9];
    int n = 0;
    for (int dy = -1; dy <= 1; ++dy) {
        int yy = min(max(y + dy, 0), h - 1);
        for (int dx = -1; dx <= 1; ++dx) {
            int xx = min(max(x + dx, 0), w - 1);
            v[n++] = src[static_cast<size_t>(yy) * w + xx];
        }
    }
    // insertion sort of 9 small ints; v[4] is the median nth_element picks
#pragma unroll
    for (int i = 1; i < 9; ++i) {
#pragma unroll
        for (int j = i; j > 0; --j) {
            int lo = min(v[j - 1], v[j]), hi = max(v[j - 1], v[j]);
            v[j - 1] = lo;
            v[j] = hi;
        }
    }
    size_t i = static_cast<size_t>(y) * w + x;
    uint8_t out = static_cast<uint8_t>(min(v[4], static_cast<int>(src[i])));
    uint8_t* dst = ch == 0 ? a0 : ch == 1 ? a1 : ch == 2 ? a2 : a3;
    dst[i] = out;
}

// --------------------------------------------------------------- census ----
// census_transform, stereo.cpp:70-96: row-major window, centre skipped,
// clamped border, bit = neighbour darker than centre.
__global__ void k_census(const float* __restrict__ img, int w, int h, int rw, int rh,
                         uint64_t* __restrict__ out) {
    int x = blockIdx.x * blockDim.x + threadIdx.x;
    int y = blockIdx.y * blockDim.y + threadIdx.y;
    if (x >= w || y >= h) return;
    const float center = img[static_cast<size_t>(y) * w + x];
    uint64_t bits = 0;
    for (int dy = -rh; dy <= rh; ++dy) {
        int yy = min(max(y + dy, 0), h - 1);
        const float* row = img + static_cast<size_t>(yy) * w;
        for (int dx = -rw; dx <= rw; ++dx) {
            if (dx == 0 && dy == 0) continue;
            int xx = min(max(x + dx, 0), w - 1);
            bits = (bits << 1) | (row[xx] < center ? 1ull : 0ull);
        }
    }
    out[static_cast<size_t>(y) * w + x] = bits;
}

// census_transform over a shared-memory tile (the clamped window of a 32x8
// block staged once), both images of a stereo pair in one launch (z).
// RW0 / RH0 > 0: the window's half sizes as compile-time constants (the
// default 9x7), so the 62 compares unroll into fixed bit positions.
template <int RW0 = 0, int RH0 = 0>
__global__ void __launch_bounds__(256) k_census_tiled(const float* __restrict__ img0, const float* __restrict__ img1,
                                                      int w, int h, int rw_, int rh_, uint64_t* __restrict__ out0,
                                                      uint64_t* __restrict__ out1) {
    extern __shared__ float tile[];  // (32 + 2 rw) x (8 + 2 rh)
    const int rw = RW0 > 0 ? RW0 : rw_, rh = RH0 > 0 ? RH0 : rh_;
    const float* img = blockIdx.z ? img1 : img0;
    uint64_t* out = blockIdx.z ? out1 : out0;
    const int tw = 32 + 2 * rw, th = 8 + 2 * rh;
    const int x0 = blockIdx.x * 32 - rw, y0 = blockIdx.y * 8 - rh;
    for (int i = threadIdx.y * 32 + threadIdx.x; i < tw * th; i += 256) {
        const int ty = i / tw, tx = i - ty * tw;
        const int yy = min(max(y0 + ty, 0), h - 1), xx = min(max(x0 + tx, 0), w - 1);
        tile[i] = img[static_cast<size_t>(yy) * w + xx];
    }
    __syncthreads();
    const int x = blockIdx.x * 32 + threadIdx.x, y = blockIdx.y * 8 + threadIdx.y;
    if (x >= w || y >= h) return;
    const float* c = tile + (threadIdx.y + rh) * tw + threadIdx.x + rw;
    const float center = *c;
    uint64_t bits = 0;
    if constexpr (RW0 > 0 && RH0 > 0) {
        // bit of (dy, dx): row-major order, centre skipped, the first compare
        // ends as the most significant of the (2RW0+1)(2RH0+1)-1 bits
        constexpr int NB = (2 * RW0 + 1) * (2 * RH0 + 1) - 1;
        uint32_t hi = 0, lo = 0;  // bits 32..NB-1, bits 0..31
#pragma unroll
        for (int dy = -RH0; dy <= RH0; ++dy) {
#pragma unroll
            for (int dx = -RW0; dx <= RW0; ++dx) {
                if (dx == 0 && dy == 0) continue;
                const int k = (dy + RH0) * (2 * RW0 + 1) + (dx + RW0) - ((dy > 0 || (dy == 0 && dx > 0)) ? 1 : 0);
                const int pos = NB - 1 - k;
                const uint32_t b = c[dy * tw + dx] < center ? 1u : 0u;
                if (pos >= 32) {
                    hi |= b << (pos - 32);
                } else {
                    lo |= b << pos;
                }
            }
        }
        bits = (static_cast<uint64_t>(hi) << 32) | lo;
    } else {
        for (int dy = -rh; dy <= rh; ++dy) {
            const float* row = c + dy * tw;
            for (int dx = -rw; dx <= rw; ++dx) {
                if (dx == 0 && dy == 0) continue;
                bits = (bits << 1) | (row[dx] < center ? 1ull : 0ull);
            }
        }
    }
    out[static_cast<size_t>(y) * w + x] = bits;
}

// ------------------------------------------------------------ cost volume --
// compute_cost_volume, stereo.cpp:106-150. One thread per (pixel, d): the
// warp spans consecutive d of one pixel, so the [p][d] store is coalesced and
// the pixel's alpha/census/luminance loads are warp-uniform broadcasts.
constexpr int kCostPix = 64;  // pixels of one row per cost-volume block

struct CostParams {
    int w, h, nd, d_min, bits;
    double lambda_ad;
    double inv_lambda;  // RN(1 / lambda_ad)
    int fast_div;       // div_lambda proven equal to the division for every |dI| in [0, 1]
    double alpha[256];
    double census[65];
};

// c / lambda from RN(1/lambda): the product and one FMA correction. For a
// given lambda the host proves it equal to the IEEE division for every
// c = |dI| * 255 with |dI| a float in [0, 1] (k_verify_div, all 1.07e9 of
// them) before enabling it; other inputs take the division.
__device__ __forceinline__ double div_lambda(double c, double lam, double inv) {
    const double q = c * inv;
    return __fma_rn(__fma_rn(-q, lam, c), inv, q);
}

__global__ void k_verify_div(double lam, double inv, unsigned* __restrict__ bad) {
    const unsigned n = 0x3f800001u;  // float bit patterns of [0, 1]
    unsigned miss = 0;
    for (unsigned u = blockIdx.x * blockDim.x + threadIdx.x; u < n; u += gridDim.x * blockDim.x) {
        const double c = static_cast<double>(__uint_as_float(u)) * 255.0;
        miss |= __double_as_longlong(div_lambda(c, lam, inv)) != __double_as_longlong(c / lam) ? 1u : 0u;
    }
    if (__any_sync(0xffffffffu, miss) && (threadIdx.x & 31) == 0) atomicOr(bad, 1u);
}

__global__ void __launch_bounds__(512) k_cost_volume(const float* __restrict__ left,
                                                     const float* __restrict__ right,
                                                     const uint64_t* __restrict__ cl,
                                                     const uint64_t* __restrict__ cr,
                                                     const uint8_t* __restrict__ armL,
                                                     const uint8_t* __restrict__ armR,
                                                     const uint8_t* __restrict__ armU,
                                                     const uint8_t* __restrict__ armD,
                                                     const __grid_constant__ CostParams prm_v,
                                                     float* __restrict__ cost) {
    const CostParams* prm = &prm_v;
    __shared__ uint64_t s_exp[2 * DCO_EXP_TABLE_N];
    __shared__ double s_census[65];
    for (int i = threadIdx.x; i < 2 * DCO_EXP_TABLE_N; i += blockDim.x) s_exp[i] = g_exp_table[i];
    for (int i = threadIdx.x; i < 65; i += blockDim.x) s_census[i] = prm->census[i];
    __syncthreads();
    // block = (32 lanes over d) x (blockDim.y pixels); a block walks kCostPix
    // pixels of one row, so no per-element index division is needed.
    const int w = prm->w, nd = prm->nd;
    const int y = blockIdx.y;
    const int lane = threadIdx.x;
    for (int xi = threadIdx.y; xi < kCostPix; xi += blockDim.y) {
        const int x = blockIdx.x * kCostPix + xi;
        if (x >= w) break;
        const size_t p = static_cast<size_t>(y) * w + x;
        const int m = min(min(armL[p], armR[p]), min(armU[p], armD[p]));
        const double alpha = prm->alpha[m];
        const double beta = 1.0 - alpha;
        const float lum = left[p];
        const uint64_t cp = cl[p];
        float* dst = cost + p * nd;
        for (int k = lane; k < nd; k += 32) {
            const int d = prm->d_min + k;
            const int qx = x - d;
            float c;
            if (qx < 0) {
                c = 2.0f;
            } else {
                const size_t q = p - static_cast<size_t>(d);
                const float adi = fabsf(lum - right[q]);
                const double c_ad = static_cast<double>(adi) * 255.0;
                // -c_ad / lambda (stereo.cpp:141): the proven fast quotient inside [0, 1]
                const double quo = (prm->fast_div && adi <= 1.0f) ? div_lambda(c_ad, prm->lambda_ad, prm->inv_lambda)
                                                                  : c_ad / prm->lambda_ad;
                double ad_term = 1.0 - dco_exp(-quo, s_exp);
                int hd = __popcll(cp ^ cr[q]);
                c = static_cast<float>(alpha * ad_term + beta * s_census[hd]);
            }
            dst[k] = c;
        }
    }
}

// ------------------------------------------------------------ aggregation --
// aggregate_costs, stereo.cpp:152-218.
// region_size (stereo.cpp:157-177): sum of horizontal spans along the vertical
// arm; integer valued, so any summation order is exact.
__global__ void k_region_size(const uint8_t* __restrict__ L, const uint8_t* __restrict__ R,
                              const uint8_t* __restrict__ U, const uint8_t* __restrict__ D, int w,
                              int h, int* __restrict__ region) {
    int x = blockIdx.x * blockDim.x + threadIdx.x;
    int y = blockIdx.y * blockDim.y + threadIdx.y;
    if (x >= w || y >= h) return;
    size_t i = static_cast<size_t>(y) * w + x;
    int s = 0;  // region_size (stereo.cpp:157-177): integer, any order
    const int y1 = y + D[i];
    constexpr int kB = 8;  // rows' loads in flight at a time
    for (int yb = y - U[i]; yb <= y1; yb += kB) {
        int v[kB];
#pragma unroll
        for (int j = 0; j < kB; ++j) {
            const size_t q = static_cast<size_t>(yb + j) * w + x;
            v[j] = yb + j <= y1 ? L[q] + R[q] + 1 : 0;
        }
#pragma unroll
        for (int j = 0; j < kB; ++j) s += v[j];
    }
    region[i] = s;
}

// Horizontal pass (stereo.cpp:191-201): one thread owns the (row y, slice k)
// chain and walks x in order, P[x+1] = P[x] + cost, exactly the reference's
// sequential double prefix. The last 2*l1+2 prefix values live in a per-thread
// shared-memory ring; pixel px is finalised once P[px+l1+1] exists:
// hsum = P[px+right+1] - P[px-left].
__global__ void k_agg_hpass(const float* __restrict__ cost, int w, int h, int nd,
                            const uint8_t* __restrict__ L, const uint8_t* __restrict__ R,
                            int lag, int ring_mask, double* __restrict__ hsum) {
    extern __shared__ double ring[];
    const int lane = threadIdx.x, tid = threadIdx.y * blockDim.x + threadIdx.x;
    const int stride = blockDim.x * blockDim.y;
    const int k = blockIdx.x * blockDim.x + lane;
    const int y = blockIdx.y * blockDim.y + threadIdx.y;
    if (y >= h || k >= nd) return;
    const float* src = cost + static_cast<size_t>(y) * w * nd + k;
    double* dst = hsum + static_cast<size_t>(y) * w * nd + k;
    const uint8_t* Lr = L + static_cast<size_t>(y) * w;
    const uint8_t* Rr = R + static_cast<size_t>(y) * w;
    double P = 0.0;
    ring[tid] = 0.0;
    // software pipeline: the next kPF costs are in flight while the current
    // kPF steps of the (inherently sequential) prefix chain execute
    constexpr int kPF = 16;
    float cur[kPF], nxt[kPF];
#pragma unroll
    for (int j = 0; j < kPF; ++j) cur[j] = j < w ? __ldg(src + static_cast<size_t>(j) * nd) : 0.0f;
    for (int x0 = 0; x0 < w; x0 += kPF) {
#pragma unroll
        for (int j = 0; j < kPF; ++j) {
            int x = x0 + kPF + j;
            nxt[j] = x < w ? __ldg(src + static_cast<size_t>(x) * nd) : 0.0f;
        }
        int la[kPF], ra[kPF];
#pragma unroll
        for (int j = 0; j < kPF; ++j) {
            int px = x0 + j + 1 - lag;
            la[j] = ra[j] = 0;
            if (px >= 0 && px < w) {
                la[j] = __ldg(Lr + px);
                ra[j] = __ldg(Rr + px);
            }
        }
#pragma unroll
        for (int j = 0; j < kPF; ++j) {
            int x = x0 + j;
            if (x < w) {
                P += static_cast<double>(cur[j]);
                ring[((x + 1) & ring_mask) * stride + tid] = P;
                int px = x + 1 - lag;
                if (px >= 0) {
                    int a = px - la[j], b = px + ra[j] + 1;
                    dst[static_cast<size_t>(px) * nd] =
                        ring[(b & ring_mask) * stride + tid] - ring[(a & ring_mask) * stride + tid];
                }
            }
        }
#pragma unroll
        for (int j = 0; j < kPF; ++j) cur[j] = nxt[j];
    }
    for (int px = max(w + 1 - lag, 0); px < w; ++px) {
        int a = px - Lr[px], b = px + Rr[px] + 1;
        dst[static_cast<size_t>(px) * nd] =
            ring[(b & ring_mask) * stride + tid] - ring[(a & ring_mask) * stride + tid];
    }
}

// Vertical pass (stereo.cpp:203-215): one thread owns the (column x, slice k)
// chain; C[y+1] = C[y] + hsum; total = C[py+down+1] - C[py-up];
// out = float(total / region_size).
__global__ void k_agg_vpass(const double* __restrict__ hsum, int w, int h, int nd,
                            const uint8_t* __restrict__ U, const uint8_t* __restrict__ D,
                            const int* __restrict__ region, int lag, int ring_mask,
                            float* __restrict__ out) {
    extern __shared__ double ring[];
    const int lane = threadIdx.x, tid = threadIdx.y * blockDim.x + threadIdx.x;
    const int stride = blockDim.x * blockDim.y;
    const int k = blockIdx.x * blockDim.x + lane;
    const int x = blockIdx.y * blockDim.y + threadIdx.y;
    if (x >= w || k >= nd) return;
    const size_t row = static_cast<size_t>(w) * nd;
    const double* src = hsum + static_cast<size_t>(x) * nd + k;
    float* dst = out + static_cast<size_t>(x) * nd + k;
    double C = 0.0;
    ring[tid] = 0.0;
    constexpr int kPF = 16;
    double cur[kPF], nxt[kPF];
#pragma unroll
    for (int j = 0; j < kPF; ++j) cur[j] = j < h ? __ldg(src + j * row) : 0.0;
    for (int y0 = 0; y0 < h; y0 += kPF) {
#pragma unroll
        for (int j = 0; j < kPF; ++j) {
            int y = y0 + kPF + j;
            nxt[j] = y < h ? __ldg(src + y * row) : 0.0;
        }
        // the arms / region sizes of the kPF pixels finalised in this chunk
        int ua[kPF], da[kPF], rg[kPF];
#pragma unroll
        for (int j = 0; j < kPF; ++j) {
            int py = y0 + j + 1 - lag;
            ua[j] = da[j] = rg[j] = 1;
            if (py >= 0 && py < h) {
                size_t i = static_cast<size_t>(py) * w + x;
                ua[j] = __ldg(U + i);
                da[j] = __ldg(D + i);
                rg[j] = __ldg(region + i);
            }
        }
#pragma unroll
        for (int j = 0; j < kPF; ++j) {
            int y = y0 + j;
            if (y < h) {
                C += cur[j];
                ring[((y + 1) & ring_mask) * stride + tid] = C;
                int py = y + 1 - lag;
                if (py >= 0) {
                    int a = py - ua[j], b = py + da[j] + 1;
                    double total = ring[(b & ring_mask) * stride + tid] - ring[(a & ring_mask) * stride + tid];
                    dst[py * row] = static_cast<float>(total / rg[j]);
                }
            }
        }
#pragma unroll
        for (int j = 0; j < kPF; ++j) cur[j] = nxt[j];
    }
    for (int py = max(h + 1 - lag, 0); py < h; ++py) {
        size_t i = static_cast<size_t>(py) * w + x;
        int a = py - U[i], b = py + D[i] + 1;
        double total = ring[(b & ring_mask) * stride + tid] - ring[(a & ring_mask) * stride + tid];
        dst[py * row] = static_cast<float>(total / region[i]);
    }
}

// Packed per-pixel arm words for the pipelined passes below:
// hinfo = left | right << 8; vinfo = up | down << 8 | region << 16 (region
// < 65536 whenever every arm <= 127, which the host checks).
__global__ void k_region_pack(const uint8_t* __restrict__ L, const uint8_t* __restrict__ R,
                              const uint8_t* __restrict__ U, const uint8_t* __restrict__ D, int w, int h,
                              uint32_t* __restrict__ hinfo, uint32_t* __restrict__ vinfo) {
    int x = blockIdx.x * blockDim.x + threadIdx.x;
    int y = blockIdx.y * blockDim.y + threadIdx.y;
    if (x >= w || y >= h) return;
    size_t i = static_cast<size_t>(y) * w + x;
    int s = 0;  // region_size (stereo.cpp:157-177): integer, any order
    const int y1 = y + D[i];
    constexpr int kB = 8;  // rows' loads in flight at a time
    for (int yb = y - U[i]; yb <= y1; yb += kB) {
        int v[kB];
#pragma unroll
        for (int j = 0; j < kB; ++j) {
            const size_t q = static_cast<size_t>(yb + j) * w + x;
            v[j] = yb + j <= y1 ? L[q] + R[q] + 1 : 0;
        }
#pragma unroll
        for (int j = 0; j < kB; ++j) s += v[j];
    }
    hinfo[i] = L[i] | (static_cast<uint32_t>(R[i]) << 8);
    vinfo[i] = U[i] | (static_cast<uint32_t>(D[i]) << 8) | (static_cast<uint32_t>(s) << 16);
}

// Pipelined horizontal pass: same chain and rounding as k_agg_hpass. Block
// = 32 slices x 4 rows (kAggThreads). The per-thread prefix ring holds
// exactly 2*l1+2 entries (modular slots, so more blocks fit per SM); the
// costs and the arm words of the next kPF steps are in flight while the
// current kPF steps execute; chunks away from the borders run without
// per-step bounds checks.
constexpr int kAggThreads = 128;

template <int kPF>
__global__ void __launch_bounds__(kAggThreads) k_agg_h2(const float* __restrict__ cost, int w, int h, int nd,
                                                        const uint32_t* __restrict__ hinfo, int lag, int ring_n,
                                                        double* __restrict__ hsum) {
    extern __shared__ double ring[];
    const int lane = threadIdx.x, tid = threadIdx.y * 32 + threadIdx.x;
    const int k = blockIdx.x * 32 + lane;
    const int y = blockIdx.y * 4 + threadIdx.y;
    if (y >= h || k >= nd) return;
    const float* lp = cost + static_cast<size_t>(y) * w * nd + k;  // next cost to load
    double* dst = hsum + static_cast<size_t>(y) * w * nd + k;
    const uint32_t* info = hinfo + static_cast<size_t>(y) * w;
    double* rg = ring + tid;
    double P = 0.0;
    rg[0] = 0.0;
    int s1 = 0;  // slot of P[x + 1] after step x
    float cur[kPF], nxt[kPF];
    uint32_t ci[kPF], ni[kPF];
#pragma unroll
    for (int j = 0; j < kPF; ++j) {
        cur[j] = j < w ? __ldg(lp) : 0.0f;
        lp += nd;
        const int px = j + 1 - lag;
        ci[j] = (px >= 0 && px < w) ? __ldg(info + px) : 0u;
    }
    auto step = [&](int x, float c, uint32_t v) {
        P += static_cast<double>(c);
        s1 = (s1 + 1 == ring_n) ? 0 : s1 + 1;
        rg[s1 * kAggThreads] = P;
        const int l = v & 255u, r = (v >> 8) & 255u;
        int ib = s1 + r + 1 - lag;  // P[px + r + 1]
        ib += ib < 0 ? ring_n : 0;
        int ia = s1 - lag - l;  // P[px - l]
        ia += ia < 0 ? ring_n : 0;
        return rg[ib * kAggThreads] - rg[ia * kAggThreads];
    };
    for (int x0 = 0; x0 < w; x0 += kPF) {
        const bool fast = x0 + 2 * kPF <= w && x0 + 1 - lag >= 0;
        if (fast) {
#pragma unroll
            for (int j = 0; j < kPF; ++j) {
                nxt[j] = __ldg(lp);
                lp += nd;
                ni[j] = __ldg(info + x0 + kPF + j + 1 - lag);
            }
            const int sb = s1;
#pragma unroll
            for (int j = 0; j < kPF; ++j) {
                P += static_cast<double>(cur[j]);
                s1 = (s1 + 1 == ring_n) ? 0 : s1 + 1;
                rg[s1 * kAggThreads] = P;
            }
            double* dp = dst + static_cast<size_t>(x0 + 1 - lag) * nd;
            int sj = sb;
#pragma unroll
            for (int j = 0; j < kPF; ++j) {
                sj = (sj + 1 == ring_n) ? 0 : sj + 1;  // slot of P[x0 + j + 1]
                const uint32_t v = ci[j];
                const int l = v & 255u, r = (v >> 8) & 255u;
                int ib = sj + r + 1 - lag;
                ib += ib < 0 ? ring_n : 0;
                int ia = sj - lag - l;
                ia += ia < 0 ? ring_n : 0;
                *dp = rg[ib * kAggThreads] - rg[ia * kAggThreads];
                dp += nd;
            }
        } else {
#pragma unroll
            for (int j = 0; j < kPF; ++j) {
                const int x = x0 + kPF + j;
                nxt[j] = x < w ? __ldg(lp) : 0.0f;
                lp += nd;
                const int px = x + 1 - lag;
                ni[j] = (px >= 0 && px < w) ? __ldg(info + px) : 0u;
            }
#pragma unroll
            for (int j = 0; j < kPF; ++j) {
                const int x = x0 + j;
                if (x < w) {
                    const int px = x + 1 - lag;
                    if (px >= 0) {
                        dst[static_cast<size_t>(px) * nd] = step(x, cur[j], ci[j]);
                    } else {
                        P += static_cast<double>(cur[j]);
                        s1 = (s1 + 1 == ring_n) ? 0 : s1 + 1;
                        rg[s1 * kAggThreads] = P;
                    }
                }
            }
        }
#pragma unroll
        for (int j = 0; j < kPF; ++j) {
            cur[j] = nxt[j];
            ci[j] = ni[j];
        }
    }
    // s1 = slot of P[w]
    for (int px = max(w + 1 - lag, 0); px < w; ++px) {
        const uint32_t v = info[px];
        const int l = v & 255u, r = (v >> 8) & 255u;
        int ib = s1 + (px + r + 1 - w);
        ib += ib < 0 ? ring_n : 0;
        int ia = s1 + (px - l - w);
        ia += ia < 0 ? ring_n : 0;
        dst[static_cast<size_t>(px) * nd] = rg[ib * kAggThreads] - rg[ia * kAggThreads];
    }
}

// Pipelined vertical pass: same chain, rounding and division as k_agg_vpass.
// Block = 32 slices x 4 columns.
// kBand (row bands, DESIGN 7): the column prefix starts at row c0 from the
// exact prefix of the rows above the band (carry_in, [d - k0][x] doubles, or
// 0) -- rows < c0 add nothing -- and the prefix before row e is exported to
// carry_out for the next band. Same chain, so the exact rows are bit-equal to
// the whole frame's. Slices [k0, k1) only (a chunk of the carry chain).
template <int kPF, bool kBand = false>
__global__ void __launch_bounds__(kAggThreads) k_agg_v2(const double* __restrict__ hsum, int w, int h, int nd,
                                                        const uint32_t* __restrict__ vinfo, int lag, int ring_n,
                                                        float* __restrict__ out, const double* __restrict__ carry_in = nullptr,
                                                        int c0 = 0, double* __restrict__ carry_out = nullptr,
                                                        int e = -1, int k0 = 0, int k1 = 0) {
    extern __shared__ double ring[];
    const int lane = threadIdx.x, tid = threadIdx.y * 32 + threadIdx.x;
    const int k = (kBand ? k0 : 0) + blockIdx.x * 32 + lane;
    const int x = blockIdx.y * 4 + threadIdx.y;
    if (x >= w || k >= (kBand ? k1 : nd)) return;
    const size_t row = static_cast<size_t>(w) * nd;
    const double* lp = hsum + static_cast<size_t>(x) * nd + k;
    float* dst = out + static_cast<size_t>(x) * nd + k;
    const uint32_t* info = vinfo + x;
    double* rg = ring + tid;
    double C = 0.0;
    if (kBand && carry_in) C = carry_in[static_cast<size_t>(k - k0) * w + x];
    rg[0] = C;
    int s1 = 0;
    auto note = [&](int y) {  // C is now the prefix before row y + 1
        if (kBand && y + 1 == e) carry_out[static_cast<size_t>(k - k0) * w + x] = C;
    };
    auto live = [&](int y) { return !kBand || y >= c0; };
    double cur[kPF], nxt[kPF];
    uint32_t ci[kPF], ni[kPF];
#pragma unroll
    for (int j = 0; j < kPF; ++j) {
        cur[j] = (j < h && live(j)) ? __ldg(lp) : 0.0;
        lp += row;
        const int py = j + 1 - lag;
        ci[j] = (py >= 0 && py < h) ? __ldg(info + static_cast<size_t>(py) * w) : 0u;
    }
    auto step = [&](double c, uint32_t v) {
        C += c;
        s1 = (s1 + 1 == ring_n) ? 0 : s1 + 1;
        rg[s1 * kAggThreads] = C;
        const int u = v & 255u, d = (v >> 8) & 255u;
        int ib = s1 + d + 1 - lag;
        ib += ib < 0 ? ring_n : 0;
        int ia = s1 - lag - u;
        ia += ia < 0 ? ring_n : 0;
        const double total = rg[ib * kAggThreads] - rg[ia * kAggThreads];
        return static_cast<float>(total / static_cast<int>(v >> 16));
    };
    for (int y0 = 0; y0 < h; y0 += kPF) {
        const bool fast = y0 + 2 * kPF <= h && y0 + 1 - lag >= 0;
        if (fast) {
            const uint32_t* ip = info + static_cast<size_t>(y0 + kPF + 1 - lag) * w;
#pragma unroll
            for (int j = 0; j < kPF; ++j) {
                nxt[j] = live(y0 + kPF + j) ? __ldg(lp) : 0.0;
                lp += row;
                ni[j] = __ldg(ip);
                ip += w;
            }
            // prefixes of the whole chunk first, then its kPF outputs: no
            // shared-memory store sits between two outputs' loads
            const int sb = s1;
#pragma unroll
            for (int j = 0; j < kPF; ++j) {
                C += cur[j];
                s1 = (s1 + 1 == ring_n) ? 0 : s1 + 1;
                rg[s1 * kAggThreads] = C;
                note(y0 + j);
            }
            float* dp = dst + static_cast<size_t>(y0 + 1 - lag) * row;
            int sj = sb;
#pragma unroll
            for (int j = 0; j < kPF; ++j) {
                sj = (sj + 1 == ring_n) ? 0 : sj + 1;  // slot of C[y0 + j + 1]
                const uint32_t v = ci[j];
                const int u = v & 255u, d = (v >> 8) & 255u;
                int ib = sj + d + 1 - lag;
                ib += ib < 0 ? ring_n : 0;
                int ia = sj - lag - u;
                ia += ia < 0 ? ring_n : 0;
                const double total = rg[ib * kAggThreads] - rg[ia * kAggThreads];
                *dp = static_cast<float>(total / static_cast<int>(v >> 16));
                dp += row;
            }
        } else {
#pragma unroll
            for (int j = 0; j < kPF; ++j) {
                const int y = y0 + kPF + j;
                nxt[j] = (y < h && live(y)) ? __ldg(lp) : 0.0;
                lp += row;
                const int py = y + 1 - lag;
                ni[j] = (py >= 0 && py < h) ? __ldg(info + static_cast<size_t>(py) * w) : 0u;
            }
#pragma unroll
            for (int j = 0; j < kPF; ++j) {
                const int y = y0 + j;
                if (y < h) {
                    const int py = y + 1 - lag;
                    if (py >= 0) {
                        dst[py * row] = step(cur[j], ci[j]);
                    } else {
                        C += cur[j];
                        s1 = (s1 + 1 == ring_n) ? 0 : s1 + 1;
                        rg[s1 * kAggThreads] = C;
                    }
                    note(y);
                }
            }
        }
#pragma unroll
        for (int j = 0; j < kPF; ++j) {
            cur[j] = nxt[j];
            ci[j] = ni[j];
        }
    }
    for (int py = max(h + 1 - lag, 0); py < h; ++py) {
        const uint32_t v = info[static_cast<size_t>(py) * w];
        const int u = v & 255u, d = (v >> 8) & 255u;
        int ib = s1 + (py + d + 1 - h);
        ib += ib < 0 ? ring_n : 0;
        int ia = s1 + (py - u - h);
        ia += ia < 0 ? ring_n : 0;
        const double total = rg[ib * kAggThreads] - rg[ia * kAggThreads];
        dst[py * row] = static_cast<float>(total / static_cast<int>(v >> 16));
    }
}

// ------------------------------------------------------------------- WTA ---
// select_disparity_wta, stereo.cpp:220-238: first strict minimum. One warp
// per pixel; lanes stride over d and the warp reduces (cost, d) with ties to
// the smaller d, which is the sequential first-minimum for non-NaN costs; a
// NaN at d_min freezes the reference's scan at 0 and is honoured explicitly.
__global__ void k_wta(const float* __restrict__ cost, int npix, int nd, int d_min,
                      float* __restrict__ disp) {
    const int lane = threadIdx.x & 31;
    const size_t p = (static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    if (p >= static_cast<size_t>(npix)) return;
    const float* c = cost + p * nd;
    float best = INFINITY;
    int bi = nd;
    for (int k = lane; k < nd; k += 32) {
        float v = c[k];
        if (v < best) {
            best = v;
            bi = k;
        }
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
        float ob = __shfl_xor_sync(0xffffffffu, best, off);
        int oi = __shfl_xor_sync(0xffffffffu, bi, off);
        if (ob < best || (ob == best && oi < bi)) {
            best = ob;
            bi = oi;
        }
    }
    if (lane == 0) {
        float c0 = c[0];
        if (c0 != c0 || bi >= nd) bi = 0;  // NaN first cost, or all remaining NaN
        // a cost equal to +inf everywhere also lands on 0 (first element wins)
        disp[p] = static_cast<float>(d_min + bi);
    }
}

// ----------------------------------------------------- histogram refine ----
// refine_disparity_histogram, stereo.cpp:240-299. bin_max over the input.
__global__ void k_bin_max(const float* __restrict__ disp, int n, int* __restrict__ out) {
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    int b = 0;
    if (i < n) {
        float v = disp[i];
        if (isfinite(v)) b = max(0, static_cast<int>(lroundf(v)));
    }
    block_atomic_max(out, b);
}

// One warp per pixel (grid-stride over pixels). The cross region — the
// horizontal spans of the pixels on the centre's vertical arm — is flattened
// so all 32 lanes sample it in parallel; per 32 samples __match_any_sync
// groups equal bins and one leader per distinct bin adds the group size to the
// warp's shared-memory histogram (no atomics needed). Mode = max count, the
// smaller bin winning ties, exactly the reference's ascending scan; only the
// touched bin range is scanned and cleared.
__global__ void __launch_bounds__(256) k_hist_refine(const float* __restrict__ cur, int w, int h,
                                                     const uint8_t* __restrict__ L, const uint8_t* __restrict__ R,
                                                     const uint8_t* __restrict__ U, const uint8_t* __restrict__ D,
                                                     const int* __restrict__ bin_max_ptr, int nbins_cap, int rows_cap,
                                                     float* __restrict__ next) {
    extern __shared__ unsigned dyn[];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int per_warp = nbins_cap + 3 * rows_cap + 1;
    unsigned* hist = dyn + static_cast<size_t>(warp) * per_warp;
    int* roff = reinterpret_cast<int*>(hist + nbins_cap);  // rows_cap + 1 offsets
    int* rx = roff + rows_cap + 1;                         // first column of each row span
    int* ry = rx + rows_cap;                               // row index
    const int bin_max = *bin_max_ptr;
    const int nb = min(bin_max + 1, nbins_cap);
    for (int b = lane; b < nb; b += 32) hist[b] = 0u;
    __syncwarp();
    const size_t npix = static_cast<size_t>(w) * h;
    const size_t nwarps = static_cast<size_t>(gridDim.x) * (blockDim.x >> 5);
    for (size_t p = static_cast<size_t>(blockIdx.x) * (blockDim.x >> 5) + warp; p < npix; p += nwarps) {
        const float center = cur[p];
        if (!isfinite(center)) {
            if (lane == 0) next[p] = center;  // removed outliers stay removed
            continue;
        }
        const int x = static_cast<int>(p % w), y = static_cast<int>(p / w);
        const int up = U[p], nrows = up + D[p] + 1;
        // row spans and their exclusive prefix (flattened offsets)
        int total = 0;
        for (int rb = 0; rb < nrows; rb += 32) {
            int r = rb + lane, len = 0;
            if (r < nrows) {
                int vy = y - up + r;
                size_t vi = static_cast<size_t>(vy) * w + x;
                int l = L[vi];
                len = l + R[vi] + 1;
                rx[r] = x - l;
                ry[r] = vy;
            }
            int inc = len;
#pragma unroll
            for (int off = 1; off < 32; off <<= 1) {
                int o = __shfl_up_sync(0xffffffffu, inc, off);
                if (lane >= off) inc += o;
            }
            if (r < nrows) roff[r] = total + inc - len;
            total += __shfl_sync(0xffffffffu, inc, 31);
        }
        if (lane == 0) roff[nrows] = total;
        __syncwarp();
        int count = 0, lo = bin_max, hi = 0, row = 0;
        for (int f0 = 0; f0 < total; f0 += 32) {
            int f = f0 + lane;
            int bin = -1;
            if (f < total) {
                while (roff[row + 1] <= f) ++row;
                float v = cur[static_cast<size_t>(ry[row]) * w + rx[row] + (f - roff[row])];
                if (isfinite(v)) {
                    bin = min(max(static_cast<int>(lroundf(v)), 0), nb - 1);
                    ++count;
                    lo = min(lo, bin);
                    hi = max(hi, bin);
                }
            }
            unsigned grp = __match_any_sync(0xffffffffu, bin);
            if (bin >= 0 && lane == __ffs(grp) - 1) hist[bin] += __popc(grp);
            __syncwarp();
        }
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) {
            count += __shfl_xor_sync(0xffffffffu, count, off);
            lo = min(lo, __shfl_xor_sync(0xffffffffu, lo, off));
            hi = max(hi, __shfl_xor_sync(0xffffffffu, hi, off));
        }
        int best_c = 0, best_b = lo;
        for (int b = lo + lane; b <= hi; b += 32) {
            int cnt = static_cast<int>(hist[b]);
            hist[b] = 0u;
            if (cnt > best_c) {
                best_c = cnt;
                best_b = b;
            }
        }
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) {
            int oc = __shfl_xor_sync(0xffffffffu, best_c, off);
            int ob = __shfl_xor_sync(0xffffffffu, best_b, off);
            if (oc > best_c || (oc == best_c && ob < best_b)) {
                best_c = oc;
                best_b = ob;
            }
        }
        if (lane == 0) {
            if (best_c == 1 && count >= 4)
                next[p] = __int_as_float(0x7fc00000);  // quiet NaN nodata
            else
                next[p] = static_cast<float>(best_b);
        }
        __syncwarp();
    }
}


// Thread per pixel: a private 16-bit histogram column per thread in shared
// memory ([bin][thread], conflict-free), filled by walking the cross region
// row by row (counts are integers: any order is exact), then the reference's
// ascending mode scan over the touched bin range, which is cleared for the
// next pixel. Used when the bin range fits (<= 256 bins); otherwise the
// warp-per-pixel kernel above.
constexpr int kHistThreads = 128;

__global__ void __launch_bounds__(kHistThreads) k_hist_refine_thread(
    const float* __restrict__ cur, int w, int h, const uint8_t* __restrict__ L, const uint8_t* __restrict__ R,
    const uint8_t* __restrict__ U, const uint8_t* __restrict__ D, const int* __restrict__ bin_max_ptr, int nbins_cap,
    float* __restrict__ next) {
    extern __shared__ unsigned short hcol[];  // [nbins_cap][kHistThreads]
    const int t = threadIdx.x;
    const int bin_max = *bin_max_ptr;
    const int nb = min(bin_max + 1, nbins_cap);
    for (int b = 0; b < nb; ++b) hcol[b * kHistThreads + t] = 0;
    const size_t npix = static_cast<size_t>(w) * h;
    for (size_t p = static_cast<size_t>(blockIdx.x) * kHistThreads + t; p < npix;
         p += static_cast<size_t>(gridDim.x) * kHistThreads) {
        const float center = cur[p];
        if (!isfinite(center)) {
            next[p] = center;  // removed outliers stay removed
            continue;
        }
        const int x = static_cast<int>(p % w), y = static_cast<int>(p / w);
        const int y0 = y - U[p], y1 = y + D[p];
        int count = 0, lo = bin_max, hi = 0;
        for (int vy = y0; vy <= y1; ++vy) {
            const size_t vi = static_cast<size_t>(vy) * w + x;
            const float* row = cur + static_cast<size_t>(vy) * w;
            const int x1 = x + R[vi];
            for (int c = x - L[vi]; c <= x1; ++c) {
                float v = row[c];
                if (!isfinite(v)) continue;
                int bin = min(max(static_cast<int>(lroundf(v)), 0), nb - 1);
                unsigned short* cell = &hcol[bin * kHistThreads + t];
                *cell = static_cast<unsigned short>(*cell + 1);
                ++count;
                lo = min(lo, bin);
                hi = max(hi, bin);
            }
        }
        int best_c = 0, best_b = lo;
        for (int b = lo; b <= hi; ++b) {
            int cnt = hcol[b * kHistThreads + t];
            hcol[b * kHistThreads + t] = 0;
            if (cnt > best_c) {
                best_c = cnt;
                best_b = b;
            }
        }
        next[p] = (best_c == 1 && count >= 4) ? __int_as_float(0x7fc00000) : static_cast<float>(best_b);
    }
}

// ---------------------------------------------------------------------------
// Histogram refinement by region extrema (stereo.cpp:240-299), the frame
// loop's default. The refined map is piecewise constant: at config B 90 % of
// the cross regions hold a single distinct disparity (95 % at most two). For
// such a region the histogram has one bin, its count is the region's valid
// count, so the mode is that value and "mode_count == 1 && region >= 4" cannot
// hold. So:
//   k_ref_hminmax : per pixel (x, y'), the min / max bin over its horizontal
//                   span in row y' (NaN skipped; empty -> min > max);
//   k_ref_vminmax : per pixel (x, y), the min / max over its vertical arm of
//                   those; a valid centre with min == max takes that bin; any
//                   other valid centre is queued (warp-aggregated atomic);
//   k_ref_slow    : warp per queued pixel: the exact histogram of its region
//                   in shared memory (lanes over a span, __match_any_sync
//                   groups equal bins so each distinct bin is added once per
//                   row chunk), then the (count, smallest bin) argmax over
//                   [lo, hi] and the reference's outlier rule.
// Min, max and counts are exact integers in any order, so every output is the
// reference's. A NaN centre stays NaN (stereo.cpp:258).
// Row runs of equal bins (NaN = bin -1): runs[y][x] = bin(x) & 0xffff |
// (last x' of the run holding x) << 16. The region scans below then step from
// run to run instead of from pixel to pixel: the refined map is piecewise
// constant, so a 35-pixel span is typically one to three runs.
__device__ __forceinline__ int ref_bin(float v, int cap) {
    return isfinite(v) ? min(max(static_cast<int>(lroundf(v)), 0), cap - 1) : -1;
}
__global__ void k_ref_runs(const float* __restrict__ cur, int w, int h, int cap, uint32_t* __restrict__ runs) {
    extern __shared__ uint32_t rr_chg[];  // bit x: the run ends at x
    const int y = blockIdx.x, lane = threadIdx.x & 31;
    const float* row = cur + static_cast<size_t>(y) * w;
    const int nwd = (w + 31) >> 5;
    for (int x0 = 0; x0 < nwd * 32; x0 += blockDim.x) {  // uniform trip count (blockDim % 32 == 0)
        const int x = x0 + static_cast<int>(threadIdx.x);
        const bool c = x >= w - 1 || ref_bin(row[x], cap) != ref_bin(row[x + 1], cap);
        const unsigned bal = __ballot_sync(0xffffffffu, c);
        if (lane == 0 && (x >> 5) < nwd) rr_chg[x >> 5] = bal;
    }
    __syncthreads();
    for (int x = threadIdx.x; x < w; x += blockDim.x) {
        int wd = x >> 5;
        unsigned m = rr_chg[wd] & (0xffffffffu << (x & 31));
        while (!m) m = rr_chg[++wd];  // bit w - 1 is set
        const int e = (wd << 5) + __ffs(m) - 1;
        runs[static_cast<size_t>(y) * w + x] =
            (static_cast<uint32_t>(ref_bin(row[x], cap)) & 0xffffu) | (static_cast<uint32_t>(e) << 16);
    }
}

__global__ void k_ref_hminmax(const uint32_t* __restrict__ runs, int w, int h, const uint8_t* __restrict__ L,
                              const uint8_t* __restrict__ R, uint2* __restrict__ mm) {
    const int x = blockIdx.x * blockDim.x + threadIdx.x, y = blockIdx.y;
    if (x >= w) return;
    const size_t i = static_cast<size_t>(y) * w + x;
    const uint32_t* row = runs + static_cast<size_t>(y) * w;
    // the span's distinct bins, up to two (a < b), their counts, and whether a
    // third exists -- the per-pixel scan's state after each run of len pixels
    int a = 0x7fff, b = -1, ca = 0, cb = 0;
    bool three = false;
    for (int c = x - L[i], e = x + R[i]; c <= e;) {
        const uint32_t v = row[c];
        const int bin = static_cast<short>(v & 0xffffu);
        const int end = min(static_cast<int>(v >> 16), e);
        const int len = end - c + 1;
        c = end + 1;
        if (bin < 0) continue;
        if (bin == a) {
            ca += len;
        } else if (bin == b) {
            cb += len;
        } else if (b < 0) {  // a second distinct bin (or the first)
            if (a == 0x7fff) {
                a = bin;
                ca = len;
            } else if (bin < a) {
                b = a;
                cb = ca;
                a = bin;
                ca = len;
            } else {
                b = bin;
                cb = len;
            }
        } else {
            // a third bin: the first pixel only moves the extrema, the rest of
            // the run then counts toward whichever extremum it became
            three = true;
            a = min(a, bin);
            b = max(b, bin);
            if (bin == a) {
                ca += len - 1;
            } else if (bin == b) {
                cb += len - 1;
            }
        }
    }
    if (b < 0 && a != 0x7fff) {  // one distinct bin: min == max
        b = a;
        cb = ca;
    }
    mm[i] = make_uint2(static_cast<uint32_t>(a & 0xffff) | (static_cast<uint32_t>(b & 0xffff) << 16),
                       static_cast<uint32_t>(min(ca, 255)) | (static_cast<uint32_t>(min(cb, 255)) << 8) |
                           (three ? 1u << 16 : 0u));
}

__global__ void k_ref_vminmax(const float* __restrict__ cur, int w, int h, const uint8_t* __restrict__ U,
                              const uint8_t* __restrict__ D, const uint2* __restrict__ mm,
                              float* __restrict__ next, int* __restrict__ queue) {
    const int x = blockIdx.x * blockDim.x + threadIdx.x, y = blockIdx.y;
    if (x >= w) return;
    const size_t i = static_cast<size_t>(y) * w + x;
    const float c = cur[i];
    if (!isfinite(c)) {  // removed outliers stay removed
        next[i] = c;
        return;
    }
    const int y0 = y - U[i], y1 = y + D[i];
    int lo = 0x7fff, hi = -1;
    bool three = false;
    // kB rows' loads in flight at a time (min / max / or: any order)
    constexpr int kB = 8;
    for (int yb = y0; yb <= y1; yb += kB) {
        uint2 v[kB];
#pragma unroll
        for (int j = 0; j < kB; ++j)
            v[j] = yb + j <= y1 ? mm[static_cast<size_t>(yb + j) * w + x] : make_uint2(0x7fffu | 0xffff0000u, 0u);
#pragma unroll
        for (int j = 0; j < kB; ++j) {
            lo = min(lo, static_cast<int>(v[j].x & 0xffffu));
            hi = max(hi, static_cast<int>(static_cast<short>(v[j].x >> 16)));
            three |= (v[j].y >> 16) != 0;
        }
    }
    if (lo == hi) {  // one bin in the region: it is the mode
        next[i] = static_cast<float>(lo);
        return;
    }
    if (!three) {
        // two bins lo < hi, if every span holds only those: counts from the spans,
        // the mode is lo on ties (smaller bin) and "mode_count == 1 && region >= 4"
        // cannot hold (both counts 1 means a region of 2)
        bool two = true;
        int nlo = 0, nhi = 0;
        for (int yy = y0; yy <= y1; ++yy) {
            const uint2 v = mm[static_cast<size_t>(yy) * w + x];
            const int a = static_cast<int>(v.x & 0xffffu), b = static_cast<int>(static_cast<short>(v.x >> 16));
            if (b < 0) continue;  // no valid value in this span
            two &= (a == lo || a == hi) && (b == lo || b == hi);
            nlo += a == lo ? static_cast<int>(v.y & 255u) : 0;
            nhi += b == hi ? static_cast<int>((v.y >> 8) & 255u) : 0;
        }
        if (two) {
            next[i] = static_cast<float>(nlo >= nhi ? lo : hi);
            return;
        }
    }
    queue[1 + atomicAdd(queue, 1)] = static_cast<int>(i);
}

constexpr int kSlowWarps = 8;
__global__ void __launch_bounds__(kSlowWarps * 32) k_ref_slow(const uint32_t* __restrict__ runs, int w, int h,
                                                              const uint8_t* __restrict__ L,
                                                              const uint8_t* __restrict__ R,
                                                              const uint8_t* __restrict__ U,
                                                              const uint8_t* __restrict__ D, int cap,
                                                              const int* __restrict__ queue,
                                                              float* __restrict__ next) {
    // per warp: cap 16-bit counts packed two per word (a region holds at most
    // 255 x 255 pixels, so a half never carries into the other)
    extern __shared__ uint32_t rs_hist[];  // [kSlowWarps][cap / 2]
    const int lane = threadIdx.x & 31, wp = threadIdx.x >> 5;
    uint32_t* hist = rs_hist + static_cast<size_t>(wp) * (cap >> 1);
    for (int b = lane; b < (cap >> 1); b += 32) hist[b] = 0;
    __syncwarp();
    const int nq = queue[0];
    for (int q = blockIdx.x * kSlowWarps + wp; q < nq; q += gridDim.x * kSlowWarps) {
        const int i = queue[1 + q];
        const int y = i / w, x = i - y * w;
        int lo = 0x7fff, hi = -1, total = 0;
        const int y0 = y - U[i], nrow = y + D[i] - y0 + 1;
        // lane j walks the runs of the span of row y0 + r0 + j
        for (int r0 = lane; r0 < nrow; r0 += 32) {
            const size_t vi = static_cast<size_t>(y0 + r0) * w + x;
            const uint32_t* row = runs + static_cast<size_t>(y0 + r0) * w;
            for (int c = x - L[vi], e = x + R[vi]; c <= e;) {
                const uint32_t v = row[c];
                const int bin = static_cast<short>(v & 0xffffu);
                const int end = min(static_cast<int>(v >> 16), e);
                const int len = end - c + 1;
                c = end + 1;
                if (bin < 0) continue;
                atomicAdd(hist + (bin >> 1), static_cast<uint32_t>(len) << (16 * (bin & 1)));
                lo = min(lo, bin);
                hi = max(hi, bin);
                total += len;
            }
        }
        __syncwarp();
        lo = __reduce_min_sync(0xffffffffu, lo);
        hi = __reduce_max_sync(0xffffffffu, static_cast<unsigned>(hi + 1)) - 1;
        total = static_cast<int>(__reduce_add_sync(0xffffffffu, static_cast<unsigned>(total)));
        // (count, smallest bin) argmax: the reference's strict '>' scan from lo (stereo.cpp:272-278)
        unsigned key = 0;
        for (int b = lo + lane; b <= hi; b += 32) {
            const unsigned cnt = (hist[b >> 1] >> (16 * (b & 1))) & 0xffffu;
            if (cnt) key = max(key, (cnt << 16) | (0xffffu - static_cast<unsigned>(b)));
        }
        __syncwarp();
        for (int b = (lo >> 1) + lane; b <= (hi >> 1); b += 32) hist[b] = 0;
        key = __reduce_max_sync(0xffffffffu, key);
        if (lane == 0) {
            const int best_c = static_cast<int>(key >> 16);
            const int best_b = static_cast<int>(0xffffu - (key & 0xffffu));
            next[i] = (best_c == 1 && total >= 4) ? __int_as_float(0x7fc00000) : static_cast<float>(best_b);
        }
        __syncwarp();
    }
}

// Histogram refinement as an exact integer cross-aggregation (the region
// histogram of stereo.cpp:252-297 is the cross-region sum of one-hot bins):
//   H(x, y', v) = #{c in the horizontal span of (x, y') : bin(c, y') == v}
//   count(x, y, v) = sum over y' on the vertical arm of (x, y) of H(x, y', v)
// Counts are integers, so any summation order is exact. k_refine_hscatter
// builds H densely; k_refine_segsum sums it per (column, row segment); the
// mode pass walks each segment of each column with a prefix ring seeded from
// the segment sums and takes the mode (max count, smallest bin on ties).
// Cost O(N * bins) instead of O(N * region) -- regions reach 35x35.

// Segmented mode pass: warp per (column x, row segment k); the prefix ring is
// seeded from the carry, so segments run in parallel. H rows are prefetched
// kPF ahead.
template <int VPL>
__global__ void k_refine_vmode2(const float* __restrict__ cur, const uint8_t* __restrict__ hcnt, int w, int h,
                                const uint8_t* __restrict__ U, const uint8_t* __restrict__ D, int lag, int ring_mask,
                                int seg, int nseg, const unsigned* __restrict__ carry, float* __restrict__ next) {
    extern __shared__ unsigned short rings[];  // per warp: [ring][32 lanes][VPL]
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int gw = blockIdx.x * (blockDim.x >> 5) + warp;
    const int x = gw / nseg, k = gw - x * nseg;
    if (x >= w) return;
    const int nbp = 32 * VPL;
    const int ring = ring_mask + 1;
    unsigned short* rg = rings + static_cast<size_t>(warp) * ring * 32 * VPL;
    auto R_at = [&](int slot, int j) -> unsigned short& { return rg[(slot * 32 + lane) * VPL + j]; };
    const int j0 = max(0, k * seg - lag);
    const int out0 = k * seg, out1 = min(h, (k + 1) * seg);
    const int yend = min(h, out1 + lag);  // rows needed: C up to out1 - 1 + maxarm + 1
    unsigned short C[VPL];
    unsigned cs[VPL];
#pragma unroll
    for (int j = 0; j < VPL; ++j) cs[j] = 0;
    for (int kk = 0; kk < k; ++kk) {  // exclusive prefix of the segment sums
        const unsigned* cin = carry + ((static_cast<size_t>(x) * nseg + kk) * 32 + lane) * VPL;
#pragma unroll
        for (int j = 0; j < VPL; ++j) cs[j] += cin[j];
    }
#pragma unroll
    for (int j = 0; j < VPL; ++j) {
        C[j] = static_cast<unsigned short>(cs[j]);
        R_at(j0 & ring_mask, j) = C[j];
    }
    auto finalize = [&](int py, float center, int up, int dn) {
        const size_t i = static_cast<size_t>(py) * w + x;
        const int a = py - up, b = py + dn + 1;
        int best_c = 0, best_b = 0x7fffffff, total = 0;
#pragma unroll
        for (int j = 0; j < VPL; ++j) {
            int cnt = static_cast<int>(R_at(b & ring_mask, j)) - static_cast<int>(R_at(a & ring_mask, j));
            total += cnt;
            if (cnt > best_c) {
                best_c = cnt;
                best_b = lane * VPL + j;
            }
        }
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) {
            total += __shfl_xor_sync(0xffffffffu, total, off);
            int oc = __shfl_xor_sync(0xffffffffu, best_c, off);
            int ob = __shfl_xor_sync(0xffffffffu, best_b, off);
            if (oc > best_c || (oc == best_c && ob < best_b)) {
                best_c = oc;
                best_b = ob;
            }
        }
        if (lane == 0) {
            float o = center;
            if (isfinite(center))
                o = (best_c == 1 && total >= 4) ? __int_as_float(0x7fc00000) : static_cast<float>(best_b);
            next[i] = o;
        }
    };
    const size_t rowstride = static_cast<size_t>(w) * nbp;
    const uint8_t* src = hcnt + static_cast<size_t>(x) * nbp + lane * VPL;
    constexpr int kPF = 8;
    uint8_t pf[kPF][VPL];
#pragma unroll
    for (int q = 0; q < kPF; ++q)
#pragma unroll
        for (int j = 0; j < VPL; ++j) pf[q][j] = (j0 + q < yend) ? src[(j0 + q) * rowstride + j] : 0;
    for (int y0 = j0; y0 < yend; y0 += kPF) {
        uint8_t nx[kPF][VPL];
#pragma unroll
        for (int q = 0; q < kPF; ++q)
#pragma unroll
            for (int j = 0; j < VPL; ++j) {
                int y = y0 + kPF + q;
                nx[q][j] = y < yend ? src[y * rowstride + j] : 0;
            }
        // the centre values / vertical arms of the rows finalised in this chunk
        float cq[kPF];
        int uq[kPF], dq[kPF];
#pragma unroll
        for (int q = 0; q < kPF; ++q) {
            const int py = y0 + q + 1 - lag;
            cq[q] = 0.0f;
            uq[q] = dq[q] = 0;
            if (py >= out0 && py < out1) {
                const size_t i = static_cast<size_t>(py) * w + x;
                cq[q] = cur[i];
                uq[q] = U[i];
                dq[q] = D[i];
            }
        }
#pragma unroll
        for (int q = 0; q < kPF; ++q) {
            const int y = y0 + q;
            if (y < yend) {
#pragma unroll
                for (int j = 0; j < VPL; ++j) {
                    C[j] = static_cast<unsigned short>(C[j] + pf[q][j]);
                    R_at((y + 1) & ring_mask, j) = C[j];
                }
                const int py = y + 1 - lag;
                if (py >= out0 && py < out1) finalize(py, cq[q], uq[q], dq[q]);
            }
        }
#pragma unroll
        for (int q = 0; q < kPF; ++q)
#pragma unroll
            for (int j = 0; j < VPL; ++j) pf[q][j] = nx[q][j];
    }
    // rows whose window reaches the image bottom
    for (int py = max(yend + 1 - lag, out0); py < out1; ++py) {
        const size_t i = static_cast<size_t>(py) * w + x;
        finalize(py, cur[i], U[i], D[i]);
    }
}

// Packed segmented mode pass (the production path): as k_refine_vmode2, but
// two u16 bin prefixes share one u32 (a column prefix never exceeds
// h * (2*l1+1) < 65536, so the halves never carry into each other and the
// packed difference of two prefixes is the pair of exact counts), one
// vector shared-memory access per slot, and the (count, -bin) argmax and the
// region total as two warp REDUX ops.
template <int VPL>
__global__ void k_refine_vmode3(const float* __restrict__ cur, const uint8_t* __restrict__ hcnt, int w, int h,
                                const uint8_t* __restrict__ U, const uint8_t* __restrict__ D, int lag, int ring_n,
                                int seg, int nseg, const unsigned* __restrict__ carry, float* __restrict__ next) {
    static_assert(VPL == 2 || VPL == 4 || VPL == 8, "packed pairs");
    constexpr int W2 = VPL / 2;
    extern __shared__ uint32_t ringw[];  // per warp: [ring_n][32 lanes][W2]
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int gw = blockIdx.x * (blockDim.x >> 5) + warp;
    const int x = gw / nseg, k = gw - x * nseg;
    if (x >= w) return;
    const int nbp = 32 * VPL;
    uint32_t* rg = ringw + static_cast<size_t>(warp) * ring_n * 32 * W2 + lane * W2;
    auto slot_ptr = [&](int slot) { return rg + slot * 32 * W2; };
    auto load_slot = [&](int slot, uint32_t (&o)[W2]) {
        const uint32_t* p = slot_ptr(slot);
        if constexpr (W2 == 1) {
            o[0] = p[0];
        } else if constexpr (W2 == 2) {
            uint2 v = *reinterpret_cast<const uint2*>(p);
            o[0] = v.x;
            o[1] = v.y;
        } else {
            uint4 v = *reinterpret_cast<const uint4*>(p);
            o[0] = v.x;
            o[1] = v.y;
            o[2] = v.z;
            o[3] = v.w;
        }
    };
    auto store_slot = [&](int slot, const uint32_t (&o)[W2]) {
        uint32_t* p = slot_ptr(slot);
        if constexpr (W2 == 1) {
            p[0] = o[0];
        } else if constexpr (W2 == 2) {
            *reinterpret_cast<uint2*>(p) = make_uint2(o[0], o[1]);
        } else {
            *reinterpret_cast<uint4*>(p) = make_uint4(o[0], o[1], o[2], o[3]);
        }
    };
    const int j0 = max(0, k * seg - lag);
    const int out0 = k * seg, out1 = min(h, (k + 1) * seg);
    const int yend = min(h, out1 + lag);
    uint32_t C[W2];
    {
        // exclusive prefix of the segment sums: the first 8 loads issue together
        unsigned cs[VPL];
#pragma unroll
        for (int j = 0; j < VPL; ++j) cs[j] = 0;
        const unsigned* cin = carry + (static_cast<size_t>(x) * nseg * 32 + lane) * VPL;
        constexpr int kU = 8;
        unsigned part[kU][VPL];
#pragma unroll
        for (int kk = 0; kk < kU; ++kk)
#pragma unroll
            for (int j = 0; j < VPL; ++j) part[kk][j] = kk < k ? cin[kk * 32 * VPL + j] : 0u;
#pragma unroll
        for (int kk = 0; kk < kU; ++kk)
#pragma unroll
            for (int j = 0; j < VPL; ++j) cs[j] += part[kk][j];
        for (int kk = kU; kk < k; ++kk)
#pragma unroll
            for (int j = 0; j < VPL; ++j) cs[j] += cin[kk * 32 * VPL + j];
#pragma unroll
        for (int q = 0; q < W2; ++q) C[q] = (cs[2 * q] & 0xffffu) | (cs[2 * q + 1] << 16);
    }
    int s1 = 0;  // slot of C after row y (prefix through row y): starts as the prefix before j0
    store_slot(0, C);
    auto finalize = [&](int sa, int sb, float center, int py) {
        uint32_t A[W2], B[W2];
        load_slot(sa, A);
        load_slot(sb, B);
        uint32_t key = 0;
        int tot = 0;
#pragma unroll
        for (int q = 0; q < W2; ++q) {
            const uint32_t dlt = B[q] - A[q];
            const uint32_t c0 = dlt & 0xffffu, c1 = dlt >> 16;
            const uint32_t b0 = static_cast<uint32_t>(lane * VPL + 2 * q);
            tot += static_cast<int>(c0 + c1);
            const uint32_t k0 = c0 ? (c0 << 16) | (0xffffu - b0) : 0u;
            const uint32_t k1 = c1 ? (c1 << 16) | (0xffffu - b0 - 1u) : 0u;
            key = max(key, max(k0, k1));
        }
        const uint32_t wkey = __reduce_max_sync(0xffffffffu, key);
        const int total = static_cast<int>(__reduce_add_sync(0xffffffffu, static_cast<unsigned>(tot)));
        if (lane == 0) {
            float o = center;  // removed outliers stay removed
            if (isfinite(center)) {
                const int best_c = static_cast<int>(wkey >> 16);
                const int best_b = static_cast<int>(0xffffu - (wkey & 0xffffu));
                o = (best_c == 1 && total >= 4) ? __int_as_float(0x7fc00000) : static_cast<float>(best_b);
            }
            next[static_cast<size_t>(py) * w + x] = o;
        }
    };
    // ring slot of the prefix through row yy (C[yy+1] in prefix terms) relative
    // to s1 = slot of the prefix through row y: slot(y) - (y - yy)
    auto rel = [&](int base_slot, int back) {
        int sl = base_slot - back;
        return sl < 0 ? sl + ring_n : sl;
    };
    const size_t rowstride = static_cast<size_t>(w) * nbp;
    // raw H words are kept as loaded (VPL bytes per lane) and unpacked into
    // u16 pairs only when consumed, so the prefetch really stays in flight
    constexpr int RW = (VPL + 3) / 4;  // raw u32 words per row (VPL=2 uses the low half)
    auto load_raw = [&](const uint8_t* p, uint32_t (&o)[RW]) {
        if constexpr (VPL == 2) {
            o[0] = *reinterpret_cast<const unsigned short*>(p);
        } else if constexpr (VPL == 4) {
            o[0] = *reinterpret_cast<const uint32_t*>(p);
        } else {
            const uint2 v = *reinterpret_cast<const uint2*>(p);
            o[0] = v.x;
            o[1] = v.y;
        }
    };
    auto unpack = [&](const uint32_t (&r)[RW], uint32_t (&o)[W2]) {
#pragma unroll
        for (int q = 0; q < RW; ++q) {
            o[2 * q] = __byte_perm(r[q], 0u, 0x4140);
            if (2 * q + 1 < W2) o[2 * q + 1] = __byte_perm(r[q], 0u, 0x4342);
        }
    };
    // hp: next H row to load
    const uint8_t* hp = hcnt + static_cast<size_t>(j0) * rowstride + static_cast<size_t>(x) * nbp + lane * VPL;
    constexpr int kPF = 8;
    uint32_t pf[kPF][RW];
    float cq[kPF];
    uint32_t uq[kPF], dq[kPF];  // arms of the row finalised at this step
    auto load_meta = [&](int y, float& c, uint32_t& a, uint32_t& b) {
        const int py = y + 1 - lag;
        c = 0.0f;
        a = b = 0u;
        if (py >= out0 && py < out1) {
            const size_t i = static_cast<size_t>(py) * w + x;
            c = cur[i];
            a = U[i];
            b = D[i];
        }
    };
#pragma unroll
    for (int q = 0; q < kPF; ++q) {
        if (j0 + q < yend) {
            load_raw(hp, pf[q]);
        } else {
#pragma unroll
            for (int t = 0; t < RW; ++t) pf[q][t] = 0u;
        }
        hp += rowstride;
        load_meta(j0 + q, cq[q], uq[q], dq[q]);
    }
    for (int y0 = j0; y0 < yend; y0 += kPF) {
        uint32_t nx[kPF][RW];
        float nc[kPF];
        uint32_t nu[kPF], nd[kPF];
        // chunk fully inside [j0, yend) with every row finalised: no per-row checks
        const bool fast = y0 + 2 * kPF <= yend && y0 + kPF + 1 - lag >= out0 && y0 + 2 * kPF - lag < out1;
        if (fast) {
            const size_t mi = static_cast<size_t>(y0 + kPF + 1 - lag) * w + x;
            const float* cp = cur + mi;
            const uint8_t* up = U + mi;
            const uint8_t* dp = D + mi;
#pragma unroll
            for (int q = 0; q < kPF; ++q) {
                load_raw(hp, nx[q]);
                hp += rowstride;
                nc[q] = *cp;
                nu[q] = *up;
                nd[q] = *dp;
                cp += w;
                up += w;
                dp += w;
            }
        } else {
#pragma unroll
            for (int q = 0; q < kPF; ++q) {
                const int y = y0 + kPF + q;
                if (y < yend) {
                    load_raw(hp, nx[q]);
                } else {
#pragma unroll
                    for (int t = 0; t < RW; ++t) nx[q][t] = 0u;
                }
                hp += rowstride;
                load_meta(y, nc[q], nu[q], nd[q]);
            }
        }
        // prefixes of the whole chunk, then its outputs
        const int sb0 = s1;
#pragma unroll
        for (int q = 0; q < kPF; ++q) {
            if (y0 + q < yend) {
                uint32_t hv[W2];
                unpack(pf[q], hv);
#pragma unroll
                for (int t = 0; t < W2; ++t) C[t] += hv[t];
                s1 = (s1 + 1 == ring_n) ? 0 : s1 + 1;
                store_slot(s1, C);
            }
        }
        __syncwarp();
        int sq = sb0;
#pragma unroll
        for (int q = 0; q < kPF; ++q) {
            const int y = y0 + q;
            if (y < yend) {
                sq = (sq + 1 == ring_n) ? 0 : sq + 1;  // slot of the prefix through row y
                const int py = y + 1 - lag;
                if (py >= out0 && py < out1) {
                    // counts over rows [py - up, py + dn] = P(py + dn) - P(py - up - 1)
                    const int sb = rel(sq, lag - 1 - static_cast<int>(dq[q]));
                    const int sa = rel(sq, lag + static_cast<int>(uq[q]));
                    finalize(sa, sb, cq[q], py);
                }
            }
        }
        __syncwarp();
#pragma unroll
        for (int q = 0; q < kPF; ++q) {
#pragma unroll
            for (int t = 0; t < RW; ++t) pf[q][t] = nx[q][t];
            cq[q] = nc[q];
            uq[q] = nu[q];
            dq[q] = nd[q];
        }
    }
    // rows whose window reaches the image bottom; s1 = slot of the prefix through row yend - 1
    for (int py = max(yend + 1 - lag, out0); py < out1; ++py) {
        const size_t i = static_cast<size_t>(py) * w + x;
        const int up = U[i], dn = D[i];
        const int last = yend - 1;
        const int sb = rel(s1, last - (py + dn));
        const int sa = rel(s1, last - (py - up - 1));
        finalize(sa, sb, cur[i], py);
    }
}

// H(x, y, .) by scattering the pixel's own span (<= 2*l1+1 values) into a
// per-thread shared-memory column of u8 counters, then streaming the dense
// row out with 16-byte stores (the zero bins included).
constexpr int kHcThreads = 128;
__global__ void __launch_bounds__(kHcThreads) k_refine_hscatter(const float* __restrict__ cur, int w, int h,
                                                                const uint8_t* __restrict__ L,
                                                                const uint8_t* __restrict__ R, int nbp,
                                                                uint8_t* __restrict__ hcnt) {
    extern __shared__ uint4 hsm4[];  // [nbp/16][kHcThreads] uint4
    uint8_t* hs = reinterpret_cast<uint8_t*>(hsm4);
    const int t = threadIdx.x;
    const int nq = nbp >> 4;
    for (int q = 0; q < nq; ++q) hsm4[q * kHcThreads + t] = make_uint4(0, 0, 0, 0);
    const size_t npix = static_cast<size_t>(w) * h;
    for (size_t p = static_cast<size_t>(blockIdx.x) * kHcThreads + t; p < npix;
         p += static_cast<size_t>(gridDim.x) * kHcThreads) {
        const int x = static_cast<int>(p % w);
        const float* row = cur + (p - x);
        const int a = x - L[p], z = x + R[p];
        int lo = nbp, hi = -1;
        for (int c = a; c <= z; ++c) {
            float v = row[c];
            if (!isfinite(v)) continue;
            int b = min(max(static_cast<int>(lroundf(v)), 0), nbp - 1);
            uint8_t* cell = &hs[((b >> 4) * kHcThreads + t) * 16 + (b & 15)];
            *cell = static_cast<uint8_t>(*cell + 1);
            lo = min(lo, b);
            hi = max(hi, b);
        }
        uint4* out = reinterpret_cast<uint4*>(hcnt + p * nbp);
        for (int q = 0; q < nq; ++q) {
            uint4 val = hsm4[q * kHcThreads + t];
            out[q] = val;
        }
        for (int q = (lo >> 4); q <= (hi >> 4) && hi >= 0; ++q) hsm4[q * kHcThreads + t] = make_uint4(0, 0, 0, 0);
    }
}

// Per (column, segment) sums of H over the rows [j0(k), j0(k+1)); the mode
// pass turns them into exclusive prefixes (integers: exact in any order).
template <int VPL>
__global__ void k_refine_segsum(const uint8_t* __restrict__ hcnt, int w, int h, int seg, int nseg, int lag,
                                unsigned* __restrict__ segsum /* [x][nseg][32][VPL] */) {
    const int lane = threadIdx.x & 31;
    const int gw = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    const int x = gw / nseg, k = gw - x * nseg;
    if (x >= w) return;
    const int nbp = 32 * VPL;
    const int y0 = max(0, k * seg - lag), y1 = (k + 1 < nseg) ? max(0, (k + 1) * seg - lag) : h;
    const size_t rowstride = static_cast<size_t>(w) * nbp;
    const uint8_t* src = hcnt + static_cast<size_t>(x) * nbp + lane * VPL;
    unsigned acc[VPL];
#pragma unroll
    for (int j = 0; j < VPL; ++j) acc[j] = 0;
#pragma unroll 8
    for (int y = y0; y < y1; ++y)
#pragma unroll
        for (int j = 0; j < VPL; ++j) acc[j] += src[y * rowstride + j];
    unsigned* dst = segsum + ((static_cast<size_t>(x) * nseg + k) * 32 + lane) * VPL;
#pragma unroll
    for (int j = 0; j < VPL; ++j) dst[j] = acc[j];
}

// k_refine_segsum with the rows of one (column, segment) split over the 4
// warps of a block (integer partial sums: exact in any order).
template <int VPL>
__global__ void __launch_bounds__(128) k_refine_segsum4(const uint8_t* __restrict__ hcnt, int w, int h, int seg,
                                                        int nseg, int lag, unsigned* __restrict__ segsum) {
    __shared__ unsigned part[4][32 * VPL];
    const int lane = threadIdx.x & 31, wp = threadIdx.x >> 5;
    const int x = blockIdx.x / nseg, k = blockIdx.x - x * nseg;
    const int nbp = 32 * VPL;
    const int y0 = max(0, k * seg - lag), y1 = (k + 1 < nseg) ? max(0, (k + 1) * seg - lag) : h;
    const size_t rowstride = static_cast<size_t>(w) * nbp;
    const uint8_t* src = hcnt + static_cast<size_t>(x) * nbp + lane * VPL;
    unsigned acc[VPL];
#pragma unroll
    for (int j = 0; j < VPL; ++j) acc[j] = 0;
#pragma unroll 4
    for (int y = y0 + wp; y < y1; y += 4)
#pragma unroll
        for (int j = 0; j < VPL; ++j) acc[j] += src[y * rowstride + j];
#pragma unroll
    for (int j = 0; j < VPL; ++j) part[wp][lane * VPL + j] = acc[j];
    __syncthreads();
    if (wp == 0) {
        unsigned* dst = segsum + ((static_cast<size_t>(x) * nseg + k) * 32 + lane) * VPL;
#pragma unroll
        for (int j = 0; j < VPL; ++j)
            dst[j] = part[0][lane * VPL + j] + part[1][lane * VPL + j] + part[2][lane * VPL + j] +
                     part[3][lane * VPL + j];
    }
}

// -------------------------------------------------------- sparse depth -----
// disparity_to_sparse_depth, stereo.cpp:301-315.
__global__ void k_sparse_depth(const float* __restrict__ disp, int w, int h, double fb, int fw,
                               int fh, float* __restrict__ out) {
    int x = blockIdx.x * blockDim.x + threadIdx.x;
    int y = blockIdx.y * blockDim.y + threadIdx.y;
    if (x >= fw || y >= fh) return;
    float v = __int_as_float(0x7fc00000);
    if (!(x & 1) && !(y & 1) && (x >> 1) < w && (y >> 1) < h) {
        float d = disp[static_cast<size_t>(y >> 1) * w + (x >> 1)];
        if (isfinite(d)) {
            double d_full = 2.0 * static_cast<double>(d);
            if (d_full > 0.0) v = static_cast<float>(fb / d_full);
        }
    }
    out[static_cast<size_t>(y) * fw + x] = v;
}

// ------------------------------------------ left-right consistency (opt-in) --
// Not in the reference (SPEC.md "Non-goals: no left-right cross-checking");
// the north_star's optional filter. The right view's disparity is the same
// chain on the mirrored pair (left' = mirror(right), right' = mirror(left):
// q' = x' - d in right' is q = x + d in the left image), mirrored back.
__global__ void k_flip_h(const float* __restrict__ in, int w, int h, float* __restrict__ out) {
    const int x = blockIdx.x * blockDim.x + threadIdx.x;
    const int y = blockIdx.y * blockDim.y + threadIdx.y;
    if (x >= w || y >= h) return;
    out[static_cast<size_t>(y) * w + x] = in[static_cast<size_t>(y) * w + (w - 1 - x)];
}

// keep d_L(x) where the right view maps back: x_r = x - d_L (integer-valued
// disparities), |d_L(x) - d_R(x_r)| <= max_diff; nodata (NaN) otherwise.
__global__ void k_lr_check(const float* __restrict__ dl, const float* __restrict__ dr, int w, int h,
                           double max_diff, float* __restrict__ out) {
    const int x = blockIdx.x * blockDim.x + threadIdx.x;
    const int y = blockIdx.y * blockDim.y + threadIdx.y;
    if (x >= w || y >= h) return;
    const size_t i = static_cast<size_t>(y) * w + x;
    const float d = dl[i];
    float v = __int_as_float(0x7fc00000);
    if (isfinite(d)) {
        const int xr = x - static_cast<int>(floorf(d + 0.5f));
        if (xr >= 0 && xr < w) {
            const float e = dr[static_cast<size_t>(y) * w + xr];
            if (isfinite(e) && fabs(static_cast<double>(d) - static_cast<double>(e)) <= max_diff) v = d;
        }
    }
    out[i] = v;
}

__global__ void k_max_arm(const uint8_t* __restrict__ a0, const uint8_t* __restrict__ a1,
                          const uint8_t* __restrict__ a2, const uint8_t* __restrict__ a3, size_t n,
                          int* __restrict__ out) {
    size_t i = static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    int m = 0;
    if (i < n) m = max(max(a0[i], a1[i]), max(a2[i], a3[i]));
    block_atomic_max(out, m);
}

inline dim3 grid2(int w, int h, dim3 b) { return dim3((w + b.x - 1) / b.x, (h + b.y - 1) / b.y); }

int ring_size(int l1) {
    int need = 2 * l1 + 2, r = 1;
    while (r < need) r <<= 1;
    return r;
}

}  // namespace

// ===================================================================== host =

int max_arm_length(dco_ctx* ctx, const uint8_t* l, const uint8_t* r, const uint8_t* u,
                   const uint8_t* d, int w, int h) {
    size_t n = static_cast<size_t>(w) * h;
    int* dm = static_cast<int*>(scratch(ctx, S_FLAG_ARM, 64));
    cuda_check(cudaMemsetAsync(dm, 0, sizeof(int), ctx->stream), "memset");
    k_max_arm<<<blocks_for(n, 256), 256, 0, ctx->stream>>>(l, r, u, d, n, dm);
    launched(ctx, "k_max_arm");
    int* hm = static_cast<int*>(pinned_host(ctx, 64));
    cuda_check(cudaMemcpyAsync(hm, dm, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream), "d2h");
    cuda_check(cudaStreamSynchronize(ctx->stream), "sync");
    return *hm;
}

void downsample_half(dco_ctx* ctx, const float* img, int w, int h, float* out) {
    require(w >= 2 && h >= 2, "downsample_half: dimensions must be at least 2x2");
    int ow = w / 2, oh = h / 2;
    dim3 b(32, 8);
    k_downsample<<<grid2(ow, oh, b), b, 0, ctx->stream>>>(img, w, h, out, ow, oh);
    launched(ctx, "k_downsample");
}

void ingest_gray8(dco_ctx* ctx, const uint8_t* g8, int w, int h, float* full, float* quarter) {
    require(w >= 2 && h >= 2, "ingest: dimensions must be at least 2x2");
    int qw = w / 2, qh = h / 2;
    dim3 b(32, 8);
    const bool v4 = (w % 8) == 0 && (reinterpret_cast<uintptr_t>(g8) & 7) == 0 &&
                    (reinterpret_cast<uintptr_t>(full) & 15) == 0 && (reinterpret_cast<uintptr_t>(quarter) & 15) == 0;
    if (v4) {
        k_ingest_gray8_v4<<<grid2(qw / 4, qh, b), b, 0, ctx->stream>>>(g8, w, h, full, quarter, qw, qh);
    } else {
        k_ingest_gray8<<<grid2(qw, qh, b), b, 0, ctx->stream>>>(g8, w, h, full, quarter, qw, qh);
    }
    launched(ctx, "k_ingest_gray8");
    int tail = ((w & 1) ? h : 0) + ((h & 1) ? w : 0);
    if (full && tail) {
        k_ingest_gray8_tail<<<blocks_for(tail, 256), 256, 0, ctx->stream>>>(g8, w, h, full);
        launched(ctx, "k_ingest_gray8_tail");
    }
}

void build_cross_windows(dco_ctx* ctx, const float* img, int w, int h, const dco_config* cfg,
                         uint8_t* l, uint8_t* r, uint8_t* u, uint8_t* d) {
    require(w >= 1 && h >= 1, "build_cross_windows: empty image");
    require(cfg->cross_arm_l1 <= 255, "build_cross_windows: cross_arm_l1 must fit the u8 arms");
    uint8_t* raw = static_cast<uint8_t*>(scratch(ctx, S_ARM_RAW, static_cast<size_t>(w) * h * 4));
    dim3 b(32, 8);
    if (!getenv("DCO_ARMS_F64")) {
        // the smallest float >= tau: (double)diff >= tau <=> diff >= it
        auto arm_threshold = [](double tau) {
            float f = static_cast<float>(tau);
            if (static_cast<double>(f) < tau) f = nextafterf(f, INFINITY);
            return f;
        };
        k_cross_arms_f<<<grid2(w, h, b), b, 0, ctx->stream>>>(img, w, h, cfg->cross_arm_l1, cfg->cross_arm_l2,
                                                              arm_threshold(cfg->cross_color_tau),
                                                              arm_threshold(cfg->cross_color_tau2), raw);
        launched(ctx, "k_cross_arms_f");
    } else {
        k_cross_arms_raw<<<grid2(w, h, b), b, 0, ctx->stream>>>(img, w, h, cfg->cross_arm_l1,
                                                                cfg->cross_arm_l2, cfg->cross_color_tau,
                                                                cfg->cross_color_tau2, raw);
        launched(ctx, "k_cross_arms_raw");
    }
    dim3 g = grid2(w, h, b);
    g.z = 4;
    k_arm_median<<<g, b, 0, ctx->stream>>>(raw, w, h, l, r, u, d);
    launched(ctx, "k_arm_median");
}

void region_pack(dco_ctx* ctx, const uint8_t* l, const uint8_t* r, const uint8_t* u, const uint8_t* d, int w, int h,
                 uint32_t* hinfo, uint32_t* vinfo) {
    dim3 b(32, 8);
    k_region_pack<<<grid2(w, h, b), b, 0, ctx->stream>>>(l, r, u, d, w, h, hinfo, vinfo);
    launched(ctx, "k_region_pack");
}

// census of a stereo pair in one tiled launch (the cost volume's inputs)
void census_pair(dco_ctx* ctx, const float* left, const float* right, int w, int h, int ww, int wh,
                 uint64_t* out_l, uint64_t* out_r) {
    const int rw = ww / 2, rh = wh / 2;
    const size_t smem = static_cast<size_t>(32 + 2 * rw) * (8 + 2 * rh) * sizeof(float);
    const dim3 grid((w + 31) / 32, (h + 7) / 8, 2);
    if (rw == 4 && rh == 3)
        k_census_tiled<4, 3><<<grid, dim3(32, 8), smem, ctx->stream>>>(left, right, w, h, rw, rh, out_l, out_r);
    else
        k_census_tiled<<<grid, dim3(32, 8), smem, ctx->stream>>>(left, right, w, h, rw, rh, out_l, out_r);
    launched(ctx, "k_census_tiled");
}

void census_transform(dco_ctx* ctx, const float* img, int w, int h, int ww, int wh, uint64_t* out) {
    if (ww % 2 == 0 || wh % 2 == 0)
        fail(DCO_CONFIG, "census_transform: window dimensions must be odd");
    if (ww * wh - 1 > 64) fail(DCO_CONFIG, "census_transform: window exceeds 64 comparison bits");
    dim3 b(32, 8);
    k_census<<<grid2(w, h, b), b, 0, ctx->stream>>>(img, w, h, ww / 2, wh / 2, out);
    launched(ctx, "k_census");
}

// Whether div_lambda equals the IEEE division for this lambda over the whole
// [0, 1] input domain: one exhaustive device check per (device, lambda),
// cached for the process.
bool lambda_division_fast(dco_ctx* ctx, double lam) {
    static std::mutex mu;
    static std::map<std::pair<int, uint64_t>, bool> known;
    uint64_t bits;
    memcpy(&bits, &lam, 8);
    const auto key = std::make_pair(ctx->device, bits);
    std::lock_guard<std::mutex> lock(mu);
    auto it = known.find(key);
    if (it != known.end()) return it->second;
    unsigned* bad = static_cast<unsigned*>(scratch(ctx, S_FLAG_DIV, 64));
    cuda_check(cudaMemsetAsync(bad, 0, sizeof(unsigned), ctx->stream), "memset");
    k_verify_div<<<148 * 8, 256, 0, ctx->stream>>>(lam, 1.0 / lam, bad);
    launched(ctx, "k_verify_div");
    unsigned host = 1;
    cuda_check(cudaMemcpyAsync(&host, bad, sizeof(unsigned), cudaMemcpyDeviceToHost, ctx->stream), "d2h");
    cuda_check(cudaStreamSynchronize(ctx->stream), "sync");
    known[key] = host == 0;
    return host == 0;
}

void compute_cost_volume(dco_ctx* ctx, const float* left, const float* right, int w, int h,
                         const uint8_t* l, const uint8_t* r, const uint8_t* u, const uint8_t* d,
                         const dco_config* cfg, float* cost) {
    validate_config(cfg);
    const size_t n = static_cast<size_t>(w) * h;
    uint64_t* census = static_cast<uint64_t*>(scratch(ctx, S_CENSUS, n * 16));
    census_pair(ctx, left, right, w, h, cfg->census_window_w, cfg->census_window_h, census, census + n);
    CostParams hp;
    hp.w = w;
    hp.h = h;
    hp.nd = cfg->d_max - cfg->d_min + 1;
    hp.d_min = cfg->d_min;
    hp.bits = cfg->census_window_w * cfg->census_window_h - 1;
    hp.lambda_ad = cfg->lambda_ad;
    hp.inv_lambda = 1.0 / cfg->lambda_ad;
    hp.fast_div = lambda_division_fast(ctx, cfg->lambda_ad) ? 1 : 0;
    StereoTables t;
    make_stereo_tables(cfg, &t);
    for (int i = 0; i < 256; ++i) hp.alpha[i] = t.alpha[i];
    for (int i = 0; i < 65; ++i) hp.census[i] = t.census[i];
    dim3 grid((w + kCostPix - 1) / kCostPix, h);
    k_cost_volume<<<grid, dim3(32, 16), 0, ctx->stream>>>(left, right, census, census + n, l, r, u, d, hp,
                                                           cost);
    launched(ctx, "k_cost_volume");
}

// A row band's aggregation (DESIGN 7), in two phases so the carry chain
// covers only the vertical pass: the packed arm words + horizontal pass into
// the context's scratch, then the vertical pass of slices [k0, k1) with the
// column prefix seeded from the band above and exported to the band below.
constexpr int kBandVPF = 8, kBandHPF = 16;

void aggregate_band_hpass(dco_ctx* ctx, const float* cost, int w, int h, int nd, const uint8_t* l, const uint8_t* r,
                          const uint8_t* u, const uint8_t* d, int max_arm) {
    require(nd >= 1, "aggregate_costs: empty disparity range");
    require(max_arm >= 0 && max_arm <= 127, "row bands: cross_arm_l1 must be <= 127");
    const size_t n = static_cast<size_t>(w) * h;
    double* hsum = static_cast<double*>(scratch(ctx, S_HSUM, n * nd * sizeof(double)));
    const int lag = max_arm + 1;
    uint32_t* hinfo = static_cast<uint32_t*>(scratch(ctx, S_REGION, 2 * n * sizeof(uint32_t)));
    uint32_t* vinfo = hinfo + n;
    dim3 b(32, 8);
    k_region_pack<<<grid2(w, h, b), b, 0, ctx->stream>>>(l, r, u, d, w, h, hinfo, vinfo);
    launched(ctx, "k_region_pack");
    const int ring_h = 2 * max_arm + 2 + kBandHPF - 1;
    dim3 tb(32, 4);
    const size_t smem_h = static_cast<size_t>(ring_h) * kAggThreads * sizeof(double);
    smem_attr(ctx, k_agg_h2<kBandHPF>, 227 * 1024, true);
    k_agg_h2<kBandHPF><<<dim3((nd + 31) / 32, (h + 3) / 4), tb, smem_h, ctx->stream>>>(cost, w, h, nd, hinfo, lag,
                                                                                      ring_h, hsum);
    launched(ctx, "k_agg_h2");
}

void aggregate_band_vpass(dco_ctx* ctx, int w, int h, int nd, int max_arm, float* out, const double* carry_in,
                          int c0, double* carry_out, int e, int k0, int k1) {
    require(0 <= k0 && k0 < k1 && k1 <= nd && k0 % 32 == 0, "row bands: slice chunk must start at a multiple of 32");
    const size_t n = static_cast<size_t>(w) * h;
    const double* hsum = static_cast<const double*>(scratch(ctx, S_HSUM, n * nd * sizeof(double)));
    const uint32_t* vinfo = static_cast<const uint32_t*>(scratch(ctx, S_REGION, 2 * n * sizeof(uint32_t))) + n;
    const int lag = max_arm + 1;
    const int ring_v = 2 * max_arm + 2 + kBandVPF - 1;
    dim3 tb(32, 4);
    const size_t smem_v = static_cast<size_t>(ring_v) * kAggThreads * sizeof(double);
    smem_attr(ctx, k_agg_v2<kBandVPF, true>, 227 * 1024, true);
    k_agg_v2<kBandVPF, true><<<dim3((k1 - k0 + 31) / 32, (w + 3) / 4), tb, smem_v, ctx->stream>>>(
        hsum, w, h, nd, vinfo, lag, ring_v, out, carry_in, c0, carry_out, e, k0, k1);
    launched(ctx, "k_agg_v2_band");
}

void aggregate_costs(dco_ctx* ctx, const float* cost, int w, int h, int nd, const uint8_t* l,
                     const uint8_t* r, const uint8_t* u, const uint8_t* d, int max_arm,
                     float* out) {
    require(nd >= 1, "aggregate_costs: empty disparity range");
    require(max_arm >= 0 && max_arm <= 255, "aggregate_costs: arm length out of range");
    const size_t n = static_cast<size_t>(w) * h;
    double* hsum = static_cast<double*>(scratch(ctx, S_HSUM, n * nd * sizeof(double)));
    const int lag = max_arm + 1;
    dim3 b(32, 8);
    if (max_arm <= 127) {
        // packed arm words (region < 65536), exact-size modular rings
        uint32_t* hinfo = static_cast<uint32_t*>(scratch(ctx, S_REGION, 2 * n * sizeof(uint32_t)));
        uint32_t* vinfo = hinfo + n;
        k_region_pack<<<grid2(w, h, b), b, 0, ctx->stream>>>(l, r, u, d, w, h, hinfo, vinfo);
        launched(ctx, "k_region_pack");
        constexpr int kVPF = 8, kHPF = 16;
        // a chunk's prefixes are all written before its outputs read the ring
        const int ring_h = 2 * max_arm + 2 + kHPF - 1, ring_v = 2 * max_arm + 2 + kVPF - 1;
        dim3 tb(32, 4);
        const size_t smem_h = static_cast<size_t>(ring_h) * kAggThreads * sizeof(double);
        const size_t smem_v = static_cast<size_t>(ring_v) * kAggThreads * sizeof(double);
        smem_attr(ctx, k_agg_h2<kHPF>, 227 * 1024, true);
        smem_attr(ctx, k_agg_v2<kVPF>, 227 * 1024, true);
        k_agg_h2<kHPF><<<dim3((nd + 31) / 32, (h + 3) / 4), tb, smem_h, ctx->stream>>>(cost, w, h, nd, hinfo, lag,
                                                                                      ring_h, hsum);
        launched(ctx, "k_agg_h2");
        k_agg_v2<kVPF><<<dim3((nd + 31) / 32, (w + 3) / 4), tb, smem_v, ctx->stream>>>(hsum, w, h, nd, vinfo, lag,
                                                                                      ring_v, out);
        launched(ctx, "k_agg_v2");
        return;
    }
    int* region = static_cast<int*>(scratch(ctx, S_REGION, n * sizeof(int)));
    k_region_size<<<grid2(w, h, b), b, 0, ctx->stream>>>(l, r, u, d, w, h, region);
    launched(ctx, "k_region_size");
    const int ring = ring_size(max_arm);
    int rows = 4;
    while (rows > 1 && static_cast<size_t>(ring) * 32 * rows * sizeof(double) > 200 * 1024) rows >>= 1;
    dim3 tb(32, rows);
    size_t smem = static_cast<size_t>(ring) * 32 * rows * sizeof(double);
    smem_attr(ctx, k_agg_hpass, 227 * 1024);
    smem_attr(ctx, k_agg_vpass, 227 * 1024);
    dim3 gh((nd + 31) / 32, (h + rows - 1) / rows);
    k_agg_hpass<<<gh, tb, smem, ctx->stream>>>(cost, w, h, nd, l, r, lag, ring - 1, hsum);
    launched(ctx, "k_agg_hpass");
    dim3 gv((nd + 31) / 32, (w + rows - 1) / rows);
    k_agg_vpass<<<gv, tb, smem, ctx->stream>>>(hsum, w, h, nd, u, d, region, lag, ring - 1, out);
    launched(ctx, "k_agg_vpass");
}

void select_disparity_wta(dco_ctx* ctx, const float* cost, int w, int h, int d_min, int nd,
                          float* disp) {
    const size_t n = static_cast<size_t>(w) * h;
    k_wta<<<blocks_for(n * 32, 256), 256, 0, ctx->stream>>>(cost, static_cast<int>(n), nd, d_min,
                                                            disp);
    launched(ctx, "k_wta");
}

void refine_disparity_histogram(dco_ctx* ctx, const float* disp, int w, int h, const uint8_t* l,
                                const uint8_t* r, const uint8_t* u, const uint8_t* d, int iters,
                                int bin_bound, int max_arm, float* out) {
    const size_t n = static_cast<size_t>(w) * h;
    require(iters >= 0, "refine_disparity_histogram: negative iteration count");
    if (iters == 0) {
        cuda_check(cudaMemcpyAsync(out, disp, n * 4, cudaMemcpyDeviceToDevice, ctx->stream), "copy");
        return;
    }
    int* bmax = static_cast<int*>(scratch(ctx, S_FLAG_BIN, 64));
    cuda_check(cudaMemsetAsync(bmax, 0, sizeof(int), ctx->stream), "memset");
    k_bin_max<<<blocks_for(n, 256), 256, 0, ctx->stream>>>(disp, static_cast<int>(n), bmax);
    launched(ctx, "k_bin_max");
    int cap = bin_bound + 1;
    if (bin_bound < 0) {  // unknown input range: read the bound back
        int hb = 0;
        cuda_check(cudaMemcpyAsync(&hb, bmax, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream), "d2h");
        cuda_check(cudaStreamSynchronize(ctx->stream), "sync");
        cap = hb + 1;
    }
    require(cap <= 8192, "refine_disparity_histogram: disparities above 8191 are not supported");
    cap = (cap + 31) & ~31;
    if (cap <= 4096 && max_arm <= 127 && w <= 65535 && !getenv("DCO_REFINE_DENSE")) {  // span counts fit a byte
        // region extrema + exact histograms only where a region holds two or more bins
        float* bufs2[2] = {static_cast<float*>(scratch(ctx, S_DISP0, n * 4)),
                           static_cast<float*>(scratch(ctx, S_DISP1, n * 4))};
        uint2* mm = static_cast<uint2*>(scratch(ctx, S_HSUM, n * sizeof(uint2)));
        int* queue = static_cast<int*>(scratch(ctx, S_TMP1, (n + 1) * sizeof(int)));
        uint32_t* runs = static_cast<uint32_t*>(scratch(ctx, S_RUNS, n * sizeof(uint32_t)));
        const int rows = 1;
        dim3 b(128, rows);
        dim3 g((w + 127) / 128, h);
        const size_t hsm = static_cast<size_t>(kSlowWarps) * (cap / 2) * sizeof(uint32_t);
        smem_attr(ctx, k_ref_slow, static_cast<int>(hsm));
        const size_t rsm = static_cast<size_t>((w + 31) / 32) * sizeof(uint32_t);
        smem_attr(ctx, k_ref_runs, static_cast<int>(rsm));
        const float* src = disp;
        for (int it = 0; it < iters; ++it) {
            float* dst = (it == iters - 1) ? out : bufs2[it & 1];
            k_ref_runs<<<h, 256, rsm, ctx->stream>>>(src, w, h, cap, runs);
            launched(ctx, "k_ref_runs");
            k_ref_hminmax<<<g, b, 0, ctx->stream>>>(runs, w, h, l, r, mm);
            launched(ctx, "k_ref_hminmax");
            cuda_check(cudaMemsetAsync(queue, 0, sizeof(int), ctx->stream), "memset");
            k_ref_vminmax<<<g, b, 0, ctx->stream>>>(src, w, h, u, d, mm, dst, queue);
            launched(ctx, "k_ref_vminmax");
            k_ref_slow<<<sm_count(ctx) * 4, kSlowWarps * 32, hsm, ctx->stream>>>(runs, w, h, l, r, u, d, cap, queue,
                                                                                 dst);
            launched(ctx, "k_ref_slow");
            src = dst;
        }
        return;
    }
    const int warps = 8;
    const int rows_cap = 2 * max_arm + 2;
    size_t smem = static_cast<size_t>(warps) * (cap + 3 * rows_cap + 1) * sizeof(unsigned);
    smem_attr(ctx, k_hist_refine, 227 * 1024);
    float* bufs[2] = {static_cast<float*>(scratch(ctx, S_DISP0, n * 4)),
                      static_cast<float*>(scratch(ctx, S_DISP1, n * 4))};
    const float* src = disp;
    const unsigned blocks = static_cast<unsigned>(std::min<size_t>(blocks_for(n, warps), 148 * 16));
    // exact integer cross-aggregation of one-hot bins (preferred, O(N*bins))
    const int nbp = cap <= 64 ? 64 : cap <= 128 ? 128 : cap <= 256 ? 256 : 0;
    uint8_t* hcnt = nbp ? static_cast<uint8_t*>(scratch(ctx, S_HSUM, n * nbp)) : nullptr;
    const int lag = max_arm + 1, ring = ring_size(max_arm);
    const int vwarps = 4;
    const size_t vsmem = static_cast<size_t>(vwarps) * ring * nbp * sizeof(unsigned short);
    const size_t hsmem = static_cast<size_t>(nbp) * ((w + 31) / 32) * sizeof(unsigned);
    smem_attr(ctx, k_refine_vmode3<2>, 227 * 1024);
    smem_attr(ctx, k_refine_vmode3<4>, 227 * 1024);
    smem_attr(ctx, k_refine_vmode3<8>, 227 * 1024);
    smem_attr(ctx, k_refine_vmode2<1>, 227 * 1024);
    smem_attr(ctx, k_refine_vmode2<2>, 227 * 1024);
    smem_attr(ctx, k_refine_vmode2<4>, 227 * 1024);
    smem_attr(ctx, k_refine_vmode2<8>, 227 * 1024);
    const bool aggregated = nbp && vsmem <= 200 * 1024 && hsmem <= 200 * 1024;
    // packed u16 pairs: every column prefix stays below 65536
    const bool packed = aggregated && nbp >= 64 && static_cast<long>(h) * (2 * max_arm + 1) < 65536;
    const int ring3 = 8 + 2 * max_arm + 2;
    const size_t vsmem3 = static_cast<size_t>(vwarps) * ring3 * 32 * (nbp / 64) * sizeof(uint32_t);
    const bool per_thread = cap <= 256;
    const size_t smem_t = static_cast<size_t>(cap) * kHistThreads * sizeof(unsigned short);
    smem_attr(ctx, k_hist_refine_thread, 227 * 1024);
    const unsigned blocks_t = static_cast<unsigned>(std::min<size_t>(blocks_for(n, kHistThreads), 148 * 8));
    for (int it = 0; it < iters; ++it) {
        float* dst = (it == iters - 1) ? out : bufs[it & 1];
        if (aggregated) {
            k_refine_hscatter<<<static_cast<unsigned>(std::min<size_t>(blocks_for(n, kHcThreads), 148 * 8)),
                                kHcThreads, static_cast<size_t>(nbp) * kHcThreads, ctx->stream>>>(src, w, h, l, r,
                                                                                                  nbp, hcnt);
            launched(ctx, "k_refine_hscatter");
            int seg = packed ? 64 : 32;
            if (const char* e = getenv("DCO_REFINE_SEG")) seg = std::max(8, atoi(e));  // tuning hook
            const int nseg = (h + seg - 1) / seg;
            unsigned* carry = static_cast<unsigned*>(scratch(ctx, S_TMP1, static_cast<size_t>(w) * nseg * nbp * 4));
            dim3 vb(32 * vwarps), vg((w * nseg + vwarps - 1) / vwarps);
            if (packed) {
                switch (nbp / 32) {
                    case 2:
                        k_refine_segsum4<2><<<w * nseg, 128, 0, ctx->stream>>>(hcnt, w, h, seg, nseg, lag, carry);
                        k_refine_vmode3<2><<<vg, vb, vsmem3, ctx->stream>>>(src, hcnt, w, h, u, d, lag, ring3, seg,
                                                                            nseg, carry, dst);
                        break;
                    case 4:
                        k_refine_segsum4<4><<<w * nseg, 128, 0, ctx->stream>>>(hcnt, w, h, seg, nseg, lag, carry);
                        k_refine_vmode3<4><<<vg, vb, vsmem3, ctx->stream>>>(src, hcnt, w, h, u, d, lag, ring3, seg,
                                                                            nseg, carry, dst);
                        break;
                    default:
                        k_refine_segsum4<8><<<w * nseg, 128, 0, ctx->stream>>>(hcnt, w, h, seg, nseg, lag, carry);
                        k_refine_vmode3<8><<<vg, vb, vsmem3, ctx->stream>>>(src, hcnt, w, h, u, d, lag, ring3, seg,
                                                                            nseg, carry, dst);
                        break;
                }
                launched(ctx, "k_refine_segsum4");
                launched(ctx, "k_refine_vmode3");
                src = dst;
                continue;
            }
            switch (nbp / 32) {
                case 1:
                    k_refine_segsum<1><<<vg, vb, 0, ctx->stream>>>(hcnt, w, h, seg, nseg, lag, carry);
                    k_refine_vmode2<1><<<vg, vb, vsmem, ctx->stream>>>(src, hcnt, w, h, u, d, lag, ring - 1, seg, nseg, carry, dst);
                    break;
                case 2:
                    k_refine_segsum<2><<<vg, vb, 0, ctx->stream>>>(hcnt, w, h, seg, nseg, lag, carry);
                    k_refine_vmode2<2><<<vg, vb, vsmem, ctx->stream>>>(src, hcnt, w, h, u, d, lag, ring - 1, seg, nseg, carry, dst);
                    break;
                case 4:
                    k_refine_segsum<4><<<vg, vb, 0, ctx->stream>>>(hcnt, w, h, seg, nseg, lag, carry);
                    k_refine_vmode2<4><<<vg, vb, vsmem, ctx->stream>>>(src, hcnt, w, h, u, d, lag, ring - 1, seg, nseg, carry, dst);
                    break;
                default:
                    k_refine_segsum<8><<<vg, vb, 0, ctx->stream>>>(hcnt, w, h, seg, nseg, lag, carry);
                    k_refine_vmode2<8><<<vg, vb, vsmem, ctx->stream>>>(src, hcnt, w, h, u, d, lag, ring - 1, seg, nseg, carry, dst);
                    break;
            }
            launched(ctx, "k_refine_segsum");
            launched(ctx, "k_refine_vmode2");
        } else if (per_thread) {
            k_hist_refine_thread<<<blocks_t, kHistThreads, smem_t, ctx->stream>>>(src, w, h, l, r, u, d, bmax, cap, dst);
            launched(ctx, "k_hist_refine_thread");
        } else {
            k_hist_refine<<<blocks, warps * 32, smem, ctx->stream>>>(src, w, h, l, r, u, d, bmax, cap, rows_cap, dst);
            launched(ctx, "k_hist_refine");
        }
        src = dst;
    }
}

void flip_horizontal(dco_ctx* ctx, const float* img, int w, int h, float* out) {
    dim3 b(32, 8);
    k_flip_h<<<grid2(w, h, b), b, 0, ctx->stream>>>(img, w, h, out);
    launched(ctx, "k_flip_h");
}

void lr_consistency(dco_ctx* ctx, const float* dl, const float* dr, int w, int h, double max_diff, float* out) {
    dim3 b(32, 8);
    k_lr_check<<<grid2(w, h, b), b, 0, ctx->stream>>>(dl, dr, w, h, max_diff, out);
    launched(ctx, "k_lr_check");
}

void disparity_to_sparse_depth(dco_ctx* ctx, const float* disp, int w, int h, const dco_config* cfg,
                               int fw, int fh, float* out) {
    if (fw < w * 2 || fh < h * 2)
        fail(DCO_INPUT, "disparity_to_sparse_depth: full dimensions too small for the quarter map");
    dim3 b(32, 8);
    k_sparse_depth<<<grid2(fw, fh, b), b, 0, ctx->stream>>>(disp, w, h, cfg->focal_px * cfg->baseline_m,
                                                            fw, fh, out);
    launched(ctx, "k_sparse_depth");
}

}  // namespace dco_gpu

using namespace dco_gpu;

extern "C" {

int dco_downsample_half(dco_ctx* ctx, const float* img, int w, int h, float* out) {
    return guarded(ctx, [&] { downsample_half(ctx, img, w, h, out); });
}

int dco_ingest_gray8(dco_ctx* ctx, const uint8_t* g8, int w, int h, float* full, float* quarter) {
    return guarded(ctx, [&] { ingest_gray8(ctx, g8, w, h, full, quarter); });
}

int dco_build_cross_windows(dco_ctx* ctx, const float* img, int w, int h, const dco_config* cfg,
                            uint8_t* l, uint8_t* r, uint8_t* u, uint8_t* d) {
    return guarded(ctx, [&] { build_cross_windows(ctx, img, w, h, cfg, l, r, u, d); });
}

int dco_census_transform(dco_ctx* ctx, const float* img, int w, int h, int ww, int wh, uint64_t* out) {
    return guarded(ctx, [&] { census_transform(ctx, img, w, h, ww, wh, out); });
}

int dco_compute_cost_volume(dco_ctx* ctx, const float* left, const float* right, int w, int h,
                            const uint8_t* l, const uint8_t* r, const uint8_t* u, const uint8_t* d,
                            const dco_config* cfg, float* cost) {
    return guarded(ctx, [&] { compute_cost_volume(ctx, left, right, w, h, l, r, u, d, cfg, cost); });
}

int dco_aggregate_costs(dco_ctx* ctx, const float* cost, int w, int h, int d_min, int d_max,
                        const uint8_t* l, const uint8_t* r, const uint8_t* u, const uint8_t* d,
                        float* out) {
    return guarded(ctx, [&] {
        require(d_max >= d_min, "aggregate_costs: empty disparity range");
        // the ring must cover the longest arm present: reduce it on the device
        aggregate_costs(ctx, cost, w, h, d_max - d_min + 1, l, r, u, d,
                        max_arm_length(ctx, l, r, u, d, w, h), out);
    });
}

int dco_select_disparity_wta(dco_ctx* ctx, const float* cost, int w, int h, int d_min, int d_max,
                             float* disp) {
    return guarded(ctx, [&] {
        require(d_max >= d_min, "select_disparity_wta: empty disparity range");
        select_disparity_wta(ctx, cost, w, h, d_min, d_max - d_min + 1, disp);
    });
}

int dco_refine_disparity_histogram(dco_ctx* ctx, const float* disp, int w, int h, const uint8_t* l,
                                   const uint8_t* r, const uint8_t* u, const uint8_t* d, int iters,
                                   float* out) {
    return guarded(ctx, [&] { refine_disparity_histogram(ctx, disp, w, h, l, r, u, d, iters, -1, max_arm_length(ctx, l, r, u, d, w, h), out); });
}

int dco_disparity_to_sparse_depth(dco_ctx* ctx, const float* disp, int w, int h, const dco_config* cfg,
                                  int fw, int fh, float* out) {
    return guarded(ctx, [&] { disparity_to_sparse_depth(ctx, disp, w, h, cfg, fw, fh, out); });
}

int dco_flip_horizontal(dco_ctx* ctx, const float* img, int w, int h, float* out) {
    return guarded(ctx, [&] {
        require(w >= 1 && h >= 1, "flip_horizontal: empty image");
        require(img != out, "flip_horizontal: in-place flip is not supported");
        flip_horizontal(ctx, img, w, h, out);
    });
}

int dco_lr_consistency(dco_ctx* ctx, const float* disp_left, const float* disp_right, int w, int h, double max_diff,
                       float* out) {
    return guarded(ctx, [&] {
        require(w >= 1 && h >= 1, "lr_consistency: empty map");
        require(max_diff >= 0.0, "lr_consistency: negative tolerance");
        lr_consistency(ctx, disp_left, disp_right, w, h, max_diff, out);
    });
}

}  // extern "C"
