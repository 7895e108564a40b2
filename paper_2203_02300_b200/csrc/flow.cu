// flow.cu — coarse-to-fine patch inverse-search optical flow (reference
// src/flow.cpp:22-205, DIS without variational refinement) on sm_100a.
//
// Per pyramid level three kernels run, for BOTH directions of the pipeline's
// bidirectional flow at once (blockIdx.z = direction; the `from` pyramid is
// shared): the flow upsample from the coarser level (flow.cpp:39-62), one
// warp per 8x8 patch for the 12-step inverse-compositional Gauss-Newton
// search (flow.cpp:72-121, double sums in the reference's (dy,dx) order), and
// one thread per pixel gathering the weighted patch mean in the reference's
// (py,px) patch order (flow.cpp:123-160). Arithmetic order matches the
// reference exactly (compiled with --fmad=false), so the field is bit-exact.
#include <math.h>

#include <algorithm>
#include <vector>

#include "common.cuh"

namespace dco_gpu {
namespace {

constexpr int kPatch = 8;
constexpr int kStride = 4;
constexpr int kIters = 12;
constexpr int kMinLevelDim = 16;

struct Level {
    int w, h;
    int nx, ny;  // patch grid
};

// patch_positions, flow.cpp:29-35: stride grid, last position pinned.
__host__ __device__ __forceinline__ int patch_count(int extent) {
    int last = extent - kPatch;
    int n = last >= 0 ? last / kStride + 1 : 0;
    if (n == 0 || (n - 1) * kStride != last) ++n;
    return n;
}
__host__ __device__ __forceinline__ int patch_pos(int j, int n, int extent) {
    int last = extent - kPatch;
    return j == n - 1 ? (last > 0 ? last : 0) : j * kStride;
}

// std::clamp semantics exactly (NaN and signed zero pass through unchanged).
__device__ __forceinline__ float clampf(float v, float lo, float hi) {
    return (v < lo) ? lo : ((hi < v) ? hi : v);
}

// sample_bilinear, image.cpp:27-39 (float arithmetic, clamped).
__device__ __forceinline__ float sample_bilinear(const float* img, int w, int h, float x, float y) {
    x = clampf(x, 0.0f, static_cast<float>(w - 1));
    y = clampf(y, 0.0f, static_cast<float>(h - 1));
    int x0 = static_cast<int>(x), y0 = static_cast<int>(y);
    int x1 = min(x0 + 1, w - 1), y1 = min(y0 + 1, h - 1);
    float fx = x - static_cast<float>(x0), fy = y - static_cast<float>(y0);
    const float* r0 = img + static_cast<size_t>(y0) * w;
    const float* r1 = img + static_cast<size_t>(y1) * w;
    float top = __ldg(r0 + x0) * (1.0f - fx) + __ldg(r0 + x1) * fx;
    float bot = __ldg(r1 + x0) * (1.0f - fx) + __ldg(r1 + x1) * fx;
    return top * (1.0f - fy) + bot * fy;
}

// downsample_half (pyramid.cpp:5-17) of up to three same-size images in one
// launch (z = image): one pyramid level of the from / to / to frames.
struct PyrLevel {
    const float* src[3];
    float* dst[3];
};
__global__ void k_pyr_level(const __grid_constant__ PyrLevel pl, int w, int ow, int oh) {
    int x = blockIdx.x * blockDim.x + threadIdx.x;
    int y = blockIdx.y * blockDim.y + threadIdx.y;
    if (x >= ow || y >= oh) return;
    const float* r0 = pl.src[blockIdx.z] + static_cast<size_t>(2 * y) * w + 2 * x;
    const float* r1 = r0 + w;
    float sum = r0[0] + r0[1] + r1[0] + r1[1];
    pl.dst[blockIdx.z][static_cast<size_t>(y) * ow + x] = sum * 0.25f;
}

// upsample_flow, flow.cpp:39-62. z = direction.
__global__ void k_flow_upsample(const float* __restrict__ cu, const float* __restrict__ cv, int cw,
                                int ch, float* __restrict__ fu, float* __restrict__ fv, int fw,
                                int fh, size_t cstride, size_t fstride) {
    int x = blockIdx.x * blockDim.x + threadIdx.x;
    int y = blockIdx.y * blockDim.y + threadIdx.y;
    if (x >= fw || y >= fh) return;
    cu += blockIdx.z * cstride;
    cv += blockIdx.z * cstride;
    fu += blockIdx.z * fstride;
    fv += blockIdx.z * fstride;
    float sy = clampf((static_cast<float>(y) + 0.5f) * 0.5f - 0.5f, 0.0f, static_cast<float>(ch - 1));
    int y0 = static_cast<int>(sy), y1 = min(y0 + 1, ch - 1);
    float fy = sy - static_cast<float>(y0);
    float sx = clampf((static_cast<float>(x) + 0.5f) * 0.5f - 0.5f, 0.0f, static_cast<float>(cw - 1));
    int x0 = static_cast<int>(sx), x1 = min(x0 + 1, cw - 1);
    float fx = sx - static_cast<float>(x0);
    size_t i00 = static_cast<size_t>(y0) * cw + x0, i10 = static_cast<size_t>(y0) * cw + x1;
    size_t i01 = static_cast<size_t>(y1) * cw + x0, i11 = static_cast<size_t>(y1) * cw + x1;
    float tu = cu[i00] * (1 - fx) + cu[i10] * fx;
    float bu = cu[i01] * (1 - fx) + cu[i11] * fx;
    float tv = cv[i00] * (1 - fx) + cv[i10] * fx;
    float bv = cv[i01] * (1 - fx) + cv[i11] * fx;
    size_t o = static_cast<size_t>(y) * fw + x;
    fu[o] = 2.0f * (tu * (1 - fy) + bu * fy);
    fv[o] = 2.0f * (tv * (1 - fy) + bv * fy);
}

// search_patch, flow.cpp:72-121, one HALF-WARP per patch (two patches per
// warp); z = direction. Lane l of a half owns samples n = l + 16 q, q < 4
// (template and gradients stay in its registers); every product gx*r, gy*r,
// r*r of two floats is exact in double, so the reference's sequential sums
// are reproduced by one lane per sum adding the exact terms in (dy, dx)
// order -- the same rounding chains, run side by side (both halves' chains
// share each instruction, as do the divisions and the step). The Hessian's
// three chains and the first iteration's three (whose samples need only the
// seed) run together on lanes 0..5 of the half: most patches converge in that
// first iteration. A half whose patch is done idles until the other's is.
// Term rows are 65 doubles apart: the chain lanes' loads fall in distinct
// bank pairs.
constexpr int kPatchWarps = 4;
constexpr int kTermPitch = 65;

__global__ void __launch_bounds__(kPatchWarps * 32) k_flow_patch_w(const float* __restrict__ from,
                                                                  const float* __restrict__ to0,
                                                                  const float* __restrict__ to1, int w, int h,
                                                                  int nx, int ny,
                                                                  const float* __restrict__ init_u_base,
                                                                  const float* __restrict__ init_v_base,
                                                                  size_t field_stride, float* __restrict__ res_base,
                                                                  size_t res_stride) {
    constexpr int N = kPatch * kPatch;
    __shared__ double s_term[kPatchWarps][2][6 * kTermPitch];
    const int lane = threadIdx.x & 31, wp = threadIdx.x >> 5;
    const int hl = lane >> 4, ll = lane & 15;
    const int j0 = (blockIdx.x * kPatchWarps + wp) * 2;
    const int np = nx * ny;
    if (j0 >= np) return;  // warp-uniform
    const int j = min(j0 + hl, np - 1);  // an odd last patch: the second half repeats it, inactive
    bool active = j0 + hl < np;
    const float* to = blockIdx.z ? to1 : to0;
    const float* iu = init_u_base + blockIdx.z * field_stride;
    const float* iv = init_v_base + blockIdx.z * field_stride;
    float* res = res_base + blockIdx.z * res_stride;
    const int jy = j / nx, jx = j - jy * nx;
    const int px = patch_pos(jx, nx, w), py = patch_pos(jy, ny, h);
    const int cx = min(px + kPatch / 2, w - 1), cy = min(py + kPatch / 2, h - 1);
    const float seed_u = iu[static_cast<size_t>(cy) * w + cx];
    const float seed_v = iv[static_cast<size_t>(cy) * w + cx];
    double* term = s_term[wp][hl];
    float tv[4], gxv[4], gyv[4];

    // template, gradients and the Hessian terms (flow.cpp:78-89), and the
    // first iteration's terms at the seed (flow.cpp:93-100)
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        const int n = ll + 16 * q;
        const int y = py + (n >> 3), x = px + (n & 7);
        const int ym = max(y - 1, 0), yp = min(y + 1, h - 1);
        const int xm = max(x - 1, 0), xp = min(x + 1, w - 1);
        const float* row = from + static_cast<size_t>(y) * w;
        tv[q] = __ldg(row + x);
        gxv[q] = 0.5f * (__ldg(row + xp) - __ldg(row + xm));
        gyv[q] = 0.5f * (__ldg(from + static_cast<size_t>(yp) * w + x) - __ldg(from + static_cast<size_t>(ym) * w + x));
        const float r =
            sample_bilinear(to, w, h, static_cast<float>(x) + seed_u, static_cast<float>(y) + seed_v) - tv[q];
        term[0 * kTermPitch + n] = static_cast<double>(gxv[q]) * gxv[q];
        term[1 * kTermPitch + n] = static_cast<double>(gxv[q]) * gyv[q];
        term[2 * kTermPitch + n] = static_cast<double>(gyv[q]) * gyv[q];
        term[3 * kTermPitch + n] = static_cast<double>(gxv[q]) * r;
        term[4 * kTermPitch + n] = static_cast<double>(gyv[q]) * r;
        term[5 * kTermPitch + n] = static_cast<double>(r) * r;
    }
    __syncwarp();
    // h00, h01, h11 (from 1e-6, 0, 1e-6) on lanes 0..2 of the half; bu, bv, sse on 3..5
    double acc = (ll == 0 || ll == 2) ? 1e-6 : 0.0;
    if (ll < 6) {
        const double* tl = term + ll * kTermPitch;
#pragma unroll 16
        for (int n = 0; n < N; ++n) acc += tl[n];
    }
    const int hb = lane & 16;  // the half's lane 0
    const double h00 = __shfl_sync(0xffffffffu, acc, hb + 0);
    const double h01 = __shfl_sync(0xffffffffu, acc, hb + 1);
    const double h11 = __shfl_sync(0xffffffffu, acc, hb + 2);
    double bu = __shfl_sync(0xffffffffu, acc, hb + 3);
    double bv = __shfl_sync(0xffffffffu, acc, hb + 4);
    double sse = __shfl_sync(0xffffffffu, acc, hb + 5);
    const double det = h00 * h11 - h01 * h01;
    const double inv00 = h11 / det, inv01 = -h01 / det, inv11 = h00 / det;

    float u = seed_u, v = seed_v;
    double mse = 0.0;
    const float fw = static_cast<float>(w), fh = static_cast<float>(h);
    for (int iter = 0; iter < kIters && __any_sync(0xffffffffu, active); ++iter) {
        if (iter > 0) {
            __syncwarp();  // previous iteration's term reads are done
            if (active) {
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    const int n = ll + 16 * q;
                    const float sx = static_cast<float>(px + (n & 7)) + u;
                    const float sy = static_cast<float>(py + (n >> 3)) + v;
                    const float r = sample_bilinear(to, w, h, sx, sy) - tv[q];
                    term[0 * kTermPitch + n] = static_cast<double>(gxv[q]) * r;
                    term[1 * kTermPitch + n] = static_cast<double>(gyv[q]) * r;
                    term[2 * kTermPitch + n] = static_cast<double>(r) * r;
                }
            }
            __syncwarp();
            double sum = 0.0;  // bu, bv, sse on lanes 0, 1, 2 of the half
            if (ll < 3 && active) {
                const double* tl = term + ll * kTermPitch;
#pragma unroll 16
                for (int n = 0; n < N; ++n) sum += tl[n];
            }
            bu = __shfl_sync(0xffffffffu, sum, hb + 0);
            bv = __shfl_sync(0xffffffffu, sum, hb + 1);
            sse = __shfl_sync(0xffffffffu, sum, hb + 2);
        }
        if (!active) continue;
        mse = sse / (kPatch * kPatch);
        const double step_u = inv00 * bu + inv01 * bv;
        const double step_v = inv01 * bu + inv11 * bv;
        u -= static_cast<float>(step_u);
        v -= static_cast<float>(step_v);
        if (!isfinite(u) || !isfinite(v)) {
            u = seed_u;
            v = seed_v;
            active = false;
            continue;
        }
        u = clampf(u, -fw, fw);
        v = clampf(v, -fh, fh);
        if (step_u * step_u + step_v * step_v < 1e-6) active = false;
    }
    if (ll == 0 && j0 + hl < np) {
        res[3 * j + 0] = u;
        res[3 * j + 1] = v;
        res[3 * j + 2] = static_cast<float>(1.0 / (mse + 1e-2));
    }
}

// estimate_level gather, flow.cpp:137-160: per pixel, the double-weighted mean
// of the covering patches accumulated in (py, px) loop order.
__global__ void k_flow_gather(const float* __restrict__ res_base, size_t res_stride, int w, int h,
                              int nx, int ny, float* __restrict__ u_base, float* __restrict__ v_base,
                              size_t field_stride, int* __restrict__ uncovered) {
    int x = blockIdx.x * blockDim.x + threadIdx.x;
    int y = blockIdx.y * blockDim.y + threadIdx.y;
    if (x >= w || y >= h) return;
    const float* res = res_base + blockIdx.z * res_stride;
    double au = 0.0, av = 0.0, aw = 0.0;
    int jy0 = max(0, (y - (kPatch - 1) + kStride - 1) / kStride - 1);
    int jx0 = max(0, (x - (kPatch - 1) + kStride - 1) / kStride - 1);
    for (int jy = jy0; jy < ny; ++jy) {
        int py = patch_pos(jy, ny, h);
        if (py > y) break;
        if (y >= py + kPatch) continue;
        for (int jx = jx0; jx < nx; ++jx) {
            int px = patch_pos(jx, nx, w);
            if (px > x) break;
            if (x >= px + kPatch) continue;
            const float* r = res + 3 * (static_cast<size_t>(jy) * nx + jx);
            float ru = r[0], rv = r[1], rw = r[2];
            au += static_cast<double>(rw) * ru;
            av += static_cast<double>(rw) * rv;
            aw += rw;
        }
    }
    size_t i = static_cast<size_t>(y) * w + x;
    float* fu = u_base + blockIdx.z * field_stride;
    float* fv = v_base + blockIdx.z * field_stride;
    if (aw > 0.0) {
        fu[i] = static_cast<float>(au / aw);
        fv[i] = static_cast<float>(av / aw);
    } else {
        fu[i] = 0.0f;
        fv[i] = 0.0f;
        atomicAdd(uncovered, 1);
    }
}

// Nearest-covered fallback of flow.cpp:162-180 (only reachable when a patch
// weight is zero, i.e. a non-finite patch error). Serial per pixel, in the
// reference's (radius, dy, dx) search order, reading the gathered weights.
__global__ void k_flow_fill(const float* __restrict__ res_base, size_t res_stride, int w, int h,
                            int nx, int ny, float* __restrict__ u_base, float* __restrict__ v_base,
                            size_t field_stride, const int* __restrict__ uncovered) {
    if (*uncovered == 0) return;  // the common case: every pixel was covered
    int x = blockIdx.x * blockDim.x + threadIdx.x;
    int y = blockIdx.y * blockDim.y + threadIdx.y;
    if (x >= w || y >= h) return;
    const float* res = res_base + blockIdx.z * res_stride;
    auto covered = [&](int qx, int qy) {
        double aw = 0.0;
        for (int jy = 0; jy < ny; ++jy) {
            int py = patch_pos(jy, ny, h);
            if (qy < py || qy >= py + kPatch) continue;
            for (int jx = 0; jx < nx; ++jx) {
                int px = patch_pos(jx, nx, w);
                if (qx < px || qx >= px + kPatch) continue;
                aw += res[3 * (static_cast<size_t>(jy) * nx + jx) + 2];
            }
        }
        return aw > 0.0;
    };
    if (covered(x, y)) return;
    float* fu = u_base + blockIdx.z * field_stride;
    float* fv = v_base + blockIdx.z * field_stride;
    size_t i = static_cast<size_t>(y) * w + x;
    int rmax = max(w, h);
    for (int radius = 1; radius < rmax; ++radius) {
        for (int dy = -radius; dy <= radius; ++dy)
            for (int dx = -radius; dx <= radius; ++dx) {
                int qx = x + dx, qy = y + dy;
                if (qx < 0 || qy < 0 || qx >= w || qy >= h) continue;
                if (covered(qx, qy)) {
                    size_t q = static_cast<size_t>(qy) * w + qx;
                    fu[i] = fu[q];  // covered pixels are final: no race
                    fv[i] = fv[q];
                    return;
                }
            }
    }
}

inline dim3 grid2(int w, int h, dim3 b, int z) {
    return dim3((w + b.x - 1) / b.x, (h + b.y - 1) / b.y, z);
}

}  // namespace

void downsample_half(dco_ctx* ctx, const float* img, int w, int h, float* out);

// compute_flow for `dirs` directions that share the `from` frame
// (flow.cpp:185-205): flow from -> to[k], written to u[k], v[k].
void compute_flow_multi(dco_ctx* ctx, const float* from, const float* const* to, int dirs, int w,
                        int h, float* const* u_out, float* const* v_out) {
    if (w < kPatch || h < kPatch) fail(DCO_INPUT, "compute_flow: frames smaller than the patch size");
    require(dirs >= 1 && dirs <= 2, "compute_flow: 1 or 2 directions");
    int levels = 1;
    while (std::min(w, h) / (1 << levels) >= kMinLevelDim) ++levels;
    std::vector<Level> lv(levels);
    size_t pyr_elems = 0, max_level = 0, max_patches = 0;
    for (int l = 0, lw = w, lh = h; l < levels; ++l, lw /= 2, lh /= 2) {
        lv[l] = {lw, lh, patch_count(lw), patch_count(lh)};
        pyr_elems += static_cast<size_t>(lw) * lh;
        max_level = std::max(max_level, static_cast<size_t>(lw) * lh);
        max_patches = std::max(max_patches, static_cast<size_t>(lv[l].nx) * lv[l].ny);
    }
    // pyramids: [from | to0 | to1] per level, level 0 aliases the inputs
    float* pyr = static_cast<float*>(scratch(ctx, S_FLOW_PYR, pyr_elems * 3 * sizeof(float)));
    std::vector<const float*> p_from(levels), p_to[2];
    p_to[0].resize(levels);
    p_to[1].resize(levels);
    size_t off = 0;
    p_from[0] = from;
    for (int k = 0; k < dirs; ++k) p_to[k][0] = to[k];
    for (int l = 1; l < levels; ++l) {
        size_t n = static_cast<size_t>(lv[l].w) * lv[l].h;
        PyrLevel pl{};
        float* f = pyr + off;
        off += n;
        pl.src[0] = p_from[l - 1];
        pl.dst[0] = f;
        p_from[l] = f;
        for (int k = 0; k < dirs; ++k) {
            float* t = pyr + off;
            off += n;
            pl.src[1 + k] = p_to[k][l - 1];
            pl.dst[1 + k] = t;
            p_to[k][l] = t;
        }
        // every level of the three pyramids in one launch (pyramid.cpp:5-17)
        require(lv[l - 1].w >= 2 && lv[l - 1].h >= 2, "downsample_half: dimensions must be at least 2x2");
        dim3 bd(32, 8);
        k_pyr_level<<<dim3((lv[l].w + 31) / 32, (lv[l].h + 7) / 8, 1 + dirs), bd, 0, ctx->stream>>>(
            pl, lv[l - 1].w, lv[l].w, lv[l].h);
        launched(ctx, "k_pyr_level");
    }
    float* res = static_cast<float*>(scratch(ctx, S_FLOW_PATCH, max_patches * 3 * 2 * sizeof(float)));
    // field ping-pong: [buf][dir][u|v][max_level]
    float* fld = static_cast<float*>(scratch(ctx, S_FLOW_ACC, max_level * 8 * sizeof(float)));
    int* uncovered = static_cast<int*>(scratch(ctx, S_FLAG_FLOW, 64));
    const size_t fs = 2 * max_level;  // direction stride inside one buffer
    auto U = [&](int buf, int k) { return fld + buf * 4 * max_level + k * fs; };
    auto V = [&](int buf, int k) { return fld + buf * 4 * max_level + k * fs + max_level; };
    int cur = 0;
    cuda_check(cudaMemsetAsync(fld, 0, max_level * 8 * sizeof(float), ctx->stream), "memset");
    smem_attr(ctx, k_flow_patch_w, 0, true);  // the whole carveout: 26 KB blocks, register-limited
    dim3 b(32, 8);
    for (int l = levels - 1; l >= 0; --l) {
        const Level& L = lv[l];
        if (l != levels - 1) {
            const Level& C = lv[l + 1];
            k_flow_upsample<<<grid2(L.w, L.h, b, dirs), b, 0, ctx->stream>>>(
                U(cur, 0), V(cur, 0), C.w, C.h, U(cur ^ 1, 0), V(cur ^ 1, 0), L.w, L.h, fs, fs);
            launched(ctx, "k_flow_upsample");
            cur ^= 1;
        }
        int np = L.nx * L.ny;
        const int npw = (np + 1) / 2;  // warps: two patches each
        k_flow_patch_w<<<dim3((npw + kPatchWarps - 1) / kPatchWarps, 1, dirs), kPatchWarps * 32, 0, ctx->stream>>>(
            p_from[l], p_to[0][l], dirs > 1 ? p_to[1][l] : p_to[0][l], L.w, L.h, L.nx, L.ny, U(cur, 0), V(cur, 0), fs, res,
            max_patches * 3);
        launched(ctx, "k_flow_patch_w");
        cuda_check(cudaMemsetAsync(uncovered, 0, sizeof(int), ctx->stream), "memset");
        k_flow_gather<<<grid2(L.w, L.h, b, dirs), b, 0, ctx->stream>>>(
            res, max_patches * 3, L.w, L.h, L.nx, L.ny, U(cur ^ 1, 0), V(cur ^ 1, 0), fs, uncovered);
        launched(ctx, "k_flow_gather");
        cur ^= 1;
        // every pixel is covered by the pinned grid unless a patch weight is 0
        // (non-finite error); the fill kernel exits at once otherwise.
        k_flow_fill<<<grid2(L.w, L.h, b, dirs), b, 0, ctx->stream>>>(
            res, max_patches * 3, L.w, L.h, L.nx, L.ny, U(cur, 0), V(cur, 0), fs, uncovered);
        launched(ctx, "k_flow_fill");
    }
    size_t n0 = static_cast<size_t>(w) * h;
    for (int k = 0; k < dirs; ++k) {
        cuda_check(cudaMemcpyAsync(u_out[k], U(cur, k), n0 * 4, cudaMemcpyDeviceToDevice, ctx->stream),
                   "copy u");
        cuda_check(cudaMemcpyAsync(v_out[k], V(cur, k), n0 * 4, cudaMemcpyDeviceToDevice, ctx->stream),
                   "copy v");
    }
}

}  // namespace dco_gpu

using namespace dco_gpu;

extern "C" int dco_compute_flow(dco_ctx* ctx, const float* from, const float* to, int w, int h,
                                const dco_config* cfg, float* u, float* v) {
    (void)cfg;  // the reference ignores cfg too (flow.cpp:186)
    return guarded(ctx, [&] {
        const float* tos[1] = {to};
        float* us[1] = {u};
        float* vs[1] = {v};
        compute_flow_multi(ctx, from, tos, 1, w, h, us, vs);
    });
}
