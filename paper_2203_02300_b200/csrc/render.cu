// render.cu -- transform_mesh + render_virtual on sm_100a (reference
// src/occlude.cpp:78-169; the composite's virtual layer,
// pose-dependent every frame, pipeline.cpp:247-252).
//
// The reference rasterises triangles in index order into a float depth
// buffer, replacing a pixel when the new perspective-correct depth z (double)
// is strictly below the STORED float depth. Because that comparison sees the
// rounded previous depth, the winner is order-dependent (not simply the
// minimum z), so every pixel must visit its covering triangles in ascending
// index order. Here:
//   k_tri_setup : per triangle, the reference's projection, area and clamped
//                 bounding box (same double expressions, --fmad=false);
//   k_tri_tiles : a warp per triangle counts, then fills, the 16x16 tiles it
//                 overlaps (list offsets from a scan of the counts);
//   k_tile_sort : each tile's list sorted ascending (bitonic, shared memory);
//   k_raster    : one thread per pixel, walking its tile's sorted list with
//                 the reference's barycentrics, depth test and colour.
// Tiles whose list exceeds the shared-memory sort walk every triangle of the
// mesh in order instead (bounding-box culled) -- exact, slower.
#include <math.h>

#include <algorithm>

#include "common.cuh"

namespace dco_gpu {
namespace {

constexpr int kTile = 16;
constexpr int kSortCap = 4096;  // tile lists up to this length are sorted in shared memory

struct TriSetup {
    double ua, va, ub, vb, uc, vc;
    double area;
    double inv_za, inv_zb, inv_zc;
    float ca[3], cb[3], cc[3];
    int x0, x1, y0, y1;  // clamped bounding box; x1 < x0 marks a skipped triangle
};

// transform_mesh, occlude.cpp:78-87 (double products, float result). The
// pose travels as a kernel parameter (no copy per frame).
struct Pose16 {
    double p[16];
};
__global__ void k_transform_mesh(const float* __restrict__ v, int nv, const __grid_constant__ Pose16 ps,
                                 float* __restrict__ out) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= nv) return;
    const double* pose = ps.p;
    const double x = v[3 * i], y = v[3 * i + 1], z = v[3 * i + 2];
    out[3 * i + 0] = static_cast<float>(pose[0] * x + pose[1] * y + pose[2] * z + pose[3]);
    out[3 * i + 1] = static_cast<float>(pose[4] * x + pose[5] * y + pose[6] * z + pose[7]);
    out[3 * i + 2] = static_cast<float>(pose[8] * x + pose[9] * y + pose[10] * z + pose[11]);
}

__device__ __forceinline__ double clampd(double v, double lo, double hi) {  // std::clamp
    return (v < lo) ? lo : ((hi < v) ? hi : v);
}
__device__ __forceinline__ double min3(double a, double b, double c) {  // std::min({a, b, c})
    double m = a;
    if (b < m) m = b;
    if (c < m) m = c;
    return m;
}
__device__ __forceinline__ double max3(double a, double b, double c) {  // std::max({a, b, c})
    double m = a;
    if (m < b) m = b;
    if (m < c) m = c;
    return m;
}

// render_virtual, occlude.cpp:118-145: per-triangle setup + tile counts.
__global__ void k_tri_setup(const float* __restrict__ v, const int* __restrict__ tris, const float* __restrict__ col,
                            int nt, double focal, double cx, double cy, int w, int h, TriSetup* __restrict__ ts) {
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= nt) return;
    TriSetup s;
    s.x0 = 0;
    s.x1 = -1;
    s.y0 = 0;
    s.y1 = -1;
    const int ia = tris[3 * t], ib = tris[3 * t + 1], ic = tris[3 * t + 2];
    const float az = v[3 * ia + 2], bz = v[3 * ib + 2], cz = v[3 * ic + 2];
    if (!(az <= 0.0f || bz <= 0.0f || cz <= 0.0f)) {  // behind camera, no clipping
        s.ua = focal * v[3 * ia] / az + cx;
        s.va = focal * v[3 * ia + 1] / az + cy;
        s.ub = focal * v[3 * ib] / bz + cx;
        s.vb = focal * v[3 * ib + 1] / bz + cy;
        s.uc = focal * v[3 * ic] / cz + cx;
        s.vc = focal * v[3 * ic + 1] / cz + cy;
        s.area = (s.ub - s.ua) * (s.vc - s.va) - (s.uc - s.ua) * (s.vb - s.va);
        if (s.area != 0.0) {
            const double bx0 = clampd(floor(min3(s.ua, s.ub, s.uc) - 0.5), 0.0, static_cast<double>(w - 1));
            const double bx1 = clampd(ceil(max3(s.ua, s.ub, s.uc) - 0.5), 0.0, static_cast<double>(w - 1));
            const double by0 = clampd(floor(min3(s.va, s.vb, s.vc) - 0.5), 0.0, static_cast<double>(h - 1));
            const double by1 = clampd(ceil(max3(s.va, s.vb, s.vc) - 0.5), 0.0, static_cast<double>(h - 1));
            s.x0 = static_cast<int>(bx0);
            s.x1 = static_cast<int>(bx1);
            s.y0 = static_cast<int>(by0);
            s.y1 = static_cast<int>(by1);
            s.inv_za = 1.0 / az;
            s.inv_zb = 1.0 / bz;
            s.inv_zc = 1.0 / cz;
            for (int k = 0; k < 3; ++k) {
                s.ca[k] = col[3 * ia + k];
                s.cb[k] = col[3 * ib + k];
                s.cc[k] = col[3 * ic + k];
            }
        }
    }
    ts[t] = s;
}

// one warp per triangle: lanes stride over the tiles its bounding box overlaps
// (count pass when lists == nullptr, fill pass otherwise)
__global__ void k_tri_tiles(const TriSetup* __restrict__ ts, int nt, int tiles_x, int* __restrict__ counts,
                            const int* __restrict__ offsets, int* __restrict__ cursor, int* __restrict__ lists, int ntiles,
                            long long cap) {
    const int t = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
    if (t >= nt) return;
    if (lists && offsets[ntiles] > cap) return;  // lists do not fit: every tile rasterises the whole mesh
    const TriSetup& s = ts[t];
    if (s.x1 < s.x0) return;
    const int tx0 = s.x0 / kTile, ty0 = s.y0 / kTile;
    const int ntx = s.x1 / kTile - tx0 + 1, nty = s.y1 / kTile - ty0 + 1;
    for (int k = lane; k < ntx * nty; k += 32) {
        const int tile = (ty0 + k / ntx) * tiles_x + tx0 + k % ntx;
        if (lists) {
            lists[offsets[tile] + atomicAdd(cursor + tile, 1)] = t;
        } else {
            atomicAdd(counts + tile, 1);
        }
    }
}

// exclusive scan of the tile counts (one block; tile counts are small)
__global__ void k_tile_scan(const int* __restrict__ counts, int n, int* __restrict__ offsets,
                            int* __restrict__ cursor) {
    __shared__ int warp_tot[32];
    __shared__ int carry;
    if (threadIdx.x == 0) carry = 0;
    __syncthreads();
    const int lane = threadIdx.x & 31, wp = threadIdx.x >> 5;
    for (int base = 0; base < n; base += blockDim.x) {
        const int i = base + threadIdx.x;
        const int c = i < n ? counts[i] : 0;
        int s = c;
#pragma unroll
        for (int off = 1; off < 32; off <<= 1) {
            const int o = __shfl_up_sync(0xffffffffu, s, off);
            if (lane >= off) s += o;
        }
        if (lane == 31) warp_tot[wp] = s;
        __syncthreads();
        if (wp == 0) {
            int tsum = lane < (blockDim.x >> 5) ? warp_tot[lane] : 0;
#pragma unroll
            for (int off = 1; off < 32; off <<= 1) {
                const int o = __shfl_up_sync(0xffffffffu, tsum, off);
                if (lane >= off) tsum += o;
            }
            warp_tot[lane] = tsum;  // inclusive over warps
        }
        __syncthreads();
        const int before = carry + (wp ? warp_tot[wp - 1] : 0);
        if (i < n) {
            offsets[i] = before + s - c;
            cursor[i] = 0;
        }
        __syncthreads();
        if (threadIdx.x == blockDim.x - 1) carry = before + s;
        __syncthreads();
    }
    if (threadIdx.x == 0) offsets[n] = carry;
}

// ascending sort of one tile's list (bitonic in shared memory); longer lists
// are left unsorted and their tiles flagged for k_raster_all
__global__ void __launch_bounds__(256) k_tile_sort(const int* __restrict__ offsets, int* __restrict__ lists,
                                                   int* __restrict__ overflow, int ntiles, long long cap) {
    __shared__ int key[kSortCap];
    const int tile = blockIdx.x;
    const int b = offsets[tile], len = offsets[tile + 1] - b;
    if (offsets[ntiles] > cap) {
        if (threadIdx.x == 0) overflow[tile] = 1;
        return;
    }
    if (len <= 1) return;
    if (len > kSortCap) {
        if (threadIdx.x == 0) overflow[tile] = 1;
        return;
    }
    int p2 = 1;
    while (p2 < len) p2 <<= 1;
    for (int i = threadIdx.x; i < p2; i += blockDim.x) key[i] = i < len ? lists[b + i] : 0x7fffffff;
    __syncthreads();
    for (int k = 2; k <= p2; k <<= 1)
        for (int j = k >> 1; j > 0; j >>= 1) {
            for (int i = threadIdx.x; i < p2; i += blockDim.x) {
                const int ixj = i ^ j;
                if (ixj > i) {
                    const bool up = (i & k) == 0;
                    const int a = key[i], c = key[ixj];
                    if ((a > c) == up) {
                        key[i] = c;
                        key[ixj] = a;
                    }
                }
            }
            __syncthreads();
        }
    for (int i = threadIdx.x; i < len; i += blockDim.x) lists[b + i] = key[i];
}

// the per-pixel body of render_virtual's inner loop (occlude.cpp:146-166)
__device__ __forceinline__ void shade(const TriSetup& s, int x, int y, float& depth, float (&rgb)[3]) {
    if (x < s.x0 || x > s.x1 || y < s.y0 || y > s.y1) return;
    const double py = y + 0.5, px = x + 0.5;
    const double l0 = ((s.ub - px) * (s.vc - py) - (s.uc - px) * (s.vb - py)) / s.area;
    const double l1 = ((s.uc - px) * (s.va - py) - (s.ua - px) * (s.vc - py)) / s.area;
    const double l2 = 1.0 - l0 - l1;
    if (l0 < 0.0 || l1 < 0.0 || l2 < 0.0) return;
    const double inv_z = l0 * s.inv_za + l1 * s.inv_zb + l2 * s.inv_zc;
    const double z = 1.0 / inv_z;
    const float prev = depth;
    if (isfinite(prev) && prev <= z) return;  // FloatMap::is_valid(prev) && prev <= z
    depth = static_cast<float>(z);
#pragma unroll
    for (int ch = 0; ch < 3; ++ch) {
        const double num = l0 * s.ca[ch] * s.inv_za + l1 * s.cb[ch] * s.inv_zb + l2 * s.cc[ch] * s.inv_zc;
        rgb[ch] = static_cast<float>(num * z);
    }
}

// one block per 16x16 tile: the tile's sorted list, staged through shared
// memory in batches
__global__ void __launch_bounds__(kTile* kTile) k_raster(const TriSetup* __restrict__ ts, int nt,
                                                         const int* __restrict__ offsets, const int* __restrict__ lists,
                                                         const int* __restrict__ overflow, int w, int h, int tiles_x,
                                                         float* __restrict__ rgb_out, float* __restrict__ depth_out) {
    constexpr int kBatch = 64;
    __shared__ TriSetup st[kBatch];
    const int tile = blockIdx.x;
    const int x = (tile % tiles_x) * kTile + (threadIdx.x & (kTile - 1));
    const int y = (tile / tiles_x) * kTile + (threadIdx.x / kTile);
    float depth = __int_as_float(0x7fc00000);  // nodata
    float rgb[3] = {0.0f, 0.0f, 0.0f};
    if (overflow[tile]) {
        // list too long for the sort (or lists did not fit): every triangle of
        // the mesh in index order, bounding-box culled -- exact, slower
        for (int t = 0; t < nt; ++t) shade(ts[t], x, y, depth, rgb);
    } else {
        const int b = offsets[tile], e = offsets[tile + 1];
        for (int k0 = b; k0 < e; k0 += kBatch) {
            const int cnt = min(kBatch, e - k0);
            __syncthreads();
            for (int i = threadIdx.x; i < cnt; i += blockDim.x) st[i] = ts[lists[k0 + i]];
            __syncthreads();
            for (int i = 0; i < cnt; ++i) shade(st[i], x, y, depth, rgb);
        }
    }
    if (x < w && y < h) {
        const size_t p = static_cast<size_t>(y) * w + x;
        depth_out[p] = depth;
        rgb_out[3 * p + 0] = rgb[0];
        rgb_out[3 * p + 1] = rgb[1];
        rgb_out[3 * p + 2] = rgb[2];
    }
}

}  // namespace

// ===================================================================== host =

// pose: 16 doubles, row-major, HOST memory (passed by value to the kernel)
void transform_mesh(dco_ctx* ctx, const float* verts, int nv, const double* pose, float* out) {
    if (nv <= 0) return;
    Pose16 ps;
    for (int i = 0; i < 16; ++i) ps.p[i] = pose[i];
    k_transform_mesh<<<blocks_for(static_cast<size_t>(nv), 128), 128, 0, ctx->stream>>>(verts, nv, ps, out);
    launched(ctx, "k_transform_mesh");
}

// render_virtual (occlude.cpp:107-169) into caller buffers: rgb (w*h*3 float,
// 0 where nothing covers) and depth (w*h float, NaN where nothing covers).
void render_virtual(dco_ctx* ctx, const float* verts, const int* tris, const float* colors, int nt, double focal_px,
                    double cx, double cy, int w, int h, float* rgb, float* depth) {
    require(w >= 1 && h >= 1, "render_virtual: output dimensions must be positive");
    const int tiles_x = (w + kTile - 1) / kTile, tiles_y = (h + kTile - 1) / kTile;
    const int ntiles = tiles_x * tiles_y;
    // scratch: setups, counts | offsets (n+1) | cursor | overflow, then the lists
    const size_t setup_bytes = static_cast<size_t>(std::max(nt, 1)) * sizeof(TriSetup);
    char* base = static_cast<char*>(scratch(ctx, S_RENDER, setup_bytes + (4 * static_cast<size_t>(ntiles) + 1) * 4));
    TriSetup* ts = reinterpret_cast<TriSetup*>(base);
    int* counts = reinterpret_cast<int*>(base + setup_bytes);
    int* offsets = counts + ntiles;
    int* cursor = offsets + ntiles + 1;
    int* overflow = cursor + ntiles;
    cuda_check(cudaMemsetAsync(counts, 0, static_cast<size_t>(ntiles) * 4, ctx->stream), "memset");
    cuda_check(cudaMemsetAsync(overflow, 0, static_cast<size_t>(ntiles) * 4, ctx->stream), "memset");
    if (nt > 0) {
        k_tri_setup<<<blocks_for(static_cast<size_t>(nt), 128), 128, 0, ctx->stream>>>(
            verts, tris, colors, nt, focal_px, cx, cy, w, h, ts);
        launched(ctx, "k_tri_setup");
        k_tri_tiles<<<blocks_for(static_cast<size_t>(nt) * 32, 256), 256, 0, ctx->stream>>>(
            ts, nt, tiles_x, counts, nullptr, nullptr, nullptr, ntiles, 0);
        launched(ctx, "k_tri_tiles");
    }
    k_tile_scan<<<1, 1024, 0, ctx->stream>>>(counts, ntiles, offsets, cursor);
    launched(ctx, "k_tile_scan");
    // list storage without a host round trip: room for every (triangle, tile)
    // pair of small meshes, 256 tiles per triangle of larger ones; a frame that
    // needs more sends every tile down the whole-mesh path (still exact)
    const long long cap = std::min<long long>(static_cast<long long>(nt) * ntiles,
                                              std::max<long long>(256LL * nt, 1 << 20));
    int* lists = static_cast<int*>(scratch(ctx, S_RENDER_LIST, static_cast<size_t>(std::max<long long>(cap, 1)) * 4));
    if (nt > 0) {
        k_tri_tiles<<<blocks_for(static_cast<size_t>(nt) * 32, 256), 256, 0, ctx->stream>>>(
            ts, nt, tiles_x, nullptr, offsets, cursor, lists, ntiles, cap);
        launched(ctx, "k_tri_tiles");
        k_tile_sort<<<ntiles, 256, 0, ctx->stream>>>(offsets, lists, overflow, ntiles, cap);
        launched(ctx, "k_tile_sort");
    }
    k_raster<<<ntiles, kTile * kTile, 0, ctx->stream>>>(ts, nt, offsets, lists, overflow, w, h, tiles_x, rgb, depth);
    launched(ctx, "k_raster");
}

}  // namespace dco_gpu

using namespace dco_gpu;

extern "C" {

int dco_transform_mesh(dco_ctx* ctx, const float* vertices, int num_vertices, const double* pose, float* out) {
    return guarded(ctx, [&] {
        require(num_vertices >= 0, "transform_mesh: negative vertex count");
        require(pose != nullptr, "transform_mesh: pose is required");
        transform_mesh(ctx, vertices, num_vertices, pose, out);
    });
}

int dco_render_virtual(dco_ctx* ctx, const float* vertices, const int* triangles, const float* colors,
                       int num_triangles, double focal_px, double cx, double cy, int width, int height,
                       float* rgb, float* depth) {
    return guarded(ctx, [&] {
        require(num_triangles >= 0, "render_virtual: negative triangle count");
        render_virtual(ctx, vertices, triangles, colors, num_triangles, focal_px, cx, cy, width, height, rgb, depth);
    });
}

}  // extern "C"
