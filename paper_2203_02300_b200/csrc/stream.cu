// stream.cu — composite (reference src/occlude.cpp:171-194) and the
// device-resident frame orchestrator that replaces run_pipeline's per-frame
// body (src/pipeline.cpp:136-258) for one stream: the 3-frame keyframe window
// (flow.cpp:10-18), the previous-dense chain (pipeline.cpp:133,235) and the
// Unsolvable fallback (pipeline.cpp:236-242) all stay on the GPU, so a frame
// is a fixed sequence of kernel launches with no host round trip unless the
// caller asks for the frame statistics.
#include <string.h>

#include <algorithm>

#include "common.cuh"

namespace dco_gpu {

// forward declarations (stereo.cu, flow.cu, contour.cu, densify.cu)
void ingest_gray8(dco_ctx* ctx, const uint8_t* g8, int w, int h, float* full, float* quarter);
void downsample_half(dco_ctx* ctx, const float* img, int w, int h, float* out);
void build_cross_windows(dco_ctx* ctx, const float* img, int w, int h, const dco_config* cfg, uint8_t* l,
                         uint8_t* r, uint8_t* u, uint8_t* d);
void compute_cost_volume(dco_ctx* ctx, const float* left, const float* right, int w, int h, const uint8_t* l,
                         const uint8_t* r, const uint8_t* u, const uint8_t* d, const dco_config* cfg,
                         float* cost);
void aggregate_costs(dco_ctx* ctx, const float* cost, int w, int h, int nd, const uint8_t* l, const uint8_t* r,
                     const uint8_t* u, const uint8_t* d, int max_arm, float* out);
void select_disparity_wta(dco_ctx* ctx, const float* cost, int w, int h, int d_min, int nd, float* disp);
// render.cu
void transform_mesh(dco_ctx* ctx, const float* verts, int nv, const double* pose, float* out);
void render_virtual(dco_ctx* ctx, const float* verts, const int* tris, const float* colors, int nt, double focal_px,
                    double cx, double cy, int w, int h, float* rgb, float* depth);
// slice-major stereo core of the frame loop (stereo_slices.cu)
bool stereo_slices_supported(int max_arm, int qh);
void cost_volume_slices(dco_ctx* ctx, const float* left, const float* right, int w, int h, const uint8_t* l,
                        const uint8_t* r, const uint8_t* u, const uint8_t* d, const dco_config* cfg, int max_arm,
                        float* cost, int* rect);
void aggregate_slices(dco_ctx* ctx, const float* cost, int w, int h, int nd, const uint8_t* l, const uint8_t* r,
                      const uint8_t* u, const uint8_t* d, int max_arm, const int* rect, float* agg);
void wta_slices(dco_ctx* ctx, const float* agg, int w, int h, int d_min, int nd, float* disp);
void refine_disparity_histogram(dco_ctx* ctx, const float* disp, int w, int h, const uint8_t* l,
                                const uint8_t* r, const uint8_t* u, const uint8_t* d, int iters, int bin_bound,
                                int max_arm, float* out);
void flip_horizontal(dco_ctx* ctx, const float* img, int w, int h, float* out);
void lr_consistency(dco_ctx* ctx, const float* dl, const float* dr, int w, int h, double max_diff, float* out);
void disparity_to_sparse_depth(dco_ctx* ctx, const float* disp, int w, int h, const dco_config* cfg, int fw,
                               int fh, float* out);
void compute_flow_multi(dco_ctx* ctx, const float* from, const float* const* to, int dirs, int w, int h,
                        float* const* u_out, float* const* v_out);
void amplitude_fuse(dco_ctx* ctx, const float* pu, const float* pv, const float* fu, const float* fv, int w,
                    int h, double k, float* out);
void box_filter(dco_ctx* ctx, const float* a, int w, int h, int radius, float* out);
void normalize_amplitude(dco_ctx* ctx, const float* a, int w, int h, float* out);
void gaussian_blur(dco_ctx* ctx, const float* img, int w, int h, double sigma, float* out);
void extract_depth_contours_prefiltered(dco_ctx* ctx, const float* blurred, int w, int h, const float* mf,
                                        int qw, int qh, const dco_config* cfg, uint8_t* edges, float* m_i);
void assemble_system_dev(dco_ctx* ctx, const float* sparse, const uint8_t* edges, const float* mf, int qw,
                         int qh, const float* mi, const float* pre, const int* pre_valid, int w, int h,
                         const dco_config* cfg, const dco_system* sys, double* const_dev,
                         unsigned long long* anchors_dev);
void solve_dense_dev(dco_ctx* ctx, const dco_system* sys, const dco_config* cfg,
                     const unsigned long long* anchors_dev, const double* const_dev, float* dense,
                     const float* fallback, const int* fallback_valid, double* hist, int hist_cap,
                     void* out_dev);
size_t solve_out_bytes();
void read_solve_out(const void* host, int* status, int* iters, double* relres, double* obj0, double* obj1);

namespace {

// composite, occlude.cpp:171-194.
// 128-bit variant (n % 4 == 0, 16-byte aligned buffers): 4 pixels per thread,
// the RGB planes as three float4, depths as float4, the mask as one u32.
__global__ void k_composite_v4(const float* __restrict__ real, const float* __restrict__ dense,
                               const float* __restrict__ vrgb, const float* __restrict__ vdepth, size_t n4,
                               float* __restrict__ out, uint8_t* __restrict__ mask) {
    const size_t i = static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= n4) return;
    bool take[4] = {false, false, false, false};
    if (vdepth) {
        const float4 vz = reinterpret_cast<const float4*>(vdepth)[i];
        const float4 rz = reinterpret_cast<const float4*>(dense)[i];
        const float v[4] = {vz.x, vz.y, vz.z, vz.w}, r[4] = {rz.x, rz.y, rz.z, rz.w};
#pragma unroll
        for (int j = 0; j < 4; ++j) take[j] = isfinite(v[j]) && !(isfinite(r[j]) && v[j] > r[j]);
    }
    float rc[12], vc[12];
    const float4* R = reinterpret_cast<const float4*>(real) + 3 * i;
    const float4 a = R[0], b = R[1], c = R[2];
    rc[0] = a.x; rc[1] = a.y; rc[2] = a.z; rc[3] = a.w; rc[4] = b.x; rc[5] = b.y;
    rc[6] = b.z; rc[7] = b.w; rc[8] = c.x; rc[9] = c.y; rc[10] = c.z; rc[11] = c.w;
    if (take[0] | take[1] | take[2] | take[3]) {
        const float4* V = reinterpret_cast<const float4*>(vrgb) + 3 * i;
        const float4 d = V[0], e = V[1], f = V[2];
        vc[0] = d.x; vc[1] = d.y; vc[2] = d.z; vc[3] = d.w; vc[4] = e.x; vc[5] = e.y;
        vc[6] = e.z; vc[7] = e.w; vc[8] = f.x; vc[9] = f.y; vc[10] = f.z; vc[11] = f.w;
#pragma unroll
        for (int j = 0; j < 12; ++j) rc[j] = take[j / 3] ? vc[j] : rc[j];
    }
    float4* O = reinterpret_cast<float4*>(out) + 3 * i;
    O[0] = make_float4(rc[0], rc[1], rc[2], rc[3]);
    O[1] = make_float4(rc[4], rc[5], rc[6], rc[7]);
    O[2] = make_float4(rc[8], rc[9], rc[10], rc[11]);
    reinterpret_cast<uint32_t*>(mask)[i] = (take[0] ? 1u : 0u) | (take[1] ? 1u << 8 : 0u) | (take[2] ? 1u << 16 : 0u) |
                                           (take[3] ? 1u << 24 : 0u);
}

__global__ void k_composite(const float* __restrict__ real, const float* __restrict__ dense,
                            const float* __restrict__ vrgb, const float* __restrict__ vdepth, size_t n,
                            float* __restrict__ out, uint8_t* __restrict__ mask) {
    size_t i = static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= n) return;
    bool take = false;
    if (vdepth) {
        float vz = vdepth[i];
        if (isfinite(vz)) {
            float rz = dense[i];
            take = !(isfinite(rz) && vz > rz);
        }
    }
    const float* src = take ? vrgb : real;
    out[3 * i] = src[3 * i];
    out[3 * i + 1] = src[3 * i + 1];
    out[3 * i + 2] = src[3 * i + 2];
    mask[i] = take ? 1 : 0;
}

// to_color (image.cpp:17-25) of the u8 gray frame, or rgb8 / 255.0f.
__global__ void k_rgb_from_u8(const uint8_t* __restrict__ gray8, const uint8_t* __restrict__ rgb8, size_t n,
                              float* __restrict__ rgb) {
    size_t i = static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= n) return;
    if (rgb8) {
        rgb[3 * i] = rgb8[3 * i] / 255.0f;
        rgb[3 * i + 1] = rgb8[3 * i + 1] / 255.0f;
        rgb[3 * i + 2] = rgb8[3 * i + 2] / 255.0f;
    } else {
        float g = gray8[i] / 255.0f;
        rgb[3 * i] = g;
        rgb[3 * i + 1] = g;
        rgb[3 * i + 2] = g;
    }
}

__global__ void k_rgb_from_f32(const float* __restrict__ gray, const float* __restrict__ rgb_in, size_t n,
                               float* __restrict__ rgb) {
    size_t i = static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= n) return;
    if (rgb_in) {
        rgb[3 * i] = rgb_in[3 * i];
        rgb[3 * i + 1] = rgb_in[3 * i + 1];
        rgb[3 * i + 2] = rgb_in[3 * i + 2];
    } else {
        float g = gray[i];
        rgb[3 * i] = g;
        rgb[3 * i + 1] = g;
        rgb[3 * i + 2] = g;
    }
}

// previous_dense = dense when the solve succeeded (pipeline.cpp:235).
// The frame's outputs in run_pipeline's file encodings (pipeline.cpp:266-267):
// the composite as write_ppm's bytes (quantize, codec.cpp:23-26, 221-229) and
// the mask as write_mask_pgm's (0 / 255, codec.cpp:243-247). Thread per pixel.
__global__ void k_encode_frame(const float* __restrict__ comp, const uint8_t* __restrict__ mask, size_t n,
                               uint8_t* __restrict__ rgb8, uint8_t* __restrict__ mask8) {
    const size_t i = static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= n) return;
#pragma unroll
    for (int c = 0; c < 3; ++c) {
        float v = comp[3 * i + c];
        v = v < 0.0f ? 0.0f : (1.0f < v ? 1.0f : v);  // std::clamp: NaN passes through
        rgb8[3 * i + c] = isnan(v) ? 0 : static_cast<uint8_t>(lroundf(v * 255.0f));
    }
    mask8[i] = mask[i] ? 255 : 0;
}

__global__ void k_keep_dense(const float* __restrict__ dense, size_t n, const int* __restrict__ status,
                             float* __restrict__ prev, int* __restrict__ prev_valid) {
    if (*status != 0) return;
    size_t i = static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i < n) prev[i] = dense[i];
    if (i == 0) *prev_valid = 1;
}

}  // namespace

void composite(dco_ctx* ctx, const float* real, const float* dense, const float* vrgb, const float* vdepth,
               int w, int h, float* out, uint8_t* mask) {
    size_t n = static_cast<size_t>(w) * h;
    auto al = [](const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; };
    if (n % 4 == 0 && al(real) && al(dense) && al(out) && (!vrgb || al(vrgb)) && (!vdepth || al(vdepth)) &&
        (reinterpret_cast<uintptr_t>(mask) & 3) == 0) {
        k_composite_v4<<<blocks_for(n / 4, 256), 256, 0, ctx->stream>>>(real, dense, vrgb, vdepth, n / 4, out, mask);
    } else {
        k_composite<<<blocks_for(n, 256), 256, 0, ctx->stream>>>(real, dense, vrgb, vdepth, n, out, mask);
    }
    launched(ctx, "k_composite");
}

}  // namespace dco_gpu

using namespace dco_gpu;

struct dco_stream {
    dco_ctx* ctx = nullptr;
    dco_config cfg;
    int fw = 0, fh = 0, qw = 0, qh = 0, nd = 0;
    uint64_t pushed = 0;
    std::vector<void*> allocs;
    // window slots (3): quarter left/right, full gray, full rgb
    float* left_q[3];
    float* right_q[3];
    float* gray[3];
    float* rgb[3];
    // opt-in left-right check (not in the reference): mirrored pair, right view, checked map
    bool lr = false;
    double lr_max = 1.0;
    float* lr_buf = nullptr;  // 4 quarter planes
    // per-frame products
    uint8_t* arms;  // 4 planes
    float* cost;
    float* agg;
    float* disp_wta;
    float* disparity;
    float* sparse;
    float* flow;  // pu, pv, fu, fv
    float* fused;
    float* boxed;
    float* m_fuse;
    float* blurred;
    float* m_i;
    uint8_t* edges;
    dco_system sys;
    double* const_dev;
    unsigned long long* anchors_dev;
    void* solve_out;
    float* dense;
    float* prev;
    int* prev_valid;
    float* comp;
    uint8_t* mask;
    float* vrgb = nullptr;
    float* vdepth = nullptr;
    bool has_virtual = false;
    // virtual mesh rendered per frame (occlude.cpp:107-169, pipeline.cpp:247-252)
    float* mesh_v = nullptr;  // device copies
    int* mesh_t = nullptr;
    float* mesh_c = nullptr;
    float* mesh_posed = nullptr;
    int mesh_nv = 0, mesh_nt = 0;
    bool has_mesh = false;
    double pose[3][16] = {};  // per window slot: the frame's manifest pose
    bool pose_set[3] = {};
    double next_pose[16] = {};
    bool next_pose_set = false;
    void* host_out = nullptr;
    uint8_t* enc = nullptr;  // encoded outputs (4 bytes per pixel), allocated on first use
    // optional per-span CUDA-event timing (StageTimings, pipeline.hpp:27-46)
    // A ring of kRing event sets so the host never waits on the frame it just
    // enqueued: set i is harvested when it is about to be reused (or flushed).
    static constexpr int kRing = 4;
    bool timing = false;
    cudaEvent_t ev[kRing][DCO_SPAN_COUNT + 1] = {};
    bool pending[kRing] = {};
    int cur_set = 0;
    double span_ms[DCO_SPAN_COUNT] = {};
    uint64_t timed_frames = 0;
    void mark(int k) {
        if (timing) cuda_check(cudaEventRecord(ev[cur_set][k], ctx->stream), "event record");
    }
    void harvest(int set) {
        if (!pending[set]) return;
        cuda_check(cudaEventSynchronize(ev[set][DCO_SPAN_COUNT]), "event sync");
        for (int k = 0; k < DCO_SPAN_COUNT; ++k) {
            float ms = 0.0f;
            cuda_check(cudaEventElapsedTime(&ms, ev[set][k], ev[set][k + 1]), "elapsed");
            span_ms[k] += ms;
        }
        ++timed_frames;
        pending[set] = false;
    }
    void take_pose(int slot) {  // the pose set for this push (pipeline.cpp:249: the record's pose)
        pose_set[slot] = next_pose_set;
        for (int i = 0; i < 16; ++i) pose[slot][i] = next_pose[i];
        next_pose_set = false;
    }
    void begin_frame() {  // before the frame's first kernel
        if (!timing) return;
        cur_set = (cur_set + 1) % kRing;
        harvest(cur_set);
        mark(0);
    }

    template <typename T>
    T* alloc(size_t count) {
        void* p = nullptr;
        cuda_check(cudaMalloc(&p, count * sizeof(T) + 256), "cudaMalloc(stream)");
        allocs.push_back(p);
        return static_cast<T*>(p);
    }
};

namespace {

// The stereo chain of the current branch (slice-major or packed exact) on an
// arbitrary quarter pair into out (the right view of the opt-in LR check).
void stereo_chain(dco_stream* s, const float* lq, const float* rq, float* out) {
    dco_ctx* ctx = s->ctx;
    const dco_config* cfg = &s->cfg;
    const int qw = s->qw, qh = s->qh;
    const size_t nq = static_cast<size_t>(qw) * qh;
    uint8_t *L = s->arms, *R = L + nq, *U = R + nq, *D = U + nq;
    build_cross_windows(ctx, lq, qw, qh, cfg, L, R, U, D);
    if (stereo_slices_supported(cfg->cross_arm_l1, s->qh)) {
        int* rect = static_cast<int*>(scratch(ctx, S_FLAG_SLICE, 2 * static_cast<size_t>(s->nd) * sizeof(int)));
        cost_volume_slices(ctx, lq, rq, qw, qh, L, R, U, D, cfg, cfg->cross_arm_l1, s->cost, rect);
        aggregate_slices(ctx, s->cost, qw, qh, s->nd, L, R, U, D, cfg->cross_arm_l1, rect, s->agg);
        wta_slices(ctx, s->agg, qw, qh, cfg->d_min, s->nd, s->disp_wta);
    } else {
        compute_cost_volume(ctx, lq, rq, qw, qh, L, R, U, D, cfg, s->cost);
        aggregate_costs(ctx, s->cost, qw, qh, s->nd, L, R, U, D, cfg->cross_arm_l1, s->agg);
        select_disparity_wta(ctx, s->agg, qw, qh, cfg->d_min, s->nd, s->disp_wta);
    }
    refine_disparity_histogram(ctx, s->disp_wta, qw, qh, L, R, U, D, cfg->hist_iterations, cfg->d_max,
                               cfg->cross_arm_l1, out);
}

void run_frame(dco_stream* s, dco_frame_result* res) {
    dco_ctx* ctx = s->ctx;
    const dco_config* cfg = &s->cfg;
    const int fw = s->fw, fh = s->fh, qw = s->qw, qh = s->qh;
    const size_t nq = static_cast<size_t>(qw) * qh, nf = static_cast<size_t>(fw) * fh;
    s->mark(DCO_SPAN_INGEST + 1);
    const uint64_t k = s->pushed;  // frames pushed so far (>= 3)
    const int past = static_cast<int>((k - 3) % 3), mid = static_cast<int>((k - 2) % 3),
              fut = static_cast<int>((k - 1) % 3);
    uint8_t* L = s->arms;
    uint8_t* R = L + nq;
    uint8_t* U = R + nq;
    uint8_t* D = U + nq;
    // --- stereo on the middle pair (pipeline.cpp:184-195)
    build_cross_windows(ctx, s->left_q[mid], qw, qh, cfg, L, R, U, D);
    s->mark(DCO_SPAN_CROSS + 1);
    if (stereo_slices_supported(cfg->cross_arm_l1, s->qh)) {
        // slice-major cost volume + exact fixed-point aggregation (stereo_slices.cu)
        int* rect = static_cast<int*>(scratch(ctx, S_FLAG_SLICE, 2 * static_cast<size_t>(s->nd) * sizeof(int)));
        cost_volume_slices(ctx, s->left_q[mid], s->right_q[mid], qw, qh, L, R, U, D, cfg, cfg->cross_arm_l1, s->cost,
                           rect);
        s->mark(DCO_SPAN_COST + 1);
        aggregate_slices(ctx, s->cost, qw, qh, s->nd, L, R, U, D, cfg->cross_arm_l1, rect, s->agg);
        s->mark(DCO_SPAN_AGGREGATE + 1);
        wta_slices(ctx, s->agg, qw, qh, cfg->d_min, s->nd, s->disp_wta);
    } else {
        compute_cost_volume(ctx, s->left_q[mid], s->right_q[mid], qw, qh, L, R, U, D, cfg, s->cost);
        s->mark(DCO_SPAN_COST + 1);
        aggregate_costs(ctx, s->cost, qw, qh, s->nd, L, R, U, D, cfg->cross_arm_l1, s->agg);
        s->mark(DCO_SPAN_AGGREGATE + 1);
        select_disparity_wta(ctx, s->agg, qw, qh, cfg->d_min, s->nd, s->disp_wta);
    }
    s->mark(DCO_SPAN_WTA + 1);
    refine_disparity_histogram(ctx, s->disp_wta, qw, qh, L, R, U, D, cfg->hist_iterations, cfg->d_max,
                               cfg->cross_arm_l1, s->disparity);
    if (s->lr) {  // opt-in: right view on the mirrored pair, then the check (counted in the refine span)
        float* fl = s->lr_buf;
        float* fr = fl + nq;
        float* dm = fr + nq;
        float* dr = dm + nq;
        flip_horizontal(ctx, s->right_q[mid], qw, qh, fl);
        flip_horizontal(ctx, s->left_q[mid], qw, qh, fr);
        stereo_chain(s, fl, fr, dm);
        flip_horizontal(ctx, dm, qw, qh, dr);
        lr_consistency(ctx, s->disparity, dr, qw, qh, s->lr_max, dm);
        cuda_check(cudaMemcpyAsync(s->disparity, dm, nq * 4, cudaMemcpyDeviceToDevice, ctx->stream), "lr copy");
    }
    s->mark(DCO_SPAN_REFINE + 1);
    disparity_to_sparse_depth(ctx, s->disparity, qw, qh, cfg, fw, fh, s->sparse);
    s->mark(DCO_SPAN_SPARSE + 1);
    // --- bidirectional flow around the middle frame (pipeline.cpp:199-202)
    const float* tos[2] = {s->left_q[past], s->left_q[fut]};
    float* us[2] = {s->flow, s->flow + 2 * nq};
    float* vs[2] = {s->flow + nq, s->flow + 3 * nq};
    compute_flow_multi(ctx, s->left_q[mid], tos, 2, qw, qh, us, vs);
    s->mark(DCO_SPAN_FLOW + 1);
    // --- amplitude + fusion + box + normalisation (pipeline.cpp:204-215);
    // amplitude is computed inside the fusion kernel (never materialised)
    amplitude_fuse(ctx, us[0], vs[0], us[1], vs[1], qw, qh, cfg->confidence_offset_k, s->fused);
    s->mark(DCO_SPAN_FUSION + 1);
    box_filter(ctx, s->fused, qw, qh, cfg->box_radius, s->boxed);
    s->mark(DCO_SPAN_BOX + 1);
    normalize_amplitude(ctx, s->boxed, qw, qh, s->m_fuse);
    s->mark(DCO_SPAN_NORMALIZE + 1);
    // --- contours at full resolution (pipeline.cpp:218-222)
    gaussian_blur(ctx, s->gray[mid], fw, fh, cfg->gauss_sigma, s->blurred);
    s->mark(DCO_SPAN_BLUR + 1);
    extract_depth_contours_prefiltered(ctx, s->blurred, fw, fh, s->m_fuse, qw, qh, cfg, s->edges, s->m_i);
    s->mark(DCO_SPAN_CONTOUR + 1);
    // --- densification seeded with the previous dense map (pipeline.cpp:225-243)
    assemble_system_dev(ctx, s->sparse, s->edges, s->m_fuse, qw, qh, s->m_i, s->prev, s->prev_valid, fw, fh,
                        cfg, &s->sys, s->const_dev, s->anchors_dev);
    s->mark(DCO_SPAN_ASSEMBLE + 1);
    solve_dense_dev(ctx, &s->sys, cfg, s->anchors_dev, s->const_dev, s->dense, s->prev, s->prev_valid,
                    nullptr, 0, s->solve_out);
    k_keep_dense<<<blocks_for(nf, 256), 256, 0, ctx->stream>>>(s->dense, nf, static_cast<const int*>(s->solve_out),
                                                               s->prev, s->prev_valid);
    launched(ctx, "k_keep_dense");
    s->mark(DCO_SPAN_SOLVE + 1);
    // --- composite (pipeline.cpp:247-258)
    if (s->has_mesh) {
        // render_virtual of the (posed) mesh for the middle frame (pipeline.cpp:249-252)
        const float* verts = s->mesh_v;
        if (s->pose_set[mid]) {
            transform_mesh(ctx, s->mesh_v, s->mesh_nv, s->pose[mid], s->mesh_posed);
            verts = s->mesh_posed;
        }
        render_virtual(ctx, verts, s->mesh_t, s->mesh_c, s->mesh_nt, cfg->focal_px, fw / 2.0, fh / 2.0, fw, fh,
                       s->vrgb, s->vdepth);
    }
    const bool layer = s->has_mesh || s->has_virtual;
    composite(ctx, s->rgb[mid], s->dense, layer ? s->vrgb : nullptr, layer ? s->vdepth : nullptr, fw, fh, s->comp,
              s->mask);
    s->mark(DCO_SPAN_COMPOSITE + 1);
    if (s->timing) s->pending[s->cur_set] = true;
    if (res) {
        void* hp = pinned_host(ctx, 256);
        cuda_check(cudaMemcpyAsync(hp, s->solve_out, solve_out_bytes(), cudaMemcpyDeviceToHost, ctx->stream),
                   "d2h");
        cuda_check(cudaStreamSynchronize(ctx->stream), "sync");
        int status, iters;
        double rr, o0, o1;
        read_solve_out(hp, &status, &iters, &rr, &o0, &o1);
        res->composited = 1;
        res->densify_skipped = status != 0;
        res->densify_iterations = status ? 0 : iters;
        res->densify_objective = status ? 0.0 : o1;
        res->relative_residual = status ? 0.0 : rr;
    }
}

void finish_push(dco_stream* s, dco_frame_result* res) {
    ++s->pushed;
    if (s->pushed < 3) {
        if (res) memset(res, 0, sizeof(*res));
        return;
    }
    run_frame(s, res);
}

}  // namespace

extern "C" {

int dco_stream_create(dco_ctx* ctx, int fw, int fh, const dco_config* cfg, dco_stream** out) {
    return guarded(ctx, [&] {
        validate_config(cfg);
        require(fw >= 32 && fh >= 32, "stream: frames must be at least 32x32");
        dco_stream* s = new dco_stream();
        try {
            s->ctx = ctx;
            s->cfg = *cfg;
            s->fw = fw;
            s->fh = fh;
            s->qw = fw / 2;
            s->qh = fh / 2;
            s->nd = cfg->d_max - cfg->d_min + 1;
            const size_t nq = static_cast<size_t>(s->qw) * s->qh, nf = static_cast<size_t>(fw) * fh;
            for (int i = 0; i < 3; ++i) {
                s->left_q[i] = s->alloc<float>(nq);
                s->right_q[i] = s->alloc<float>(nq);
                s->gray[i] = s->alloc<float>(nf);
                s->rgb[i] = s->alloc<float>(3 * nf);
            }
            s->arms = s->alloc<uint8_t>(4 * nq);
            s->cost = s->alloc<float>(nq * s->nd);
            s->agg = s->alloc<float>(nq * s->nd);
            s->disp_wta = s->alloc<float>(nq);
            s->disparity = s->alloc<float>(nq);
            s->sparse = s->alloc<float>(nf);
            s->flow = s->alloc<float>(4 * nq);
            s->fused = s->alloc<float>(nq);
            s->boxed = s->alloc<float>(nq);
            s->m_fuse = s->alloc<float>(nq);
            s->blurred = s->alloc<float>(nf);
            s->m_i = s->alloc<float>(nf);
            s->edges = s->alloc<uint8_t>(nf);
            s->sys.width = fw;
            s->sys.height = fh;
            s->sys.diag = s->alloc<double>(nf);
            s->sys.coup_h = s->alloc<double>(nf);
            s->sys.coup_v = s->alloc<double>(nf);
            s->sys.rhs = s->alloc<double>(nf);
            s->sys.initial = s->alloc<double>(nf);
            s->sys.anchored = s->alloc<uint8_t>(nf);
            s->sys.constant_term = 0.0;
            s->sys.anchor_count = 0;
            s->const_dev = s->alloc<double>(1);
            s->anchors_dev = s->alloc<unsigned long long>(1);
            s->solve_out = s->alloc<char>(256);
            s->dense = s->alloc<float>(nf);
            s->prev = s->alloc<float>(nf);
            s->prev_valid = s->alloc<int>(1);
            s->comp = s->alloc<float>(3 * nf);
            s->mask = s->alloc<uint8_t>(nf);
            cuda_check(cudaMemsetAsync(s->prev_valid, 0, sizeof(int), ctx->stream), "memset");
        } catch (...) {
            for (void* p : s->allocs) cudaFree(p);
            delete s;
            throw;
        }
        *out = s;
    });
}

void dco_stream_destroy(dco_stream* s) {
    if (!s) return;
    cudaStreamSynchronize(s->ctx->stream);
    for (auto& set : s->ev)
        for (auto& e : set)
            if (e) cudaEventDestroy(e);
    for (void* p : s->allocs) cudaFree(p);
    if (s->host_out) cudaFreeHost(s->host_out);
    delete s;
}

int dco_stream_set_virtual(dco_stream* s, const float* vrgb, const float* vdepth) {
    if (!s) return DCO_INPUT;
    return guarded(s->ctx, [&] {
        const size_t nf = static_cast<size_t>(s->fw) * s->fh;
        if (!vrgb || !vdepth) {
            s->has_virtual = false;
            return;
        }
        if (!s->vrgb) {
            s->vrgb = s->alloc<float>(3 * nf);
            s->vdepth = s->alloc<float>(nf);
        }
        cuda_check(cudaMemcpyAsync(s->vrgb, vrgb, 3 * nf * 4, cudaMemcpyDeviceToDevice, s->ctx->stream), "copy");
        cuda_check(cudaMemcpyAsync(s->vdepth, vdepth, nf * 4, cudaMemcpyDeviceToDevice, s->ctx->stream), "copy");
        s->has_virtual = true;
    });
}

int dco_stream_set_mesh(dco_stream* s, const float* vertices, int num_vertices, const int* triangles,
                        int num_triangles, const float* colors) {
    if (!s) return DCO_INPUT;
    return guarded(s->ctx, [&] {
        if (!vertices || !triangles || !colors || num_vertices <= 0) {
            s->has_mesh = false;
            return;
        }
        require(num_triangles >= 0, "set_mesh: negative triangle count");
        for (int t = 0; t < 3 * num_triangles; ++t)
            require(triangles[t] >= 0 && triangles[t] < num_vertices, "set_mesh: triangle index out of range");
        const size_t nf = static_cast<size_t>(s->fw) * s->fh;
        if (!s->vrgb) {
            s->vrgb = s->alloc<float>(3 * nf);
            s->vdepth = s->alloc<float>(nf);
        }
        if (num_vertices > s->mesh_nv || !s->mesh_v) {
            s->mesh_v = s->alloc<float>(3 * static_cast<size_t>(num_vertices));
            s->mesh_c = s->alloc<float>(3 * static_cast<size_t>(num_vertices));
            s->mesh_posed = s->alloc<float>(3 * static_cast<size_t>(num_vertices));
        }
        if (num_triangles > s->mesh_nt || !s->mesh_t)
            s->mesh_t = s->alloc<int>(3 * static_cast<size_t>(std::max(num_triangles, 1)));
        cuda_check(cudaMemcpy(s->mesh_v, vertices, 12 * static_cast<size_t>(num_vertices), cudaMemcpyHostToDevice),
                   "h2d");
        cuda_check(cudaMemcpy(s->mesh_c, colors, 12 * static_cast<size_t>(num_vertices), cudaMemcpyHostToDevice),
                   "h2d");
        if (num_triangles)
            cuda_check(cudaMemcpy(s->mesh_t, triangles, 12 * static_cast<size_t>(num_triangles),
                                  cudaMemcpyHostToDevice),
                       "h2d");
        s->mesh_nv = num_vertices;
        s->mesh_nt = num_triangles;
        s->has_mesh = true;
    });
}

int dco_stream_set_next_pose(dco_stream* s, const double* pose) {
    if (!s) return DCO_INPUT;
    s->next_pose_set = pose != nullptr;
    if (pose)
        for (int i = 0; i < 16; ++i) s->next_pose[i] = pose[i];
    return DCO_OK;
}

int dco_stream_push_gray8(dco_stream* s, const uint8_t* left8, const uint8_t* right8, const uint8_t* rgb8,
                          dco_frame_result* res) {
    if (!s) return DCO_INPUT;
    return guarded(s->ctx, [&] {
        dco_ctx* ctx = s->ctx;
        if (s->pushed + 1 >= 3) s->begin_frame();
        int slot = static_cast<int>(s->pushed % 3);
        s->take_pose(slot);
        ingest_gray8(ctx, left8, s->fw, s->fh, s->gray[slot], s->left_q[slot]);
        ingest_gray8(ctx, right8, s->fw, s->fh, nullptr, s->right_q[slot]);
        size_t nf = static_cast<size_t>(s->fw) * s->fh;
        k_rgb_from_u8<<<blocks_for(nf, 256), 256, 0, ctx->stream>>>(left8, rgb8, nf, s->rgb[slot]);
        launched(ctx, "k_rgb_from_u8");
        finish_push(s, res);
    });
}

int dco_run_streams(dco_stream* const* streams, int n, const uint8_t* const* left8, const uint8_t* const* right8,
                    int frames_per_stream, dco_frame_result* results) {
    if (!streams || n < 1 || !left8 || !right8 || frames_per_stream < 0) return DCO_INPUT;
    for (int k = 0; k < n; ++k)
        if (!streams[k] || !left8[k] || !right8[k]) return DCO_INPUT;
    // frame f of every stream, then f + 1: each stream's launches go to its own
    // context stream, so the streams' frames overlap on the device
    for (int f = 0; f < frames_per_stream; ++f) {
        for (int k = 0; k < n; ++k) {
            dco_stream* s = streams[k];
            const size_t nf = static_cast<size_t>(s->fw) * s->fh;
            dco_frame_result* r = results ? &results[static_cast<size_t>(k) * frames_per_stream + f] : nullptr;
            const int st = dco_stream_push_gray8(s, left8[k] + f * nf, right8[k] + f * nf, nullptr, r);
            if (st != DCO_OK) return st;
        }
    }
    return DCO_OK;
}

int dco_stream_push_f32(dco_stream* s, const float* left, const float* right, const float* rgb,
                        dco_frame_result* res) {
    if (!s) return DCO_INPUT;
    return guarded(s->ctx, [&] {
        dco_ctx* ctx = s->ctx;
        if (s->pushed + 1 >= 3) s->begin_frame();
        int slot = static_cast<int>(s->pushed % 3);
        s->take_pose(slot);
        size_t nf = static_cast<size_t>(s->fw) * s->fh;
        cuda_check(cudaMemcpyAsync(s->gray[slot], left, nf * 4, cudaMemcpyDeviceToDevice, ctx->stream), "copy");
        downsample_half(ctx, left, s->fw, s->fh, s->left_q[slot]);
        downsample_half(ctx, right, s->fw, s->fh, s->right_q[slot]);
        k_rgb_from_f32<<<blocks_for(nf, 256), 256, 0, ctx->stream>>>(left, rgb, nf, s->rgb[slot]);
        launched(ctx, "k_rgb_from_f32");
        finish_push(s, res);
    });
}

int dco_stream_push_gray8_host(dco_stream* s, const uint8_t* left8, const uint8_t* right8, float* comp_out,
                               uint8_t* mask_out, float* dense_out, dco_frame_result* res) {
    if (!s) return DCO_INPUT;
    return guarded(s->ctx, [&] {
        dco_ctx* ctx = s->ctx;
        size_t nf = static_cast<size_t>(s->fw) * s->fh;
        uint8_t* staging = static_cast<uint8_t*>(scratch(ctx, S_STAGE, 2 * nf));
        cuda_check(cudaMemcpyAsync(staging, left8, nf, cudaMemcpyHostToDevice, ctx->stream), "h2d");
        cuda_check(cudaMemcpyAsync(staging + nf, right8, nf, cudaMemcpyHostToDevice, ctx->stream), "h2d");
        if (s->pushed + 1 >= 3) s->begin_frame();
        int slot = static_cast<int>(s->pushed % 3);
        s->take_pose(slot);
        ingest_gray8(ctx, staging, s->fw, s->fh, s->gray[slot], s->left_q[slot]);
        ingest_gray8(ctx, staging + nf, s->fw, s->fh, nullptr, s->right_q[slot]);
        k_rgb_from_u8<<<blocks_for(nf, 256), 256, 0, ctx->stream>>>(staging, nullptr, nf, s->rgb[slot]);
        launched(ctx, "k_rgb_from_u8");
        finish_push(s, res);
        if (s->pushed >= 3) {
            if (comp_out)
                cuda_check(cudaMemcpyAsync(comp_out, s->comp, 3 * nf * 4, cudaMemcpyDeviceToHost, ctx->stream), "d2h");
            if (mask_out)
                cuda_check(cudaMemcpyAsync(mask_out, s->mask, nf, cudaMemcpyDeviceToHost, ctx->stream), "d2h");
            if (dense_out)
                cuda_check(cudaMemcpyAsync(dense_out, s->dense, nf * 4, cudaMemcpyDeviceToHost, ctx->stream), "d2h");
        }
        cuda_check(cudaStreamSynchronize(ctx->stream), "sync");
    });
}

int dco_stream_push_gray8_host_encoded(dco_stream* s, const uint8_t* left8, const uint8_t* right8,
                                       uint8_t* composite_rgb8, uint8_t* mask8, float* dense_out,
                                       dco_frame_result* res) {
    if (!s) return DCO_INPUT;
    return guarded(s->ctx, [&] {
        dco_ctx* ctx = s->ctx;
        size_t nf = static_cast<size_t>(s->fw) * s->fh;
        if (!s->enc) s->enc = s->alloc<uint8_t>(4 * nf);
        uint8_t* staging = static_cast<uint8_t*>(scratch(ctx, S_STAGE, 2 * nf));
        cuda_check(cudaMemcpyAsync(staging, left8, nf, cudaMemcpyHostToDevice, ctx->stream), "h2d");
        cuda_check(cudaMemcpyAsync(staging + nf, right8, nf, cudaMemcpyHostToDevice, ctx->stream), "h2d");
        if (s->pushed + 1 >= 3) s->begin_frame();
        int slot = static_cast<int>(s->pushed % 3);
        s->take_pose(slot);
        ingest_gray8(ctx, staging, s->fw, s->fh, s->gray[slot], s->left_q[slot]);
        ingest_gray8(ctx, staging + nf, s->fw, s->fh, nullptr, s->right_q[slot]);
        k_rgb_from_u8<<<blocks_for(nf, 256), 256, 0, ctx->stream>>>(staging, nullptr, nf, s->rgb[slot]);
        launched(ctx, "k_rgb_from_u8");
        finish_push(s, res);
        if (s->pushed >= 3) {
            if (composite_rgb8 || mask8) {
                k_encode_frame<<<blocks_for(nf, 256), 256, 0, ctx->stream>>>(s->comp, s->mask, nf, s->enc,
                                                                              s->enc + 3 * nf);
                launched(ctx, "k_encode_frame");
            }
            if (composite_rgb8)
                cuda_check(cudaMemcpyAsync(composite_rgb8, s->enc, 3 * nf, cudaMemcpyDeviceToHost, ctx->stream),
                           "d2h");
            if (mask8)
                cuda_check(cudaMemcpyAsync(mask8, s->enc + 3 * nf, nf, cudaMemcpyDeviceToHost, ctx->stream), "d2h");
            if (dense_out)
                cuda_check(cudaMemcpyAsync(dense_out, s->dense, nf * 4, cudaMemcpyDeviceToHost, ctx->stream), "d2h");
        }
        cuda_check(cudaStreamSynchronize(ctx->stream), "sync");
    });
}

int dco_stream_set_lr_check(dco_stream* s, int enable, double max_diff) {
    if (!s) return DCO_INPUT;
    return guarded(s->ctx, [&] {
        require(max_diff >= 0.0, "stream: negative left-right tolerance");
        if (enable && !s->lr_buf) s->lr_buf = s->alloc<float>(4 * static_cast<size_t>(s->qw) * s->qh);
        s->lr = enable != 0;
        s->lr_max = max_diff;
    });
}

int dco_stream_set_timing(dco_stream* s, int enable) {
    if (!s) return DCO_INPUT;
    return guarded(s->ctx, [&] {
        if (enable && !s->ev[0][0])
            for (auto& set : s->ev)
                for (auto& e : set) cuda_check(cudaEventCreate(&e), "event create");
        for (int i = 0; i < dco_stream::kRing; ++i) s->pending[i] = false;
        for (double& v : s->span_ms) v = 0.0;
        s->timed_frames = 0;
        s->timing = enable != 0;
    });
}

int dco_stream_span_times(dco_stream* s, double* ms, uint64_t* frames) {
    if (!s) return DCO_INPUT;
    return guarded(s->ctx, [&] {
        for (int i = 0; i < dco_stream::kRing; ++i) s->harvest(i);
        for (int k = 0; k < DCO_SPAN_COUNT; ++k) ms[k] = s->span_ms[k];
        if (frames) *frames = s->timed_frames;
    });
}

int dco_stream_views(const dco_stream* s, dco_frame_views* v) {
    if (!s || !v) return DCO_INPUT;
    const size_t nq = static_cast<size_t>(s->qw) * s->qh;
    v->full_w = s->fw;
    v->full_h = s->fh;
    v->quarter_w = s->qw;
    v->quarter_h = s->qh;
    v->disparity = s->disparity;
    v->sparse = s->sparse;
    v->m_fuse = s->m_fuse;
    v->m_i = s->m_i;
    v->edges = s->edges;
    v->dense = s->dense;
    v->composite = s->comp;
    v->mask = s->mask;
    v->flow_past_u = s->flow;
    v->flow_past_v = s->flow + nq;
    v->flow_future_u = s->flow + 2 * nq;
    v->flow_future_v = s->flow + 3 * nq;
    v->cost_volume = s->cost;
    v->aggregated = s->agg;
    v->volume_layout = stereo_slices_supported(s->cfg.cross_arm_l1, s->qh) ? 1 : 0;
    v->num_disparities = s->nd;
    return DCO_OK;
}

// state = {pushed, window slots (left_q, right_q, gray, rgb) x3, prev, prev_valid}
size_t dco_stream_state_size(const dco_stream* s) {
    if (!s) return 0;
    const size_t nq = static_cast<size_t>(s->qw) * s->qh, nf = static_cast<size_t>(s->fw) * s->fh;
    return 16 + 3 * (2 * nq + nf + 3 * nf) * 4 + nf * 4 + 4;
}

int dco_stream_save_state(dco_stream* s, void* buf, size_t len) {
    if (!s) return DCO_INPUT;
    return guarded(s->ctx, [&] {
        require(len >= dco_stream_state_size(s), "stream state: buffer too small");
        const size_t nq = static_cast<size_t>(s->qw) * s->qh, nf = static_cast<size_t>(s->fw) * s->fh;
        char* p = static_cast<char*>(buf);
        memcpy(p, &s->pushed, 8);
        p += 16;
        auto d2h = [&](const void* src, size_t bytes) {
            cuda_check(cudaMemcpyAsync(p, src, bytes, cudaMemcpyDeviceToHost, s->ctx->stream), "d2h");
            p += bytes;
        };
        for (int i = 0; i < 3; ++i) {
            d2h(s->left_q[i], nq * 4);
            d2h(s->right_q[i], nq * 4);
            d2h(s->gray[i], nf * 4);
            d2h(s->rgb[i], 3 * nf * 4);
        }
        d2h(s->prev, nf * 4);
        d2h(s->prev_valid, 4);
        cuda_check(cudaStreamSynchronize(s->ctx->stream), "sync");
    });
}

int dco_stream_load_state(dco_stream* s, const void* buf, size_t len) {
    if (!s) return DCO_INPUT;
    return guarded(s->ctx, [&] {
        require(len >= dco_stream_state_size(s), "stream state: buffer too small");
        const size_t nq = static_cast<size_t>(s->qw) * s->qh, nf = static_cast<size_t>(s->fw) * s->fh;
        const char* p = static_cast<const char*>(buf);
        memcpy(&s->pushed, p, 8);
        p += 16;
        auto h2d = [&](void* dst, size_t bytes) {
            cuda_check(cudaMemcpyAsync(dst, p, bytes, cudaMemcpyHostToDevice, s->ctx->stream), "h2d");
            p += bytes;
        };
        for (int i = 0; i < 3; ++i) {
            h2d(s->left_q[i], nq * 4);
            h2d(s->right_q[i], nq * 4);
            h2d(s->gray[i], nf * 4);
            h2d(s->rgb[i], 3 * nf * 4);
        }
        h2d(s->prev, nf * 4);
        h2d(s->prev_valid, 4);
        cuda_check(cudaStreamSynchronize(s->ctx->stream), "sync");
    });
}

int dco_composite(dco_ctx* ctx, const float* real, const float* dense, const float* vrgb, const float* vdepth,
                  int w, int h, float* out, uint8_t* mask) {
    return guarded(ctx, [&] { composite(ctx, real, dense, vrgb, vdepth, w, h, out, mask); });
}

int dco_stereo_sparse_depth(dco_ctx* ctx, const float* left_q, const float* right_q, int w, int h,
                            const dco_config* cfg, int fw, int fh, float* disparity, float* sparse) {
    return guarded(ctx, [&] {
        validate_config(cfg);
        const size_t nq = static_cast<size_t>(w) * h;
        const int nd = cfg->d_max - cfg->d_min + 1;
        uint8_t* arms = static_cast<uint8_t*>(scratch(ctx, S_ARMS, 4 * nq));
        float* cost = static_cast<float*>(scratch(ctx, S_COST, nq * nd * 4));
        float* agg = static_cast<float*>(scratch(ctx, S_AGG, nq * nd * 4));
        float* d0 = static_cast<float*>(scratch(ctx, S_TMP0, nq * 4 * 2));
        float* d1 = d0 + nq;
        uint8_t *L = arms, *R = arms + nq, *U = arms + 2 * nq, *D = arms + 3 * nq;
        build_cross_windows(ctx, left_q, w, h, cfg, L, R, U, D);
        if (stereo_slices_supported(cfg->cross_arm_l1, h)) {
            int* rect = static_cast<int*>(scratch(ctx, S_FLAG_SLICE, 2 * static_cast<size_t>(nd) * sizeof(int)));
            cost_volume_slices(ctx, left_q, right_q, w, h, L, R, U, D, cfg, cfg->cross_arm_l1, cost, rect);
            aggregate_slices(ctx, cost, w, h, nd, L, R, U, D, cfg->cross_arm_l1, rect, agg);
            wta_slices(ctx, agg, w, h, cfg->d_min, nd, d0);
        } else {
            compute_cost_volume(ctx, left_q, right_q, w, h, L, R, U, D, cfg, cost);
            aggregate_costs(ctx, cost, w, h, nd, L, R, U, D, cfg->cross_arm_l1, agg);
            select_disparity_wta(ctx, agg, w, h, cfg->d_min, nd, d0);
        }
        float* disp = disparity ? disparity : d1;
        refine_disparity_histogram(ctx, d0, w, h, L, R, U, D, cfg->hist_iterations, cfg->d_max, cfg->cross_arm_l1, disp);
        disparity_to_sparse_depth(ctx, disp, w, h, cfg, fw, fh, sparse);
    });
}

}  // extern "C"
