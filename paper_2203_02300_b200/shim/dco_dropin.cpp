// dco_dropin.cpp — the drop-in: the reference's L2 stage API (namespace dco,
// /root/reference/proj/include/dco/{pyramid,stereo,flow,contour,densify,
// occlude}.hpp) implemented on top of the C-ABI of libdco_gpu.so.
//
// Compiled against the reference's own headers, this object replaces
// pyramid.o stereo.o flow.o contour.o densify.o and occlude.o's composite()
// at link time (src/CMakeLists.txt:1-13), so unmodified reference callers —
// tests/acceptance.cpp, src/pipeline.cpp, tools/dco.cpp — run on the B200
// kernels. Each function: host value types -> device buffers (H2D), the
// C-ABI call, D2H, and dco_status -> the reference's exception classes
// (include/dco/error.hpp:10-32). Build recipe: scripts/build_dropin.sh.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <stdexcept>
#include <cstring>
#include <string>
#include <vector>

#include "dco/contour.hpp"
#include "dco/densify.hpp"
#include "dco/error.hpp"
#include "dco/flow.hpp"
#include "dco/occlude.hpp"
#include "dco/pyramid.hpp"
#include "dco/stereo.hpp"
#include "dco_gpu.h"

namespace {

dco_ctx* ctx() {
    static dco_ctx* c = [] {
        dco_ctx* h = nullptr;
        if (dco_create(0, &h) != DCO_OK) throw std::runtime_error("dco_create: no CUDA device");
        return h;
    }();
    return c;
}

void check(int st) {
    if (st == DCO_OK) return;
    std::string msg = dco_last_error(ctx());
    switch (st) {
        case DCO_CONFIG: throw dco::ConfigError(msg);
        case DCO_INPUT: throw dco::InputError(msg);
        case DCO_CODEC: throw dco::CodecError(msg);
        case DCO_UNSOLVABLE: throw dco::UnsolvableFrameError(msg);
        default: throw std::runtime_error("dco_gpu: " + msg);
    }
}

void cu(cudaError_t e) {
    if (e != cudaSuccess) throw std::runtime_error(std::string("cuda: ") + cudaGetErrorString(e));
}

// RAII device buffer
template <typename T>
struct Dev {
    T* p = nullptr;
    size_t n = 0;
    explicit Dev(size_t count) : n(count) { cu(cudaMalloc(&p, (count ? count : 1) * sizeof(T))); }
    Dev(const T* host, size_t count) : Dev(count) {
        if (count) cu(cudaMemcpy(p, host, count * sizeof(T), cudaMemcpyHostToDevice));
    }
    explicit Dev(const std::vector<T>& v) : Dev(v.data(), v.size()) {}
    ~Dev() { cudaFree(p); }
    Dev(const Dev&) = delete;
    Dev& operator=(const Dev&) = delete;
    void get(T* host) const {
        cu(cudaDeviceSynchronize());
        if (n) cu(cudaMemcpy(host, p, n * sizeof(T), cudaMemcpyDeviceToHost));
    }
    void get(std::vector<T>& v) const {
        v.resize(n);
        get(v.data());
    }
};

dco_config cfg_of(const dco::PipelineConfig& p) {
    dco_config c;
    c.lambda_ad = p.lambda_ad;
    c.lambda_census = p.lambda_census;
    c.gamma_l = p.gamma_l;
    c.epsilon = p.epsilon;
    c.t_high = p.t_high;
    c.t_low = p.t_low;
    c.t_depth = p.t_depth;
    c.lambda_d = p.lambda_d;
    c.lambda_s = p.lambda_s;
    c.lambda_s2 = p.lambda_s2;
    c.d_min = p.d_min;
    c.d_max = p.d_max;
    c.focal_px = p.focal_px;
    c.baseline_m = p.baseline_m;
    c.census_window_w = p.census_window_w;
    c.census_window_h = p.census_window_h;
    c.cross_color_tau = p.cross_color_tau;
    c.cross_color_tau2 = p.cross_color_tau2;
    c.cross_arm_l1 = p.cross_arm_l1;
    c.cross_arm_l2 = p.cross_arm_l2;
    c.box_radius = p.box_radius;
    c.gauss_sigma = p.gauss_sigma;
    c.confidence_offset_k = p.confidence_offset_k;
    c.hist_iterations = p.hist_iterations;
    c.solver_tol = p.solver_tol;
    c.solver_max_iter = p.solver_max_iter;
    return c;
}

struct DevArms {
    Dev<uint8_t> l, r, u, d;
    explicit DevArms(const dco::CrossWindowField& f) : l(f.left), r(f.right), u(f.up), d(f.down) {}
};

}  // namespace

namespace dco {

// ---------------------------------------------------------------- pyramid
GrayImage downsample_half(const GrayImage& img) {
    if (img.width < 2 || img.height < 2) throw InputError("downsample_half: dimensions must be at least 2x2");
    Dev<float> in(img.data);
    GrayImage out(img.width / 2, img.height / 2);
    Dev<float> o(out.data.size());
    check(dco_downsample_half(ctx(), in.p, img.width, img.height, o.p));
    o.get(out.data);
    return out;
}

std::vector<GrayImage> build_pyramid(const GrayImage& img, int levels) {
    if (levels < 1) throw InputError("build_pyramid: levels must be >= 1");
    int w = img.width, h = img.height;
    for (int i = 1; i < levels; ++i) w /= 2, h /= 2;
    if (w < 8 || h < 8) throw InputError("build_pyramid: coarsest level would drop below 8 px");
    std::vector<GrayImage> pyr{img};
    for (int i = 1; i < levels; ++i) pyr.push_back(downsample_half(pyr.back()));
    return pyr;
}

// ----------------------------------------------------------------- stereo
CrossWindowField build_cross_windows(const GrayImage& img, const PipelineConfig& cfg) {
    dco_config c = cfg_of(cfg);
    Dev<float> in(img.data);
    size_t n = img.pixel_count();
    Dev<uint8_t> l(n), r(n), u(n), d(n);
    check(dco_build_cross_windows(ctx(), in.p, img.width, img.height, &c, l.p, r.p, u.p, d.p));
    CrossWindowField f(img.width, img.height);
    l.get(f.left);
    r.get(f.right);
    u.get(f.up);
    d.get(f.down);
    return f;
}

CensusMap census_transform(const GrayImage& img, int ww, int wh) {
    Dev<float> in(img.data);
    Dev<uint64_t> o(img.pixel_count());
    check(dco_census_transform(ctx(), in.p, img.width, img.height, ww, wh, o.p));
    CensusMap m;
    m.width = img.width;
    m.height = img.height;
    m.bits = ww * wh - 1;
    o.get(m.data);
    return m;
}

int hamming_distance(uint64_t a, uint64_t b) { return __builtin_popcountll(a ^ b); }

double adaptive_alpha(int l_min, const PipelineConfig& cfg) {
    return 1.0 - std::exp(-cfg.gamma_l / (static_cast<double>(l_min) + cfg.epsilon));
}

CostVolume compute_cost_volume(const GrayImage& left, const GrayImage& right, const CrossWindowField& windows,
                               const PipelineConfig& cfg) {
    if (left.width != right.width || left.height != right.height)
        throw InputError("compute_cost_volume: left/right dimensions differ");
    if (windows.width != left.width || windows.height != left.height)
        throw InputError("compute_cost_volume: cross windows built on different dimensions");
    dco_config c = cfg_of(cfg);
    Dev<float> l(left.data), r(right.data);
    DevArms a(windows);
    CostVolume v;
    v.width = left.width;
    v.height = left.height;
    v.d_min = cfg.d_min;
    v.d_max = cfg.d_max;
    Dev<float> o(left.pixel_count() * static_cast<size_t>(cfg.d_max - cfg.d_min + 1 > 0 ? cfg.d_max - cfg.d_min + 1 : 1));
    check(dco_compute_cost_volume(ctx(), l.p, r.p, left.width, left.height, a.l.p, a.r.p, a.u.p, a.d.p, &c, o.p));
    o.get(v.cost);
    return v;
}

CostVolume aggregate_costs(const CostVolume& vol, const CrossWindowField& windows) {
    if (windows.width != vol.width || windows.height != vol.height)
        throw InputError("aggregate_costs: cross windows built on different dimensions");
    Dev<float> in(vol.cost), o(vol.cost.size());
    DevArms a(windows);
    check(dco_aggregate_costs(ctx(), in.p, vol.width, vol.height, vol.d_min, vol.d_max, a.l.p, a.r.p, a.u.p, a.d.p,
                              o.p));
    CostVolume out = vol;
    o.get(out.cost);
    return out;
}

DisparityMap select_disparity_wta(const CostVolume& vol) {
    Dev<float> in(vol.cost);
    DisparityMap d(vol.width, vol.height);
    Dev<float> o(d.disparity.size());
    check(dco_select_disparity_wta(ctx(), in.p, vol.width, vol.height, vol.d_min, vol.d_max, o.p));
    o.get(d.disparity);
    return d;
}

DisparityMap refine_disparity_histogram(const DisparityMap& disp, const CrossWindowField& windows, int iterations) {
    if (windows.width != disp.width || windows.height != disp.height)
        throw InputError("refine_disparity_histogram: cross windows built on different dimensions");
    Dev<float> in(disp.disparity), o(disp.disparity.size());
    DevArms a(windows);
    check(dco_refine_disparity_histogram(ctx(), in.p, disp.width, disp.height, a.l.p, a.r.p, a.u.p, a.d.p,
                                         iterations, o.p));
    DisparityMap out = disp;
    o.get(out.disparity);
    return out;
}

SparseDepthMap disparity_to_sparse_depth(const DisparityMap& disp, const PipelineConfig& cfg, int full_width,
                                         int full_height) {
    dco_config c = cfg_of(cfg);
    Dev<float> in(disp.disparity);
    SparseDepthMap out(full_width > 0 ? full_width : 0, full_height > 0 ? full_height : 0);
    Dev<float> o(out.data.size());
    check(dco_disparity_to_sparse_depth(ctx(), in.p, disp.width, disp.height, &c, full_width, full_height, o.p));
    o.get(out.data);
    return out;
}

// ------------------------------------------------------------------- flow
std::optional<KeyframeWindow> KeyframeBuffer::push_frame(GrayImage frame) {
    if (!frames_.empty() && (frame.width != frames_.front().width || frame.height != frames_.front().height))
        throw InputError("push_frame: frame dimensions differ from buffered frames");
    frames_.push_back(std::move(frame));
    if (frames_.size() > 3) frames_.pop_front();
    if (frames_.size() < 3) return std::nullopt;
    return KeyframeWindow{frames_[0], frames_[1], frames_[2]};
}

FlowField compute_flow(const GrayImage& from, const GrayImage& to, const PipelineConfig& cfg) {
    if (from.width != to.width || from.height != to.height) throw InputError("compute_flow: frame dimensions differ");
    dco_config c = cfg_of(cfg);
    Dev<float> f(from.data), t(to.data);
    FlowField out(from.width, from.height);
    Dev<float> u(out.u.size()), v(out.v.size());
    check(dco_compute_flow(ctx(), f.p, t.p, from.width, from.height, &c, u.p, v.p));
    u.get(out.u);
    v.get(out.v);
    return out;
}

// ---------------------------------------------------------------- contour
PolarFlowField flow_to_polar(const FlowField& flow) {
    Dev<float> u(flow.u), v(flow.v), r(flow.u.size()), t(flow.u.size());
    check(dco_flow_to_polar(ctx(), u.p, v.p, flow.width, flow.height, r.p, t.p));
    PolarFlowField p;
    p.width = flow.width;
    p.height = flow.height;
    r.get(p.r);
    t.get(p.theta);
    return p;
}

AmplitudeMap gradient_amplitude(const PolarFlowField& polar) {
    Dev<float> r(polar.r);
    AmplitudeMap out(polar.width, polar.height, 0.0f);
    Dev<float> o(out.data.size());
    check(dco_gradient_amplitude(ctx(), r.p, polar.width, polar.height, o.p));
    o.get(out.data);
    return out;
}

AmplitudeMap fuse_amplitudes(const FlowField& fp, const FlowField& ff, const AmplitudeMap& mp, const AmplitudeMap& mf,
                             const PipelineConfig& cfg) {
    const int w = mp.width, h = mp.height;
    if (fp.width != w || fp.height != h || ff.width != w || ff.height != h || mf.width != w || mf.height != h)
        throw InputError("fuse_amplitudes: input dimensions differ");
    dco_config c = cfg_of(cfg);
    Dev<float> pu(fp.u), pv(fp.v), fu(ff.u), fv(ff.v), a(mp.data), b(mf.data), o(mp.data.size());
    check(dco_fuse_amplitudes(ctx(), pu.p, pv.p, fu.p, fv.p, a.p, b.p, w, h, &c, o.p));
    AmplitudeMap out(w, h, 0.0f);
    o.get(out.data);
    return out;
}

AmplitudeMap box_filter(const AmplitudeMap& amp, int radius) {
    Dev<float> in(amp.data), o(amp.data.size());
    check(dco_box_filter(ctx(), in.p, amp.width, amp.height, radius, o.p));
    AmplitudeMap out(amp.width, amp.height, 0.0f);
    o.get(out.data);
    return out;
}

AmplitudeMap normalize_amplitude(const AmplitudeMap& amp) {
    Dev<float> in(amp.data), o(amp.data.size());
    check(dco_normalize_amplitude(ctx(), in.p, amp.width, amp.height, o.p));
    AmplitudeMap out = amp;
    o.get(out.data);
    return out;
}

GrayImage gaussian_blur(const GrayImage& img, double sigma) {
    Dev<float> in(img.data), o(img.data.size());
    check(dco_gaussian_blur(ctx(), in.p, img.width, img.height, sigma, o.p));
    GrayImage out(img.width, img.height);
    o.get(out.data);
    return out;
}

ContourResult extract_depth_contours_prefiltered(const GrayImage& blurred, const AmplitudeMap& m_fuse,
                                                 const PipelineConfig& cfg) {
    dco_config c = cfg_of(cfg);
    Dev<float> b(blurred.data), m(m_fuse.data), mi(blurred.data.size());
    Dev<uint8_t> e(blurred.data.size());
    check(dco_extract_depth_contours_prefiltered(ctx(), b.p, blurred.width, blurred.height, m.p, m_fuse.width,
                                                 m_fuse.height, &c, e.p, mi.p));
    ContourResult r{EdgeMask(blurred.width, blurred.height, 0), IntensityGradientMap(blurred.width, blurred.height, 0.0f)};
    e.get(r.edges.data);
    mi.get(r.m_i.data);
    return r;
}

ContourResult extract_depth_contours(const GrayImage& gray, const AmplitudeMap& m_fuse, const PipelineConfig& cfg) {
    return extract_depth_contours_prefiltered(gaussian_blur(gray, cfg.gauss_sigma), m_fuse, cfg);
}

// ---------------------------------------------------------------- densify
double smoothness_weight(int px, int py, int qx, int qy, const EdgeMask& b_dp, const AmplitudeMap& m_fuse,
                         const IntensityGradientMap& m_i) {
    Dev<uint8_t> e(b_dp.data);
    Dev<float> f(m_fuse.data), mi(m_i.data);
    double out = 0.0;
    check(dco_smoothness_weight(ctx(), px, py, qx, qy, e.p, b_dp.width, b_dp.height, f.p, m_fuse.width,
                                m_fuse.height, mi.p, &out));
    return out;
}

ConstraintSystem assemble_system(const SparseDepthMap& d_sparse, const EdgeMask& b_dp, const AmplitudeMap& m_fuse,
                                 const IntensityGradientMap& m_i, const FloatMap* d_pre, const PipelineConfig& cfg) {
    const int w = d_sparse.width, h = d_sparse.height;
    if (b_dp.width != w || b_dp.height != h || m_i.width != w || m_i.height != h)
        throw InputError("assemble_system: full-resolution inputs disagree on dimensions");
    if (d_pre && (d_pre->width != w || d_pre->height != h))
        throw InputError("assemble_system: previous dense map has different dimensions");
    dco_config c = cfg_of(cfg);
    size_t n = d_sparse.pixel_count();
    Dev<float> s(d_sparse.data), f(m_fuse.data), mi(m_i.data);
    Dev<uint8_t> e(b_dp.data);
    Dev<float> pre(d_pre ? d_pre->data.size() : 0);
    if (d_pre) cu(cudaMemcpy(pre.p, d_pre->data.data(), n * 4, cudaMemcpyHostToDevice));
    Dev<double> diag(n), ch(n), cv(n), rhs(n), init(n);
    Dev<uint8_t> anch(n);
    dco_system sys{w, h, diag.p, ch.p, cv.p, rhs.p, init.p, anch.p, 0.0, 0};
    check(dco_assemble_system(ctx(), s.p, e.p, f.p, m_fuse.width, m_fuse.height, mi.p, d_pre ? pre.p : nullptr, w, h,
                              &c, &sys));
    ConstraintSystem out;
    out.width = w;
    out.height = h;
    diag.get(out.diag);
    ch.get(out.coup_h);
    cv.get(out.coup_v);
    rhs.get(out.rhs);
    init.get(out.initial);
    anch.get(out.anchored);
    out.constant_term = sys.constant_term;
    out.anchor_count = sys.anchor_count;
    return out;
}

namespace {
struct DevSys {
    Dev<double> diag, ch, cv, rhs, init;
    Dev<uint8_t> anch;
    dco_system s;
    explicit DevSys(const ConstraintSystem& sys)
        : diag(sys.diag), ch(sys.coup_h), cv(sys.coup_v), rhs(sys.rhs), init(sys.initial), anch(sys.anchored) {
        s = dco_system{sys.width, sys.height, diag.p, ch.p, cv.p, rhs.p, init.p, anch.p, sys.constant_term,
                       static_cast<uint64_t>(sys.anchor_count)};
    }
};
}  // namespace

void apply_system(const ConstraintSystem& sys, const std::vector<double>& x, std::vector<double>& out) {
    DevSys d(sys);
    Dev<double> xd(x), o(sys.size());
    check(dco_apply_system(ctx(), &d.s, xd.p, o.p));
    o.get(out);
}

double objective_value(const ConstraintSystem& sys, const std::vector<double>& x) {
    DevSys d(sys);
    Dev<double> xd(x);
    double v = 0.0;
    check(dco_objective_value(ctx(), &d.s, xd.p, &v));
    return v;
}

DenseDepthMap solve_dense_depth(const ConstraintSystem& sys, const PipelineConfig& cfg, SolveStats* stats) {
    if (sys.anchor_count == 0)
        throw UnsolvableFrameError("solve_dense_depth: no pixel carries a data or stability constraint");
    dco_config c = cfg_of(cfg);
    DevSys d(sys);
    DenseDepthMap out(sys.width, sys.height);
    Dev<float> o(sys.size());
    std::vector<double> hist(static_cast<size_t>(cfg.solver_max_iter) + 1);
    dco_solve_stats st{0, 0.0, 0.0, 0.0, hist.data(), static_cast<int>(hist.size())};
    check(dco_solve_dense_depth(ctx(), &d.s, &c, o.p, &st));
    o.get(out.data);
    if (stats) {
        stats->iterations = st.iterations;
        stats->relative_residual = st.relative_residual;
        stats->objective_initial = st.objective_initial;
        stats->objective_final = st.objective_final;
        stats->residual_history.assign(hist.begin(), hist.begin() + std::min<size_t>(hist.size(), st.iterations + 1));
    }
    return out;
}

// -------------------------------------------------------------- composite
// transform_mesh / render_virtual, occlude.cpp:78-169 (dco_transform_mesh,
// dco_render_virtual; the renderer is bit-exact with the index-ordered z-buffer)
TriangleMesh transform_mesh(const TriangleMesh& mesh, const std::array<double, 16>& pose) {
    const int nv = static_cast<int>(mesh.vertices.size());
    std::vector<float> flat(3 * static_cast<size_t>(nv));
    for (int i = 0; i < nv; ++i)
        for (int k = 0; k < 3; ++k) flat[3 * i + k] = mesh.vertices[i][k];
    Dev<float> v(flat), o(flat.size());
    check(dco_transform_mesh(ctx(), v.p, nv, pose.data(), o.p));
    o.get(flat);
    TriangleMesh out = mesh;
    for (int i = 0; i < nv; ++i)
        for (int k = 0; k < 3; ++k) out.vertices[i][k] = flat[3 * i + k];
    return out;
}

VirtualLayer render_virtual(const TriangleMesh& mesh, double focal_px, double cx, double cy, int out_width,
                            int out_height) {
    if (out_width < 1 || out_height < 1) throw InputError("render_virtual: output dimensions must be positive");
    const size_t nv = mesh.vertices.size(), nt = mesh.triangles.size();
    std::vector<float> fv(3 * nv), fc(3 * nv);
    std::vector<int> ft(3 * nt);
    for (size_t i = 0; i < nv; ++i)
        for (int k = 0; k < 3; ++k) {
            fv[3 * i + k] = mesh.vertices[i][k];
            fc[3 * i + k] = mesh.colors[i][k];
        }
    for (size_t t = 0; t < nt; ++t)
        for (int k = 0; k < 3; ++k) ft[3 * t + k] = mesh.triangles[t][k];
    Dev<float> v(fv), c(fc);
    Dev<int> tr(ft);
    const size_t n = static_cast<size_t>(out_width) * out_height;
    Dev<float> rgb(3 * n), depth(n);
    check(dco_render_virtual(ctx(), v.p, tr.p, c.p, static_cast<int>(nt), focal_px, cx, cy, out_width, out_height,
                             rgb.p, depth.p));
    VirtualLayer layer;
    layer.color = ColorImage(out_width, out_height);
    layer.depth = FloatMap(out_width, out_height);
    rgb.get(layer.color.data);
    depth.get(layer.depth.data);
    return layer;
}

CompositeResult composite(const ColorImage& real, const DenseDepthMap& dense, const VirtualLayer& virt) {
    const int w = real.width, h = real.height;
    if (dense.width != w || dense.height != h || virt.color.width != w || virt.color.height != h ||
        virt.depth.width != w || virt.depth.height != h)
        throw InputError("composite: input dimensions differ");
    Dev<float> r(real.data), dd(dense.data), vc(virt.color.data), vd(virt.depth.data), o(real.data.size());
    Dev<uint8_t> m(real.pixel_count());
    check(dco_composite(ctx(), r.p, dd.p, vc.p, vd.p, w, h, o.p, m.p));
    CompositeResult res;
    res.color = ColorImage(w, h);
    res.mask = OcclusionMask(w, h, 0);
    o.get(res.color.data);
    m.get(res.mask.data);
    return res;
}

}  // namespace dco
