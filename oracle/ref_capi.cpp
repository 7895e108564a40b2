// ref_capi.cpp — extern "C" access to the UNMODIFIED reference library
// (/root/reference/proj/src, compiled by oracle/Makefile into oracle/_ref).
//
// TEST INFRASTRUCTURE ONLY. This file is the checker's doorway: tests/,
// __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference leg
// load oracle/_ref/libdco_ref.so through it. No product code links it.
//
// Every ref_* function converts plain host pointers into the reference's
// value types, calls the reference stage function named in its comment, and
// copies the result out. Exceptions map to the status codes of dco_gpu.h.
#include <cstring>
#include <exception>
#include <string>

#include "dco/codec.hpp"
#include "dco/config.hpp"
#include "dco/contour.hpp"
#include "dco/densify.hpp"
#include "dco/error.hpp"
#include "dco/flow.hpp"
#include "dco/occlude.hpp"
#include "dco/pipeline.hpp"
#include "dco/pyramid.hpp"
#include "dco/stereo.hpp"
#include "dco/synth.hpp"
#include "dco_gpu.h"

using namespace dco;

namespace {

thread_local std::string g_err;

template <typename F>
int guarded(F&& fn) {
    try {
        fn();
        return DCO_OK;
    } catch (const ConfigError& e) {
        g_err = e.what();
        return DCO_CONFIG;
    } catch (const InputError& e) {
        g_err = e.what();
        return DCO_INPUT;
    } catch (const CodecError& e) {
        g_err = e.what();
        return DCO_CODEC;
    } catch (const UnsolvableFrameError& e) {
        g_err = e.what();
        return DCO_UNSOLVABLE;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 99;
    }
}

PipelineConfig to_cfg(const dco_config* c) {
    PipelineConfig p;
    p.lambda_ad = c->lambda_ad;
    p.lambda_census = c->lambda_census;
    p.gamma_l = c->gamma_l;
    p.epsilon = c->epsilon;
    p.t_high = c->t_high;
    p.t_low = c->t_low;
    p.t_depth = c->t_depth;
    p.lambda_d = c->lambda_d;
    p.lambda_s = c->lambda_s;
    p.lambda_s2 = c->lambda_s2;
    p.d_min = c->d_min;
    p.d_max = c->d_max;
    p.focal_px = c->focal_px;
    p.baseline_m = c->baseline_m;
    p.census_window_w = c->census_window_w;
    p.census_window_h = c->census_window_h;
    p.cross_color_tau = c->cross_color_tau;
    p.cross_color_tau2 = c->cross_color_tau2;
    p.cross_arm_l1 = c->cross_arm_l1;
    p.cross_arm_l2 = c->cross_arm_l2;
    p.box_radius = c->box_radius;
    p.gauss_sigma = c->gauss_sigma;
    p.confidence_offset_k = c->confidence_offset_k;
    p.hist_iterations = c->hist_iterations;
    p.solver_tol = c->solver_tol;
    p.solver_max_iter = c->solver_max_iter;
    return p;
}

GrayImage gray_in(const float* p, int w, int h) {
    GrayImage g(w, h);
    std::memcpy(g.data.data(), p, sizeof(float) * g.data.size());
    return g;
}

FloatMap map_in(const float* p, int w, int h) {
    FloatMap m(w, h);
    std::memcpy(m.data.data(), p, sizeof(float) * m.data.size());
    return m;
}

BinaryMask mask_in(const uint8_t* p, int w, int h) {
    BinaryMask m(w, h);
    std::memcpy(m.data.data(), p, m.data.size());
    return m;
}

CrossWindowField arms_in(const uint8_t* l, const uint8_t* r, const uint8_t* u, const uint8_t* d,
                         int w, int h) {
    CrossWindowField f(w, h);
    size_t n = static_cast<size_t>(w) * h;
    std::memcpy(f.left.data(), l, n);
    std::memcpy(f.right.data(), r, n);
    std::memcpy(f.up.data(), u, n);
    std::memcpy(f.down.data(), d, n);
    return f;
}

template <typename T>
void copy_out(const std::vector<T>& v, T* out) {
    std::memcpy(out, v.data(), sizeof(T) * v.size());
}

ConstraintSystem sys_in(int w, int h, const double* diag, const double* ch, const double* cv,
                        const double* rhs, const double* initial, const uint8_t* anchored,
                        double constant_term) {
    ConstraintSystem s;
    s.width = w;
    s.height = h;
    size_t n = static_cast<size_t>(w) * h;
    s.diag.assign(diag, diag + n);
    s.coup_h.assign(ch, ch + n);
    s.coup_v.assign(cv, cv + n);
    s.rhs.assign(rhs, rhs + n);
    s.initial.assign(initial, initial + n);
    s.anchored.assign(anchored, anchored + n);
    s.constant_term = constant_term;
    s.anchor_count = 0;
    for (uint8_t a : s.anchored) s.anchor_count += a;
    return s;
}

} // namespace

extern "C" {

const char* ref_last_error(void) { return g_err.c_str(); }

// PipelineConfig defaults, config.hpp:13-56.
void ref_config_default(dco_config* c) {
    PipelineConfig p;
    c->lambda_ad = p.lambda_ad;
    c->lambda_census = p.lambda_census;
    c->gamma_l = p.gamma_l;
    c->epsilon = p.epsilon;
    c->t_high = p.t_high;
    c->t_low = p.t_low;
    c->t_depth = p.t_depth;
    c->lambda_d = p.lambda_d;
    c->lambda_s = p.lambda_s;
    c->lambda_s2 = p.lambda_s2;
    c->d_min = p.d_min;
    c->d_max = p.d_max;
    c->focal_px = p.focal_px;
    c->baseline_m = p.baseline_m;
    c->census_window_w = p.census_window_w;
    c->census_window_h = p.census_window_h;
    c->cross_color_tau = p.cross_color_tau;
    c->cross_color_tau2 = p.cross_color_tau2;
    c->cross_arm_l1 = p.cross_arm_l1;
    c->cross_arm_l2 = p.cross_arm_l2;
    c->box_radius = p.box_radius;
    c->gauss_sigma = p.gauss_sigma;
    c->confidence_offset_k = p.confidence_offset_k;
    c->hist_iterations = p.hist_iterations;
    c->solver_tol = p.solver_tol;
    c->solver_max_iter = p.solver_max_iter;
}

// PipelineConfig::validate, config.cpp:10-36.
int ref_config_validate(const dco_config* c) {
    return guarded([&] { to_cfg(c).validate(); });
}

// load_config, config.cpp:119-144 (the strict key=value parser).
int ref_load_config(const char* path, dco_config* out) {
    return guarded([&] {
        PipelineConfig p = load_config(path);
        ref_config_default(out);
        out->lambda_ad = p.lambda_ad;
        out->lambda_census = p.lambda_census;
        out->gamma_l = p.gamma_l;
        out->epsilon = p.epsilon;
        out->t_high = p.t_high;
        out->t_low = p.t_low;
        out->t_depth = p.t_depth;
        out->lambda_d = p.lambda_d;
        out->lambda_s = p.lambda_s;
        out->lambda_s2 = p.lambda_s2;
        out->d_min = p.d_min;
        out->d_max = p.d_max;
        out->focal_px = p.focal_px;
        out->baseline_m = p.baseline_m;
        out->census_window_w = p.census_window_w;
        out->census_window_h = p.census_window_h;
        out->cross_color_tau = p.cross_color_tau;
        out->cross_color_tau2 = p.cross_color_tau2;
        out->cross_arm_l1 = p.cross_arm_l1;
        out->cross_arm_l2 = p.cross_arm_l2;
        out->box_radius = p.box_radius;
        out->gauss_sigma = p.gauss_sigma;
        out->confidence_offset_k = p.confidence_offset_k;
        out->hist_iterations = p.hist_iterations;
        out->solver_tol = p.solver_tol;
        out->solver_max_iter = p.solver_max_iter;
    });
}

// render_synth_frame, synth.cpp:68-135. Any output pointer may be NULL.
int ref_render_synth_frame(int width, int height, double z_fg, double z_bg, double focal_px,
                           double baseline_m, int square_size, double square_x0,
                           double square_y0, double shift_x, double shift_y, uint64_t seed,
                           int index, float* left, float* right, float* gt_depth,
                           uint8_t* gt_boundary, float* gt_u, float* gt_v) {
    return guarded([&] {
        SceneSpec s;
        s.width = width;
        s.height = height;
        s.z_fg = z_fg;
        s.z_bg = z_bg;
        s.focal_px = focal_px;
        s.baseline_m = baseline_m;
        s.square_size = square_size;
        s.square_x0 = square_x0;
        s.square_y0 = square_y0;
        s.shift_x = shift_x;
        s.shift_y = shift_y;
        s.seed = seed;
        SynthFrame f = render_synth_frame(s, index);
        if (left) copy_out(f.left.data, left);
        if (right) copy_out(f.right.data, right);
        if (gt_depth) copy_out(f.gt_depth.data, gt_depth);
        if (gt_boundary) copy_out(f.gt_boundary.data, gt_boundary);
        if (gt_u) copy_out(f.gt_flow.u, gt_u);
        if (gt_v) copy_out(f.gt_flow.v, gt_v);
    });
}

// write_pgm (codec.cpp:211-229) followed by read_gray (codec.cpp:59-82):
// the 8-bit round trip every CLI/pipeline input goes through. bytes (may be
// NULL) receives the PGM payload, back (may be NULL) the re-read floats.
int ref_pgm_roundtrip(const float* img, int w, int h, const char* tmp_path, uint8_t* bytes,
                      float* back) {
    return guarded([&] {
        write_pgm(gray_in(img, w, h), tmp_path);
        GrayImage g = read_gray(tmp_path);
        if (back) copy_out(g.data, back);
        if (bytes)
            for (size_t i = 0; i < g.data.size(); ++i)
                bytes[i] = static_cast<uint8_t>(g.data[i] * 255.0f + 0.5f);
    });
}

// write_pgm / write_ppm / write_pfm (codec.cpp:211-229, 293-309), read_pnm via
// read_gray / read_color (codec.cpp:59-82, 199-209), to_gray (image.cpp:7-15).
int ref_write_pgm(const float* img, int w, int h, const char* path) {
    return guarded([&] { write_pgm(gray_in(img, w, h), path); });
}

int ref_write_ppm(const float* rgb, int w, int h, const char* path) {
    return guarded([&] {
        ColorImage c(w, h);
        std::memcpy(c.data.data(), rgb, sizeof(float) * c.data.size());
        write_ppm(c, path);
    });
}

int ref_write_pfm(const float* map, int w, int h, const char* path) {
    return guarded([&] { write_pfm(map_in(map, w, h), path); });
}

// read_pnm of a P5 (color = 0) or P6 file; out (may be NULL) receives the
// floats (bytes / 255.0f), w and h the dimensions.
int ref_read_pnm(const char* path, int color, float* out, size_t cap, int* w, int* h) {
    return guarded([&] {
        LoadedImage img = read_image(path, color ? ImageFormat::Ppm : ImageFormat::Pgm);  // = read_pnm(path, color)
        if (color) {
            const ColorImage& c = std::get<ColorImage>(img);
            *w = c.width;
            *h = c.height;
            if (out && cap >= c.data.size()) copy_out(c.data, out);
        } else {
            const GrayImage& g = std::get<GrayImage>(img);
            *w = g.width;
            *h = g.height;
            if (out && cap >= g.data.size()) copy_out(g.data, out);
        }
    });
}

int ref_to_gray(const float* rgb, int w, int h, float* out) {
    return guarded([&] {
        ColorImage c(w, h);
        std::memcpy(c.data.data(), rgb, sizeof(float) * c.data.size());
        copy_out(to_gray(c).data, out);
    });
}

// downsample_half, pyramid.cpp:5-17.
int ref_downsample_half(const float* img, int w, int h, float* out) {
    return guarded([&] { copy_out(downsample_half(gray_in(img, w, h)).data, out); });
}

// build_cross_windows, stereo.cpp:52-68.
int ref_build_cross_windows(const float* img, int w, int h, const dco_config* c, uint8_t* l,
                            uint8_t* r, uint8_t* u, uint8_t* d) {
    return guarded([&] {
        CrossWindowField f = build_cross_windows(gray_in(img, w, h), to_cfg(c));
        copy_out(f.left, l);
        copy_out(f.right, r);
        copy_out(f.up, u);
        copy_out(f.down, d);
    });
}

// census_transform, stereo.cpp:70-96.
int ref_census_transform(const float* img, int w, int h, int ww, int wh, uint64_t* out) {
    return guarded([&] { copy_out(census_transform(gray_in(img, w, h), ww, wh).data, out); });
}

// adaptive_alpha, stereo.cpp:102-104.
double ref_adaptive_alpha(int l_min, const dco_config* c) { return adaptive_alpha(l_min, to_cfg(c)); }

// compute_cost_volume, stereo.cpp:106-150.
int ref_compute_cost_volume(const float* left, const float* right, int w, int h, const uint8_t* l,
                            const uint8_t* r, const uint8_t* u, const uint8_t* d,
                            const dco_config* c, float* cost) {
    return guarded([&] {
        CostVolume v = compute_cost_volume(gray_in(left, w, h), gray_in(right, w, h),
                                           arms_in(l, r, u, d, w, h), to_cfg(c));
        copy_out(v.cost, cost);
    });
}

// aggregate_costs, stereo.cpp:152-218.
int ref_aggregate_costs(const float* cost, int w, int h, int d_min, int d_max, const uint8_t* l,
                        const uint8_t* r, const uint8_t* u, const uint8_t* d, float* out) {
    return guarded([&] {
        CostVolume v;
        v.width = w;
        v.height = h;
        v.d_min = d_min;
        v.d_max = d_max;
        v.cost.assign(cost, cost + static_cast<size_t>(w) * h * (d_max - d_min + 1));
        copy_out(aggregate_costs(v, arms_in(l, r, u, d, w, h)).cost, out);
    });
}

// select_disparity_wta, stereo.cpp:220-238.
int ref_select_disparity_wta(const float* cost, int w, int h, int d_min, int d_max, float* disp) {
    return guarded([&] {
        CostVolume v;
        v.width = w;
        v.height = h;
        v.d_min = d_min;
        v.d_max = d_max;
        v.cost.assign(cost, cost + static_cast<size_t>(w) * h * (d_max - d_min + 1));
        copy_out(select_disparity_wta(v).disparity, disp);
    });
}

// refine_disparity_histogram, stereo.cpp:240-299.
int ref_refine_disparity_histogram(const float* disp, int w, int h, const uint8_t* l,
                                   const uint8_t* r, const uint8_t* u, const uint8_t* d, int iters,
                                   float* out) {
    return guarded([&] {
        DisparityMap m(w, h);
        std::memcpy(m.disparity.data(), disp, sizeof(float) * m.disparity.size());
        copy_out(refine_disparity_histogram(m, arms_in(l, r, u, d, w, h), iters).disparity, out);
    });
}

// disparity_to_sparse_depth, stereo.cpp:301-315.
int ref_disparity_to_sparse_depth(const float* disp, int w, int h, const dco_config* c, int fw,
                                  int fh, float* out) {
    return guarded([&] {
        DisparityMap m(w, h);
        std::memcpy(m.disparity.data(), disp, sizeof(float) * m.disparity.size());
        copy_out(disparity_to_sparse_depth(m, to_cfg(c), fw, fh).data, out);
    });
}

// compute_flow, flow.cpp:185-205.
int ref_compute_flow(const float* from, const float* to, int w, int h, const dco_config* c,
                     float* u, float* v) {
    return guarded([&] {
        FlowField f = compute_flow(gray_in(from, w, h), gray_in(to, w, h), to_cfg(c));
        copy_out(f.u, u);
        copy_out(f.v, v);
    });
}

// flow_to_polar, contour.cpp:10-25.
int ref_flow_to_polar(const float* u, const float* v, int w, int h, float* r, float* theta) {
    return guarded([&] {
        FlowField f(w, h);
        std::memcpy(f.u.data(), u, sizeof(float) * f.u.size());
        std::memcpy(f.v.data(), v, sizeof(float) * f.v.size());
        PolarFlowField p = flow_to_polar(f);
        copy_out(p.r, r);
        if (theta) copy_out(p.theta, theta);
    });
}

// gradient_amplitude, contour.cpp:27-42.
int ref_gradient_amplitude(const float* r, int w, int h, float* amp) {
    return guarded([&] {
        PolarFlowField p;
        p.width = w;
        p.height = h;
        p.r.assign(r, r + static_cast<size_t>(w) * h);
        p.theta.assign(p.r.size(), 0.0f);
        copy_out(gradient_amplitude(p).data, amp);
    });
}

// fuse_amplitudes, contour.cpp:82-106.
int ref_fuse_amplitudes(const float* pu, const float* pv, const float* fu, const float* fv,
                        const float* mp, const float* mf, int w, int h, const dco_config* c,
                        float* out) {
    return guarded([&] {
        FlowField past(w, h), future(w, h);
        size_t n = static_cast<size_t>(w) * h;
        std::memcpy(past.u.data(), pu, 4 * n);
        std::memcpy(past.v.data(), pv, 4 * n);
        std::memcpy(future.u.data(), fu, 4 * n);
        std::memcpy(future.v.data(), fv, 4 * n);
        copy_out(fuse_amplitudes(past, future, map_in(mp, w, h), map_in(mf, w, h), to_cfg(c)).data,
                 out);
    });
}

// box_filter, contour.cpp:108-136.
int ref_box_filter(const float* amp, int w, int h, int radius, float* out) {
    return guarded([&] { copy_out(box_filter(map_in(amp, w, h), radius).data, out); });
}

// normalize_amplitude, contour.cpp:138-147.
int ref_normalize_amplitude(const float* amp, int w, int h, float* out) {
    return guarded([&] { copy_out(normalize_amplitude(map_in(amp, w, h)).data, out); });
}

// gaussian_blur, contour.cpp:149-175.
int ref_gaussian_blur(const float* img, int w, int h, double sigma, float* out) {
    return guarded([&] { copy_out(gaussian_blur(gray_in(img, w, h), sigma).data, out); });
}

// extract_depth_contours_prefiltered, contour.cpp:177-279.
int ref_extract_depth_contours_prefiltered(const float* blurred, int w, int h, const float* mf,
                                           int qw, int qh, const dco_config* c, uint8_t* edges,
                                           float* m_i) {
    return guarded([&] {
        ContourResult r =
            extract_depth_contours_prefiltered(gray_in(blurred, w, h), map_in(mf, qw, qh), to_cfg(c));
        copy_out(r.edges.data, edges);
        copy_out(r.m_i.data, m_i);
    });
}

// smoothness_weight, densify.cpp:26-35.
int ref_smoothness_weight(int px, int py, int qx, int qy, const uint8_t* edges, int w, int h,
                          const float* mf, int qw, int qh, const float* m_i, double* out) {
    return guarded([&] {
        *out = smoothness_weight(px, py, qx, qy, mask_in(edges, w, h), map_in(mf, qw, qh),
                                 map_in(m_i, w, h));
    });
}

// assemble_system, densify.cpp:37-116. d_pre may be NULL.
int ref_assemble_system(const float* sparse, const uint8_t* edges, const float* mf, int qw, int qh,
                        const float* m_i, const float* d_pre, int w, int h, const dco_config* c,
                        double* diag, double* ch, double* cv, double* rhs, double* initial,
                        uint8_t* anchored, double* constant_term, uint64_t* anchor_count) {
    return guarded([&] {
        FloatMap pre;
        if (d_pre) pre = map_in(d_pre, w, h);
        ConstraintSystem s = assemble_system(map_in(sparse, w, h), mask_in(edges, w, h),
                                             map_in(mf, qw, qh), map_in(m_i, w, h),
                                             d_pre ? &pre : nullptr, to_cfg(c));
        copy_out(s.diag, diag);
        copy_out(s.coup_h, ch);
        copy_out(s.coup_v, cv);
        copy_out(s.rhs, rhs);
        copy_out(s.initial, initial);
        copy_out(s.anchored, anchored);
        *constant_term = s.constant_term;
        *anchor_count = s.anchor_count;
    });
}

// apply_system, densify.cpp:118-133.
int ref_apply_system(int w, int h, const double* diag, const double* ch, const double* cv,
                     const double* x, double* out) {
    return guarded([&] {
        size_t n = static_cast<size_t>(w) * h;
        std::vector<uint8_t> none(n, 0);
        std::vector<double> zero(n, 0.0);
        ConstraintSystem s = sys_in(w, h, diag, ch, cv, zero.data(), zero.data(), none.data(), 0.0);
        std::vector<double> xv(x, x + n), o;
        apply_system(s, xv, o);
        copy_out(o, out);
    });
}

// solve_dense_depth, densify.cpp:141-222 (+ SolveStats, densify.hpp:50-56).
int ref_solve_dense_depth(int w, int h, const double* diag, const double* ch, const double* cv,
                          const double* rhs, const double* initial, const uint8_t* anchored,
                          double constant_term, const dco_config* c, float* dense, int* iterations,
                          double* relative_residual, double* obj_initial, double* obj_final,
                          double* history, int history_cap) {
    return guarded([&] {
        ConstraintSystem s = sys_in(w, h, diag, ch, cv, rhs, initial, anchored, constant_term);
        SolveStats st;
        FloatMap d = solve_dense_depth(s, to_cfg(c), &st);
        copy_out(d.data, dense);
        if (iterations) *iterations = st.iterations;
        if (relative_residual) *relative_residual = st.relative_residual;
        if (obj_initial) *obj_initial = st.objective_initial;
        if (obj_final) *obj_final = st.objective_final;
        if (history)
            for (int i = 0; i < history_cap && i < static_cast<int>(st.residual_history.size()); ++i)
                history[i] = st.residual_history[i];
    });
}

// composite, occlude.cpp:171-194.
int ref_composite(const float* real, const float* dense, const float* vrgb, const float* vdepth,
                  int w, int h, float* out_rgb, uint8_t* mask) {
    return guarded([&] {
        ColorImage r(w, h);
        std::memcpy(r.data.data(), real, sizeof(float) * r.data.size());
        VirtualLayer v;
        v.color = ColorImage(w, h);
        std::memcpy(v.color.data.data(), vrgb, sizeof(float) * v.color.data.size());
        v.depth = map_in(vdepth, w, h);
        CompositeResult res = composite(r, map_in(dense, w, h), v);
        copy_out(res.color.data, out_rgb);
        copy_out(res.mask.data, mask);
    });
}

// make_cube_mesh + render_virtual (occlude.cpp:89-169): the composite's input
// generator (render_virtual is outside the hot path).
int ref_render_cube(float cx, float cy, float cz, float side, double focal_px, int w, int h,
                    float* vrgb, float* vdepth) {
    return guarded([&] {
        TriangleMesh m = make_cube_mesh(cx, cy, cz, side);
        VirtualLayer v = render_virtual(m, focal_px, w / 2.0, h / 2.0, w, h);
        copy_out(v.color.data, vrgb);
        copy_out(v.depth.data, vdepth);
    });
}

// transform_mesh + render_virtual (occlude.cpp:78-169) on an arbitrary mesh:
// vertices / colours are nv x 3 floats, triangles nt x 3 ints; pose (16
// doubles, row-major) may be NULL (no transform, pipeline.cpp:249-250).
int ref_render_virtual(const float* verts, int nv, const int* tris, int nt, const float* colors,
                       const double* pose, double focal_px, double cx, double cy, int w, int h, float* vrgb,
                       float* vdepth) {
    return guarded([&] {
        TriangleMesh m;
        for (int i = 0; i < nv; ++i) {
            m.vertices.push_back({verts[3 * i], verts[3 * i + 1], verts[3 * i + 2]});
            m.colors.push_back({colors[3 * i], colors[3 * i + 1], colors[3 * i + 2]});
        }
        for (int t = 0; t < nt; ++t) m.triangles.push_back({tris[3 * t], tris[3 * t + 1], tris[3 * t + 2]});
        if (pose) {
            std::array<double, 16> p;
            for (int i = 0; i < 16; ++i) p[i] = pose[i];
            m = transform_mesh(m, p);
        }
        VirtualLayer v = render_virtual(m, focal_px, cx, cy, w, h);
        copy_out(v.color.data, vrgb);
        copy_out(v.depth.data, vdepth);
    });
}

int ref_transform_mesh(const float* verts, int nv, const double* pose, float* out) {
    return guarded([&] {
        TriangleMesh m;
        for (int i = 0; i < nv; ++i) {
            m.vertices.push_back({verts[3 * i], verts[3 * i + 1], verts[3 * i + 2]});
            m.colors.push_back({0.0f, 0.0f, 0.0f});
        }
        std::array<double, 16> p;
        for (int i = 0; i < 16; ++i) p[i] = pose[i];
        TriangleMesh o = transform_mesh(m, p);
        for (int i = 0; i < nv; ++i)
            for (int k = 0; k < 3; ++k) out[3 * i + k] = o.vertices[i][k];
    });
}

// One composited frame of run_pipeline (pipeline.cpp:183-258) on in-memory
// inputs: past/middle/future quarter lefts, the middle's full gray, quarter
// right, colour, optional previous dense map and virtual layer. Outputs: dense
// (full), composite RGB, mask, edges; iterations/objective. Used for the CPU
// baseline and end-to-end parity. Returns DCO_UNSOLVABLE when densify throws
// (dense then holds the fallback, as pipeline.cpp:236-242 does).
int ref_pipeline_frame(int fw, int fh, const float* past_q, const float* mid_q,
                       const float* future_q, const float* mid_gray, const float* right_q,
                       const float* mid_rgb, const float* d_pre, const float* vrgb,
                       const float* vdepth, const dco_config* c, float* dense_out,
                       float* composite_out, uint8_t* mask_out, uint8_t* edges_out,
                       float* sparse_out, int* iterations, double* objective) {
    return guarded([&] {
        PipelineConfig cfg = to_cfg(c);
        const int qw = fw / 2, qh = fh / 2;
        GrayImage past = gray_in(past_q, qw, qh), mid = gray_in(mid_q, qw, qh),
                  fut = gray_in(future_q, qw, qh), gray = gray_in(mid_gray, fw, fh),
                  right = gray_in(right_q, qw, qh);
        CrossWindowField cross = build_cross_windows(mid, cfg);
        CostVolume vol = compute_cost_volume(mid, right, cross, cfg);
        DisparityMap disp = select_disparity_wta(aggregate_costs(vol, cross));
        disp = refine_disparity_histogram(disp, cross, cfg.hist_iterations);
        SparseDepthMap sparse = disparity_to_sparse_depth(disp, cfg, fw, fh);
        FlowField fp = compute_flow(mid, past, cfg);
        FlowField ff = compute_flow(mid, fut, cfg);
        AmplitudeMap mp = gradient_amplitude(flow_to_polar(fp));
        AmplitudeMap mfut = gradient_amplitude(flow_to_polar(ff));
        AmplitudeMap fused = fuse_amplitudes(fp, ff, mp, mfut, cfg);
        fused = normalize_amplitude(box_filter(fused, cfg.box_radius));
        GrayImage blurred = gaussian_blur(gray, cfg.gauss_sigma);
        ContourResult cont = extract_depth_contours_prefiltered(blurred, fused, cfg);
        FloatMap pre;
        if (d_pre) pre = map_in(d_pre, fw, fh);
        FloatMap dense;
        bool unsolvable = false;
        try {
            ConstraintSystem sys =
                assemble_system(sparse, cont.edges, fused, cont.m_i, d_pre ? &pre : nullptr, cfg);
            SolveStats st;
            dense = solve_dense_depth(sys, cfg, &st);
            if (iterations) *iterations = st.iterations;
            if (objective) *objective = st.objective_final;
        } catch (const UnsolvableFrameError&) {
            unsolvable = true;
            dense = d_pre ? pre : FloatMap(fw, fh);
        }
        ColorImage real(fw, fh);
        std::memcpy(real.data.data(), mid_rgb, sizeof(float) * real.data.size());
        CompositeResult comp;
        if (vrgb && vdepth) {
            VirtualLayer v;
            v.color = ColorImage(fw, fh);
            std::memcpy(v.color.data.data(), vrgb, sizeof(float) * v.color.data.size());
            v.depth = map_in(vdepth, fw, fh);
            comp = composite(real, dense, v);
        } else {
            comp.color = real;
            comp.mask = OcclusionMask(fw, fh, 0);
        }
        if (dense_out) copy_out(dense.data, dense_out);
        if (composite_out) copy_out(comp.color.data, composite_out);
        if (mask_out) copy_out(comp.mask.data, mask_out);
        if (edges_out) copy_out(cont.edges.data, edges_out);
        if (sparse_out) copy_out(sparse.data, sparse_out);
        if (unsolvable) throw UnsolvableFrameError("solve_dense_depth: no anchored pixel");
    });
}

// run_pipeline (pipeline.cpp:108-321), the reference's own public frame loop:
// config file, manifest of PGM frames with per-frame poses, OBJ mesh, outputs
// under out_dir. Per composited frame (in index order, at most cap): the 14
// StageTimings values + the frame total (15 doubles, pipeline.cpp:57-82) into
// stage_ms, the CG iteration count into iterations and the frame index into
// index. *n = number of composited frames.
int ref_run_pipeline(const char* config_path, const char* manifest, const char* out_dir, const char* mesh_path,
                     int cap, double* stage_ms, int* iterations, int* index, int* n) {
    return guarded([&] {
        RunOptions o;
        o.config_path = config_path ? config_path : "";
        o.manifest_path = manifest;
        o.output_dir = out_dir;
        o.mesh_path = mesh_path ? mesh_path : "";
        RunSummary sum = run_pipeline(o);
        int k = 0;
        for (const FrameResult& f : sum.frames) {
            if (!f.composited || k >= cap) continue;
            std::vector<double> v = f.timings.stage_values();
            for (size_t i = 0; i < v.size(); ++i) stage_ms[15 * k + i] = v[i];
            stage_ms[15 * k + 14] = f.timings.total;
            iterations[k] = f.densify_iterations;
            index[k] = f.index;
            ++k;
        }
        *n = k;
    });
}

// format_bench_report / write_bench_csv (pipeline.cpp:366-391) of a report
// whose 14 rows carry the StageTimings::stage_names() (pipeline.cpp:57-75) and
// whose total is "frame processing"; mmm = 15 x (mean, min, max). The text goes
// to out (NUL-terminated, truncated to cap); csv_path may be NULL.
int ref_format_bench_report(int repetitions, const double* mmm, char* out, size_t cap, const char* csv_path) {
    return guarded([&] {
        BenchReport r;
        r.repetitions = repetitions;
        const auto& names = StageTimings::stage_names();
        for (size_t i = 0; i < names.size(); ++i)
            r.rows.push_back({names[i], mmm[3 * i], mmm[3 * i + 1], mmm[3 * i + 2]});
        r.total = {"frame processing", mmm[3 * 14], mmm[3 * 14 + 1], mmm[3 * 14 + 2]};
        std::string text = format_bench_report(r);
        std::strncpy(out, text.c_str(), cap - 1);
        out[cap - 1] = 0;
        if (csv_path) write_bench_csv(r, csv_path);
    });
}

} // extern "C"
