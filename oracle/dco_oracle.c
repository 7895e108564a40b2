/* dco_oracle.c — plain-C restatement of the reference DCO hot path.
 * TEST INFRASTRUCTURE ONLY; see dco_oracle.h. Built without -march and with
 * -ffp-contract=off so its float/double arithmetic rounds exactly like the
 * reference's Release build; libm calls (exp, hypot, hypotf, atan2f) are the
 * host's, as in the reference. Reference file:line citations are relative to
 * /root/reference/proj. */
#include "dco_oracle.h"

#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

static char g_msg[256];

static int err(int status, const char* msg) {
    snprintf(g_msg, sizeof g_msg, "%s", msg);
    return status;
}

const char* dco_o_error(void) { return g_msg; }

#define NODATA ((float)NAN)
#define IDX(x, y, w) ((size_t)(y) * (size_t)(w) + (size_t)(x))

static int clampi(int v, int lo, int hi) { return v < lo ? lo : (v > hi ? hi : v); }
/* std::clamp(v, lo, hi) for floats: NaN and signed zeros pass through */
static float clampf_std(float v, float lo, float hi) { return v < lo ? lo : (hi < v ? hi : v); }
static float maxf_std(float a, float b) { return a < b ? b : a; } /* std::max */

/* PipelineConfig::validate, src/config.cpp:10-36 */
int dco_o_validate(const dco_config* c) {
    if (c->d_min >= c->d_max) return err(DCO_CONFIG, "config: d_min must be below d_max");
    if (c->t_low < 0.0 || c->t_low >= c->t_high || c->t_high > 1.0)
        return err(DCO_CONFIG, "config: need 0 <= t_low < t_high <= 1");
    if (c->t_depth < 0.0 || c->t_depth > 1.0) return err(DCO_CONFIG, "config: t_depth outside [0,1]");
    if (c->lambda_ad <= 0.0 || c->lambda_census <= 0.0 || c->lambda_d <= 0.0 || c->lambda_s <= 0.0 ||
        c->lambda_s2 <= 0.0)
        return err(DCO_CONFIG, "config: every lambda must be positive");
    if (c->gamma_l <= 0.0 || c->epsilon <= 0.0)
        return err(DCO_CONFIG, "config: gamma_l and epsilon must be positive");
    if (c->census_window_w % 2 == 0 || c->census_window_h % 2 == 0)
        return err(DCO_CONFIG, "config: census window dimensions must be odd");
    if (c->census_window_w < 1 || c->census_window_h < 1 || c->census_window_w * c->census_window_h - 1 > 64)
        return err(DCO_CONFIG, "config: census window must fit 64 bits");
    if (c->cross_arm_l1 < 1 || c->cross_arm_l2 < 1 || c->cross_arm_l2 > c->cross_arm_l1)
        return err(DCO_CONFIG, "config: need 1 <= cross_arm_l2 <= cross_arm_l1");
    if (c->cross_color_tau <= 0.0 || c->cross_color_tau2 <= 0.0)
        return err(DCO_CONFIG, "config: color thresholds must be positive");
    if (c->box_radius < 1) return err(DCO_CONFIG, "config: box_radius must be >= 1");
    if (c->gauss_sigma <= 0.0) return err(DCO_CONFIG, "config: gauss_sigma must be positive");
    if (c->confidence_offset_k <= 0.0) return err(DCO_CONFIG, "config: confidence_offset_k must be positive");
    if (c->hist_iterations < 0) return err(DCO_CONFIG, "config: hist_iterations must be >= 0");
    if (c->focal_px <= 0.0 || c->baseline_m <= 0.0)
        return err(DCO_CONFIG, "config: focal_px and baseline_m must be positive");
    if (c->solver_tol <= 0.0 || c->solver_max_iter < 1)
        return err(DCO_CONFIG, "config: solver_tol must be positive, solver_max_iter >= 1");
    if (c->d_min < 0) return err(DCO_CONFIG, "config: d_min must be >= 0");
    return DCO_OK;
}

/* ---------------------------------------------------------------- pyramid */
/* downsample_half, src/pyramid.cpp:5-17 */
int dco_o_downsample_half(const float* img, int w, int h, float* out) {
    if (w < 2 || h < 2) return err(DCO_INPUT, "downsample_half: dimensions must be at least 2x2");
    int ow = w / 2, oh = h / 2;
    for (int y = 0; y < oh; ++y)
        for (int x = 0; x < ow; ++x) {
            const float* a = img + IDX(2 * x, 2 * y, w);
            float s = a[0] + a[1];
            s = s + a[w];
            s = s + a[w + 1];
            out[IDX(x, y, ow)] = s * 0.25f;
        }
    return DCO_OK;
}

/* ----------------------------------------------------------------- stereo */
/* grow_arm, src/stereo.cpp:14-26 */
static int arm_reach(const float* img, int w, int h, int x, int y, int sx, int sy, const dco_config* c) {
    float mid = img[IDX(x, y, w)];
    int reach = 0;
    for (int step = 1; step <= c->cross_arm_l1; ++step) {
        int qx = x + step * sx, qy = y + step * sy;
        if (qx < 0 || qy < 0 || qx >= w || qy >= h) break;
        double limit = step <= c->cross_arm_l2 ? c->cross_color_tau : c->cross_color_tau2;
        if ((double)fabsf(img[IDX(qx, qy, w)] - mid) >= limit) break;
        reach = step;
    }
    return reach;
}

/* smooth_arm_channel, src/stereo.cpp:30-48: 5th smallest of the clamped 3x3
 * neighbourhood (what nth_element(.., +4, ..) leaves at index 4), then min
 * with the unsmoothed arm */
static void median_clamp(uint8_t* arm, int w, int h) {
    size_t n = (size_t)w * h;
    uint8_t* raw = malloc(n);
    memcpy(raw, arm, n);
    for (int y = 0; y < h; ++y)
        for (int x = 0; x < w; ++x) {
            int hist[256] = {0};
            for (int dy = -1; dy <= 1; ++dy)
                for (int dx = -1; dx <= 1; ++dx) hist[raw[IDX(clampi(x + dx, 0, w - 1), clampi(y + dy, 0, h - 1), w)]]++;
            int seen = 0, med = 0;
            for (int v = 0; v < 256; ++v) {
                seen += hist[v];
                if (seen >= 5) {
                    med = v;
                    break;
                }
            }
            uint8_t r = raw[IDX(x, y, w)];
            arm[IDX(x, y, w)] = (uint8_t)(med < r ? med : r);
        }
    free(raw);
}

/* build_cross_windows, src/stereo.cpp:52-68 */
int dco_o_cross_windows(const float* img, int w, int h, const dco_config* c, uint8_t* l, uint8_t* r, uint8_t* u,
                        uint8_t* d) {
    for (int y = 0; y < h; ++y)
        for (int x = 0; x < w; ++x) {
            size_t i = IDX(x, y, w);
            l[i] = (uint8_t)arm_reach(img, w, h, x, y, -1, 0, c);
            r[i] = (uint8_t)arm_reach(img, w, h, x, y, 1, 0, c);
            u[i] = (uint8_t)arm_reach(img, w, h, x, y, 0, -1, c);
            d[i] = (uint8_t)arm_reach(img, w, h, x, y, 0, 1, c);
        }
    median_clamp(l, w, h);
    median_clamp(r, w, h);
    median_clamp(u, w, h);
    median_clamp(d, w, h);
    return DCO_OK;
}

/* census_transform, src/stereo.cpp:70-96 */
int dco_o_census(const float* img, int w, int h, int ww, int wh, uint64_t* out) {
    if (ww % 2 == 0 || wh % 2 == 0) return err(DCO_CONFIG, "census_transform: window dimensions must be odd");
    if (ww * wh - 1 > 64) return err(DCO_CONFIG, "census_transform: window exceeds 64 comparison bits");
    for (int y = 0; y < h; ++y)
        for (int x = 0; x < w; ++x) {
            float mid = img[IDX(x, y, w)];
            uint64_t code = 0;
            for (int dy = -(wh / 2); dy <= wh / 2; ++dy)
                for (int dx = -(ww / 2); dx <= ww / 2; ++dx) {
                    if (!dx && !dy) continue;
                    float q = img[IDX(clampi(x + dx, 0, w - 1), clampi(y + dy, 0, h - 1), w)];
                    code = (code << 1) | (uint64_t)(q < mid);
                }
            out[IDX(x, y, w)] = code;
        }
    return DCO_OK;
}

/* compute_cost_volume, src/stereo.cpp:106-150 (adaptive_alpha :102-104) */
int dco_o_cost_volume(const float* left, const float* right, int w, int h, const uint8_t* l, const uint8_t* r,
                      const uint8_t* u, const uint8_t* d, const dco_config* c, float* cost) {
    int st = dco_o_validate(c);
    if (st) return st;
    size_t n = (size_t)w * h;
    uint64_t* cl = malloc(n * 8);
    uint64_t* cr = malloc(n * 8);
    st = dco_o_census(left, w, h, c->census_window_w, c->census_window_h, cl);
    if (!st) st = dco_o_census(right, w, h, c->census_window_w, c->census_window_h, cr);
    if (st) {
        free(cl);
        free(cr);
        return st;
    }
    int bits = c->census_window_w * c->census_window_h - 1;
    double tc[65];
    for (int k = 0; k <= bits; ++k) tc[k] = 1.0 - exp(-(double)k / c->lambda_census);
    int nd = c->d_max - c->d_min + 1;
    for (int y = 0; y < h; ++y)
        for (int x = 0; x < w; ++x) {
            size_t i = IDX(x, y, w);
            int m = l[i];
            if (r[i] < m) m = r[i];
            if (u[i] < m) m = u[i];
            if (d[i] < m) m = d[i];
            double alpha = 1.0 - exp(-c->gamma_l / ((double)m + c->epsilon));
            float* out = cost + i * nd;
            for (int k = 0; k < nd; ++k) {
                int qx = x - (c->d_min + k);
                if (qx < 0) {
                    out[k] = 2.0f;
                    continue;
                }
                size_t j = IDX(qx, y, w);
                double ad = (double)fabsf(left[i] - right[j]) * 255.0;
                double t_ad = 1.0 - exp(-ad / c->lambda_ad);
                int hd = __builtin_popcountll(cl[i] ^ cr[j]);
                out[k] = (float)(alpha * t_ad + (1.0 - alpha) * tc[hd]);
            }
        }
    free(cl);
    free(cr);
    return DCO_OK;
}

/* aggregate_costs, src/stereo.cpp:152-218: per slice, sequential double row
 * prefixes, hsum = P[x+right+1] - P[x-left]; then sequential column prefixes of
 * hsum, total = C[y+down+1] - C[y-up]; out = float(total / region_size). */
int dco_o_aggregate(const float* cost, int w, int h, int nd, const uint8_t* l, const uint8_t* r, const uint8_t* u,
                    const uint8_t* d, float* out) {
    size_t n = (size_t)w * h;
    int* region = malloc(n * sizeof(int));
    for (int y = 0; y < h; ++y)
        for (int x = 0; x < w; ++x) {
            int s = 0;
            for (int yy = y - u[IDX(x, y, w)]; yy <= y + d[IDX(x, y, w)]; ++yy) s += l[IDX(x, yy, w)] + r[IDX(x, yy, w)] + 1;
            region[IDX(x, y, w)] = s;
        }
    double* pre = malloc(sizeof(double) * (size_t)((w > h ? w : h) + 1));
    double* hs = malloc(sizeof(double) * n);
    for (int k = 0; k < nd; ++k) {
        for (int y = 0; y < h; ++y) {
            pre[0] = 0.0;
            for (int x = 0; x < w; ++x) pre[x + 1] = pre[x] + (double)cost[IDX(x, y, w) * nd + k];
            for (int x = 0; x < w; ++x) {
                size_t i = IDX(x, y, w);
                hs[i] = pre[x + r[i] + 1] - pre[x - l[i]];
            }
        }
        for (int x = 0; x < w; ++x) {
            pre[0] = 0.0;
            for (int y = 0; y < h; ++y) pre[y + 1] = pre[y] + hs[IDX(x, y, w)];
            for (int y = 0; y < h; ++y) {
                size_t i = IDX(x, y, w);
                double total = pre[y + d[i] + 1] - pre[y - u[i]];
                out[i * nd + k] = (float)(total / region[i]);
            }
        }
    }
    free(pre);
    free(hs);
    free(region);
    return DCO_OK;
}

/* select_disparity_wta, src/stereo.cpp:220-238 */
int dco_o_wta(const float* cost, int w, int h, int d_min, int nd, float* disp) {
    for (size_t i = 0; i < (size_t)w * h; ++i) {
        const float* cv = cost + i * nd;
        int arg = 0;
        for (int k = 1; k < nd; ++k)
            if (cv[k] < cv[arg]) arg = k;
        disp[i] = (float)(d_min + arg);
    }
    return DCO_OK;
}

/* refine_disparity_histogram, src/stereo.cpp:240-299 */
int dco_o_refine(const float* disp, int w, int h, const uint8_t* l, const uint8_t* r, const uint8_t* u,
                 const uint8_t* d, int iters, float* out) {
    size_t n = (size_t)w * h;
    long top = 0;
    for (size_t i = 0; i < n; ++i)
        if (isfinite(disp[i]) && lroundf(disp[i]) > top) top = lroundf(disp[i]);
    int* counts = calloc((size_t)top + 1, sizeof(int));
    float* cur = malloc(n * 4);
    memcpy(cur, disp, n * 4);
    float* nxt = malloc(n * 4);
    for (int it = 0; it < iters; ++it) {
        memcpy(nxt, cur, n * 4);
        for (int y = 0; y < h; ++y)
            for (int x = 0; x < w; ++x) {
                size_t i = IDX(x, y, w);
                if (!isfinite(cur[i])) continue;
                int members = 0, lo = (int)top, hi = 0;
                for (int yy = y - u[i]; yy <= y + d[i]; ++yy) {
                    size_t vi = IDX(x, yy, w);
                    for (int xx = x - l[vi]; xx <= x + r[vi]; ++xx) {
                        float v = cur[IDX(xx, yy, w)];
                        if (!isfinite(v)) continue;
                        int b = (int)lroundf(v);
                        counts[b]++;
                        members++;
                        if (b < lo) lo = b;
                        if (b > hi) hi = b;
                    }
                }
                int mode = lo, best = 0;
                for (int b = lo; b <= hi; ++b) {
                    if (counts[b] > best) {
                        best = counts[b];
                        mode = b;
                    }
                    counts[b] = 0;
                }
                nxt[i] = (best == 1 && members >= 4) ? NODATA : (float)mode;
            }
        float* t = cur;
        cur = nxt;
        nxt = t;
    }
    memcpy(out, cur, n * 4);
    free(cur);
    free(nxt);
    free(counts);
    return DCO_OK;
}

/* disparity_to_sparse_depth, src/stereo.cpp:301-315 */
int dco_o_sparse_depth(const float* disp, int w, int h, const dco_config* c, int fw, int fh, float* out) {
    if (fw < 2 * w || fh < 2 * h)
        return err(DCO_INPUT, "disparity_to_sparse_depth: full dimensions too small for the quarter map");
    for (size_t i = 0; i < (size_t)fw * fh; ++i) out[i] = NODATA;
    for (int y = 0; y < h; ++y)
        for (int x = 0; x < w; ++x) {
            float v = disp[IDX(x, y, w)];
            if (!isfinite(v)) continue;
            double full = 2.0 * v;
            if (full <= 0.0) continue;
            out[IDX(2 * x, 2 * y, fw)] = (float)(c->focal_px * c->baseline_m / full);
        }
    return DCO_OK;
}

/* ------------------------------------------------------------------- flow */
/* sample_bilinear, src/image.cpp:27-39 */
static float bilerp(const float* img, int w, int h, float x, float y) {
    x = clampf_std(x, 0.0f, (float)(w - 1));
    y = clampf_std(y, 0.0f, (float)(h - 1));
    int x0 = (int)x, y0 = (int)y;
    int x1 = x0 + 1 < w ? x0 + 1 : w - 1, y1 = y0 + 1 < h ? y0 + 1 : h - 1;
    float fx = x - (float)x0, fy = y - (float)y0;
    float a = img[IDX(x0, y0, w)] * (1.0f - fx) + img[IDX(x1, y0, w)] * fx;
    float b = img[IDX(x0, y1, w)] * (1.0f - fx) + img[IDX(x1, y1, w)] * fx;
    return a * (1.0f - fy) + b * fy;
}

/* patch_positions, src/flow.cpp:29-35 */
static int patch_grid(int extent, int* pos) {
    int last = extent - 8, n = 0;
    for (int p = 0; p <= last; p += 4) pos[n++] = p;
    if (n == 0 || pos[n - 1] != last) pos[n++] = last > 0 ? last : 0;
    return n;
}

/* search_patch, src/flow.cpp:72-121 */
static void patch_search(const float* from, const float* to, int w, int h, int px, int py, float su, float sv,
                         float* ou, float* ov, float* ow) {
    float tpl[64], gxs[64], gys[64];
    double a00 = 1e-6, a01 = 0.0, a11 = 1e-6;
    for (int k = 0; k < 64; ++k) {
        int x = px + (k & 7), y = py + (k >> 3);
        tpl[k] = from[IDX(x, y, w)];
        gxs[k] = 0.5f * (from[IDX(clampi(x + 1, 0, w - 1), y, w)] - from[IDX(clampi(x - 1, 0, w - 1), y, w)]);
        gys[k] = 0.5f * (from[IDX(x, clampi(y + 1, 0, h - 1), w)] - from[IDX(x, clampi(y - 1, 0, h - 1), w)]);
        a00 += (double)gxs[k] * gxs[k];
        a01 += (double)gxs[k] * gys[k];
        a11 += (double)gys[k] * gys[k];
    }
    double det = a00 * a11 - a01 * a01;
    double i00 = a11 / det, i01 = -a01 / det, i11 = a00 / det;
    float u = su, v = sv;
    double err2 = 0.0;
    for (int it = 0; it < 12; ++it) {
        double eu = 0.0, ev = 0.0, e2 = 0.0;
        for (int k = 0; k < 64; ++k) {
            float res = bilerp(to, w, h, (float)(px + (k & 7)) + u, (float)(py + (k >> 3)) + v) - tpl[k];
            eu += (double)gxs[k] * res;
            ev += (double)gys[k] * res;
            e2 += (double)res * res;
        }
        err2 = e2 / 64;
        double du = i00 * eu + i01 * ev, dv = i01 * eu + i11 * ev;
        u -= (float)du;
        v -= (float)dv;
        if (!isfinite(u) || !isfinite(v)) {
            u = su;
            v = sv;
            break;
        }
        u = clampf_std(u, (float)-w, (float)w);
        v = clampf_std(v, (float)-h, (float)h);
        if (du * du + dv * dv < 1e-6) break;
    }
    *ou = u;
    *ov = v;
    *ow = (float)(1.0 / (err2 + 1e-2));
}

/* estimate_level, src/flow.cpp:123-181 */
static void flow_level(const float* from, const float* to, int w, int h, const float* iu, const float* iv,
                       float* ou, float* ov) {
    int* xs = malloc(sizeof(int) * (w / 4 + 3));
    int* ys = malloc(sizeof(int) * (h / 4 + 3));
    int nx = patch_grid(w, xs), ny = patch_grid(h, ys);
    size_t n = (size_t)w * h;
    double* su = calloc(n, sizeof(double));
    double* sv = calloc(n, sizeof(double));
    double* sw = calloc(n, sizeof(double));
    for (int a = 0; a < ny; ++a)
        for (int b = 0; b < nx; ++b) {
            int px = xs[b], py = ys[a];
            int cx = px + 4 < w - 1 ? px + 4 : w - 1, cy = py + 4 < h - 1 ? py + 4 : h - 1;
            float pu, pv, pw;
            patch_search(from, to, w, h, px, py, iu[IDX(cx, cy, w)], iv[IDX(cx, cy, w)], &pu, &pv, &pw);
            for (int dy = 0; dy < 8 && py + dy < h; ++dy)
                for (int dx = 0; dx < 8 && px + dx < w; ++dx) {
                    size_t i = IDX(px + dx, py + dy, w);
                    su[i] += (double)pw * pu;
                    sv[i] += (double)pw * pv;
                    sw[i] += pw;
                }
        }
    for (size_t i = 0; i < n; ++i) {
        ou[i] = sw[i] > 0.0 ? (float)(su[i] / sw[i]) : 0.0f;
        ov[i] = sw[i] > 0.0 ? (float)(sv[i] / sw[i]) : 0.0f;
    }
    /* nearest covered pixel for uncovered ones (flow.cpp:162-180) */
    for (int y = 0; y < h; ++y)
        for (int x = 0; x < w; ++x) {
            if (sw[IDX(x, y, w)] > 0.0) continue;
            int done = 0;
            for (int rad = 1; rad < (w > h ? w : h) && !done; ++rad)
                for (int dy = -rad; dy <= rad && !done; ++dy)
                    for (int dx = -rad; dx <= rad && !done; ++dx) {
                        int qx = x + dx, qy = y + dy;
                        if (qx < 0 || qy < 0 || qx >= w || qy >= h || !(sw[IDX(qx, qy, w)] > 0.0)) continue;
                        ou[IDX(x, y, w)] = ou[IDX(qx, qy, w)];
                        ov[IDX(x, y, w)] = ov[IDX(qx, qy, w)];
                        done = 1;
                    }
        }
    free(xs);
    free(ys);
    free(su);
    free(sv);
    free(sw);
}

/* upsample_flow, src/flow.cpp:39-62 */
static void flow_up(const float* cu, const float* cv, int cw, int chh, float* fu, float* fv, int fw, int fh) {
    for (int y = 0; y < fh; ++y) {
        float sy = clampf_std(((float)y + 0.5f) * 0.5f - 0.5f, 0.0f, (float)(chh - 1));
        int y0 = (int)sy, y1 = y0 + 1 < chh ? y0 + 1 : chh - 1;
        float ty = sy - (float)y0;
        for (int x = 0; x < fw; ++x) {
            float sx = clampf_std(((float)x + 0.5f) * 0.5f - 0.5f, 0.0f, (float)(cw - 1));
            int x0 = (int)sx, x1 = x0 + 1 < cw ? x0 + 1 : cw - 1;
            float tx = sx - (float)x0;
            const float* comp[2] = {cu, cv};
            float* dst[2] = {fu, fv};
            for (int c = 0; c < 2; ++c) {
                const float* s = comp[c];
                float a = s[IDX(x0, y0, cw)] * (1 - tx) + s[IDX(x1, y0, cw)] * tx;
                float b = s[IDX(x0, y1, cw)] * (1 - tx) + s[IDX(x1, y1, cw)] * tx;
                dst[c][IDX(x, y, fw)] = 2.0f * (a * (1 - ty) + b * ty);
            }
        }
    }
}

/* compute_flow, src/flow.cpp:185-205 (build_pyramid, src/pyramid.cpp:19-33) */
int dco_o_flow(const float* from, const float* to, int w, int h, float* u, float* v) {
    if (w < 8 || h < 8) return err(DCO_INPUT, "compute_flow: frames smaller than the patch size");
    int nlev = 1;
    while ((w < h ? w : h) / (1 << nlev) >= 16) ++nlev;
    const float* pf[16];
    const float* pt[16];
    int lw[16], lh[16];
    float* owned[32];
    int no = 0;
    pf[0] = from;
    pt[0] = to;
    lw[0] = w;
    lh[0] = h;
    for (int i = 1; i < nlev; ++i) {
        lw[i] = lw[i - 1] / 2;
        lh[i] = lh[i - 1] / 2;
        float* a = malloc((size_t)lw[i] * lh[i] * 4);
        float* b = malloc((size_t)lw[i] * lh[i] * 4);
        dco_o_downsample_half(pf[i - 1], lw[i - 1], lh[i - 1], a);
        dco_o_downsample_half(pt[i - 1], lw[i - 1], lh[i - 1], b);
        pf[i] = a;
        pt[i] = b;
        owned[no++] = a;
        owned[no++] = b;
    }
    size_t cap = (size_t)w * h;
    float* fu = calloc(cap, 4);
    float* fv = calloc(cap, 4);
    float* gu = calloc(cap, 4);
    float* gv = calloc(cap, 4);
    for (int lev = nlev - 1; lev >= 0; --lev) {
        if (lev != nlev - 1) {
            flow_up(fu, fv, lw[lev + 1], lh[lev + 1], gu, gv, lw[lev], lh[lev]);
            float* t = fu;
            fu = gu;
            gu = t;
            t = fv;
            fv = gv;
            gv = t;
        }
        flow_level(pf[lev], pt[lev], lw[lev], lh[lev], fu, fv, gu, gv);
        float* t = fu;
        fu = gu;
        gu = t;
        t = fv;
        fv = gv;
        gv = t;
    }
    memcpy(u, fu, cap * 4);
    memcpy(v, fv, cap * 4);
    free(fu);
    free(fv);
    free(gu);
    free(gv);
    for (int i = 0; i < no; ++i) free(owned[i]);
    return DCO_OK;
}

/* ---------------------------------------------------------------- contour */
/* flow_to_polar, src/contour.cpp:10-25 */
int dco_o_polar(const float* u, const float* v, int n, float* r, float* theta) {
    for (int i = 0; i < n; ++i) {
        r[i] = hypotf(u[i], v[i]);
        if (theta) {
            float t = atan2f(v[i], u[i]);
            theta[i] = t <= -(float)3.141592653589793 ? (float)3.141592653589793 : t;
        }
    }
    return DCO_OK;
}

/* gradient_amplitude, src/contour.cpp:27-42 */
int dco_o_gradient_amplitude(const float* r, int w, int h, float* amp) {
    for (int y = 0; y < h; ++y)
        for (int x = 0; x < w; ++x) {
            float c = r[IDX(x, y, w)];
            float gu = x + 1 < w ? r[IDX(x + 1, y, w)] - c : (w > 1 ? c - r[IDX(x - 1, y, w)] : 0.0f);
            float gv = y + 1 < h ? r[IDX(x, y + 1, w)] - c : (h > 1 ? c - r[IDX(x, y - 1, w)] : 0.0f);
            amp[IDX(x, y, w)] = maxf_std(fabsf(gu), fabsf(gv));
        }
    return DCO_OK;
}

/* projection_confidence, src/contour.cpp:65-78 (sample_component :46-60) */
static double growth(const float* fu, const float* fv, int w, int h, int x, int y, double k) {
    float u = fu[IDX(x, y, w)], v = fv[IDX(x, y, w)];
    double mag = hypot((double)u, (double)v);
    if (mag < 1e-3) return 0.0;
    double ex = u / mag, ey = v / mag;
    float bx = (float)(x - k * ex), by = (float)(y - k * ey);
    float ax = (float)(x + k * ex), ay = (float)(y + k * ey);
    double back = bilerp(fu, w, h, bx, by) * ex + bilerp(fv, w, h, bx, by) * ey;
    double ahead = bilerp(fu, w, h, ax, ay) * ex + bilerp(fv, w, h, ax, ay) * ey;
    return ahead - back;
}

/* fuse_amplitudes, src/contour.cpp:82-106 */
int dco_o_fuse(const float* pu, const float* pv, const float* fu, const float* fv, const float* mp, const float* mf,
               int w, int h, double k, float* out) {
    for (int y = 0; y < h; ++y)
        for (int x = 0; x < w; ++x) {
            double gp = growth(pu, pv, w, h, x, y, k), gf = growth(fu, fv, w, h, x, y, k);
            size_t i = IDX(x, y, w);
            out[i] = gp > gf ? mp[i] : (gf > gp ? mf[i] : maxf_std(mp[i], mf[i]));
        }
    return DCO_OK;
}

/* box_filter, src/contour.cpp:108-136 */
int dco_o_box(const float* a, int w, int h, int radius, float* out) {
    if (radius < 1) return err(DCO_INPUT, "box_filter: radius must be >= 1");
    size_t W = (size_t)w + 1;
    double* sat = calloc(W * (h + 1), sizeof(double));
    for (int y = 0; y < h; ++y) {
        double run = 0.0;
        for (int x = 0; x < w; ++x) {
            run += a[IDX(x, y, w)];
            sat[(y + 1) * W + x + 1] = sat[y * W + x + 1] + run;
        }
    }
    for (int y = 0; y < h; ++y)
        for (int x = 0; x < w; ++x) {
            int y0 = y - radius < 0 ? 0 : y - radius, y1 = y + radius > h - 1 ? h - 1 : y + radius;
            int x0 = x - radius < 0 ? 0 : x - radius, x1 = x + radius > w - 1 ? w - 1 : x + radius;
            double s = sat[(y1 + 1) * W + x1 + 1] - sat[y0 * W + x1 + 1] - sat[(y1 + 1) * W + x0] + sat[y0 * W + x0];
            out[IDX(x, y, w)] = (float)(s / ((y1 - y0 + 1) * (x1 - x0 + 1)));
        }
    free(sat);
    return DCO_OK;
}

/* normalize_amplitude, src/contour.cpp:138-147 */
int dco_o_normalize(const float* a, int n, float* out) {
    float peak = 0.0f;
    for (int i = 0; i < n; ++i)
        if (isfinite(a[i])) peak = maxf_std(peak, a[i]);
    for (int i = 0; i < n; ++i) out[i] = (peak > 0.0f && isfinite(a[i])) ? a[i] / peak : a[i];
    return DCO_OK;
}

/* gaussian_blur, src/contour.cpp:149-175 */
int dco_o_gauss(const float* img, int w, int h, double sigma, float* out) {
    if (sigma <= 0.0) return err(DCO_INPUT, "gaussian_blur: sigma must be positive");
    double k[5], s = 0.0;
    for (int i = -2; i <= 2; ++i) {
        k[i + 2] = exp(-(i * i) / (2.0 * sigma * sigma));
        s += k[i + 2];
    }
    for (int i = 0; i < 5; ++i) k[i] /= s;
    float* tmp = malloc((size_t)w * h * 4);
    for (int y = 0; y < h; ++y)
        for (int x = 0; x < w; ++x) {
            double acc = 0.0;
            for (int i = -2; i <= 2; ++i) acc += k[i + 2] * img[IDX(clampi(x + i, 0, w - 1), y, w)];
            tmp[IDX(x, y, w)] = (float)acc;
        }
    for (int y = 0; y < h; ++y)
        for (int x = 0; x < w; ++x) {
            double acc = 0.0;
            for (int i = -2; i <= 2; ++i) acc += k[i + 2] * tmp[IDX(x, clampi(y + i, 0, h - 1), w)];
            out[IDX(x, y, w)] = (float)acc;
        }
    free(tmp);
    return DCO_OK;
}

/* extract_depth_contours_prefiltered, src/contour.cpp:177-279 */
int dco_o_contours(const float* b, int w, int h, const float* mf, int qw, int qh, const dco_config* c,
                   uint8_t* edges, float* m_i) {
    size_t n = (size_t)w * h;
    float* gx = malloc(n * 4);
    float* gy = malloc(n * 4);
    float* mag = malloc(n * 4);
    uint8_t* keep = calloc(n, 1);
#define B(xx, yy) b[IDX(clampi(xx, 0, w - 1), clampi(yy, 0, h - 1), w)]
    float peak = 0.0f;
    for (int y = 0; y < h; ++y)
        for (int x = 0; x < w; ++x) {
            size_t i = IDX(x, y, w);
            gx[i] = (B(x + 1, y - 1) + 2 * B(x + 1, y) + B(x + 1, y + 1)) -
                    (B(x - 1, y - 1) + 2 * B(x - 1, y) + B(x - 1, y + 1));
            gy[i] = (B(x - 1, y + 1) + 2 * B(x, y + 1) + B(x + 1, y + 1)) -
                    (B(x - 1, y - 1) + 2 * B(x, y - 1) + B(x + 1, y - 1));
            mag[i] = hypotf(gx[i], gy[i]);
            peak = maxf_std(peak, mag[i]);
        }
#undef B
    if (peak > 0.0f)
        for (size_t i = 0; i < n; ++i) mag[i] /= peak;
    memcpy(m_i, mag, n * 4);
#define M(xx, yy) mag[IDX(clampi(xx, 0, w - 1), clampi(yy, 0, h - 1), w)]
    for (int y = 0; y < h; ++y)
        for (int x = 0; x < w; ++x) {
            size_t i = IDX(x, y, w);
            if (mag[i] <= 0.0f) continue;
            double ang = atan2f(gy[i], gx[i]);
            if (ang < 0) ang += 3.141592653589793;
            double deg = ang * 180.0 / 3.141592653589793;
            float a1, a2;
            if (deg < 22.5 || deg >= 157.5) {
                a1 = M(x + 1, y);
                a2 = M(x - 1, y);
            } else if (deg < 67.5) {
                a1 = M(x + 1, y + 1);
                a2 = M(x - 1, y - 1);
            } else if (deg < 112.5) {
                a1 = M(x, y + 1);
                a2 = M(x, y - 1);
            } else {
                a1 = M(x - 1, y + 1);
                a2 = M(x + 1, y - 1);
            }
            keep[i] = mag[i] >= a1 && mag[i] >= a2;
            if (keep[i]) {
                int mx = x / 2 < qw - 1 ? x / 2 : qw - 1, my = y / 2 < qh - 1 ? y / 2 : qh - 1;
                float conf = mf[IDX(mx, my, qw)];
                if (!isfinite(conf) || conf < c->t_depth) keep[i] = 0;
            }
        }
#undef M
    /* hysteresis (contour.cpp:250-277): explicit stack flood, 8-connected */
    memset(edges, 0, n);
    size_t* stack = malloc(n * sizeof(size_t));
    size_t top = 0;
    for (size_t i = 0; i < n; ++i)
        if (keep[i] && mag[i] > c->t_high) {
            edges[i] = 1;
            stack[top++] = i;
        }
    while (top) {
        size_t i = stack[--top];
        int x = (int)(i % w), y = (int)(i / w);
        for (int dy = -1; dy <= 1; ++dy)
            for (int dx = -1; dx <= 1; ++dx) {
                int qx = x + dx, qy = y + dy;
                if ((!dx && !dy) || qx < 0 || qy < 0 || qx >= w || qy >= h) continue;
                size_t j = IDX(qx, qy, w);
                if (!edges[j] && keep[j] && mag[j] >= c->t_low) {
                    edges[j] = 1;
                    stack[top++] = j;
                }
            }
    }
    free(stack);
    free(gx);
    free(gy);
    free(mag);
    free(keep);
    return DCO_OK;
}

/* ---------------------------------------------------------------- densify */
/* fused_confidence + smoothness_weight, src/densify.cpp:11-16, 26-35 */
static double conf_at(const float* mf, int qw, int qh, int x, int y) {
    float v = mf[IDX(x / 2 < qw - 1 ? x / 2 : qw - 1, y / 2 < qh - 1 ? y / 2 : qh - 1, qw)];
    return isfinite(v) ? v : 0.0;
}
static double pair_weight(const uint8_t* e, const float* mf, int qw, int qh, const float* mi, int w, int px, int py,
                          int qx, int qy) {
    if ((e[IDX(px, py, w)] != 0) + (e[IDX(qx, qy, w)] != 0) == 1) return 0.0;
    double a = conf_at(mf, qw, qh, px, py) * mi[IDX(px, py, w)];
    double b = conf_at(mf, qw, qh, qx, qy) * mi[IDX(qx, qy, w)];
    double m = b < a ? b : a;
    double r = 1.0 - m;
    return r < 0.0 ? 0.0 : r;
}

/* assemble_system, src/densify.cpp:37-116 */
int dco_o_assemble(const float* sparse, const uint8_t* edges, const float* mf, int qw, int qh, const float* mi,
                   const float* pre, int w, int h, const dco_config* c, double* diag, double* ch, double* cv,
                   double* rhs, double* init, uint8_t* anchored, double* constant_term, uint64_t* anchor_count) {
    size_t n = (size_t)w * h;
    if (c->lambda_s2 <= 0.0) pre = NULL;
    double sum = 0.0;
    size_t cnt = 0;
    for (size_t i = 0; i < n; ++i)
        if (isfinite(sparse[i])) {
            sum += sparse[i];
            ++cnt;
        }
    double mean = cnt ? sum / cnt : 0.0;
    double ct = 0.0;
    uint64_t anchors = 0;
    for (size_t i = 0; i < n; ++i) {
        diag[i] = ch[i] = cv[i] = rhs[i] = 0.0;
        anchored[i] = 0;
        double start = mean;
        if (isfinite(sparse[i])) {
            double s = sparse[i];
            diag[i] += c->lambda_d;
            rhs[i] += c->lambda_d * s;
            ct += c->lambda_d * s * s;
            anchored[i] = 1;
            start = s;
        } else if (pre && isfinite(pre[i])) {
            start = pre[i];
        }
        if (pre && isfinite(pre[i])) {
            double q = pre[i];
            diag[i] += c->lambda_s2;
            rhs[i] += c->lambda_s2 * q;
            ct += c->lambda_s2 * q * q;
            anchored[i] = 1;
        }
        init[i] = start;
        anchors += anchored[i];
    }
    for (int y = 0; y < h; ++y)
        for (int x = 0; x < w; ++x) {
            size_t i = IDX(x, y, w);
            if (x + 1 < w) {
                double k = 2.0 * c->lambda_s * pair_weight(edges, mf, qw, qh, mi, w, x, y, x + 1, y);
                ch[i] = k;
                diag[i] += k;
                diag[i + 1] += k;
            }
            if (y + 1 < h) {
                double k = 2.0 * c->lambda_s * pair_weight(edges, mf, qw, qh, mi, w, x, y, x, y + 1);
                cv[i] = k;
                diag[i] += k;
                diag[i + w] += k;
            }
        }
    *constant_term = ct;
    *anchor_count = anchors;
    return DCO_OK;
}

/* apply_system, src/densify.cpp:118-133 */
int dco_o_apply(int w, int h, const double* diag, const double* ch, const double* cv, const double* x,
                double* out) {
    for (int y = 0; y < h; ++y)
        for (int xx = 0; xx < w; ++xx) {
            size_t i = IDX(xx, y, w);
            double s = diag[i] * x[i];
            if (xx + 1 < w) s -= ch[i] * x[i + 1];
            if (xx > 0) s -= ch[i - 1] * x[i - 1];
            if (y + 1 < h) s -= cv[i] * x[i + w];
            if (y > 0) s -= cv[i - w] * x[i - w];
            out[i] = s;
        }
    return DCO_OK;
}

static double dotp(const double* a, const double* b, size_t n) {
    double s = 0.0;
    for (size_t i = 0; i < n; ++i) s += a[i] * b[i];
    return s;
}

/* objective_value, src/densify.cpp:135-139 */
static double objective(int w, int h, const double* diag, const double* ch, const double* cv, const double* rhs,
                        double ct, const double* x, double* tmp) {
    dco_o_apply(w, h, diag, ch, cv, x, tmp);
    size_t n = (size_t)w * h;
    return dotp(x, tmp, n) - 2.0 * dotp(rhs, x, n) + ct;
}

/* solve_dense_depth, src/densify.cpp:141-222 */
int dco_o_solve(int w, int h, const double* diag, const double* ch, const double* cv, const double* rhs,
                const double* init, uint64_t anchor_count, double constant_term, const dco_config* c, float* dense,
                int* iterations, double* relres, double* obj0, double* obj1) {
    if (anchor_count == 0)
        return err(DCO_UNSOLVABLE, "solve_dense_depth: no pixel carries a data or stability constraint");
    size_t n = (size_t)w * h;
    double* buf = malloc(sizeof(double) * n * 9);
    double *x = buf, *m = buf + n, *r = buf + 2 * n, *z = buf + 3 * n, *p = buf + 4 * n, *q = buf + 5 * n,
           *xs = buf + 6 * n, *rs = buf + 7 * n, *tmp = buf + 8 * n;
    memcpy(x, init, n * 8);
    for (size_t i = 0; i < n; ++i) m[i] = diag[i] > 0.0 ? 1.0 / diag[i] : 1.0;
    dco_o_apply(w, h, diag, ch, cv, x, q);
    for (size_t i = 0; i < n; ++i) r[i] = rhs[i] - q[i];
    double bn = sqrt(dotp(rhs, rhs, n));
    double den = bn > 0.0 ? bn : 1.0;
    memcpy(xs, x, n * 8);
    memcpy(rs, r, n * 8);
    double sn = sqrt(dotp(rs, rs, n));
    *obj0 = objective(w, h, diag, ch, cv, rhs, constant_term, init, tmp);
    for (size_t i = 0; i < n; ++i) z[i] = m[i] * r[i];
    memcpy(p, z, n * 8);
    double rho = dotp(r, z, n);
    int it = 0;
    while (it < c->solver_max_iter && sn / den > c->solver_tol) {
        dco_o_apply(w, h, diag, ch, cv, p, q);
        double pq = dotp(p, q, n);
        if (pq <= 0.0) break;
        double alpha = rho / pq, rn = 0.0;
        for (size_t i = 0; i < n; ++i) {
            x[i] += alpha * p[i];
            r[i] -= alpha * q[i];
            z[i] = m[i] * r[i];
            rn += r[i] * z[i];
        }
        double beta = rn / rho;
        rho = rn;
        for (size_t i = 0; i < n; ++i) p[i] = z[i] + beta * p[i];
        double sd = 0.0, dd = 0.0;
        for (size_t i = 0; i < n; ++i) {
            double di = r[i] - rs[i];
            sd += rs[i] * di;
            dd += di * di;
        }
        double eta = 0.0;
        if (dd > 0.0) {
            eta = -sd / dd;
            eta = eta < 0.0 ? 0.0 : (eta > 1.0 ? 1.0 : eta);
        }
        double s2 = 0.0;
        for (size_t i = 0; i < n; ++i) {
            if (eta > 0.0) {
                rs[i] += eta * (r[i] - rs[i]);
                xs[i] += eta * (x[i] - xs[i]);
            }
            s2 += rs[i] * rs[i];
        }
        sn = sqrt(s2);
        ++it;
    }
    *iterations = it;
    *relres = sn / den;
    *obj1 = objective(w, h, diag, ch, cv, rhs, constant_term, xs, tmp);
    for (size_t i = 0; i < n; ++i) dense[i] = (float)(xs[i] < 0.0 ? 0.0 : xs[i]);
    free(buf);
    return DCO_OK;
}

/* -------------------------------------------------------------- composite */
/* composite, src/occlude.cpp:171-194 */
int dco_o_composite(const float* real, const float* dense, const float* vrgb, const float* vdepth, int w, int h,
                    float* out, uint8_t* mask) {
    size_t n = (size_t)w * h;
    memcpy(out, real, n * 3 * 4);
    for (size_t i = 0; i < n; ++i) {
        mask[i] = 0;
        if (!isfinite(vdepth[i])) continue;
        if (isfinite(dense[i]) && vdepth[i] > dense[i]) continue;
        mask[i] = 1;
        memcpy(out + 3 * i, vrgb + 3 * i, 12);
    }
    return DCO_OK;
}
