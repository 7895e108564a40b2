// bands.cu -- row-band split of the stereo chain for frames spread over
// several GPUs (BASELINE config D). See include/dco_gpu.h and
// DESIGN 7 for the halo and the column-prefix carry; the kernels are the
// whole-frame ones on the band's sub-image, plus k_agg_v2<.., kBand>.
#include <algorithm>

#include "common.cuh"

namespace dco_gpu {

void build_cross_windows(dco_ctx* ctx, const float* img, int w, int h, const dco_config* cfg, uint8_t* l,
                         uint8_t* r, uint8_t* u, uint8_t* d);
void compute_cost_volume(dco_ctx* ctx, const float* left, const float* right, int w, int h, const uint8_t* l,
                         const uint8_t* r, const uint8_t* u, const uint8_t* d, const dco_config* cfg,
                         float* cost);
void aggregate_band_hpass(dco_ctx* ctx, const float* cost, int w, int h, int nd, const uint8_t* l, const uint8_t* r,
                          const uint8_t* u, const uint8_t* d, int max_arm);
void aggregate_band_vpass(dco_ctx* ctx, int w, int h, int nd, int max_arm, float* out, const double* carry_in,
                          int c0, double* carry_out, int e, int k0, int k1);
void select_disparity_wta(dco_ctx* ctx, const float* cost, int w, int h, int d_min, int nd, float* disp);
void refine_disparity_histogram(dco_ctx* ctx, const float* disp, int w, int h, const uint8_t* l,
                                const uint8_t* r, const uint8_t* u, const uint8_t* d, int iters, int bin_bound,
                                int max_arm, float* out);
void disparity_to_sparse_depth(dco_ctx* ctx, const float* disp, int w, int h, const dco_config* cfg, int fw,
                               int fh, float* out);

namespace {

// Rows of recompute halo: an owned row's disparity depends on quarter rows
// within (I+1)*l1 + max(Rc,1): census +-Rc and horizontal arms +-1 (3x3 median)
// for the cost and hsum rows; aggregation +-l1; each refinement pass +-l1;
// vertical arms +-(l1+1), which the sum covers.
int band_halo(const dco_config* cfg) {
    const int rc = std::max(cfg->census_window_h / 2, 1);
    return (cfg->hist_iterations + 1) * cfg->cross_arm_l1 + rc;
}

dco_band plan(const dco_config* cfg, int fw, int fh, int bands, int k) {
    const int qh = fh / 2;
    const int reach = (cfg->hist_iterations + 1) * cfg->cross_arm_l1;  // prefix rows an owned row reads above it
    const int rc = std::max(cfg->census_window_h / 2, 1);
    auto row0 = [&](int j) { return static_cast<int>(static_cast<long long>(j) * qh / bands); };
    auto carry = [&](int j) { return std::max(0, row0(j) - reach); };
    dco_band b;
    b.row0 = row0(k);
    b.row1 = row0(k + 1);
    b.halo = band_halo(cfg);
    b.carry_row = carry(k);
    b.sub0 = std::max(0, b.carry_row - rc);
    b.sub1 = std::min(qh, b.row1 + b.halo);
    b.carry_out_row = (k + 1 < bands && carry(k + 1) > 0) ? carry(k + 1) : -1;
    b.frow0 = 2 * b.row0;
    b.frow1 = k + 1 == bands ? fh : 2 * b.row1;
    return b;
}

}  // namespace
}  // namespace dco_gpu

using namespace dco_gpu;

extern "C" {

int dco_band_plan(const dco_config* cfg, int fw, int fh, int bands, int index, dco_band* out) {
    try {
        validate_config(cfg);
        require(out != nullptr, "dco_band_plan: null output");
        require(fw >= 2 && fh >= 2, "dco_band_plan: frame smaller than 2x2");
        require(bands >= 1 && bands <= fh / 2, "dco_band_plan: bands must be in [1, quarter height]");
        require(index >= 0 && index < bands, "dco_band_plan: band index out of range");
        require(cfg->cross_arm_l1 <= 127, "dco_band_plan: cross_arm_l1 must be <= 127");
        *out = plan(cfg, fw, fh, bands, index);
        return static_cast<int>(DCO_OK);
    } catch (const Failure& f) {
        return f.status;
    }
}

size_t dco_band_carry_bytes(const dco_config* cfg, int fw) {
    return static_cast<size_t>(fw / 2) * static_cast<size_t>(cfg->d_max - cfg->d_min + 1) * sizeof(double);
}

}  // extern "C"

namespace dco_gpu {
namespace {

struct BandBufs {
    int qw, hs, nd;
    size_t n;
    uint8_t *L, *R, *U, *D;
    float *cost, *agg, *d0, *d1;
};

BandBufs band_bufs(dco_ctx* ctx, const dco_band& b, const dco_config* cfg, int fw, int fh) {
    BandBufs z;
    z.qw = fw / 2;
    const int qh = fh / 2;
    require(z.qw >= 1 && qh >= 1, "dco_stereo_band: frame smaller than 2x2");
    require(0 <= b.sub0 && b.sub0 <= b.carry_row && b.carry_row <= b.row0 && b.row0 < b.row1 && b.row1 <= b.sub1 &&
                b.sub1 <= qh,
            "dco_stereo_band: inconsistent band (use dco_band_plan)");
    require(b.carry_out_row < 0 || (b.carry_out_row > b.carry_row && b.carry_out_row < b.sub1),
            "dco_stereo_band: carry_out_row outside the band's exact rows");
    require(b.frow0 == 2 * b.row0 && b.frow1 >= 2 * b.row1 && b.frow1 <= fh, "dco_stereo_band: bad full rows");
    z.hs = b.sub1 - b.sub0;
    z.n = static_cast<size_t>(z.qw) * z.hs;
    z.nd = cfg->d_max - cfg->d_min + 1;
    uint8_t* arms = static_cast<uint8_t*>(scratch(ctx, S_ARMS, 4 * z.n));
    z.L = arms;
    z.R = arms + z.n;
    z.U = arms + 2 * z.n;
    z.D = arms + 3 * z.n;
    z.cost = static_cast<float*>(scratch(ctx, S_COST, z.n * z.nd * 4));
    z.agg = static_cast<float*>(scratch(ctx, S_AGG, z.n * z.nd * 4));
    z.d0 = static_cast<float*>(scratch(ctx, S_TMP0, z.n * 4 * 2));
    z.d1 = z.d0 + z.n;
    return z;
}

void band_begin(dco_ctx* ctx, const float* left_sub, const float* right_sub, const dco_band& b,
                const dco_config* cfg, int fw, int fh) {
    BandBufs z = band_bufs(ctx, b, cfg, fw, fh);
    build_cross_windows(ctx, left_sub, z.qw, z.hs, cfg, z.L, z.R, z.U, z.D);
    compute_cost_volume(ctx, left_sub, right_sub, z.qw, z.hs, z.L, z.R, z.U, z.D, cfg, z.cost);
    aggregate_band_hpass(ctx, z.cost, z.qw, z.hs, z.nd, z.L, z.R, z.U, z.D, cfg->cross_arm_l1);
}

void band_vpass(dco_ctx* ctx, const dco_band& b, const dco_config* cfg, int fw, int fh, int d0, int d1,
                const double* carry_in, double* carry_out) {
    BandBufs z = band_bufs(ctx, b, cfg, fw, fh);
    require(b.carry_row == 0 || carry_in != nullptr, "dco_stereo_band: band needs the carry from the band above");
    require(b.carry_out_row < 0 || carry_out != nullptr, "dco_stereo_band: band exports a carry; carry_out is null");
    aggregate_band_vpass(ctx, z.qw, z.hs, z.nd, cfg->cross_arm_l1, z.agg, b.carry_row > 0 ? carry_in : nullptr,
                         b.carry_row - b.sub0, carry_out, b.carry_out_row >= 0 ? b.carry_out_row - b.sub0 : -1, d0,
                         d1);
}

void band_end(dco_ctx* ctx, const dco_band& b, const dco_config* cfg, int fw, int fh, float* disparity,
              float* sparse) {
    BandBufs z = band_bufs(ctx, b, cfg, fw, fh);
    select_disparity_wta(ctx, z.agg, z.qw, z.hs, cfg->d_min, z.nd, z.d0);
    refine_disparity_histogram(ctx, z.d0, z.qw, z.hs, z.L, z.R, z.U, z.D, cfg->hist_iterations, cfg->d_max,
                               cfg->cross_arm_l1, z.d1);
    const float* own = z.d1 + static_cast<size_t>(b.row0 - b.sub0) * z.qw;
    const int rows = b.row1 - b.row0;
    if (disparity)
        cuda_check(cudaMemcpyAsync(disparity, own, static_cast<size_t>(rows) * z.qw * 4, cudaMemcpyDeviceToDevice,
                                   ctx->stream),
                   "band disparity");
    if (sparse) disparity_to_sparse_depth(ctx, own, z.qw, rows, cfg, fw, b.frow1 - b.frow0, sparse);
}

}  // namespace
}  // namespace dco_gpu

extern "C" {

int dco_stereo_band(dco_ctx* ctx, const float* left_sub, const float* right_sub, const dco_band* band,
                    const dco_config* cfg, int fw, int fh, const double* carry_in, double* carry_out,
                    float* disparity, float* sparse) {
    return guarded(ctx, [&] {
        validate_config(cfg);
        require(band != nullptr, "dco_stereo_band: null band");
        band_begin(ctx, left_sub, right_sub, *band, cfg, fw, fh);
        band_vpass(ctx, *band, cfg, fw, fh, 0, cfg->d_max - cfg->d_min + 1, carry_in, carry_out);
        band_end(ctx, *band, cfg, fw, fh, disparity, sparse);
    });
}

int dco_stereo_band_begin(dco_ctx* ctx, const float* left_sub, const float* right_sub, const dco_band* band,
                          const dco_config* cfg, int fw, int fh) {
    return guarded(ctx, [&] {
        validate_config(cfg);
        require(band != nullptr, "dco_stereo_band: null band");
        band_begin(ctx, left_sub, right_sub, *band, cfg, fw, fh);
    });
}

int dco_stereo_band_vpass(dco_ctx* ctx, const dco_band* band, const dco_config* cfg, int fw, int fh, int d0, int d1,
                          const double* carry_in, double* carry_out) {
    return guarded(ctx, [&] {
        validate_config(cfg);
        require(band != nullptr, "dco_stereo_band: null band");
        band_vpass(ctx, *band, cfg, fw, fh, d0, d1, carry_in, carry_out);
    });
}

int dco_stereo_band_end(dco_ctx* ctx, const dco_band* band, const dco_config* cfg, int fw, int fh, float* disparity,
                        float* sparse) {
    return guarded(ctx, [&] {
        validate_config(cfg);
        require(band != nullptr, "dco_stereo_band: null band");
        band_end(ctx, *band, cfg, fw, fh, disparity, sparse);
    });
}

}  // extern "C"
