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
void aggregate_costs_band(dco_ctx* ctx, const float* cost, int w, int h, int nd, const uint8_t* l,
                          const uint8_t* r, const uint8_t* u, const uint8_t* d, int max_arm, float* out,
                          const double* carry_in, int c0, double* carry_out, int e);
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

int dco_stereo_band(dco_ctx* ctx, const float* left_sub, const float* right_sub, const dco_band* band,
                    const dco_config* cfg, int fw, int fh, const double* carry_in, double* carry_out,
                    float* disparity, float* sparse) {
    return guarded(ctx, [&] {
        validate_config(cfg);
        require(band != nullptr, "dco_stereo_band: null band");
        const dco_band& b = *band;
        const int qw = fw / 2, qh = fh / 2;
        require(qw >= 1 && qh >= 1, "dco_stereo_band: frame smaller than 2x2");
        require(0 <= b.sub0 && b.sub0 <= b.carry_row && b.carry_row <= b.row0 && b.row0 < b.row1 &&
                    b.row1 <= b.sub1 && b.sub1 <= qh,
                "dco_stereo_band: inconsistent band (use dco_band_plan)");
        require(b.carry_row == 0 || carry_in != nullptr, "dco_stereo_band: band needs the carry from the band above");
        require(b.carry_out_row < 0 || carry_out != nullptr, "dco_stereo_band: band exports a carry; carry_out is null");
        require(b.carry_out_row < 0 || (b.carry_out_row > b.carry_row && b.carry_out_row < b.sub1),
                "dco_stereo_band: carry_out_row outside the band's exact rows");
        require(b.frow0 == 2 * b.row0 && b.frow1 >= 2 * b.row1 && b.frow1 <= fh, "dco_stereo_band: bad full rows");
        const int hs = b.sub1 - b.sub0;
        const size_t n = static_cast<size_t>(qw) * hs;
        const int nd = cfg->d_max - cfg->d_min + 1;
        uint8_t* arms = static_cast<uint8_t*>(scratch(ctx, S_ARMS, 4 * n));
        float* cost = static_cast<float*>(scratch(ctx, S_COST, n * nd * 4));
        float* agg = static_cast<float*>(scratch(ctx, S_AGG, n * nd * 4));
        float* d0 = static_cast<float*>(scratch(ctx, S_TMP0, n * 4 * 2));
        float* d1 = d0 + n;
        uint8_t *L = arms, *R = arms + n, *U = arms + 2 * n, *D = arms + 3 * n;
        build_cross_windows(ctx, left_sub, qw, hs, cfg, L, R, U, D);
        compute_cost_volume(ctx, left_sub, right_sub, qw, hs, L, R, U, D, cfg, cost);
        aggregate_costs_band(ctx, cost, qw, hs, nd, L, R, U, D, cfg->cross_arm_l1, agg,
                             b.carry_row > 0 ? carry_in : nullptr, b.carry_row - b.sub0, carry_out,
                             b.carry_out_row >= 0 ? b.carry_out_row - b.sub0 : -1);
        select_disparity_wta(ctx, agg, qw, hs, cfg->d_min, nd, d0);
        refine_disparity_histogram(ctx, d0, qw, hs, L, R, U, D, cfg->hist_iterations, cfg->d_max, cfg->cross_arm_l1,
                                   d1);
        const float* own = d1 + static_cast<size_t>(b.row0 - b.sub0) * qw;
        const int rows = b.row1 - b.row0;
        if (disparity)
            cuda_check(cudaMemcpyAsync(disparity, own, static_cast<size_t>(rows) * qw * 4, cudaMemcpyDeviceToDevice,
                                       ctx->stream),
                       "band disparity");
        if (sparse) disparity_to_sparse_depth(ctx, own, qw, rows, cfg, fw, b.frow1 - b.frow0, sparse);
    });
}

}  // extern "C"
