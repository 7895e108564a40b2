// ctx.cu — context lifetime, scratch pool, config defaults/validation and the
// host-computed lookup tables. Mirrors include/dco/config.hpp:11-60 and
// src/config.cpp:10-36.
#include <math.h>
#include <string.h>

#include <map>
#include <mutex>

#include "common.cuh"

namespace dco_gpu {

void* scratch(dco_ctx* ctx, Slot s, size_t bytes) {
    DevBuf& b = ctx->slots[s];
    if (b.bytes < bytes) {
        if (b.ptr) cuda_check(cudaFree(b.ptr), "cudaFree(scratch)");
        b.ptr = nullptr;
        b.bytes = 0;
        size_t want = bytes + bytes / 8 + 256;
        cuda_check(cudaMalloc(&b.ptr, want), "cudaMalloc(scratch)");
        b.bytes = want;
    }
    return b.ptr;
}

void* pinned_host(dco_ctx* ctx, size_t bytes) {
    if (ctx->pinned_bytes < bytes) {
        if (ctx->pinned) cudaFreeHost(ctx->pinned);
        ctx->pinned = nullptr;
        ctx->pinned_bytes = 0;
        cuda_check(cudaMallocHost(&ctx->pinned, bytes), "cudaMallocHost");
        ctx->pinned_bytes = bytes;
    }
    return ctx->pinned;
}

void validate_config(const dco_config* c) {
    require(c != nullptr, "config: null");
    auto bad = [](const char* m) { fail(DCO_CONFIG, m); };
    if (c->d_min >= c->d_max) bad("config: d_min must be below d_max");
    if (c->t_low < 0.0 || c->t_low >= c->t_high || c->t_high > 1.0)
        bad("config: need 0 <= t_low < t_high <= 1");
    if (c->t_depth < 0.0 || c->t_depth > 1.0) bad("config: t_depth outside [0,1]");
    if (c->lambda_ad <= 0.0 || c->lambda_census <= 0.0 || c->lambda_d <= 0.0 ||
        c->lambda_s <= 0.0 || c->lambda_s2 <= 0.0)
        bad("config: every lambda must be positive");
    if (c->gamma_l <= 0.0 || c->epsilon <= 0.0)
        bad("config: gamma_l and epsilon must be positive");
    if (c->census_window_w % 2 == 0 || c->census_window_h % 2 == 0)
        bad("config: census window dimensions must be odd");
    if (c->census_window_w < 1 || c->census_window_h < 1 ||
        c->census_window_w * c->census_window_h - 1 > 64)
        bad("config: census window must fit 64 bits");
    if (c->cross_arm_l1 < 1 || c->cross_arm_l2 < 1 || c->cross_arm_l2 > c->cross_arm_l1)
        bad("config: need 1 <= cross_arm_l2 <= cross_arm_l1");
    if (c->cross_color_tau <= 0.0 || c->cross_color_tau2 <= 0.0)
        bad("config: color thresholds must be positive");
    if (c->box_radius < 1) bad("config: box_radius must be >= 1");
    if (c->gauss_sigma <= 0.0) bad("config: gauss_sigma must be positive");
    if (c->confidence_offset_k <= 0.0) bad("config: confidence_offset_k must be positive");
    if (c->hist_iterations < 0) bad("config: hist_iterations must be >= 0");
    if (c->focal_px <= 0.0 || c->baseline_m <= 0.0)
        bad("config: focal_px and baseline_m must be positive");
    if (c->solver_tol <= 0.0 || c->solver_max_iter < 1)
        bad("config: solver_tol must be positive, solver_max_iter >= 1");
    if (c->d_min < 0) bad("config: d_min must be >= 0");
}

void make_stereo_tables(const dco_config* cfg, StereoTables* t) {
    for (int l = 0; l < 256; ++l)
        t->alpha[l] = 1.0 - exp(-cfg->gamma_l / (static_cast<double>(l) + cfg->epsilon));
    for (int h = 0; h <= 64; ++h)
        t->census[h] = 1.0 - exp(-static_cast<double>(h) / cfg->lambda_census);
}

void smem_attr(dco_ctx* ctx, const void* fn, int bytes, bool carveout) {
    static std::mutex mu;
    static std::map<std::pair<int, const void*>, int> done;
    std::lock_guard<std::mutex> lock(mu);
    int& have = done[{ctx->device, fn}];  // bytes + 1 once set (0 = never)
    if (have > bytes) return;
    if (bytes > 0)
        cuda_check(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes), "smem attr");
    if (carveout)
        cuda_check(cudaFuncSetAttribute(fn, cudaFuncAttributePreferredSharedMemoryCarveout, 100), "carveout");
    have = bytes + 1;
}

int sm_count(dco_ctx* ctx) {
    static std::mutex mu;
    static std::map<int, int> cache;
    std::lock_guard<std::mutex> lock(mu);
    auto it = cache.find(ctx->device);
    if (it != cache.end()) return it->second;
    int n = 0;
    cuda_check(cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, ctx->device), "sm count");
    cache[ctx->device] = n;
    return n;
}

}  // namespace dco_gpu

using namespace dco_gpu;

extern "C" {

int dco_abi_version(void) { return DCO_ABI_VERSION; }

int dco_create(int device, dco_ctx** out) {
    if (!out) return DCO_INPUT;
    *out = nullptr;
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess || n == 0) {
        cudaGetLastError();
        return DCO_CUDA;
    }
    if (device < 0 || device >= n) return DCO_INPUT;
    if (cudaSetDevice(device) != cudaSuccess) return DCO_CUDA;
    dco_ctx* c = new dco_ctx();
    c->device = device;
    *out = c;
    return DCO_OK;
}

void dco_destroy(dco_ctx* ctx) {
    if (!ctx) return;
    cudaSetDevice(ctx->device);
    cudaStreamSynchronize(ctx->stream);
    for (auto& b : ctx->slots)
        if (b.ptr) cudaFree(b.ptr);
    if (ctx->pinned) cudaFreeHost(ctx->pinned);
    delete ctx;
}

const char* dco_last_error(const dco_ctx* ctx) { return ctx ? ctx->err.c_str() : "null context"; }

int dco_set_stream(dco_ctx* ctx, void* stream) {
    return guarded(ctx, [&] { ctx->stream = static_cast<cudaStream_t>(stream); });
}

int dco_synchronize(dco_ctx* ctx) {
    return guarded(ctx, [&] { cuda_check(cudaStreamSynchronize(ctx->stream), "synchronize"); });
}

uint64_t dco_kernel_launches(const dco_ctx* ctx) { return ctx ? ctx->launches : 0; }

const char* dco_last_solver(const dco_ctx* ctx) { return ctx ? ctx->last_solver : ""; }

void dco_config_default(dco_config* c) {
    if (!c) return;
    c->lambda_ad = 10.0;
    c->lambda_census = 40.0;
    c->gamma_l = 1.0;
    c->epsilon = 0.8;
    c->t_high = 0.06;
    c->t_low = 0.03;
    c->t_depth = 0.03;
    c->lambda_d = 0.8;
    c->lambda_s = 1.2;
    c->lambda_s2 = 0.02;
    c->d_min = 0;
    c->d_max = 64;
    c->focal_px = 400.0;
    c->baseline_m = 0.12;
    c->census_window_w = 9;
    c->census_window_h = 7;
    c->cross_color_tau = 20.0 / 255.0;
    c->cross_color_tau2 = 6.0 / 255.0;
    c->cross_arm_l1 = 17;
    c->cross_arm_l2 = 8;
    c->box_radius = 5;
    c->gauss_sigma = 1.4;
    c->confidence_offset_k = 2.0;
    c->hist_iterations = 2;
    c->solver_tol = 1e-5;
    c->solver_max_iter = 400;
}

int dco_config_validate(const dco_config* cfg, char* msg, size_t msg_len) {
    try {
        validate_config(cfg);
        if (msg && msg_len) msg[0] = 0;
        return DCO_OK;
    } catch (const Failure& f) {
        if (msg && msg_len) {
            strncpy(msg, f.what(), msg_len - 1);
            msg[msg_len - 1] = 0;
        }
        return f.status;
    }
}

}  // extern "C"
