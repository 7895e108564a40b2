/*
 * dco_gpu.h — C-ABI of the B200-native depth-contour-occlusion (DCO) hot path.
 *
 * Every entry point below replaces one free function of the reference's L2
 * stage API (namespace dco, /root/reference/proj/include/dco/ *.hpp). The
 * mapping is one-to-one and cited per function. Differences are mechanical:
 *   - plain pointers + sizes instead of std::vector-owning structs;
 *   - stage inputs/outputs are DEVICE pointers owned by the caller (cudaMalloc
 *     or a torch tensor), unless the function name ends in _host;
 *   - exceptions become status codes (dco_status) plus dco_last_error(ctx):
 *       InputError -> DCO_INPUT, ConfigError -> DCO_CONFIG (an InputError,
 *       CLI exit 1), CodecError -> DCO_CODEC (exit 2), UnsolvableFrameError ->
 *       DCO_UNSOLVABLE (exit 3)   (error.hpp:10-32, tools/dco.cpp:203-224);
 *   - work is enqueued on the context's CUDA stream (dco_set_stream); calls
 *     return after enqueueing unless they must report a host-side scalar
 *     (solve statistics, anchor counts), in which case they synchronise.
 * Layouts are the reference's: row-major rasters, nodata = quiet NaN
 * (image.hpp:71), cost volumes [y][x][d - d_min] (stereo.hpp:50-63), cross
 * arms as four u8 planes (stereo.hpp:13-35), flow as SoA u/v planes
 * (flow.hpp:13-26), RGB interleaved (image.hpp:40-63).
 * There is no CPU fallback: without a CUDA device every compute call fails
 * with DCO_CUDA.
 */
#ifndef DCO_GPU_H
#define DCO_GPU_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif
#if defined(__GNUC__)
#pragma GCC visibility push(default)
#endif

#define DCO_ABI_VERSION 3

typedef enum dco_status {
    DCO_OK = 0,
    DCO_INPUT = 1,      /* dco::InputError */
    DCO_CONFIG = 5,     /* dco::ConfigError (maps to CLI exit 1 like InputError) */
    DCO_CODEC = 2,      /* dco::CodecError */
    DCO_UNSOLVABLE = 3, /* dco::UnsolvableFrameError */
    DCO_CUDA = 4        /* device / driver failure (no reference analogue) */
} dco_status;

/* Mirrors dco::PipelineConfig field for field, same order and defaults
 * (include/dco/config.hpp:11-60). */
typedef struct dco_config {
    double lambda_ad, lambda_census, gamma_l, epsilon;
    double t_high, t_low, t_depth;
    double lambda_d, lambda_s, lambda_s2;
    int d_min, d_max;
    double focal_px, baseline_m;
    int census_window_w, census_window_h;
    double cross_color_tau, cross_color_tau2;
    int cross_arm_l1, cross_arm_l2;
    int box_radius;
    double gauss_sigma;
    double confidence_offset_k;
    int hist_iterations;
    double solver_tol;
    int solver_max_iter;
} dco_config;

/* Device-resident ConstraintSystem (densify.hpp:19-33). Arrays are caller-owned
 * device buffers of width*height elements; scalars are filled on the host. */
typedef struct dco_system {
    int width, height;
    double* diag;
    double* coup_h;
    double* coup_v;
    double* rhs;
    double* initial;
    uint8_t* anchored;
    double constant_term;
    uint64_t anchor_count;
} dco_system;

/* SolveStats (densify.hpp:50-56). residual_history is optional: when
 * history != NULL it receives min(iterations+1, history_cap) norms. */
typedef struct dco_solve_stats {
    int iterations;
    double relative_residual;
    double objective_initial;
    double objective_final;
    double* history;
    int history_cap;
} dco_solve_stats;

typedef struct dco_ctx dco_ctx;

/* ---- context ---------------------------------------------------------- */
int dco_abi_version(void);
int dco_create(int device, dco_ctx** out);
void dco_destroy(dco_ctx* ctx);
const char* dco_last_error(const dco_ctx* ctx);
/* cudaStream_t passed as void* so this header needs no CUDA include. */
int dco_set_stream(dco_ctx* ctx, void* stream);
int dco_synchronize(dco_ctx* ctx);
/* Number of kernels this context has launched (for the bench's launch count). */
uint64_t dco_kernel_launches(const dco_ctx* ctx);
/* Kernel instance that ran this context's last dense solve, e.g.
 * "k_pcg_tmem<7>" (tests pin the headline instance; "" before any solve). */
const char* dco_last_solver(const dco_ctx* ctx);

/* ---- config (config.hpp:11-60, config.cpp:10-36) ----------------------- */
void dco_config_default(dco_config* cfg);
/* PipelineConfig::validate (config.cpp:10-36); message copied into msg. */
int dco_config_validate(const dco_config* cfg, char* msg, size_t msg_len);

/* ---- pyramid (pyramid.hpp:11-15) --------------------------------------- */
/* downsample_half, pyramid.cpp:5-17. out is (w/2) x (h/2). */
int dco_downsample_half(dco_ctx* ctx, const float* img, int w, int h, float* out);
/* read_pnm u8 -> float (codec.cpp:80) fused with downsample_half: gray8 is a
 * w x h byte image; full receives bytes/255.0f, quarter its 2x2 mean. */
int dco_ingest_gray8(dco_ctx* ctx, const uint8_t* gray8, int w, int h, float* full,
                     float* quarter);

/* ---- stereo (stereo.hpp:86-119) ---------------------------------------- */
/* build_cross_windows, stereo.cpp:52-68. */
int dco_build_cross_windows(dco_ctx* ctx, const float* img, int w, int h, const dco_config* cfg,
                            uint8_t* left, uint8_t* right, uint8_t* up, uint8_t* down);
/* census_transform, stereo.cpp:70-96. */
int dco_census_transform(dco_ctx* ctx, const float* img, int w, int h, int window_w,
                         int window_h, uint64_t* out);
/* compute_cost_volume, stereo.cpp:106-150. cost: w*h*(d_max-d_min+1) floats. */
int dco_compute_cost_volume(dco_ctx* ctx, const float* left, const float* right, int w, int h,
                            const uint8_t* arm_left, const uint8_t* arm_right,
                            const uint8_t* arm_up, const uint8_t* arm_down,
                            const dco_config* cfg, float* cost);
/* aggregate_costs, stereo.cpp:152-218. out may not alias cost. */
int dco_aggregate_costs(dco_ctx* ctx, const float* cost, int w, int h, int d_min, int d_max,
                        const uint8_t* arm_left, const uint8_t* arm_right, const uint8_t* arm_up,
                        const uint8_t* arm_down, float* out);
/* select_disparity_wta, stereo.cpp:220-238. */
int dco_select_disparity_wta(dco_ctx* ctx, const float* cost, int w, int h, int d_min, int d_max,
                             float* disparity);
/* refine_disparity_histogram, stereo.cpp:240-299. out may not alias disp. */
int dco_refine_disparity_histogram(dco_ctx* ctx, const float* disp, int w, int h,
                                   const uint8_t* arm_left, const uint8_t* arm_right,
                                   const uint8_t* arm_up, const uint8_t* arm_down, int iterations,
                                   float* out);
/* disparity_to_sparse_depth, stereo.cpp:301-315. */
int dco_disparity_to_sparse_depth(dco_ctx* ctx, const float* disp, int w, int h,
                                  const dco_config* cfg, int full_w, int full_h, float* sparse);
/* The whole stereo chain of pipeline.cpp:184-195 in one call: cross windows,
 * cost, aggregation, WTA, histogram refinement, sparse depth. Intermediates
 * live in the context's scratch pool. disparity (w*h) may be NULL. */
int dco_stereo_sparse_depth(dco_ctx* ctx, const float* left_q, const float* right_q, int w, int h,
                            const dco_config* cfg, int full_w, int full_h, float* disparity,
                            float* sparse);

/* Left-right consistency -- opt-in, not part of the reference (SPEC.md
 * "Non-goals: no left-right cross-checking"). The right view's disparity is the
 * stereo chain on the mirrored pair: dco_flip_horizontal both quarter images,
 * run with left' = mirror(right), right' = mirror(left), mirror the result
 * back. dco_lr_consistency keeps d_L(x) where the right view at x - d_L agrees
 * within max_diff, NaN (nodata) elsewhere. */
int dco_flip_horizontal(dco_ctx* ctx, const float* img, int w, int h, float* out);
int dco_lr_consistency(dco_ctx* ctx, const float* disp_left, const float* disp_right, int w, int h, double max_diff,
                       float* out);

/* ---- flow (flow.hpp:35-50) --------------------------------------------- */
/* compute_flow, flow.cpp:185-205 (pyramid, upsample, DIS patch search). */
int dco_compute_flow(dco_ctx* ctx, const float* from, const float* to, int w, int h,
                     const dco_config* cfg, float* u, float* v);

/* ---- contour (contour.hpp:31-72) --------------------------------------- */
/* flow_to_polar, contour.cpp:10-25. theta may be NULL (unused downstream). */
int dco_flow_to_polar(dco_ctx* ctx, const float* u, const float* v, int w, int h, float* r,
                      float* theta);
/* gradient_amplitude, contour.cpp:27-42. */
int dco_gradient_amplitude(dco_ctx* ctx, const float* r, int w, int h, float* amp);
/* fuse_amplitudes, contour.cpp:82-106. */
int dco_fuse_amplitudes(dco_ctx* ctx, const float* past_u, const float* past_v,
                        const float* future_u, const float* future_v, const float* m_past,
                        const float* m_future, int w, int h, const dco_config* cfg, float* out);
/* box_filter, contour.cpp:108-136. */
int dco_box_filter(dco_ctx* ctx, const float* amp, int w, int h, int radius, float* out);
/* normalize_amplitude, contour.cpp:138-147. out may alias amp. */
int dco_normalize_amplitude(dco_ctx* ctx, const float* amp, int w, int h, float* out);
/* gaussian_blur, contour.cpp:149-175. */
int dco_gaussian_blur(dco_ctx* ctx, const float* img, int w, int h, double sigma, float* out);
/* extract_depth_contours_prefiltered, contour.cpp:177-279. m_fuse is qw x qh. */
int dco_extract_depth_contours_prefiltered(dco_ctx* ctx, const float* blurred, int w, int h,
                                           const float* m_fuse, int qw, int qh,
                                           const dco_config* cfg, uint8_t* edges, float* m_i);
/* extract_depth_contours, contour.cpp:281-285 (blur + the above). */
int dco_extract_depth_contours(dco_ctx* ctx, const float* gray, int w, int h, const float* m_fuse,
                               int qw, int qh, const dco_config* cfg, uint8_t* edges, float* m_i);

/* ---- densify (densify.hpp:41-70) --------------------------------------- */
/* smoothness_weight, densify.cpp:26-35, evaluated for one pair (host scalar). */
int dco_smoothness_weight(dco_ctx* ctx, int px, int py, int qx, int qy, const uint8_t* edges,
                          int w, int h, const float* m_fuse, int qw, int qh, const float* m_i,
                          double* out);
/* assemble_system, densify.cpp:37-116. d_pre may be NULL. sys arrays must be
 * allocated by the caller (w*h each); scalars are written. */
int dco_assemble_system(dco_ctx* ctx, const float* sparse, const uint8_t* edges, const float* m_fuse,
                        int qw, int qh, const float* m_i, const float* d_pre, int w, int h,
                        const dco_config* cfg, dco_system* sys);
/* apply_system, densify.cpp:118-133. */
int dco_apply_system(dco_ctx* ctx, const dco_system* sys, const double* x, double* out);
/* objective_value, densify.cpp:135-139. */
int dco_objective_value(dco_ctx* ctx, const dco_system* sys, const double* x, double* out);
/* solve_dense_depth, densify.cpp:141-222. stats may be NULL. */
int dco_solve_dense_depth(dco_ctx* ctx, const dco_system* sys, const dco_config* cfg,
                          float* dense, dco_solve_stats* stats);

/* ---- composite (occlude.hpp:47-54) ------------------------------------- */
/* composite, occlude.cpp:171-194. real/virt_rgb/out_rgb: 3*w*h floats. */
int dco_composite(dco_ctx* ctx, const float* real_rgb, const float* dense, const float* virt_rgb,
                  const float* virt_depth, int w, int h, float* out_rgb, uint8_t* mask);

/* ---- virtual layer (occlude.hpp:36-48) ----------------- */
/* transform_mesh, occlude.cpp:78-87. vertices/out: 3*num_vertices floats
 * (device); pose: 16 doubles, row-major (HOST). */
int dco_transform_mesh(dco_ctx* ctx, const float* vertices, int num_vertices, const double* pose,
                       float* out);
/* render_virtual, occlude.cpp:107-169. vertices / colors: 3 floats per vertex,
 * triangles: 3 ints per triangle (device). rgb: 3*w*h floats (0 where nothing
 * covers), depth: w*h floats (NaN where nothing covers). Bit-exact with the
 * reference's index-ordered z-buffer (tile-binned, per-pixel ordered). */
int dco_render_virtual(dco_ctx* ctx, const float* vertices, const int* triangles, const float* colors,
                       int num_triangles, double focal_px, double cx, double cy, int width, int height,
                       float* rgb, float* depth);

/* ---- frame orchestration (pipeline.cpp:136-258) ------------------------- */
/* One stream of the pipeline: the KeyframeBuffer window (flow.cpp:10-18), the
 * previous dense map chain (pipeline.cpp:133, 235) and the Unsolvable fallback
 * (pipeline.cpp:236-242), all device-resident. */
typedef struct dco_stream dco_stream;

typedef struct dco_frame_result {
    int composited;          /* 0 until the 3-frame window is full */
    int densify_skipped;     /* UnsolvableFrameError was caught */
    int densify_iterations;
    double densify_objective;
    double relative_residual;
} dco_frame_result;

/* Device outputs of the last composited frame (owned by the stream). */
typedef struct dco_frame_views {
    int full_w, full_h, quarter_w, quarter_h;
    const float* disparity;   /* quarter */
    const float* sparse;      /* full */
    const float* m_fuse;      /* quarter, normalised */
    const float* m_i;         /* full */
    const uint8_t* edges;     /* full */
    const float* dense;       /* full */
    const float* composite;   /* full RGB */
    const uint8_t* mask;      /* full */
    const float* flow_past_u, *flow_past_v, *flow_future_u, *flow_future_v; /* quarter */
    /* the frame's quarter-scale cost and aggregated volumes (stereo.cpp:106-218);
     * volume_layout 0 = the reference's [y][x][d], 1 = slice-major [d][y][x]
     * (the frame loop's fast path) */
    const float* cost_volume;
    const float* aggregated;
    int volume_layout;
    int num_disparities;
} dco_frame_views;

int dco_stream_create(dco_ctx* ctx, int full_w, int full_h, const dco_config* cfg,
                      dco_stream** out);
void dco_stream_destroy(dco_stream* s);
/* Virtual layer used by composite (render_virtual output; device pointers,
 * copied into the stream). NULL clears it: the frame then passes the real
 * colour through with an empty mask (pipeline.cpp:254-257). */
int dco_stream_set_virtual(dco_stream* s, const float* virt_rgb, const float* virt_depth);
/* Virtual mesh rendered on the device for every composited frame
 * (pipeline.cpp:247-252: transform_mesh by the frame's pose, then
 * render_virtual with focal_px and the image centre). HOST arrays, copied:
 * vertices / colors 3 floats per vertex, triangles 3 ints each. Takes
 * precedence over dco_stream_set_virtual; NULL vertices clear it. */
int dco_stream_set_mesh(dco_stream* s, const float* vertices, int num_vertices, const int* triangles,
                        int num_triangles, const float* colors);
/* Pose (16 doubles, row-major, host) of the NEXT pushed frame -- the manifest
 * record's pose (pipeline.cpp:42-47). NULL: that frame's mesh is not
 * transformed. */
int dco_stream_set_next_pose(dco_stream* s, const double* pose);
/* Push one frame (device buffers): 8-bit left/right gray and the left colour
 * as 8-bit RGB (read_color / read_gray of the same PGM give rgb = gray x3;
 * rgb8 may be NULL to mean exactly that). */
int dco_stream_push_gray8(dco_stream* s, const uint8_t* left8, const uint8_t* right8,
                          const uint8_t* rgb8, dco_frame_result* result);
/* Same with float [0,1] inputs (GrayImage/ColorImage data). rgb may be NULL. */
/* The batched throughput entry point (SURVEY 8b "dco_run_streams"):
 * frames_per_stream frames for each of n streams, interleaved (frame f of every
 * stream, then f + 1). left8[k] / right8[k]: frames_per_stream consecutive
 * device-resident w*h u8 frames of stream k. results (may be NULL):
 * n * frames_per_stream entries, stream-major; asking for them synchronises
 * every frame. Errors stop at the failing frame (its stream's error string). */
int dco_run_streams(dco_stream* const* streams, int n, const uint8_t* const* left8, const uint8_t* const* right8,
                    int frames_per_stream, dco_frame_result* results);
int dco_stream_push_f32(dco_stream* s, const float* left, const float* right, const float* rgb,
                        dco_frame_result* result);
/* Host-buffer variant: H2D of the frame, the full frame pipeline, D2H of the
 * composite (3*w*h floats), mask and dense map into the given host buffers
 * (any may be NULL to skip that copy). */
int dco_stream_push_gray8_host(dco_stream* s, const uint8_t* left8, const uint8_t* right8,
                               float* composite_out, uint8_t* mask_out, float* dense_out,
                               dco_frame_result* result);
/* Host-buffer variant with the frame's outputs in the encodings run_pipeline
 * writes them (pipeline.cpp:266-268): the composite as write_ppm's 8-bit RGB
 * bytes (quantize, codec.cpp:23-26 and 221-229; 3*w*h bytes), the mask as
 * write_mask_pgm's bytes (0 / 255, codec.cpp:243-247; w*h), the dense map as
 * the floats write_pfm stores (w*h). Quantised on the device, so 7.4 MB per
 * 1280x720 frame cross PCIe instead of 15.7 MB. Any output may be NULL. */
int dco_stream_push_gray8_host_encoded(dco_stream* s, const uint8_t* left8, const uint8_t* right8,
                                       uint8_t* composite_rgb8, uint8_t* mask8, float* dense_out,
                                       dco_frame_result* result);
int dco_stream_views(const dco_stream* s, dco_frame_views* views);

/* Per-span CUDA-event timing of composited frames: the device-side
 * counterpart of StageTimings (pipeline.hpp:27-46, pipeline.cpp:57-82). The
 * spans refine the reference's 14 stages (cost/aggregate/wta make up
 * "initial parallax"; assemble + solve make up "densification"). */
enum {
    DCO_SPAN_INGEST = 0, /* u8 decode + downsample of the pushed frame    */
    DCO_SPAN_CROSS,      /* adaptive filter area construction            */
    DCO_SPAN_COST,       /* census + AD-census cost volume               */
    DCO_SPAN_AGGREGATE,  /* cross-region aggregation                     */
    DCO_SPAN_WTA,        /* winner-takes-all                              */
    DCO_SPAN_REFINE,     /* parallax optimisation (histogram refinement)  */
    DCO_SPAN_SPARSE,     /* sparse map                                    */
    DCO_SPAN_FLOW,       /* bidirectional optical flow                    */
    DCO_SPAN_FUSION,     /* amplitude + fusion (one kernel)               */
    DCO_SPAN_BOX,        /* box filter                                    */
    DCO_SPAN_NORMALIZE,  /* normalisation                                 */
    DCO_SPAN_BLUR,       /* Gaussian filtering                            */
    DCO_SPAN_CONTOUR,    /* depth contour extraction                      */
    DCO_SPAN_ASSEMBLE,   /* densification: assemble_system                */
    DCO_SPAN_SOLVE,      /* densification: PCG + MR solve                 */
    DCO_SPAN_COMPOSITE,  /* rendering (composite)                         */
    DCO_SPAN_COUNT
};
/* Opt-in left-right consistency on every frame's disparity before the sparse
 * map (not in the reference; default off): see dco_lr_consistency. */
int dco_stream_set_lr_check(dco_stream* s, int enable, double max_diff);
/* Enables (and resets) timing; events ride the stream, no host waits. */
int dco_stream_set_timing(dco_stream* s, int enable);
/* Sum of each span's milliseconds over the timed frames (synchronises). */
int dco_stream_span_times(dco_stream* s, double* ms, uint64_t* frames);
/* Serialisable per-stream state (SURVEY §5 checkpoint): number of bytes. */
size_t dco_stream_state_size(const dco_stream* s);
int dco_stream_save_state(dco_stream* s, void* host_buf, size_t len);
int dco_stream_load_state(dco_stream* s, const void* host_buf, size_t len);

/* ---- ingest / egress (codec.cpp, image.cpp) ------------
 * quantize (codec.cpp:23-26) and to_gray (image.cpp:7-15) on the device, so
 * only bytes cross PCIe; the file formats on the host, byte-for-byte the
 * reference's. The host functions need no context: err (may be NULL)
 * receives the reference's message, e.g. "<path>: truncated payload (byte
 * offset N)"; status DCO_CODEC as CodecError. */
int dco_quantize_u8(dco_ctx* ctx, const float* in, size_t n, uint8_t* out);
int dco_to_gray(dco_ctx* ctx, const float* rgb, int w, int h, float* gray);
/* read_pnm (codec.cpp:59-82): P5 (gray) or P6 (expect_color) with maxval 255.
 * bytes == NULL reads the header only (w, h). */
int dco_read_pnm(const char* path, int expect_color, uint8_t* bytes, size_t cap, int* w, int* h, char* err,
                 size_t err_len);
/* write_pgm / write_ppm (codec.cpp:211-229) of already-quantised bytes. */
int dco_write_pnm(const char* path, const uint8_t* bytes, int w, int h, int channels, char* err, size_t err_len);
/* write_pfm (codec.cpp:293-309): rows bottom-up, nodata written as +inf. */
int dco_write_pfm(const char* path, const float* map, int w, int h, char* err, size_t err_len);

/* ---- row bands (3840x2160 over G GPUs) ------------
 * The quarter-scale rows split into G contiguous bands. Band k computes the
 * stereo chain on its rows plus a recompute halo of (I+1)*l1 + max(Rc,1)
 * rows each side (I = hist_iterations, Rc = census half-height), so every
 * owned row is bit-equal to the whole frame's. The one true exchange is the
 * aggregation's sequential column prefix (stereo.cpp:203-215): band k starts
 * it at carry_row from band k-1's exact prefix (nd * qw doubles, [d][x]) and
 * exports its prefix at carry_out_row to band k+1 -- a chain over bands. No
 * reference function is replaced; this is the multi-GPU split of
 * dco_stereo_sparse_depth (pipeline.cpp:184-195). */
typedef struct dco_band {
    int row0, row1;       /* owned quarter rows [row0, row1)                      */
    int sub0, sub1;       /* quarter rows computed: owned + halo, clipped          */
    int carry_row;        /* quarter row the prefix arrives at; 0 = no carry in     */
    int carry_out_row;    /* row whose prefix goes to band k+1; -1 = none           */
    int frow0, frow1;     /* full-resolution rows of the band's sparse depth        */
    int halo;             /* recompute halo in quarter rows                        */
} dco_band;
int dco_band_plan(const dco_config* cfg, int full_w, int full_h, int bands, int index, dco_band* out);
/* Bytes of one carry buffer: (d_max - d_min + 1) * (full_w / 2) doubles, [d][x]. */
size_t dco_band_carry_bytes(const dco_config* cfg, int full_w);
/* Stereo chain of one band. left_sub / right_sub: quarter rows [sub0, sub1)
 * (qw = full_w / 2 wide). carry_in: required when carry_row > 0; carry_out:
 * written when carry_out_row >= 0. disparity: (row1-row0)*qw, may be NULL;
 * sparse: full rows [frow0, frow1) of full_w. */
int dco_stereo_band(dco_ctx* ctx, const float* left_sub, const float* right_sub, const dco_band* band,
                    const dco_config* cfg, int full_w, int full_h, const double* carry_in, double* carry_out,
                    float* disparity, float* sparse);
/* The same in three phases, so that under a multi-GPU chain only the vertical
 * pass waits for the carry, and the carry can travel in disparity chunks:
 * begin (cross windows, cost, horizontal pass), vpass over slices [d0, d1)
 * (d0 a multiple of 32; carry buffers of (d1-d0) * qw doubles, [d][x]), end
 * (WTA, refinement, sparse). State lives in the context between the calls:
 * no other stereo call on ctx until end. */
int dco_stereo_band_begin(dco_ctx* ctx, const float* left_sub, const float* right_sub, const dco_band* band,
                          const dco_config* cfg, int full_w, int full_h);
int dco_stereo_band_vpass(dco_ctx* ctx, const dco_band* band, const dco_config* cfg, int full_w, int full_h, int d0,
                          int d1, const double* carry_in, double* carry_out);
int dco_stereo_band_end(dco_ctx* ctx, const dco_band* band, const dco_config* cfg, int full_w, int full_h,
                        float* disparity, float* sparse);

/* Row-band densify (SURVEY 8e "1-row p halo per SpMV plus an all-reduce of
 * the scalar groups per iteration"): the PCG + MR solve of one frame's system
 * with rank k owning full rows [row0, row0 + rows). One persistent kernel per
 * GPU; the per-iteration reduction and the p halo cross GPUs through peer
 * memory (CUDA IPC over NVLink), not NCCL calls between launches. The
 * system passed to a solve is the band's: width x rows arrays starting at the
 * band's first row, coup_v readable one row above it when row0 > 0. The
 * Krylov scalars are the same on every rank; the result matches
 * dco_solve_dense_depth within the solver tolerance (densify.cpp:141-222). */
/* Row-band assembly (densify.cpp:37-116). The frame-wide sparse mean
 * (densify.cpp:60-68) is the one global input: every band reports
 * {sum, sum of |v|, count, min ulp exponent} of its owned rows (host doubles),
 * the ranks exchange them, and dco_band_sparse_mean combines them in rank
 * order -- exact (the sequential sum's bits) whenever the guard holds
 * (*exact = 1); otherwise the caller gathers the full sparse map and uses
 * dco_sparse_mean. dco_band_assemble fills the system of the sub-frame rows it
 * is given (inputs offset to the sub-frame's first row, an even full row;
 * m_fuse offset by half of it) with the frame's mean, and returns anchors and
 * constant term of the owned sub-frame rows [own0, own0 + own_rows). */
int dco_band_sparse_stats(dco_ctx* ctx, const float* sparse_rows, size_t n, double* out4);
int dco_band_sparse_mean(const double* stats, int bands, double* mean, int* exact);
int dco_sparse_mean(dco_ctx* ctx, const float* sparse, size_t n, double* mean);
int dco_band_assemble(dco_ctx* ctx, const float* sparse, const uint8_t* edges, const float* m_fuse, int qw, int qh,
                      const float* m_i, const float* d_pre, int w, int h, int own0, int own_rows,
                      const dco_config* cfg, double sparse_mean, dco_system* sys, uint64_t* anchors,
                      double* constant);

#define DCO_BAND_HANDLE_BYTES 128
typedef struct dco_band_solver dco_band_solver;
int dco_band_solver_create(dco_ctx* ctx, int ranks, int rank, int width, int row0, int rows, int full_height,
                           dco_band_solver** out);
void dco_band_solver_destroy(dco_band_solver* s);
/* One process per GPU: export this rank's handle (DCO_BAND_HANDLE_BYTES), gather
 * every rank's (e.g. over torch.distributed), connect with the rank-ordered table. */
int dco_band_solver_export(dco_band_solver* s, void* handle);
int dco_band_solver_connect(dco_band_solver* s, const void* handles);
int dco_band_solve(dco_band_solver* s, const dco_system* sys, const dco_config* cfg, uint64_t anchors_total,
                   double constant_total, float* dense, dco_solve_stats* stats);
/* Every rank in this process on one context (fewer GPUs than ranks): one
 * cooperative launch runs all ranks as block groups. sys, dense, stats: [ranks]. */
int dco_band_solver_connect_local(dco_band_solver* const* solvers, int ranks);
int dco_band_solve_local(dco_band_solver* const* solvers, int ranks, const dco_system* sys, const dco_config* cfg,
                         uint64_t anchors_total, double constant_total, float* const* dense,
                         dco_solve_stats* stats);

#if defined(__GNUC__)
#pragma GCC visibility pop
#endif
#ifdef __cplusplus
}
#endif

#endif /* DCO_GPU_H */
