/* dco_oracle.h — plain-C restatement of the reference's DCO hot path.
 *
 * TEST INFRASTRUCTURE ONLY (the checker, never the product): used by tests/,
 * __graft_entry__.smoke() and bench.py's CPU legs. Each function restates the
 * reference function named in its comment (paths relative to
 * /root/reference/proj), calls the host libm exactly where the reference does,
 * and is pinned bit-for-bit against the compiled reference (oracle/_ref) by
 * tests/test_oracle_port.py. Arrays are row-major; NaN = nodata; return value
 * 0 = ok, otherwise a dco_status code (include/dco_gpu.h). */
#ifndef DCO_ORACLE_H
#define DCO_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#include "../include/dco_gpu.h"

#ifdef __cplusplus
extern "C" {
#endif

const char* dco_o_error(void);
int dco_o_validate(const dco_config* c);

int dco_o_downsample_half(const float* img, int w, int h, float* out);
int dco_o_cross_windows(const float* img, int w, int h, const dco_config* c, uint8_t* l, uint8_t* r, uint8_t* u,
                        uint8_t* d);
int dco_o_census(const float* img, int w, int h, int ww, int wh, uint64_t* out);
int dco_o_cost_volume(const float* left, const float* right, int w, int h, const uint8_t* l, const uint8_t* r,
                      const uint8_t* u, const uint8_t* d, const dco_config* c, float* cost);
int dco_o_aggregate(const float* cost, int w, int h, int nd, const uint8_t* l, const uint8_t* r, const uint8_t* u,
                    const uint8_t* d, float* out);
int dco_o_wta(const float* cost, int w, int h, int d_min, int nd, float* disp);
int dco_o_refine(const float* disp, int w, int h, const uint8_t* l, const uint8_t* r, const uint8_t* u,
                 const uint8_t* d, int iters, float* out);
int dco_o_sparse_depth(const float* disp, int w, int h, const dco_config* c, int fw, int fh, float* out);

int dco_o_flow(const float* from, const float* to, int w, int h, float* u, float* v);

int dco_o_polar(const float* u, const float* v, int n, float* r, float* theta);
int dco_o_gradient_amplitude(const float* r, int w, int h, float* amp);
int dco_o_fuse(const float* pu, const float* pv, const float* fu, const float* fv, const float* mp, const float* mf,
               int w, int h, double k, float* out);
int dco_o_box(const float* a, int w, int h, int radius, float* out);
int dco_o_normalize(const float* a, int n, float* out);
int dco_o_gauss(const float* img, int w, int h, double sigma, float* out);
int dco_o_contours(const float* blurred, int w, int h, const float* mf, int qw, int qh, const dco_config* c,
                   uint8_t* edges, float* m_i);

int dco_o_assemble(const float* sparse, const uint8_t* edges, const float* mf, int qw, int qh, const float* mi,
                   const float* pre, int w, int h, const dco_config* c, double* diag, double* ch, double* cv,
                   double* rhs, double* init, uint8_t* anchored, double* constant_term, uint64_t* anchor_count);
int dco_o_apply(int w, int h, const double* diag, const double* ch, const double* cv, const double* x,
                double* out);
int dco_o_solve(int w, int h, const double* diag, const double* ch, const double* cv, const double* rhs,
                const double* init, uint64_t anchor_count, double constant_term, const dco_config* c, float* dense,
                int* iterations, double* relres, double* obj0, double* obj1);
int dco_o_composite(const float* real, const float* dense, const float* vrgb, const float* vdepth, int w, int h,
                    float* out, uint8_t* mask);

#ifdef __cplusplus
}
#endif

#endif
