// densify.cu — the three-constraint quadratic densification (reference
// src/densify.cpp): assembly of the 5-point normal equations and the
// Jacobi-preconditioned CG with minimal-residual smoothing, in FP64.
//
// assemble_system is bit-exact: per-pixel terms are evaluated in the
// reference's order (diag: data, stability, up-coupling, left-coupling, own
// right, own down — densify.cpp:70-114) and the sparse mean uses a double
// tree that is provably exact whenever every partial sum is representable
// (checked on the device; otherwise the reference's sequential sum runs).
//
// solve_dense_depth is ONE persistent cooperative kernel: every block owns a
// fixed slice of the unknowns, the four reductions per iteration (pq, rho +
// MR numerators, |rs|^2) are fixed-shape trees, and the loop/termination
// logic of densify.cpp:174-211 runs on the device, so an entire solve is one
// launch with no host round trip. Reductions are deterministic (bit-stable
// run to run) but not in the reference's sequential order, so the dense map
// matches the oracle within tolerance, not bit for bit.
#include <cooperative_groups.h>
#include <math.h>

#include <mutex>
#include <set>
#include <string>

#include "common.cuh"
#include "grid_reduce.cuh"

namespace cg = cooperative_groups;

namespace dco_gpu {
namespace {

__device__ __forceinline__ double dmin(double a, double b) { return (b < a) ? b : a; }   // std::min
__device__ __forceinline__ double dmax0(double a) { return (a < 0.0) ? 0.0 : a; }        // std::max(a, 0.0)

// fused_confidence, densify.cpp:11-16.
__device__ __forceinline__ double fused_conf(const float* mf, int qw, int qh, int x, int y) {
    int mx = min(x / 2, qw - 1), my = min(y / 2, qh - 1);
    float v = mf[static_cast<size_t>(my) * qw + mx];
    return isfinite(v) ? static_cast<double>(v) : 0.0;
}

// smoothness_weight, densify.cpp:26-35: smooth_w_s in k_assemble.

struct AsmArgs {
    int w, h, qw, qh;
    double lambda_d, lambda_s, lambda_s2;
    const float* sparse;
    const uint8_t* edges;
    const float* mf;
    const float* mi;
    const float* pre;      // nullable
    const int* pre_valid;  // nullable: pre is used only when *pre_valid != 0
    double* diag;
    double* ch;
    double* cv;
    double* rhs;
    double* init;
    uint8_t* anchored;
    const double* sparse_mean;  // device scalar
};

// assemble_system per-pixel part, densify.cpp:70-114.
// One 32x8 block per tile; s = fused_conf * m_i and the contour flag of the
// tile and its one-pixel halo are computed once into shared memory, so each
// of the four edge weights reads them there (smoothness_weight would compute
// each endpoint's s twice per edge and every s four times per frame).
__device__ __forceinline__ double smooth_w_s(uint8_t ep, uint8_t eq, double sp, double sq) {
    if ((ep ? 1 : 0) + (eq ? 1 : 0) == 1) return 0.0;  // densify.cpp:26-35
    return dmax0(1.0 - dmin(sp, sq));
}
__global__ void __launch_bounds__(256) k_assemble(AsmArgs a) {
    __shared__ double s_s[10][34];
    __shared__ uint8_t s_e[10][34];
    const int w = a.w, h = a.h;
    const int bx0 = blockIdx.x * blockDim.x - 1, by0 = blockIdx.y * blockDim.y - 1;
    for (int k = threadIdx.y * blockDim.x + threadIdx.x; k < 10 * 34; k += blockDim.x * blockDim.y) {
        const int ty = k / 34, tx = k - ty * 34;
        const int gx = bx0 + tx, gy = by0 + ty;
        double sv = 0.0;
        uint8_t ev = 0;
        if (gx >= 0 && gx < w && gy >= 0 && gy < h) {
            const size_t ip = static_cast<size_t>(gy) * w + gx;
            ev = a.edges[ip];
            sv = fused_conf(a.mf, a.qw, a.qh, gx, gy) * a.mi[ip];
        }
        s_s[ty][tx] = sv;
        s_e[ty][tx] = ev;
    }
    __syncthreads();
    int x = blockIdx.x * blockDim.x + threadIdx.x;
    int y = blockIdx.y * blockDim.y + threadIdx.y;
    if (x >= w || y >= h) return;
    const int tx = threadIdx.x + 1, ty = threadIdx.y + 1;
    size_t i = static_cast<size_t>(y) * w + x;
    if (a.pre && a.pre_valid && *a.pre_valid == 0) a.pre = nullptr;
    const double two_ls = 2.0 * a.lambda_s;
    double diag = 0.0, rhs = 0.0, init = *a.sparse_mean;
    uint8_t anch = 0;
    float s = a.sparse[i];
    if (isfinite(s)) {
        double ds = s;
        diag += a.lambda_d;
        rhs += a.lambda_d * ds;
        anch = 1;
        init = ds;
    } else if (a.pre && isfinite(a.pre[i])) {
        init = a.pre[i];
    }
    if (a.pre && isfinite(a.pre[i])) {
        double dp = a.pre[i];
        diag += a.lambda_s2;
        rhs += a.lambda_s2 * dp;
        anch = 1;
    }
    const uint8_t e0 = s_e[ty][tx];
    const double s0 = s_s[ty][tx];
    if (y > 0) diag += two_ls * smooth_w_s(s_e[ty - 1][tx], e0, s_s[ty - 1][tx], s0);
    if (x > 0) diag += two_ls * smooth_w_s(s_e[ty][tx - 1], e0, s_s[ty][tx - 1], s0);
    double chv = 0.0, cvv = 0.0;
    if (x + 1 < w) {
        chv = two_ls * smooth_w_s(e0, s_e[ty][tx + 1], s0, s_s[ty][tx + 1]);
        diag += chv;
    }
    if (y + 1 < h) {
        cvv = two_ls * smooth_w_s(e0, s_e[ty + 1][tx], s0, s_s[ty + 1][tx]);
        diag += cvv;
    }
    a.diag[i] = diag;
    a.ch[i] = chv;
    a.cv[i] = cvv;
    a.rhs[i] = rhs;
    a.init[i] = init;
    a.anchored[i] = anch;
}

// Block-wide deterministic sum of K doubles per thread (fixed shuffle tree).
template <int K>
__device__ __forceinline__ void block_sum(double (&v)[K], double* smem /* [32*K] */) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
#pragma unroll
    for (int k = 0; k < K; ++k)
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) v[k] += __shfl_xor_sync(0xffffffffu, v[k], off);
    __syncthreads();
    if (lane == 0)
#pragma unroll
        for (int k = 0; k < K; ++k) smem[warp * K + k] = v[k];
    __syncthreads();
    if (warp == 0) {
#pragma unroll
        for (int k = 0; k < K; ++k) {
            double t = lane < nw ? smem[lane * K + k] : 0.0;
#pragma unroll
            for (int off = 16; off > 0; off >>= 1) t += __shfl_xor_sync(0xffffffffu, t, off);
            v[k] = t;
        }
    }
    __syncthreads();
    if (threadIdx.x == 0)
#pragma unroll
        for (int k = 0; k < K; ++k) smem[k] = v[k];
    __syncthreads();
#pragma unroll
    for (int k = 0; k < K; ++k) v[k] = smem[k];
    __syncthreads();
}

// Sparse statistics: valid count, min ulp exponent, sum of |v| and the double
// tree sum (exact under the guard), anchor count and constant term partials.
struct SparseStats {
    unsigned long long count;
    int min_exp;
    double abs_sum;
    double sum;
};

__global__ void k_sparse_stats(const float* __restrict__ s, size_t n, double* __restrict__ part,
                               unsigned long long* __restrict__ count, int* __restrict__ min_exp) {
    __shared__ double sm[32 * 2];
    double v[2] = {0.0, 0.0};
    unsigned long long c = 0;
    int me = 1 << 20;
    constexpr int kB = 4;  // loads of kB elements in flight, grid-stride order kept
    const size_t stride = static_cast<size_t>(gridDim.x) * blockDim.x;
    for (size_t i0 = static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x; i0 < n; i0 += kB * stride) {
        float fs[kB];
#pragma unroll
        for (int j = 0; j < kB; ++j) fs[j] = i0 + j * stride < n ? s[i0 + j * stride] : __int_as_float(0x7fc00000);
#pragma unroll
        for (int j = 0; j < kB; ++j) {
            const float f = fs[j];
            if (isfinite(f)) {
                v[0] += f;
                v[1] += fabs(static_cast<double>(f));
                ++c;
                if (f != 0.0f) {
                    int e;
                    frexpf(f, &e);  // f = m * 2^e, m in [0.5,1): ulp = 2^(e-24), denormal-safe bound
                    me = min(me, max(e - 24, -149));
                }
            }
        }
    }
    block_sum<2>(v, sm);
    if (threadIdx.x == 0) {
        part[2 * blockIdx.x] = v[0];
        part[2 * blockIdx.x + 1] = v[1];
    }
    block_atomic_add(count, c);
    block_atomic_min(min_exp, me, 1 << 20);
}

// Finishes the sparse mean (densify.cpp:60-68): exact tree when the guard
// holds, the reference's sequential loop otherwise (single thread, rare).
__global__ void k_sparse_mean(const float* __restrict__ s, size_t n, const double* __restrict__ part,
                              int nparts, const unsigned long long* __restrict__ count,
                              const int* __restrict__ min_exp, double* __restrict__ mean) {
    __shared__ double sm[32 * 2];
    double v[2] = {0.0, 0.0};
    for (int b = threadIdx.x; b < nparts; b += blockDim.x) {
        v[0] += part[2 * b];
        v[1] += part[2 * b + 1];
    }
    block_sum<2>(v, sm);
    if (threadIdx.x != 0) return;
    unsigned long long c = *count;
    if (c == 0) {
        *mean = 0.0;
        return;
    }
    double sum = v[0];
    // all partial sums are multiples of 2^min_exp bounded by abs_sum: exact
    // in double iff abs_sum < 2^(53 + min_exp) (margin for the bound's own rounding)
    double limit = ldexp(1.0, 53 + *min_exp);
    if (!(v[1] * (1.0 + 1e-9) < limit)) {
        sum = 0.0;
        for (size_t i = 0; i < n; ++i) {
            float f = s[i];
            if (isfinite(f)) sum += f;
        }
    }
    *mean = sum / static_cast<double>(c);
}

// anchor count and constant term (densify.cpp:70-94, 113): tree sums.
__global__ void k_anchor_const(const uint8_t* __restrict__ anch, const float* __restrict__ s,
                               const float* __restrict__ pre, const int* __restrict__ pre_valid, size_t n,
                               double ld, double ls2, unsigned long long* __restrict__ count,
                               double* __restrict__ part) {
    __shared__ double sm[32];
    if (pre && pre_valid && *pre_valid == 0) pre = nullptr;
    double v[1] = {0.0};
    unsigned long long c = 0;
    // the thread's elements in the same order as a plain grid-stride loop,
    // with the loads of kB of them issued before any is used
    constexpr int kB = 4;
    const size_t stride = static_cast<size_t>(gridDim.x) * blockDim.x;
    for (size_t i0 = static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x; i0 < n; i0 += kB * stride) {
        float f[kB], g[kB];
        unsigned a[kB];
#pragma unroll
        for (int j = 0; j < kB; ++j) {
            const size_t i = i0 + j * stride;
            const bool in = i < n;
            a[j] = in ? anch[i] : 0u;
            f[j] = in ? s[i] : __int_as_float(0x7fc00000);
            g[j] = in && pre ? pre[i] : __int_as_float(0x7fc00000);
        }
#pragma unroll
        for (int j = 0; j < kB; ++j) {
            c += a[j];
            if (isfinite(f[j])) {
                double ds = f[j];
                v[0] += ld * ds * ds;
            }
            if (isfinite(g[j])) {
                double dp = g[j];
                v[0] += ls2 * dp * dp;
            }
        }
    }
    block_sum<1>(v, sm);
    if (threadIdx.x == 0) part[blockIdx.x] = v[0];
    block_atomic_add(count, c);
}

// (sum, |sum|) of k_sparse_stats' block partials
__global__ void k_sparse_pair_sums(const double* __restrict__ part, int nparts, double* __restrict__ out) {
    __shared__ double sm[32 * 2];
    double v[2] = {0.0, 0.0};
    for (int b = threadIdx.x; b < nparts; b += blockDim.x) {
        v[0] += part[2 * b];
        v[1] += part[2 * b + 1];
    }
    block_sum<2>(v, sm);
    if (threadIdx.x == 0) {
        out[0] = v[0];
        out[1] = v[1];
    }
}

__global__ void k_reduce_parts(const double* __restrict__ part, int nparts, double* __restrict__ out) {
    __shared__ double sm[32];
    double v[1] = {0.0};
    for (int b = threadIdx.x; b < nparts; b += blockDim.x) v[0] += part[b];
    block_sum<1>(v, sm);
    if (threadIdx.x == 0) *out = v[0];
}

// apply_system, densify.cpp:118-133 (stencil order kept).
__device__ __forceinline__ double apply_at(const double* __restrict__ diag, const double* __restrict__ ch,
                                           const double* __restrict__ cv, const double* __restrict__ x,
                                           int w, int h, size_t i, int xx, int y) {
    double acc = diag[i] * x[i];
    if (xx + 1 < w) acc -= ch[i] * x[i + 1];
    if (xx > 0) acc -= ch[i - 1] * x[i - 1];
    if (y + 1 < h) acc -= cv[i] * x[i + w];
    if (y > 0) acc -= cv[i - w] * x[i - w];
    return acc;
}

__global__ void k_apply(const double* __restrict__ diag, const double* __restrict__ ch,
                        const double* __restrict__ cv, const double* __restrict__ x, int w, int h,
                        double* __restrict__ out) {
    int xx = blockIdx.x * blockDim.x + threadIdx.x;
    int y = blockIdx.y * blockDim.y + threadIdx.y;
    if (xx >= w || y >= h) return;
    size_t i = static_cast<size_t>(y) * w + xx;
    out[i] = apply_at(diag, ch, cv, x, w, h, i, xx, y);
}

// objective_value partials: dot(x, Ax) and dot(b, x).
__global__ void k_objective(const double* __restrict__ diag, const double* __restrict__ ch,
                            const double* __restrict__ cv, const double* __restrict__ rhs,
                            const double* __restrict__ x, int w, int h, double* __restrict__ part) {
    __shared__ double sm[64];
    double v[2] = {0.0, 0.0};
    size_t n = static_cast<size_t>(w) * h;
    for (size_t i = static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
         i += static_cast<size_t>(gridDim.x) * blockDim.x) {
        int xx = static_cast<int>(i % w), y = static_cast<int>(i / w);
        v[0] += x[i] * apply_at(diag, ch, cv, x, w, h, i, xx, y);
        v[1] += rhs[i] * x[i];
    }
    block_sum<2>(v, sm);
    if (threadIdx.x == 0) {
        part[2 * blockIdx.x] = v[0];
        part[2 * blockIdx.x + 1] = v[1];
    }
}
__global__ void k_objective_finish(const double* __restrict__ part, int nparts, double c,
                                   double* __restrict__ out) {
    __shared__ double sm[64];
    double v[2] = {0.0, 0.0};
    for (int b = threadIdx.x; b < nparts; b += blockDim.x) {
        v[0] += part[2 * b];
        v[1] += part[2 * b + 1];
    }
    block_sum<2>(v, sm);
    if (threadIdx.x == 0) *out = v[0] - 2.0 * v[1] + c;
}

// ----------------------------------------------------------------- solver --
struct SolveOut {
    int status;  // 0 ok, 3 unsolvable
    int iterations;
    double relative_residual;
    double objective_initial;
    double objective_final;
};

struct CGArgs {
    int w, h;
    size_t n;
    const double* diag;
    const double* ch;
    const double* cv;
    const double* rhs;
    const double* init;
    double constant_term_host;
    const double* constant_term_dev;  // used when non-null
    const unsigned long long* anchors_dev;
    unsigned long long anchors_host;
    double* prec;
    double* x;
    double* r;
    double* z;
    double* p;
    double* q;
    double* rs;
    double* xs;
    double* part;  // [gridDim.x][4]
    double* hist;
    int hist_cap;
    int max_iter;
    double tol;
    float* dense;
    const float* fallback;    // unsolvable: dense = fallback (or NaN when null)
    const int* fallback_valid;  // nullable: fallback usable only when *fallback_valid
    SolveOut* out;
    long long* dbg;  // optional per-phase clock64 stamps of block 0 (DCO_PCG_DEBUG)
};


// ------------------------------------------------- on-chip resident solver --
// Same Krylov iterates as k_pcg, but each of the grid's blocks (one per SM,
// 1024 threads) owns a contiguous chunk of unknowns for the whole solve: r and
// x in registers (EPT per thread), p / xs / rs / q in shared memory. Only a
// one-row halo crosses blocks per iteration; the coefficient arrays and the
// Jacobi preconditioner stream from L2. One grid barrier + deterministic
// all-reduce per iteration (grid_reduce.cuh).
template <int EPT, int THREADS>
__global__ void __launch_bounds__(THREADS, 1) k_pcg_onchip(CGArgs a, int chunk, GridBar* bar) {
    // Block b owns [base, base + size): sizes differ by at most one. r and x
    // in registers; p (with a one-row halo either side), xs, rs, q in shared
    // memory. One grid barrier per iteration: every scalar of iteration k
    // (pq, rho_{k+1}, sd, dd) is a polynomial in alpha_k of sums that are
    // known once q_k = A p_k is, so they ride on one reduction:
    //   rho_{k+1} = S1 - 2 a S2 + a^2 S3   (S = sum prec r r, prec r q, prec q q)
    //   sd        = T1 - a T2              (T = sum rs (r - rs), rs q)
    //   dd        = U1 - 2 a U2 + a^2 U3   (U = sum (r-rs)^2, (r-rs) q, q q)
    // The vector updates of iteration k then run at the head of phase k+1,
    // together with |rs|^2 (the reported norm, one phase late). The halo of
    // p_{k+1} is recomputed from the (r, q, p) rows the neighbouring blocks
    // publish in phase k, with the owner's FMA sequence (same bits). Same
    // Krylov iterates as densify.cpp:172-207 in exact arithmetic; tolerance-
    // matched (not bit-exact) in floating point.
    extern __shared__ double sx[];  // p [w + chunk + w], then xs, rs, q [chunk] each
    __shared__ double sm[32 * 16];
    __shared__ double s_w1[32 * 4];  // per-warp P1 sums
    const int w = a.w, h = a.h;
    const int n = static_cast<int>(a.n);
    const int nb = gridDim.x;
    const int qn = n / nb, rem = n - qn * nb;
    const int base = blockIdx.x * qn + min(static_cast<int>(blockIdx.x), rem);
    const int size = qn + (static_cast<int>(blockIdx.x) < rem ? 1 : 0);
    const int t = threadIdx.x;
    const int nv = size > t ? (size - t + THREADS - 1) / THREADS : 0;  // occupied register slots
    double* s_p = sx + w + t;
    double* s_xs = sx + 2 * w + chunk + t;
    double* s_rs = sx + 2 * w + 2 * chunk + t;
    double* s_q = sx + 2 * w + 3 * chunk + t;
    const double* __restrict__ diag = a.diag + base + t;
    const double* __restrict__ ch = a.ch + base + t;
    const double* __restrict__ cv = a.cv + base + t;
    const double* __restrict__ prec = a.prec + base + t;
    // halo rows published per phase parity: (r, q, p) in (a.r, a.q, a.p) / (a.x, a.z, a.rs)
    unsigned gen = 0;  // barriers completed in this solve (bar->count was zeroed at launch)
    double r[EPT], x[EPT];
    uint64_t nbr = 0;  // 4 bits per slot (EPT <= 16): 1 right, 2 left, 4 down, 8 up
    unsigned pub = 0;  // bit k: slot k lies in a row other blocks read as halo
#define DCO_OK(k) ((k) < nv)
#define KO(k) ((k) * THREADS)

    unsigned long long anchors = a.anchors_dev ? *a.anchors_dev : a.anchors_host;
    if (anchors == 0) {
        const float* fb = (a.fallback && (!a.fallback_valid || *a.fallback_valid)) ? a.fallback : nullptr;
        for (int i = base + t; i < base + size; i += THREADS) a.dense[i] = fb ? fb[i] : __int_as_float(0x7fc00000);
        if (blockIdx.x == 0 && t == 0) {
            a.out->status = 3;
            a.out->iterations = 0;
        }
        return;
    }
    const double cterm = a.constant_term_dev ? *a.constant_term_dev : a.constant_term_host;

    // setup (densify.cpp:147-166): x = initial, r = b - A x, z = M r, p = z
    // (p_0 published whole in a.xs for phase 0's halo)
    double tot[5] = {0.0, 0.0, 0.0, 0.0, 0.0};  // b.b, r.r, r.z, x.Ax, b.x
    {
#pragma unroll
        for (int k = 0; k < EPT; ++k) {
            r[k] = 0.0;
            x[k] = 0.0;
            if (DCO_OK(k)) {
                const int i = base + t + KO(k);
                const int xx = i % w, y = i / w;
                nbr |= static_cast<uint64_t>((xx + 1 < w ? 1u : 0u) | (xx > 0 ? 2u : 0u) | (y + 1 < h ? 4u : 0u) |
                                             (y > 0 ? 8u : 0u)) << (4 * k);
                if (t + KO(k) < w || t + KO(k) >= size - w) pub |= 1u << k;
                double ax = apply_at(a.diag, a.ch, a.cv, a.init, w, h, i, xx, y);
                double xi = a.init[i];
                double b = a.rhs[i];
                double d = a.diag[i];
                double pr = d > 0.0 ? 1.0 / d : 1.0;
                double ri = b - ax;
                double zi = pr * ri;
                x[k] = xi;
                s_xs[KO(k)] = xi;
                s_rs[KO(k)] = ri;
                s_p[KO(k)] = zi;
                a.prec[i] = pr;
                r[k] = ri;
                a.xs[i] = zi;
                tot[0] += b * b;
                tot[1] += ri * ri;
                tot[2] += ri * zi;
                tot[3] += xi * ax;
                tot[4] += b * xi;
            }
        }
        barrier_reduce<5>(tot, bar, a.part, gen, sm, tot);
    }
    const double bnorm = sqrt(tot[0]);
    const double denom = bnorm > 0.0 ? bnorm : 1.0;
    double snorm = sqrt(tot[1]);
    double rho = tot[2];
    if (blockIdx.x == 0 && t == 0) {
        if (a.hist_cap > 0) a.hist[0] = snorm;
        a.out->objective_initial = tot[3] - 2.0 * tot[4] + cterm;
    }

    int iter = 0;
    double alpha = 0.0, beta = 0.0, eta = 0.0;  // iteration iter-1's scalars, applied at the head of phase iter
#define STAMP(j)                                                                                      \
    if (a.dbg && t == 0 && iter < 64) {                                                               \
        if (blockIdx.x == 0 || blockIdx.x == gridDim.x - 1)                                           \
            a.dbg[(blockIdx.x ? 640 : 0) + iter * 10 + (j)] = clock64();                              \
        if ((j) < 3) {                                                                                \
            unsigned long long gt;                                                                    \
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(gt));                                   \
            a.dbg[1280 + (iter * 1024 + blockIdx.x) * 3 + (j)] = static_cast<long long>(gt);          \
        }                                                                                             \
    }
    if (a.max_iter > 0 && snorm / denom > a.tol) {
        for (;;) {
            STAMP(0)
            // opaque per iteration: keeps the compiler from hoisting (and
            // spilling) per-slot bit tests out of the loop
            asm volatile("" : "+r"(pub), "+l"(nbr));
            const int par = iter & 1;
            double* const hr_in = par ? a.r : a.x;  // published in phase iter-1
            double* const hq_in = par ? a.q : a.z;
            double* const hp_in = par ? a.p : a.rs;
            double* const hr_out = par ? a.x : a.r;
            double* const hq_out = par ? a.z : a.q;
            double* const hp_out = par ? a.rs : a.p;
            // halo rows [-w, 0) and [size, size + w): p_iter of the neighbours,
            // recomputed with the owner's FMA sequence
            {
                constexpr int kHalo = 3;
                double h0[kHalo], h1[kHalo], h2[kHalo], h3[kHalo];
#pragma unroll
                for (int u = 0; u < kHalo; ++u) {
                    const int e = t + u * THREADS;
                    const int j = base + (e < w ? e - w : size + (e - w));
                    h0[u] = h1[u] = h2[u] = h3[u] = 0.0;
                    if (e < 2 * w && j >= 0 && j < n) {
                        if (iter) {
                            h0[u] = __ldcg(hr_in + j);
                            h1[u] = __ldcg(hq_in + j);
                            h2[u] = __ldcg(hp_in + j);
                            h3[u] = __ldg(a.prec + j);
                        } else {
                            h2[u] = __ldcg(a.xs + j);
                        }
                    }
                }
#pragma unroll
                for (int u = 0; u < kHalo; ++u) {
                    const int e = t + u * THREADS;
                    const int l = e < w ? e - w : size + (e - w);
                    const int j = base + l;
                    if (e < 2 * w && j >= 0 && j < n)
                        sx[w + l] = iter ? __fma_rn(beta, h2[u], h3[u] * __fma_rn(-alpha, h1[u], h0[u])) : h2[u];
                }
                for (int e = t + kHalo * THREADS; e < 2 * w; e += THREADS) {  // w > 1.5 * THREADS only
                    const int l = e < w ? e - w : size + (e - w);
                    const int j = base + l;
                    if (j >= 0 && j < n) {
                        double pj;
                        if (iter) {
                            const double rj = __fma_rn(-alpha, __ldcg(hq_in + j), __ldcg(hr_in + j));
                            pj = __fma_rn(beta, __ldcg(hp_in + j), __ldg(a.prec + j) * rj);
                        } else {
                            pj = __ldcg(a.xs + j);
                        }
                        sx[w + l] = pj;
                    }
                }
            }
            // P1: vector updates of iteration iter-1 (densify.cpp:178-201), then
            // sums over the updated r / rs: |rs|^2, S1, T1, U1; publish (r, p) rows
            double v[10];
#pragma unroll
            for (int c = 0; c < 10; ++c) v[c] = 0.0;
#pragma unroll
            for (int k = 0; k < EPT; ++k) {
                if (DCO_OK(k)) {
                    const int o = KO(k);
                    double pk = s_p[o];
                    double ri = r[k];
                    double rsi = s_rs[o];
                    const double pr = prec[o];
                    if (iter) {
                        x[k] = __fma_rn(alpha, pk, x[k]);
                        ri = __fma_rn(-alpha, s_q[o], ri);
                        pk = __fma_rn(beta, pk, pr * ri);
                        r[k] = ri;
                        s_p[o] = pk;
                        if (eta > 0.0) {
                            rsi = __fma_rn(eta, ri - rsi, rsi);
                            s_rs[o] = rsi;
                            double xsi = s_xs[o];
                            s_xs[o] = __fma_rn(eta, x[k] - xsi, xsi);
                        }
                    }
                    const double e = ri - rsi;
                    v[1] = __fma_rn(rsi, rsi, v[1]);
                    v[2] = __fma_rn(pr * ri, ri, v[2]);
                    v[3] = __fma_rn(rsi, e, v[3]);
                    v[4] = __fma_rn(e, e, v[4]);
                    if (pub & (1u << k)) {  // rows other blocks read as halo
                        __stcg(hr_out + base + t + o, ri);
                        __stcg(hp_out + base + t + o, pk);
                    }
                }
            }
            // P1 sums -> per-warp partials in shared memory (frees registers for P2)
            {
                const int lane = t & 31, warp = t >> 5;
#pragma unroll
                for (int c = 1; c <= 4; ++c) {
#pragma unroll
                    for (int off = 16; off > 0; off >>= 1) v[c] += __shfl_xor_sync(0xffffffffu, v[c], off);
                    if (lane == 0) s_w1[warp * 4 + (c - 1)] = v[c];
                    v[c] = 0.0;
                }
            }
            __syncthreads();
            // P2: q = A p -- stencil order of densify.cpp:125-129; pq, S2, S3, T2, U2, U3
#pragma unroll
            for (int k = 0; k < EPT; ++k) {
                if (DCO_OK(k)) {
                    const unsigned m = static_cast<unsigned>(nbr >> (4 * k));
                    const int o = KO(k);
                    const double pk = s_p[o];
                    double acc = diag[o] * pk;
                    if (m & 1u) acc = __fma_rn(-ch[o], s_p[o + 1], acc);
                    if (m & 2u) acc = __fma_rn(-ch[o - 1], s_p[o - 1], acc);
                    if (m & 4u) acc = __fma_rn(-cv[o], s_p[o + w], acc);
                    if (m & 8u) acc = __fma_rn(-cv[o - w], s_p[o - w], acc);
                    s_q[o] = acc;
                    const double ri = r[k], rsi = s_rs[o];
                    const double pq_ = prec[o] * acc;
                    v[0] = __fma_rn(pk, acc, v[0]);
                    v[5] = __fma_rn(pq_, ri, v[5]);
                    v[6] = __fma_rn(pq_, acc, v[6]);
                    v[7] = __fma_rn(rsi, acc, v[7]);
                    v[8] = __fma_rn(ri - rsi, acc, v[8]);
                    v[9] = __fma_rn(acc, acc, v[9]);
                    if (pub & (1u << k)) __stcg(hq_out + base + t + o, acc);
                }
            }
            if ((t & 31) == 0) {
#pragma unroll
                for (int c = 1; c <= 4; ++c) v[c] = s_w1[(t >> 5) * 4 + (c - 1)];
            }
            STAMP(1)
            double res[10];
            barrier_reduce<10>(v, bar, a.part, gen, sm, res);
            STAMP(2)
            if (iter > 0) {
                snorm = sqrt(res[1]);
                if (blockIdx.x == 0 && t == 0 && iter < a.hist_cap) a.hist[iter] = snorm;
            }
            if (!(iter < a.max_iter && snorm / denom > a.tol)) break;  // densify.cpp:172 (uniform)
            const double pq = res[0];
            if (pq <= 0.0) break;
            alpha = rho / pq;
            const double rho_next = __fma_rn(alpha * alpha, res[6], __fma_rn(-2.0 * alpha, res[5], res[2]));
            const double sd = __fma_rn(-alpha, res[7], res[3]);
            const double dd = __fma_rn(alpha * alpha, res[9], __fma_rn(-2.0 * alpha, res[8], res[4]));
            beta = rho_next / rho;
            rho = rho_next;
            eta = 0.0;
            if (dd > 0.0) {
                eta = -sd / dd;
                eta = eta < 0.0 ? 0.0 : (1.0 < eta ? 1.0 : eta);
            }
            ++iter;
        }
    }
#undef STAMP
#undef DCO_OK
#undef KO
    // publish xs for the final objective's stencil, dense map
    for (int i = base + t; i < base + size; i += THREADS) {
        double xsi = sx[2 * w + chunk + (i - base)];  // s_xs
        a.xs[i] = xsi;
        a.dense[i] = static_cast<float>(dmax0(xsi));
    }
    {
        double z[1] = {0.0}, dummy[1];
        barrier_reduce<1>(z, bar, a.part, gen, sm, dummy);  // xs visible grid-wide
    }
    double o[2] = {0.0, 0.0};
    for (int i = base + t; i < base + size; i += THREADS) {
        int xx = i % w, y = i / w;
        double xsi = __ldcg(a.xs + i);
        o[0] += xsi * apply_at(a.diag, a.ch, a.cv, a.xs, w, h, i, xx, y);
        o[1] += a.rhs[i] * xsi;
    }
    barrier_reduce<2>(o, bar, a.part, gen, sm, o);
    if (blockIdx.x == 0 && t == 0) {
        a.out->objective_final = o[0] - 2.0 * o[1] + cterm;
        a.out->status = 0;
        a.out->iterations = iter;
        a.out->relative_residual = snorm / denom;
    }
}

}  // namespace
}  // namespace dco_gpu

#include "pcg_tmem.cuh"
#include "pcg_big.cuh"
#include "pcg_stream.cuh"
#include "pcg_band.cuh"

namespace dco_gpu {
namespace {

inline dim3 grid2(int w, int h, dim3 b) { return dim3((w + b.x - 1) / b.x, (h + b.y - 1) / b.y); }

long long* g_pcg_dbg = nullptr;
constexpr int kDbgLen = 1280 + 64 * 1024 * 3 + 1024;  // + per-block globaltimer stamps, per-block SM ids

// "k_pcg_tmem<7>"-style instance names with stable storage (dco_last_solver)
const char* instance_name(const char* base, int ept, int threads = 0) {
    static std::mutex mu;
    static std::set<std::string> names;
    std::lock_guard<std::mutex> lock(mu);
    std::string s = std::string(base) + "<" + std::to_string(ept);
    if (threads) s += ", " + std::to_string(threads);
    return names.insert(s + ">").first->c_str();
}

typedef void (*OnchipKernel)(CGArgs, int, GridBar*);
constexpr int kOnchipThreadsUsed = 1024;
constexpr int kOnchipSmemMax = 222 * 1024;  // + 2.6 KB static reduction scratch <= 227 KB
// k_pcg_tmem<E, 640>: 20 warps (5 per TMEM lane quarter, 96 columns each), 96 registers
constexpr int kTmem640 = 640;
OnchipKernel tmem640_for(int ept) {
    switch (ept) {
        case 9: return k_pcg_tmem<9, kTmem640>;
        case 10: return k_pcg_tmem<10, kTmem640>;
        case 11: return k_pcg_tmem<11, kTmem640>;  // EPT 12: a chunk > 7040, more shared memory than a CTA has
        default: return nullptr;
    }
}
// k_pcg_tmem<E, 512>: 16 warps (4 per TMEM lane quarter, 128 columns each), 128 registers
constexpr int kTmem512 = 512;
OnchipKernel tmem512_for(int ept) {
    switch (ept) {
        case 5: return k_pcg_tmem<5, kTmem512>;
        case 6: return k_pcg_tmem<6, kTmem512>;
        case 7: return k_pcg_tmem<7, kTmem512>;
        case 8: return k_pcg_tmem<8, kTmem512>;
        case 9: return k_pcg_tmem<9, kTmem512>;
        case 10: return k_pcg_tmem<10, kTmem512>;
        default: return nullptr;
    }
}
OnchipKernel tmem_for(int ept) {
    switch (ept) {
        case 1: return k_pcg_tmem<1>;
        case 2: return k_pcg_tmem<2>;
        case 3: return k_pcg_tmem<3>;
        case 4: return k_pcg_tmem<4>;
        case 5: return k_pcg_tmem<5>;
        case 6: return k_pcg_tmem<6>;
        case 7: return k_pcg_tmem<7>;
        case 8: return k_pcg_tmem<8>;
        default: return nullptr;
    }
}
typedef void (*BigKernel)(CGArgs, int, GridBar*, double*);
BigKernel share_for(int ept) {
    switch (ept) {
        case 9: return k_pcg_big<9, kShareThreads, kShareCols, true>;
        case 10: return k_pcg_big<10, kShareThreads, kShareCols, true>;
        case 11: return k_pcg_big<11, kShareThreads, kShareCols, true>;
        case 12: return k_pcg_big<12, kShareThreads, kShareCols, true>;
        case 13: return k_pcg_big<13, kShareThreads, kShareCols, true>;
        case 14: return k_pcg_big<14, kShareThreads, kShareCols, true>;
        case 15: return k_pcg_big<15, kShareThreads, kShareCols, true>;
        case 16: return k_pcg_big<16, kShareThreads, kShareCols, true>;
        default: return nullptr;
    }
}
BigKernel big1024_for(int ept) {
    switch (ept) {
        case 8: return k_pcg_big<8, 1024, 64, false>;
        case 9: return k_pcg_big<9, 1024, 64, false>;
        case 10: return k_pcg_big<10, 1024, 64, false>;
        case 11: return k_pcg_big<11, 1024, 64, false>;
        case 12: return k_pcg_big<12, 1024, 64, false>;
        case 13: return k_pcg_big<13, 1024, 64, false>;
        case 14: return k_pcg_big<14, 1024, 64, false>;
        case 15: return k_pcg_big<15, 1024, 64, false>;
        case 16: return k_pcg_big<16, 1024, 64, false>;
        default: return nullptr;
    }
}
BigKernel big_for(int ept) {
    switch (ept) {
        case 9: return k_pcg_big<9, kBigThreads, kBigCols, false>;
        case 10: return k_pcg_big<10, kBigThreads, kBigCols, false>;
        case 11: return k_pcg_big<11, kBigThreads, kBigCols, false>;
        case 12: return k_pcg_big<12, kBigThreads, kBigCols, false>;
        case 13: return k_pcg_big<13, kBigThreads, kBigCols, false>;
        case 14: return k_pcg_big<14, kBigThreads, kBigCols, false>;
        case 15: return k_pcg_big<15, kBigThreads, kBigCols, false>;
        case 16: return k_pcg_big<16, kBigThreads, kBigCols, false>;
        case 17: return k_pcg_big<17, kBigThreads, kBigCols, false>;
        case 18: return k_pcg_big<18, kBigThreads, kBigCols, false>;
        case 19: return k_pcg_big<19, kBigThreads, kBigCols, false>;
        case 20: return k_pcg_big<20, kBigThreads, kBigCols, false>;
        case 21: return k_pcg_big<21, kBigThreads, kBigCols, false>;
        default: return nullptr;
    }
}
OnchipKernel onchip_for(int threads, int ept) {
    if (threads != 1024) return nullptr;
    switch (ept) {
        case 1: return k_pcg_onchip<1, 1024>;
        case 2: return k_pcg_onchip<2, 1024>;
        case 3: return k_pcg_onchip<3, 1024>;
        case 4: return k_pcg_onchip<4, 1024>;
        case 5: return k_pcg_onchip<5, 1024>;
        case 6: return k_pcg_onchip<6, 1024>;
        case 7: return k_pcg_onchip<7, 1024>;
        case 8: return k_pcg_onchip<8, 1024>;
        default: return nullptr;
    }
}

}  // namespace

// ===================================================================== host =

// assemble into caller buffers; scalars stay on the device (const_dev,
// anchors_dev) unless the caller reads them back.
void assemble_system_dev(dco_ctx* ctx, const float* sparse, const uint8_t* edges, const float* mf,
                         int qw, int qh, const float* mi, const float* pre, const int* pre_valid, int w,
                         int h, const dco_config* cfg, const dco_system* sys, double* const_dev,
                         unsigned long long* anchors_dev) {
    require(qw >= 1 && qh >= 1, "assemble_system: empty m_fuse");
    if (cfg->lambda_s2 <= 0.0) pre = nullptr;  // densify.cpp:48
    const size_t n = static_cast<size_t>(w) * h;
    const int nblk = 296;
    char* scr = static_cast<char*>(scratch(ctx, S_STATS, 4096 + nblk * 2 * sizeof(double) * 2));
    (void)0;
    unsigned long long* count = reinterpret_cast<unsigned long long*>(scr);
    int* min_exp = reinterpret_cast<int*>(scr + 8);
    double* mean = reinterpret_cast<double*>(scr + 16);
    double* part = reinterpret_cast<double*>(scr + 4096);
    cuda_check(cudaMemsetAsync(scr, 0, 16, ctx->stream), "memset");
    cuda_check(cudaMemsetAsync(min_exp, 0x3f, sizeof(int), ctx->stream), "memset");
    k_sparse_stats<<<nblk, 256, 0, ctx->stream>>>(sparse, n, part, count, min_exp);
    launched(ctx, "k_sparse_stats");
    k_sparse_mean<<<1, 256, 0, ctx->stream>>>(sparse, n, part, nblk, count, min_exp, mean);
    launched(ctx, "k_sparse_mean");
    AsmArgs a;
    a.w = w;
    a.h = h;
    a.qw = qw;
    a.qh = qh;
    a.lambda_d = cfg->lambda_d;
    a.lambda_s = cfg->lambda_s;
    a.lambda_s2 = cfg->lambda_s2;
    a.sparse = sparse;
    a.edges = edges;
    a.mf = mf;
    a.mi = mi;
    a.pre = pre;
    a.pre_valid = pre_valid;
    a.diag = sys->diag;
    a.ch = sys->coup_h;
    a.cv = sys->coup_v;
    a.rhs = sys->rhs;
    a.init = sys->initial;
    a.anchored = sys->anchored;
    a.sparse_mean = mean;
    dim3 b(32, 8);
    k_assemble<<<grid2(w, h, b), b, 0, ctx->stream>>>(a);
    launched(ctx, "k_assemble");
    cuda_check(cudaMemsetAsync(anchors_dev, 0, sizeof(unsigned long long), ctx->stream), "memset");
    k_anchor_const<<<nblk, 256, 0, ctx->stream>>>(sys->anchored, sparse, pre, pre_valid, n, cfg->lambda_d,
                                                  cfg->lambda_s2, anchors_dev, part);
    launched(ctx, "k_anchor_const");
    k_reduce_parts<<<1, 256, 0, ctx->stream>>>(part, nblk, const_dev);
    launched(ctx, "k_reduce_parts");
}

// Grid-wide cooperative solves from different contexts/streams must never be
// co-scheduled (two partially-resident persistent grids could wait on each
// other forever): every cooperative launch in the process is chained after
// the previous one on the device through one event.
void launch_cooperative_serialized(dco_ctx* ctx, void* fn, dim3 grid, dim3 block, void** params, size_t smem) {
    static std::mutex mu;
    static cudaEvent_t done[64] = {};
    std::lock_guard<std::mutex> lock(mu);
    cudaEvent_t& ev = done[ctx->device & 63];
    if (!ev) cuda_check(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming), "event create");
    cuda_check(cudaStreamWaitEvent(ctx->stream, ev, 0), "wait previous solve");
    cuda_check(cudaLaunchCooperativeKernel(fn, grid, block, params, smem, ctx->stream), "cooperative launch");
    cuda_check(cudaEventRecord(ev, ctx->stream), "record solve");
}

// The whole PCG+MR solve, one cooperative launch. Scalars (anchors, constant
// term) may live on the device. out_dev receives SolveOut.
void solve_dense_dev(dco_ctx* ctx, const dco_system* sys, const dco_config* cfg,
                     const unsigned long long* anchors_dev, const double* const_dev, float* dense,
                     const float* fallback, const int* fallback_valid, double* hist, int hist_cap,
                     void* out_dev) {
    const int w = sys->width, h = sys->height;
    const size_t n = static_cast<size_t>(w) * h;
    double* wk = static_cast<double*>(scratch(ctx, S_CG, (8 * n + 48 * 1024 + 64) * sizeof(double)));
    CGArgs a;
    a.w = w;
    a.h = h;
    a.n = n;
    a.diag = sys->diag;
    a.ch = sys->coup_h;
    a.cv = sys->coup_v;
    a.rhs = sys->rhs;
    a.init = sys->initial;
    a.constant_term_host = sys->constant_term;
    a.constant_term_dev = const_dev;
    a.anchors_dev = anchors_dev;
    a.anchors_host = sys->anchor_count;
    a.prec = wk;
    a.x = wk + n;
    a.r = wk + 2 * n;
    a.z = wk + 3 * n;
    a.p = wk + 4 * n;
    a.q = wk + 5 * n;
    a.rs = wk + 6 * n;
    a.xs = wk + 7 * n;
    a.part = wk + 8 * n;
    a.hist = hist;
    a.hist_cap = hist ? hist_cap : 0;
    a.max_iter = cfg->solver_max_iter;
    a.tol = cfg->solver_tol;
    a.dense = dense;
    a.fallback = fallback;
    a.fallback_valid = fallback_valid;
    a.out = static_cast<SolveOut*>(out_dev);
    a.dbg = nullptr;
    if (getenv("DCO_PCG_DEBUG")) {
        static long long* dbg = nullptr;
        if (!dbg) cuda_check(cudaMalloc(&dbg, kDbgLen * sizeof(long long)), "dbg");
        a.dbg = dbg;
        g_pcg_dbg = dbg;
    }
    // on-chip resident path: one 1024-thread block per SM, chunk of unknowns
    // per block with 4 doubles each in shared memory, <= 8 per thread
    // DCO_PCG_BLOCKS=k (tests): a k-block grid instead of one block per SM, so
    // a small system reaches the per-thread slot counts (EPT) of a large one
    int sms = sm_count(ctx);
    if (const char* fb = getenv("DCO_PCG_BLOCKS")) sms = std::max(1, std::min(sms, atoi(fb)));
    const int chunk = static_cast<int>((n + sms - 1) / sms);
    const int threads = kOnchipThreadsUsed;
    const int ept = (chunk + threads - 1) / threads;
    const size_t smem = (static_cast<size_t>(chunk) * 4 + 2 * static_cast<size_t>(w)) * sizeof(double);
    // registers + TMEM + shared memory (pcg_tmem.cuh); DCO_PCG_NO_TMEM=1 selects
    // the registers + shared-memory variant
    const bool no_tmem = getenv("DCO_PCG_NO_TMEM") != nullptr;
    OnchipKernel kern = no_tmem ? onchip_for(threads, ept) : tmem_for(ept);
    // systems whose 1024-thread chunk needs 6 or more slots run k_pcg_tmem<E, 640>
    // (20 warps, 96 registers, 96 TMEM columns per warp): 0.708 against 0.762 ms
    // at config B (EPT 10 against 7; 896 / 768 / 512 / 384 threads: 0.738 / 0.750
    // / 0.730 / 0.800). DCO_PCG_1024=1 keeps 1024 threads.
    int tthreads = threads, tept = ept;
    if (!no_tmem && ept >= 6 && !getenv("DCO_PCG_1024")) {
        const int e640 = (chunk + kTmem640 - 1) / kTmem640;
        if (OnchipKernel k640 = tmem640_for(e640)) {
            kern = k640;
            tthreads = kTmem640;
            tept = e640;
        }
    } else if (!no_tmem && ept >= 3 && !getenv("DCO_PCG_1024")) {
        // 3..5 slots at 1024 threads (config A: 0.470 ms at 512 threads against
        // 0.539 at 1024; 768 / 640 / 384: 0.487 / 0.484 / 0.474)
        const int e512 = (chunk + kTmem512 - 1) / kTmem512;
        if (OnchipKernel k512 = tmem512_for(e512)) {
            kern = k512;
            tthreads = kTmem512;
            tept = e512;
        }
    }
    // DCO_PCG_FORCE_BIG=1 / DCO_PCG_FORCE_STREAM=1 (tests): the large-frame /
    // any-size kernel even when the state fits on chip
    const bool force_stream = getenv("DCO_PCG_FORCE_STREAM") != nullptr;
    const bool force_big = force_stream || getenv("DCO_PCG_FORCE_BIG") != nullptr;
    // k_pcg_big / k_pcg_share split the unknowns in units of 32 (pcg_big.cuh)
    const int chunk_a = static_cast<int>(32 * (((n + 31) / 32 + sms - 1) / sms));
    // DCO_PCG_SHARE=1: the co-residency variant (512 threads, p-only shared memory)
    if (getenv("DCO_PCG_SHARE") && sms <= 1024) {
        const int ept_s = std::max(9, (chunk_a + kShareThreads - 1) / kShareThreads);
        const size_t smem_s = (static_cast<size_t>(chunk_a) + 2 * static_cast<size_t>(w)) * sizeof(double);
        BigKernel sk = share_for(ept_s);
        if (sk && smem_s <= kOnchipSmemMax) {
            smem_attr(ctx, sk, static_cast<int>(smem_s));
            int chunk_arg = chunk_a;
            GridBar* bar = static_cast<GridBar*>(scratch(ctx, S_RED, sizeof(GridBar)));
            cuda_check(cudaMemsetAsync(bar, 0, sizeof(GridBar), ctx->stream), "memset bar");
            double* hb = static_cast<double*>(scratch(ctx, S_TMP1, 7 * n * sizeof(double)));
            void* params[] = {&a, &chunk_arg, &bar, &hb};
            launch_cooperative_serialized(ctx, reinterpret_cast<void*>(sk), dim3(sms), dim3(kShareThreads), params,
                                          smem_s);
            launched(ctx, "k_pcg_share");
            ctx->last_solver = instance_name("k_pcg_share", ept_s);
            return;
        }
    }
    if (kern && !force_big && smem <= kOnchipSmemMax && sms <= 1024) {
        // Whole blocks where that idles at most 4 SMs: every block then holds
        // exactly tept * tthreads unknowns and all its slots (config B: 144 x
        // 6400 = 921,600, five whole rows per block; solve 0.690 -> 0.653 ms
        // against 148 blocks of 6227). DCO_PCG_PARTIAL=1 keeps one block per SM.
        int nb = sms, chunk_l = chunk;
        size_t smem_l = smem;
        if (!no_tmem && !getenv("DCO_PCG_BLOCKS") && !getenv("DCO_PCG_PARTIAL")) {
            const long long per = static_cast<long long>(tept) * tthreads;
            const int nbw = static_cast<int>((static_cast<long long>(n) + per - 1) / per);
            const int cw = static_cast<int>((n + nbw - 1) / nbw);
            const size_t sw = (static_cast<size_t>(cw) * 4 + 2 * static_cast<size_t>(w)) * sizeof(double);
            if (nbw < sms && nbw >= sms - 4 && static_cast<long long>(n / nbw) >= per - tthreads &&
                sw <= static_cast<size_t>(kOnchipSmemMax)) {
                nb = nbw;
                chunk_l = cw;
                smem_l = sw;
            }
        }
        // dynamic shared memory: exactly this launch's need (static scratch
        // comes on top, 227 KB per CTA in total)
        smem_attr(ctx, kern, static_cast<int>(smem_l));
        int chunk_arg = chunk_l;
        GridBar* bar = static_cast<GridBar*>(scratch(ctx, S_RED, sizeof(GridBar)));
        cuda_check(cudaMemsetAsync(bar, 0, sizeof(GridBar), ctx->stream), "memset bar");
        void* params[] = {&a, &chunk_arg, &bar};
        launch_cooperative_serialized(ctx, reinterpret_cast<void*>(kern), dim3(nb), dim3(tthreads),
                                      params, smem_l);
        launched(ctx, no_tmem ? "k_pcg_onchip" : "k_pcg_tmem");
        ctx->last_solver = tthreads != threads ? instance_name("k_pcg_tmem", tept, tthreads)
                                               : instance_name(no_tmem ? "k_pcg_onchip" : "k_pcg_tmem", ept);
        return;
    }
    // larger frames: p on chip, q/rs in TMEM, r in registers, the rest L2-resident
    {
        const int ept_b = (chunk_a + kBigThreads - 1) / kBigThreads;
        const size_t smem_b = (static_cast<size_t>(chunk_a) + 2 * static_cast<size_t>(w)) * sizeof(double);
        // 1024 threads (EPT <= 16, 64 TMEM columns per warp) where the chunk
        // fits, else 768 (EPT <= 21): at 1920x1080 3.31 against 3.79 ms
        // (896 threads: 3.46, 640: 4.23). DCO_PCG_BIG768=1 keeps 768.
        const int ept_k = std::max(8, (chunk_a + 1023) / 1024);
        BigKernel bk = getenv("DCO_PCG_BIG768") ? nullptr : big1024_for(ept_k);
        int bthreads = 1024, e = ept_k;
        if (!bk) {
            e = ept_b < 9 ? 9 : ept_b;
            bk = big_for(e);
            bthreads = kBigThreads;
        }
        if (bk && !force_stream && smem_b <= kOnchipSmemMax && sms <= 1024 && !getenv("DCO_PCG_NO_BIG")) {
            smem_attr(ctx, bk, static_cast<int>(smem_b));
            int chunk_arg = chunk_a;
            GridBar* bar = static_cast<GridBar*>(scratch(ctx, S_RED, sizeof(GridBar)));
            cuda_check(cudaMemsetAsync(bar, 0, sizeof(GridBar), ctx->stream), "memset bar");
            double* hb = static_cast<double*>(scratch(ctx, S_TMP1, 7 * n * sizeof(double)));
            void* params[] = {&a, &chunk_arg, &bar, &hb};
            launch_cooperative_serialized(ctx, reinterpret_cast<void*>(bk), dim3(sms), dim3(bthreads), params,
                                          smem_b);
            launched(ctx, "k_pcg_big");
            ctx->last_solver = bthreads == 1024 ? instance_name("k_pcg_big", e, 1024) : instance_name("k_pcg_big", e);
            return;
        }
    }
    // any size: every vector in global memory, one grid barrier per iteration
    {
        StreamVecs sv;
        double* sb = static_cast<double*>(scratch(ctx, S_TMP1, 6 * n * sizeof(double)));
        for (int k = 0; k < 2; ++k) {
            sv.p[k] = sb + (0 + k) * n;
            sv.r[k] = sb + (2 + k) * n;
            sv.q[k] = sb + (4 + k) * n;
        }
        sv.x = a.x;
        sv.xs = a.xs;
        sv.rs = a.rs;
        GridBar* bar = static_cast<GridBar*>(scratch(ctx, S_RED, sizeof(GridBar)));
        cuda_check(cudaMemsetAsync(bar, 0, sizeof(GridBar), ctx->stream), "memset bar");
        void* params[] = {&a, &sv, &bar};
        // 512 threads x 2 batched elements: 16.7 ms at 3840x2160 (768 x 1 the
        // same; 1024 x 1 18.3, 384 x 2 18.0, 256 x 4 19.4, 512 x 3 spills)
        void* fn = reinterpret_cast<void*>(k_pcg_stream<512, 2>);
        const int threads = 512;
        launch_cooperative_serialized(ctx, fn, dim3(sms), dim3(threads), params, 0);
        launched(ctx, "k_pcg_stream");
        ctx->last_solver = "k_pcg_stream<512,2>";
    }
}

size_t solve_out_bytes() { return sizeof(SolveOut); }

void read_solve_out(const void* host, int* status, int* iters, double* relres, double* obj0,
                    double* obj1) {
    const SolveOut* o = static_cast<const SolveOut*>(host);
    *status = o->status;
    *iters = o->iterations;
    *relres = o->relative_residual;
    *obj0 = o->objective_initial;
    *obj1 = o->objective_final;
}

}  // namespace dco_gpu

using namespace dco_gpu;

extern "C" {

// debug: copies the last solve's per-phase clock64 stamps (DCO_PCG_DEBUG)
__attribute__((visibility("default"))) int dco_debug_pcg_stamps(long long* host, int n) {
    if (!g_pcg_dbg) return 1;
    cudaDeviceSynchronize();
    return cudaMemcpy(host, g_pcg_dbg, n * sizeof(long long), cudaMemcpyDeviceToHost) == cudaSuccess ? 0 : 4;
}

int dco_smoothness_weight(dco_ctx* ctx, int px, int py, int qx, int qy, const uint8_t* edges, int w,
                          int h, const float* mf, int qw, int qh, const float* mi, double* out) {
    return guarded(ctx, [&] {
        if (abs(px - qx) + abs(py - qy) != 1) fail(DCO_INPUT, "smoothness_weight: q must be 4-adjacent to p");
        require(px >= 0 && py >= 0 && qx >= 0 && qy >= 0 && px < w && qx < w && py < h && qy < h,
                "smoothness_weight: pixel outside the map");
        // evaluate on the host from the few device values involved
        uint8_t ep = 0, eq = 0;
        float mp = 0, mq = 0, fp = 0, fq = 0;
        auto get8 = [&](const uint8_t* src, int x, int y, uint8_t* dst) {
            cuda_check(cudaMemcpy(dst, src + static_cast<size_t>(y) * w + x, 1, cudaMemcpyDeviceToHost), "d2h");
        };
        auto getf = [&](const float* src, int stride, int x, int y, float* dst) {
            cuda_check(cudaMemcpy(dst, src + static_cast<size_t>(y) * stride + x, 4, cudaMemcpyDeviceToHost), "d2h");
        };
        get8(edges, px, py, &ep);
        get8(edges, qx, qy, &eq);
        int on = (ep ? 1 : 0) + (eq ? 1 : 0);
        if (on == 1) {
            *out = 0.0;
            return;
        }
        getf(mi, w, px, py, &mp);
        getf(mi, w, qx, qy, &mq);
        getf(mf, qw, std::min(px / 2, qw - 1), std::min(py / 2, qh - 1), &fp);
        getf(mf, qw, std::min(qx / 2, qw - 1), std::min(qy / 2, qh - 1), &fq);
        double cp = std::isfinite(fp) ? static_cast<double>(fp) : 0.0;
        double cq = std::isfinite(fq) ? static_cast<double>(fq) : 0.0;
        double sp = cp * mp, sq = cq * mq;
        double m = (sq < sp) ? sq : sp;
        double r = 1.0 - m;
        *out = (r < 0.0) ? 0.0 : r;
    });
}

int dco_assemble_system(dco_ctx* ctx, const float* sparse, const uint8_t* edges, const float* mf, int qw,
                        int qh, const float* mi, const float* pre, int w, int h, const dco_config* cfg,
                        dco_system* sys) {
    return guarded(ctx, [&] {
        require(sys && sys->diag && sys->coup_h && sys->coup_v && sys->rhs && sys->initial && sys->anchored,
                "assemble_system: system buffers missing");
        sys->width = w;
        sys->height = h;
        char* scr = static_cast<char*>(scratch(ctx, S_FLAG_ASM, 64));
        double* cdev = reinterpret_cast<double*>(scr);
        unsigned long long* adev = reinterpret_cast<unsigned long long*>(scr + 8);
        assemble_system_dev(ctx, sparse, edges, mf, qw, qh, mi, pre, nullptr, w, h, cfg, sys, cdev, adev);
        double* hp = static_cast<double*>(pinned_host(ctx, 64));
        cuda_check(cudaMemcpyAsync(hp, scr, 16, cudaMemcpyDeviceToHost, ctx->stream), "d2h");
        cuda_check(cudaStreamSynchronize(ctx->stream), "sync");
        sys->constant_term = hp[0];
        sys->anchor_count = reinterpret_cast<unsigned long long*>(hp)[1];
    });
}

// ---------------------------------------------------- row-band assembly ---
int dco_band_sparse_stats(dco_ctx* ctx, const float* sparse, size_t n, double* out) {
    return guarded(ctx, [&] {
        require(out != nullptr, "band_sparse_stats: null output");
        const int nblk = 296;
        char* scr = static_cast<char*>(scratch(ctx, S_STATS, 4096 + nblk * 2 * sizeof(double) * 2));
        unsigned long long* count = reinterpret_cast<unsigned long long*>(scr);
        int* min_exp = reinterpret_cast<int*>(scr + 8);
        double* sums = reinterpret_cast<double*>(scr + 16);
        double* part = reinterpret_cast<double*>(scr + 4096);
        cuda_check(cudaMemsetAsync(scr, 0, 16, ctx->stream), "memset");
        cuda_check(cudaMemsetAsync(min_exp, 0x3f, sizeof(int), ctx->stream), "memset");
        k_sparse_stats<<<nblk, 256, 0, ctx->stream>>>(sparse, n, part, count, min_exp);
        launched(ctx, "k_sparse_stats");
        // band totals: a fixed tree over the block partials (exact under the guard)
        k_sparse_pair_sums<<<1, 256, 0, ctx->stream>>>(part, nblk, sums);
        launched(ctx, "k_sparse_pair_sums");
        char* hp = static_cast<char*>(pinned_host(ctx, 64));
        cuda_check(cudaMemcpyAsync(hp, scr, 32, cudaMemcpyDeviceToHost, ctx->stream), "d2h");
        cuda_check(cudaStreamSynchronize(ctx->stream), "sync");
        const unsigned long long c = *reinterpret_cast<unsigned long long*>(hp);
        const int me = *reinterpret_cast<int*>(hp + 8);
        out[0] = reinterpret_cast<double*>(hp + 16)[0];
        out[1] = reinterpret_cast<double*>(hp + 16)[1];
        out[2] = static_cast<double>(c);
        out[3] = static_cast<double>(me);
    });
}

int dco_band_sparse_mean(const double* stats, int bands, double* mean, int* exact) {
    if (!stats || !mean || !exact || bands < 1) return DCO_INPUT;
    double sum = 0.0, abs_sum = 0.0, count = 0.0, me = 1e300;
    for (int k = 0; k < bands; ++k) {
        sum += stats[4 * k];
        abs_sum += stats[4 * k + 1];
        count += stats[4 * k + 2];
        if (stats[4 * k + 2] > 0.0) me = std::min(me, stats[4 * k + 3]);
    }
    *exact = 1;
    if (count == 0.0) {
        *mean = 0.0;
        return DCO_OK;
    }
    // the guard of k_sparse_mean, frame-wide: every partial sum of the valid
    // values is a multiple of 2^min_exp below 2^(53 + min_exp), so every band's
    // sum and their sum here are exact -- the sequential sum's bits
    if (!(abs_sum * (1.0 + 1e-9) < ldexp(1.0, 53 + static_cast<int>(me)))) {
        *exact = 0;
        return DCO_OK;
    }
    *mean = sum / count;
    return DCO_OK;
}

int dco_sparse_mean(dco_ctx* ctx, const float* sparse, size_t n, double* mean) {
    return guarded(ctx, [&] {
        const int nblk = 296;
        char* scr = static_cast<char*>(scratch(ctx, S_STATS, 4096 + nblk * 2 * sizeof(double) * 2));
        unsigned long long* count = reinterpret_cast<unsigned long long*>(scr);
        int* min_exp = reinterpret_cast<int*>(scr + 8);
        double* m = reinterpret_cast<double*>(scr + 16);
        double* part = reinterpret_cast<double*>(scr + 4096);
        cuda_check(cudaMemsetAsync(scr, 0, 16, ctx->stream), "memset");
        cuda_check(cudaMemsetAsync(min_exp, 0x3f, sizeof(int), ctx->stream), "memset");
        k_sparse_stats<<<nblk, 256, 0, ctx->stream>>>(sparse, n, part, count, min_exp);
        launched(ctx, "k_sparse_stats");
        k_sparse_mean<<<1, 256, 0, ctx->stream>>>(sparse, n, part, nblk, count, min_exp, m);
        launched(ctx, "k_sparse_mean");
        double* hp = static_cast<double*>(pinned_host(ctx, 64));
        cuda_check(cudaMemcpyAsync(hp, m, 8, cudaMemcpyDeviceToHost, ctx->stream), "d2h");
        cuda_check(cudaStreamSynchronize(ctx->stream), "sync");
        *mean = hp[0];
    });
}

int dco_band_assemble(dco_ctx* ctx, const float* sparse, const uint8_t* edges, const float* mf, int qw, int qh,
                      const float* mi, const float* pre, int w, int h, int own0, int own_rows,
                      const dco_config* cfg, double sparse_mean, dco_system* sys, uint64_t* anchors,
                      double* constant) {
    return guarded(ctx, [&] {
        require(sys && sys->diag && sys->coup_h && sys->coup_v && sys->rhs && sys->initial && sys->anchored,
                "band_assemble: system buffers missing");
        require(anchors && constant, "band_assemble: null outputs");
        require(qw >= 1 && qh >= 1 && w >= 1 && h >= 1, "band_assemble: empty inputs");
        require(own0 >= 0 && own_rows >= 1 && own0 + own_rows <= h, "band_assemble: owned rows outside the sub-frame");
        if (cfg->lambda_s2 <= 0.0) pre = nullptr;  // densify.cpp:48
        sys->width = w;
        sys->height = h;
        char* scr = static_cast<char*>(scratch(ctx, S_FLAG_ASM, 64));
        double* mean_dev = reinterpret_cast<double*>(scr + 16);
        cuda_check(cudaMemcpyAsync(mean_dev, &sparse_mean, 8, cudaMemcpyHostToDevice, ctx->stream), "mean");
        AsmArgs a;
        a.w = w;
        a.h = h;
        a.qw = qw;
        a.qh = qh;
        a.lambda_d = cfg->lambda_d;
        a.lambda_s = cfg->lambda_s;
        a.lambda_s2 = cfg->lambda_s2;
        a.sparse = sparse;
        a.edges = edges;
        a.mf = mf;
        a.mi = mi;
        a.pre = pre;
        a.pre_valid = nullptr;
        a.diag = sys->diag;
        a.ch = sys->coup_h;
        a.cv = sys->coup_v;
        a.rhs = sys->rhs;
        a.init = sys->initial;
        a.anchored = sys->anchored;
        a.sparse_mean = mean_dev;
        dim3 b(32, 8);
        k_assemble<<<grid2(w, h, b), b, 0, ctx->stream>>>(a);
        launched(ctx, "k_assemble");
        // anchors and constant term of the owned rows only
        const size_t off = static_cast<size_t>(own0) * w, n = static_cast<size_t>(own_rows) * w;
        const int nblk = 296;
        double* part = static_cast<double*>(scratch(ctx, S_STATS, 4096 + nblk * 2 * sizeof(double) * 2));
        unsigned long long* adev = reinterpret_cast<unsigned long long*>(scr + 8);
        double* cdev = reinterpret_cast<double*>(scr);
        cuda_check(cudaMemsetAsync(adev, 0, 8, ctx->stream), "memset");
        k_anchor_const<<<nblk, 256, 0, ctx->stream>>>(sys->anchored + off, sparse + off, pre ? pre + off : nullptr,
                                                      nullptr, n, cfg->lambda_d, cfg->lambda_s2, adev, part);
        launched(ctx, "k_anchor_const");
        k_reduce_parts<<<1, 256, 0, ctx->stream>>>(part, nblk, cdev);
        launched(ctx, "k_reduce_parts");
        double* hp = static_cast<double*>(pinned_host(ctx, 64));
        cuda_check(cudaMemcpyAsync(hp, scr, 16, cudaMemcpyDeviceToHost, ctx->stream), "d2h");
        cuda_check(cudaStreamSynchronize(ctx->stream), "sync");
        *constant = hp[0];
        *anchors = reinterpret_cast<unsigned long long*>(hp)[1];
        sys->constant_term = *constant;
        sys->anchor_count = *anchors;
    });
}

int dco_apply_system(dco_ctx* ctx, const dco_system* sys, const double* x, double* out) {
    return guarded(ctx, [&] {
        dim3 b(32, 8);
        k_apply<<<grid2(sys->width, sys->height, b), b, 0, ctx->stream>>>(sys->diag, sys->coup_h, sys->coup_v,
                                                                           x, sys->width, sys->height, out);
        launched(ctx, "k_apply");
    });
}

int dco_objective_value(dco_ctx* ctx, const dco_system* sys, const double* x, double* out) {
    return guarded(ctx, [&] {
        const int nblk = 296;
        double* part = static_cast<double*>(scratch(ctx, S_RED, (2 * nblk + 8) * sizeof(double)));
        k_objective<<<nblk, 256, 0, ctx->stream>>>(sys->diag, sys->coup_h, sys->coup_v, sys->rhs, x,
                                                   sys->width, sys->height, part);
        launched(ctx, "k_objective");
        k_objective_finish<<<1, 256, 0, ctx->stream>>>(part, nblk, sys->constant_term, part + 2 * nblk);
        launched(ctx, "k_objective_finish");
        double* hp = static_cast<double*>(pinned_host(ctx, 64));
        cuda_check(cudaMemcpyAsync(hp, part + 2 * nblk, 8, cudaMemcpyDeviceToHost, ctx->stream), "d2h");
        cuda_check(cudaStreamSynchronize(ctx->stream), "sync");
        *out = hp[0];
    });
}

// ------------------------------------------------------ row-band solver ---
// One rank's share of a system split into row bands (pcg_band.cuh): its
// vectors, exchange table and flags in ONE device arena, so a single IPC
// handle exports everything the peers touch.
struct dco_band_solver {
    dco_ctx* ctx = nullptr;
    int ranks = 1, rank = 0, w = 0, row0 = 0, rows = 0, H = 0;
    size_t n = 0;
    char* arena = nullptr;
    size_t arena_bytes = 0;
    dco_gpu::BandRank desc{};      // host copy; completed per solve
    dco_gpu::BandRank* desc_dev = nullptr;
    void* peer_base[dco_gpu::kMaxBandRanks] = {};  // mapped arenas (IPC) or local ones
    int peer_rows[dco_gpu::kMaxBandRanks] = {};
    bool ipc_opened[dco_gpu::kMaxBandRanks] = {};
    bool connected = false;
    bool local = false;  // connected with dco_band_solver_connect_local
};

namespace dco_gpu {
namespace {

constexpr int kBandVecs = 10;  // p0 p1 r0 r1 q0 q1 prec x xs rs
constexpr size_t kBandMaxBlocks = 1024;

struct BandLayout {
    size_t words, xslots, xflags, xgen, bar, out, part, total;
};

BandLayout band_layout(size_t n) {
    BandLayout L;
    L.words = (kBandVecs * n * sizeof(double) + 255) / 256 * 256;
    L.xslots = L.words;
    L.xflags = L.xslots + 2 * kMaxBandRanks * 16 * sizeof(double);
    L.xgen = L.xflags + kMaxBandRanks * 32 * sizeof(unsigned);
    L.bar = L.xgen + 256;
    L.out = L.bar + (sizeof(GridBar) + 255) / 256 * 256;
    L.part = L.out + 256;
    L.total = L.part + 2 * 16 * kBandMaxBlocks * sizeof(double);
    return L;
}

// The neighbour's boundary row `row` of an arena holding `n` unknowns.
BandSide band_side(char* base, size_t n, size_t row_off) {
    double* v = reinterpret_cast<double*>(base);
    BandSide S;
    for (int k = 0; k < 2; ++k) {
        S.p[k] = v + (0 + k) * n + row_off;
        S.r[k] = v + (2 + k) * n + row_off;
        S.q[k] = v + (4 + k) * n + row_off;
    }
    S.prec = v + 6 * n + row_off;
    S.x = v + 7 * n + row_off;
    S.xs = v + 8 * n + row_off;
    return S;
}

// Wires the peer pointers of s once peer_base / peer_rows are known.
void band_wire(dco_band_solver* s) {
    BandLayout L = band_layout(s->n);
    BandRank& R = s->desc;
    R.rank = s->rank;
    R.ranks = s->ranks;
    R.y0 = s->row0;
    R.H = s->H;
    double* v = reinterpret_cast<double*>(s->arena);
    for (int k = 0; k < 2; ++k) {
        R.sv.p[k] = v + (0 + k) * s->n;
        R.sv.r[k] = v + (2 + k) * s->n;
        R.sv.q[k] = v + (4 + k) * s->n;
    }
    R.sv.x = v + 7 * s->n;
    R.sv.xs = v + 8 * s->n;
    R.sv.rs = v + 9 * s->n;
    R.bar = reinterpret_cast<GridBar*>(s->arena + L.bar);
    R.xslots = reinterpret_cast<double*>(s->arena + L.xslots);
    R.xflags = reinterpret_cast<unsigned*>(s->arena + L.xflags);
    R.xgen = reinterpret_cast<unsigned*>(s->arena + L.xgen);
    for (int r = 0; r < kMaxBandRanks; ++r) {
        R.peer_slots[r] = nullptr;
        R.peer_flags[r] = nullptr;
    }
    for (int r = 0; r < s->ranks; ++r) {
        char* b = static_cast<char*>(s->peer_base[r]);
        const size_t pn = static_cast<size_t>(s->w) * s->peer_rows[r];
        BandLayout P = band_layout(pn);
        R.peer_slots[r] = reinterpret_cast<double*>(b + P.xslots);
        R.peer_flags[r] = reinterpret_cast<unsigned*>(b + P.xflags);
    }
    memset(&R.up, 0, sizeof(R.up));
    memset(&R.dn, 0, sizeof(R.dn));
    if (s->rank > 0) {
        const size_t pn = static_cast<size_t>(s->w) * s->peer_rows[s->rank - 1];
        R.up = band_side(static_cast<char*>(s->peer_base[s->rank - 1]), pn, pn - s->w);
    }
    if (s->rank + 1 < s->ranks) {
        const size_t pn = static_cast<size_t>(s->w) * s->peer_rows[s->rank + 1];
        R.dn = band_side(static_cast<char*>(s->peer_base[s->rank + 1]), pn, 0);
    }
    s->connected = true;
}

// Completes the per-solve fields of a rank's descriptor.
void band_fill(dco_band_solver* s, const dco_system* sys, const dco_config* cfg, unsigned long long anchors,
               double cterm, float* dense, double* hist, int hist_cap) {
    require(s->connected, "band solver: not connected");
    require(sys->width == s->w && sys->height == s->rows, "band solver: system is not this band's");
    BandLayout L = band_layout(s->n);
    CGArgs& a = s->desc.a;
    memset(&a, 0, sizeof(a));
    a.w = s->w;
    a.h = s->rows;
    a.n = s->n;
    a.diag = sys->diag;
    a.ch = sys->coup_h;
    a.cv = sys->coup_v;
    a.rhs = sys->rhs;
    a.init = sys->initial;
    a.constant_term_host = cterm;
    a.anchors_host = anchors;
    double* v = reinterpret_cast<double*>(s->arena);
    a.prec = v + 6 * s->n;
    a.x = v + 7 * s->n;
    a.xs = v + 8 * s->n;
    a.rs = v + 9 * s->n;
    a.part = reinterpret_cast<double*>(s->arena + L.part);
    a.hist = hist;
    a.hist_cap = hist ? hist_cap : 0;
    a.max_iter = cfg->solver_max_iter;
    a.tol = cfg->solver_tol;
    a.dense = dense;
    a.out = reinterpret_cast<SolveOut*>(s->arena + L.out);
}

void band_launch(dco_ctx* ctx, dco_band_solver* const* ss, int count) {
    const int sms = sm_count(ctx);
    const int bpr = std::min<int>(static_cast<int>(kBandMaxBlocks), sms / count);
    require(bpr >= 1, "band solver: more ranks on this GPU than SMs");
    BandRank* dd = ss[0]->desc_dev;
    for (int k = 0; k < count; ++k) {
        BandLayout L = band_layout(ss[k]->n);
        cuda_check(cudaMemsetAsync(ss[k]->arena + L.bar, 0, sizeof(GridBar), ctx->stream), "memset bar");
        cuda_check(cudaMemcpyAsync(dd + k, &ss[k]->desc, sizeof(BandRank), cudaMemcpyHostToDevice, ctx->stream),
                   "band desc");
    }
    // the descriptors are read by the kernel; keep the host copies stable until it has them
    cuda_check(cudaStreamSynchronize(ctx->stream), "band desc sync");
    int bpr_arg = bpr;
    void* params[] = {&dd, &bpr_arg};
    // 384 threads x 2 batched elements: 16.9 ms at 3840x2160 in one band
    // (512 x 2 spills: 19.2; 512 x 1 19.1; 768 x 1 17.8)
    void* fn = reinterpret_cast<void*>(k_pcg_band<kBandThreads, kBandB>);
    const int threads = kBandThreads;
    launch_cooperative_serialized(ctx, fn, dim3(bpr * count), dim3(threads), params, 0);
    launched(ctx, "k_pcg_band");
}

void band_stats(dco_ctx* ctx, dco_band_solver* s, dco_solve_stats* stats, double* hist) {
    BandLayout L = band_layout(s->n);
    void* hp = pinned_host(ctx, 256);
    cuda_check(cudaMemcpyAsync(hp, s->arena + L.out, solve_out_bytes(), cudaMemcpyDeviceToHost, ctx->stream), "d2h");
    cuda_check(cudaStreamSynchronize(ctx->stream), "sync");
    int status, iters;
    double rr, o0, o1;
    read_solve_out(hp, &status, &iters, &rr, &o0, &o1);
    if (status == 3) fail(DCO_UNSOLVABLE, "solve_dense_depth: no pixel carries a data or stability constraint");
    if (stats) {
        stats->iterations = iters;
        stats->relative_residual = rr;
        stats->objective_initial = o0;
        stats->objective_final = o1;
        if (hist && stats->history_cap > 0) {
            const int m = std::min(stats->history_cap, iters + 1);
            cuda_check(cudaMemcpy(stats->history, hist, m * sizeof(double), cudaMemcpyDeviceToHost), "d2h");
        }
    }
}

struct IpcBlob {
    cudaIpcMemHandle_t handle;
    int rows, w, rank, magic;
};
static_assert(sizeof(IpcBlob) <= 128, "DCO_BAND_HANDLE_BYTES");

}  // namespace
}  // namespace dco_gpu

int dco_band_solver_create(dco_ctx* ctx, int ranks, int rank, int width, int row0, int rows, int full_height,
                           dco_band_solver** out) {
    return guarded(ctx, [&] {
        require(out != nullptr, "band solver: null output");
        require(ranks >= 1 && ranks <= kMaxBandRanks, "band solver: 1..8 ranks");
        require(rank >= 0 && rank < ranks, "band solver: rank out of range");
        require(width >= 1 && rows >= 1 && row0 >= 0 && row0 + rows <= full_height, "band solver: bad band rows");
        require(rank > 0 || row0 == 0, "band solver: rank 0 owns the top row");
        require(rank + 1 < ranks || row0 + rows == full_height, "band solver: the last rank owns the bottom row");
        auto* s = new dco_band_solver;
        s->ctx = ctx;
        s->ranks = ranks;
        s->rank = rank;
        s->w = width;
        s->row0 = row0;
        s->rows = rows;
        s->H = full_height;
        s->n = static_cast<size_t>(width) * rows;
        BandLayout L = band_layout(s->n);
        s->arena_bytes = L.total;
        cudaError_t e = cudaMalloc(&s->arena, L.total);
        if (e != cudaSuccess) {
            delete s;
            fail(DCO_CUDA, std::string("band solver arena: ") + cudaGetErrorString(e));
        }
        cuda_check(cudaMemset(s->arena + L.words, 0, L.total - L.words), "band arena clear");
        e = cudaMalloc(&s->desc_dev, kMaxBandRanks * sizeof(BandRank));
        if (e != cudaSuccess) {
            cudaFree(s->arena);
            delete s;
            fail(DCO_CUDA, std::string("band solver desc: ") + cudaGetErrorString(e));
        }
        *out = s;
    });
}

void dco_band_solver_destroy(dco_band_solver* s) {
    if (!s) return;
    for (int r = 0; r < kMaxBandRanks; ++r)
        if (s->ipc_opened[r]) cudaIpcCloseMemHandle(s->peer_base[r]);
    cudaFree(s->desc_dev);
    cudaFree(s->arena);
    delete s;
}

int dco_band_solver_export(dco_band_solver* s, void* handle) {
    if (!s) return DCO_INPUT;
    return guarded(s->ctx, [&] {
        require(handle != nullptr, "band solver: null handle buffer");
        IpcBlob b;
        memset(&b, 0, sizeof(b));
        cuda_check(cudaIpcGetMemHandle(&b.handle, s->arena), "cudaIpcGetMemHandle");
        b.rows = s->rows;
        b.w = s->w;
        b.rank = s->rank;
        b.magic = 0x44434f42;
        memset(handle, 0, DCO_BAND_HANDLE_BYTES);
        memcpy(handle, &b, sizeof(b));
    });
}

int dco_band_solver_connect(dco_band_solver* s, const void* handles) {
    if (!s) return DCO_INPUT;
    return guarded(s->ctx, [&] {
        require(handles != nullptr, "band solver: null handles");
        const char* h = static_cast<const char*>(handles);
        for (int r = 0; r < s->ranks; ++r) {
            IpcBlob b;
            memcpy(&b, h + static_cast<size_t>(r) * DCO_BAND_HANDLE_BYTES, sizeof(b));
            require(b.magic == 0x44434f42 && b.rank == r && b.w == s->w, "band solver: handle table is not rank-ordered");
            s->peer_rows[r] = b.rows;
            if (r == s->rank) {
                s->peer_base[r] = s->arena;
                continue;
            }
            void* p = nullptr;
            cuda_check(cudaIpcOpenMemHandle(&p, b.handle, cudaIpcMemLazyEnablePeerAccess), "cudaIpcOpenMemHandle");
            s->peer_base[r] = p;
            s->ipc_opened[r] = true;
        }
        band_wire(s);
    });
}

int dco_band_solver_connect_local(dco_band_solver* const* ss, int ranks) {
    if (!ss || ranks < 1 || !ss[0]) return DCO_INPUT;
    return guarded(ss[0]->ctx, [&] {
        for (int k = 0; k < ranks; ++k) {
            require(ss[k] && ss[k]->ranks == ranks && ss[k]->rank == k && ss[k]->w == ss[0]->w &&
                        ss[k]->ctx == ss[0]->ctx,
                    "band solver: local ranks must be rank-ordered on one context");
            require(k == 0 || ss[k]->row0 == ss[k - 1]->row0 + ss[k - 1]->rows, "band solver: bands must tile the frame");
        }
        for (int k = 0; k < ranks; ++k) {
            for (int r = 0; r < ranks; ++r) {
                ss[k]->peer_base[r] = ss[r]->arena;
                ss[k]->peer_rows[r] = ss[r]->rows;
            }
            band_wire(ss[k]);
            ss[k]->local = true;
        }
    });
}

int dco_band_solve(dco_band_solver* s, const dco_system* sys, const dco_config* cfg, uint64_t anchors_total,
                   double constant_total, float* dense, dco_solve_stats* stats) {
    if (!s) return DCO_INPUT;
    return guarded(s->ctx, [&] {
        require(!s->local || s->ranks == 1, "band solver: connected locally; use dco_band_solve_local");
        const int cap = (stats && stats->history) ? stats->history_cap : 0;
        double* hist = cap > 0 ? static_cast<double*>(scratch(s->ctx, S_HIST, cap * sizeof(double))) : nullptr;
        band_fill(s, sys, cfg, anchors_total, constant_total, dense, hist, cap);
        dco_band_solver* one[1] = {s};
        band_launch(s->ctx, one, 1);
        band_stats(s->ctx, s, stats, hist);
    });
}

int dco_band_solve_local(dco_band_solver* const* ss, int ranks, const dco_system* sys, const dco_config* cfg,
                         uint64_t anchors_total, double constant_total, float* const* dense,
                         dco_solve_stats* stats) {
    if (!ss || ranks < 1 || !ss[0]) return DCO_INPUT;
    return guarded(ss[0]->ctx, [&] {
        dco_ctx* ctx = ss[0]->ctx;
        const int cap = (stats && stats->history) ? stats->history_cap : 0;
        double* hist = cap > 0 ? static_cast<double*>(scratch(ctx, S_HIST, cap * sizeof(double))) : nullptr;
        for (int k = 0; k < ranks; ++k) {
            require(ss[k]->ranks == ranks && ss[k]->ctx == ctx, "band solver: local ranks must share a context");
            band_fill(ss[k], &sys[k], cfg, anchors_total, constant_total, dense[k], k == 0 ? hist : nullptr,
                      k == 0 ? cap : 0);
        }
        band_launch(ctx, ss, ranks);
        for (int k = 0; k < ranks; ++k) band_stats(ctx, ss[k], stats ? &stats[k] : nullptr, k == 0 ? hist : nullptr);
    });
}

int dco_solve_dense_depth(dco_ctx* ctx, const dco_system* sys, const dco_config* cfg, float* dense,
                          dco_solve_stats* stats) {
    return guarded(ctx, [&] {
        if (sys->anchor_count == 0)
            fail(DCO_UNSOLVABLE, "solve_dense_depth: no pixel carries a data or stability constraint");
        int cap = (stats && stats->history) ? stats->history_cap : 0;
        double* hist = nullptr;
        if (cap > 0) hist = static_cast<double*>(scratch(ctx, S_HIST, cap * sizeof(double)));
        void* od = scratch(ctx, S_SCALAR, 256);
        solve_dense_dev(ctx, sys, cfg, nullptr, nullptr, dense, nullptr, nullptr, hist, cap, od);
        void* hp = pinned_host(ctx, 256);
        cuda_check(cudaMemcpyAsync(hp, od, solve_out_bytes(), cudaMemcpyDeviceToHost, ctx->stream), "d2h");
        cuda_check(cudaStreamSynchronize(ctx->stream), "sync");
        int status, iters;
        double rr, o0, o1;
        read_solve_out(hp, &status, &iters, &rr, &o0, &o1);
        if (stats) {
            stats->iterations = iters;
            stats->relative_residual = rr;
            stats->objective_initial = o0;
            stats->objective_final = o1;
            if (cap > 0) {
                int m = std::min(cap, iters + 1);
                cuda_check(cudaMemcpy(stats->history, hist, m * sizeof(double), cudaMemcpyDeviceToHost), "d2h");
            }
        }
    });
}

}  // extern "C"
