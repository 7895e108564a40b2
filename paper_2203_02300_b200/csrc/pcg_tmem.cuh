// pcg_tmem.cuh -- the on-chip PCG solver with its per-unknown state spread
// over all three on-SM stores of sm_100a (included by densify.cu).
//
// Same algorithm, iterates and single grid barrier per iteration as
// k_pcg_onchip (see there for the recurrences). What moves:
//   registers : r, x (x of the first slots: TMEM)  (<= 2 doubles / unknown)
//   TMEM      : q, xs, rs, diag                    (4 doubles / unknown)
//   shared    : p (+ one-row halo each side), coup_h, coup_v, prec
// so the SpMV reads every coefficient on chip; the only per-iteration L2
// traffic left is the one-row halo between neighbouring blocks (plus the
// coupling of the first row / first unknown, which belongs to the previous
// block). Tensor memory is used here as 256 KB of per-thread storage: each
// warp owns the 32 lanes of its quarter and a disjoint 8*EPT-column range
// (8 warps per quarter x 64 columns = 512), slot k of a thread holding
// [q | xs | rs | diag] in columns 8k .. 8k+7 of its lane and, in the spare
// columns above 8*EPT, the x of as many slots as fit.
#pragma once

#include <type_traits>

namespace dco_gpu {
namespace {

// lane base of the warp's quarter, and its 64-column range (8 warps per quarter)
__device__ __forceinline__ uint32_t tm_lane_col(uint32_t base, int warp) {
    return base + (static_cast<uint32_t>(32 * (warp & 3)) << 16) + static_cast<uint32_t>((warp >> 2) * 64);
}
__device__ __forceinline__ void tm_ld8(uint32_t a, uint32_t (&v)[8]) {
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
                 : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7])
                 : "r"(a)
                 : "memory");
}
__device__ __forceinline__ void tm_ld4(uint32_t a, uint32_t (&v)[4]) {
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0, %1, %2, %3}, [%4];"
                 : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3])
                 : "r"(a)
                 : "memory");
}
__device__ __forceinline__ void tm_ld2(uint32_t a, uint32_t (&v)[2]) {
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x2.b32 {%0, %1}, [%2];" : "=r"(v[0]), "=r"(v[1]) : "r"(a) : "memory");
}
__device__ __forceinline__ void tm_st8(uint32_t a, const uint32_t (&v)[8]) {
    asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};" ::"r"(a), "r"(v[0]),
                 "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7])
                 : "memory");
}
__device__ __forceinline__ void tm_st4(uint32_t a, const uint32_t (&v)[4]) {
    asm volatile("tcgen05.st.sync.aligned.32x32b.x4.b32 [%0], {%1, %2, %3, %4};" ::"r"(a), "r"(v[0]), "r"(v[1]),
                 "r"(v[2]), "r"(v[3])
                 : "memory");
}
__device__ __forceinline__ void tm_st2(uint32_t a, const uint32_t (&v)[2]) {
    asm volatile("tcgen05.st.sync.aligned.32x32b.x2.b32 [%0], {%1, %2};" ::"r"(a), "r"(v[0]), "r"(v[1]) : "memory");
}
__device__ __forceinline__ void tm_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void tm_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }
// explicit 32-bit shared-window accesses: base register + immediate, so the
// compiler neither rematerialises the window base per access nor spends a
// register per array
template <int IMM>
__device__ __forceinline__ double lds(uint32_t a) {
    double v;
    asm volatile("ld.shared.f64 %0, [%1+%2];" : "=d"(v) : "r"(a), "n"(IMM) : "memory");
    return v;
}
template <int IMM>
__device__ __forceinline__ void sts(uint32_t a, double v) {
    asm volatile("st.shared.f64 [%0+%1], %2;" ::"r"(a), "n"(IMM), "d"(v) : "memory");
}
template <int K, int N, typename F>
__device__ __forceinline__ void static_for(F&& f) {
    if constexpr (K < N) {
        f(std::integral_constant<int, K>{});
        static_for<K + 1, N>(f);
    }
}
__device__ __forceinline__ double u2d(uint32_t lo, uint32_t hi) {
    return __hiloint2double(static_cast<int>(hi), static_cast<int>(lo));
}
__device__ __forceinline__ void d2u(double d, uint32_t& lo, uint32_t& hi) {
    lo = static_cast<uint32_t>(__double2loint(d));
    hi = static_cast<uint32_t>(__double2hiint(d));
}

// THREADS = 896 (28 warps, 7 per lane quarter, 72 TMEM columns each): up to 72
// registers per thread and room in TMEM for the x of every slot up to EPT 7.
template <int EPT, int THREADS = 1024>
__global__ void __launch_bounds__(THREADS, 1) k_pcg_tmem(CGArgs a, int chunk, GridBar* bar) {
    constexpr int CPW = THREADS == 1024 ? 64 : ((512 / (THREADS / 128)) & ~7);  // TMEM columns per warp
    static_assert(THREADS % 128 == 0 && THREADS <= 1024, "whole lane quarters");
    static_assert(EPT >= 1 && 8 * EPT <= CPW, "8*EPT TMEM columns per warp");
    extern __shared__ double sx[];  // p [w + chunk + w], coup_h, coup_v, prec [chunk] each
    __shared__ double sm[32 * 16];
    __shared__ double s_w1[32 * 4];  // per-warp P1 sums
    __shared__ uint32_t s_tmem;
    const int w = a.w, h = a.h;
    const int n = static_cast<int>(a.n);
    const int nb = gridDim.x;
    const int qn = n / nb, rem = n - qn * nb;
    const int base = blockIdx.x * qn + min(static_cast<int>(blockIdx.x), rem);
    const int size = qn + (static_cast<int>(blockIdx.x) < rem ? 1 : 0);
    const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
    const int nv = size > t ? (size - t + THREADS - 1) / THREADS : 0;  // occupied slots
    double* s_p = sx + w + t;
    double* s_ch = sx + 2 * w + chunk + t;
    double* s_cv = sx + 2 * w + 2 * chunk + t;
    double* s_pr = sx + 2 * w + 3 * chunk + t;
    // shared-window byte addresses of this thread's slot 0 (loop accesses)
    // opaque to the compiler: kept (or spilled) rather than rebuilt from the
    // shared-window base at every use
    auto opaque = [](uint32_t v) {
        asm volatile("" : "+r"(v));
        return v;
    };
    const uint32_t aP = opaque(static_cast<uint32_t>(__cvta_generic_to_shared(s_p)));
    const uint32_t aCH = opaque(static_cast<uint32_t>(__cvta_generic_to_shared(s_ch)));
    const uint32_t aCV = opaque(static_cast<uint32_t>(__cvta_generic_to_shared(s_cv)));
    const uint32_t aPR = opaque(static_cast<uint32_t>(__cvta_generic_to_shared(s_pr)));
    const uint32_t wb = 8u * static_cast<uint32_t>(w);
    unsigned gen = 0;
    double r[EPT], x[EPT];
    unsigned pub = 0;  // bit k: slot k lies in a row other blocks read as halo
    // The host picks EPT = ceil(chunk / THREADS) with chunk = ceil(n / nb), so
    // (EPT - 1) * THREADS <= chunk - 1 <= qn <= size: slots 0 .. EPT-2 are
    // occupied in every thread of every block (DCO_FULL: only the last slot is
    // tested). A launch breaking this is a host bug.
    if (qn < (EPT - 1) * THREADS) __trap();
#define DCO_OK(k) ((k) < nv)
#define DCO_FULL(k) ((k) < EPT - 1 || (k) < nv)
#define KO(k) ((k) * THREADS)

    if (a.dbg && t == 0 && blockIdx.x == 0) {  // kernel entry (DCO_PCG_DEBUG)
        unsigned long long gt_;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(gt_));
        a.dbg[636] = static_cast<long long>(gt_);
    }
    if (a.dbg && t == 0) {  // this block's SM (DCO_PCG_DEBUG)
        unsigned smid_;
        asm volatile("mov.u32 %0, %%smid;" : "=r"(smid_));
        a.dbg[1280 + 64 * 1024 * 3 + blockIdx.x] = smid_;
    }
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
    // tensor memory: all 512 columns (this CTA is alone on its SM)
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
                         static_cast<uint32_t>(__cvta_generic_to_shared(&s_tmem)))
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    // this warp's column 0, lane base: quarter warp % 4, column range (warp / 4) * CPW
    const uint32_t tm = s_tmem + (static_cast<uint32_t>(32 * (warp & 3)) << 16) +
                        static_cast<uint32_t>((warp >> 2) * CPW);
    // x of the first XT slots lives in the spare columns 8*EPT.. (2 per slot),
    // the rest in registers
    constexpr int XT = (CPW - 8 * EPT) / 2 < EPT ? (CPW - 8 * EPT) / 2 : EPT;
    const uint32_t tmx = tm + 8 * EPT;
    if (a.dbg && t == 0 && blockIdx.x == 0) {  // globaltimer: setup / teardown split (DCO_PCG_DEBUG)
        unsigned long long gt_;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(gt_));
        a.dbg[6] = static_cast<long long>(gt_);
    }
    const double cterm = a.constant_term_dev ? *a.constant_term_dev : a.constant_term_host;

    // setup (densify.cpp:147-166): x = initial, r = b - A x, z = M r, p = z
    // (p_0 published whole in a.xs for phase 0's halo)
    double tot[5] = {0.0, 0.0, 0.0, 0.0, 0.0};  // b.b, r.r, r.z, x.Ax, b.x
#pragma unroll
    for (int k = 0; k < EPT; ++k) {
        r[k] = 0.0;
        x[k] = 0.0;
        double xi = 0.0, ri = 0.0, d = 0.0;
        if (DCO_OK(k)) {
            const int i = base + t + KO(k);
            const int xx = i % w, y = i / w;
            if (t + KO(k) < w || t + KO(k) >= size - w) pub |= 1u << k;
            const double ax = apply_at(a.diag, a.ch, a.cv, a.init, w, h, i, xx, y);
            xi = a.init[i];
            const double b = a.rhs[i];
            d = a.diag[i];
            const double pr = d > 0.0 ? 1.0 / d : 1.0;
            ri = b - ax;
            const double zi = pr * ri;
            x[k] = xi;
            r[k] = ri;
            s_p[KO(k)] = zi;
            // couplings to missing neighbours forced to 0: the SpMV below then
            // needs no per-neighbour branch (a 0 coefficient times a finite p
            // adds an exact 0, as the reference's skipped term does)
            s_ch[KO(k)] = xx + 1 < w ? a.ch[i] : 0.0;
            s_cv[KO(k)] = y + 1 < h ? a.cv[i] : 0.0;
            s_pr[KO(k)] = pr;
            a.prec[i] = pr;
            a.xs[i] = zi;
            tot[0] += b * b;
            tot[1] += ri * ri;
            tot[2] += ri * zi;
            tot[3] += xi * ax;
            tot[4] += b * xi;
        }
        uint32_t v8[8];
        v8[0] = v8[1] = 0u;  // q
        d2u(xi, v8[2], v8[3]);
        d2u(ri, v8[4], v8[5]);
        d2u(d, v8[6], v8[7]);
        tm_st8(tm + 8 * k, v8);
        if (k < XT) {
            uint32_t v2[2];
            d2u(xi, v2[0], v2[1]);
            tm_st2(tmx + 2 * k, v2);
        }
    }
    barrier_reduce<5>(tot, bar, a.part, gen, sm, tot);
    if (a.dbg && t == 0 && blockIdx.x == 0) {  // globaltimer: setup / teardown split (DCO_PCG_DEBUG)
        unsigned long long gt_;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(gt_));
        a.dbg[7] = static_cast<long long>(gt_);
    }
    const double bnorm = sqrt(tot[0]);
    const double denom = bnorm > 0.0 ? bnorm : 1.0;
    double snorm = sqrt(tot[1]);
    double rho = tot[2];
    if (blockIdx.x == 0 && t == 0) {
        if (a.hist_cap > 0) a.hist[0] = snorm;
        a.out->objective_initial = tot[3] - 2.0 * tot[4] + cterm;
    }
    // couplings of the first unknown / first row that belong to the previous block
    const double ch_left0 = (base % w) != 0 ? a.ch[base - 1] : 0.0;

    int iter = 0;
    double alpha = 0.0, beta = 0.0, eta = 0.0;  // iteration iter-1's scalars
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
            asm volatile("" : "+r"(pub));
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
                constexpr int kHalo = THREADS <= 640 ? 4 : 3;  // 2w <= kHalo * THREADS at w = 1280
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
                            h3[u] = __ldcg(a.prec + j);
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
                    if (e < 2 * w)  // outside the grid: 0 (multiplied by a 0 coupling)
                        sx[w + l] = (j >= 0 && j < n)
                                        ? (iter ? __fma_rn(beta, h2[u], h3[u] * __fma_rn(-alpha, h1[u], h0[u])) : h2[u])
                                        : 0.0;
                }
                for (int e = t + kHalo * THREADS; e < 2 * w; e += THREADS) {  // w > 1.5 * THREADS only
                    const int l = e < w ? e - w : size + (e - w);
                    const int j = base + l;
                    double pj = 0.0;
                    if (j >= 0 && j < n) {
                        if (iter) {
                            const double rj = __fma_rn(-alpha, __ldcg(hq_in + j), __ldcg(hr_in + j));
                            pj = __fma_rn(beta, __ldcg(hp_in + j), __ldcg(a.prec + j) * rj);
                        } else {
                            pj = __ldcg(a.xs + j);
                        }
                    }
                    sx[w + l] = pj;
                }
            }
            STAMP(3)
            // P1: vector updates of iteration iter-1, then |rs|^2, S1, T1, U1
            double v[10];
#pragma unroll
            for (int c = 0; c < 10; ++c) v[c] = 0.0;
            tm_wait_st();  // last phase's q / xs / rs stores have landed
            // slot k + 1's q, xs, rs (and x) are loaded while slot k computes
            uint32_t c4[4], c2[2], cx[2] = {0u, 0u};
            tm_ld4(tm, c4);      // q, xs
            tm_ld2(tm + 4, c2);  // rs
            if (XT > 0) tm_ld2(tmx, cx);
            tm_wait_ld();
            static_for<0, EPT>([&](auto kc) {
                constexpr int k = decltype(kc)::value;
                uint32_t n4[4], n2[2], nx[2] = {0u, 0u};
                if constexpr (k + 1 < EPT) {
                    tm_ld4(tm + 8 * (k + 1), n4);
                    tm_ld2(tm + 8 * (k + 1) + 4, n2);
                    if (k + 1 < XT) tm_ld2(tmx + 2 * (k + 1), nx);
                }
                const double qk = u2d(c4[0], c4[1]);
                double xsi = u2d(c4[2], c4[3]);
                double rsi = u2d(c2[0], c2[1]);
                double xk = k < XT ? u2d(cx[0], cx[1]) : x[k];
                if (DCO_FULL(k)) {
                    const int o = KO(k);
                    double pk = lds<8 * KO(k)>(aP);
                    double ri = r[k];
                    const double pr = lds<8 * KO(k)>(aPR);
                    if (iter) {
                        xk = __fma_rn(alpha, pk, xk);
                        ri = __fma_rn(-alpha, qk, ri);
                        pk = __fma_rn(beta, pk, pr * ri);
                        r[k] = ri;
                        sts<8 * KO(k)>(aP, pk);
                        if (eta > 0.0) {
                            rsi = __fma_rn(eta, ri - rsi, rsi);
                            xsi = __fma_rn(eta, xk - xsi, xsi);
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
                if (k >= XT) x[k] = xk;
                if (iter && k < XT) {  // warp-uniform
                    uint32_t s2x[2];
                    d2u(xk, s2x[0], s2x[1]);
                    tm_st2(tmx + 2 * k, s2x);
                }
                if (iter && eta > 0.0) {  // warp-uniform
                    uint32_t s4[4];
                    d2u(xsi, s4[0], s4[1]);
                    d2u(rsi, s4[2], s4[3]);
                    tm_st4(tm + 8 * k + 2, s4);
                }
                if constexpr (k + 1 < EPT) {
                    tm_wait_ld();
#pragma unroll
                    for (int c = 0; c < 4; ++c) c4[c] = n4[c];
                    c2[0] = n2[0];
                    c2[1] = n2[1];
                    cx[0] = nx[0];
                    cx[1] = nx[1];
                }
            });
            // P1 sums -> per-warp partials in shared memory (frees registers for P2)
            // recursive halving: 6 double shuffles for the 4 sums instead of 20
            {
                double u[4] = {v[1], v[2], v[3], v[4]};
                warp_halving_reduce<4>(u, lane);
                if ((lane & 7) == 0) s_w1[warp * 4 + grid_reduce_index<4>(lane)] = u[0];
#pragma unroll
                for (int c = 1; c <= 4; ++c) v[c] = 0.0;
            }
            tm_wait_st();  // P2 reads rs back
            STAMP(4)
            __syncthreads();
            STAMP(5)
            // P2: q = A p -- stencil order of densify.cpp:125-129; pq, S2, S3, T2, U2, U3
            uint32_t cur4[4];
            tm_ld4(tm + 4, cur4);  // rs, diag of slot 0
            tm_wait_ld();
            static_for<0, EPT>([&](auto kc) {
                constexpr int k = decltype(kc)::value;
                uint32_t nxt4[4];
                if (k + 1 < EPT) tm_ld4(tm + 8 * (k + 1) + 4, nxt4);  // in flight during slot k
                const double rsi = u2d(cur4[0], cur4[1]);
                const double dg = u2d(cur4[2], cur4[3]);
                double acc = 0.0;
                if (DCO_FULL(k)) {
                    const int o = KO(k);
                    const int l = t + o;
                    const double pk = lds<8 * KO(k)>(aP);
                    double cl, cu;  // couplings to the left / upper neighbour
                    if (k == 0 && l == 0) {
                        cl = ch_left0;
                    } else {
                        cl = lds<8 * KO(k) - 8>(aCH);
                    }
                    if (KO(k) + THREADS <= w || l < w) {  // first row: the previous block's couplings
                        const int j = base + l - w;
                        cu = j >= 0 ? __ldg(a.cv + j) : 0.0;
                    } else {
                        cu = lds<8 * KO(k)>(aCV - wb);
                    }
                    acc = dg * pk;
                    acc = __fma_rn(-lds<8 * KO(k)>(aCH), lds<8 * KO(k) + 8>(aP), acc);
                    acc = __fma_rn(-cl, lds<8 * KO(k) - 8>(aP), acc);
                    acc = __fma_rn(-lds<8 * KO(k)>(aCV), lds<8 * KO(k)>(aP + wb), acc);
                    acc = __fma_rn(-cu, lds<8 * KO(k)>(aP - wb), acc);
                    const double ri = r[k];
                    const double pq_ = lds<8 * KO(k)>(aPR) * acc;
                    v[0] = __fma_rn(pk, acc, v[0]);
                    v[5] = __fma_rn(pq_, ri, v[5]);
                    v[6] = __fma_rn(pq_, acc, v[6]);
                    v[7] = __fma_rn(rsi, acc, v[7]);
                    v[8] = __fma_rn(ri - rsi, acc, v[8]);
                    v[9] = __fma_rn(acc, acc, v[9]);
                    if (pub & (1u << k)) __stcg(hq_out + base + l, acc);
                }
                uint32_t s2[2];
                d2u(acc, s2[0], s2[1]);
                tm_st2(tm + 8 * k, s2);
                if (k + 1 < EPT) {
                    tm_wait_ld();
#pragma unroll
                    for (int c = 0; c < 4; ++c) cur4[c] = nxt4[c];
                }
            });
            if (lane == 0) {
#pragma unroll
                for (int c = 1; c <= 4; ++c) v[c] = s_w1[warp * 4 + (c - 1)];
            }
            STAMP(1)
            double res[10];
            barrier_reduce<10, false>(v, bar, a.part, gen, sm, res);  // CTA barrier before P2 guards sm
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
    if (a.dbg && t == 0 && blockIdx.x == 0) {
        unsigned long long gt_;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(gt_));
        a.dbg[8] = static_cast<long long>(gt_);
    }
    // publish xs for the final objective's stencil, dense map
    tm_wait_st();
#pragma unroll
    for (int k = 0; k < EPT; ++k) {
        uint32_t v2[2];
        tm_ld2(tm + 8 * k + 2, v2);
        tm_wait_ld();
        if (DCO_OK(k)) {
            const int i = base + t + KO(k);
            const double xsi = u2d(v2[0], v2[1]);
            a.xs[i] = xsi;
            a.dense[i] = static_cast<float>(dmax0(xsi));
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    {
        double z[1] = {0.0}, dummy[1];
        barrier_reduce<1>(z, bar, a.part, gen, sm, dummy);  // xs visible grid-wide (and a CTA barrier)
    }
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(s_tmem) : "memory");
    double o[2] = {0.0, 0.0};
    // the thread's elements in order, unrolled so their loads overlap
    static_for<0, EPT>([&](auto kc) {
        constexpr int k = decltype(kc)::value;
        if (DCO_OK(k)) {
            const int i = base + t + KO(k);
            const int xx = i % w, y = i / w;
            const double xsi = __ldcg(a.xs + i);
            o[0] += xsi * apply_at(a.diag, a.ch, a.cv, a.xs, w, h, i, xx, y);
            o[1] += a.rhs[i] * xsi;
        }
    });
    barrier_reduce<2>(o, bar, a.part, gen, sm, o);
    if (a.dbg && t == 0 && blockIdx.x == 0) {  // globaltimer: setup / teardown split (DCO_PCG_DEBUG)
        unsigned long long gt_;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(gt_));
        a.dbg[9] = static_cast<long long>(gt_);
    }
    if (blockIdx.x == 0 && t == 0) {
        a.out->objective_final = o[0] - 2.0 * o[1] + cterm;
        a.out->status = 0;
        a.out->iterations = iter;
        a.out->relative_residual = snorm / denom;
    }
#undef STAMP
#undef DCO_OK
#undef DCO_FULL
#undef KO
}

}  // namespace
}  // namespace dco_gpu
