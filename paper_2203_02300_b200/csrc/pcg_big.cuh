// pcg_big.cuh -- the single-barrier PCG for frames whose solver state does
// not fit on chip (1920x1080 and up to ~2.5 M unknowns; included by
// densify.cu after pcg_tmem.cuh).
//
// Same recurrences, reductions and halo scheme as k_pcg_tmem. Placement for
// a per-SM chunk of up to 768 * 21 unknowns:
//   shared    : p with a one-row halo each side           (the SpMV operand)
//   TMEM      : q, rs                                      (4 columns / slot)
//   registers : r
//   global    : x, xs, diag, coup_h, coup_v -- 40 B per unknown, about 83 MB
//               at 1920x1080, L2-resident between iterations. The Jacobi
//               preconditioner is recomputed as 1/diag where it is used (the
//               setup's expression, so the same bits as the stored prec, which
//               only the halo recompute still reads): 4.25 -> 3.87 ms.
// 768 threads: 24 warps, 6 per TMEM lane quarter, so each warp owns 84
// columns (21 slots of [q | rs]) and a thread has 85 registers.
#pragma once

namespace dco_gpu {
namespace {

constexpr int kBigThreads = 768;
constexpr int kBigCols = 84;  // TMEM columns per warp (6 warps per lane quarter)
// The co-residency variant (DCO_PCG_SHARE): 512 threads at <= 64 registers and
// only p in shared memory, so the solve leaves half the register file and
// ~150 KB of shared memory per SM to other streams' kernels; x and xs move to
// TMEM too (4 warps per quarter: 128 columns = [q | rs | x | xs] x 16 slots).
constexpr int kShareThreads = 512;
constexpr int kShareCols = 128;

template <int EPT, int THREADS, int COLS, bool XT>
__global__ void __launch_bounds__(THREADS, XT ? 2 : 1) k_pcg_big(CGArgs a, int chunk, GridBar* bar, double* hb) {
    constexpr int SL = XT ? 8 : 4;  // TMEM columns per slot
    static_assert(SL * EPT <= COLS, "slot state in the warp's TMEM columns");
    extern __shared__ double sx[];  // p [w + chunk + w]
    __shared__ double sm[32 * 16];
    __shared__ double s_w1[32 * 4];
    __shared__ uint32_t s_tmem;
    const int w = a.w, h = a.h;
    const int n = static_cast<int>(a.n);
    const int nb = gridDim.x;
    // an even split in units of 32 unknowns: every block starts on a 256 B
    // boundary, so its rows, halos and the L2-resident vectors stay line-aligned
    // (the host sizes chunk = 32 * ceil(ceil(n / 32) / nb))
    const int bi = static_cast<int>(blockIdx.x);
    const int units = (n + 31) >> 5, qu = units / nb, ru = units - qu * nb;
    const int base = 32 * (bi * qu + min(bi, ru));
    const int size = max(0, min(32 * (qu + (bi < ru ? 1 : 0)), n - base));
    const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
    const int nv = size > t ? (size - t + THREADS - 1) / THREADS : 0;
    double* s_p = sx + w + t;
    // halo buffers: parity 0 (r, q, p), parity 1 (r, q, p), p_0
    double* const h0r = hb;
    double* const h0q = hb + n;
    double* const h0p = hb + 2 * static_cast<size_t>(n);
    double* const h1r = hb + 3 * static_cast<size_t>(n);
    double* const h1q = hb + 4 * static_cast<size_t>(n);
    double* const h1p = hb + 5 * static_cast<size_t>(n);
    double* const hp0 = hb + 6 * static_cast<size_t>(n);
    unsigned gen = 0;
    double r[EPT];
    uint64_t nbr0 = 0, nbr1 = 0;  // 4 bits per slot (slots 0-15, 16-31): 1 right, 2 left, 4 down, 8 up
    uint32_t pub = 0;   // bit k: slot k lies in a row other blocks read as halo
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
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
                         static_cast<uint32_t>(__cvta_generic_to_shared(&s_tmem)))
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    // lane quarter = warp % 4; the 6 warps of a quarter own 84-column ranges
    const uint32_t tm = s_tmem + (static_cast<uint32_t>(32 * (warp & 3)) << 16) +
                        static_cast<uint32_t>((warp >> 2) * COLS);
    const double cterm = a.constant_term_dev ? *a.constant_term_dev : a.constant_term_host;

    // setup (densify.cpp:147-166)
    double tot[5] = {0.0, 0.0, 0.0, 0.0, 0.0};
#pragma unroll
    for (int k = 0; k < EPT; ++k) {
        r[k] = 0.0;
        double ri = 0.0, xi0 = 0.0;
        if (DCO_OK(k)) {
            const int i = base + t + KO(k);
            const int xx = i % w, y = i / w;
            const uint64_t mk = (xx + 1 < w ? 1u : 0u) | (xx > 0 ? 2u : 0u) | (y + 1 < h ? 4u : 0u) | (y > 0 ? 8u : 0u);
            if (k < 16) {
                nbr0 |= mk << (4 * k);
            } else {
                nbr1 |= mk << (4 * (k - 16));
            }
            if (t + KO(k) < w || t + KO(k) >= size - w) pub |= 1u << k;
            const double ax = apply_at(a.diag, a.ch, a.cv, a.init, w, h, i, xx, y);
            const double xi = a.init[i];
            const double b = a.rhs[i];
            const double d = a.diag[i];
            const double pr = d > 0.0 ? 1.0 / d : 1.0;
            ri = b - ax;
            const double zi = pr * ri;
            r[k] = ri;
            s_p[KO(k)] = zi;
            a.prec[i] = pr;
            if (!XT) {
                a.x[i] = xi;
                a.xs[i] = xi;
            }
            xi0 = xi;
            hp0[i] = zi;
            tot[0] += b * b;
            tot[1] += ri * ri;
            tot[2] += ri * zi;
            tot[3] += xi * ax;
            tot[4] += b * xi;
        }
        uint32_t v4[4];
        v4[0] = v4[1] = 0u;  // q
        d2u(ri, v4[2], v4[3]);
        tm_st4(tm + SL * k, v4);
        if (XT) {  // x, xs
            d2u(xi0, v4[0], v4[1]);
            d2u(xi0, v4[2], v4[3]);
            tm_st4(tm + SL * k + 4, v4);
        }
    }
    barrier_reduce<5>(tot, bar, a.part, gen, sm, tot);
    const double bnorm = sqrt(tot[0]);
    const double denom = bnorm > 0.0 ? bnorm : 1.0;
    double snorm = sqrt(tot[1]);
    double rho = tot[2];
    if (blockIdx.x == 0 && t == 0) {
        if (a.hist_cap > 0) a.hist[0] = snorm;
        a.out->objective_initial = tot[3] - 2.0 * tot[4] + cterm;
    }

    int iter = 0;
    double alpha = 0.0, beta = 0.0, eta = 0.0;
    if (a.max_iter > 0 && snorm / denom > a.tol) {
        for (;;) {
            asm volatile("" : "+r"(pub), "+l"(nbr0), "+l"(nbr1));
            const int par = iter & 1;
            const double* const hr_in = par ? h0r : h1r;  // published in phase iter-1
            const double* const hq_in = par ? h0q : h1q;
            const double* const hp_in = par ? h0p : h1p;
            double* const hr_out = par ? h1r : h0r;
            double* const hq_out = par ? h1q : h0q;
            double* const hp_out = par ? h1p : h0p;
            // halo rows: p_iter of the neighbours, owner's FMA sequence
            for (int e = t; e < 2 * w; e += THREADS) {
                const int l = e < w ? e - w : size + (e - w);
                const int j = base + l;
                double pj = 0.0;
                if (j >= 0 && j < n) {
                    if (iter) {
                        const double rj = __fma_rn(-alpha, __ldcg(hq_in + j), __ldcg(hr_in + j));
                        pj = __fma_rn(beta, __ldcg(hp_in + j), __ldcg(a.prec + j) * rj);
                    } else {
                        pj = __ldcg(hp0 + j);
                    }
                }
                sx[w + l] = pj;
            }
            // P1: updates of iteration iter-1, then |rs|^2, S1, T1, U1
            double v[10];
#pragma unroll
            for (int c = 0; c < 10; ++c) v[c] = 0.0;
            tm_wait_st();
#pragma unroll
            for (int k = 0; k < EPT; ++k) {
                uint32_t c4[4], cx4[4];
                tm_ld4(tm + SL * k, c4);  // q, rs
                if (XT) tm_ld4(tm + SL * k + 4, cx4);  // x, xs
                tm_wait_ld();
                const double qk = u2d(c4[0], c4[1]);
                double rsi = u2d(c4[2], c4[3]);
                double xk_t = XT ? u2d(cx4[0], cx4[1]) : 0.0, xs_t = XT ? u2d(cx4[2], cx4[3]) : 0.0;
                if (DCO_OK(k)) {
                    const int o = KO(k);
                    const int i = base + t + o;
                    double pk = s_p[o];
                    double ri = r[k];
                    const double dgi = __ldg(a.diag + i);
                    const double pr = dgi > 0.0 ? 1.0 / dgi : 1.0;  // = the stored prec's bits
                    if (iter) {
                        const double xk = __fma_rn(alpha, pk, XT ? xk_t : __ldcg(a.x + i));
                        if (XT) {
                            xk_t = xk;
                        } else {
                            __stcg(a.x + i, xk);
                        }
                        ri = __fma_rn(-alpha, qk, ri);
                        pk = __fma_rn(beta, pk, pr * ri);
                        r[k] = ri;
                        s_p[o] = pk;
                        if (eta > 0.0) {
                            rsi = __fma_rn(eta, ri - rsi, rsi);
                            const double xsi = XT ? xs_t : __ldcg(a.xs + i);
                            const double xsn = __fma_rn(eta, xk - xsi, xsi);
                            if (XT) {
                                xs_t = xsn;
                            } else {
                                __stcg(a.xs + i, xsn);
                            }
                        }
                    }
                    const double e = ri - rsi;
                    v[1] = __fma_rn(rsi, rsi, v[1]);
                    v[2] = __fma_rn(pr * ri, ri, v[2]);
                    v[3] = __fma_rn(rsi, e, v[3]);
                    v[4] = __fma_rn(e, e, v[4]);
                    if (pub & (1u << k)) {
                        __stcg(hr_out + i, ri);
                        __stcg(hp_out + i, pk);
                    }
                }
                if (iter && eta > 0.0) {  // warp-uniform
                    uint32_t s2[2];
                    d2u(rsi, s2[0], s2[1]);
                    tm_st2(tm + SL * k + 2, s2);
                }
                if (XT && iter) {  // x (and xs, unchanged when eta == 0)
                    uint32_t s4[4];
                    d2u(xk_t, s4[0], s4[1]);
                    d2u(xs_t, s4[2], s4[3]);
                    tm_st4(tm + SL * k + 4, s4);
                }
            }
#pragma unroll
            for (int c = 1; c <= 4; ++c) {
#pragma unroll
                for (int off = 16; off > 0; off >>= 1) v[c] += __shfl_xor_sync(0xffffffffu, v[c], off);
                if (lane == 0) s_w1[warp * 4 + (c - 1)] = v[c];
                v[c] = 0.0;
            }
            tm_wait_st();
            __syncthreads();
            // P2: q = A p (densify.cpp:125-129), pq, S2, S3, T2, U2, U3 (no
            // register headroom at 85/thread for a slot-ahead prefetch: it
            // spills 700 B and runs slower)
#pragma unroll
            for (int k = 0; k < EPT; ++k) {
                uint32_t c2[2];
                tm_ld2(tm + SL * k + 2, c2);  // rs
                tm_wait_ld();
                const double rsi = u2d(c2[0], c2[1]);
                double acc = 0.0;
                if (DCO_OK(k)) {
                    const unsigned m = static_cast<unsigned>(k < 16 ? (nbr0 >> (4 * k)) : (nbr1 >> (4 * (k - 16))));
                    const int o = KO(k);
                    const int i = base + t + o;
                    const double pk = s_p[o];
                    const double dg = __ldg(a.diag + i);
                    acc = dg * pk;
                    if (m & 1u) acc = __fma_rn(-__ldg(a.ch + i), s_p[o + 1], acc);
                    if (m & 2u) acc = __fma_rn(-__ldg(a.ch + i - 1), s_p[o - 1], acc);
                    if (m & 4u) acc = __fma_rn(-__ldg(a.cv + i), s_p[o + w], acc);
                    if (m & 8u) acc = __fma_rn(-__ldg(a.cv + i - w), s_p[o - w], acc);
                    const double ri = r[k];
                    // prec = 1/diag recomputed (setup's expression, same bits): one L2
                    // stream fewer per iteration for a DDIV
                    const double pq_ = (dg > 0.0 ? 1.0 / dg : 1.0) * acc;
                    v[0] = __fma_rn(pk, acc, v[0]);
                    v[5] = __fma_rn(pq_, ri, v[5]);
                    v[6] = __fma_rn(pq_, acc, v[6]);
                    v[7] = __fma_rn(rsi, acc, v[7]);
                    v[8] = __fma_rn(ri - rsi, acc, v[8]);
                    v[9] = __fma_rn(acc, acc, v[9]);
                    if (pub & (1u << k)) __stcg(hq_out + i, acc);
                }
                uint32_t s2[2];
                d2u(acc, s2[0], s2[1]);
                tm_st2(tm + SL * k, s2);
            }
            if (lane == 0) {
#pragma unroll
                for (int c = 1; c <= 4; ++c) v[c] = s_w1[warp * 4 + (c - 1)];
            }
            double res[10];
            barrier_reduce<10, false>(v, bar, a.part, gen, sm, res);  // CTA barrier before P2 guards sm
            if (iter > 0) {
                snorm = sqrt(res[1]);
                if (blockIdx.x == 0 && t == 0 && iter < a.hist_cap) a.hist[iter] = snorm;
            }
            if (!(iter < a.max_iter && snorm / denom > a.tol)) break;  // densify.cpp:172
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
    // dense map from xs (in a.xs for the objective's stencil)
    tm_wait_st();
    if (XT) {
#pragma unroll
        for (int k = 0; k < EPT; ++k) {
            uint32_t v2[2];
            tm_ld2(tm + SL * k + 6, v2);
            tm_wait_ld();
            if (DCO_OK(k)) a.xs[base + t + KO(k)] = u2d(v2[0], v2[1]);
        }
    }
    for (int i = base + t; i < base + size; i += THREADS) a.dense[i] = static_cast<float>(dmax0(__ldcg(a.xs + i)));
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    {
        double z[1] = {0.0}, dummy[1];
        barrier_reduce<1>(z, bar, a.part, gen, sm, dummy);  // xs visible grid-wide (and a CTA barrier)
    }
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(s_tmem) : "memory");
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
#undef DCO_OK
#undef KO
}

}  // namespace
}  // namespace dco_gpu
