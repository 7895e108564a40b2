// pcg_stream.cuh -- the single-barrier PCG with every vector in global memory,
// for frames too large for any on-chip placement (3840x2160: 8.3 M unknowns;
// included by densify.cu after pcg_big.cuh).
//
// Same recurrences and one grid barrier + 10-value deterministic all-reduce
// per iteration as k_pcg_tmem. Each block owns a contiguous chunk; threads
// stride over it. p, r and q are double-buffered by phase parity so the halo
// recompute of phase k+1 (p_{k+1} = z_k + beta p_k for the neighbouring
// blocks' boundary rows, from their phase-k r, q, p) never races the
// neighbours' own phase-(k+1) writes; x, xs and rs are per-unknown and owned.
// Per iteration about 160 B per unknown stream through HBM (the reference's
// own formulation moves 104 B over three passes and three reductions).
#pragma once

namespace dco_gpu {
namespace {


struct StreamVecs {
    double* p[2];
    double* r[2];
    double* q[2];
    double* x;
    double* xs;
    double* rs;
};

// THREADS per block (one block per SM); kB elements per thread whose loads
// are batched ahead of the stores
template <int THREADS, int kB>
__global__ void __launch_bounds__(THREADS, 1) k_pcg_stream(CGArgs a, StreamVecs sv, GridBar* bar) {
    __shared__ double sm[32 * 16];
    __shared__ double s_w1[32 * 4];
    const int w = a.w, h = a.h;
    const int n = static_cast<int>(a.n);
    const int nb = gridDim.x;
    const int qn = n / nb, rem = n - qn * nb;
    const int base = blockIdx.x * qn + min(static_cast<int>(blockIdx.x), rem);
    const int size = qn + (static_cast<int>(blockIdx.x) < rem ? 1 : 0);
    const int end = base + size;
    const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
    unsigned gen = 0;

    unsigned long long anchors = a.anchors_dev ? *a.anchors_dev : a.anchors_host;
    if (anchors == 0) {
        const float* fb = (a.fallback && (!a.fallback_valid || *a.fallback_valid)) ? a.fallback : nullptr;
        for (int i = base + t; i < end; i += THREADS) a.dense[i] = fb ? fb[i] : __int_as_float(0x7fc00000);
        if (blockIdx.x == 0 && t == 0) {
            a.out->status = 3;
            a.out->iterations = 0;
        }
        return;
    }
    const double cterm = a.constant_term_dev ? *a.constant_term_dev : a.constant_term_host;

    // setup (densify.cpp:147-166): x = initial, r = b - A x, z = M r, p = z
    double tot[5] = {0.0, 0.0, 0.0, 0.0, 0.0};
    for (int i = base + t; i < end; i += THREADS) {
        const int xx = i % w, y = i / w;
        const double ax = apply_at(a.diag, a.ch, a.cv, a.init, w, h, i, xx, y);
        const double xi = a.init[i];
        const double b = a.rhs[i];
        const double d = a.diag[i];
        const double pr = d > 0.0 ? 1.0 / d : 1.0;
        const double ri = b - ax;
        const double zi = pr * ri;
        a.prec[i] = pr;
        sv.x[i] = xi;
        sv.xs[i] = xi;
        sv.rs[i] = ri;
        sv.r[0][i] = ri;
        sv.p[0][i] = zi;
        sv.q[0][i] = 0.0;
        tot[0] += b * b;
        tot[1] += ri * ri;
        tot[2] += ri * zi;
        tot[3] += xi * ax;
        tot[4] += b * xi;
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
    double alpha = 0.0, beta = 0.0, eta = 0.0;  // iteration iter-1's scalars
    // p_iter at index j: its owner's P1 value inside this block, the halo
    // recompute outside (identical FMA sequence, identical bits)
    if (a.max_iter > 0 && snorm / denom > a.tol) {
        for (;;) {
            const int cur = iter & 1, prv = cur ^ 1;  // buffers of phase iter / iter-1
            double* const p_c = sv.p[cur];
            double* const r_c = sv.r[cur];
            double* const q_c = sv.q[cur];
            const double* const p_p = sv.p[prv];
            const double* const r_p = sv.r[prv];
            const double* const q_p = sv.q[prv];
            double v[10];
#pragma unroll
            for (int c = 0; c < 10; ++c) v[c] = 0.0;
            // P1: updates of iteration iter-1 into the phase-iter buffers. Every
            // element's loads of a batch of kB are issued before any store (the
            // vectors may alias as far as the compiler knows), for bytes in flight.
            for (int i0 = base + t; i0 < end; i0 += kB * THREADS) {
                double pr[kB], rsi[kB], ri[kB], pold[kB], xo[kB], qo[kB], xso[kB];
#pragma unroll
                for (int u = 0; u < kB; ++u) {
                    const int i = i0 + u * THREADS;
                    if (i < end) {
                        pr[u] = a.prec[i];
                        rsi[u] = sv.rs[i];
                        if (iter) {
                            pold[u] = p_p[i];
                            xo[u] = sv.x[i];
                            qo[u] = q_p[i];
                            ri[u] = r_p[i];
                            if (eta > 0.0) xso[u] = sv.xs[i];
                        } else {
                            ri[u] = r_c[i];
                        }
                    }
                }
#pragma unroll
                for (int u = 0; u < kB; ++u) {
                    const int i = i0 + u * THREADS;
                    if (i >= end) break;
                    if (iter) {
                        const double xk = __fma_rn(alpha, pold[u], xo[u]);
                        sv.x[i] = xk;
                        ri[u] = __fma_rn(-alpha, qo[u], ri[u]);
                        r_c[i] = ri[u];
                        p_c[i] = __fma_rn(beta, pold[u], pr[u] * ri[u]);
                        if (eta > 0.0) {
                            rsi[u] = __fma_rn(eta, ri[u] - rsi[u], rsi[u]);
                            sv.rs[i] = rsi[u];
                            sv.xs[i] = __fma_rn(eta, xk - xso[u], xso[u]);
                        }
                    }
                    const double e = ri[u] - rsi[u];
                    v[1] = __fma_rn(rsi[u], rsi[u], v[1]);
                    v[2] = __fma_rn(pr[u] * ri[u], ri[u], v[2]);
                    v[3] = __fma_rn(rsi[u], e, v[3]);
                    v[4] = __fma_rn(e, e, v[4]);
                }
            }
#pragma unroll
            for (int c = 1; c <= 4; ++c) {
#pragma unroll
                for (int off = 16; off > 0; off >>= 1) v[c] += __shfl_xor_sync(0xffffffffu, v[c], off);
                if (lane == 0) s_w1[warp * 4 + (c - 1)] = v[c];
                v[c] = 0.0;
            }
            __syncthreads();  // this block's p_iter is complete (global memory, block scope)
            // P2: q = A p (densify.cpp:125-129), pq, S2, S3, T2, U2, U3
            auto p_at = [&](int j) -> double {
                if (j >= base && j < end) return p_c[j];  // this block's P1 (CTA barrier above)
                if (!iter) return __ldcg(p_c + j);         // p_0, written in setup before the barrier
                // neighbouring block: its p_iter from its phase-(iter-1) values
                const double rj = __fma_rn(-alpha, __ldcg(q_p + j), __ldcg(r_p + j));
                return __fma_rn(beta, __ldcg(p_p + j), __ldcg(a.prec + j) * rj);
            };
            // (x, y) of i advanced incrementally (no per-element division); loads
            // of a batch of kB elements first, as in P1
            int xx = (base + t) % w, y = (base + t) / w;
            const int sx = THREADS % w, sy = THREADS / w;
            for (int i0 = base + t; i0 < end; i0 += kB * THREADS) {
                double pk[kB], dg[kB], ce[kB], cw[kB], cs[kB], cn[kB], pe[kB], pw[kB], ps[kB], pn[kB];
                double ri[kB], rsi[kB], pr[kB];
                int ux[kB], uy[kB];
#pragma unroll
                for (int u = 0; u < kB; ++u) {
                    ux[u] = xx;
                    uy[u] = y;
                    xx += sx;
                    y += sy;
                    if (xx >= w) {
                        xx -= w;
                        ++y;
                    }
                }
#pragma unroll
                for (int u = 0; u < kB; ++u) {
                    const int i = i0 + u * THREADS;
                    if (i < end) {
                        pk[u] = p_c[i];
                        dg[u] = a.diag[i];
                        ri[u] = r_c[i];
                        rsi[u] = sv.rs[i];
                        pr[u] = a.prec[i];
                        if (ux[u] + 1 < w) {
                            ce[u] = a.ch[i];
                            pe[u] = p_at(i + 1);
                        }
                        if (ux[u] > 0) {
                            cw[u] = a.ch[i - 1];
                            pw[u] = p_at(i - 1);
                        }
                        if (uy[u] + 1 < h) {
                            cs[u] = a.cv[i];
                            ps[u] = p_at(i + w);
                        }
                        if (uy[u] > 0) {
                            cn[u] = a.cv[i - w];
                            pn[u] = p_at(i - w);
                        }
                    }
                }
#pragma unroll
                for (int u = 0; u < kB; ++u) {
                    const int i = i0 + u * THREADS;
                    if (i >= end) break;
                    double acc = dg[u] * pk[u];
                    if (ux[u] + 1 < w) acc = __fma_rn(-ce[u], pe[u], acc);
                    if (ux[u] > 0) acc = __fma_rn(-cw[u], pw[u], acc);
                    if (uy[u] + 1 < h) acc = __fma_rn(-cs[u], ps[u], acc);
                    if (uy[u] > 0) acc = __fma_rn(-cn[u], pn[u], acc);
                    q_c[i] = acc;
                    const double pq_ = pr[u] * acc;
                    v[0] = __fma_rn(pk[u], acc, v[0]);
                    v[5] = __fma_rn(pq_, ri[u], v[5]);
                    v[6] = __fma_rn(pq_, acc, v[6]);
                    v[7] = __fma_rn(rsi[u], acc, v[7]);
                    v[8] = __fma_rn(ri[u] - rsi[u], acc, v[8]);
                    v[9] = __fma_rn(acc, acc, v[9]);
                }
            }
            if (lane == 0) {
#pragma unroll
                for (int c = 1; c <= 4; ++c) v[c] = s_w1[warp * 4 + (c - 1)];
            }
            double res[10];
            barrier_reduce<10, false>(v, bar, a.part, gen, sm, res);  // the next P1/P2 CTA barrier guards sm
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
    for (int i = base + t; i < end; i += THREADS) {
        a.xs[i] = sv.xs[i];
        a.dense[i] = static_cast<float>(dmax0(sv.xs[i]));
    }
    {
        double z[1] = {0.0}, dummy[1];
        barrier_reduce<1>(z, bar, a.part, gen, sm, dummy);  // xs visible grid-wide
    }
    double o[2] = {0.0, 0.0};
    for (int i = base + t; i < end; i += THREADS) {
        const int xx = i % w, y = i / w;
        const double xsi = __ldcg(a.xs + i);
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
