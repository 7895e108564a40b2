// pcg_band.cuh -- the single-barrier PCG + MR solve of ONE system split into
// row bands over several ranks ("1-row p halo per SpMV plus an
// all-reduce of the scalar groups per iteration"), with the exchange fused
// into the persistent kernel instead of NCCL calls between launches:
//  * each rank's blocks reduce their 10 values with the deterministic grid
//    barrier of grid_reduce.cuh over that rank's blocks only;
//  * block 0 of every rank stores the rank's vector into slot [rank] of every
//    rank's exchange table (peer memory over NVLink, st.release.sys on a
//    monotonic per-rank flag); every block polls its own table's flags and
//    sums the ranks' vectors in rank order, so all ranks hold the same bits
//    and take the same branch at every iteration;
//  * the p halo of the band's first / last row is recomputed from the
//    neighbouring rank's phase buffers (r, q, p, prec of its boundary row,
//    read over NVLink), exactly as within a rank.
// With fewer GPUs than ranks the ranks run as block groups of ONE cooperative
// launch over all ranks' data on one GPU (B200_PROFILING: no separate kernels
// that wait on each other); the code path is the same, only the pointers are
// local. Included by densify.cu after pcg_stream.cuh.
#pragma once

namespace dco_gpu {
namespace {

constexpr int kMaxBandRanks = 8;
constexpr int kBandThreads = 384;
constexpr int kBandB = 2;

// Per-rank arena layout (doubles): p[2], r[2], q[2], prec, x, xs, rs (n each),
// then the exchange table [2][kMaxBandRanks][16] and the partials of the
// local barrier; flags / counters live in a separate word area.
struct BandSide {
    const double* p[2];
    const double* r[2];
    const double* q[2];
    const double* prec;
    const double* x;     // initial iterate (setup)
    const double* xs;    // smoothed solution (final objective)
};  // all pointing at the neighbour's boundary row; null when there is none

struct BandRank {
    CGArgs a;      // this rank's system: n = owned unknowns, h = owned rows,
                   // cv readable one row above the band when y0 > 0
    StreamVecs sv;
    int y0, H;     // global row of local row 0; full height
    int rank, ranks;
    BandSide up, dn;
    GridBar* bar;
    double* xslots;                       // this rank's table [2][kMaxBandRanks][16]
    unsigned* xflags;                     // this rank's flags [kMaxBandRanks][32]
    unsigned* xgen;                       // exchanges done by earlier solves (same on all ranks)
    double* peer_slots[kMaxBandRanks];    // every rank's table (this one included)
    unsigned* peer_flags[kMaxBandRanks];  // every rank's flags
};

struct BandRed {
    const BandRank* R;
    int nb, lb;
    unsigned gen;   // local barrier generation
    unsigned xg;    // cross-rank exchange generation
};

// Local barrier-reduce over this rank's blocks, then the rank-ordered sum of
// every rank's totals.
template <int K>
__device__ __forceinline__ void band_reduce(double (&v)[K], BandRed& st, double* sm, double (&res)[K]) {
    const BandRank& R = *st.R;
    double loc[K];
    barrier_reduce_of<K, true>(v, R.bar, R.a.part, st.gen, sm, loc, st.nb, st.lb);
    const unsigned g = ++st.xg;
    if (st.lb == 0 && threadIdx.x == 0) {
        const size_t off = (static_cast<size_t>(g & 1u) * kMaxBandRanks + R.rank) * 16;
        for (int r = 0; r < R.ranks; ++r) {
#pragma unroll
            for (int k = 0; k < K; ++k) __stcg(R.peer_slots[r] + off + k, loc[k]);
        }
        for (int r = 0; r < R.ranks; ++r)
            asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(R.peer_flags[r] + R.rank * 32), "r"(g)
                         : "memory");
    }
    if (threadIdx.x < R.ranks) {
        unsigned c;
        do {
            asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(c) : "l"(R.xflags + threadIdx.x * 32) : "memory");
        } while (static_cast<int>(c - g) < 0);
    }
    __syncthreads();
    double* sres = sm + 32 * 16 - 16;
    if (threadIdx.x < K) {
        const double* t = R.xslots + static_cast<size_t>(g & 1u) * kMaxBandRanks * 16 + threadIdx.x;
        double s = 0.0;
        for (int r = 0; r < R.ranks; ++r) s += __ldcg(t + r * 16);
        sres[threadIdx.x] = s;
    }
    __syncthreads();
#pragma unroll
    for (int k = 0; k < K; ++k) res[k] = sres[k];
    __syncthreads();
}

// desc: the ranks this launch runs (all of them in the one-GPU emulation, one
// per GPU otherwise); bpr blocks per rank.
template <int THREADS, int kB>
__global__ void __launch_bounds__(THREADS, 1) k_pcg_band(const BandRank* __restrict__ desc, int bpr) {
    __shared__ double sm[32 * 16];
    __shared__ double s_w1[32 * 4];
    __shared__ BandRank s_R;
    if (threadIdx.x == 0) s_R = desc[blockIdx.x / bpr];
    __syncthreads();
    const BandRank& R = s_R;
    const CGArgs& a = R.a;
    const StreamVecs& sv = R.sv;
    BandRed st;
    st.R = &R;
    st.nb = bpr;
    st.lb = blockIdx.x % bpr;
    st.gen = 0;
    st.xg = *R.xgen;  // exchanges of earlier solves (read before this solve's first exchange)
    const unsigned xg0 = st.xg;
    const int w = a.w;
    const int n = static_cast<int>(a.n);
    const int nb = bpr, lb = st.lb;
    const int qn = n / nb, rem = n - qn * nb;
    const int base = lb * qn + min(lb, rem);
    const int size = qn + (lb < rem ? 1 : 0);
    const int end = base + size;
    const int t = threadIdx.x, lane = t & 31, warp = t >> 5;

    const unsigned long long anchors = a.anchors_dev ? *a.anchors_dev : a.anchors_host;
    if (anchors == 0) {
        const float* fb = (a.fallback && (!a.fallback_valid || *a.fallback_valid)) ? a.fallback : nullptr;
        for (int i = base + t; i < end; i += THREADS) a.dense[i] = fb ? fb[i] : __int_as_float(0x7fc00000);
        if (lb == 0 && t == 0) {
            a.out->status = 3;
            a.out->iterations = 0;
        }
        return;
    }
    const double cterm = a.constant_term_dev ? *a.constant_term_dev : a.constant_term_host;
    // x of a pixel's 4 neighbours: the band's own rows locally, the rows
    // outside the band from the neighbouring rank (valid only where the
    // global row exists)
    auto apply_band = [&](const double* xv, const double* up_x, const double* dn_x, int i, int xx, int y) {
        const int gy = R.y0 + y;
        // (other blocks' and ranks' values: L2 loads, after an exchange)
        double acc = a.diag[i] * __ldcg(xv + i);
        if (xx + 1 < w) acc = __fma_rn(-a.ch[i], __ldcg(xv + i + 1), acc);
        if (xx > 0) acc = __fma_rn(-a.ch[i - 1], __ldcg(xv + i - 1), acc);
        if (gy + 1 < R.H) acc = __fma_rn(-a.cv[i], i + w < n ? __ldcg(xv + i + w) : __ldcg(dn_x + (i + w - n)), acc);
        if (gy > 0) acc = __fma_rn(-a.cv[i - w], i - w >= 0 ? __ldcg(xv + i - w) : __ldcg(up_x + i), acc);
        return acc;
    };

    // setup (densify.cpp:147-166): x = initial, r = b - A x, z = M r, p = z.
    // A x0 needs the neighbours' initial rows: x0 = initial is published in
    // sv.x before a first exchange.
    for (int i = base + t; i < end; i += THREADS) {
        sv.x[i] = a.init[i];
        const double d = a.diag[i];
        a.prec[i] = d > 0.0 ? 1.0 / d : 1.0;
    }
    {
        double z[1] = {0.0}, dummy[1];
        band_reduce<1>(z, st, sm, dummy);  // x0 and prec visible to the neighbouring ranks
    }
    double tot[5] = {0.0, 0.0, 0.0, 0.0, 0.0};
    for (int i = base + t; i < end; i += THREADS) {
        const int xx = i % w, y = i / w;
        const double ax = apply_band(sv.x, R.up.x, R.dn.x, i, xx, y);
        const double xi = sv.x[i];
        const double b = a.rhs[i];
        const double pr = a.prec[i];
        const double ri = b - ax;
        const double zi = pr * ri;
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
    band_reduce<5>(tot, st, sm, tot);
    const double bnorm = sqrt(tot[0]);
    const double denom = bnorm > 0.0 ? bnorm : 1.0;
    double snorm = sqrt(tot[1]);
    double rho = tot[2];
    if (lb == 0 && t == 0) {
        if (a.hist_cap > 0) a.hist[0] = snorm;
        a.out->objective_initial = tot[3] - 2.0 * tot[4] + cterm;
    }

    int iter = 0;
    double alpha = 0.0, beta = 0.0, eta = 0.0;
    if (a.max_iter > 0 && snorm / denom > a.tol) {
        for (;;) {
            const int cur = iter & 1, prv = cur ^ 1;
            double* const p_c = sv.p[cur];
            double* const r_c = sv.r[cur];
            double* const q_c = sv.q[cur];
            const double* const p_p = sv.p[prv];
            const double* const r_p = sv.r[prv];
            const double* const q_p = sv.q[prv];
            double v[10];
#pragma unroll
            for (int c = 0; c < 10; ++c) v[c] = 0.0;
            // P1: updates of iteration iter-1 into the phase-iter buffers
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
            __syncthreads();
            // P2: q = A p. p_iter of an index outside this block: recomputed
            // from its owner's phase-(iter-1) values (identical FMA sequence),
            // from this rank's buffers or the neighbouring rank's boundary row.
            auto p_side = [&](const BandSide& S, int x) -> double {
                if (!iter) return __ldcg(S.p[cur] + x);
                const double rj = __fma_rn(-alpha, __ldcg(S.q[prv] + x), __ldcg(S.r[prv] + x));
                return __fma_rn(beta, __ldcg(S.p[prv] + x), __ldcg(S.prec + x) * rj);
            };
            auto p_at = [&](int j) -> double {
                if (j >= base && j < end) return p_c[j];
                if (j < 0) return p_side(R.up, j + w);
                if (j >= n) return p_side(R.dn, j - n);
                if (!iter) return __ldcg(p_c + j);
                const double rj = __fma_rn(-alpha, __ldcg(q_p + j), __ldcg(r_p + j));
                return __fma_rn(beta, __ldcg(p_p + j), __ldcg(a.prec + j) * rj);
            };
            int xx = (base + t) % w, y = (base + t) / w;
            const int sx = THREADS % w, sy = THREADS / w;
            for (int i0 = base + t; i0 < end; i0 += kB * THREADS) {
                double pk[kB], dg[kB], ce[kB], cw[kB], cs[kB], cn[kB], pe[kB], pw[kB], ps[kB], pn[kB];
                double ri[kB], rsi[kB], pr[kB];
                int ux[kB], uy[kB];
#pragma unroll
                for (int u = 0; u < kB; ++u) {
                    ux[u] = xx;
                    uy[u] = R.y0 + y;  // global row
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
                        if (uy[u] + 1 < R.H) {
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
                    if (uy[u] + 1 < R.H) acc = __fma_rn(-cs[u], ps[u], acc);
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
            band_reduce<10>(v, st, sm, res);
            if (iter > 0) {
                snorm = sqrt(res[1]);
                if (lb == 0 && t == 0 && iter < a.hist_cap) a.hist[iter] = snorm;
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
        band_reduce<1>(z, st, sm, dummy);  // xs visible to this rank and its neighbours
    }
    double o[2] = {0.0, 0.0};
    for (int i = base + t; i < end; i += THREADS) {
        const int xx = i % w, y = i / w;
        const double xsi = __ldcg(a.xs + i);
        o[0] += xsi * apply_band(a.xs, R.up.xs, R.dn.xs, i, xx, y);
        o[1] += a.rhs[i] * xsi;
    }
    band_reduce<2>(o, st, sm, o);
    if (lb == 0 && t == 0) {
        a.out->objective_final = o[0] - 2.0 * o[1] + cterm;
        a.out->status = 0;
        a.out->iterations = iter;
        a.out->relative_residual = snorm / denom;
    }
    if (lb == 0 && t == 0) *R.xgen = st.xg;  // every block of the rank read xgen before its first exchange
    (void)xg0;
}

}  // namespace
}  // namespace dco_gpu
