/*
 * dco_libm.h — bit-exact device (and host) replicas of the four glibc 2.39
 * libm routines the reference calls per pixel on its hot path:
 *
 *   exp(double)          AD term of the matching cost      stereo.cpp:142
 *   hypotf(float,float)  polar radius, Sobel magnitude      contour.cpp:18,194
 *   hypot(double,double) projection-confidence magnitude    contour.cpp:68
 *   atan2f(float,float)  NMS gradient sector               contour.cpp:217
 *
 * CUDA's own exp/hypotf/atan2f are accurate but not glibc's, so their last
 * bits differ from the CPU oracle. These restate glibc's published algorithms
 * operation for operation (ARM optimized-routines exp, FMA build as selected
 * by glibc's x86-64 ifunc on FMA hosts; the 2.35 double-precision hypotf; the
 * 2.35 hypot kernel without FMA; fdlibm atanf/atan2f). Constants are the
 * algorithms' published constants; the 128-entry exp table is regenerated
 * from its definition (oracle/gen_exp_table.py, which checks it against the
 * host libm). tests/test_cpu_boundary.py (with oracle/libm_check.c) pins every routine against the host
 * libm on large random + edge-case sweeps (exhaustively for the exp argument
 * domain the cost volume uses).
 *
 * Compile device code with --fmad=false (or host code with
 * -ffp-contract=off): every non-fused multiply-add below must stay unfused.
 */
#ifndef DCO_LIBM_H
#define DCO_LIBM_H

#include <stdint.h>

#if defined(__CUDACC__)
#define DCO_HD __host__ __device__ __forceinline__
#else
#include <math.h>
#include <string.h>
#define DCO_HD static inline
#endif

DCO_HD uint64_t dco_asu64(double x) {
#if defined(__CUDA_ARCH__)
    return (uint64_t)__double_as_longlong(x);
#else
    uint64_t u;
    memcpy(&u, &x, 8);
    return u;
#endif
}

DCO_HD double dco_asf64(uint64_t u) {
#if defined(__CUDA_ARCH__)
    return __longlong_as_double((long long)u);
#else
    double x;
    memcpy(&x, &u, 8);
    return x;
#endif
}

DCO_HD uint32_t dco_asu32(float x) {
#if defined(__CUDA_ARCH__)
    return (uint32_t)__float_as_uint(x);
#else
    uint32_t u;
    memcpy(&u, &x, 4);
    return u;
#endif
}

DCO_HD float dco_asf32(uint32_t u) {
#if defined(__CUDA_ARCH__)
    return __uint_as_float(u);
#else
    float x;
    memcpy(&x, &u, 4);
    return x;
#endif
}

DCO_HD double dco_fma(double a, double b, double c) {
#if defined(__CUDA_ARCH__)
    return __fma_rn(a, b, c);
#else
    return fma(a, b, c);
#endif
}

DCO_HD double dco_sqrt(double x) {
#if defined(__CUDA_ARCH__)
    return __dsqrt_rn(x);
#else
    return sqrt(x);
#endif
}

/* ---------------------------------------------------------------- exp --- */
/* glibc exp, EXP_TABLE_BITS = 7, FMA build. tab = dco_exp_table (256 u64),
 * passed in so device callers can stage it in shared memory. */
DCO_HD double dco_exp(double x, const uint64_t* tab) {
    const double inv_ln2_n = 0x1.71547652b82fep7;     /* N / ln 2 */
    const double shift = 0x1.8p52;
    const double neg_ln2_hi_n = -0x1.62e42fefa0000p-8; /* -ln2/N, split */
    const double neg_ln2_lo_n = -0x1.cf79abc9e3b3ap-47;
    const double c2 = 0x1.ffffffffffdbdp-2, c3 = 0x1.555555555543cp-3;
    const double c4 = 0x1.55555cf172b91p-5, c5 = 0x1.1111167a4d017p-7;

    uint32_t abstop = (uint32_t)(dco_asu64(x) >> 52) & 0x7ff;
    if (abstop - 0x3c9u >= 0x3fu) {
        if ((int32_t)(abstop - 0x3c9u) < 0) return 1.0 + x; /* |x| < 2^-54 */
        if (abstop >= 0x409u) {                                /* |x| >= 1024 */
            if (dco_asu64(x) == 0xfff0000000000000ull) return 0.0;
            if (abstop >= 0x7ffu) return 1.0 + x;
            return (dco_asu64(x) >> 63) ? 0.0 : dco_asf64(0x7ff0000000000000ull);
        }
        abstop = 0; /* 512 <= |x| < 1024: finish in the scaled branch */
    }
    double kd = dco_fma(x, inv_ln2_n, shift);
    uint64_t ki = dco_asu64(kd);
    kd -= shift;
    double r = dco_fma(kd, neg_ln2_hi_n, x);
    r = dco_fma(kd, neg_ln2_lo_n, r);
    uint32_t idx = 2u * (uint32_t)(ki & 127u);
    uint64_t top = ki << 45;
    double tail = dco_asf64(tab[idx]);
    uint64_t sbits = tab[idx + 1] + top;
    double r2 = r * r;
    double p23 = dco_fma(r, c3, c2);
    double p45 = dco_fma(r, c5, c4);
    double tmp = dco_fma(p23, r2, r + tail);
    tmp = dco_fma(r2 * r2, p45, tmp);
    if (abstop == 0) {
        double scale, y;
        if ((ki & 0x80000000u) == 0) {
            sbits -= 1009ull << 52;
            scale = dco_asf64(sbits);
            y = dco_fma(scale, tmp, scale);
            return 0x1p1009 * y;
        }
        sbits += 1022ull << 52;
        scale = dco_asf64(sbits);
        double st = scale * tmp;
        y = scale + st;
        if (y < 1.0) {
            double hi = y + 1.0;
            double lo = (scale - y) + st;
            y = ((1.0 - hi) + y) + lo;
            y = (y + hi) - 1.0;
            if (y == 0.0) y = 0.0;
        }
        return 0x1p-1022 * y;
    }
    double scale = dco_asf64(sbits);
    return dco_fma(scale, tmp, scale);
}

/* ------------------------------------------------------------- hypotf --- */
/* glibc >= 2.35 __ieee754_hypotf: one double-precision sqrt. */
DCO_HD float dco_hypotf(float x, float y) {
    uint32_t ax = dco_asu32(x) & 0x7fffffffu, ay = dco_asu32(y) & 0x7fffffffu;
    if (ax >= 0x7f800000u || ay >= 0x7f800000u) {
        if (ax == 0x7f800000u || ay == 0x7f800000u) return dco_asf32(0x7f800000u);
        return x + y; /* NaN */
    }
    double xd = (double)x, yd = (double)y;
    return (float)dco_sqrt(xd * xd + yd * yd);
}

/* -------------------------------------------------------------- hypot --- */
/* glibc >= 2.35 __hypot, non-FMA kernel (the x86-64 build has no FMA ifunc
 * for hypot). Scaling branches kept for completeness. */
DCO_HD double dco_hypot_kernel(double ax, double ay) {
    double h = dco_sqrt(ax * ax + ay * ay);
    double t1, t2;
    if (h <= 2.0 * ay) {
        double delta = h - ay;
        t1 = ax * (2.0 * delta - ax);
        t2 = (delta - 2.0 * (ax - ay)) * delta;
    } else {
        double delta = h - ax;
        t1 = 2.0 * delta * (ax - 2.0 * ay);
        t2 = (4.0 * delta - ay) * ay + delta * delta;
    }
    h -= (t1 + t2) / (2.0 * h);
    return h;
}

DCO_HD double dco_hypot(double x, double y) {
    const double large = 0x1p511, tiny = 0x1p-459, eps = 0x1p-54;
    const double scale = 0x1p-600;
    uint64_t ux = dco_asu64(x) & 0x7fffffffffffffffull, uy = dco_asu64(y) & 0x7fffffffffffffffull;
    if (ux >= 0x7ff0000000000000ull || uy >= 0x7ff0000000000000ull) {
        if (ux == 0x7ff0000000000000ull || uy == 0x7ff0000000000000ull)
            return dco_asf64(0x7ff0000000000000ull);
        return x + y;
    }
    x = dco_asf64(ux);
    y = dco_asf64(uy);
    double ax = x < y ? y : x;
    double ay = x < y ? x : y;
    if (ax > large) {
        if (ay <= ax * eps) return ax + ay;
        return dco_hypot_kernel(ax * scale, ay * scale) / scale;
    }
    if (ay < tiny) {
        if (ax >= ay / eps) return ax + ay;
        ax = dco_hypot_kernel(ax / scale, ay / scale) * scale;
        return ax;
    }
    if (ay <= ax * eps) return ax + ay;
    return dco_hypot_kernel(ax, ay);
}

/* ------------------------------------------------------- atanf/atan2f --- */
/* fdlibm s_atanf.c as built into glibc 2.39 (plain SSE float arithmetic). */
DCO_HD float dco_atanf(float x) {
    const float atanhi[4] = {dco_asf32(0x3eed6338u), dco_asf32(0x3f490fdau),
                             dco_asf32(0x3f7b985eu), dco_asf32(0x3fc90fdau)};
    const float atanlo[4] = {dco_asf32(0x31ac3769u), dco_asf32(0x33222168u),
                             dco_asf32(0x33140fb4u), dco_asf32(0x33a22168u)};
    const float at0 = dco_asf32(0x3eaaaaabu), at1 = dco_asf32(0xbe4ccccdu),
                at2 = dco_asf32(0x3e124925u), at3 = dco_asf32(0xbde38e38u),
                at4 = dco_asf32(0x3dba2e6eu), at5 = dco_asf32(0xbd9d8795u),
                at6 = dco_asf32(0x3d886b35u), at7 = dco_asf32(0xbd6ef16bu),
                at8 = dco_asf32(0x3d4bda59u), at9 = dco_asf32(0xbd15a221u),
                at10 = dco_asf32(0x3c8569d7u);
    uint32_t hx = dco_asu32(x);
    uint32_t ix = hx & 0x7fffffffu;
    int id;
    if (ix >= 0x4c000000u) { /* |x| >= 2^25 */
        if (ix > 0x7f800000u) return x + x;
        return (int32_t)hx > 0 ? atanhi[3] + atanlo[3] : -atanhi[3] - atanlo[3];
    }
    if (ix < 0x3ee00000u) {     /* |x| < 7/16 */
        if (ix < 0x31000000u) { /* |x| < 2^-29 */
            return x;           /* huge + x > 1: inexact, returns x */
        }
        id = -1;
    } else {
        x = dco_asf32(ix); /* fabsf */
        if (ix < 0x3f980000u) {     /* |x| < 1.1875 */
            if (ix < 0x3f300000u) { /* 7/16 <= |x| < 11/16 */
                id = 0;
                x = ((x + x) - 1.0f) / (x + 2.0f);
            } else { /* 11/16 <= |x| < 19/16 */
                id = 1;
                x = (x - 1.0f) / (x + 1.0f);
            }
        } else {
            if (ix < 0x401c0000u) { /* |x| < 2.4375 */
                id = 2;
                x = (x - 1.5f) / (x * 1.5f + 1.0f);
            } else { /* 2.4375 <= |x| < 2^25 */
                id = 3;
                x = -1.0f / x;
            }
        }
    }
    float z = x * x;
    float w = z * z;
    float s1 = z * (at0 + w * (at2 + w * (at4 + w * (at6 + w * (at8 + w * at10)))));
    float s2 = w * (at1 + w * (at3 + w * (at5 + w * (at7 + w * at9))));
    if (id < 0) return x - x * (s1 + s2);
    z = atanhi[id] - ((x * (s1 + s2) - atanlo[id]) - x);
    return ((int32_t)hx < 0) ? -z : z;
}

/* fdlibm e_atan2f.c as built into glibc 2.39: atan2f(y, x). */
DCO_HD float dco_atan2f(float y, float x) {
    const float pi_o_4 = dco_asf32(0x3f490fdbu), pi_o_2 = dco_asf32(0x3fc90fdbu),
                pi = dco_asf32(0x40490fdbu), pi_lo = dco_asf32(0xb3bbbd2eu);
    const float tiny = 1.0e-30f;
    uint32_t hx = dco_asu32(x), hy = dco_asu32(y);
    uint32_t ix = hx & 0x7fffffffu, iy = hy & 0x7fffffffu;
    if (ix > 0x7f800000u || iy > 0x7f800000u) return x + y; /* NaN */
    if (hx == 0x3f800000u) return dco_atanf(y);              /* x == 1 */
    uint32_t m = ((hy >> 31) & 1u) | ((hx >> 30) & 2u);
    if (iy == 0) {
        switch (m) {
            case 0:
            case 1: return y;
            case 2: return pi + tiny;
            default: return -pi - tiny;
        }
    }
    if (ix == 0) return ((int32_t)hy < 0) ? -pi_o_2 - tiny : pi_o_2 + tiny;
    if (ix == 0x7f800000u) {
        if (iy == 0x7f800000u) {
            switch (m) {
                case 0: return pi_o_4 + tiny;
                case 1: return -pi_o_4 - tiny;
                case 2: return 3.0f * pi_o_4 + tiny;
                default: return -3.0f * pi_o_4 - tiny;
            }
        }
        switch (m) {
            case 0: return 0.0f;
            case 1: return -0.0f;
            case 2: return pi + tiny;
            default: return -pi - tiny;
        }
    }
    if (iy == 0x7f800000u) return ((int32_t)hy < 0) ? -pi_o_2 - tiny : pi_o_2 + tiny;
    int32_t k = ((int32_t)iy - (int32_t)ix) >> 23;
    float z;
    if (k > 60) {
        z = pi_o_2 + 0.5f * pi_lo;
    } else if ((int32_t)hx < 0 && k < -60) {
        z = 0.0f;
    } else {
        float q = y / x;
        z = dco_atanf(dco_asf32(dco_asu32(q) & 0x7fffffffu));
    }
    switch (m) {
        case 0: return z;
        case 1: return dco_asf32(dco_asu32(z) ^ 0x80000000u);
        case 2: return pi - (z - pi_lo);
        default: return (z - pi_lo) - pi;
    }
}

#endif /* DCO_LIBM_H */
