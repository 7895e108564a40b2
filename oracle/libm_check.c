/* libm_check.c — pins paper_2203_02300_b200/csrc/dco_libm.h (the device
 * replicas) against this host's glibc libm, which is what the reference and
 * the C restatement call. Test infrastructure (run by
 * tests/test_libm_replica.py). Each mode prints "<mode> <checked> <mismatches>".
 *
 *   exp_ad <lambda_ad> [step]  every float f in [0,1] (stride step): the exact
 *                              argument -(double)f*255/lambda_ad of the AD term
 *                              (stereo.cpp:142)
 *   exp_rand <n>               random doubles over [-800, 720] + edge cases
 *   hypotf <n>                 random float pairs (flow-sized and wide)
 *   hypot <n>                  random float pairs promoted to double (contour.cpp:68)
 *   atan2f <n>                 random pairs + pairs near the NMS sector edges
 */
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "../paper_2203_02300_b200/csrc/dco_exp_table.h"
#include "../paper_2203_02300_b200/csrc/dco_libm.h"

static uint64_t rng_state = 0x9E3779B97F4A7C15ull;
static uint64_t rnd(void) {
    rng_state ^= rng_state >> 12;
    rng_state ^= rng_state << 25;
    rng_state ^= rng_state >> 27;
    return rng_state * 0x2545F4914F6CDD1Dull;
}
static double uni(double lo, double hi) { return lo + (hi - lo) * ((rnd() >> 11) * 0x1.0p-53); }
static float rfloat_bits(void) {
    /* random finite float over all exponents */
    uint32_t u;
    do {
        u = (uint32_t)rnd();
    } while ((u & 0x7f800000u) == 0x7f800000u);
    return dco_asf32(u);
}

static int same64(double a, double b) { return dco_asu64(a) == dco_asu64(b); }
static int same32(float a, float b) { return dco_asu32(a) == dco_asu32(b); }

int main(int argc, char** argv) {
    if (argc < 2) return 2;
    const char* mode = argv[1];
    unsigned long long checked = 0, bad = 0;
    if (!strcmp(mode, "exp_ad")) {
        double lambda = argc > 2 ? atof(argv[2]) : 10.0;
        uint32_t step = argc > 3 ? (uint32_t)atoi(argv[3]) : 1;
        for (uint32_t u = 0; u <= 0x3f800000u; u += step) {
            float f = dco_asf32(u);
            double c_ad = (double)f * 255.0;
            double x = -c_ad / lambda;
            double want = exp(x), got = dco_exp(x, dco_exp_table);
            ++checked;
            if (!same64(want, got)) {
                if (bad < 5) fprintf(stderr, "exp mismatch x=%a want=%a got=%a\n", x, want, got);
                ++bad;
            }
            if (u > 0x3f800000u - step) break;
        }
    } else if (!strcmp(mode, "exp_rand")) {
        long n = atol(argv[2]);
        const double edges[] = {0.0, -0.0, 0x1p-60, -0x1p-60, 0x1p-54, -0x1p-54, 511.9, -511.9,
                                512.0, -512.0, 700.0, -700.0, -708.4, -709.1, -720.0, -744.0,
                                -745.2, -746.0, 709.7, 710.0, 1e-300, -1e-300, 1.0, -1.0};
        for (size_t i = 0; i < sizeof(edges) / sizeof(edges[0]); ++i) {
            ++checked;
            if (!same64(exp(edges[i]), dco_exp(edges[i], dco_exp_table))) {
                fprintf(stderr, "exp edge mismatch x=%a\n", edges[i]);
                ++bad;
            }
        }
        for (long i = 0; i < n; ++i) {
            double x = (i & 1) ? uni(-800.0, 720.0) : uni(-30.0, 1.0);
            ++checked;
            if (!same64(exp(x), dco_exp(x, dco_exp_table))) {
                if (bad < 5) fprintf(stderr, "exp mismatch x=%a\n", x);
                ++bad;
            }
        }
    } else if (!strcmp(mode, "hypotf")) {
        long n = atol(argv[2]);
        for (long i = 0; i < n; ++i) {
            float a, b;
            if (i % 3 == 0) {
                a = rfloat_bits();
                b = rfloat_bits();
            } else {
                a = (float)uni(-40.0, 40.0);
                b = (i % 3 == 1) ? (float)uni(-40.0, 40.0) : (float)uni(-1e-3, 1e-3);
            }
            ++checked;
            if (!same32(hypotf(a, b), dco_hypotf(a, b))) {
                if (bad < 5) fprintf(stderr, "hypotf mismatch %a %a\n", a, b);
                ++bad;
            }
        }
    } else if (!strcmp(mode, "hypot")) {
        long n = atol(argv[2]);
        for (long i = 0; i < n; ++i) {
            float a, b;
            if (i % 4 == 0) {
                a = rfloat_bits();
                b = rfloat_bits();
            } else if (i % 4 == 3) {
                a = (float)uni(-40.0, 40.0);
                b = 0.0f;
            } else {
                a = (float)uni(-40.0, 40.0);
                b = (float)uni(-40.0, 40.0);
            }
            ++checked;
            if (!same64(hypot((double)a, (double)b), dco_hypot((double)a, (double)b))) {
                if (bad < 5) fprintf(stderr, "hypot mismatch %a %a\n", a, b);
                ++bad;
            }
        }
    } else if (!strcmp(mode, "atan2f")) {
        long n = atol(argv[2]);
        const double edges_deg[] = {22.5, 67.5, 112.5, 157.5};
        for (long i = 0; i < n; ++i) {
            float y, x;
            int kind = (int)(i % 4);
            if (kind == 0) {
                y = rfloat_bits();
                x = rfloat_bits();
            } else if (kind == 1) {
                y = (float)uni(-8.0, 8.0);
                x = (float)uni(-8.0, 8.0);
            } else {
                /* near a sector boundary: angle = edge +- a few ulps */
                double e = edges_deg[rnd() & 3] * 3.14159265358979323846 / 180.0;
                double mag = uni(1e-3, 8.0);
                double t = e + uni(-1e-6, 1e-6);
                x = (float)(mag * cos(t));
                y = (float)(mag * sin(t));
                if (kind == 3) {
                    x = -x;
                    y = -y;
                }
            }
            ++checked;
            if (!same32(atan2f(y, x), dco_atan2f(y, x))) {
                if (bad < 5) fprintf(stderr, "atan2f mismatch %a %a\n", y, x);
                ++bad;
            }
        }
        const float specials[] = {0.0f, -0.0f, 1.0f, -1.0f, INFINITY, -INFINITY, 1e-40f, -1e-40f, 3.0f};
        for (size_t i = 0; i < 9; ++i)
            for (size_t j = 0; j < 9; ++j) {
                ++checked;
                if (!same32(atan2f(specials[i], specials[j]), dco_atan2f(specials[i], specials[j]))) {
                    fprintf(stderr, "atan2f special mismatch %a %a\n", specials[i], specials[j]);
                    ++bad;
                }
            }
    } else {
        return 2;
    }
    printf("%s %llu %llu\n", mode, checked, bad);
    return bad ? 1 : 0;
}
