/*
 * TEST INFRASTRUCTURE ONLY -- the CPU oracle for the multi-level F/B estimator.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
 * reference legs may load this library, and only as the checker (or as the
 * timed CPU baseline).  The product path (paper_2006_14970_b200) never links
 * or calls it.
 *
 * This file restates, in plain C, the reference algorithm of arXiv 2006.14970
 * as implemented in /root/reference/proj (fgmatte).  Every function names the
 * reference lines it follows.  The double-precision build is compiled with
 * -ffp-contract=off exactly like the reference (proj/CMakeLists.txt:23-24), so
 * that it is bitwise equal to the reference itself (checked against
 * oracle/_ref in tests/test_oracle.py).  A float instantiation of the same code
 * is provided only to calibrate the fp32 tolerance of the GPU path.
 *
 * Layout (same as the reference, image.hpp:12-26): planar, plane(c)[y*w + x].
 */
#include <math.h>
#include <stddef.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#include "fgm_oracle.h"

/* ---- level schedule: multilevel.cpp:17-44 --------------------------------- */
static int bit_width_u32(unsigned v) { return v ? 32 - __builtin_clz(v) : 0; }

int fgmo_num_levels(int w, int h) {
    if (w < 1 || h < 1) return -1;
    unsigned m = (unsigned)(w > h ? w : h);
    int n = m > 1 ? bit_width_u32(m - 1) : 0; /* multilevel.cpp:25-26 */
    return n < 1 ? 1 : n;
}

int fgmo_level_schedule(int w, int h, int low_res_threshold, int iters_low, int iters_high,
                        int* out_w, int* out_h, int* out_iters, int cap) {
    int n = fgmo_num_levels(w, h);
    if (n < 0) return -1;
    if (n > cap) return -2;
    for (int l = 1; l <= n; ++l) {
        int lw, lh;
        if (l == n) { /* multilevel.cpp:32-34 */
            lw = w;
            lh = h;
        } else {      /* multilevel.cpp:36-38 */
            double e = (double)l / (double)n;
            lw = (int)llround(pow((double)w, e));
            lh = (int)llround(pow((double)h, e));
        }
        int mx = lw > lh ? lw : lh;
        out_w[l - 1] = lw;
        out_h[l - 1] = lh;
        out_iters[l - 1] = mx <= low_res_threshold ? iters_low : iters_high; /* :40 */
    }
    return n;
}

/* ---- taps: image.cpp:71-83 ------------------------------------------------ */
typedef struct { int i0, i1; double t; } tap_t;

static void make_taps(int src, int dst, tap_t* taps) {
    const double scale = (double)src / (double)dst;
    for (int d = 0; d < dst; ++d) {
        double f = (d + 0.5) * scale - 0.5;
        if (f < 0.0) f = 0.0;
        const double max_f = (double)(src - 1);
        if (f > max_f) f = max_f;
        const int i0 = (int)f;
        taps[d].i0 = i0;
        taps[d].i1 = i0 + 1 < src - 1 ? i0 + 1 : src - 1;
        taps[d].t = f - (double)i0;
    }
}

void fgmo_make_taps(int src, int dst, int* i0, int* i1, double* t) {
    tap_t* taps = (tap_t*)malloc(sizeof(tap_t) * (size_t)dst);
    make_taps(src, dst, taps);
    for (int d = 0; d < dst; ++d) {
        i0[d] = taps[d].i0;
        i1[d] = taps[d].i1;
        t[d] = taps[d].t;
    }
    free(taps);
}

/* ---- the precision-generic core (instantiated for double and float) ------ */
#define REAL double
#define SFX(name) name##_f64
#include "fgm_oracle_core.inc"
#undef REAL
#undef SFX

#define REAL float
#define SFX(name) name##_f32
#include "fgm_oracle_core.inc"
#undef REAL
#undef SFX

/* ---- one pixel: multilevel.cpp:48-79 (solve_pixel_impl) ------------------- */
int fgmo_solve_pixel(double alpha_i, const double intensity[3], int n, const double* nalpha,
                     const double* nfg /* n x 3 */, const double* nbg /* n x 3 */, double omega,
                     double eps_r, int clamp, double fg_out[3], double bg_out[3]) {
    if (!(omega >= 0.0) || !(eps_r > 0.0)) return 1;  /* MlParams::validate, :10-15 */
    if (n < 1) return 1;                              /* :55 */
    const double u[2] = {alpha_i, 1.0 - alpha_i};     /* PixelSystem::init, multilevel.hpp:50-56 */
    double diag[2] = {u[0] * u[0], u[1] * u[1]};
    const double off = u[0] * u[1];
    double rhs[2][3];
    for (int k = 0; k < 2; ++k)
        for (int c = 0; c < 3; ++c) rhs[k][c] = intensity[c] * u[k];
    for (int j = 0; j < n; ++j) {                     /* add_neighbor, multilevel.hpp:58-64 */
        const double d = eps_r + omega * fabs(alpha_i - nalpha[j]);
        const double* nb[2] = {nfg + 3 * j, nbg + 3 * j};
        for (int k = 0; k < 2; ++k) {
            diag[k] += d;
            for (int c = 0; c < 3; ++c) rhs[k][c] += d * nb[k][c];
        }
    }
    const double det = diag[0] * diag[1] - off * off; /* :66 */
    if (!(det > 0.0) || !isfinite(1.0 / det)) return 2;
    const double inv_det = 1.0 / det;
    double* out[2] = {fg_out, bg_out};
    for (int c = 0; c < 3; ++c)                       /* solve_raw, multilevel.hpp:69-74 */
        for (int k = 0; k < 2; ++k) {
            double v = (diag[1 - k] * rhs[k][c] - off * rhs[1 - k][c]) * inv_det;
            if (clamp) v = v < 0.0 ? 0.0 : (v > 1.0 ? 1.0 : v); /* clamp01, image.hpp:64 */
            out[k][c] = v;
        }
    return 0;
}
