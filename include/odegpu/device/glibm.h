/*
 * glibm.h — the glibc 2.39 libm routines the reference solver calls,
 * restated for the exact-parity build (and compiled unchanged on the host,
 * where tests/test_glibm_cpu.py checks them bit for bit against the live
 * libm).
 *
 * Why: the reference (/root/reference/proj, g++ -O3, no -march) evaluates
 * std::cos (Duffing forcing, models/duffing.hpp:37-42), the sin/cos pairs of
 * the Keller-Miksis excitation (g++ merges them into sincos,
 * models/keller_miksis.hpp:93-99), std::pow in the Keller-Miksis RHS
 * (keller_miksis.hpp:90) and std::pow(ratio, -0.2) in the step controller
 * (steppers.hpp:185) through glibc's libm. Its accept / reject decisions and
 * event detections therefore depend on glibc's last-bit rounding, and
 * libdevice (what nvcc's ::cos / ::pow are) differs from glibc in ~16 % of
 * cos / sincos results (scripts/glibm_call_stats.py). Exact parity of integer
 * counts needs glibc's own arithmetic on the device.
 *
 * What: on x86_64 with FMA + AVX2 (this image's CPUs) glibc resolves its
 * ifuncs to the "_fma" builds of
 *   - sysdeps/ieee754/dbl-64/s_sin.c and s_sincos.c — the IBM Accurate
 *     Mathematical Library: Cody-Waite reduction by pi/2 in three parts
 *     (reduce_sincos), a 128-point table of sin / cos with correction terms
 *     (__sincostab) and short polynomials around the table point (do_sin,
 *     do_cos), a Taylor polynomial near 0 (TAYLOR_SIN);
 *   - sysdeps/ieee754/dbl-64/e_pow.c — the Arm optimized-routines pow:
 *     log(x) to ~68 bits from a 128-entry table (log_inline), y log x as a
 *     double-double, exp from a 128-entry table of 2^(j/128) (exp_inline).
 * Every function below follows those sources operation for operation, with
 * the a*b+c contractions the _fma objects contain (read from their machine
 * code: the operand order of each vfmadd / vfnmadd / vfmsub is kept), and the
 * constants of glibm_tables.h (generated from the installed libm.so.6 by
 * scripts/gen_glibm_tables.py). Device code uses __dadd_rn / __dmul_rn /
 * __fma_rn so no compiler contraction can intervene; host code must be
 * compiled with -ffp-contract=off (plain + - * are then IEEE operations).
 *
 * Scope: |x| < 105414350 for cos / sincos (glibc's simple-reduction range;
 * beyond it glibc calls __branred, which is not restated: glm_trig_in_range()
 * tells the caller to use another path); pow for every input class the
 * solver can produce (the special-case branches of e_pow.c are restated too).
 */
#ifndef ODEGPU_DEVICE_GLIBM_H
#define ODEGPU_DEVICE_GLIBM_H

#include <math.h>
#include <stdint.h>
#include <string.h>

#include "odegpu/device/glibm_tables.h"

#if defined(__CUDACC__)
#define GLM_FN static __device__ __forceinline__ /* host code calls libm itself */
#else
#define GLM_FN static inline
#endif

/* IEEE operations, round to nearest, never contracted. */
#if defined(__CUDA_ARCH__)
#define GLM_ADD(a, b) __dadd_rn((a), (b))
#define GLM_SUB(a, b) __dsub_rn((a), (b))
#define GLM_MUL(a, b) __dmul_rn((a), (b))
#define GLM_FMA(a, b, c) __fma_rn((a), (b), (c))
#else
#define GLM_ADD(a, b) ((a) + (b))
#define GLM_SUB(a, b) ((a) - (b))
#define GLM_MUL(a, b) ((a) * (b))
#define GLM_FMA(a, b, c) fma((a), (b), (c))
#endif

GLM_FN double glm_asdouble(uint64_t u) {
#if defined(__CUDA_ARCH__)
    return __longlong_as_double((long long)u);
#else
    double d;
    memcpy(&d, &u, sizeof d);
    return d;
#endif
}

GLM_FN uint64_t glm_asuint64(double d) {
#if defined(__CUDA_ARCH__)
    return (uint64_t)__double_as_longlong(d);
#else
    uint64_t u;
    memcpy(&u, &d, sizeof u);
    return u;
#endif
}

#if defined(__CUDA_ARCH__)
#define GLM_LD(table, i) glm_asdouble(__ldg(&(table)[i]))
#else
#define GLM_LD(table, i) glm_asdouble((table)[i])
#endif
#define GLM_C(name) glm_asdouble(GLM_K_##name)

GLM_FN double glm_fabs(double x) { return glm_asdouble(glm_asuint64(x) & 0x7fffffffffffffffull); }
GLM_FN double glm_neg(double x) { return glm_asdouble(glm_asuint64(x) ^ 0x8000000000000000ull); }
GLM_FN double glm_copysign(double m, double s) {
    return glm_asdouble((glm_asuint64(m) & 0x7fffffffffffffffull) | (glm_asuint64(s) & 0x8000000000000000ull));
}

/* ---------------------------------------------------------------- s_sin.c */

/* TAYLOR_SIN (s_sin.c): a + (((((s5 xx + s4) xx + s3) xx + s2) xx + s1) a
 * - da/2) xx + da, for |a| < 0.126. */
GLM_FN double glm_taylor_sin(double a, double da) {
    const double xx = GLM_MUL(a, a);
    double p = GLM_FMA(xx, GLM_C(s5), GLM_C(s4));
    p = GLM_FMA(xx, p, GLM_C(s3));
    p = GLM_FMA(xx, p, GLM_C(s2));
    p = GLM_FMA(xx, p, GLM_C(s1));
    const double h = GLM_MUL(da, 0.5);
    const double q = GLM_FMA(p, a, glm_neg(h));
    const double t = GLM_FMA(xx, q, da);
    return GLM_ADD(a, t);
}

/* Table point of |x| < 0.855469: u = big + |x| rounds |x| to a multiple of
 * 1/128; returns the offset x - point and the __sincostab index. */
GLM_FN double glm_table_point(double ax, int* k4) {
    const double u = GLM_ADD(ax, GLM_C(big));
    *k4 = (int)((uint32_t)glm_asuint64(u) << 2);
    return GLM_SUB(ax, GLM_SUB(u, GLM_C(big)));
}

/* do_sin (s_sin.c) for |x| >= 0.126 without the final copysign:
 * sin(ax + dx), ax = |x| and dx already negated for x <= 0. */
GLM_FN double glm_do_sin_core(double ax, double dx) {
    int k;
    const double x = glm_table_point(ax, &k);
    const double xx = GLM_MUL(x, x);
    const double p = GLM_FMA(xx, GLM_C(sn5), GLM_C(sn3));
    const double s = GLM_ADD(x, GLM_FMA(GLM_MUL(x, xx), p, dx));
    const double c = GLM_FMA(x, dx, GLM_MUL(xx, GLM_FMA(xx, GLM_FMA(xx, GLM_C(cs6), GLM_C(cs4)), GLM_C(cs2))));
    const double sn = GLM_LD(glm_sincostab, k), ssn = GLM_LD(glm_sincostab, k + 1);
    const double cs = GLM_LD(glm_sincostab, k + 2), ccs = GLM_LD(glm_sincostab, k + 3);
    /* cor = (ssn + s * ccs - sn * c) + cs * s */
    const double cor = GLM_FMA(s, cs, GLM_FMA(glm_neg(c), sn, GLM_FMA(s, ccs, ssn)));
    return GLM_ADD(sn, cor);
}

/* do_sin (s_sin.c): sin(x + dx). */
GLM_FN double glm_do_sin(double x, double dx) {
    if (glm_fabs(x) < GLM_C(taylor_bound)) return glm_taylor_sin(x, dx);
    if (x <= 0) dx = glm_neg(dx);
    return glm_copysign(glm_do_sin_core(glm_fabs(x), dx), x);
}

/* do_cos (s_sin.c): cos(x + dx). */
GLM_FN double glm_do_cos(double x, double dx) {
    if (x < 0) dx = glm_neg(dx);
    int k;
    const double x0 = GLM_ADD(glm_table_point(glm_fabs(x), &k), dx);
    const double xx = GLM_MUL(x0, x0);
    const double s = GLM_FMA(GLM_MUL(x0, xx), GLM_FMA(xx, GLM_C(sn5), GLM_C(sn3)), x0);
    const double c = GLM_MUL(xx, GLM_FMA(xx, GLM_FMA(xx, GLM_C(cs6), GLM_C(cs4)), GLM_C(cs2)));
    const double sn = GLM_LD(glm_sincostab, k), ssn = GLM_LD(glm_sincostab, k + 1);
    const double cs = GLM_LD(glm_sincostab, k + 2), ccs = GLM_LD(glm_sincostab, k + 3);
    /* cor = (ccs - s * ssn - cs * c) - sn * s */
    const double cor = GLM_FMA(glm_neg(s), sn, GLM_FMA(glm_neg(c), cs, GLM_FMA(glm_neg(s), ssn, ccs)));
    return GLM_ADD(cs, cor);
}

/* reduce_sincos (s_sin.c): x = n pi/2 + (a + da), |x| < 105414350. */
GLM_FN int glm_reduce_sincos(double x, double* a, double* da) {
    const double t = GLM_FMA(x, GLM_C(hpinv), GLM_C(toint));
    const double xn = GLM_SUB(t, GLM_C(toint));
    const int n = (int)(glm_asuint64(t) & 3u);
    const double nxn = glm_neg(xn);
    double y = GLM_FMA(nxn, GLM_C(mp1), x);
    y = GLM_FMA(nxn, GLM_C(mp2), y);
    const double t2 = GLM_FMA(nxn, GLM_C(pp3), y);
    double db = GLM_FMA(nxn, GLM_C(pp3), GLM_SUB(y, t2));
    const double b = GLM_FMA(nxn, GLM_C(pp4), t2);
    db = GLM_ADD(db, GLM_FMA(nxn, GLM_C(pp4), GLM_SUB(t2, b)));
    *a = b;
    *da = db;
    return n;
}

/* do_sincos (s_sin.c): sin(a + da + n pi/2). */
GLM_FN double glm_do_sincos(double a, double da, int n) {
    const double r = (n & 1) ? glm_do_cos(a, da) : glm_do_sin(a, da);
    return (n & 2) ? glm_neg(r) : r;
}

/* Whether glm_cos / glm_sincos restate glibc for x (|x| < 105414350, or
 * inf / NaN); beyond that glibc reduces with __branred, not restated. */
GLM_FN int glm_trig_in_range(double x) {
    const uint32_t k = (uint32_t)(glm_asuint64(x) >> 32) & 0x7fffffffu;
    return k < 0x419921fbu || k >= 0x7ff00000u;
}

/* __cos (s_sin.c). */
GLM_FN double glm_cos(double x) {
    const uint32_t k = (uint32_t)(glm_asuint64(x) >> 32) & 0x7fffffffu;
    if (k < 0x3e400000u) return 1.0;                     /* |x| < 2^-27 */
    if (k < 0x3feb6000u) return glm_do_cos(x, 0.0);      /* |x| < 0.855469 */
    if (k < 0x400368fdu) {                               /* |x| < 2.426265 */
        const double y = GLM_SUB(GLM_C(hp0), glm_fabs(x));
        const double a = GLM_ADD(y, GLM_C(hp1));
        const double da = GLM_ADD(GLM_SUB(y, a), GLM_C(hp1));
        return glm_do_sin(a, da);
    }
    if (k < 0x419921fbu) {                               /* |x| < 105414350 */
        double a, da;
        const int n = glm_reduce_sincos(x, &a, &da);
        return glm_do_sincos(a, da, n + 1);
    }
    return x / x; /* inf / NaN -> NaN (the __branred range is not restated: glm_trig_in_range) */
}

/* __sincos (s_sincos.c). */
GLM_FN void glm_sincos(double x, double* sinx, double* cosx) {
    const uint32_t k = (uint32_t)(glm_asuint64(x) >> 32) & 0x7fffffffu;
    if (k < 0x400368fdu) {
        if (k < 0x3e400000u) { /* |x| < 2^-27 */
            *sinx = x;
            *cosx = 1.0;
            return;
        }
        if (k < 0x3feb6000u) { /* |x| < 0.855469 */
            *sinx = glm_do_sin(x, 0.0);
            *cosx = glm_do_cos(x, 0.0);
            return;
        }
        const double y = GLM_SUB(GLM_C(hp0), glm_fabs(x));
        const double a = GLM_ADD(y, GLM_C(hp1));
        const double da = GLM_ADD(GLM_SUB(y, a), GLM_C(hp1));
        *sinx = glm_copysign(glm_do_cos(a, da), x);
        *cosx = glm_do_sin(a, da);
        return;
    }
    if (k < 0x419921fbu) {
        double a, da;
        const int n = glm_reduce_sincos(x, &a, &da);
        *sinx = glm_do_sincos(a, da, n);
        *cosx = glm_do_sincos(a, da, n + 1);
        return;
    }
    *sinx = *cosx = x / x; /* inf / NaN -> NaN (the __branred range is not restated: glm_trig_in_range) */
}

/* ---------------------------------------------------------------- e_pow.c */

#define GLM_POW_OFF 0x3fe6955500000000ull

/* log_inline (e_pow.c, __FP_FAST_FMA form): log(x) = hi + *tail. */
GLM_FN double glm_log_inline(uint64_t ix, double* tail) {
    const uint64_t tmp = ix - GLM_POW_OFF;
    const int i = (int)((tmp >> 45) % 128u);
    const int k = (int)((int64_t)tmp >> 52);
    const uint64_t iz = ix - (tmp & (0xfffull << 52));
    const double z = glm_asdouble(iz);
    const double kd = (double)k;
    const double invc = GLM_LD(glm_pow_tab, 4 * i), logc = GLM_LD(glm_pow_tab, 4 * i + 2);
    const double logctail = GLM_LD(glm_pow_tab, 4 * i + 3);
    const double r = GLM_FMA(z, invc, -1.0);
    const double t1 = GLM_FMA(kd, GLM_C(ln2hi), logc);
    const double t2 = GLM_ADD(r, t1);
    const double lo1 = GLM_FMA(kd, GLM_C(ln2lo), logctail);
    const double lo2 = GLM_ADD(GLM_SUB(t1, t2), r);
    const double ar = GLM_MUL(r, GLM_LD(glm_pow_poly, 0)); /* A[0] = -0.5 */
    const double ar2 = GLM_MUL(r, ar);
    const double ar3 = GLM_MUL(r, ar2);
    const double hi = GLM_ADD(t2, ar2);
    const double lo3 = GLM_FMA(ar, r, glm_neg(ar2));
    const double lo4 = GLM_ADD(GLM_SUB(t2, hi), ar2);
    /* p = ar3 (A1 + r A2 + ar2 (A3 + r A4 + ar2 (A5 + r A6))) */
    const double q56 = GLM_FMA(r, GLM_LD(glm_pow_poly, 6), GLM_LD(glm_pow_poly, 5));
    const double q34 = GLM_FMA(r, GLM_LD(glm_pow_poly, 4), GLM_LD(glm_pow_poly, 3));
    const double q12 = GLM_FMA(r, GLM_LD(glm_pow_poly, 2), GLM_LD(glm_pow_poly, 1));
    const double q = GLM_FMA(ar2, GLM_FMA(q56, ar2, q34), q12);
    /* lo = lo1 + lo2 + lo3 + lo4 + p, the last add fused with p's product */
    const double lo = GLM_FMA(ar3, q, GLM_ADD(GLM_ADD(GLM_ADD(lo1, lo2), lo3), lo4));
    const double y = GLM_ADD(hi, lo);
    *tail = GLM_ADD(GLM_SUB(hi, y), lo);
    return y;
}

/* specialcase (e_pow.c): scale (1 + tmp) near overflow / underflow. */
GLM_FN double glm_exp_specialcase(double tmp, uint64_t sbits, uint64_t ki) {
    if ((ki & 0x80000000u) == 0) {
        sbits -= 1009ull << 52;
        const double scale = glm_asdouble(sbits);
        return GLM_MUL(GLM_FMA(scale, tmp, scale), glm_asdouble(0x7f00000000000000ull)); /* 2^1009 */
    }
    sbits += 1022ull << 52;
    const double scale = glm_asdouble(sbits);
    const double st = GLM_MUL(tmp, scale);
    double y = GLM_ADD(scale, st);
    if (glm_fabs(y) < 1.0) {
        const double one = (y < 0.0) ? -1.0 : 1.0;
        double lo = GLM_ADD(GLM_SUB(scale, y), st);
        const double hi = GLM_ADD(one, y);
        lo = GLM_ADD(GLM_ADD(GLM_SUB(one, hi), y), lo);
        y = GLM_SUB(GLM_ADD(hi, lo), one);
        if (y == 0) y = glm_asdouble(sbits & 0x8000000000000000ull);
    }
    return GLM_MUL(y, glm_asdouble(0x0010000000000000ull)); /* 2^-1022 */
}

/* exp_inline (e_pow.c): sign * exp(x + xtail). */
GLM_FN double glm_exp_inline(double x, double xtail, uint64_t sign_bias) {
    uint32_t abstop = (uint32_t)(glm_asuint64(x) >> 52) & 0x7ffu;
    if (abstop - 0x3c9u >= 0x408u - 0x3c9u) {
        if ((int32_t)(abstop - 0x3c9u) < 0) { /* tiny x: 1 + x */
            const double one = GLM_ADD(x, 1.0);
            return sign_bias ? glm_neg(one) : one;
        }
        if (abstop >= 0x409u) { /* overflow / underflow */
            const double big = (glm_asuint64(x) >> 63) ? 0.0 : glm_asdouble(0x7ff0000000000000ull);
            return sign_bias ? glm_neg(big) : big;
        }
        abstop = 0; /* large x: specialcase below */
    }
    const double kd0 = GLM_FMA(x, GLM_C(invln2N), GLM_C(shift));
    const uint64_t ki = glm_asuint64(kd0);
    const double kd = GLM_SUB(kd0, GLM_C(shift));
    double r = GLM_FMA(kd, GLM_C(negln2loN), GLM_FMA(kd, GLM_C(negln2hiN), x));
    r = GLM_ADD(xtail, r);
    const uint64_t idx = 2 * (ki % 128u);
    const uint64_t top = (ki + sign_bias) << 45;
    const double tail = GLM_LD(glm_exp_tab, idx);
    const uint64_t sbits = glm_exp_tab[idx + 1] + top;
    const double r2 = GLM_MUL(r, r);
    /* tmp = tail + r + r2 (C2 + r C3) + r2 r2 (C4 + r C5) */
    const double p23 = GLM_FMA(r, GLM_C(C3), GLM_C(C2));
    const double p45 = GLM_FMA(r, GLM_C(C5), GLM_C(C4));
    const double tmp = GLM_FMA(p45, GLM_MUL(r2, r2), GLM_FMA(p23, r2, GLM_ADD(r, tail)));
    if (abstop == 0) return glm_exp_specialcase(tmp, sbits, ki);
    const double scale = glm_asdouble(sbits);
    return GLM_FMA(tmp, scale, scale);
}

/* checkint (e_pow.c): 0 not an integer, 1 odd integer, 2 even integer. */
GLM_FN int glm_checkint(uint64_t iy) {
    const int e = (int)(iy >> 52 & 0x7ff);
    if (e < 0x3ff) return 0;
    if (e > 0x3ff + 52) return 2;
    if (iy & ((1ull << (0x3ff + 52 - e)) - 1)) return 0;
    if (iy & (1ull << (0x3ff + 52 - e))) return 1;
    return 2;
}

GLM_FN int glm_zeroinfnan(uint64_t i) { return 2 * i - 1 >= 2 * 0x7ff0000000000000ull - 1; }
GLM_FN int glm_issignaling(uint64_t i) { return 2 * (i ^ 0x0008000000000000ull) > 2 * 0x7ff8000000000000ull; }

/* __pow (e_pow.c). */
GLM_FN double glm_pow(double x, double y) {
    uint64_t sign_bias = 0;
    uint64_t ix = glm_asuint64(x), iy = glm_asuint64(y);
    uint32_t topx = (uint32_t)(ix >> 52), topy = (uint32_t)(iy >> 52);
    if (topx - 0x001u >= 0x7ffu - 0x001u || (topy & 0x7ffu) - 0x3beu >= 0x43eu - 0x3beu) {
        if (glm_zeroinfnan(iy)) {
            if (2 * iy == 0) return glm_issignaling(ix) ? GLM_ADD(x, y) : 1.0;
            if (ix == glm_asuint64(1.0)) return glm_issignaling(iy) ? GLM_ADD(x, y) : 1.0;
            if (2 * ix > 2 * 0x7ff0000000000000ull || 2 * iy > 2 * 0x7ff0000000000000ull)
                return GLM_ADD(x, y);
            if (2 * ix == 2 * glm_asuint64(1.0)) return 1.0;
            if ((2 * ix < 2 * glm_asuint64(1.0)) == !(iy >> 63)) return 0.0;
            return GLM_MUL(y, y);
        }
        if (glm_zeroinfnan(ix)) {
            double x2 = GLM_MUL(x, x);
            if ((ix >> 63) && glm_checkint(iy) == 1) x2 = glm_neg(x2);
            return (iy >> 63) ? 1.0 / x2 : x2;
        }
        if (ix >> 63) { /* finite x < 0 */
            const int yint = glm_checkint(iy);
            if (yint == 0) return (x - x) / (x - x);
            if (yint == 1) sign_bias = 0x800ull << 7;
            ix &= 0x7fffffffffffffffull;
            topx &= 0x7ffu;
        }
        if ((topy & 0x7ffu) - 0x3beu >= 0x43eu - 0x3beu) {
            if (ix == glm_asuint64(1.0)) return 1.0;
            if ((topy & 0x7ffu) < 0x3beu) return ix > glm_asuint64(1.0) ? GLM_ADD(1.0, y) : GLM_SUB(1.0, y);
            return (ix > glm_asuint64(1.0)) == (topy < 0x800u) ? glm_asdouble(0x7ff0000000000000ull) : 0.0;
        }
        if (topx == 0) { /* subnormal x: normalise */
            ix = glm_asuint64(GLM_MUL(x, 4503599627370496.0)); /* x * 2^52 */
            ix &= 0x7fffffffffffffffull;
            ix -= 52ull << 52;
        }
    }
    double lo;
    const double hi = glm_log_inline(ix, &lo);
    const double ehi = GLM_MUL(y, hi);
    const double elo = GLM_FMA(y, lo, GLM_FMA(hi, y, glm_neg(ehi)));
    return glm_exp_inline(ehi, elo, sign_bias);
}

#endif /* ODEGPU_DEVICE_GLIBM_H */
