// vr_glibc_pow.h -- glibc's pow, restated for the device (and the host check).
//
// The reference raises floats with numba's `**` (_kernels.py:204 the Phong
// power, :489/:519 the opacity correction (1 - a)^(step/ref_step), :569 the
// pre-integrated specular), which numba lowers to libm's pow.  glibc 2.39's
// pow (the ARM optimized-routines algorithm, sysdeps/ieee754/dbl-64/e_pow.c;
// on x86-64 CPUs with FMA the ifunc picks its FMA build) is accurate to <= 0.52
// ulp but not correctly rounded: 0.09 % of pow(x, 32) on x in [0, 1] differ
// from the correctly rounded power.  To reproduce the reference bit for bit,
// the kernels run the same algorithm on the same tables (vr_pow_tables.h,
// extracted from libm by tools/gen_pow_tables.py, which also checks this file
// against libm's pow on 2e7 random inputs):
//
//   log(x) = k ln2 + log(c) + log1p(z/c - 1) in double-double (128-entry table
//   of 1/c, log c), y * log(x) split exactly with an FMA, then
//   exp(hi + lo) = 2^(k/128) * exp(r) with a 256-entry table and a degree-5
//   polynomial, the tail rounded once.
//
// Every operation below is one IEEE operation in the C source's order.  The
// FMA build of glibc is compiled with GCC's default contraction, which fuses
// every product whose only uses are additions in the same basic block into
// them; those fusions are
// written out here as fma() calls (this file itself is compiled without
// contraction: -fmad=false / -ffp-contract=off).  Special cases cover what the kernels can pass: x in
// [0, +inf), y finite (zero, subnormal and huge y included).
#pragma once

#include <stdint.h>
#include <string.h>

#ifdef __CUDACC__
#define VR_POW_FN __host__ __device__ __forceinline__
#define VR_POW_TABLE static __device__ const
#else
#define VR_POW_FN static inline
#define VR_POW_TABLE static const
#endif

#include "vr_pow_tables.h"

VR_POW_FN uint64_t vr_asu64(double x) {
#ifdef __CUDA_ARCH__
    return (uint64_t)__double_as_longlong(x);
#else
    uint64_t u;
    memcpy(&u, &x, 8);
    return u;
#endif
}

VR_POW_FN double vr_asf64(uint64_t u) {
#ifdef __CUDA_ARCH__
    return __longlong_as_double((long long)u);
#else
    double x;
    memcpy(&x, &u, 8);
    return x;
#endif
}

VR_POW_FN double vr_pow_log_entry(int i, int j) {
#ifdef __CUDA_ARCH__
    return __ldg(&vr_pow_log_tab[i][j]);
#else
    return vr_pow_log_tab[i][j];
#endif
}

VR_POW_FN uint64_t vr_exp_entry(int i) {
#ifdef __CUDA_ARCH__
    return __ldg(&vr_exp_tab[i]);
#else
    return vr_exp_tab[i];
#endif
}

// e_pow.c log_inline (FMA build): log(x) as hi + *tail
VR_POW_FN double vr_pow_log_inline(uint64_t ix, double *tail) {
    const uint64_t OFF = 0x3fe6955500000000ull;
    const uint64_t tmp = ix - OFF;
    const int i = (int)((tmp >> (52 - 7)) % 128);
    const int k = (int)((int64_t)tmp >> 52);
    const uint64_t iz = ix - (tmp & (0xfffull << 52));
    const double z = vr_asf64(iz);
    const double kd = (double)k;
    const double invc = vr_pow_log_entry(i, 0);
    const double logc = vr_pow_log_entry(i, 1);
    const double logctail = vr_pow_log_entry(i, 2);
    // 1/c is j/128 or j/256 with |z/c - 1| < 1/128: r is exact with the FMA
    const double r = fma(z, invc, -1.0);
    const double t1 = fma(kd, VR_POW_LN2HI, logc);
    const double t2 = t1 + r;
    const double lo1 = fma(kd, VR_POW_LN2LO, logctail);
    const double lo2 = t1 - t2 + r;
    const double ar = VR_POW_A0 * r;
    const double ar2 = r * ar;
    const double ar3 = r * ar2;
    const double hi = t2 + ar2;
    const double lo3 = fma(ar, r, -ar2);
    const double lo4 = t2 - hi + ar2;
    const double q = fma(ar2, fma(ar2, fma(r, VR_POW_A6, VR_POW_A5), fma(r, VR_POW_A4, VR_POW_A3)),
                         fma(r, VR_POW_A2, VR_POW_A1));
    const double lo = fma(ar3, q, ((lo1 + lo2) + lo3) + lo4);  // ... + p, p = ar3 * q
    const double y = hi + lo;
    *tail = hi - y + lo;
    return y;
}

// e_exp.c / e_pow.c specialcase: results whose scale left the normal range
VR_POW_FN double vr_pow_specialcase(double tmp, uint64_t sbits, uint64_t ki) {
    if ((ki & 0x80000000ull) == 0) {
        // k > 0: the exponent of scale may have overflowed by <= 460
        sbits -= 1009ull << 52;
        const double scale = vr_asf64(sbits);
        return 0x1p1009 * fma(scale, tmp, scale);
    }
    // k < 0: careful rounding in the subnormal range
    sbits += 1022ull << 52;
    const double scale = vr_asf64(sbits);
    // scale * tmp is also used inside the branch below (another basic block),
    // so GCC does not fuse it here: plain multiply and add
    const double st = scale * tmp;
    double y = scale + st;
    if (fabs(y) < 1.0) {
        const double one = y < 0.0 ? -1.0 : 1.0;
        double lo = scale - y + st;
        const double hi = one + y;
        lo = one - hi + y + lo;
        y = (hi + lo) - one;
        if (y == 0) y = vr_asf64(sbits & 0x8000000000000000ull);
    }
    return 0x1p-1022 * y;
}

// e_pow.c exp_inline: exp(x + xtail) (sign_bias 0: x >= 0 here)
VR_POW_FN double vr_pow_exp_inline(double x, double xtail) {
    uint32_t abstop = (uint32_t)(vr_asu64(x) >> 52) & 0x7ff;
    const uint32_t top_tiny = 0x3c9;  // top12(0x1p-54)
    const uint32_t top_512 = 0x408;   // top12(512.0)
    if (abstop - top_tiny >= top_512 - top_tiny) {
        if (abstop - top_tiny >= 0x80000000u) return 1.0;  // tiny x: avoid spurious underflow
        if (abstop >= 0x409) {                              // top12(1024.0)
            return (vr_asu64(x) >> 63) ? 0.0 : vr_asf64(0x7ff0000000000000ull);  // underflow / overflow
        }
        abstop = 0;  // large x: special-cased below
    }
    double kd = fma(VR_EXP_INVLN2N, x, VR_EXP_SHIFT);
    const uint64_t ki = vr_asu64(kd);
    kd -= VR_EXP_SHIFT;
    double r = fma(kd, VR_EXP_NEGLN2LON, fma(kd, VR_EXP_NEGLN2HIN, x));
    r += xtail;
    const uint64_t idx = 2 * (ki % 128);
    const uint64_t top = ki << (52 - 7);
    const double tail = vr_asf64(vr_exp_entry((int)idx));
    const uint64_t sbits = vr_exp_entry((int)idx + 1) + top;
    const double r2 = r * r;
    const double tmp = fma(r2 * r2, fma(r, VR_EXP_C5, VR_EXP_C4), fma(r2, fma(r, VR_EXP_C3, VR_EXP_C2), tail + r));
    if (abstop == 0) return vr_pow_specialcase(tmp, sbits, ki);
    const double scale = vr_asf64(sbits);
    return fma(scale, tmp, scale);
}

// pow(x, y) for x >= 0 (or +inf) and finite y, bit-identical to glibc 2.39's
VR_POW_FN double vr_glibc_pow(double x, double y) {
    uint64_t ix = vr_asu64(x);
    const uint64_t iy = vr_asu64(y);
    const uint32_t topx = (uint32_t)(ix >> 52);
    const uint32_t topy = (uint32_t)(iy >> 52);
    if (topx - 0x001 >= 0x7ff - 0x001 || (topy & 0x7ff) - 0x3be >= 0x43e - 0x3be) {
        // zero / subnormal / inf x, or |y| tiny or huge
        const int y_zero = 2 * iy == 0;
        if (y_zero) return 1.0;
        if (ix == 0x3ff0000000000000ull) return 1.0;
        if (2 * ix - 1 >= 2 * 0x7ff0000000000000ull - 1) {  // x == 0 or inf (zeroinfnan)
            const double x2 = x * x;
            return (iy >> 63) ? 1.0 / x2 : x2;
        }
        if ((topy & 0x7ff) - 0x3be >= 0x43e - 0x3be) {
            if ((topy & 0x7ff) < 0x3be) return ix > 0x3ff0000000000000ull ? 1.0 + y : 1.0 - y;  // |y| tiny
            const int big = (ix > 0x3ff0000000000000ull) == (topy < 0x800);
            return big ? vr_asf64(0x7ff0000000000000ull) : 0.0;
        }
        if (topx == 0) {  // subnormal x: normalise so the exponent becomes negative
            ix = vr_asu64(x * 0x1p52);
            ix &= 0x7fffffffffffffffull;
            ix -= 52ull << 52;
        }
    }
    double lo;
    const double hi = vr_pow_log_inline(ix, &lo);
    const double ehi = y * hi;
    const double elo = fma(y, lo, fma(y, hi, -ehi));
    return vr_pow_exp_inline(ehi, elo);
}
