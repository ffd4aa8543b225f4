// vr_common.cuh -- device helpers shared by the sm_100a kernels.
//
// Parity mode: every translation unit that includes this file is compiled
// with -fmad=false, so each float64 multiply and add below rounds separately,
// in the same association as the reference's numba kernels
// (/root/reference/pkg/src/voxelray/_kernels.py), which the survey checked
// carry no FMA contraction.  Division and sqrt are IEEE correctly rounded on
// the device (nvcc default -prec-div=true -prec-sqrt=true for double).
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

#define VR_HD __host__ __device__ __forceinline__
#define VR_D __device__ __forceinline__

namespace vr {

VR_HD double clampf(double v, double lo, double hi) {
    if (v < lo) return lo;
    if (v > hi) return hi;
    return v;
}

VR_HD int clampi(int v, int lo, int hi) {
    if (v < lo) return lo;
    if (v > hi) return hi;
    return v;
}

// Python's max(a, 0.0)
VR_HD double pymax0(double a) { return (0.0 > a) ? 0.0 : a; }

// Exact int16 -> float64 (the reference promotes taps with 1.0 * data[p]).
VR_D double tap(const int16_t *p) { return (double)__ldg(p); }
VR_D double tap(const uint8_t *p) { return (double)__ldg(p); }

// ---------------------------------------------------------------- divide
// x / s where s is a positive constant.  When s is a power of two, x * (1/s)
// is bit-identical to x / s (no subnormals in range), and avoids the DDIV
// sequence; otherwise fall back to the correctly rounded division.
struct Divisor {
    double s;
    double inv;
    int pow2;
};

inline Divisor make_divisor(double s) {
    Divisor d;
    d.s = s;
    d.inv = 1.0 / s;
    int e = 0;
    double m = frexp(s, &e);
    d.pow2 = (m == 0.5) ? 1 : 0;
    return d;
}

VR_D double divide(double x, const Divisor &d) { return d.pow2 ? x * d.inv : x / d.s; }

// floor((x - 1) / stride) clamped to [0, nb-1], as the reference's block
// attribution does (_kernels.py:226-228, 372-374).  The quotient is first
// estimated with a reciprocal multiply; only when that estimate sits within
// 1e-9 of an integer (where the correctly rounded quotient could round across
// it) is the exact division evaluated.
VR_D int owner_block(double x, double stride, double inv_stride, int nb) {
    if (nb == 1) return 0;
    double a = x - 1.0;
    double q = a * inv_stride;
    double f = floor(q);
    double fr = q - f;
    if (fr < 1e-9 || fr > 1.0 - 1e-9) f = floor(a / stride);
    // clamp in the float domain first so huge values cannot overflow the int
    if (f < 0.0) return 0;
    if (f > (double)(nb - 1)) return nb - 1;
    return (int)f;
}

// ----------------------------------------------------------- Catmull-Rom
// _kernels.py:83-91
VR_D void cr_weights(double t, double &w0, double &w1, double &w2, double &w3) {
    double t2 = t * t;
    double t3 = t2 * t;
    w0 = 0.5 * ((-t3 + 2.0 * t2) - t);
    w1 = 0.5 * ((3.0 * t3 - 5.0 * t2) + 2.0);
    w2 = 0.5 * ((-3.0 * t3 + 4.0 * t2) + t);
    w3 = 0.5 * (t3 - t2);
}

// A block of the volume seen through the reference's atlas addressing: local
// coordinates in [0, e), voxels at base[(k*py) + (j*px) + i] with the global
// pitches (the atlas copy of a block holds the same voxels, blocks.py:269-294).
template <class T>
struct Brick {
    const T *base;
    long long pz, py;  // plane and row pitch in elements
    int ex, ey, ez;    // block extents
};

// _kernels.py:52-80
template <class T>
VR_D double tri_sample(const Brick<T> &b, double x, double y, double z) {
    x = clampf(x, 0.0, b.ex - 1.0);
    y = clampf(y, 0.0, b.ey - 1.0);
    z = clampf(z, 0.0, b.ez - 1.0);
    int i0 = clampi((int)x, 0, b.ex - 2);
    int j0 = clampi((int)y, 0, b.ey - 2);
    int k0 = clampi((int)z, 0, b.ez - 2);
    double fx = x - (double)i0;
    double fy = y - (double)j0;
    double fz = z - (double)k0;
    const T *p = b.base + (long long)k0 * b.pz + (long long)j0 * b.py + i0;
    const T *q = p + b.pz;
    double v000 = tap(p), v100 = tap(p + 1), v010 = tap(p + b.py), v110 = tap(p + b.py + 1);
    double v001 = tap(q), v101 = tap(q + 1), v011 = tap(q + b.py), v111 = tap(q + b.py + 1);
    double c00 = v000 + (v100 - v000) * fx;
    double c10 = v010 + (v110 - v010) * fx;
    double c01 = v001 + (v101 - v001) * fx;
    double c11 = v011 + (v111 - v011) * fx;
    double c0 = c00 + (c10 - c00) * fy;
    double c1 = c01 + (c11 - c01) * fy;
    return c0 + (c1 - c0) * fz;
}

// _kernels.py:94-143: taps clamped to the block, rows summed x -> y -> z.
template <class T>
VR_D double cub_sample(const Brick<T> &b, double x, double y, double z) {
    x = clampf(x, 0.0, b.ex - 1.0);
    y = clampf(y, 0.0, b.ey - 1.0);
    z = clampf(z, 0.0, b.ez - 1.0);
    int i0 = clampi((int)x, 0, b.ex - 1);
    int j0 = clampi((int)y, 0, b.ey - 1);
    int k0 = clampi((int)z, 0, b.ez - 1);
    double wx0, wx1, wx2, wx3, wy0, wy1, wy2, wy3, wz0, wz1, wz2, wz3;
    cr_weights(x - (double)i0, wx0, wx1, wx2, wx3);
    cr_weights(y - (double)j0, wy0, wy1, wy2, wy3);
    cr_weights(z - (double)k0, wz0, wz1, wz2, wz3);
    int ia = max(i0 - 1, 0), ic = min(i0 + 1, b.ex - 1), id = min(i0 + 2, b.ex - 1);
    long long ja = (long long)max(j0 - 1, 0) * b.py, jb = (long long)j0 * b.py;
    long long jc = (long long)min(j0 + 1, b.ey - 1) * b.py, jd = (long long)min(j0 + 2, b.ey - 1) * b.py;
    long long kz[4] = {(long long)max(k0 - 1, 0) * b.pz, (long long)k0 * b.pz,
                       (long long)min(k0 + 1, b.ez - 1) * b.pz,
                       (long long)min(k0 + 2, b.ez - 1) * b.pz};
    double pl[4];
#pragma unroll
    for (int c = 0; c < 4; ++c) {
        const T *pb = b.base + kz[c];
        const T *r0 = pb + ja, *r1 = pb + jb, *r2 = pb + jc, *r3 = pb + jd;
        double s0 = ((wx0 * tap(r0 + ia) + wx1 * tap(r0 + i0)) + wx2 * tap(r0 + ic)) + wx3 * tap(r0 + id);
        double s1 = ((wx0 * tap(r1 + ia) + wx1 * tap(r1 + i0)) + wx2 * tap(r1 + ic)) + wx3 * tap(r1 + id);
        double s2 = ((wx0 * tap(r2 + ia) + wx1 * tap(r2 + i0)) + wx2 * tap(r2 + ic)) + wx3 * tap(r2 + id);
        double s3 = ((wx0 * tap(r3 + ia) + wx1 * tap(r3 + i0)) + wx2 * tap(r3 + ic)) + wx3 * tap(r3 + id);
        pl[c] = ((wy0 * s0 + wy1 * s1) + wy2 * s2) + wy3 * s3;
    }
    return ((wz0 * pl[0] + wz1 * pl[1]) + wz2 * pl[2]) + wz3 * pl[3];
}

template <class T>
VR_D double sample(const Brick<T> &b, double x, double y, double z, bool cubic) {
    return cubic ? cub_sample(b, x, y, z) : tri_sample(b, x, y, z);
}

// ------------------------------------------------------------ block layout
// blocks.py:100-107: origins i*stride, extents min(B, n - origin).
struct Layout {
    int n[3];       // nx, ny, nz
    int nb[3];      // blocks per axis
    int bsize;      // block_size (max(n) for the monolithic single block)
    int stride;     // block_size - overlap (max(n) for monolithic)
    double strided; // (double)stride
    double inv_stride;
    long long py, pz;  // global pitches
};

VR_HD int block_origin(const Layout &L, int b) { return b * L.stride; }
VR_HD int block_extent(const Layout &L, int a, int b) {
    int e = L.n[a] - b * L.stride;
    return e < L.bsize ? e : L.bsize;
}

// ---------------------------------------------------------- exact powers
// Error-free double-double product (fma is exact; the explicit call is not
// affected by -fmad=false).
VR_D void two_prod(double a, double b, double &p, double &e) {
    p = a * b;
    e = fma(a, b, -p);
}

VR_D void two_sum(double a, double b, double &s, double &e) {
    s = a + b;
    double bb = s - a;
    e = (a - (s - bb)) + (b - bb);
}

// x^n for a non-negative integer n in double-double (about 100 significant
// bits), rounded once: agrees with a correctly rounded pow (glibc's pow, used
// by the reference's `**`) except in cases closer to a rounding midpoint
// than ~2^-95 relative.
VR_D double pow_int_dd(double x, int n) {
    double rh = 1.0, rl = 0.0;
    double bh = x, bl = 0.0;
    while (n > 0) {
        if (n & 1) {
            double p, e;
            two_prod(rh, bh, p, e);
            e += rh * bl + rl * bh;
            two_sum(p, e, rh, rl);
        }
        n >>= 1;
        if (n) {
            double p, e;
            two_prod(bh, bh, p, e);
            e += 2.0 * bh * bl;
            two_sum(p, e, bh, bl);
        }
    }
    return rh + rl;
}

// pow(x, y) for the two exponents the reference raises at run time:
// the opacity correction (1 - a)^(step/ref_step) (_kernels.py:489,519) and
// the Phong exponent (_kernels.py:204,569).  Integer exponents use the
// double-double ladder, y == 0.5 is sqrt (correctly rounded, as is a
// correctly rounded pow), anything else the CUDA pow (<= 2 ulp).
struct PowSpec {
    int kind;  // 0 identity (y == 1), 1 integer, 2 sqrt, 3 general
    int n;
    double y;
};

inline PowSpec make_pow(double y) {
    PowSpec p;
    p.y = y;
    p.n = 0;
    if (y == 1.0) {
        p.kind = 0;
    } else if (y >= 0.0 && y <= 4096.0 && y == (double)(int)y) {
        p.kind = 1;
        p.n = (int)y;
    } else if (y == 0.5) {
        p.kind = 2;
    } else {
        p.kind = 3;
    }
    return p;
}

VR_D double vr_pow(double x, const PowSpec &p) {
    switch (p.kind) {
        case 0: return x;
        case 1: return (x == 0.0 && p.n == 0) ? 1.0 : pow_int_dd(x, p.n);
        case 2: return sqrt(x);
        default: return pow(x, p.y);
    }
}

}  // namespace vr
