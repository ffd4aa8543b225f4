// vr_common.cuh -- device helpers shared by the sm_100a kernels.
//
// Parity mode: every translation unit that includes this file is compiled
// with -fmad=false, so each float64 multiply and add below rounds separately,
// in the same association as the reference's numba kernels
// (/root/reference/pkg/src/voxelray/_kernels.py), which the survey checked
// carry no FMA contraction.  Division and sqrt are IEEE correctly rounded on
// the device (nvcc default -prec-div=true -prec-sqrt=true for double).
#pragma once
#include <climits>

#include <cstdint>
#include <cstdlib>
#include <utility>
#include <cuda_runtime.h>

#include "vr_glibc_pow.h"

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

// Programmatic dependent launch between the frame's kernels (visibility
// setup -> ray casters -> hit count).  Each such kernel starts with
// pdl_enter(): it waits for its predecessor grid to complete (and its writes
// to be visible) before touching memory, then lets its own successor launch,
// so the successor's launch and CTA rasterisation overlap this kernel instead
// of following it.  The data dependences are those of plain stream order.
VR_D void pdl_enter() {
    asm volatile("griddepcontrol.wait;" ::: "memory");
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

// Launch with the programmatic-serialisation attribute (build with
// -DVR_NO_PDL for plain stream order, A/B).  Only kernels that begin with
// pdl_enter() may be launched this way.
#ifdef VR_NO_PDL
constexpr int kPdl = 0;
#else
constexpr int kPdl = 1;
#endif
template <typename... P, typename... A>
cudaError_t launch_pdl(void (*k)(P...), dim3 grid, dim3 block, size_t smem, cudaStream_t s, A &&...args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = kPdl;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, k, std::forward<A>(args)...);
}

// SM count of the current device, queried once per device (grids of the
// persistent and grid-stride kernels are sized from it).
int device_sms();

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

// Rare paths live out of line so the hot loops stay within the instruction
// cache (an inlined IEEE double division is ~20 instructions plus a slow
// path, and the kernels call these from many sites).
static __device__ __noinline__ double div_rn(double x, double s) { return x / s; }
static __device__ __noinline__ double floor_div(double a, double s) { return floor(a / s); }

VR_D double divide(double x, const Divisor &d) { return d.pow2 ? x * d.inv : div_rn(x, d.s); }

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
    if (fr < 1e-9 || fr > 1.0 - 1e-9) f = floor_div(a, stride);
    // clamp in the float domain first so huge values cannot overflow the int
    if (f < 0.0) return 0;
    if (f > (double)(nb - 1)) return nb - 1;
    return (int)f;
}

// _kernels.py:190-192 _lut_bin
VR_D int lut_bin(double s, double lo, double inv_w, int nbins) {
    double q = (s - lo) * inv_w;
    // int() truncates toward zero; clamp in the float domain to stay in range
    if (q <= -1.0) return 0;
    if (q >= (double)nbins) return nbins - 1;
    return clampi((int)q, 0, nbins - 1);
}

// Integer value thresholds of the LUT's visible bin range: every integer s
// with s < vlo has lut_bin(s) < first_vis and every s > vhi has lut_bin(s) >
// last_vis (lut_bin is monotone), so an integer bound can be tested without
// floating point.  vlo = INT_MAX / vhi = INT_MIN when no bin is visible.
VR_D void visible_value_range(double lo, double inv_w, int nbins, int first_vis, int last_vis, int &vlo,
                              int &vhi) {
    const int L = -(1 << 24), R = 1 << 24;
    if (first_vis >= nbins || last_vis < 0) {
        vlo = INT_MAX;
        vhi = INT_MIN;
        return;
    }
    int a = L, b = R;  // smallest s in [L, R] with lut_bin(s) >= first_vis (R when none... bin(R) = nbins-1)
    while (a < b) {
        const int m = a + (b - a) / 2;
        if (lut_bin((double)m, lo, inv_w, nbins) >= first_vis) b = m; else a = m + 1;
    }
    vlo = a;
    a = L;
    b = R;  // largest s with lut_bin(s) <= last_vis
    while (a < b) {
        const int m = a + (b - a + 1) / 2;
        if (lut_bin((double)m, lo, inv_w, nbins) <= last_vis) a = m; else b = m - 1;
    }
    vhi = a;
}

// The same thresholds with every thread of a T-thread CTA (all must call it; the
// results are in vlo / vhi on return in every thread).  lut_bin is
// nondecreasing in s, so each threshold is the first s of a false->true
// predicate: a T-ary search (T = 1024: 3 rounds over [-2^24, 2^24 + 1]) instead of
// the 2 x 25 dependent bisection steps of one thread.
//   vlo = first s in [L, R] with lut_bin(s) >= first_vis (R when none)
//   vhi = (first s in [L+1, R+1] with lut_bin(s) > last_vis) - 1 (R when none)
// which is exactly what the bisections above return.
template <int T>
VR_D void block_value_range(double lo, double inv_w, int nbins, int first_vis, int last_vis, int &vlo, int &vhi) {
    __shared__ int lo_a, lo_b, hi_a, hi_b, lo_t, hi_t;
    const int L = -(1 << 24), R = 1 << 24;
    const int tid = (int)threadIdx.x;
    const bool none = first_vis >= nbins || last_vis < 0;
    if (tid == 0) {
        lo_a = L;
        lo_b = R;
        hi_a = L + 1;
        hi_b = R + 1;
    }
    __syncthreads();
    for (;;) {
        const int a0 = lo_a, b0 = lo_b, a1 = hi_a, b1 = hi_b;
        if (none || (a0 >= b0 && a1 >= b1)) break;
        const int st0 = (b0 - a0 + T - 1) / T, st1 = (b1 - a1 + T - 1) / T;
        __syncthreads();  // everyone read the interval before it changes
        if (tid == 0) {
            lo_t = T;
            hi_t = T;
        }
        __syncthreads();
        if (a0 < b0) {
            const long long m = (long long)a0 + (long long)tid * st0;
            if (m < b0 && lut_bin((double)m, lo, inv_w, nbins) >= first_vis) atomicMin(&lo_t, tid);
        }
        if (a1 < b1) {
            const long long m = (long long)a1 + (long long)tid * st1;
            if (m < b1 && lut_bin((double)m, lo, inv_w, nbins) > last_vis) atomicMin(&hi_t, tid);
        }
        __syncthreads();
        if (tid == 0) {
            // probes a + t*step (t < T, below b): the first true probe t* bounds
            // the answer to (probe t*-1, probe t*]; none true: (last probe, b]
            if (a0 < b0) {
                const int t = lo_t;
                if (t < T) {
                    lo_b = a0 + t * st0;
                    lo_a = t > 0 ? a0 + (t - 1) * st0 + 1 : a0;
                } else {
                    const int last = (b0 - 1 - a0) / st0;  // last probe below b
                    lo_a = a0 + last * st0 + 1;
                }
            }
            if (a1 < b1) {
                const int t = hi_t;
                if (t < T) {
                    hi_b = a1 + t * st1;
                    hi_a = t > 0 ? a1 + (t - 1) * st1 + 1 : a1;
                } else {
                    const int last = (b1 - 1 - a1) / st1;
                    hi_a = a1 + last * st1 + 1;
                }
            }
        }
        __syncthreads();
    }
    if (none) {
        vlo = INT_MAX;
        vhi = INT_MIN;
    } else {
        vlo = lo_a;
        vhi = hi_a - 1;
    }
    __syncthreads();  // the shared state may be reused by a later call
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

// ------------------------------------------------------------ volume views
// Voxel access by global index (x, y, z).  Three layouts: the x-fastest
// linear volume (ScalarVolume.values order), the same for uint8 planes
// (pre-classified RGBA), and the 4x4x4-brick layout K1 builds for the ray
// caster -- one brick is one 128-byte line, so the 4x4x4 Catmull-Rom
// neighbourhood of a sample touches at most 8 lines, and neighbouring rays of
// a warp share them, whatever the view direction.
struct LinearVol {
    const int16_t *p;
    long long py, pz;
    VR_D const int16_t *at_ptr(int x, int y, int z) const { return p + (long long)z * pz + (long long)y * py + x; }
    VR_D double at(int x, int y, int z) const { return tap(at_ptr(x, y, z)); }
    VR_D void row4(int x, int y, int z, double v[4]) const {
        const int16_t *q = at_ptr(x, y, z);
        v[0] = tap(q);
        v[1] = tap(q + 1);
        v[2] = tap(q + 2);
        v[3] = tap(q + 3);
    }
    VR_D void row2(int x, int y, int z, double v[2]) const {
        const int16_t *q = at_ptr(x, y, z);
        v[0] = tap(q);
        v[1] = tap(q + 1);
    }
};

struct LinearU8 {
    const uint8_t *p;
    long long py, pz;
    VR_D const uint8_t *at_ptr(int x, int y, int z) const { return p + (long long)z * pz + (long long)y * py + x; }
    VR_D double at(int x, int y, int z) const { return tap(at_ptr(x, y, z)); }
    VR_D void row4(int x, int y, int z, double v[4]) const {
        const uint8_t *q = at_ptr(x, y, z);
        v[0] = tap(q);
        v[1] = tap(q + 1);
        v[2] = tap(q + 2);
        v[3] = tap(q + 3);
    }
    VR_D void row2(int x, int y, int z, double v[2]) const {
        const uint8_t *q = at_ptr(x, y, z);
        v[0] = tap(q);
        v[1] = tap(q + 1);
    }
};

// Bounds-checked builds (-DVR_BOUNDS_CHECK, test only: compute-sanitizer is
// closed on this GPU pool): every brick-window load traps when it leaves the
// allocation.
#ifdef VR_BOUNDS_CHECK
#define VR_CHECK_SPAN(base, n, q, len)                                                   \
    do {                                                                                 \
        if ((const void *)(q) < (const void *)(base) ||                                  \
            (const char *)((q) + (len)) > (const char *)((base) + (n))) __trap();         \
    } while (0)
#else
#define VR_CHECK_SPAN(base, n, q, len) ((void)0)
#endif

struct BrickVol {
    const int16_t *p;
    long long bpy, bpz;  // int16 elements per row of bricks / per plane of bricks
    long long n;         // int16 elements of the allocation (bounds-checked builds)
    VR_D const int16_t *row_ptr(int x, int y, int z) const {
        return p + (long long)(z >> 2) * bpz + (long long)(y >> 2) * bpy + ((long long)(x >> 2) << 6) +
               ((z & 3) << 4) + ((y & 3) << 2);
    }
    VR_D double at(int x, int y, int z) const {
        VR_CHECK_SPAN(p, n, row_ptr(x, y, z) + (x & 3), 1);
        return tap(row_ptr(x, y, z) + (x & 3));
    }
    // four (two) consecutive voxels from x: the 8-byte brick row holding x,
    // plus the next brick's row when the run crosses into it
    VR_D unsigned long long run(int x, int y, int z, int len) const {
        const int16_t *q = row_ptr(x, y, z);
        VR_CHECK_SPAN(p, n, q, 4);
        unsigned long long lo = __ldg(reinterpret_cast<const unsigned long long *>(q));
        const int o = x & 3;
        if (o + len > 4) {
            VR_CHECK_SPAN(p, n, q + 64, 4);
            unsigned long long hi = __ldg(reinterpret_cast<const unsigned long long *>(q + 64));
            lo = (lo >> (16 * o)) | (hi << (64 - 16 * o));
        } else {
            lo >>= 16 * o;
        }
        return lo;
    }
    VR_D void row4(int x, int y, int z, double v[4]) const {
        unsigned long long w = run(x, y, z, 4);
        v[0] = (double)(short)(w & 0xffff);
        v[1] = (double)(short)((w >> 16) & 0xffff);
        v[2] = (double)(short)((w >> 32) & 0xffff);
        v[3] = (double)(short)(w >> 48);
    }
    VR_D void row2(int x, int y, int z, double v[2]) const {
        unsigned long long w = run(x, y, z, 2);
        v[0] = (double)(short)(w & 0xffff);
        v[1] = (double)(short)((w >> 16) & 0xffff);
    }
};

// The pre-classified volume interleaved as one uchar4 (r, g, b, a) per voxel
// -- the (nz, ny, nx, 4) uint8 array transfer.py:142-145 returns -- so one
// 4-byte load serves all four channels of a tap.
struct LinearRGBA {
    const uchar4 *p;
    long long py, pz;
    VR_D uchar4 at(int x, int y, int z) const { return __ldg(p + (long long)z * pz + (long long)y * py + x); }
};

// A block of the decomposition seen through the reference's atlas
// addressing: local coordinates in [0, e) per axis, local voxel i at global
// index origin + i (the atlas copy of a block holds exactly those voxels,
// blocks.py:269-294).
template <class V>
struct Block {
    V vol;
    int ox, oy, oz;
    int ex, ey, ez;
};

// _kernels.py:52-80
template <class V>
VR_D double tri_sample(const Block<V> &b, double x, double y, double z) {
    x = clampf(x, 0.0, b.ex - 1.0);
    y = clampf(y, 0.0, b.ey - 1.0);
    z = clampf(z, 0.0, b.ez - 1.0);
    int i0 = clampi((int)x, 0, b.ex - 2);
    int j0 = clampi((int)y, 0, b.ey - 2);
    int k0 = clampi((int)z, 0, b.ez - 2);
    double fx = x - (double)i0;
    double fy = y - (double)j0;
    double fz = z - (double)k0;
    const int gx = b.ox + i0, gy = b.oy + j0, gz = b.oz + k0;
    double r00[2], r10[2], r01[2], r11[2];
    b.vol.row2(gx, gy, gz, r00);
    b.vol.row2(gx, gy + 1, gz, r10);
    b.vol.row2(gx, gy, gz + 1, r01);
    b.vol.row2(gx, gy + 1, gz + 1, r11);
    double c00 = r00[0] + (r00[1] - r00[0]) * fx;
    double c10 = r10[0] + (r10[1] - r10[0]) * fx;
    double c01 = r01[0] + (r01[1] - r01[0]) * fx;
    double c11 = r11[0] + (r11[1] - r11[0]) * fx;
    double c0 = c00 + (c10 - c00) * fy;
    double c1 = c01 + (c11 - c01) * fy;
    return c0 + (c1 - c0) * fz;
}

// _kernels.py:94-143: taps clamped to the block, rows summed x -> y -> z.
template <class V>
VR_D double cub_sample(const Block<V> &b, double x, double y, double z) {
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
    const int gx[4] = {b.ox + max(i0 - 1, 0), b.ox + i0, b.ox + min(i0 + 1, b.ex - 1), b.ox + min(i0 + 2, b.ex - 1)};
    const int gy[4] = {b.oy + max(j0 - 1, 0), b.oy + j0, b.oy + min(j0 + 1, b.ey - 1), b.oy + min(j0 + 2, b.ey - 1)};
    const int gz[4] = {b.oz + max(k0 - 1, 0), b.oz + k0, b.oz + min(k0 + 1, b.ez - 1), b.oz + min(k0 + 2, b.ez - 1)};
    // unclamped rows are four consecutive voxels
    const bool run = i0 >= 1 && i0 + 2 <= b.ex - 1;
    double pl[4];
#pragma unroll
    for (int c = 0; c < 4; ++c) {
        double s[4];
#pragma unroll
        for (int r = 0; r < 4; ++r) {
            double v[4];
            if (run) {
                b.vol.row4(gx[0], gy[r], gz[c], v);
            } else {
                v[0] = b.vol.at(gx[0], gy[r], gz[c]);
                v[1] = b.vol.at(gx[1], gy[r], gz[c]);
                v[2] = b.vol.at(gx[2], gy[r], gz[c]);
                v[3] = b.vol.at(gx[3], gy[r], gz[c]);
            }
            s[r] = ((wx0 * v[0] + wx1 * v[1]) + wx2 * v[2]) + wx3 * v[3];
        }
        pl[c] = ((wy0 * s[0] + wy1 * s[1]) + wy2 * s[2]) + wy3 * s[3];
    }
    return ((wz0 * pl[0] + wz1 * pl[1]) + wz2 * pl[2]) + wz3 * pl[3];
}

// ---------------------------------------------------- brick-layout sampling

// The brick volume is read in 8-voxel windows: the 8-byte row of the brick
// holding `base` (= first tap index rounded down to a multiple of 4) and the
// same row of the next brick in x.  Every tap of a row lies in that window
// (taps span at most 4 consecutive indices, clamping only pulls them
// inwards), so all rows of a sample are fetched with independent loads
// issued before any arithmetic -- one L2 round trip per interpolation instead
// of one per row -- and each tap is a shift of the window.
VR_D double window_tap(unsigned long long lo, unsigned long long hi, unsigned s) {
    const unsigned long long w = s < 64 ? (lo >> s) : (hi >> (s - 64));
    // (an exact magic-number conversion on the FP64 pipe measured slower
    // than I2F: the sampler is latency-bound, not XU-bound)
    return (double)(short)(w & 0xffffull);
}

// The signed 16-bit halves of a 32-bit word as float64 (exact): one
// conversion each, reading the half in place (no shift or mask first).
VR_D double s16_lo(unsigned w) {
    double d;
    asm("{ .reg .b16 l, h; mov.b32 {l, h}, %1; cvt.rn.f64.s16 %0, l; }" : "=d"(d) : "r"(w));
    return d;
}
VR_D double s16_hi(unsigned w) {
    double d;
    asm("{ .reg .b16 l, h; mov.b32 {l, h}, %1; cvt.rn.f64.s16 %0, h; }" : "=d"(d) : "r"(w));
    return d;
}

// Row offsets relative to the brick row/plane of the first tap g0 (taps span
// at most two bricks per axis), in 32-bit arithmetic: the sample's base
// pointer carries the 64-bit part once.
VR_D unsigned brick_dy(const BrickVol &v, int gy, int gy0) {
    return ((gy >> 2) != (gy0 >> 2) ? (unsigned)v.bpy : 0u) + ((unsigned)(gy & 3) << 2);
}
VR_D unsigned brick_dz(const BrickVol &v, int gz, int gz0) {
    return ((gz >> 2) != (gz0 >> 2) ? (unsigned)v.bpz : 0u) + ((unsigned)(gz & 3) << 4);
}
VR_D const int16_t *brick_base(const BrickVol &v, int base, int gy0, int gz0) {
    return v.p + (long long)(gz0 >> 2) * v.bpz + (long long)(gy0 >> 2) * v.bpy + ((long long)(base >> 2) << 6);
}

// _kernels.py:52-80 on the brick layout
VR_D double tri_sample(const Block<BrickVol> &b, double x, double y, double z) {
    x = clampf(x, 0.0, b.ex - 1.0);
    y = clampf(y, 0.0, b.ey - 1.0);
    z = clampf(z, 0.0, b.ez - 1.0);
    int i0 = clampi((int)x, 0, b.ex - 2);
    int j0 = clampi((int)y, 0, b.ey - 2);
    int k0 = clampi((int)z, 0, b.ez - 2);
    double fx = x - (double)i0;
    double fy = y - (double)j0;
    double fz = z - (double)k0;
    const int gx = b.ox + i0, base = gx & ~3;
    const unsigned s0 = 16u * (unsigned)(gx - base), s1 = s0 + 16u;
    const bool need_hi = (gx - base) == 3;
    const int gy = b.oy + j0, gz = b.oz + k0;
    const int16_t *px = brick_base(b.vol, base, gy, gz);
    const unsigned y0 = brick_dy(b.vol, gy, gy), y1 = brick_dy(b.vol, gy + 1, gy);
    const unsigned z0 = brick_dz(b.vol, gz, gz), z1 = brick_dz(b.vol, gz + 1, gz);
    const unsigned long long *q00 = reinterpret_cast<const unsigned long long *>(px + (y0 + z0));
    const unsigned long long *q10 = reinterpret_cast<const unsigned long long *>(px + (y1 + z0));
    const unsigned long long *q01 = reinterpret_cast<const unsigned long long *>(px + (y0 + z1));
    const unsigned long long *q11 = reinterpret_cast<const unsigned long long *>(px + (y1 + z1));
    VR_CHECK_SPAN(b.vol.p, b.vol.n, px + (y0 + z0), need_hi ? 68 : 4);
    VR_CHECK_SPAN(b.vol.p, b.vol.n, px + (y1 + z1), need_hi ? 68 : 4);
    const unsigned long long l00 = __ldg(q00), l10 = __ldg(q10), l01 = __ldg(q01), l11 = __ldg(q11);
    unsigned long long h00 = 0, h10 = 0, h01 = 0, h11 = 0;
    if (need_hi) {
        h00 = __ldg(q00 + 16);
        h10 = __ldg(q10 + 16);
        h01 = __ldg(q01 + 16);
        h11 = __ldg(q11 + 16);
    }
    double v000 = window_tap(l00, h00, s0), v100 = window_tap(l00, h00, s1);
    double v010 = window_tap(l10, h10, s0), v110 = window_tap(l10, h10, s1);
    double v001 = window_tap(l01, h01, s0), v101 = window_tap(l01, h01, s1);
    double v011 = window_tap(l11, h11, s0), v111 = window_tap(l11, h11, s1);
    double c00 = v000 + (v100 - v000) * fx;
    double c10 = v010 + (v110 - v010) * fx;
    double c01 = v001 + (v101 - v001) * fx;
    double c11 = v011 + (v111 - v011) * fx;
    double c0 = c00 + (c10 - c00) * fy;
    double c1 = c01 + (c11 - c01) * fy;
    return c0 + (c1 - c0) * fz;
}

// _kernels.py:94-143 on the brick layout: same taps, same x -> y -> z sums.
// FUNNEL selects the tap extraction (same values): per-tap 128-bit window
// shifts, or per row one funnel shift, two byte permutes and four in-place
// half conversions (18 instructions per row instead of 22, and fewer live
// registers).  The ray casters use the funnel form (C3-stress +8 %, C3
// +1.8 %, C3-soft +2.8 %, C2 +1.5 % over the window shifts).
template <bool FUNNEL>
VR_D double cub_sample_brick(const Block<BrickVol> &b, double x, double y, double z) {
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
    const int gx0 = b.ox + max(i0 - 1, 0), gx3 = b.ox + min(i0 + 2, b.ex - 1);
    const int base = gx0 & ~3;
    const unsigned s0 = 16u * (unsigned)(gx0 - base);
    const unsigned s1 = 16u * (unsigned)(b.ox + i0 - base);
    const unsigned s2 = 16u * (unsigned)(b.ox + min(i0 + 1, b.ex - 1) - base);
    const unsigned s3 = 16u * (unsigned)(gx3 - base);
    const bool need_hi = (gx3 - base) >= 4;
    const int gy0 = b.oy + max(j0 - 1, 0), gz0 = b.oz + max(k0 - 1, 0);
    const int16_t *px = brick_base(b.vol, base, gy0, gz0);
    const unsigned yo[4] = {brick_dy(b.vol, gy0, gy0), brick_dy(b.vol, b.oy + j0, gy0),
                            brick_dy(b.vol, b.oy + min(j0 + 1, b.ey - 1), gy0),
                            brick_dy(b.vol, b.oy + min(j0 + 2, b.ey - 1), gy0)};
    const unsigned zo[4] = {brick_dz(b.vol, gz0, gz0), brick_dz(b.vol, b.oz + k0, gz0),
                            brick_dz(b.vol, b.oz + min(k0 + 1, b.ez - 1), gz0),
                            brick_dz(b.vol, b.oz + min(k0 + 2, b.ez - 1), gz0)};
    unsigned long long lo[16], hi[16];
#pragma unroll
    for (int c = 0; c < 4; ++c)
#pragma unroll
        for (int r = 0; r < 4; ++r) {
            const unsigned long long *q = reinterpret_cast<const unsigned long long *>(px + (zo[c] + yo[r]));
            VR_CHECK_SPAN(b.vol.p, b.vol.n, px + (zo[c] + yo[r]), need_hi ? 68 : 4);
            lo[4 * c + r] = __ldg(q);
            hi[4 * c + r] = need_hi ? __ldg(q + 16) : 0ull;
        }
    double pl[4];
    // (FUNNEL) one funnel shift per row brings the row's taps into a 64-bit
    // word starting at tap 0
    const unsigned q0 = s0 >> 5, r0 = s0 & 31u;
    const unsigned d1 = s1 - s0, d2 = s2 - s0, d3 = s3 - s0;
    // tap k is the 16-bit half at offset d_k of the shifted window (wl, wh):
    // one byte permute per tap pair gathers (tap0, tap1) and (tap2, tap3)
    // into the halves of two words (the identity away from the block's x
    // faces, where d = 16, 32, 48), each then converted in place
    const unsigned p01 = 0x10u | ((d1 >> 3) << 8) | (((d1 >> 3) + 1u) << 12);
    const unsigned p23 = (d2 >> 3) | (((d2 >> 3) + 1u) << 4) | ((d3 >> 3) << 8) | (((d3 >> 3) + 1u) << 12);
#pragma unroll
    for (int c = 0; c < 4; ++c) {
        double s[4];
#pragma unroll
        for (int r = 0; r < 4; ++r) {
            const unsigned long long l = lo[4 * c + r], h = hi[4 * c + r];
            if (FUNNEL) {
            const unsigned W0 = (unsigned)l, W1 = (unsigned)(l >> 32), W2 = (unsigned)h, W3 = (unsigned)(h >> 32);
            const unsigned a0 = q0 ? W1 : W0, a1 = q0 ? W2 : W1, a2 = q0 ? W3 : W2;
            const unsigned wl = __funnelshift_r(a0, a1, r0), wh = __funnelshift_r(a1, a2, r0);
            const unsigned t01 = __byte_perm(wl, wh, p01), t23 = __byte_perm(wl, wh, p23);
            s[r] = ((wx0 * s16_lo(t01) + wx1 * s16_hi(t01)) + wx2 * s16_lo(t23)) + wx3 * s16_hi(t23);
            } else {
            s[r] = ((wx0 * window_tap(l, h, s0) + wx1 * window_tap(l, h, s1)) + wx2 * window_tap(l, h, s2)) +
                   wx3 * window_tap(l, h, s3);
            }
        }
        pl[c] = ((wy0 * s[0] + wy1 * s[1]) + wy2 * s[2]) + wy3 * s[3];
    }
    return ((wz0 * pl[0] + wz1 * pl[1]) + wz2 * pl[2]) + wz3 * pl[3];
}

VR_D double cub_sample(const Block<BrickVol> &b, double x, double y, double z) {
    return cub_sample_brick<false>(b, x, y, z);
}

// ------------------------------------------------- texture sampling path
// The sampling-path A/B of the north star ("texture path or shared-memory-
// staged bricks, whichever ncu shows is faster"), built with
// -DVR_SAMPLER_TEX=1: a 3-D texture of x-quads (texel (x, y, z) = the int16
// voxels x .. x+3 of row (y, z), short4, point-sampled), so a row of four
// consecutive Catmull-Rom taps is ONE texture fetch through the texture
// cache's 3-D-blocked layout instead of one or two 8-byte brick-window loads
// and per-tap shifts.  Same taps, same sums: bit-identical results.
#ifndef VR_SAMPLER_TEX
#define VR_SAMPLER_TEX 0
#endif
struct TexVol {
    unsigned long long tex;  // cudaTextureObject_t
    VR_D short4 quad(int x, int y, int z) const {
        return tex3D<short4>((cudaTextureObject_t)tex, (float)x + 0.5f, (float)y + 0.5f, (float)z + 0.5f);
    }
};

// _kernels.py:52-80 through the texture
VR_D double tri_sample(const Block<TexVol> &b, double x, double y, double z) {
    x = clampf(x, 0.0, b.ex - 1.0);
    y = clampf(y, 0.0, b.ey - 1.0);
    z = clampf(z, 0.0, b.ez - 1.0);
    int i0 = clampi((int)x, 0, b.ex - 2);
    int j0 = clampi((int)y, 0, b.ey - 2);
    int k0 = clampi((int)z, 0, b.ez - 2);
    double fx = x - (double)i0;
    double fy = y - (double)j0;
    double fz = z - (double)k0;
    const int gx = b.ox + i0, gy = b.oy + j0, gz = b.oz + k0;
    const short4 q00 = b.vol.quad(gx, gy, gz), q10 = b.vol.quad(gx, gy + 1, gz);
    const short4 q01 = b.vol.quad(gx, gy, gz + 1), q11 = b.vol.quad(gx, gy + 1, gz + 1);
    double c00 = (double)q00.x + ((double)q00.y - (double)q00.x) * fx;
    double c10 = (double)q10.x + ((double)q10.y - (double)q10.x) * fx;
    double c01 = (double)q01.x + ((double)q01.y - (double)q01.x) * fx;
    double c11 = (double)q11.x + ((double)q11.y - (double)q11.x) * fx;
    double c0 = c00 + (c10 - c00) * fy;
    double c1 = c01 + (c11 - c01) * fy;
    return c0 + (c1 - c0) * fz;
}

// _kernels.py:94-143 through the texture: a row of consecutive taps is one
// fetch; a row clamped at the block's edge fetches each tap
VR_D double cub_sample(const Block<TexVol> &b, double x, double y, double z) {
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
    const int gx[4] = {b.ox + max(i0 - 1, 0), b.ox + i0, b.ox + min(i0 + 1, b.ex - 1), b.ox + min(i0 + 2, b.ex - 1)};
    const int gy[4] = {b.oy + max(j0 - 1, 0), b.oy + j0, b.oy + min(j0 + 1, b.ey - 1), b.oy + min(j0 + 2, b.ey - 1)};
    const int gz[4] = {b.oz + max(k0 - 1, 0), b.oz + k0, b.oz + min(k0 + 1, b.ez - 1), b.oz + min(k0 + 2, b.ez - 1)};
    const bool run = i0 >= 1 && i0 + 2 <= b.ex - 1;
    short4 q[16];
#pragma unroll
    for (int c = 0; c < 4; ++c)
#pragma unroll
        for (int r = 0; r < 4; ++r) q[4 * c + r] = b.vol.quad(gx[0], gy[r], gz[c]);
    double pl[4];
#pragma unroll
    for (int c = 0; c < 4; ++c) {
        double s[4];
#pragma unroll
        for (int r = 0; r < 4; ++r) {
            double v0, v1, v2, v3;
            if (run) {
                const short4 w = q[4 * c + r];
                v0 = w.x;
                v1 = w.y;
                v2 = w.z;
                v3 = w.w;
            } else {
                v0 = q[4 * c + r].x;
                v1 = b.vol.quad(gx[1], gy[r], gz[c]).x;
                v2 = b.vol.quad(gx[2], gy[r], gz[c]).x;
                v3 = b.vol.quad(gx[3], gy[r], gz[c]).x;
            }
            s[r] = ((wx0 * v0 + wx1 * v1) + wx2 * v2) + wx3 * v3;
        }
        pl[c] = ((wy0 * s[0] + wy1 * s[1]) + wy2 * s[2]) + wy3 * s[3];
    }
    return ((wz0 * pl[0] + wz1 * pl[1]) + wz2 * pl[2]) + wz3 * pl[3];
}

// _kernels.py:52-143 for the four pre-classified channels at once: the same
// taps and the same sums as four separate single-channel samples (c = r, g,
// b, a in out[0..3]), each channel's arithmetic unchanged.
VR_D void tri_sample4(const Block<LinearRGBA> &b, double x, double y, double z, double out[4]) {
    x = clampf(x, 0.0, b.ex - 1.0);
    y = clampf(y, 0.0, b.ey - 1.0);
    z = clampf(z, 0.0, b.ez - 1.0);
    int i0 = clampi((int)x, 0, b.ex - 2);
    int j0 = clampi((int)y, 0, b.ey - 2);
    int k0 = clampi((int)z, 0, b.ez - 2);
    double fx = x - (double)i0;
    double fy = y - (double)j0;
    double fz = z - (double)k0;
    const int gx = b.ox + i0, gy = b.oy + j0, gz = b.oz + k0;
    const uchar4 t000 = b.vol.at(gx, gy, gz), t100 = b.vol.at(gx + 1, gy, gz);
    const uchar4 t010 = b.vol.at(gx, gy + 1, gz), t110 = b.vol.at(gx + 1, gy + 1, gz);
    const uchar4 t001 = b.vol.at(gx, gy, gz + 1), t101 = b.vol.at(gx + 1, gy, gz + 1);
    const uchar4 t011 = b.vol.at(gx, gy + 1, gz + 1), t111 = b.vol.at(gx + 1, gy + 1, gz + 1);
#pragma unroll
    for (int ch = 0; ch < 4; ++ch) {
        auto C = [ch](uchar4 q) { return (double)(ch == 0 ? q.x : ch == 1 ? q.y : ch == 2 ? q.z : q.w); };
        const double c00 = C(t000) + (C(t100) - C(t000)) * fx;
        const double c10 = C(t010) + (C(t110) - C(t010)) * fx;
        const double c01 = C(t001) + (C(t101) - C(t001)) * fx;
        const double c11 = C(t011) + (C(t111) - C(t011)) * fx;
        const double c0 = c00 + (c10 - c00) * fy;
        const double c1 = c01 + (c11 - c01) * fy;
        out[ch] = c0 + (c1 - c0) * fz;
    }
}

VR_D void cub_sample4(const Block<LinearRGBA> &b, double x, double y, double z, double out[4]) {
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
    const int gx[4] = {b.ox + max(i0 - 1, 0), b.ox + i0, b.ox + min(i0 + 1, b.ex - 1), b.ox + min(i0 + 2, b.ex - 1)};
    const int gy[4] = {b.oy + max(j0 - 1, 0), b.oy + j0, b.oy + min(j0 + 1, b.ey - 1), b.oy + min(j0 + 2, b.ey - 1)};
    const int gz[4] = {b.oz + max(k0 - 1, 0), b.oz + k0, b.oz + min(k0 + 1, b.ez - 1), b.oz + min(k0 + 2, b.ez - 1)};
    double acc[4] = {0.0, 0.0, 0.0, 0.0};  // the z sum, built in the reference's order
#pragma unroll
    for (int c = 0; c < 4; ++c) {
        double pl[4] = {0.0, 0.0, 0.0, 0.0};  // per channel, the plane sum over rows
#pragma unroll
        for (int r = 0; r < 4; ++r) {
            const uchar4 q0 = b.vol.at(gx[0], gy[r], gz[c]), q1 = b.vol.at(gx[1], gy[r], gz[c]);
            const uchar4 q2 = b.vol.at(gx[2], gy[r], gz[c]), q3 = b.vol.at(gx[3], gy[r], gz[c]);
            const double wy = r == 0 ? wy0 : r == 1 ? wy1 : r == 2 ? wy2 : wy3;
#pragma unroll
            for (int ch = 0; ch < 4; ++ch) {
                auto C = [ch](uchar4 q) { return (double)(ch == 0 ? q.x : ch == 1 ? q.y : ch == 2 ? q.z : q.w); };
                const double srow = ((wx0 * C(q0) + wx1 * C(q1)) + wx2 * C(q2)) + wx3 * C(q3);
                // ((wy0 s0 + wy1 s1) + wy2 s2) + wy3 s3, accumulated row by row
                pl[ch] = r == 0 ? wy * srow : pl[ch] + wy * srow;
            }
        }
        const double wz = c == 0 ? wz0 : c == 1 ? wz1 : c == 2 ? wz2 : wz3;
#pragma unroll
        for (int ch = 0; ch < 4; ++ch) acc[ch] = c == 0 ? wz * pl[ch] : acc[ch] + wz * pl[ch];
    }
#pragma unroll
    for (int ch = 0; ch < 4; ++ch) out[ch] = acc[ch];
}

template <class V>
VR_D double sample(const Block<V> &b, double x, double y, double z, bool cubic) {
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

// ---------------------------------------------------------------- powers
// pow(x, y) for the exponents the reference raises at run time: the
// opacity correction (1 - a)^(step/ref_step) (_kernels.py:489,519) and the
// Phong exponent (_kernels.py:204,569).  The reference's `**` is libm's pow
// (glibc 2.39), accurate to <= 0.52 ulp but not correctly rounded, so the
// kernels run glibc's own algorithm on its own tables (vr_glibc_pow.h,
// checked bit for bit against libm by tools/gen_pow_tables.py).  y == 1 (the
// default step) is the identity, exactly as libm's pow(x, 1) == x.
struct PowSpec {
    int kind;  // 0 identity (y == 1), 1 glibc pow
    double y;
};

inline PowSpec make_pow(double y) {
    PowSpec p;
    p.y = y;
    p.kind = (y == 1.0) ? 0 : 1;
    return p;
}

// out of line: one copy of the ~80-instruction pow serves every call site
static __device__ __noinline__ double pow_glibc(double x, double y) { return vr_glibc_pow(x, y); }

// (+0)^y = +0 for y > 0 without the call: the Phong base max(2 (n.l)^2 - 1, 0)
// is zero for most shaded samples
VR_D double vr_pow(double x, const PowSpec &p) {
    if (p.kind == 0) return x;
    if (x == 0.0 && p.y > 0.0) return 0.0;
    return pow_glibc(x, p.y);
}

}  // namespace vr
