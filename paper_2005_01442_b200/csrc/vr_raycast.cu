// vr_raycast.cu -- K3: ray generation, box clipping, empty-space leaping,
// Catmull-Rom / trilinear sampling, classification, headlight shading and
// front-to-back compositing with early ray termination, fused with the
// straight-alpha uint8 epilogue and the stats reduction.
//
// Follows _kernels.march (/root/reference/pkg/src/voxelray/_kernels.py:279-594)
// sample for sample: the n-th sample of a ray sits at t = t0 + (n + 0.5)*step,
// block attribution is floor((x - 1)/stride), and every taken sample is
// classified and composited with the reference's float64 operation order.
// What differs is how skipped samples are found: instead of testing the skip
// predicate at every step (_kernels.py:377-399), a ray in a skippable region
// leaps to the last sample that is provably still inside it -- the exit of its
// ownership cell, the entry of the block's visibility box, or the entry of the
// union of all visibility boxes, each shrunk by a 1e-6-voxel guard and one
// sample -- then re-evaluates the exact predicate there.  samples_taken /
// samples_skipped therefore match the reference exactly while the work per
// ray is O(cells crossed near visible matter).
//
// The kernel is specialised per (mode/classification, interpolation,
// lighting, leaping) so each instantiation carries only its own path: one
// kernel holding every branch spilled the instruction cache (ncu: 16% of warp
// samples stalled on no_instructions) and needed 154 registers.
#include <cfloat>
#include <climits>
#include <mutex>

#include "vr_raycast.cuh"

namespace vr {
namespace {

enum Kind { kPost = 0, kPre = 1, kPreint = 2, kIso = 3 };

struct Ray {
    double ox, oy, oz, dx, dy, dz;
};

// One view's camera: basis and image-plane half extents.
struct ViewCam {
    double pos[3], fwd[3], right[3], up[3];
    double half_w, half_h;
};

// Ray-setup divisions (once per ray): out of line in A/B builds
#ifndef VR_SETUP_DIV_OOL
#define VR_SETUP_DIV_OOL 1  // C3 +0.5 %, C3-soft +2.6 % (a smaller per-lane kernel)
#endif
#if VR_SETUP_DIV_OOL
VR_D double sdiv(double x, double y) { return div_rn(x, y); }
#else
VR_D double sdiv(double x, double y) { return x / y; }
#endif

VR_D ViewCam view_cam(const RenderArgs &a, int v) {
    ViewCam c;
    if (a.views) {
        const double *p = a.views + 14 * (long long)v;
#pragma unroll
        for (int k = 0; k < 3; ++k) {
            c.pos[k] = __ldg(p + k);
            c.fwd[k] = __ldg(p + 3 + k);
            c.right[k] = __ldg(p + 6 + k);
            c.up[k] = __ldg(p + 9 + k);
        }
        c.half_w = __ldg(p + 12);
        c.half_h = __ldg(p + 13);
    } else {
#pragma unroll
        for (int k = 0; k < 3; ++k) {
            c.pos[k] = a.pos[k];
            c.fwd[k] = a.fwd[k];
            c.right[k] = a.right[k];
            c.up[k] = a.up[k];
        }
        c.half_w = a.half_w;
        c.half_h = a.half_h;
    }
    return c;
}

// render.py:125-144 (pinhole) per pixel, or the orthographic variant.
VR_D Ray make_ray(const RenderArgs &a, const ViewCam &c, int px, int py) {
    Ray r;
    double v = (1.0 - sdiv(2.0 * ((double)py + 0.5), (double)a.H)) * c.half_h;
    double u = (sdiv(2.0 * ((double)px + 0.5), (double)a.W) - 1.0) * c.half_w;
    if (a.projection == 0) {
        double d0 = (c.fwd[0] + u * c.right[0]) + v * c.up[0];
        double d1 = (c.fwd[1] + u * c.right[1]) + v * c.up[1];
        double d2 = (c.fwd[2] + u * c.right[2]) + v * c.up[2];
        double nrm = sqrt((d0 * d0 + d1 * d1) + d2 * d2);
        r.dx = sdiv(d0, nrm);
        r.dy = sdiv(d1, nrm);
        r.dz = sdiv(d2, nrm);
        r.ox = c.pos[0];
        r.oy = c.pos[1];
        r.oz = c.pos[2];
    } else {
        r.ox = (c.pos[0] + u * c.right[0]) + v * c.up[0];
        r.oy = (c.pos[1] + u * c.right[1]) + v * c.up[1];
        r.oz = (c.pos[2] + u * c.right[2]) + v * c.up[2];
        r.dx = c.fwd[0];
        r.dy = c.fwd[1];
        r.dz = c.fwd[2];
    }
    return r;
}

// Per-view sample counts of one lane: accumulated while the lane's rays belong
// to one view, added to that view's totals when the view changes (a lane's
// rays come in increasing item order, so at most once per view) and at exit.
struct ViewTotals {
    int view = -1;
    unsigned long long taken = 0, skipped = 0;
    VR_D void add(const RenderArgs &a, int v, long long t, long long s) {
        if (v != view) {
            flush(a);
            view = v;
        }
        taken += (unsigned long long)t;
        skipped += (unsigned long long)s;
    }
    VR_D void flush(const RenderArgs &a) {
        if (view >= 0 && a.totals && (taken | skipped)) {
            atomicAdd(a.totals + 5 * (long long)view, taken);
            atomicAdd(a.totals + 5 * (long long)view + 1, skipped);
        }
        taken = skipped = 0;
    }
    // exit: lanes holding the same view combine their counts first (one
    // atomic pair per view per warp; all lanes of the warp must call this)
    VR_D void flush_warp(const RenderArgs &a) {
        const unsigned same = __match_any_sync(0xffffffffu, view);
        const unsigned t = __reduce_add_sync(same, (unsigned)taken);
        const unsigned sk = __reduce_add_sync(same, (unsigned)skipped);
        if ((int)(threadIdx.x & 31) == __ffs(same) - 1) {
            taken = t;
            skipped = sk;
            flush(a);
        }
    }
};

// render.py:147-156
VR_D void clip_to_bounds(const Ray &r, const double ext[3], double &tmin, double &tmax) {
    const double tiny = 1e-300;
    const double o[3] = {r.ox, r.oy, r.oz};
    const double d[3] = {r.dx, r.dy, r.dz};
    double lo_max = 0.0, hi_min = 0.0;
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        double dd = d[k];
        if (fabs(dd) < tiny) dd = (dd < 0) ? -tiny : tiny;
        double lo = sdiv(0.0 - o[k], dd);
        double hi = sdiv(ext[k] - o[k], dd);
        double mn = lo < hi ? lo : hi;
        double mx = lo > hi ? lo : hi;
        if (k == 0 || mn > lo_max) lo_max = mn;
        if (k == 0 || mx < hi_min) hi_min = mx;
    }
    tmin = lo_max > 0.0 ? lo_max : 0.0;
    tmax = hi_min;
}

VR_D int owner(const RenderArgs &a, int axis, double v) {
    return owner_block(v, a.L.strided, a.L.inv_stride, a.L.nb[axis]);
}

// _attr_sample (_kernels.py:211-233) with the owning block already known:
// local coordinates x - origin, taps clamped to the block, voxels read in
// place from the volume (the atlas copy holds the same voxels).
template <bool CUBIC, class V>
VR_D double sample_in(const V &vol, const RenderArgs &a, int bi, int bj, int bk, double x, double y, double z) {
    Block<V> b;
    b.vol = vol;
    b.ox = block_origin(a.L, bi);
    b.oy = block_origin(a.L, bj);
    b.oz = block_origin(a.L, bk);
    b.ex = block_extent(a.L, 0, bi);
    b.ey = block_extent(a.L, 1, bj);
    b.ez = block_extent(a.L, 2, bk);
    const double lx = x - (double)b.ox, ly = y - (double)b.oy, lz = z - (double)b.oz;
    return CUBIC ? cub_sample(b, lx, ly, lz) : tri_sample(b, lx, ly, lz);
}

// the ray casters' interpolant: brick windows through L1 (default) or the
// x-quad texture (VR_SAMPLER_TEX A/B builds)
// (FUNNEL: the brick sampler's funnel + byte-permute tap extraction)
#ifndef VR_LIT_FUNNEL
#define VR_LIT_FUNNEL 1  // 0: per-tap window shifts in the lit kernels (A/B builds)
#endif
template <bool CUBIC, bool FUNNEL = (VR_LIT_FUNNEL != 0)>
VR_D double vol_sample(const RenderArgs &a, int bi, int bj, int bk, double x, double y, double z) {
#if VR_SAMPLER_TEX
    return sample_in<CUBIC>(a.tv, a, bi, bj, bk, x, y, z);
#else
    if (CUBIC && FUNNEL) {
        Block<BrickVol> b;
        b.vol = a.bv;
        b.ox = block_origin(a.L, bi);
        b.oy = block_origin(a.L, bj);
        b.oz = block_origin(a.L, bk);
        b.ex = block_extent(a.L, 0, bi);
        b.ey = block_extent(a.L, 1, bj);
        b.ez = block_extent(a.L, 2, bk);
        return cub_sample_brick<true>(b, x - (double)b.ox, y - (double)b.oy, z - (double)b.oz);
    }
    return sample_in<CUBIC>(a.bv, a, bi, bj, bk, x, y, z);
#endif
}

template <bool CUBIC>
VR_D double attr_sample(const RenderArgs &a, double x, double y, double z) {
    return vol_sample<CUBIC>(a, owner(a, 0, x), owner(a, 1, y), owner(a, 2, z), x, y, z);
}

// _attr_grad (_kernels.py:236-253): six taps at +-0.5 voxel, each attributed
// to its own block (only the displaced axis can change owner), then / spacing.
// One loop body so the interpolant is instantiated once for all six.
template <bool CUBIC>
VR_D void attr_grad(const RenderArgs &a, double x, double y, double z, int bi, int bj, int bk, double g[3]) {
    double plus = 0.0;
#pragma unroll 1
    for (int q = 0; q < 6; ++q) {
        const int axis = q >> 1;
        const double h = (q & 1) ? -0.5 : 0.5;
        double px = x, py = y, pz = z;
        int qi = bi, qj = bj, qk = bk;
        if (axis == 0) {
            px = x + h;
            qi = owner(a, 0, px);
        } else if (axis == 1) {
            py = y + h;
            qj = owner(a, 1, py);
        } else {
            pz = z + h;
            qk = owner(a, 2, pz);
        }
        double s = vol_sample<CUBIC>(a, qi, qj, qk, px, py, pz);
        if (q & 1)
            g[axis] = plus - s;
        else
            plus = s;
    }
    g[0] = divide(g[0], a.dsx);
    g[1] = divide(g[1], a.dsy);
    g[2] = divide(g[2], a.dsz);
}

// _attr_rgba (_kernels.py:256-276) for the four channels at once: out =
// (r, g, b, a), each clamp(v / 255, 0, 1) exactly as the per-channel call
template <bool CUBIC>
VR_D void attr_rgba4(const RenderArgs &a, int bi, int bj, int bk, double x, double y, double z, double out[4]) {
    Block<LinearRGBA> b;
    b.vol.p = reinterpret_cast<const uchar4 *>(a.rgba);
    b.vol.py = a.L.py;
    b.vol.pz = a.L.pz;
    b.ox = block_origin(a.L, bi);
    b.oy = block_origin(a.L, bj);
    b.oz = block_origin(a.L, bk);
    b.ex = block_extent(a.L, 0, bi);
    b.ey = block_extent(a.L, 1, bj);
    b.ez = block_extent(a.L, 2, bk);
    const double lx = x - (double)b.ox, ly = y - (double)b.oy, lz = z - (double)b.oz;
    if (CUBIC)
        cub_sample4(b, lx, ly, lz, out);
    else
        tri_sample4(b, lx, ly, lz, out);
#pragma unroll
    for (int c = 0; c < 4; ++c) out[c] = clampf(out[c] / 255.0, 0.0, 1.0);
}

// _kernels.py:190-192

// _kernels.py:195-208
VR_D void shade(const RenderArgs &a, double &r, double &g, double &b, double nx, double ny, double nz,
                double lx, double ly, double lz) {
    double ndl = (nx * lx + ny * ly) + nz * lz;
    double diff = a.kd * pymax0(ndl);
    double rv = 2.0 * ndl * ndl - 1.0;
    double spec = a.ks * vr_pow(pymax0(rv), a.shin);
    r = clampf(r * (a.ka + diff) + spec, 0.0, 1.0);
    g = clampf(g * (a.ka + diff) + spec, 0.0, 1.0);
    b = clampf(b * (a.ka + diff) + spec, 0.0, 1.0);
}

VR_D double dmin(double a, double b) { return a < b ? a : b; }
VR_D double dmax(double a, double b) { return a > b ? a : b; }

// Per-frame skip state of one block, 32 bytes (box_kernel, vr_prep.cu): the
// visibility box +- margin (integers +- 2 or 3, exact in float32) and the
// empty flag, fetched with two 16-byte loads.
struct BlockRec {
    float4 lo;  // x, y, z, empty (1.0f / 0.0f)
    float4 hi;  // x, y, z, unused
};

VR_D BlockRec block_rec(const RenderArgs &a, int b) {
    const float4 *p = reinterpret_cast<const float4 *>(a.box) + 2 * (long long)b;
    BlockRec r;
    r.lo = __ldg(p);
    r.hi = __ldg(p + 1);
    return r;
}

// The reference's DVR skip predicate (_kernels.py:381-391) for block b.
VR_D bool dvr_skippable(const BlockRec &r, double x, double y, double z) {
    return r.lo.w != 0.0f || x < (double)r.lo.x || x > (double)r.hi.x || y < (double)r.lo.y ||
           y > (double)r.hi.y || z < (double)r.lo.z || z > (double)r.hi.z;
}

// Whether the interpolated value at (x, y, z) provably classifies to a
// zero-opacity LUT bin, so the reference's sample would contribute nothing
// (_kernels.py:513-515: alpha == 0 -> no compositing).  The bounds come from
// K1 (launch_interp_bounds): per unit cube g = floor(clamp(coordinate)) the
// range of the trilinear / Catmull-Rom interpolant under any block-local tap
// clamping, and per 4^3 cell the union of its cubes' ranges.  Returns 0 (not
// provable), 1 (the whole cell is transparent: culled_run may leap to the
// cell exit) or 2 (this sample's unit cube is: a leap to the cube's exit, the
// cube bound covering every sample based in it).  A bound at the
// int16 limit is saturated and proves nothing on that side.  Before the cell,
// the 16^3 macro cell (union of 64 cells) is tried: 3 = transparent there,
// culled_run may leap to the macro-cell exit.
VR_D bool bounds_transparent(short2 b, int vlo, int vhi) {
    // integer thresholds of the visible bins (visible_value_range); a bound at
    // the int16 limit is saturated: unbounded on that side
    const int up = b.y >= 32767 ? INT_MAX : (int)b.y;
    const int dn = b.x <= -32768 ? INT_MIN : (int)b.x;
    return up < vlo || dn > vhi;
}

template <bool CUBIC>
VR_D int provably_transparent(const RenderArgs &a, double x, double y, double z, int vlo, int vhi) {
    // == (int)clamp(v, 0, n-1): truncation then an integer clamp (|v| << 2^31)
    const int gx = clampi((int)x, 0, a.L.n[0] - 1);
    const int gy = clampi((int)y, 0, a.L.n[1] - 1);
    const int gz = clampi((int)z, 0, a.L.n[2] - 1);
    if (a.mcells &&
        bounds_transparent(__ldg(a.mcells + ((long long)(gz >> 4) * a.nmy + (gy >> 4)) * a.nmx + (gx >> 4)), vlo, vhi))
        return 3;
    if (bounds_transparent(__ldg(a.cells + ((long long)(gz >> 2) * a.ncy + (gy >> 2)) * a.ncx + (gx >> 2)), vlo, vhi))
        return 1;
    if (!a.cubes) return 0;
    const long long ci = (long long)(gz >> 2) * a.bv.bpz + (long long)(gy >> 2) * a.bv.bpy +
                         ((long long)(gx >> 2) << 6) + ((gz & 3) << 4) + ((gy & 3) << 2) + (gx & 3);
    VR_CHECK_SPAN(a.cubes, a.bv.n, a.cubes + ci, 1);  // (one bound per voxel, brick order)
    const short2 w = __ldg(a.cubes + ci);
    return bounds_transparent(w, vlo, vhi) ? 2 : 0;
}

// The cell level of provably_transparent alone: every sample based in the
// 4^3 cell around (x, y, z) classifies to a zero-opacity bin.
VR_D bool cell_transparent(const RenderArgs &a, double x, double y, double z, int vlo, int vhi) {
    const int gx = clampi((int)x, 0, a.L.n[0] - 1);
    const int gy = clampi((int)y, 0, a.L.n[1] - 1);
    const int gz = clampi((int)z, 0, a.L.n[2] - 1);
    return bounds_transparent(__ldg(a.cells + ((long long)(gz >> 2) * a.ncy + (gy >> 2)) * a.ncx + (gx >> 2)), vlo,
                              vhi);
}

// Chained modes (iso, pre-integrated), the analogue of provably_transparent:
// the level (3 macro cell, 1 cell, 2 unit cube; 0 none) of the largest
// region around (x, y, z) whose interpolant bound [lo, hi] guarantees that
// consecutive samples inside it change nothing the reference composites:
//  - iso: the bound excludes the isovalue, so every sample lies strictly on
//    one side -- no sign change, no exact hit (_kernels.py:446-465);
//  - pre-integrated: every table cell (front bin, back bin) with both bins in
//    [bin(lo), bin(hi)] has zero opacity (_kernels.py:555-558: seg_a == 0,
//    nothing composited).  a.tbl_nz is the 2-D prefix count of cells with
//    alpha > 0, so the square test is four lookups.
template <int KIND>
VR_D bool chain_bound_ok(const RenderArgs &a, short2 b) {
    if (b.x <= -32768 || b.y >= 32767) return false;  // saturated: unbounded
    if (KIND == kIso) return (double)b.y < a.isovalue || (double)b.x > a.isovalue;
    const int i0 = lut_bin((double)b.x, a.tbl_lo, a.tbl_inv_w, a.ntbl);
    const int i1 = lut_bin((double)b.y, a.tbl_lo, a.tbl_inv_w, a.ntbl) + 1;
    const long long w = a.ntbl + 1;
    const int cnt = __ldg(a.tbl_nz + i1 * w + i1) - __ldg(a.tbl_nz + i0 * w + i1) - __ldg(a.tbl_nz + i1 * w + i0) +
                    __ldg(a.tbl_nz + i0 * w + i0);
    return cnt == 0;
}

template <int KIND>
VR_D int chain_transparent(const RenderArgs &a, double x, double y, double z, short2 *bound = nullptr) {
    const int gx = clampi((int)x, 0, a.L.n[0] - 1);
    const int gy = clampi((int)y, 0, a.L.n[1] - 1);
    const int gz = clampi((int)z, 0, a.L.n[2] - 1);
    if (a.mcells) {
        const short2 w = __ldg(a.mcells + ((long long)(gz >> 4) * a.nmy + (gy >> 4)) * a.nmx + (gx >> 4));
        if (chain_bound_ok<KIND>(a, w)) {
            if (bound) *bound = w;
            return 3;
        }
    }
    const short2 c = __ldg(a.cells + ((long long)(gz >> 2) * a.ncy + (gy >> 2)) * a.ncx + (gx >> 2));
    if (chain_bound_ok<KIND>(a, c)) {
        if (bound) *bound = c;
        return 1;
    }
    if (!a.cubes) return 0;
    const long long ci = (long long)(gz >> 2) * a.bv.bpz + (long long)(gy >> 2) * a.bv.bpy +
                         ((long long)(gx >> 2) << 6) + ((gz & 3) << 4) + ((gy & 3) << 2) + (gx & 3);
    VR_CHECK_SPAN(a.cubes, a.bv.n, a.cubes + ci, 1);  // (one bound per voxel, brick order)
    const short2 w = __ldg(a.cubes + ci);
    if (!chain_bound_ok<KIND>(a, w)) return 0;
    if (bound) *bound = w;
    return 2;
}

// Pre-classified culling: the level (4 macro cell, 2 cell; 0 none) of the
// region around (x, y, z) whose raw footprint bound (a.cells / a.mcells hold
// raw voxel ranges in this mode) lies outside the frame's non-zero-alpha
// value range: every tap of every sample based there has a zero alpha plane.
VR_D int pre_transparent(const RenderArgs &a, double x, double y, double z) {
    const int gx = clampi((int)x, 0, a.L.n[0] - 1), gy = clampi((int)y, 0, a.L.n[1] - 1);
    const int gz = clampi((int)z, 0, a.L.n[2] - 1);
    const int plo = __ldg(a.pre_range), phi = __ldg(a.pre_range + 1);
    const short2 mb = __ldg(a.mcells + ((long long)(gz >> 4) * a.nmy + (gy >> 4)) * a.nmx + (gx >> 4));
    if ((int)mb.y < plo || (int)mb.x > phi) return 4;
    const short2 cb = __ldg(a.cells + ((long long)(gz >> 2) * a.ncy + (gy >> 2)) * a.ncx + (gx >> 2));
    return ((int)cb.y < plo || (int)cb.x > phi) ? 2 : 0;
}

// Parameter interval in which the (exact) ray lies inside the box [lo, hi]
// expanded by delta on every side; returns false when it never does.  For an
// axis the ray does not move along, the computed coordinate is exactly
// constant, so the test uses the unexpanded bounds on it.
VR_D bool slab(const double o[3], const double d[3], const double inv[3], const double s[3], const double p[3],
               const double lo[3], const double hi[3], double delta, double &tin, double &tout) {
    tin = -DBL_MAX;
    tout = DBL_MAX;
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        if (d[k] == 0.0) {
            if (p[k] < lo[k] || p[k] > hi[k]) return false;
        } else {
            double ta = ((lo[k] - delta) * s[k] - o[k]) * inv[k];
            double tb = ((hi[k] + delta) * s[k] - o[k]) * inv[k];
            tin = dmax(tin, dmin(ta, tb));
            tout = dmin(tout, dmax(ta, tb));
        }
    }
    return tin <= tout;
}

// Number k >= 1 of samples, starting at the skippable sample n (parameter t,
// computed position p, owner block (bidx, b)), that are guaranteed skippable.
// Every sample strictly before the returned safe parameter lies, in exact
// arithmetic, at least `delta` voxel inside the current ownership cell and
// outside the block's box (when it is non-empty), or outside the union of
// all visibility boxes; computed positions err by < 1e-11 voxel, so they give
// the same verdict.  One sample of slack absorbs the rounding of t itself;
// reciprocal multiplies stand in for divisions for the same reason.
template <int KIND>
VR_D long long leap_count(const RenderArgs &a, const Ray &r, const double inv[3], double t0, long long n,
                          double t, const double p[3], const int bidx[3], const BlockRec &rec, bool cell_only) {
    const double delta = 1e-6;
    const double d[3] = {r.dx, r.dy, r.dz};
    const double o[3] = {r.ox, r.oy, r.oz};
    const double s[3] = {a.dsx.s, a.dsy.s, a.dsz.s};
    double t_safe = DBL_MAX;
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        if (d[k] > 0.0 && bidx[k] < a.L.nb[k] - 1) {
            double X = (1.0 + (double)((bidx[k] + 1) * a.L.stride)) - delta;
            t_safe = dmin(t_safe, (X * s[k] - o[k]) * inv[k]);
        } else if (d[k] < 0.0 && bidx[k] > 0) {
            double X = (1.0 + (double)(bidx[k] * a.L.stride)) + delta;
            t_safe = dmin(t_safe, (X * s[k] - o[k]) * inv[k]);
        }
    }
    if (KIND != kIso) {
        if (!cell_only) {
            const double lo[3] = {(double)rec.lo.x, (double)rec.lo.y, (double)rec.lo.z};
            const double hi[3] = {(double)rec.hi.x, (double)rec.hi.y, (double)rec.hi.z};
            double tin, tout;
            if (slab(o, d, inv, s, p, lo, hi, delta, tin, tout) && tout >= t)
                t_safe = (tin > t) ? dmin(t_safe, tin) : t;
        }
        // union of every non-empty block's box: outside it nothing is visible
        double tin, tout;
        double ut;
        const int u0 = __ldg(a.uni), u3 = __ldg(a.uni + 3);
        const double ulo[3] = {(double)u0 - a.margin, (double)__ldg(a.uni + 1) - a.margin,
                               (double)__ldg(a.uni + 2) - a.margin};
        const double uhi[3] = {(double)u3 + a.margin, (double)__ldg(a.uni + 4) + a.margin,
                               (double)__ldg(a.uni + 5) + a.margin};
        if (u0 > u3) {
            ut = DBL_MAX;  // no visible block at all
        } else if (!slab(o, d, inv, s, p, ulo, uhi, delta, tin, tout) || tout < t) {
            ut = DBL_MAX;
        } else {
            ut = tin > t ? tin : t;
        }
        t_safe = dmax(t_safe, ut);
    }
    if (!(t_safe > t)) return 1;
    double q = (t_safe - t0) * a.inv_step - 0.5;
    if (q > 4.0e15) return LLONG_MAX / 4;
    long long m = (long long)floor(q) - 1;
    long long k = m - n + 1;
    return k < 1 ? 1 : k;
}

// Number k >= 1 of samples, starting at the taken, provably transparent sample
// n, that are all taken and provably transparent: they stay in the same
// dilated culling cell (so the same min/max bound applies) and, on the block
// path, in the same ownership cell and inside the same visibility box (so
// the skip predicate stays false).  Computed positions are monotone in n, so
// only the exit side of each interval needs the delta guard; the one-sample
// slack absorbs the rounding of t.
template <bool SKIP, bool BOX = true>
VR_D long long culled_run(const RenderArgs &a, const Ray &r, const double inv[3], double t0, long long n, double t,
                          const double p[3], const int bidx[3], const BlockRec &rec, int shift) {
    const double delta = 1e-6;
    const double d[3] = {r.dx, r.dy, r.dz};
    const double o[3] = {r.ox, r.oy, r.oz};
    const double s[3] = {a.dsx.s, a.dsy.s, a.dsz.s};
    double t_safe = DBL_MAX;
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        if (d[k] == 0.0) continue;
        const int g = clampi((int)p[k], 0, a.L.n[k] - 1);  // == (int)clamp(p, 0, n-1)
        const int c = g >> shift, clast = (a.L.n[k] - 1) >> shift;
        const double size = (double)(1 << shift);
        if (d[k] > 0.0 && c < clast) t_safe = dmin(t_safe, ((size * (c + 1) - delta) * s[k] - o[k]) * inv[k]);
        if (d[k] < 0.0 && c > 0) t_safe = dmin(t_safe, ((size * c + delta) * s[k] - o[k]) * inv[k]);
        if (SKIP) {
            if (d[k] > 0.0 && bidx[k] < a.L.nb[k] - 1) {
                double X = (1.0 + (double)((bidx[k] + 1) * a.L.stride)) - delta;
                t_safe = dmin(t_safe, (X * s[k] - o[k]) * inv[k]);
            } else if (d[k] < 0.0 && bidx[k] > 0) {
                double X = (1.0 + (double)(bidx[k] * a.L.stride)) + delta;
                t_safe = dmin(t_safe, (X * s[k] - o[k]) * inv[k]);
            }
            if (BOX) {  // (iso's skip predicate is per block, without a box)
                const float lo_k = k == 0 ? rec.lo.x : (k == 1 ? rec.lo.y : rec.lo.z);
                const float hi_k = k == 0 ? rec.hi.x : (k == 1 ? rec.hi.y : rec.hi.z);
                const double edge = d[k] > 0.0 ? (double)hi_k - delta : (double)lo_k + delta;
                t_safe = dmin(t_safe, (edge * s[k] - o[k]) * inv[k]);
            }
        }
    }
    if (!(t_safe > t)) return 1;
    double q = (t_safe - t0) * a.inv_step - 0.5;
    if (q > 4.0e15) return LLONG_MAX / 4;
    long long m = (long long)floor(q) - 1;
    long long k = m - n + 1;
    return k < 1 ? 1 : k;
}

struct RayResult {
    double r, g, b, a;
    double depth;
    long long taken, skipped, shaded, eval, iter;
};

// One pixel of _kernels.march (:343-594).
template <int KIND, bool CUBIC, bool LIGHT, bool SKIP>
VR_D RayResult march(const RenderArgs &a, const Ray &r, double t0, double t1, uint8_t *hits) {
    constexpr bool chained = (KIND == kIso) || (KIND == kPreint);  // _kernels.py:341
    RayResult res;
    double acc_r = 0.0, acc_g = 0.0, acc_b = 0.0, acc_a = 0.0;
    long long n_taken = 0, n_skip = 0, n_shaded = 0, n_eval = 0, n_iter = 0;
    double depth = __longlong_as_double(0x7ff8000000000000LL);  // NaN
    if (t1 >= t0) {
        const double step = a.step;
        long long nsteps = (long long)ceil((t1 - t0) / step);
        if (nsteps < 1) nsteps = 1;
        // the reference breaks at the first t > t1; t(n) is monotone in n, so
        // the samples it visits are exactly the prefix [0, N)
        long long N = nsteps;
        while (N > 0 && (t0 + ((double)(N - 1) + 0.5) * step) > t1) --N;
        const int nbx = a.L.nb[0], nby = a.L.nb[1];
        double inv[3] = {0.0, 0.0, 0.0};
        if (SKIP || a.cull) {
            inv[0] = r.dx != 0.0 ? 1.0 / r.dx : 0.0;
            inv[1] = r.dy != 0.0 ? 1.0 / r.dy : 0.0;
            inv[2] = r.dz != 0.0 ? 1.0 / r.dz : 0.0;
        }
        double prev_s = 0.0;
        bool prev_valid = false, prev_skippable = false;
        int last_hit = -1;
        int first_vis = INT_MIN, last_vis = INT_MAX;  // value thresholds (vlo, vhi)
        const bool cull = KIND == kPost && a.cull;
        // chained modes: after a culled run the previous sample's value was not
        // computed; the next evaluated sample recomputes it at that sample's
        // own position (the reference interpolated it there)
        const bool chain_cull = (KIND == kIso || KIND == kPreint) && a.cull;
        bool prev_pending = false;
        if (cull) {
            first_vis = __ldg(a.lut_range + 2);
            last_vis = __ldg(a.lut_range + 3);
        }
        long long n = 0;
        while (n < N) {
            ++n_iter;
            const double t = t0 + ((double)n + 0.5) * step;
            const double x = divide(r.ox + t * r.dx, a.dsx);
            const double y = divide(r.oy + t * r.dy, a.dsy);
            const double z = divide(r.oz + t * r.dz, a.dsz);
            const int bi = owner(a, 0, x), bj = owner(a, 1, y), bk = owner(a, 2, z);
            const int b = (bk * nby + bj) * nbx + bi;

            BlockRec rec = {};
            if (SKIP) {
                bool skippable, cell_only = true;
                if (KIND == kIso) {
                    skippable = (double)__ldg(a.vmax + b) < a.isovalue || (double)__ldg(a.vmin + b) > a.isovalue;
                } else {
                    rec = block_rec(a, b);
                    skippable = dvr_skippable(rec, x, y, z);
                    cell_only = rec.lo.w != 0.0f;
                }
                if (skippable && (prev_skippable || !chained)) {
                    const double p[3] = {x, y, z};
                    const int bidx[3] = {bi, bj, bk};
                    long long k = leap_count<KIND>(a, r, inv, t0, n, t, p, bidx, rec, cell_only);
                    long long m = (N - n < k) ? N : n + k;
                    n_skip += m - n;
                    n = m;
                    prev_valid = false;
                    prev_pending = false;
                    prev_skippable = true;
                    continue;
                }
                prev_skippable = skippable;
            }
            if (b != last_hit) {
                if (hits) hits[b] = 1;
                last_hit = b;
            }
            n_taken += 1;

            if (chain_cull && prev_pending) {
                // sample n-1 was taken inside a culled run: its exact value
                const double tq = t0 + ((double)(n - 1) + 0.5) * step;
                prev_s = attr_sample<CUBIC>(a, divide(r.ox + tq * r.dx, a.dsx), divide(r.oy + tq * r.dy, a.dsy),
                                            divide(r.oz + tq * r.dz, a.dsz));
                prev_valid = true;
                prev_pending = false;
            }
            if (KIND == kIso) {
                // _kernels.py:405-468
                double s = vol_sample<CUBIC>(a, bi, bj, bk, x, y, z);
                if (!prev_valid && n > 0) {
                    double tp = t - step;
                    prev_s = attr_sample<CUBIC>(a, divide(r.ox + tp * r.dx, a.dsx), divide(r.oy + tp * r.dy, a.dsy),
                                                divide(r.oz + tp * r.dz, a.dsz));
                    prev_valid = true;
                }
                bool hit = false;
                double t_hit = t;
                if (prev_valid && (prev_s - a.isovalue) * (s - a.isovalue) < 0.0) {
                    double lo_t = t - step, hi_t = t, lo_s = prev_s;
#pragma unroll 1
                    for (int it = 0; it < 8; ++it) {
                        double mid = 0.5 * (lo_t + hi_t);
                        double ms = attr_sample<CUBIC>(a, divide(r.ox + mid * r.dx, a.dsx),
                                                       divide(r.oy + mid * r.dy, a.dsy),
                                                       divide(r.oz + mid * r.dz, a.dsz));
                        if ((lo_s - a.isovalue) * (ms - a.isovalue) <= 0.0) {
                            hi_t = mid;
                        } else {
                            lo_t = mid;
                            lo_s = ms;
                        }
                    }
                    t_hit = 0.5 * (lo_t + hi_t);
                    hit = true;
                } else if (s == a.isovalue) {
                    hit = true;
                }
                if (hit) {
                    double hx = divide(r.ox + t_hit * r.dx, a.dsx);
                    double hy = divide(r.oy + t_hit * r.dy, a.dsy);
                    double hz = divide(r.oz + t_hit * r.dz, a.dsz);
                    int ib = lut_bin(a.isovalue, a.lut_lo, a.lut_inv_w, a.nlut);
                    double cr = __ldg(a.lut + 4 * ib), cg = __ldg(a.lut + 4 * ib + 1), cb = __ldg(a.lut + 4 * ib + 2);
                    double g[3];
                    attr_grad<CUBIC>(a, hx, hy, hz, owner(a, 0, hx), owner(a, 1, hy), owner(a, 2, hz), g);
                    n_shaded += 1;
                    double norm = sqrt((g[0] * g[0] + g[1] * g[1]) + g[2] * g[2]);
                    if (LIGHT && norm > 1e-12)
                        shade(a, cr, cg, cb, -g[0] / norm, -g[1] / norm, -g[2] / norm, -r.dx, -r.dy, -r.dz);
                    acc_r = cr;
                    acc_g = cg;
                    acc_b = cb;
                    acc_a = 1.0;
                    depth = t_hit;
                    break;
                }
                prev_s = s;
                prev_valid = true;
                // (not from a skippable sample taken as the first of a gap: the
                // reference skips the samples after it)
                if (chain_cull && !prev_skippable) {
                    // samples n+1 .. n+k-1 lie in the region of sample n, whose
                    // bound excludes the isovalue: no sign change, no hit
                    const int lvl = chain_transparent<kIso>(a, x, y, z);
                    if (lvl) {
                        const double p[3] = {x, y, z};
                        const int bidx[3] = {bi, bj, bk};
                        long long k = culled_run<SKIP, false>(a, r, inv, t0, n, t, p, bidx, rec,
                                                             lvl == 3 ? 4 : lvl == 1 ? 2 : 0);
                        if (k > N - n) k = N - n;
                        if (k > 1) {
                            n_taken += k - 1;
                            n += k;
                            prev_pending = true;
                            continue;
                        }
                    }
                }
            } else if (KIND == kPre) {
                // pre-classified (_kernels.py:471-507).  Culling: when every voxel
                // a sample in this cell (macro cell) can read has a zero alpha
                // plane, its interpolated alpha is exactly 0 -- nothing composited
                if (a.cull) {
                    const int lvl = pre_transparent(a, x, y, z);
                    if (lvl) {
                        const double p[3] = {x, y, z};
                        const int bidx[3] = {bi, bj, bk};
                        long long k = culled_run<SKIP>(a, r, inv, t0, n, t, p, bidx, rec, lvl);
                        if (k > N - n) k = N - n;
                        n_taken += k - 1;
                        n += k;
                        continue;
                    }
                }
                ++n_eval;
                double c4[4];
                attr_rgba4<CUBIC>(a, bi, bj, bk, x, y, z, c4);
                double sa = c4[3];
                if (sa > 0.0) {
                    double sr = c4[0], sg = c4[1], sb = c4[2];
                    double ahat = 1.0 - vr_pow(1.0 - sa, a.corr);
                    if (LIGHT) {
                        double g[3];
                        attr_grad<CUBIC>(a, x, y, z, bi, bj, bk, g);
                        n_shaded += 1;
                        double norm = sqrt((g[0] * g[0] + g[1] * g[1]) + g[2] * g[2]);
                        if (norm > 1e-12)
                            shade(a, sr, sg, sb, -g[0] / norm, -g[1] / norm, -g[2] / norm, -r.dx, -r.dy, -r.dz);
                    }
                    double w = (1.0 - acc_a) * ahat;
                    acc_r += w * sr;
                    acc_g += w * sg;
                    acc_b += w * sb;
                    acc_a += w;
                    if (acc_a >= a.term_alpha) break;
                }
            } else if (KIND == kPost) {
                // post-classified (_kernels.py:508-537)
                const int pt = cull ? provably_transparent<CUBIC>(a, x, y, z, first_vis, last_vis) : 0;
                if (pt) {
                    const double p[3] = {x, y, z};
                    const int bidx[3] = {bi, bj, bk};
                    long long k = culled_run<SKIP>(a, r, inv, t0, n, t, p, bidx, rec, pt == 3 ? 4 : pt == 1 ? 2 : 0);
                    if (k > N - n) k = N - n;
                    n_taken += k - 1;
                    n += k;
                    continue;
                }
                ++n_eval;
                double s = vol_sample<CUBIC>(a, bi, bj, bk, x, y, z);
                int sbin = lut_bin(s, a.lut_lo, a.lut_inv_w, a.nlut);
                double sa = __ldg(a.lut + 4 * sbin + 3);
                if (sa > 0.0) {
                    double sr = __ldg(a.lut + 4 * sbin), sg = __ldg(a.lut + 4 * sbin + 1), sb = __ldg(a.lut + 4 * sbin + 2);
                    double ahat = 1.0 - vr_pow(1.0 - sa, a.corr);
                    if (LIGHT) {
                        double g[3];
                        attr_grad<CUBIC>(a, x, y, z, bi, bj, bk, g);
                        n_shaded += 1;
                        double norm = sqrt((g[0] * g[0] + g[1] * g[1]) + g[2] * g[2]);
                        if (norm > 1e-12)
                            shade(a, sr, sg, sb, -g[0] / norm, -g[1] / norm, -g[2] / norm, -r.dx, -r.dy, -r.dz);
                    }
                    double w = (1.0 - acc_a) * ahat;
                    acc_r += w * sr;
                    acc_g += w * sg;
                    acc_b += w * sb;
                    acc_a += w;
                    if (acc_a >= a.term_alpha) break;
                }
            } else {
                // pre-integrated (_kernels.py:538-581)
                double s = vol_sample<CUBIC>(a, bi, bj, bk, x, y, z);
                if (!prev_valid && n > 0) {
                    double tp = t - step;
                    prev_s = attr_sample<CUBIC>(a, divide(r.ox + tp * r.dx, a.dsx), divide(r.oy + tp * r.dy, a.dsy),
                                                divide(r.oz + tp * r.dz, a.dsz));
                    prev_valid = true;
                }
                double sf = prev_valid ? prev_s : s;
                int fbin = lut_bin(sf, a.tbl_lo, a.tbl_inv_w, a.ntbl);
                int bbin = lut_bin(s, a.tbl_lo, a.tbl_inv_w, a.ntbl);
                const double *cell = a.table + 4 * ((long long)fbin * a.ntbl + bbin);
                double seg_a = __ldg(cell + 3);
                if (seg_a > 0.0) {
                    double seg_r = __ldg(cell), seg_g = __ldg(cell + 1), seg_b = __ldg(cell + 2);
                    if (LIGHT) {
                        double g[3];
                        attr_grad<CUBIC>(a, x, y, z, bi, bj, bk, g);
                        n_shaded += 1;
                        double norm = sqrt((g[0] * g[0] + g[1] * g[1]) + g[2] * g[2]);
                        if (norm > 1e-12) {
                            double ndl = fabs(((g[0] * -r.dx + g[1] * -r.dy) + g[2] * -r.dz) / norm);
                            double scale = a.ka + a.kd * ndl;
                            double spec = a.ks * vr_pow(ndl, a.shin) * seg_a;
                            seg_r = clampf(scale * seg_r + spec, 0.0, 1.0);
                            seg_g = clampf(scale * seg_g + spec, 0.0, 1.0);
                            seg_b = clampf(scale * seg_b + spec, 0.0, 1.0);
                        }
                    }
                    double w = 1.0 - acc_a;
                    acc_r += w * seg_r;
                    acc_g += w * seg_g;
                    acc_b += w * seg_b;
                    acc_a += w * seg_a;
                    if (acc_a >= a.term_alpha) break;
                }
                prev_s = s;
                prev_valid = true;
                if (chain_cull && !prev_skippable) {
                    // samples n+1 .. n+k-1 lie in the region of sample n, every
                    // segment between two of them has zero opacity
                    const int lvl = chain_transparent<kPreint>(a, x, y, z);
                    if (lvl) {
                        const double p[3] = {x, y, z};
                        const int bidx[3] = {bi, bj, bk};
                        long long k = culled_run<SKIP>(a, r, inv, t0, n, t, p, bidx, rec,
                                                       lvl == 3 ? 4 : lvl == 1 ? 2 : 0);
                        if (k > N - n) k = N - n;
                        if (k > 1) {
                            n_taken += k - 1;
                            n += k;
                            prev_pending = true;
                            continue;
                        }
                    }
                }
            }
            ++n;
        }
    }
    // composite over the background (_kernels.py:583-588)
    double w = 1.0 - acc_a;
    acc_r += w * a.bg[0] * a.bg[3];
    acc_g += w * a.bg[1] * a.bg[3];
    acc_b += w * a.bg[2] * a.bg[3];
    acc_a += w * a.bg[3];
    res.r = acc_r;
    res.g = acc_g;
    res.b = acc_b;
    res.a = acc_a;
    res.depth = depth;
    res.taken = n_taken;
    res.skipped = n_skip;
    res.shaded = n_shaded;
    res.eval = (KIND == kPost || KIND == kPre) ? n_eval : n_taken;
    res.iter = n_iter;
    return res;
}

// render.py:454-459: straight = premult / max(alpha, 1e-12) where alpha > 0,
// rint(clip(.,0,1) * 255) with round-half-even.
VR_D unsigned char to_u8(double v) { return (unsigned char)rint(clampf(v, 0.0, 1.0) * 255.0); }

// Sum over the (converged) warp with one REDUX; a lane's per-launch counts
// stay far below 2^32 (a lane handles at most a few hundred rays of at most a
// few thousand samples), the 64-bit totals accumulate in global atomics.
VR_D unsigned long long warp_sum(unsigned long long v) {
    return (unsigned long long)__reduce_add_sync(0xffffffffu, (unsigned)v);
}

template <int KIND, bool CUBIC, bool LIGHT, bool SKIP>
#ifndef VR_RAYCAST_MIN_BLOCKS
#define VR_RAYCAST_MIN_BLOCKS 1
#endif
__global__ void __launch_bounds__(kThreads, VR_RAYCAST_MIN_BLOCKS) raycast_kernel(const __grid_constant__ RenderArgs a) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int lx = (warp & 1) * 8 + (lane & 7);   // 0..15 inside the 16x8 cell
    const int ly = (warp >> 1) * 4 + (lane >> 3);  // 0..7; each warp an 8x4 tile
    const int local_view = (int)(blockIdx.x / (unsigned)a.slots);
    const int slot = (int)(blockIdx.x - (unsigned)local_view * (unsigned)a.slots);
    const int view = a.view0 + local_view;
    const int cell = a.il_n > 1 ? slot * a.il_n + a.il_k : slot;
    const int cx = (cell % a.cells_x) * kTileW + lx;
    const int cy = (cell / a.cells_x) * kTileH + ly;
    const bool active = cell < a.ncells && cx < a.tw && cy < a.th;
    unsigned long long taken = 0, skipped = 0, shaded = 0, evals = 0, iters = 0;
    if (active) {
        Ray r = make_ray(a, view_cam(a, view), a.tx + cx, a.ty + cy);
        double t0, t1;
        clip_to_bounds(r, a.ext_mm, t0, t1);
        RayResult res = march<KIND, CUBIC, LIGHT, SKIP>(
            a, r, t0, t1, a.blocks_hit ? a.blocks_hit + (long long)view * a.nblocks : nullptr);
        const long long p = (long long)view * a.view_pix +
                            (a.il_packed ? (long long)slot * (kTileW * kTileH) + ly * kTileW + lx
                                         : (long long)cy * a.tw + cx);
        if (a.premult) {
            double4 *o = reinterpret_cast<double4 *>(a.premult) + p;
            *o = make_double4(res.r, res.g, res.b, res.a);
        }
        if (a.pixels) {
            double alpha = res.a;
            double r0 = 0.0, g0 = 0.0, b0 = 0.0;
            if (alpha > 0.0) {
                double den = alpha > 1e-12 ? alpha : 1e-12;
                r0 = res.r / den;
                g0 = res.g / den;
                b0 = res.b / den;
            }
            reinterpret_cast<uchar4 *>(a.pixels)[p] = make_uchar4(to_u8(r0), to_u8(g0), to_u8(b0), to_u8(alpha));
        }
        if (a.depth) a.depth[p] = res.depth;
        if (a.taken) a.taken[p] = res.taken;
        if (a.skipped) a.skipped[p] = res.skipped;
        taken = (unsigned long long)res.taken;
        skipped = (unsigned long long)res.skipped;
        shaded = (unsigned long long)res.shaded;
        evals = (unsigned long long)res.eval;
        iters = (unsigned long long)res.iter;
    }
    taken = warp_sum(taken);
    skipped = warp_sum(skipped);
    if (lane == 0 && a.totals && (taken | skipped)) {
        atomicAdd(a.totals + 5 * (long long)view, taken);
        atomicAdd(a.totals + 5 * (long long)view + 1, skipped);
    }
    if (a.work) {
        shaded = warp_sum(shaded);
        evals = warp_sum(evals);
        iters = warp_sum(iters);
        if (lane == 0) {
            if (shaded) atomicAdd(a.work, shaded);
            if (evals) atomicAdd(a.work + 1, evals);
            if (iters) atomicAdd(a.work + 2, iters);
        }
    }
}

// ------------------------------------------------- persistent post-classified
// The headline path (post-classified DVR, _kernels.py:343-404, 508-537,
// 583-594) as a persistent kernel.  Ray cost is extremely uneven (a grazing
// ray near bone takes ~700 samples, most rays none), so one ray per thread
// leaves a warp's lanes idle behind its slowest ray.  Here every lane pulls
// rays from a global counter (work items in 8x4-tile order, so a warp's rays
// stay coherent) and takes the next one as soon as its ray ends.  Each trip a
// lane advances its ray by a bounded number of cheap steps -- skip-predicate
// leaps, culled runs -- until it needs an interpolation, then all lanes with
// pending work evaluate one interpolation together: the sample (stage 0) or
// one of the six gradient taps (stages 1..6, in the reference's
// +x,-x,+y,-y,+z,-z order).  Every sample's arithmetic is unchanged.

struct PostRay {
    Ray r;
    double inv[3];
    double t0;
    long long n, N;
    double acc_r, acc_g, acc_b, acc_a;
    double x, y, z;
    double sr, sg, sb, ahat, gplus, gx, gy, gz;
    long long taken, skipped;
    int bi, bj, bk;
    int stage;     // -1 none pending, 0 sample, 1..6 gradient taps
    int last_hit;
    int work;      // steps spent on this ray by this lane
    int nvis;      // samples composited so far
    long long out;  // output index of the pixel
    long long item; // work item (pixel) the ray came from
    int view;       // batched views: the view the item belongs to
    bool live;
};

#ifndef VR_PHASE_A_CAP
#define VR_PHASE_A_CAP 32  // swept 4..64: 32 best (C2 1656 -> 2279 fps vs 8; C3 +1 %)
#endif
constexpr int kPhaseACap = VR_PHASE_A_CAP;  // cheap steps a lane may take per trip
#ifndef VR_DENSE_BURST
#define VR_DENSE_BURST 64  // (C3-stress: 8 -> 31.9, 32 -> 38.2, 64 -> 39.0 fps)
#endif
constexpr int kDenseBurst = VR_DENSE_BURST;
#ifndef VR_COOP_GRAD
#define VR_COOP_GRAD 1  // lit per-lane kernel: a shaded sample's six gradient taps spread over its warp
#endif
constexpr bool kCoopGrad = VR_COOP_GRAD != 0;
#ifndef VR_CHAIN_COOP
#define VR_CHAIN_COOP 1  // chained per-lane kernel: cooperative gradients (pre-classified)
#endif
#ifndef VR_HEAVY_SMEM
#define VR_HEAVY_SMEM 7  // cooperative kernel, chunk exchange through shared memory: 1 scans, 2 tap positions, 4 tap values
#endif  // consecutive interpolated samples per trip (unlit, no skip)

// A long ray handed from the per-lane kernel to the warp-cooperative one:
// everything needed to continue it exactly where it stopped.
struct HeavyRay {
    long long item;
    long long n;
    double acc[4];
    long long taken, skipped;
    double o[3], d[3];  // the ray and its clipped sample range, so the
    double t0;          // cooperative kernel does not redo make_ray / clip
    long long N;
};
static_assert(sizeof(HeavyRay) == kHeavyRayBytes, "HeavyRay layout");

// Work item -> pixel.  Items are numbered view by view, then cell slot by cell
// slot, 128 per slot, each 32-item group one 8x4 warp tile (the layout of
// raycast_kernel).  (cx, cy) in the rectangle, the output index and the view;
// false for padding items
template <bool MV>
VR_D bool item_pixel(const RenderArgs &a, long long item, int &cx, int &cy, long long &out, int &view) {
    const int local_view = MV ? (int)(item / a.items_per_view) : 0;
    item -= (long long)local_view * a.items_per_view;
    view = MV ? a.view0 + local_view : 0;
    const int slot = (int)(item >> 7), local = (int)(item & 127);
    const int w = local >> 5, l = local & 31;
    const int lx = (w & 1) * 8 + (l & 7), ly = (w >> 1) * 4 + (l >> 3);
    int cell = a.il_n > 1 ? slot * a.il_n + a.il_k : slot;
    if (a.cell_order) cell = __ldg(a.cell_order + cell);  // centre-first visiting order
    cx = (cell % a.cells_x) * kTileW + lx;
    cy = (cell / a.cells_x) * kTileH + ly;
    out = (MV ? (long long)view * a.view_pix : 0ll) +
          (a.il_packed ? (long long)slot * (kTileW * kTileH) + ly * kTileW + lx : (long long)cy * a.tw + cx);
    return !(cell >= a.ncells || cx >= a.tw || cy >= a.th);
}

template <bool MV>
VR_D bool start_ray(const RenderArgs &a, long long item, PostRay &R) {
    int cx, cy;
    if (!item_pixel<MV>(a, item, cx, cy, R.out, R.view)) return false;
    R.r = make_ray(a, MV ? view_cam(a, R.view) : view_cam(a, 0), a.tx + cx, a.ty + cy);
    double t0, t1;
    clip_to_bounds(R.r, a.ext_mm, t0, t1);
    R.t0 = t0;
    R.N = 0;
    if (t1 >= t0) {
        long long nsteps = (long long)ceil(sdiv(t1 - t0, a.step));
        if (nsteps < 1) nsteps = 1;
        long long N = nsteps;
        while (N > 0 && (t0 + ((double)(N - 1) + 0.5) * a.step) > t1) --N;
        R.N = N;
    }
    R.inv[0] = R.r.dx != 0.0 ? sdiv(1.0, R.r.dx) : 0.0;
    R.inv[1] = R.r.dy != 0.0 ? sdiv(1.0, R.r.dy) : 0.0;
    R.inv[2] = R.r.dz != 0.0 ? sdiv(1.0, R.r.dz) : 0.0;
    R.n = 0;
    R.acc_r = R.acc_g = R.acc_b = R.acc_a = 0.0;
    R.taken = R.skipped = 0;
    R.stage = -1;
    R.last_hit = -1;
    R.work = 0;
    R.nvis = 0;
    R.item = item;
    R.live = true;
    return true;
}

// Background composite, straight-alpha uint8 epilogue and per-pixel outputs
// of a finished ray (_kernels.py:583-594, render.py:454-459).
VR_D void finish_ray(const RenderArgs &a, long long p, double acc_r, double acc_g, double acc_b, double acc_a,
                     long long taken, long long skipped) {
    const double w = 1.0 - acc_a;
    const double rr = acc_r + w * a.bg[0] * a.bg[3];
    const double gg = acc_g + w * a.bg[1] * a.bg[3];
    const double bb = acc_b + w * a.bg[2] * a.bg[3];
    const double aa = acc_a + w * a.bg[3];
    if (a.premult) reinterpret_cast<double4 *>(a.premult)[p] = make_double4(rr, gg, bb, aa);
    if (a.pixels) {
        double r0 = 0.0, g0 = 0.0, b0 = 0.0;
        if (aa > 0.0) {
            const double den = aa > 1e-12 ? aa : 1e-12;
            r0 = rr / den;
            g0 = gg / den;
            b0 = bb / den;
        }
        reinterpret_cast<uchar4 *>(a.pixels)[p] = make_uchar4(to_u8(r0), to_u8(g0), to_u8(b0), to_u8(aa));
    }
    if (a.depth) a.depth[p] = __longlong_as_double(0x7ff8000000000000LL);
    if (a.taken) a.taken[p] = taken;
    if (a.skipped) a.skipped[p] = skipped;
}

// MV: batched views (vr_render_views); the single-frame instantiation carries
// no per-view indexing in its hot loop
template <bool CUBIC, bool LIGHT, bool SKIP, bool MV>
#ifndef VR_POST_MIN_BLOCKS
#define VR_POST_MIN_BLOCKS 4  // <= 128 registers: 16 warps/SM (latency-bound; swept 1..5)
#endif
#ifndef VR_UNLIT_MIN_BLOCKS
#define VR_UNLIT_MIN_BLOCKS 5  // unlit: <= 96 registers, 20 warps/SM (C3-stress +4 % over 16; 24: -1 %)
#endif
__global__ void __launch_bounds__(kPersistThreads,
                                  (LIGHT ? VR_POST_MIN_BLOCKS : VR_UNLIT_MIN_BLOCKS) * (kThreads / kPersistThreads))
    raycast_post_kernel(const __grid_constant__ RenderArgs a) {
    pdl_enter();
#ifdef VR_DEBUG_STATS
    // rays finished here without / with taken samples (count, trip-steps), rays handed over (count, trip-steps)
    unsigned long long dbg[6] = {};
#endif
    const int lane = threadIdx.x & 31;
    const unsigned full = 0xffffffffu;
    const long long total = a.items_per_view * a.nviews;
#if VR_COOP_GRAD
    // (lit) per warp: positions of the samples being shaded this trip and
    // their gradient-tap values, spread over the warp's lanes
    constexpr int kW = kPersistThreads / 32;
    __shared__ double s_px[kW][32], s_py[kW][32], s_pz[kW][32];
    __shared__ int4 s_blk[kW][32];
    __shared__ double s_tap[kW][6 * 32];
    const int wib = threadIdx.x >> 5;
#endif
    const int nbx = a.L.nb[0], nby = a.L.nb[1];
    const int first_vis = a.cull ? __ldg(a.lut_range + 2) : INT_MIN;  // value thresholds (vlo, vhi)
    const int last_vis = a.cull ? __ldg(a.lut_range + 3) : INT_MAX;
    // a LUT whose first and last bins are visible can never prove a sample transparent
    const bool cull = a.cull != 0 && (first_vis > -32768 || last_vis < 32767);
    unsigned long long c_taken = 0, c_skip = 0, c_shaded = 0, c_eval = 0, c_iter = 0;
    ViewTotals vt;
    PostRay R;
    R.live = false;
    R.view = 0;
    bool exhausted = false;
    // no more rays than lanes (the grid is capped at one lane per ray)
    const bool starved = total <= (long long)gridDim.x * blockDim.x;
#ifdef VR_DEBUG_TIMES
    unsigned long long t_begin, t_drain = 0, n_trips_after = 0;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_begin));
    unsigned long long n_rays = 0;
#endif
    for (;;) {
        // ---- fetch rays for idle lanes (one atomic per warp)
        const bool want = !R.live && !exhausted;
        const unsigned m = __ballot_sync(full, want);
        if (m) {
            const int leader = __ffs(m) - 1;
            unsigned long long base = 0;
            if (lane == leader) base = atomicAdd(a.work_counter, (unsigned long long)__popc(m));
            base = __shfl_sync(full, base, leader);
            if (want) {
                const long long item = (long long)base + __popc(m & ((1u << lane) - 1u));
                if (item >= total)
                    exhausted = true;
                else
                    start_ray<MV>(a, item, R);
            }
        }
        if (__all_sync(full, !R.live && exhausted)) break;
        // the queue head is global: a warp whose lanes are all busy with long
        // rays must still learn that the queue has drained
        // (batched views: "drained" per view -- the queue has moved past this
        // ray's view, so it is one of that view's tail rays)
        bool drained;
        if (MV) {
            unsigned long long head = 0;
            if (lane == 0 && a.heavy) head = *reinterpret_cast<volatile unsigned long long *>(a.work_counter);
            head = __shfl_sync(full, head, 0);
            const unsigned long long view_end =
                (unsigned long long)(R.view - a.view0 + 1) * (unsigned long long)a.items_per_view;
            // (the vote first: the per-lane test below may differ across lanes)
            const bool any_exhausted = __any_sync(full, exhausted);
            drained = any_exhausted || (a.heavy && head >= view_end);
        } else {
            int head_done = 0;
            if (lane == 0 && a.heavy)
                head_done = *reinterpret_cast<volatile unsigned long long *>(a.work_counter) >= (unsigned long long)total;
            drained = __shfl_sync(full, head_done, 0) != 0 || __any_sync(full, exhausted);
        }
#ifdef VR_DEBUG_TIMES
        if (drained && t_drain == 0) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_drain));
        n_trips_after += drained ? 1 : 0;
#endif
        // (lit, cooperative gradients: idle lanes stay for the trip -- they
        // take gradient taps of the warp's shaded samples)
        if (!(kCoopGrad && LIGHT) && !R.live) continue;

        // ---- once the ray queue has drained, hand long rays to the
        // warp-cooperative kernel (at a clean point, nothing pending): the
        // frame would otherwise end with a few warps finishing grazing rays
        // of ~700 samples while every other SM idles.
        // A ray fetched as the queue drains first gets one trip here: most
        // rays end (or pass their long empty stretch) within it, cheaper than
        // a hand-off record and a warp's fetch (C3 +3 %, C2 +4 %).  A frame
        // with fewer rays than this kernel has lanes hands them over at once:
        // one lane per ray cannot fill the GPU (C1: 7,300 vs 2,900 frames/s).
        if (R.live && a.heavy && ((drained && (R.work > 0 || starved)) || R.work > a.heavy_after || (R.nvis >= a.heavy_vis && R.acc_a < a.heavy_vis_alpha)) &&
            R.work >= 0 && R.stage < 0 &&
            R.N - R.n >= a.heavy_min_left) {
            // long rays go to their own queue, which the cooperative kernel
            // drains first (longest work first shortens its tail)
            const bool lng = R.N - R.n >= a.heavy_long;
            const unsigned long long slot = atomicAdd(lng ? a.heavy_count_long : a.heavy_count, 1ull);
            if (slot < (unsigned long long)a.heavy_cap) {
                HeavyRay h;
                h.item = R.item;
                h.n = R.n;
                h.acc[0] = R.acc_r;
                h.acc[1] = R.acc_g;
                h.acc[2] = R.acc_b;
                h.acc[3] = R.acc_a;
                h.taken = R.taken;
                h.skipped = R.skipped;
                h.o[0] = R.r.ox;
                h.o[1] = R.r.oy;
                h.o[2] = R.r.oz;
                h.d[0] = R.r.dx;
                h.d[1] = R.r.dy;
                h.d[2] = R.r.dz;
                h.t0 = R.t0;
                h.N = R.N;
                static_cast<HeavyRay *>(a.heavy)[lng ? a.heavy_cap + slot : slot] = h;
                R.live = false;
#ifdef VR_DEBUG_STATS
                dbg[4] += 1;
                dbg[5] += (unsigned long long)R.work;
#endif
                if (!(kCoopGrad && LIGHT)) continue;
            } else {
                R.work = INT_MIN;  // queue full: keep it here
            }
        }

        // ---- phase A: cheap steps until an interpolation is needed
        int steps = 0;
        while (R.live && R.stage < 0 && R.n < R.N && steps < a.phase_cap) {
            ++steps;
            ++c_iter;
            const long long n = R.n;
            const double t = R.t0 + ((double)n + 0.5) * a.step;
            const double x = divide(R.r.ox + t * R.r.dx, a.dsx);
            const double y = divide(R.r.oy + t * R.r.dy, a.dsy);
            const double z = divide(R.r.oz + t * R.r.dz, a.dsz);
            const int bi = owner(a, 0, x), bj = owner(a, 1, y), bk = owner(a, 2, z);
            const int b = (bk * nby + bj) * nbx + bi;
            const double p[3] = {x, y, z};
            const int bidx[3] = {bi, bj, bk};
            BlockRec rec = {};
            if (SKIP) {
                rec = block_rec(a, b);
                const bool skippable = dvr_skippable(rec, x, y, z);
                const bool cell_only = rec.lo.w != 0.0f;
                if (skippable) {
                    long long k = leap_count<kPost>(a, R.r, R.inv, R.t0, n, t, p, bidx, rec, cell_only);
                    if (k > R.N - n) k = R.N - n;
                    R.skipped += k;
                    R.n = n + k;
                    continue;
                }
            }
            if (b != R.last_hit) {
                if (a.blocks_hit) a.blocks_hit[(MV ? (long long)R.view * a.nblocks : 0ll) + b] = 1;
                R.last_hit = b;
            }
            const int pt = cull ? provably_transparent<CUBIC>(a, x, y, z, first_vis, last_vis) : 0;
            if (pt) {
                long long k =
                    culled_run<SKIP>(a, R.r, R.inv, R.t0, n, t, p, bidx, rec, pt == 3 ? 4 : pt == 1 ? 2 : 0);
                if (k > R.N - n) k = R.N - n;
                R.taken += k;
                R.n = n + k;
                continue;
            }
            R.taken += 1;
            R.x = x;
            R.y = y;
            R.z = z;
            R.bi = bi;
            R.bj = bj;
            R.bk = bk;
            R.stage = 0;
        }

        // ---- phase B: one interpolation per lane with pending work
        bool finished = false;
#if VR_COOP_GRAD
        if (LIGHT) {
            // Cooperative gradients: the lanes whose sample turns out visible
            // get all six taps this trip, computed by the whole warp (32 taps
            // per round, as in the cooperative kernel) instead of one tap per
            // trip each: a shaded sample takes one trip, not seven, and every
            // lane of a tap round does useful work.
            __syncwarp();
            const bool need = R.live && R.stage == 0;
            if (__any_sync(full, need)) {
                bool shading = false;
                int ntaps = 0, rank = 0;
#pragma unroll 1
                for (int base = -32; base < ntaps; base += 32) {
                    double px = 0.0, py = 0.0, pz = 0.0;  // (idle lanes: a valid position)
                    int qi = 0, qj = 0, qk = 0;
                    const int id = base + lane;
                    const bool act = base < 0 ? need : id < ntaps;
                    if (base < 0) {
                        if (need) {
                            px = R.x;
                            py = R.y;
                            pz = R.z;
                            qi = R.bi;
                            qj = R.bj;
                            qk = R.bk;
                        }
                    } else if (act) {
                        const int k = id / 6, g = id - 6 * k;
                        px = s_px[wib][k];
                        py = s_py[wib][k];
                        pz = s_pz[wib][k];
                        const int4 q = s_blk[wib][k];
                        // tap g: +x, -x, +y, -y, +z, -z (_kernels.py:236-253)
                        const double hh = (g & 1) ? -0.5 : 0.5;
                        const int axis = g >> 1;
                        px = axis == 0 ? px + hh : px;
                        py = axis == 1 ? py + hh : py;
                        pz = axis == 2 ? pz + hh : pz;
                        const int o = owner(a, axis, axis == 0 ? px : axis == 1 ? py : pz);
                        qi = axis == 0 ? o : q.x;
                        qj = axis == 1 ? o : q.y;
                        qk = axis == 2 ? o : q.z;
                    }
                    const double v = vol_sample<CUBIC, VR_LIT_FUNNEL>(a, qi, qj, qk, px, py, pz);
                    if (base < 0) {
                        if (need) {
                            ++c_eval;
                            const int sbin = lut_bin(v, a.lut_lo, a.lut_inv_w, a.nlut);
                            const double sa = __ldg(a.lut + 4 * sbin + 3);
                            if (sa > 0.0) {
                                R.sr = __ldg(a.lut + 4 * sbin);
                                R.sg = __ldg(a.lut + 4 * sbin + 1);
                                R.sb = __ldg(a.lut + 4 * sbin + 2);
                                R.ahat = 1.0 - vr_pow(1.0 - sa, a.corr);
                                shading = true;
                            } else {
                                R.stage = -1;
                                R.n += 1;
                            }
                        }
                        const unsigned gm = __ballot_sync(full, shading);
                        ntaps = 6 * __popc(gm);
                        rank = __popc(gm & ((1u << lane) - 1u));
                        if (shading) {
                            s_px[wib][rank] = R.x;
                            s_py[wib][rank] = R.y;
                            s_pz[wib][rank] = R.z;
                            s_blk[wib][rank] = make_int4(R.bi, R.bj, R.bk, 0);
                        }
                        __syncwarp();
                    } else if (act) {
                        s_tap[wib][id] = v;
                    }
                }
                __syncwarp();
                if (shading) {
                    const double *tp = s_tap[wib] + 6 * rank;
                    const double gx = divide(tp[0] - tp[1], a.dsx), gy = divide(tp[2] - tp[3], a.dsy),
                                 gz = divide(tp[4] - tp[5], a.dsz);
                    ++c_shaded;
                    const double norm = sqrt((gx * gx + gy * gy) + gz * gz);
                    if (norm > 1e-12)
                        shade(a, R.sr, R.sg, R.sb, -gx / norm, -gy / norm, -gz / norm, -R.r.dx, -R.r.dy, -R.r.dz);
                    ++R.nvis;
                    const double w = (1.0 - R.acc_a) * R.ahat;
                    R.acc_r += w * R.sr;
                    R.acc_g += w * R.sg;
                    R.acc_b += w * R.sb;
                    R.acc_a += w;
                    R.stage = -1;
                    R.n += 1;
                    if (R.acc_a >= a.term_alpha) finished = true;  // early ray termination
                }
                __syncwarp();  // the shared arrays are refilled next trip
            }
        } else
#endif
        if (R.stage >= 0) {
            double px = R.x, py = R.y, pz = R.z;
            int qi = R.bi, qj = R.bj, qk = R.bk;
            if (LIGHT && R.stage > 0) {
                const int q = R.stage - 1;
                const double h = (q & 1) ? -0.5 : 0.5;
                if (q < 2) {
                    px = R.x + h;
                    qi = owner(a, 0, px);
                } else if (q < 4) {
                    py = R.y + h;
                    qj = owner(a, 1, py);
                } else {
                    pz = R.z + h;
                    qk = owner(a, 2, pz);
                }
            }
            const double v = vol_sample<CUBIC, !LIGHT || VR_LIT_FUNNEL>(a, qi, qj, qk, px, py, pz);
            c_eval += R.stage == 0;  // sample interpolations (gradient taps: 6 per shaded sample)
            bool composite = false;
            if (R.stage == 0) {
                const int sbin = lut_bin(v, a.lut_lo, a.lut_inv_w, a.nlut);
                const double sa = __ldg(a.lut + 4 * sbin + 3);
                if (sa > 0.0) {
                    R.sr = __ldg(a.lut + 4 * sbin);
                    R.sg = __ldg(a.lut + 4 * sbin + 1);
                    R.sb = __ldg(a.lut + 4 * sbin + 2);
                    R.ahat = 1.0 - vr_pow(1.0 - sa, a.corr);
                    if (LIGHT)
                        R.stage = 1;
                    else
                        composite = true;
                } else {
                    R.stage = -1;
                    R.n += 1;
                }
            } else {
                const int q = R.stage - 1;
                if (q & 1) {
                    const double dg = R.gplus - v;
                    if (q == 1) R.gx = dg;
                    else if (q == 3) R.gy = dg;
                    else R.gz = dg;
                } else {
                    R.gplus = v;
                }
                if (R.stage < 6) {
                    R.stage += 1;
                } else {
                    const double gx = divide(R.gx, a.dsx), gy = divide(R.gy, a.dsy), gz = divide(R.gz, a.dsz);
                    ++c_shaded;
                    const double norm = sqrt((gx * gx + gy * gy) + gz * gz);
                    if (norm > 1e-12)
                        shade(a, R.sr, R.sg, R.sb, -gx / norm, -gy / norm, -gz / norm, -R.r.dx, -R.r.dy, -R.r.dz);
                    composite = true;
                }
            }
            if (composite) {
                ++R.nvis;
                const double w = (1.0 - R.acc_a) * R.ahat;
                R.acc_r += w * R.sr;
                R.acc_g += w * R.sg;
                R.acc_b += w * R.sb;
                R.acc_a += w;
                R.stage = -1;
                R.n += 1;
                if (R.acc_a >= a.term_alpha) finished = true;  // early ray termination
            }
            // Dense burst (unlit, no skip predicate): once a sample needed its
            // interpolation, the following ones usually do too -- march them
            // here, consecutively, without a trip each (a trip's queue visit,
            // cheap-step phase and culling hierarchy cost as much as the
            // interpolation).  The burst stops at the first sample whose 4^3
            // cell is provably transparent, where the next trip's phase A
            // takes over with its culled runs; the samples are the
            // reference's (_kernels.py:508-537), in order.
            if (!LIGHT && !SKIP && !MV && !finished && R.stage < 0) {
                int burst = 0;
#pragma unroll 1
                while (burst < kDenseBurst && R.n < R.N) {
                    const long long n = R.n;
                    const double t = R.t0 + ((double)n + 0.5) * a.step;
                    const double x = divide(R.r.ox + t * R.r.dx, a.dsx);
                    const double y = divide(R.r.oy + t * R.r.dy, a.dsy);
                    const double z = divide(R.r.oz + t * R.r.dz, a.dsz);
                    if (cull && cell_transparent(a, x, y, z, first_vis, last_vis)) break;
                    const int bi = owner(a, 0, x), bj = owner(a, 1, y), bk = owner(a, 2, z);
                    const int b = (bk * nby + bj) * nbx + bi;
                    if (b != R.last_hit) {
                        if (a.blocks_hit) a.blocks_hit[b] = 1;
                        R.last_hit = b;
                    }
                    const double v = vol_sample<CUBIC, true>(a, bi, bj, bk, x, y, z);
                    ++burst;
                    R.taken += 1;
                    R.n = n + 1;
                    const int sbin = lut_bin(v, a.lut_lo, a.lut_inv_w, a.nlut);
                    const double sa = __ldg(a.lut + 4 * sbin + 3);
                    if (sa > 0.0) {
                        ++R.nvis;
                        const double ahat = 1.0 - vr_pow(1.0 - sa, a.corr);
                        const double w = (1.0 - R.acc_a) * ahat;
                        R.acc_r += w * __ldg(a.lut + 4 * sbin);
                        R.acc_g += w * __ldg(a.lut + 4 * sbin + 1);
                        R.acc_b += w * __ldg(a.lut + 4 * sbin + 2);
                        R.acc_a += w;
                        if (R.acc_a >= a.term_alpha) {  // early ray termination
                            finished = true;
                            break;
                        }
                    }
                }
                c_eval += burst;
                c_iter += burst;
                R.work += burst;
            }
        }
        if (R.live && R.stage < 0 && R.n >= R.N) finished = true;
        R.work += steps + 1;

        // ---- finish: background, epilogue, per-pixel outputs
        if (finished) {
            finish_ray(a, R.out, R.acc_r, R.acc_g, R.acc_b, R.acc_a, R.taken, R.skipped);
            if (MV) {
                vt.add(a, R.view, R.taken, R.skipped);
            } else {
                c_taken += (unsigned long long)R.taken;
                c_skip += (unsigned long long)R.skipped;
            }
            R.live = false;
#ifdef VR_DEBUG_STATS
            dbg[R.taken == 0 ? 0 : 2] += 1;
            dbg[R.taken == 0 ? 1 : 3] += (unsigned long long)R.work;
#endif
        }
    }
#ifdef VR_DEBUG_STATS
    if (a.debug_times)
        for (int i = 0; i < 6; ++i) atomicAdd(a.debug_times + 4 * 148 * 64 + 20 + i, dbg[i]);
#endif
#ifdef VR_DEBUG_TIMES
    if (a.debug_times) {
        unsigned long long t_end;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_end));
        const unsigned long long rays = warp_sum(c_iter ? 1ull : 0ull);
        if (lane == 0) {
            const long long w = (long long)blockIdx.x * (kPersistThreads / 32) + (threadIdx.x >> 5);
            unsigned sm;
            asm volatile("mov.u32 %0, %%smid;" : "=r"(sm));
            a.debug_times[4 * w] = t_begin;
            a.debug_times[4 * w + 1] = t_end;
            a.debug_times[4 * w + 2] = t_drain;
            a.debug_times[4 * w + 3] = n_trips_after;
            (void)sm;
            (void)rays;
        }
    }
#endif
    if (MV) {
        vt.flush_warp(a);
    } else {
        c_taken = warp_sum(c_taken);
        c_skip = warp_sum(c_skip);
        if (lane == 0 && a.totals && (c_taken | c_skip)) {
            atomicAdd(a.totals, c_taken);
            atomicAdd(a.totals + 1, c_skip);
        }
    }
    if (a.work) {
        c_shaded = warp_sum(c_shaded);
        c_eval = warp_sum(c_eval);
        c_iter = warp_sum(c_iter);
        if (lane == 0) {
            if (c_shaded) atomicAdd(a.work, c_shaded);
            if (c_eval) atomicAdd(a.work + 1, c_eval);
            if (c_iter) atomicAdd(a.work + 2, c_iter);
        }
    }
}

// --------------------------------------------- warp-cooperative long rays
// Continues the rays raycast_post_kernel handed over.  One warp owns one ray
// and walks it 32 consecutive samples at a time, one per lane: each lane
// evaluates its sample's exact skip predicate, transparency bound and, when
// needed, interpolation and classification (in parallel).  The opacity
// recurrence is then replayed in sample order -- every lane runs the same
// float64 updates on shuffled values -- to find the early-termination sample
// before any gradient is computed: at a bone surface a chunk is typically all
// visible while the ray terminates within a few samples, so gradients past
// that sample would be wasted.  The gradient taps of the samples up to it are
// spread over the lanes, and colours composited in order, so colour and
// counts are those of the sequential march.  Chunks with nothing to evaluate
// extend by the same provable leaps as the per-lane kernel, taken from the
// chunk's last sample.
// position of the k-th (0-based) set bit of m (k < popc(m))
VR_D int nth_bit(unsigned m, int k) {
    int pos = 0;
#pragma unroll
    for (int w = 16; w >= 1; w >>= 1) {
        const int c = __popc(m & ((1u << w) - 1u));
        if (k >= c) {
            k -= c;
            m >>= w;
            pos += w;
        }
    }
    return pos;
}

template <bool CUBIC, bool LIGHT, bool SKIP, bool MV>
#ifndef VR_HEAVY_MIN_BLOCKS
#define VR_HEAVY_MIN_BLOCKS 4  // <= 128 registers: 16 warps/SM (swept 3..8 with phase-A cap 32)
#endif
__global__ void __launch_bounds__(kPersistThreads, VR_HEAVY_MIN_BLOCKS *(kThreads / kPersistThreads))
    raycast_heavy_kernel(const __grid_constant__ RenderArgs a) {
    pdl_enter();
    const int lane = threadIdx.x & 31;
    const unsigned full = 0xffffffffu;
#if VR_HEAVY_SMEM
    // per warp: the chunk's sample opacities and premultiplied colours (read
    // in sample order by the serial scans, one broadcast load per sample
    // instead of shuffles) and the positions of its visible samples (read by
    // the lanes that take their gradient taps)
    constexpr int kW = kPersistThreads / 32;
    __shared__ double s_ahat[kW][32];
    __shared__ double4 s_col[kW][32];
#if VR_HEAVY_SMEM & 4
    __shared__ double s_tap[kW][6 * 32];
#endif
#if VR_HEAVY_SMEM & 2
    __shared__ double s_px[kW][32], s_py[kW][32], s_pz[kW][32];
    __shared__ int4 s_blk[kW][32];
#endif
    const int wib = threadIdx.x >> 5;
#endif
    const int nbx = a.L.nb[0], nby = a.L.nb[1];
    const int first_vis = a.cull ? __ldg(a.lut_range + 2) : INT_MIN;  // value thresholds (vlo, vhi)
    const int last_vis = a.cull ? __ldg(a.lut_range + 3) : INT_MAX;
    // a LUT whose first and last bins are visible can never prove a sample transparent
    const bool cull = a.cull != 0 && (first_vis > -32768 || last_vis < 32767);
    const unsigned long long pushed = *a.heavy_count, pushed_long = *a.heavy_count_long;
    const long long n_short = (long long)(pushed < (unsigned long long)a.heavy_cap ? pushed : a.heavy_cap);
    const long long n_long = (long long)(pushed_long < (unsigned long long)a.heavy_cap ? pushed_long : a.heavy_cap);
    const long long count = n_long + n_short;
    unsigned long long c_taken = 0, c_skip = 0, c_shaded = 0, c_eval = 0, c_iter = 0;
    ViewTotals vt;
#ifdef VR_DEBUG_TIMES
    unsigned long long t_begin, n_rays = 0;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_begin));
#endif
#ifdef VR_DEBUG_STATS
    // warp statistics (lane 0): chunks, chunks with candidates, candidates,
    // contributions, leaps, leapt samples, ET rays, rays, samples left at
    // hand-off, then a histogram of candidates per chunk: 0, 1-4, 5-16, 17-32
    unsigned long long st[18] = {};  // + histogram of visible samples per chunk: 1-2, 3-5, 6-10, 11-32
#endif
    for (;;) {
        unsigned long long idx = 0;
        if (lane == 0) idx = atomicAdd(a.heavy_head, 1ull);
        idx = __shfl_sync(full, idx, 0);
        if ((long long)idx >= count) break;
        // the long queue (stored after the short one) first
        const long long rec = (long long)idx < n_long ? a.heavy_cap + (long long)idx : (long long)idx - n_long;
        const HeavyRay h = static_cast<const HeavyRay *>(a.heavy)[rec];
        PostRay R;
        {
            int cx, cy;
            item_pixel<MV>(a, h.item, cx, cy, R.out, R.view);
        }
        uint8_t *hits = a.blocks_hit ? a.blocks_hit + (MV ? (long long)R.view * a.nblocks : 0ll) : nullptr;
        R.r.ox = h.o[0];
        R.r.oy = h.o[1];
        R.r.oz = h.o[2];
        R.r.dx = h.d[0];
        R.r.dy = h.d[1];
        R.r.dz = h.d[2];
        R.t0 = h.t0;
        R.N = h.N;
        R.inv[0] = R.r.dx != 0.0 ? 1.0 / R.r.dx : 0.0;  // as start_ray
        R.inv[1] = R.r.dy != 0.0 ? 1.0 / R.r.dy : 0.0;
        R.inv[2] = R.r.dz != 0.0 ? 1.0 / R.r.dz : 0.0;
        long long n = h.n;
        double acc_r = h.acc[0], acc_g = h.acc[1], acc_b = h.acc[2], acc_a = h.acc[3];
        long long taken = h.taken, skipped = h.skipped;
        while (n < R.N) {
            ++c_iter;
            const long long m = n + lane;
            const bool valid = m < R.N;
            bool skippable = false, cell_only = true, cand = false;
            int run_shift = -1;  // culled run leapable to the exit of a 2^run_shift cell (-1: none)
            double x = 0.0, y = 0.0, z = 0.0, t = 0.0;
            int bi = 0, bj = 0, bk = 0, b = 0;
            BlockRec rec = {};
            if (valid) {
                t = R.t0 + ((double)m + 0.5) * a.step;
                x = divide(R.r.ox + t * R.r.dx, a.dsx);
                y = divide(R.r.oy + t * R.r.dy, a.dsy);
                z = divide(R.r.oz + t * R.r.dz, a.dsz);
                bi = owner(a, 0, x);
                bj = owner(a, 1, y);
                bk = owner(a, 2, z);
                b = (bk * nby + bj) * nbx + bi;
                if (SKIP) {
                    rec = block_rec(a, b);
                    skippable = dvr_skippable(rec, x, y, z);
                    cell_only = rec.lo.w != 0.0f;
                }
                if (!skippable) {
                    const int pt = cull ? provably_transparent<CUBIC>(a, x, y, z, first_vis, last_vis) : 0;
                    cand = pt == 0;
                    run_shift = pt == 3 ? 4 : pt == 1 ? 2 : pt == 2 ? 0 : -1;
                }
            }
            // Evaluate the chunk.  Round 0 interpolates every candidate sample
            // on its own lane and classifies it.  Opacity alone decides early
            // termination, so the alpha recurrence is replayed right away (in
            // sample order, identically on every lane) to find the terminating
            // sample; only the visible samples up to it need a gradient.  Their
            // six taps each (+x,-x,+y,-y,+z,-z) are spread over the lanes, 32 per
            // round, and shuffled back to their sample's lane.  One loop body
            // keeps a single copy of the interpolant in the kernel.
            double sr = 0.0, sg = 0.0, sb = 0.0, ahat = 0.0;
            double tp[6] = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
            bool contrib = false;
            double wself = 0.0;  // compositing weight of this lane's sample
            unsigned vis = 0u;  // visible lanes up to the terminating sample
            int ntaps = 0, rank = 0, et_lane = 32;
            const bool any_cand = __any_sync(full, cand);
#pragma unroll 1
            for (int base = -32; any_cand && base < ntaps; base += 32) {
                bool act = cand;
                double px = x, py = y, pz = z;
                int qi = bi, qj = bj, qk = bk;
                if (base >= 0) {
                    const int id = base + lane;
                    act = id < ntaps;
                    const int k = id / 6, g = id - 6 * k;
#if VR_HEAVY_SMEM & 2
                    if (act) {  // (inactive lanes interpolate at their own position)
                        px = s_px[wib][k];
                        py = s_py[wib][k];
                        pz = s_pz[wib][k];
                        const int4 q = s_blk[wib][k];
                        qi = q.x;
                        qj = q.y;
                        qk = q.z;
                    }
#else
                    const int src = act ? nth_bit(vis, k) : lane;
                    px = __shfl_sync(full, x, src);
                    py = __shfl_sync(full, y, src);
                    pz = __shfl_sync(full, z, src);
                    qi = __shfl_sync(full, bi, src);
                    qj = __shfl_sync(full, bj, src);
                    qk = __shfl_sync(full, bk, src);
#endif
                    // branch-free: lanes of a round take different taps, and a
                    // divergent branch here lets the compiler split the warp
                    const double hh = (g & 1) ? -0.5 : 0.5;
                    const int axis = g >> 1;
                    px = axis == 0 ? px + hh : px;
                    py = axis == 1 ? py + hh : py;
                    pz = axis == 2 ? pz + hh : pz;
                    const int o = owner(a, axis, axis == 0 ? px : axis == 1 ? py : pz);
                    qi = axis == 0 ? o : qi;
                    qj = axis == 1 ? o : qj;
                    qk = axis == 2 ? o : qk;
                }
                // every lane interpolates (inactive lanes at a valid position):
                // no divergent branch around the interpolant
                const double v = vol_sample<CUBIC>(a, qi, qj, qk, px, py, pz);
                if (base < 0) {
                    if (act) {
                        const int sbin = lut_bin(v, a.lut_lo, a.lut_inv_w, a.nlut);
                        const double sa = __ldg(a.lut + 4 * sbin + 3);
                        if (sa > 0.0) {  // else transparent: nothing to composite
                            contrib = true;
                            sr = __ldg(a.lut + 4 * sbin);
                            sg = __ldg(a.lut + 4 * sbin + 1);
                            sb = __ldg(a.lut + 4 * sbin + 2);
                            ahat = 1.0 - vr_pow(1.0 - sa, a.corr);
                        }
                    }
                    // the terminating sample (_kernels.py:531-537: A += (1 - A) * a)
                    unsigned cm = __ballot_sync(full, contrib);
                    double A = acc_a;
#if VR_HEAVY_SMEM
                    s_ahat[wib][lane] = ahat;
                    __syncwarp();
#endif
                    while (cm) {
                        const int src = __ffs(cm) - 1;
                        cm &= cm - 1;
#if VR_HEAVY_SMEM
                        const double w = (1.0 - A) * s_ahat[wib][src];
#else
                        const double w = (1.0 - A) * __shfl_sync(full, ahat, src);
#endif
                        if (lane == src) wself = w;  // this sample's weight, reused by the composite
                        A += w;
                        if (A >= a.term_alpha) {
                            et_lane = src;
                            break;
                        }
                    }
                    if (LIGHT) {
                        const unsigned upto = et_lane >= 31 ? full : ((2u << et_lane) - 1u);
                        vis = __ballot_sync(full, contrib) & upto;
                        ntaps = 6 * __popc(vis);
                        rank = __popc(vis & ((1u << lane) - 1u));
#if VR_HEAVY_SMEM & 2
                        if ((vis >> lane) & 1u) {
                            s_px[wib][rank] = x;
                            s_py[wib][rank] = y;
                            s_pz[wib][rank] = z;
                            s_blk[wib][rank] = make_int4(bi, bj, bk, 0);
                        }
                        __syncwarp();
#endif
                    }
                } else {
#if VR_HEAVY_SMEM & 4
                    if (act) s_tap[wib][base + lane] = v;
#else
#pragma unroll
                    for (int g = 0; g < 6; ++g) {
                        const int s = 6 * rank + g - base;
                        const double w = __shfl_sync(full, v, s & 31);
                        if (s >= 0 && s < 32) tp[g] = w;
                    }
#endif
                }
            }
#if VR_HEAVY_SMEM & 4
            if (LIGHT && ntaps) {
                __syncwarp();
                if ((vis >> lane) & 1u) {
#pragma unroll
                    for (int g = 0; g < 6; ++g) tp[g] = s_tap[wib][6 * rank + g];
                }
            }
#endif
            if (LIGHT && ((vis >> lane) & 1u)) {
                const double gx = divide(tp[0] - tp[1], a.dsx);
                const double gy = divide(tp[2] - tp[3], a.dsy);
                const double gz = divide(tp[4] - tp[5], a.dsz);
                const double norm = sqrt((gx * gx + gy * gy) + gz * gz);
                if (norm > 1e-12)
                    shade(a, sr, sg, sb, -gx / norm, -gy / norm, -gz / norm, -R.r.dx, -R.r.dy, -R.r.dz);
            }
            // composite up to the terminating sample, in sample order,
            // identically on every lane (_kernels.py:531-537)
            {
                const unsigned upto = et_lane >= 31 ? full : ((2u << et_lane) - 1u);
                unsigned cm = __ballot_sync(full, contrib) & upto;
#if VR_HEAVY_SMEM
                // each lane's products w * colour (the reference's products,
                // formed in parallel); only the sums run in sample order.
                // w == (1 - acc_a) * ahat: the same operations on the same
                // values as in the termination scan above
                __syncwarp();
                s_col[wib][lane] = make_double4(wself * sr, wself * sg, wself * sb, wself);
                __syncwarp();
                while (cm) {
                    const int src = __ffs(cm) - 1;
                    cm &= cm - 1;
                    const double4 c = s_col[wib][src];
                    acc_r += c.x;
                    acc_g += c.y;
                    acc_b += c.z;
                    acc_a += c.w;
                }
                __syncwarp();
#else
                while (cm) {
                    const int src = __ffs(cm) - 1;
                    cm &= cm - 1;
                    const double r_ = __shfl_sync(full, sr, src), g_ = __shfl_sync(full, sg, src);
                    const double b_ = __shfl_sync(full, sb, src);
                    // == (1 - acc_a) * ahat: the same operations on the same
                    // values as in the termination scan above
                    const double w = __shfl_sync(full, wself, src);
                    acc_r += w * r_;
                    acc_g += w * g_;
                    acc_b += w * b_;
                    acc_a += w;
                }
#endif
            }
            // counts up to and including the terminating sample
            const unsigned upto = et_lane >= 31 ? full : ((2u << et_lane) - 1u);
            const bool is_taken = valid && !skippable;
            const unsigned tmask = __ballot_sync(full, is_taken) & upto;
            const unsigned smask = __ballot_sync(full, valid && skippable) & upto;
            taken += __popc(tmask);
            skipped += __popc(smask);
            // work the sequential march would do (lanes past the terminating
            // sample were evaluated speculatively and are not counted)
            const unsigned emask = __ballot_sync(full, cand) & upto;
            const unsigned cmask = __ballot_sync(full, contrib) & upto;
            if (lane == 0) {
                c_eval += __popc(emask);
                if (LIGHT) c_shaded += __popc(cmask);
            }
#ifdef VR_DEBUG_STATS
            {
                const int nc = __popc(__ballot_sync(full, cand));
                st[0] += 1;
                st[1] += nc > 0;
                st[2] += nc;
                st[3] += __popc(cmask);
                st[nc == 0 ? 10 : nc <= 4 ? 11 : nc <= 16 ? 12 : 13] += 1;
                const int nv = __popc(__ballot_sync(full, contrib));
                if (nv) st[nv <= 2 ? 14 : nv <= 5 ? 15 : nv <= 10 ? 16 : 17] += 1;
                if (et_lane < 32) st[6] += 1;
            }
#endif
            if (is_taken && lane <= et_lane && hits) hits[b] = 1;
            if (et_lane < 32) break;
            // advance; a chunk with nothing to evaluate extends by a provable run
            long long next = n + 32;
            if (!any_cand && n + 31 < R.N) {
                long long k = 1;
                if (lane == 31) {
                    const double p[3] = {x, y, z};
                    const int bidx[3] = {bi, bj, bk};
                    k = skippable ? leap_count<kPost>(a, R.r, R.inv, R.t0, m, t, p, bidx, rec, cell_only)
                        : run_shift >= 0 ? culled_run<SKIP>(a, R.r, R.inv, R.t0, m, t, p, bidx, rec, run_shift)
                                   : 1;
                }
                k = __shfl_sync(full, k, 31);
                const bool last_skip = __shfl_sync(full, skippable, 31);
                const long long last = n + 31;
                if (k > R.N - last) k = R.N - last;
                if (k > 1) {
                    if (last_skip)
                        skipped += k - 1;
                    else
                        taken += k - 1;
                    next = last + k;
#ifdef VR_DEBUG_STATS
                    st[4] += 1;
                    st[5] += k - 1;
#endif
                }
            }
            n = next;
        }
        if (lane == 0) {
            finish_ray(a, R.out, acc_r, acc_g, acc_b, acc_a, taken, skipped);
            if (MV) {
                vt.add(a, R.view, taken, skipped);
            } else {
                c_taken += (unsigned long long)taken;
                c_skip += (unsigned long long)skipped;
            }
        }
#ifdef VR_DEBUG_TIMES
        ++n_rays;
#endif
#ifdef VR_DEBUG_STATS
        st[7] += 1;
        st[8] += (unsigned long long)(R.N - h.n);
#endif
    }
#ifdef VR_DEBUG_STATS
    if (a.debug_times && lane == 0)
        for (int i = 0; i < 18; ++i) atomicAdd(a.debug_times + 4 * 148 * 64 + i, st[i]);
#endif
#ifdef VR_DEBUG_TIMES
    if (a.debug_times && lane == 0) {
        unsigned long long t_end;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_end));
        const long long w = 148 * 32 + (long long)blockIdx.x * (kPersistThreads / 32) + (threadIdx.x >> 5);
        a.debug_times[4 * w] = t_begin;
        a.debug_times[4 * w + 1] = t_end;
        a.debug_times[4 * w + 2] = count;  // rays handed over
        a.debug_times[4 * w + 3] = n_rays;
    }
#endif
    if (MV) {
        vt.flush_warp(a);
    } else {
        c_taken = warp_sum(c_taken);
        c_skip = warp_sum(c_skip);
        if (lane == 0 && a.totals && (c_taken | c_skip)) {
            atomicAdd(a.totals, c_taken);
            atomicAdd(a.totals + 1, c_skip);
        }
    }
    if (a.work) {
        c_shaded = warp_sum(c_shaded);
        c_eval = warp_sum(c_eval);
        c_iter = warp_sum(c_iter);
        if (lane == 0) {
            if (c_shaded) atomicAdd(a.work, c_shaded);
            if (c_eval) atomicAdd(a.work + 1, c_eval);
            if (c_iter) atomicAdd(a.work + 2, c_iter);
        }
    }
}

// ---------------------------------------- persistent chained modes (iso, preint)
// The isosurface and pre-integrated modes (_kernels.py:405-468, 538-581) on
// the persistent scheduler: every lane pulls rays from the global queue (as
// raycast_post_kernel) and advances its ray by trips -- cheap steps (skip
// leaps) until an interpolation is needed, then ONE interpolation per trip,
// whatever it is for: the sample itself, the previous sample (after a gap,
// at t - step, as the reference re-evaluates it; after a culled run, at its
// own position), one of the 8 bisection points of an iso crossing, or one of
// the 6 gradient taps.  The lanes of a warp stay on one instruction stream
// while their rays are at different places, and a lane whose ray ends takes
// the next ray at once.  After each evaluated sample, a run of samples whose
// interpolant bound rules out any contribution (chain_transparent) is
// counted as taken and leapt over, exactly as raycast_kernel does.
enum ChainStage { kcNone = -1, kcSample = 0, kcPrevExact = 1, kcPrevGap = 2, kcBisect = 3, kcGrad = 11 };

// A chained-mode ray handed to the cooperative kernel: everything needed to
// continue it exactly where it stopped.
struct ChainRec {
    long long out, n, N;
    double t0;
    double o[3], d[3];
    double acc[4];
    long long taken, skipped;
    double prev_s;
    int flags;  // 1 prev_valid, 2 prev_pending (previous sample culled), 4 prev_skippable
    int pad;
};
static_assert(sizeof(ChainRec) == kChainRecBytes, "ChainRec layout");

struct ChainRay {
    Ray r;
    double inv[3];
    double t0;
    long long n, N;
    double acc_r, acc_g, acc_b, acc_a;
    double x, y, z, t;      // the current sample
    double prev_s, s;
    double lo_t, hi_t, lo_s, t_hit;  // iso bisection
    double hx, hy, hz;      // gradient centre
    double cr, cg, cb, ca;  // colour pending composite (iso: LUT colour; preint: segment)
    double gplus, gx, gy, gz;
    long long taken, skipped;
    long long out;
    int bi, bj, bk, hbi, hbj, hbk;
    int stage;
    int last_hit;
    int nvis;  // samples composited so far (dense-ray hand-off)
    bool prev_valid, prev_pending, prev_skippable, live;
};

template <int KIND, bool CUBIC, bool LIGHT, bool SKIP>
#ifndef VR_CHAIN_MIN_BLOCKS
#define VR_CHAIN_MIN_BLOCKS 4
#endif
__global__ void __launch_bounds__(kPersistThreads, VR_CHAIN_MIN_BLOCKS *(kThreads / kPersistThreads))
    raycast_chain_kernel(const __grid_constant__ RenderArgs a) {
    const int lane = threadIdx.x & 31;
    const unsigned full = 0xffffffffu;
    const long long total = a.items_per_view;
    const int nbx = a.L.nb[0], nby = a.L.nb[1];
    const bool chain_cull = a.cull != 0;
    unsigned long long c_taken = 0, c_skip = 0, c_shaded = 0, c_eval = 0, c_iter = 0;
    ChainRay R;
    R.live = false;
    bool exhausted = false;
#if VR_CHAIN_COOP
    constexpr int kW = kPersistThreads / 32;
    __shared__ double s_px[kW][32], s_py[kW][32], s_pz[kW][32];
    __shared__ int4 s_blk[kW][32];
    __shared__ double s_tap[kW][6 * 32];
    const int wib = threadIdx.x >> 5;
    // (pre-classified only: iso and pre-integrated measured slower with it,
    // their kernels spill more)
    constexpr bool coop = LIGHT && KIND == kPre;
#else
    constexpr bool coop = false;
#endif
    for (;;) {
        // ---- fetch rays for idle lanes (one atomic per warp)
        const bool want = !R.live && !exhausted;
        const unsigned m = __ballot_sync(full, want);
        if (m) {
            const int leader = __ffs(m) - 1;
            unsigned long long base = 0;
            if (lane == leader) base = atomicAdd(a.work_counter, (unsigned long long)__popc(m));
            base = __shfl_sync(full, base, leader);
            if (want) {
                const long long item = (long long)base + __popc(m & ((1u << lane) - 1u));
                int cx, cy, view;
                if (item >= total) {
                    exhausted = true;
                } else if (item_pixel<false>(a, item, cx, cy, R.out, view)) {
                    R.r = make_ray(a, view_cam(a, 0), a.tx + cx, a.ty + cy);
                    double t0, t1;
                    clip_to_bounds(R.r, a.ext_mm, t0, t1);
                    R.t0 = t0;
                    R.N = 0;
                    if (t1 >= t0) {
                        long long nsteps = (long long)ceil((t1 - t0) / a.step);
                        if (nsteps < 1) nsteps = 1;
                        long long N = nsteps;
                        while (N > 0 && (t0 + ((double)(N - 1) + 0.5) * a.step) > t1) --N;
                        R.N = N;
                    }
                    R.inv[0] = R.r.dx != 0.0 ? 1.0 / R.r.dx : 0.0;
                    R.inv[1] = R.r.dy != 0.0 ? 1.0 / R.r.dy : 0.0;
                    R.inv[2] = R.r.dz != 0.0 ? 1.0 / R.r.dz : 0.0;
                    R.n = 0;
                    R.acc_r = R.acc_g = R.acc_b = R.acc_a = 0.0;
                    R.taken = R.skipped = 0;
                    R.prev_s = 0.0;
                    R.prev_valid = R.prev_pending = R.prev_skippable = false;
                    R.t_hit = __longlong_as_double(0x7ff8000000000000LL);  // NaN: no hit
                    R.stage = kcNone;
                    R.last_hit = -1;
                    R.nvis = 0;
                    R.live = true;
                }
            }
        }
        if (__all_sync(full, !R.live && exhausted)) break;
        // the queue head is global: a warp whose lanes are all busy must still
        // learn that it has drained
        int head_done = 0;
        if (lane == 0 && a.heavy)
            head_done = *reinterpret_cast<volatile unsigned long long *>(a.work_counter) >= (unsigned long long)total;
        const bool drained = __shfl_sync(full, head_done, 0) != 0 || __any_sync(full, exhausted);
        if (!coop && !R.live) continue;

        // ---- once the queue has drained, long rays go to the cooperative
        // kernel at a clean point (the frame would otherwise end with a few
        // lanes walking long rays alone)
        // (dense lit rays -- several composited samples, still far from
        // termination -- go at once: the cooperative kernel spreads their
        // gradient taps over the warp)
        if (R.live && a.heavy && R.stage == kcNone && R.N - R.n >= a.heavy_min_left &&
            (drained || (R.nvis >= a.heavy_vis && R.acc_a < a.heavy_vis_alpha))) {
            const unsigned long long slot = atomicAdd(a.heavy_count, 1ull);
            if (slot < (unsigned long long)a.heavy_cap) {
                ChainRec h;
                h.out = R.out;
                h.n = R.n;
                h.N = R.N;
                h.t0 = R.t0;
                h.o[0] = R.r.ox;
                h.o[1] = R.r.oy;
                h.o[2] = R.r.oz;
                h.d[0] = R.r.dx;
                h.d[1] = R.r.dy;
                h.d[2] = R.r.dz;
                h.acc[0] = R.acc_r;
                h.acc[1] = R.acc_g;
                h.acc[2] = R.acc_b;
                h.acc[3] = R.acc_a;
                h.taken = R.taken;
                h.skipped = R.skipped;
                h.prev_s = R.prev_s;
                h.flags = (R.prev_valid ? 1 : 0) | (R.prev_pending ? 2 : 0) | (R.prev_skippable ? 4 : 0);
                static_cast<ChainRec *>(a.heavy)[slot] = h;
                R.live = false;
                if (!coop) continue;
            }
        }

        // ---- phase A: skip leaps until a taken sample needs an interpolation
        int steps = 0;
        while (R.live && R.stage == kcNone && R.n < R.N && steps < kPhaseACap) {
            ++steps;
            ++c_iter;
            const long long n = R.n;
            const double t = R.t0 + ((double)n + 0.5) * a.step;
            const double x = divide(R.r.ox + t * R.r.dx, a.dsx);
            const double y = divide(R.r.oy + t * R.r.dy, a.dsy);
            const double z = divide(R.r.oz + t * R.r.dz, a.dsz);
            const int bi = owner(a, 0, x), bj = owner(a, 1, y), bk = owner(a, 2, z);
            const int b = (bk * nby + bj) * nbx + bi;
            BlockRec rec = {};
            if (SKIP) {
                bool skippable, cell_only = true;
                if (KIND == kIso) {
                    skippable = (double)__ldg(a.vmax + b) < a.isovalue || (double)__ldg(a.vmin + b) > a.isovalue;
                } else {
                    rec = block_rec(a, b);
                    skippable = dvr_skippable(rec, x, y, z);
                    cell_only = rec.lo.w != 0.0f;
                }
                // chained modes take the first sample of a gap; pre skips every skippable sample
                if (skippable && (KIND == kPre || R.prev_skippable)) {
                    const double p[3] = {x, y, z};
                    const int bidx[3] = {bi, bj, bk};
                    long long k = leap_count<KIND>(a, R.r, R.inv, R.t0, n, t, p, bidx, rec, cell_only);
                    if (k > R.N - n) k = R.N - n;
                    R.skipped += k;
                    R.n = n + k;
                    R.prev_valid = false;
                    R.prev_pending = false;
                    continue;
                }
                R.prev_skippable = skippable;
            }
            if (b != R.last_hit) {
                if (a.blocks_hit) a.blocks_hit[b] = 1;
                R.last_hit = b;
            }
            R.taken += 1;
            if (KIND == kPre && chain_cull) {
                // every voxel a sample in this (macro) cell can read has a zero
                // alpha plane: its interpolated alpha is exactly 0
                const int lvl = pre_transparent(a, x, y, z);
                if (lvl) {
                    const double p[3] = {x, y, z};
                    const int bidx[3] = {bi, bj, bk};
                    long long k = culled_run<SKIP>(a, R.r, R.inv, R.t0, n, t, p, bidx, rec, lvl);
                    if (k > R.N - n) k = R.N - n;
                    if (k < 1) k = 1;
                    R.taken += k - 1;
                    R.n = n + k;
                    continue;
                }
            }
            if (KIND == kIso && chain_cull && !R.prev_pending && (R.prev_valid || n == 0)) {
                // A sample whose region bound excludes the isovalue needs no
                // interpolation: only the sign of s - iso is ever used (the
                // crossing test, the bisection bracket), and the bound's end
                // nearest the isovalue has it.  No crossing into it: the whole
                // run in the region is hit-free; a crossing: bisect.
                short2 bd;
                if (chain_transparent<kIso>(a, x, y, z, &bd)) {
                    const double stand = (double)bd.x > a.isovalue ? (double)bd.x : (double)bd.y;
                    if (R.prev_valid && (R.prev_s - a.isovalue) * (stand - a.isovalue) < 0.0) {
                        R.lo_t = t - a.step;
                        R.hi_t = t;
                        R.lo_s = R.prev_s;
                        R.stage = kcBisect;
                        break;
                    }
                    long long k = 1;
                    if (!R.prev_skippable) {
                        const double p[3] = {x, y, z};
                        const int bidx[3] = {bi, bj, bk};
                        const BlockRec rec = {};
                        const int lvl = chain_transparent<kIso>(a, x, y, z);
                        k = culled_run<SKIP, false>(a, R.r, R.inv, R.t0, n, t, p, bidx, rec,
                                                    lvl == 3 ? 4 : lvl == 1 ? 2 : 0);
                        if (k > R.N - n) k = R.N - n;
                        if (k < 1) k = 1;
                    }
                    R.taken += k - 1;
                    R.n = n + k;
                    R.prev_s = stand;
                    R.prev_valid = true;
                    continue;
                }
            }
            R.x = x;
            R.y = y;
            R.z = z;
            R.t = t;
            R.bi = bi;
            R.bj = bj;
            R.bk = bk;
            R.stage = KIND == kPre ? kcSample
                                   : (R.prev_pending ? kcPrevExact : ((!R.prev_valid && n > 0) ? kcPrevGap : kcSample));
        }

        // ---- phase B: one interpolation
        bool finished = false;
        auto gradient_done = [&](double dgx, double dgy, double dgz) {
            const double gx = divide(dgx, a.dsx), gy = divide(dgy, a.dsy), gz = divide(dgz, a.dsz);
            ++c_shaded;
            const double norm = sqrt((gx * gx + gy * gy) + gz * gz);
            if (KIND == kPre) {
                double sr = R.cr, sg = R.cg, sb = R.cb;
                if (norm > 1e-12) shade(a, sr, sg, sb, -gx / norm, -gy / norm, -gz / norm, -R.r.dx, -R.r.dy, -R.r.dz);
                const double w = (1.0 - R.acc_a) * R.ca;
                R.acc_r += w * sr;
                R.acc_g += w * sg;
                R.acc_b += w * sb;
                R.acc_a += w;
                ++R.nvis;
                R.stage = kcNone;
                R.n += 1;
                if (R.acc_a >= a.term_alpha) finished = true;
            } else if (KIND == kIso) {
                const int ib = lut_bin(a.isovalue, a.lut_lo, a.lut_inv_w, a.nlut);
                double cr = __ldg(a.lut + 4 * ib), cg = __ldg(a.lut + 4 * ib + 1), cb = __ldg(a.lut + 4 * ib + 2);
                if (LIGHT && norm > 1e-12)
                    shade(a, cr, cg, cb, -gx / norm, -gy / norm, -gz / norm, -R.r.dx, -R.r.dy, -R.r.dz);
                R.acc_r = cr;
                R.acc_g = cg;
                R.acc_b = cb;
                R.acc_a = 1.0;
                finished = true;
            } else {
                double seg_r = R.cr, seg_g = R.cg, seg_b = R.cb;
                const double seg_a = R.ca;
                if (norm > 1e-12) {
                    const double ndl = fabs(((gx * -R.r.dx + gy * -R.r.dy) + gz * -R.r.dz) / norm);
                    const double scale = a.ka + a.kd * ndl;
                    const double spec = a.ks * vr_pow(ndl, a.shin) * seg_a;
                    seg_r = clampf(scale * seg_r + spec, 0.0, 1.0);
                    seg_g = clampf(scale * seg_g + spec, 0.0, 1.0);
                    seg_b = clampf(scale * seg_b + spec, 0.0, 1.0);
                }
                const double w = 1.0 - R.acc_a;
                R.acc_r += w * seg_r;
                R.acc_g += w * seg_g;
                R.acc_b += w * seg_b;
                R.acc_a += w * seg_a;
                ++R.nvis;
                if (R.acc_a >= a.term_alpha) {
                    finished = true;
                } else {
                    R.prev_s = R.s;
                    R.prev_valid = true;
                    R.stage = kcNone;
                    R.n += 1;
                }
            }
        };
        if (R.live && R.stage != kcNone && !(coop && R.stage >= kcGrad)) {
            double px = R.x, py = R.y, pz = R.z;
            int qi = R.bi, qj = R.bj, qk = R.bk;
            bool own = false;  // position not attributed yet (owner from the position)
            if (R.stage == kcPrevExact || R.stage == kcPrevGap) {
                const double tq = R.stage == kcPrevExact ? R.t0 + ((double)(R.n - 1) + 0.5) * a.step : R.t - a.step;
                px = divide(R.r.ox + tq * R.r.dx, a.dsx);
                py = divide(R.r.oy + tq * R.r.dy, a.dsy);
                pz = divide(R.r.oz + tq * R.r.dz, a.dsz);
                own = true;
            } else if (KIND == kIso && R.stage >= kcBisect && R.stage < kcGrad) {
                const double mid = 0.5 * (R.lo_t + R.hi_t);
                px = divide(R.r.ox + mid * R.r.dx, a.dsx);
                py = divide(R.r.oy + mid * R.r.dy, a.dsy);
                pz = divide(R.r.oz + mid * R.r.dz, a.dsz);
                own = true;
            } else if (R.stage >= kcGrad) {
                const int q = R.stage - kcGrad;
                const double h = (q & 1) ? -0.5 : 0.5;
                px = R.hx;
                py = R.hy;
                pz = R.hz;
                qi = R.hbi;
                qj = R.hbj;
                qk = R.hbk;
                if (q < 2) {
                    px = R.hx + h;
                    qi = owner(a, 0, px);
                } else if (q < 4) {
                    py = R.hy + h;
                    qj = owner(a, 1, py);
                } else {
                    pz = R.hz + h;
                    qk = owner(a, 2, pz);
                }
            }
            if (own) {
                qi = owner(a, 0, px);
                qj = owner(a, 1, py);
                qk = owner(a, 2, pz);
            }
            double v = 0.0;
            double c4[4] = {0.0, 0.0, 0.0, 0.0};
            if (KIND == kPre && R.stage == kcSample) {
                // the pre-classified channels (_attr_rgba, _kernels.py:256-276), all four at once
                attr_rgba4<CUBIC>(a, R.bi, R.bj, R.bk, R.x, R.y, R.z, c4);
            } else {
                v = vol_sample<CUBIC>(a, qi, qj, qk, px, py, pz);
            }
            if (KIND == kPre && R.stage == kcSample) {
                // _kernels.py:471-507
                ++c_eval;
                if (c4[3] > 0.0) {
                    R.ca = 1.0 - vr_pow(1.0 - c4[3], a.corr);  // ahat
                    R.cr = c4[0];
                    R.cg = c4[1];
                    R.cb = c4[2];
                    if (LIGHT) {
                        R.hx = R.x;
                        R.hy = R.y;
                        R.hz = R.z;
                        R.hbi = R.bi;
                        R.hbj = R.bj;
                        R.hbk = R.bk;
                        R.stage = kcGrad;
                    } else {
                        const double w = (1.0 - R.acc_a) * R.ca;
                        R.acc_r += w * R.cr;
                        R.acc_g += w * R.cg;
                        R.acc_b += w * R.cb;
                        R.acc_a += w;
                        ++R.nvis;
                        R.stage = kcNone;
                        R.n += 1;
                        if (R.acc_a >= a.term_alpha) finished = true;
                    }
                } else {
                    R.stage = kcNone;
                    R.n += 1;
                }
            } else if (R.stage == kcPrevExact || R.stage == kcPrevGap) {
                R.prev_s = v;
                R.prev_valid = true;
                R.prev_pending = false;
                R.stage = kcSample;
            } else if (R.stage == kcSample) {
                ++c_eval;
                R.s = v;
                bool cont = true;  // the ray goes on past this sample
                if (KIND == kIso) {
                    if (R.prev_valid && (R.prev_s - a.isovalue) * (v - a.isovalue) < 0.0) {
                        R.lo_t = R.t - a.step;
                        R.hi_t = R.t;
                        R.lo_s = R.prev_s;
                        R.stage = kcBisect;
                        cont = false;
                    } else if (v == a.isovalue) {
                        R.t_hit = R.t;
                        R.hx = R.x;
                        R.hy = R.y;
                        R.hz = R.z;
                        R.hbi = owner(a, 0, R.hx);
                        R.hbj = owner(a, 1, R.hy);
                        R.hbk = owner(a, 2, R.hz);
                        R.stage = kcGrad;
                        cont = false;
                    }
                } else {
                    const double sf = R.prev_valid ? R.prev_s : v;
                    const int fbin = lut_bin(sf, a.tbl_lo, a.tbl_inv_w, a.ntbl);
                    const int bbin = lut_bin(v, a.tbl_lo, a.tbl_inv_w, a.ntbl);
                    const double *cell = a.table + 4 * ((long long)fbin * a.ntbl + bbin);
                    const double seg_a = __ldg(cell + 3);
                    if (seg_a > 0.0) {
                        R.cr = __ldg(cell);
                        R.cg = __ldg(cell + 1);
                        R.cb = __ldg(cell + 2);
                        R.ca = seg_a;
                        if (LIGHT) {
                            R.hx = R.x;
                            R.hy = R.y;
                            R.hz = R.z;
                            R.hbi = R.bi;
                            R.hbj = R.bj;
                            R.hbk = R.bk;
                            R.stage = kcGrad;
                            cont = false;
                        } else {
                            const double w = 1.0 - R.acc_a;
                            R.acc_r += w * R.cr;
                            R.acc_g += w * R.cg;
                            R.acc_b += w * R.cb;
                            R.acc_a += w * R.ca;
                            ++R.nvis;
                            if (R.acc_a >= a.term_alpha) finished = true;
                        }
                    }
                }
                if (cont && !finished) {
                    // sample done: a run of samples that provably change nothing
                    R.prev_s = v;
                    R.prev_valid = true;
                    R.stage = kcNone;
                    long long k = 1;
                    if (chain_cull && !R.prev_skippable) {
                        const int lvl = chain_transparent<KIND>(a, R.x, R.y, R.z);
                        if (lvl) {
                            const double p[3] = {R.x, R.y, R.z};
                            const int bidx[3] = {R.bi, R.bj, R.bk};
                            BlockRec rec = {};
                            if (SKIP && KIND != kIso) rec = block_rec(a, (R.bk * nby + R.bj) * nbx + R.bi);
                            k = KIND == kIso ? culled_run<SKIP, false>(a, R.r, R.inv, R.t0, R.n, R.t, p, bidx, rec,
                                                                        lvl == 3 ? 4 : lvl == 1 ? 2 : 0)
                                             : culled_run<SKIP>(a, R.r, R.inv, R.t0, R.n, R.t, p, bidx, rec,
                                                                lvl == 3 ? 4 : lvl == 1 ? 2 : 0);
                            if (k > R.N - R.n) k = R.N - R.n;
                            if (k < 1) k = 1;
                        }
                    }
                    if (k > 1) {
                        R.taken += k - 1;
                        R.prev_pending = true;
                    }
                    R.n += k;
                }
            } else if (KIND == kIso && R.stage < kcGrad) {
                // bisection round (_kernels.py:447-461)
                const double mid = 0.5 * (R.lo_t + R.hi_t);
                if ((R.lo_s - a.isovalue) * (v - a.isovalue) <= 0.0) {
                    R.hi_t = mid;
                } else {
                    R.lo_t = mid;
                    R.lo_s = v;
                }
                if (++R.stage == kcGrad) {
                    R.t_hit = 0.5 * (R.lo_t + R.hi_t);
                    R.hx = divide(R.r.ox + R.t_hit * R.r.dx, a.dsx);
                    R.hy = divide(R.r.oy + R.t_hit * R.r.dy, a.dsy);
                    R.hz = divide(R.r.oz + R.t_hit * R.r.dz, a.dsz);
                    R.hbi = owner(a, 0, R.hx);
                    R.hbj = owner(a, 1, R.hy);
                    R.hbk = owner(a, 2, R.hz);
                }
            } else {
                // gradient tap (_kernels.py:236-253): +x, -x, +y, -y, +z, -z
                const int q = R.stage - kcGrad;
                if (q & 1) {
                    const double dg = R.gplus - v;
                    if (q == 1) R.gx = dg;
                    else if (q == 3) R.gy = dg;
                    else R.gz = dg;
                } else {
                    R.gplus = v;
                }
                if (q < 5) {
                    R.stage += 1;
                } else {
                    gradient_done(R.gx, R.gy, R.gz);
                }
            }
        }
#if VR_CHAIN_COOP
        if (coop) {
            __syncwarp();
            const bool grad = R.live && R.stage == kcGrad;
            const unsigned gm = __ballot_sync(full, grad);
            if (gm) {
                const int ntaps = 6 * __popc(gm);
                const int rank = __popc(gm & ((1u << lane) - 1u));
                if (grad) {
                    s_px[wib][rank] = R.hx;
                    s_py[wib][rank] = R.hy;
                    s_pz[wib][rank] = R.hz;
                    s_blk[wib][rank] = make_int4(R.hbi, R.hbj, R.hbk, 0);
                }
                __syncwarp();
#pragma unroll 1
                for (int base = 0; base < ntaps; base += 32) {
                    const int id = base + lane;
                    const bool act = id < ntaps;
                    double px = 0.0, py = 0.0, pz = 0.0;
                    int qi = 0, qj = 0, qk = 0;
                    if (act) {
                        const int k = id / 6, g = id - 6 * k;
                        px = s_px[wib][k];
                        py = s_py[wib][k];
                        pz = s_pz[wib][k];
                        const int4 q = s_blk[wib][k];
                        const double hh = (g & 1) ? -0.5 : 0.5;
                        const int axis = g >> 1;
                        px = axis == 0 ? px + hh : px;
                        py = axis == 1 ? py + hh : py;
                        pz = axis == 2 ? pz + hh : pz;
                        const int o = owner(a, axis, axis == 0 ? px : axis == 1 ? py : pz);
                        qi = axis == 0 ? o : q.x;
                        qj = axis == 1 ? o : q.y;
                        qk = axis == 2 ? o : q.z;
                    }
                    const double v = vol_sample<CUBIC>(a, qi, qj, qk, px, py, pz);
                    if (act) s_tap[wib][id] = v;
                }
                __syncwarp();
                if (grad) {
                    const double *tp = s_tap[wib] + 6 * rank;
                    gradient_done(tp[0] - tp[1], tp[2] - tp[3], tp[4] - tp[5]);
                }
                __syncwarp();
            }
        }
#endif
        if (R.live && R.stage == kcNone && R.n >= R.N) finished = true;

        if (finished) {
            // background, epilogue, per-pixel outputs (_kernels.py:583-594)
            const double w = 1.0 - R.acc_a;
            const double rr = R.acc_r + w * a.bg[0] * a.bg[3];
            const double gg = R.acc_g + w * a.bg[1] * a.bg[3];
            const double bb = R.acc_b + w * a.bg[2] * a.bg[3];
            const double aa = R.acc_a + w * a.bg[3];
            const long long p = R.out;
            if (a.premult) reinterpret_cast<double4 *>(a.premult)[p] = make_double4(rr, gg, bb, aa);
            if (a.pixels) {
                double r0 = 0.0, g0 = 0.0, b0 = 0.0;
                if (aa > 0.0) {
                    const double den = aa > 1e-12 ? aa : 1e-12;
                    r0 = rr / den;
                    g0 = gg / den;
                    b0 = bb / den;
                }
                reinterpret_cast<uchar4 *>(a.pixels)[p] = make_uchar4(to_u8(r0), to_u8(g0), to_u8(b0), to_u8(aa));
            }
            if (a.depth) a.depth[p] = R.t_hit;
            if (a.taken) a.taken[p] = R.taken;
            if (a.skipped) a.skipped[p] = R.skipped;
            c_taken += (unsigned long long)R.taken;
            c_skip += (unsigned long long)R.skipped;
            R.live = false;
        }
    }
    c_taken = warp_sum(c_taken);
    c_skip = warp_sum(c_skip);
    if (lane == 0 && a.totals && (c_taken | c_skip)) {
        atomicAdd(a.totals, c_taken);
        atomicAdd(a.totals + 1, c_skip);
    }
    if (a.work) {
        c_shaded = warp_sum(c_shaded);
        c_eval = warp_sum(c_eval);
        c_iter = warp_sum(c_iter);
        if (lane == 0) {
            if (c_shaded) atomicAdd(a.work, c_shaded);
            if (c_eval) atomicAdd(a.work + 1, c_eval);
            if (c_iter) atomicAdd(a.work + 2, c_iter);
        }
    }
}

using KernelFn = void (*)(RenderArgs);

template <bool CUBIC, bool LIGHT, bool MV>
KernelFn pick_heavy(bool skip) {
    return skip ? raycast_heavy_kernel<CUBIC, LIGHT, true, MV> : raycast_heavy_kernel<CUBIC, LIGHT, false, MV>;
}

KernelFn pick_cooperative(const RenderArgs &a) {
    const bool c = a.cubic != 0, l = a.lighting != 0, s = a.skip_empty != 0;
    if (a.nviews > 1) {
        if (c) return l ? pick_heavy<true, true, true>(s) : pick_heavy<true, false, true>(s);
        return l ? pick_heavy<false, true, true>(s) : pick_heavy<false, false, true>(s);
    }
    if (c) return l ? pick_heavy<true, true, false>(s) : pick_heavy<true, false, false>(s);
    return l ? pick_heavy<false, true, false>(s) : pick_heavy<false, false, false>(s);
}

template <bool CUBIC, bool LIGHT, bool MV>
KernelFn pick_post(bool skip) {
    return skip ? raycast_post_kernel<CUBIC, LIGHT, true, MV> : raycast_post_kernel<CUBIC, LIGHT, false, MV>;
}

KernelFn pick_persistent(const RenderArgs &a) {
    const bool c = a.cubic != 0, l = a.lighting != 0, s = a.skip_empty != 0;
    if (a.nviews > 1) {
        if (c) return l ? pick_post<true, true, true>(s) : pick_post<true, false, true>(s);
        return l ? pick_post<false, true, true>(s) : pick_post<false, false, true>(s);
    }
    if (c) return l ? pick_post<true, true, false>(s) : pick_post<true, false, false>(s);
    return l ? pick_post<false, true, false>(s) : pick_post<false, false, false>(s);
}

template <int KIND, bool CUBIC, bool LIGHT>
KernelFn pick_skip(bool skip) {
    return skip ? raycast_kernel<KIND, CUBIC, LIGHT, true> : raycast_kernel<KIND, CUBIC, LIGHT, false>;
}

template <int KIND, bool CUBIC>
KernelFn pick_light(bool light, bool skip) {
    return light ? pick_skip<KIND, CUBIC, true>(skip) : pick_skip<KIND, CUBIC, false>(skip);
}

template <int KIND>
KernelFn pick_cubic(bool cubic, bool light, bool skip) {
    return cubic ? pick_light<KIND, true>(light, skip) : pick_light<KIND, false>(light, skip);
}

// Resident CTAs per SM of a persistent kernel on the current device, queried
// once per (device, kernel) and cached (two runtime queries per frame were
// host time on the end-to-end path).  Reentrant callers share the cache
// under a lock.
std::mutex g_occ_mu;

int persistent_ctas_per_sm(KernelFn k) {
    static int keys_dev[64];
    static KernelFn keys[64];
    static int vals[64];
    static int n = 0;
    int dev = 0;
    cudaGetDevice(&dev);
    std::lock_guard<std::mutex> g(g_occ_mu);
    for (int i = 0; i < n; ++i)
        if (keys[i] == k && keys_dev[i] == dev) return vals[i];
    int per_sm = 1;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k, kPersistThreads, 0) != cudaSuccess || per_sm < 1)
        per_sm = 1;
    if (n < 64) {
        keys_dev[n] = dev;
        keys[n] = k;
        vals[n] = per_sm;
        ++n;
    }
    return per_sm;
}

// ------------------------------------- warp-cooperative chained-mode long rays
// Continues the rays raycast_chain_kernel handed over: one warp per ray, 32
// consecutive samples per chunk, one per lane.  Every lane evaluates its
// sample's skip predicate (the chained gap rule -- a skippable sample is
// taken when its predecessor was not -- needs only the neighbour's flag),
// interpolates it if taken, and, when its predecessor was skipped (or, for
// the chunk's first lane, culled in the per-lane kernel), the previous sample
// as the reference re-evaluates it.  Then, in sample order:
//  - iso: the first lane whose pair (prev, s) changes sign or hits exactly is
//    the hit; its 8 bisection points run on that lane, its 6 gradient taps on
//    6 lanes (_kernels.py:405-468);
//  - pre-integrated: the segment opacities decide the terminating sample by
//    replaying A += (1 - A) a; the gradient taps of the contributing samples
//    up to it are spread over the lanes, 32 per round; colours composite in
//    order (_kernels.py:538-581).
// Counts stop at the hit / terminating sample, as the sequential march does.
template <int KIND, bool CUBIC, bool LIGHT, bool SKIP>
#ifndef VR_CHAIN_COOP_MIN_BLOCKS
#define VR_CHAIN_COOP_MIN_BLOCKS 4
#endif
__global__ void __launch_bounds__(kPersistThreads, VR_CHAIN_COOP_MIN_BLOCKS *(kThreads / kPersistThreads))
    raycast_chain_coop_kernel(const __grid_constant__ RenderArgs a) {
    pdl_enter();
    const int lane = threadIdx.x & 31;
    const unsigned full = 0xffffffffu;
    const unsigned lower = (1u << lane) - 1u;
    const int nbx = a.L.nb[0], nby = a.L.nb[1];
    const unsigned long long pushed = *a.heavy_count;
    const long long count = (long long)(pushed < (unsigned long long)a.heavy_cap ? pushed : a.heavy_cap);
    unsigned long long c_taken = 0, c_skip = 0, c_shaded = 0, c_eval = 0, c_iter = 0;
    for (;;) {
        unsigned long long idx = 0;
        if (lane == 0) idx = atomicAdd(a.heavy_head, 1ull);
        idx = __shfl_sync(full, idx, 0);
        if ((long long)idx >= count) break;
        const ChainRec h = static_cast<const ChainRec *>(a.heavy)[idx];
        Ray r;
        r.ox = h.o[0];
        r.oy = h.o[1];
        r.oz = h.o[2];
        r.dx = h.d[0];
        r.dy = h.d[1];
        r.dz = h.d[2];
        double inv[3];
        inv[0] = r.dx != 0.0 ? 1.0 / r.dx : 0.0;
        inv[1] = r.dy != 0.0 ? 1.0 / r.dy : 0.0;
        inv[2] = r.dz != 0.0 ? 1.0 / r.dz : 0.0;
        double acc_r = h.acc[0], acc_g = h.acc[1], acc_b = h.acc[2], acc_a = h.acc[3];
        long long taken = h.taken, skipped = h.skipped;
        // carried state of the sample before the chunk
        double c_prev = h.prev_s;
        bool c_prev_valid = (h.flags & 1) != 0, c_pending = (h.flags & 2) != 0, c_prev_skip = (h.flags & 4) != 0;
        double t_hit = __longlong_as_double(0x7ff8000000000000LL);
        long long n = h.n;
        bool done = false;
        while (KIND == kPre && n < h.N) {
            // ---- pre-classified chunk (_kernels.py:471-507): not chained
            ++c_iter;
            const long long m = n + lane;
            const bool valid = m < h.N;
            double t = 0.0, x = 0.0, y = 0.0, z = 0.0;
            int bi = 0, bj = 0, bk = 0, b = 0, lvl = 0;
            bool skippable = false, cell_only = true;
            BlockRec rec = {};
            if (valid) {
                t = h.t0 + ((double)m + 0.5) * a.step;
                x = divide(r.ox + t * r.dx, a.dsx);
                y = divide(r.oy + t * r.dy, a.dsy);
                z = divide(r.oz + t * r.dz, a.dsz);
                bi = owner(a, 0, x);
                bj = owner(a, 1, y);
                bk = owner(a, 2, z);
                b = (bk * nby + bj) * nbx + bi;
                if (SKIP) {
                    rec = block_rec(a, b);
                    skippable = dvr_skippable(rec, x, y, z);
                    cell_only = rec.lo.w != 0.0f;
                }
                if (!skippable && a.cull) lvl = pre_transparent(a, x, y, z);
            }
            const bool tk = valid && !skippable;
            const bool cand = tk && lvl == 0;
            const unsigned tmask = __ballot_sync(full, tk), vmask = __ballot_sync(full, valid);
            const unsigned candm = __ballot_sync(full, cand);
            if (candm == 0u) {
                // nothing to evaluate: extend by a provable run from the last sample
                long long k = 1;
                if (lane == 31 && valid) {
                    const double p[3] = {x, y, z};
                    const int bidx[3] = {bi, bj, bk};
                    k = skippable ? leap_count<kPre>(a, r, inv, h.t0, m, t, p, bidx, rec, cell_only)
                                  : culled_run<SKIP>(a, r, inv, h.t0, m, t, p, bidx, rec, lvl);
                }
                k = __shfl_sync(full, k, 31);
                const bool last_skip = __shfl_sync(full, skippable, 31);
                taken += __popc(tmask);
                skipped += __popc(vmask & ~tmask);
                if (tk && a.blocks_hit) a.blocks_hit[b] = 1;
                long long next = n + 32;
                const long long last = n + 31;
                if (last < h.N && k > 1) {
                    if (k > h.N - last) k = h.N - last;
                    if (last_skip)
                        skipped += k - 1;
                    else
                        taken += k - 1;
                    next = last + k;
                }
                n = next;
                continue;
            }
            // alpha of every candidate, then the terminating sample by replaying
            // A += (1 - A) ahat in sample order
            double sa = 0.0, ahat = 0.0, c4[4] = {0.0, 0.0, 0.0, 0.0};
            if (cand) attr_rgba4<CUBIC>(a, bi, bj, bk, x, y, z, c4);
            sa = c4[3];
            const bool contrib = cand && sa > 0.0;
            if (contrib) ahat = 1.0 - vr_pow(1.0 - sa, a.corr);
            const unsigned cm = __ballot_sync(full, contrib);
            int stop = 32;
            {
                double A = acc_a;
                unsigned mm = cm;
                while (mm) {
                    const int src = __ffs(mm) - 1;
                    mm &= mm - 1;
                    A += (1.0 - A) * __shfl_sync(full, ahat, src);
                    if (A >= a.term_alpha) {
                        stop = src;
                        break;
                    }
                }
            }
            const unsigned upto = stop >= 31 ? full : ((2u << stop) - 1u);
            const unsigned vis = cm & upto;
            // the 6 gradient taps of every visible sample (lighting), spread
            // over the lanes, 32 per round
            double sr = c4[0], sg = c4[1], sb = c4[2];
            if (LIGHT && vis) {
                double tp[6] = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
                const int njobs = 6 * __popc(vis);
                const int rank = __popc(vis & lower);
                for (int base = 0; base < njobs; base += 32) {
                    const int id = base + lane;
                    const bool act = id < njobs;
                    const int k = id / 6, g = id - 6 * k;
                    const int src = act ? nth_bit(vis, k) : lane;
                    double px = __shfl_sync(full, x, src), py = __shfl_sync(full, y, src);
                    double pz = __shfl_sync(full, z, src);
                    int qi = __shfl_sync(full, bi, src), qj = __shfl_sync(full, bj, src);
                    int qk = __shfl_sync(full, bk, src);
                    const double hh = (g & 1) ? -0.5 : 0.5;
                    const int axis = g >> 1;
                    px = axis == 0 ? px + hh : px;
                    py = axis == 1 ? py + hh : py;
                    pz = axis == 2 ? pz + hh : pz;
                    const int o = owner(a, axis, axis == 0 ? px : axis == 1 ? py : pz);
                    qi = axis == 0 ? o : qi;
                    qj = axis == 1 ? o : qj;
                    qk = axis == 2 ? o : qk;
                    const double v = vol_sample<CUBIC>(a, qi, qj, qk, px, py, pz);
#pragma unroll
                    for (int gg = 0; gg < 6; ++gg) {
                        const int sidx = 6 * rank + gg - base;
                        const double w = __shfl_sync(full, v, sidx & 31);
                        if (sidx >= 0 && sidx < 32) tp[gg] = w;
                    }
                }
                if ((vis >> lane) & 1u) {
                    const double gx = divide(tp[0] - tp[1], a.dsx), gy = divide(tp[2] - tp[3], a.dsy),
                                 gz = divide(tp[4] - tp[5], a.dsz);
                    const double norm = sqrt((gx * gx + gy * gy) + gz * gz);
                    if (norm > 1e-12) shade(a, sr, sg, sb, -gx / norm, -gy / norm, -gz / norm, -r.dx, -r.dy, -r.dz);
                }
            }
            if (LIGHT && lane == 0) c_shaded += __popc(vis);
            {
                unsigned mm = vis;
                while (mm) {
                    const int src = __ffs(mm) - 1;
                    mm &= mm - 1;
                    const double w = (1.0 - acc_a) * __shfl_sync(full, ahat, src);
                    acc_r += w * __shfl_sync(full, sr, src);
                    acc_g += w * __shfl_sync(full, sg, src);
                    acc_b += w * __shfl_sync(full, sb, src);
                    acc_a += w;
                }
            }
            taken += __popc(tmask & upto);
            skipped += __popc(vmask & ~tmask & upto);
            if (lane == 0) c_eval += __popc(candm & upto);
            if (tk && lane <= stop && a.blocks_hit) a.blocks_hit[b] = 1;
            if (stop < 32) break;
            n += 32;
        }
        while (KIND != kPre && n < h.N && !done) {
            ++c_iter;
            const long long m = n + lane;
            const bool valid = m < h.N;
            double t = 0.0, x = 0.0, y = 0.0, z = 0.0;
            int bi = 0, bj = 0, bk = 0, b = 0;
            bool skippable = false, cell_only = true;
            BlockRec rec = {};
            if (valid) {
                t = h.t0 + ((double)m + 0.5) * a.step;
                x = divide(r.ox + t * r.dx, a.dsx);
                y = divide(r.oy + t * r.dy, a.dsy);
                z = divide(r.oz + t * r.dz, a.dsz);
                bi = owner(a, 0, x);
                bj = owner(a, 1, y);
                bk = owner(a, 2, z);
                b = (bk * nby + bj) * nbx + bi;
                if (SKIP) {
                    if (KIND == kIso) {
                        skippable = (double)__ldg(a.vmax + b) < a.isovalue || (double)__ldg(a.vmin + b) > a.isovalue;
                    } else {
                        rec = block_rec(a, b);
                        skippable = dvr_skippable(rec, x, y, z);
                        cell_only = rec.lo.w != 0.0f;
                    }
                }
            }
            // the chained gap rule: skipped iff skippable and the previous sample was
            const bool pskip_lane = __shfl_up_sync(full, skippable, 1);
            const bool prev_skip = lane == 0 ? c_prev_skip : pskip_lane;
            const bool tk = valid && !(skippable && prev_skip);
            const unsigned tmask = __ballot_sync(full, tk);
            const unsigned vmask = __ballot_sync(full, valid);
            // a chunk with nothing taken extends by a provable leap from its last sample
            if (tmask == 0u) {
                const unsigned smask = vmask;
                long long k = 1;
                if (lane == 31 && valid && skippable) {
                    const double p[3] = {x, y, z};
                    const int bidx[3] = {bi, bj, bk};
                    k = leap_count<KIND>(a, r, inv, h.t0, m, t, p, bidx, rec, cell_only);
                }
                k = __shfl_sync(full, k, 31);
                const long long last = n + 31;
                skipped += __popc(smask);
                long long next = n + 32;
                if (last < h.N && k > 1) {
                    if (k > h.N - last) k = h.N - last;
                    skipped += k - 1;
                    next = last + k;
                }
                c_prev_valid = false;
                c_pending = false;
                c_prev_skip = __shfl_sync(full, skippable, 31) || !__shfl_sync(full, valid, 31);
                n = next;
                continue;
            }
            // round 1: every taken sample -- except, for iso, samples whose
            // region bound excludes the isovalue: only the sign of s - iso is
            // ever used for them (crossing tests, bisection bracket), and the
            // bound's end nearest the isovalue carries it
            double sv = 0.0;
            bool cull_iso = false;
            if (KIND == kIso && tk && a.cull) {
                short2 bd;
                if (chain_transparent<kIso>(a, x, y, z, &bd)) {
                    cull_iso = true;
                    sv = (double)bd.x > a.isovalue ? (double)bd.x : (double)bd.y;
                }
            }
            if (tk && !cull_iso) {
                sv = vol_sample<CUBIC>(a, bi, bj, bk, x, y, z);
            }
            // round 2: previous values the chunk does not hold -- after a
            // skipped predecessor (t - step, the reference's gap rule) or, on
            // lane 0, after a culled run (the predecessor's own position)
            const bool pred_taken_lane = __shfl_up_sync(full, tk, 1);
            const double pred_s_lane = __shfl_up_sync(full, sv, 1);
            bool pvalid;
            double pv = 0.0;
            bool need = false;
            double tq = 0.0;
            if (lane == 0) {
                if (c_pending) {
                    need = tk;
                    tq = h.t0 + ((double)(m - 1) + 0.5) * a.step;
                    pvalid = true;
                } else if (c_prev_valid) {
                    pvalid = true;
                    pv = c_prev;
                } else {
                    need = tk && m > 0;
                    tq = t - a.step;
                    pvalid = m > 0;
                }
            } else if (pred_taken_lane) {
                pvalid = true;
                pv = pred_s_lane;
            } else {
                need = tk;  // predecessor skipped: prev at t - step (m > 0 here)
                tq = t - a.step;
                pvalid = true;
            }
            if (__any_sync(full, need)) {
                double qx = x, qy = y, qz = z;
                int qi = bi, qj = bj, qk = bk;
                if (need) {
                    qx = divide(r.ox + tq * r.dx, a.dsx);
                    qy = divide(r.oy + tq * r.dy, a.dsy);
                    qz = divide(r.oz + tq * r.dz, a.dsz);
                    qi = owner(a, 0, qx);
                    qj = owner(a, 1, qy);
                    qk = owner(a, 2, qz);
                }
                const double q = vol_sample<CUBIC>(a, qi, qj, qk, qx, qy, qz);
                if (need) pv = q;
            }
            if (!tk) pvalid = false;
            int stop = 32;  // the lane whose sample ends the ray (hit / termination); 32: none
            if (KIND == kIso) {
                const bool crossing = tk && pvalid && (pv - a.isovalue) * (sv - a.isovalue) < 0.0;
                const bool exact = tk && sv == a.isovalue;
                const unsigned hm = __ballot_sync(full, crossing || exact);
                if (hm) {
                    const int hl = __ffs(hm) - 1;
                    stop = hl;
                    const bool hc = __shfl_sync(full, crossing, hl);
                    const double ht = __shfl_sync(full, t, hl);
                    double thit = ht;
                    if (hc) {
                        // 8 bisection rounds on the warp (the hit lane's interval)
                        double lo_t = ht - a.step, hi_t = ht, lo_s = __shfl_sync(full, pv, hl);
                        for (int it = 0; it < 8; ++it) {
                            const double mid = 0.5 * (lo_t + hi_t);
                            const double mx = divide(r.ox + mid * r.dx, a.dsx);
                            const double my = divide(r.oy + mid * r.dy, a.dsy);
                            const double mz = divide(r.oz + mid * r.dz, a.dsz);
                            const double ms = vol_sample<CUBIC>(a, owner(a, 0, mx), owner(a, 1, my), owner(a, 2, mz),
                                                                mx, my, mz);
                            if ((lo_s - a.isovalue) * (ms - a.isovalue) <= 0.0) {
                                hi_t = mid;
                            } else {
                                lo_t = mid;
                                lo_s = ms;
                            }
                        }
                        thit = 0.5 * (lo_t + hi_t);
                    }
                    const double hx = divide(r.ox + thit * r.dx, a.dsx);
                    const double hy = divide(r.oy + thit * r.dy, a.dsy);
                    const double hz = divide(r.oz + thit * r.dz, a.dsz);
                    const int hbi = owner(a, 0, hx), hbj = owner(a, 1, hy), hbk = owner(a, 2, hz);
                    // gradient: lane q < 6 takes tap q (+x,-x,+y,-y,+z,-z)
                    double gpx = hx, gpy = hy, gpz = hz;
                    int gi = hbi, gj = hbj, gk = hbk;
                    const int q = lane < 6 ? lane : 0;
                    const double hh = (q & 1) ? -0.5 : 0.5;
                    const int axis = q >> 1;
                    gpx = axis == 0 ? hx + hh : hx;
                    gpy = axis == 1 ? hy + hh : hy;
                    gpz = axis == 2 ? hz + hh : hz;
                    const int o = owner(a, axis, axis == 0 ? gpx : axis == 1 ? gpy : gpz);
                    gi = axis == 0 ? o : gi;
                    gj = axis == 1 ? o : gj;
                    gk = axis == 2 ? o : gk;
                    const double tv = vol_sample<CUBIC>(a, gi, gj, gk, gpx, gpy, gpz);
                    const double tp0 = __shfl_sync(full, tv, 0), tp1 = __shfl_sync(full, tv, 1);
                    const double tp2 = __shfl_sync(full, tv, 2), tp3 = __shfl_sync(full, tv, 3);
                    const double tp4 = __shfl_sync(full, tv, 4), tp5 = __shfl_sync(full, tv, 5);
                    const double gx = divide(tp0 - tp1, a.dsx), gy = divide(tp2 - tp3, a.dsy),
                                 gz = divide(tp4 - tp5, a.dsz);
                    if (lane == 0) ++c_shaded;
                    const double norm = sqrt((gx * gx + gy * gy) + gz * gz);
                    const int ib = lut_bin(a.isovalue, a.lut_lo, a.lut_inv_w, a.nlut);
                    double cr = __ldg(a.lut + 4 * ib), cg = __ldg(a.lut + 4 * ib + 1), cb = __ldg(a.lut + 4 * ib + 2);
                    if (LIGHT && norm > 1e-12)
                        shade(a, cr, cg, cb, -gx / norm, -gy / norm, -gz / norm, -r.dx, -r.dy, -r.dz);
                    acc_r = cr;
                    acc_g = cg;
                    acc_b = cb;
                    acc_a = 1.0;
                    t_hit = thit;
                }
            } else {
                // pre-integrated segments
                bool contrib = false;
                double sr = 0.0, sg = 0.0, sb = 0.0, sa = 0.0;
                if (tk) {
                    const double sf = pvalid ? pv : sv;
                    const int fbin = lut_bin(sf, a.tbl_lo, a.tbl_inv_w, a.ntbl);
                    const int bbin = lut_bin(sv, a.tbl_lo, a.tbl_inv_w, a.ntbl);
                    const double *cell = a.table + 4 * ((long long)fbin * a.ntbl + bbin);
                    sa = __ldg(cell + 3);
                    if (sa > 0.0) {
                        contrib = true;
                        sr = __ldg(cell);
                        sg = __ldg(cell + 1);
                        sb = __ldg(cell + 2);
                    }
                }
                // the terminating sample: replay A += (1 - A) a in order
                unsigned cm = __ballot_sync(full, contrib);
                {
                    double A = acc_a;
                    unsigned mm = cm;
                    while (mm) {
                        const int src = __ffs(mm) - 1;
                        mm &= mm - 1;
                        A += (1.0 - A) * __shfl_sync(full, sa, src);
                        if (A >= a.term_alpha) {
                            stop = src;
                            break;
                        }
                    }
                }
                const unsigned upto = stop >= 31 ? full : ((2u << stop) - 1u);
                const unsigned vis = cm & upto;
                if (LIGHT && vis) {
                    // 6 gradient taps per contributing sample, 32 per round
                    const int ntaps = 6 * __popc(vis);
                    const int rank = __popc(vis & lower);
                    double tp[6] = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
                    for (int base = 0; base < ntaps; base += 32) {
                        const int id = base + lane;
                        const bool act = id < ntaps;
                        const int k = id / 6, g = id - 6 * k;
                        const int src = act ? nth_bit(vis, k) : lane;
                        double px = __shfl_sync(full, x, src), py = __shfl_sync(full, y, src);
                        double pz = __shfl_sync(full, z, src);
                        int qi = __shfl_sync(full, bi, src), qj = __shfl_sync(full, bj, src);
                        int qk = __shfl_sync(full, bk, src);
                        const double hh = (g & 1) ? -0.5 : 0.5;
                        const int axis = g >> 1;
                        px = axis == 0 ? px + hh : px;
                        py = axis == 1 ? py + hh : py;
                        pz = axis == 2 ? pz + hh : pz;
                        const int o = owner(a, axis, axis == 0 ? px : axis == 1 ? py : pz);
                        qi = axis == 0 ? o : qi;
                        qj = axis == 1 ? o : qj;
                        qk = axis == 2 ? o : qk;
                        const double v = vol_sample<CUBIC>(a, qi, qj, qk, px, py, pz);
#pragma unroll
                        for (int gg = 0; gg < 6; ++gg) {
                            const int sidx = 6 * rank + gg - base;
                            const double w = __shfl_sync(full, v, sidx & 31);
                            if (sidx >= 0 && sidx < 32) tp[gg] = w;
                        }
                    }
                    if ((vis >> lane) & 1u) {
                        const double gx = divide(tp[0] - tp[1], a.dsx), gy = divide(tp[2] - tp[3], a.dsy),
                                     gz = divide(tp[4] - tp[5], a.dsz);
                        const double norm = sqrt((gx * gx + gy * gy) + gz * gz);
                        if (norm > 1e-12) {
                            const double ndl = fabs(((gx * -r.dx + gy * -r.dy) + gz * -r.dz) / norm);
                            const double scale = a.ka + a.kd * ndl;
                            const double spec = a.ks * vr_pow(ndl, a.shin) * sa;
                            sr = clampf(scale * sr + spec, 0.0, 1.0);
                            sg = clampf(scale * sg + spec, 0.0, 1.0);
                            sb = clampf(scale * sb + spec, 0.0, 1.0);
                        }
                    }
                    if (lane == 0) c_shaded += __popc(vis);
                }
                // composite in sample order (_kernels.py:574-579)
                unsigned mm = vis;
                while (mm) {
                    const int src = __ffs(mm) - 1;
                    mm &= mm - 1;
                    const double w = 1.0 - acc_a;
                    acc_r += w * __shfl_sync(full, sr, src);
                    acc_g += w * __shfl_sync(full, sg, src);
                    acc_b += w * __shfl_sync(full, sb, src);
                    acc_a += w * __shfl_sync(full, sa, src);
                }
            }
            // counts up to and including the stopping sample; blocks hit
            const unsigned upto = stop >= 31 ? full : ((2u << stop) - 1u);
            taken += __popc(tmask & upto);
            skipped += __popc(vmask & ~tmask & upto);
            if (lane == 0) c_eval += __popc(tmask & upto);  // (samples evaluated or provably one-sided)
            if (tk && lane <= stop && a.blocks_hit) a.blocks_hit[b] = 1;
            if (stop < 32) {
                done = true;
                break;
            }
            // carry the chunk's last sample into the next chunk
            const bool last_tk = __shfl_sync(full, tk, 31);
            c_prev = __shfl_sync(full, sv, 31);
            c_prev_valid = last_tk;
            c_pending = false;
            c_prev_skip = __shfl_sync(full, skippable, 31);
            n += 32;
        }
        if (lane == 0) {
            const double w = 1.0 - acc_a;
            const double rr = acc_r + w * a.bg[0] * a.bg[3];
            const double gg = acc_g + w * a.bg[1] * a.bg[3];
            const double bb = acc_b + w * a.bg[2] * a.bg[3];
            const double aa = acc_a + w * a.bg[3];
            const long long p = h.out;
            if (a.premult) reinterpret_cast<double4 *>(a.premult)[p] = make_double4(rr, gg, bb, aa);
            if (a.pixels) {
                double r0 = 0.0, g0 = 0.0, b0 = 0.0;
                if (aa > 0.0) {
                    const double den = aa > 1e-12 ? aa : 1e-12;
                    r0 = rr / den;
                    g0 = gg / den;
                    b0 = bb / den;
                }
                reinterpret_cast<uchar4 *>(a.pixels)[p] = make_uchar4(to_u8(r0), to_u8(g0), to_u8(b0), to_u8(aa));
            }
            if (a.depth) a.depth[p] = t_hit;
            if (a.taken) a.taken[p] = taken;
            if (a.skipped) a.skipped[p] = skipped;
            c_taken += (unsigned long long)taken;
            c_skip += (unsigned long long)skipped;
        }
    }
    c_taken = warp_sum(c_taken);
    c_skip = warp_sum(c_skip);
    if (lane == 0 && a.totals && (c_taken | c_skip)) {
        atomicAdd(a.totals, c_taken);
        atomicAdd(a.totals + 1, c_skip);
    }
    if (a.work) {
        c_shaded = warp_sum(c_shaded);
        c_eval = warp_sum(c_eval);
        c_iter = warp_sum(c_iter);
        if (lane == 0) {
            if (c_shaded) atomicAdd(a.work, c_shaded);
            if (c_eval) atomicAdd(a.work + 1, c_eval);
            if (c_iter) atomicAdd(a.work + 2, c_iter);
        }
    }
}

template <int KIND, bool CUBIC, bool LIGHT>
KernelFn pick_chain_skip(bool skip) {
    return skip ? raycast_chain_kernel<KIND, CUBIC, LIGHT, true> : raycast_chain_kernel<KIND, CUBIC, LIGHT, false>;
}

template <int KIND>
KernelFn pick_chain_kind(const RenderArgs &a) {
    const bool c = a.cubic != 0, l = a.lighting != 0, s = a.skip_empty != 0;
    if (c) return l ? pick_chain_skip<KIND, true, true>(s) : pick_chain_skip<KIND, true, false>(s);
    return l ? pick_chain_skip<KIND, false, true>(s) : pick_chain_skip<KIND, false, false>(s);
}

KernelFn pick_chain(const RenderArgs &a) {
    if (a.mode == 1) return pick_chain_kind<kIso>(a);
    return a.classify == 1 ? pick_chain_kind<kPre>(a) : pick_chain_kind<kPreint>(a);
}

template <int KIND, bool CUBIC, bool LIGHT>
KernelFn pick_chain_coop_skip(bool skip) {
    return skip ? raycast_chain_coop_kernel<KIND, CUBIC, LIGHT, true> : raycast_chain_coop_kernel<KIND, CUBIC, LIGHT, false>;
}

template <int KIND>
KernelFn pick_chain_coop_kind(const RenderArgs &a) {
    const bool c = a.cubic != 0, l = a.lighting != 0, s = a.skip_empty != 0;
    if (c) return l ? pick_chain_coop_skip<KIND, true, true>(s) : pick_chain_coop_skip<KIND, true, false>(s);
    return l ? pick_chain_coop_skip<KIND, false, true>(s) : pick_chain_coop_skip<KIND, false, false>(s);
}

KernelFn pick_chain_coop(const RenderArgs &a) {
    if (a.mode == 1) return pick_chain_coop_kind<kIso>(a);
    return a.classify == 1 ? pick_chain_coop_kind<kPre>(a) : pick_chain_coop_kind<kPreint>(a);
}

KernelFn pick(const RenderArgs &a) {
    const bool c = a.cubic != 0, l = a.lighting != 0, s = a.skip_empty != 0;
    if (a.mode == 1) return pick_cubic<kIso>(c, l, s);
    switch (a.classify) {
        case 1: return pick_cubic<kPre>(c, l, s);
        case 2: return pick_cubic<kPreint>(c, l, s);
        default: return pick_cubic<kPost>(c, l, s);
    }
}

}  // namespace

int device_sms() {
    static int sms[64] = {};
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev < 0 || dev >= 64) dev = 0;
    std::lock_guard<std::mutex> g(g_occ_mu);
    if (sms[dev] == 0) {
        int v = 0;
        if (cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || v < 1) {
            cudaGetLastError();
            v = 148;  // B200
        }
        sms[dev] = v;
    }
    return sms[dev];
}

cudaError_t launch_raycast(const RenderArgs &a, cudaStream_t stream) {
    if (a.tw <= 0 || a.th <= 0) return cudaSuccess;
    if (a.slots <= 0) return cudaSuccess;
    if (a.mode == 0 && a.classify == 0 && a.work_counter) {
        // persistent: enough CTAs to fill every SM at the kernel's occupancy.
        // A batched sweep runs in chunks of kViewChunk views, each a
        // per-lane pass then the cooperative pass over its handed-over rays:
        // the hand-off queues stay bounded and every chunk's long rays are
        // handed over as its views' items drain (per view, as in a frame).
        KernelFn k = pick_persistent(a);
        KernelFn h = a.heavy ? pick_cooperative(a) : nullptr;
        const int sms = device_sms(), per_sm = persistent_ctas_per_sm(k);
        const int hctas = h ? sms * persistent_ctas_per_sm(h) : 0;
        for (int v0 = 0; v0 < a.nviews; v0 += kViewChunk) {
            RenderArgs c = a;
            c.view0 = a.view0 + v0;
            c.nviews = a.nviews - v0 < kViewChunk ? a.nviews - v0 : kViewChunk;
            if (v0 > 0) {  // the first chunk's counters were zeroed by the frame's setup kernel
                cudaError_t e = cudaMemsetAsync(a.work_counter, 0, 4 * sizeof(unsigned long long), stream);
                if (e != cudaSuccess) return e;
            }
            long long ctas = (long long)sms * per_sm;
            const long long most = (long long)c.slots * c.nviews * (kThreads / kPersistThreads);  // a warp per 32 rays at most
            if (ctas > most) ctas = most;
            cudaError_t e = launch_pdl(k, (unsigned)ctas, kPersistThreads, 0, stream, c);
            if (e != cudaSuccess) return e;
            if (h) {
                e = launch_pdl(h, (unsigned)hctas, kPersistThreads, 0, stream, c);
                if (e != cudaSuccess) return e;
            }
        }
        return cudaGetLastError();
    }
    const bool chained = a.mode == 1 || (a.mode == 0 && a.classify != 0);  // iso, pre-integrated, pre
    if (chained && a.work_counter && a.nviews == 1) {
        // persistent chained modes (queue counters zeroed by the frame's first kernel)
        KernelFn k = pick_chain(a);
        long long ctas = (long long)device_sms() * persistent_ctas_per_sm(k);
        const long long most = (long long)a.slots * (kThreads / kPersistThreads);
        if (ctas > most) ctas = most;
        k<<<(unsigned)ctas, kPersistThreads, 0, stream>>>(a);
        if (a.heavy) {
            KernelFn h = pick_chain_coop(a);
            cudaError_t e = launch_pdl(h, (unsigned)(device_sms() * persistent_ctas_per_sm(h)), kPersistThreads, 0,
                                       stream, a);
            if (e != cudaSuccess) return e;
        }
        return cudaGetLastError();
    }
    pick(a)<<<(unsigned)((long long)a.slots * a.nviews), kThreads, 0, stream>>>(a);
    return cudaGetLastError();
}

}  // namespace vr
