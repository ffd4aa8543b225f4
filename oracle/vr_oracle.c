/*
 * oracle/vr_oracle.c -- CPU restatement of the voxelray hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  Nothing in the product package links, loads or
 * calls this file.  It is imported by tests/, by __graft_entry__.smoke() and by
 * bench.py's cpu_baseline / --impl reference legs, and only as the checker or
 * the timed CPU baseline.
 *
 * Parity pin: tests/test_oracle_golden.py checks every function here against
 * golden vectors produced by the unmodified reference (tests/golden/make_golden.py
 * imports /root/reference/pkg/src/voxelray and calls its own functions).  The
 * restatement keeps the reference's operation order, so that with
 * -ffp-contract=off (no FMA contraction, like numba's LLVM output, which the
 * survey checked has no vfmadd) it reproduces the float64 results bit for bit.
 *
 * Reference anchors (paths relative to /root/reference/pkg/src/voxelray/):
 *   _kernels.py:52-80   _tri_sample         -> vro_tri_sample
 *   _kernels.py:83-143  _cr_weights/_row4/_plane4/_cub_sample -> vro_cub_sample
 *   _kernels.py:153-166 _grad_voxel         -> vro_grad_voxel
 *   _kernels.py:169-187 sample_points / gradient_points
 *   _kernels.py:190-192 _lut_bin            -> lut_bin
 *   _kernels.py:195-208 _shade              -> shade
 *   _kernels.py:211-276 _attr_sample/_attr_grad/_attr_rgba
 *   _kernels.py:279-594 march               -> vro_march
 *   render.py:125-144   _ray_grid           -> vro_ray_grid
 *   render.py:147-156   _clip_to_bounds     -> vro_clip_to_bounds
 *   blocks.py:100-158   _axis_layout/decompose -> vro_axis_layout / vro_block_minmax
 *   blocks.py:161-220   cull_empty/fit_bounding_box/with_visibility -> vro_visibility
 *   blocks.py:269-294   build_atlas         -> vro_build_atlas
 *   phantoms.py:76-111  torso phantom       (numpy restatement lives in oracle.py)
 *   K4 (no voxel function in the reference): vro_threshold_count,
 *   vro_ball_counts, vro_threshold_measure, vro_ball_measure -- S and V of the
 *   method of spheres (morphology.py:70-306)
 *   restated on the voxel grid; parity unpinned (no reference function), the
 *   semantics pinned by the analytic oracles of SPEC.md:472-473 instead.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define MODE_DVR 0
#define MODE_ISO 1
#define CLS_POST 0
#define CLS_PRE 1
#define CLS_PREINT 2

static inline double clampf(double v, double lo, double hi) {
    if (v < lo) return lo;
    if (v > hi) return hi;
    return v;
}

static inline int64_t clampi(int64_t v, int64_t lo, int64_t hi) {
    if (v < lo) return lo;
    if (v > hi) return hi;
    return v;
}

/* Python's max(a, 0.0): returns a unless 0.0 > a */
static inline double pymax0(double a) { return (0.0 > a) ? 0.0 : a; }

/* ---------------------------------------------------------- interpolation */

/* _kernels.py:52-80 */
static double vro_tri_sample(const int16_t *data, int64_t base, int64_t ex, int64_t ey,
                             int64_t ez, double x, double y, double z) {
    x = clampf(x, 0.0, ex - 1.0);
    y = clampf(y, 0.0, ey - 1.0);
    z = clampf(z, 0.0, ez - 1.0);
    int64_t i0 = clampi((int64_t)x, 0, ex - 2);
    int64_t j0 = clampi((int64_t)y, 0, ey - 2);
    int64_t k0 = clampi((int64_t)z, 0, ez - 2);
    double fx = x - (double)i0;
    double fy = y - (double)j0;
    double fz = z - (double)k0;
    int64_t p = base + (k0 * ey + j0) * ex + i0;
    int64_t q = p + ey * ex;
    double v000 = (double)data[p];
    double v100 = (double)data[p + 1];
    double v010 = (double)data[p + ex];
    double v110 = (double)data[p + ex + 1];
    double v001 = (double)data[q];
    double v101 = (double)data[q + 1];
    double v011 = (double)data[q + ex];
    double v111 = (double)data[q + ex + 1];
    double c00 = v000 + (v100 - v000) * fx;
    double c10 = v010 + (v110 - v010) * fx;
    double c01 = v001 + (v101 - v001) * fx;
    double c11 = v011 + (v111 - v011) * fx;
    double c0 = c00 + (c10 - c00) * fy;
    double c1 = c01 + (c11 - c01) * fy;
    return c0 + (c1 - c0) * fz;
}

/* _kernels.py:83-91 -- Catmull-Rom weights, same association as the Python */
static inline void cr_weights(double t, double w[4]) {
    double t2 = t * t;
    double t3 = t2 * t;
    w[0] = 0.5 * ((-t3 + 2.0 * t2) - t);
    w[1] = 0.5 * ((3.0 * t3 - 5.0 * t2) + 2.0);
    w[2] = 0.5 * ((-3.0 * t3 + 4.0 * t2) + t);
    w[3] = 0.5 * (t3 - t2);
}

/* _kernels.py:94-111 for one row; generic element type through a macro so the
 * same code serves the int16 atlas and the uint8 preclassified atlas */
#define ROW4(data, row, ii, w)                                                     \
    ((((w)[0] * (double)(data)[(row) + (ii)[0]] + (w)[1] * (double)(data)[(row) + (ii)[1]]) + \
      (w)[2] * (double)(data)[(row) + (ii)[2]]) +                                   \
     (w)[3] * (double)(data)[(row) + (ii)[3]])

#define DEFINE_CUB(NAME, T)                                                          \
    static double NAME(const T *data, int64_t base, int64_t ex, int64_t ey, int64_t ez, \
                       double x, double y, double z) {                              \
        x = clampf(x, 0.0, ex - 1.0);                                                \
        y = clampf(y, 0.0, ey - 1.0);                                                \
        z = clampf(z, 0.0, ez - 1.0);                                                \
        int64_t i0 = clampi((int64_t)x, 0, ex - 1);                                  \
        int64_t j0 = clampi((int64_t)y, 0, ey - 1);                                  \
        int64_t k0 = clampi((int64_t)z, 0, ez - 1);                                  \
        double wx[4], wy[4], wz[4];                                                  \
        cr_weights(x - (double)i0, wx);                                              \
        cr_weights(y - (double)j0, wy);                                              \
        cr_weights(z - (double)k0, wz);                                              \
        int64_t ii[4] = {clampi(i0 - 1, 0, ex - 1), i0, clampi(i0 + 1, 0, ex - 1),   \
                         clampi(i0 + 2, 0, ex - 1)};                                 \
        int64_t jj[4] = {clampi(j0 - 1, 0, ey - 1), j0, clampi(j0 + 1, 0, ey - 1),   \
                         clampi(j0 + 2, 0, ey - 1)};                                 \
        int64_t kk[4] = {clampi(k0 - 1, 0, ez - 1), k0, clampi(k0 + 1, 0, ez - 1),   \
                         clampi(k0 + 2, 0, ez - 1)};                                 \
        int64_t plane = ey * ex;                                                     \
        double pl[4];                                                                \
        for (int c = 0; c < 4; ++c) {                                                \
            int64_t pb = base + kk[c] * plane;                                       \
            double r0 = ROW4(data, pb + jj[0] * ex, ii, wx);                         \
            double r1 = ROW4(data, pb + jj[1] * ex, ii, wx);                         \
            double r2 = ROW4(data, pb + jj[2] * ex, ii, wx);                         \
            double r3 = ROW4(data, pb + jj[3] * ex, ii, wx);                         \
            pl[c] = ((wy[0] * r0 + wy[1] * r1) + wy[2] * r2) + wy[3] * r3;           \
        }                                                                            \
        return ((wz[0] * pl[0] + wz[1] * pl[1]) + wz[2] * pl[2]) + wz[3] * pl[3];    \
    }

/* _kernels.py:114-143 */
DEFINE_CUB(vro_cub_sample, int16_t)
DEFINE_CUB(vro_cub_sample_u8, uint8_t)

/* trilinear over uint8 data (preclassified planes), same formula as _tri_sample */
static double vro_tri_sample_u8(const uint8_t *data, int64_t base, int64_t ex, int64_t ey,
                                int64_t ez, double x, double y, double z) {
    x = clampf(x, 0.0, ex - 1.0);
    y = clampf(y, 0.0, ey - 1.0);
    z = clampf(z, 0.0, ez - 1.0);
    int64_t i0 = clampi((int64_t)x, 0, ex - 2);
    int64_t j0 = clampi((int64_t)y, 0, ey - 2);
    int64_t k0 = clampi((int64_t)z, 0, ez - 2);
    double fx = x - (double)i0;
    double fy = y - (double)j0;
    double fz = z - (double)k0;
    int64_t p = base + (k0 * ey + j0) * ex + i0;
    int64_t q = p + ey * ex;
    double v000 = (double)data[p];
    double v100 = (double)data[p + 1];
    double v010 = (double)data[p + ex];
    double v110 = (double)data[p + ex + 1];
    double v001 = (double)data[q];
    double v101 = (double)data[q + 1];
    double v011 = (double)data[q + ex];
    double v111 = (double)data[q + ex + 1];
    double c00 = v000 + (v100 - v000) * fx;
    double c10 = v010 + (v110 - v010) * fx;
    double c01 = v001 + (v101 - v001) * fx;
    double c11 = v011 + (v111 - v011) * fx;
    double c0 = c00 + (c10 - c00) * fy;
    double c1 = c01 + (c11 - c01) * fy;
    return c0 + (c1 - c0) * fz;
}

/* _kernels.py:146-150 */
static inline double vro_sample(const int16_t *data, int64_t base, int64_t ex, int64_t ey,
                                int64_t ez, double x, double y, double z, int cubic) {
    if (cubic) return vro_cub_sample(data, base, ex, ey, ez, x, y, z);
    return vro_tri_sample(data, base, ex, ey, ez, x, y, z);
}

static inline double vro_sample_u8(const uint8_t *data, int64_t base, int64_t ex, int64_t ey,
                                   int64_t ez, double x, double y, double z, int cubic) {
    if (cubic) return vro_cub_sample_u8(data, base, ex, ey, ez, x, y, z);
    return vro_tri_sample_u8(data, base, ex, ey, ez, x, y, z);
}

/* _kernels.py:153-166 */
static void vro_grad_voxel(const int16_t *data, int64_t base, int64_t ex, int64_t ey,
                           int64_t ez, double x, double y, double z, int cubic, double g[3]) {
    const double h = 0.5;
    g[0] = vro_sample(data, base, ex, ey, ez, x + h, y, z, cubic) -
           vro_sample(data, base, ex, ey, ez, x - h, y, z, cubic);
    g[1] = vro_sample(data, base, ex, ey, ez, x, y + h, z, cubic) -
           vro_sample(data, base, ex, ey, ez, x, y - h, z, cubic);
    g[2] = vro_sample(data, base, ex, ey, ez, x, y, z + h, cubic) -
           vro_sample(data, base, ex, ey, ez, x, y, z - h, cubic);
}

/* _kernels.py:169-174 */
void vro_sample_points(const int16_t *data, int64_t ex, int64_t ey, int64_t ez,
                       const double *pts, int64_t n, int cubic, double *out) {
    for (int64_t i = 0; i < n; ++i)
        out[i] = vro_sample(data, 0, ex, ey, ez, pts[3 * i], pts[3 * i + 1], pts[3 * i + 2], cubic);
}

/* _kernels.py:177-187 */
void vro_gradient_points(const int16_t *data, int64_t ex, int64_t ey, int64_t ez,
                         const double *pts, int64_t n, int cubic, double sx, double sy,
                         double sz, double *out) {
    for (int64_t i = 0; i < n; ++i) {
        double g[3];
        vro_grad_voxel(data, 0, ex, ey, ez, pts[3 * i], pts[3 * i + 1], pts[3 * i + 2], cubic, g);
        out[3 * i] = g[0] / sx;
        out[3 * i + 1] = g[1] / sy;
        out[3 * i + 2] = g[2] / sz;
    }
}

/* _kernels.py:190-192; int() truncates toward zero before the clamp */
static inline int64_t lut_bin(double s, double lo, double inv_w, int64_t nbins) {
    return clampi((int64_t)((s - lo) * inv_w), 0, nbins - 1);
}

#ifdef VRO_CR_POW
/* Diagnostics build only (never the oracle proper): x^n for integer n as a
 * double-double ladder rounded once, i.e. a correctly rounded power, to tell
 * glibc pow's <= 0.52-ulp rounding apart from other differences. */
static double vro_pow(double x, double y) {
    if (y != floor(y) || y < 0 || y > 4096) return pow(x, y);
    int n = (int)y;
    double rh = 1.0, rl = 0.0, bh = x, bl = 0.0;
    while (n > 0) {
        if (n & 1) {
            double p = rh * bh, e = fma(rh, bh, -p);
            e += rh * bl + rl * bh;
            double s = p + e, bb = s - p;
            rl = (p - (s - bb)) + (e - bb);
            rh = s;
        }
        n >>= 1;
        if (n) {
            double p = bh * bh, e = fma(bh, bh, -p);
            e += 2.0 * bh * bl;
            double s = p + e, bb = s - p;
            bl = (p - (s - bb)) + (e - bb);
            bh = s;
        }
    }
    return rh + rl;
}
#define SHADE_POW vro_pow
#else
#define SHADE_POW pow
#endif

/* _kernels.py:195-208 */
static inline void shade(double *r, double *g, double *b, double nx, double ny, double nz,
                         double lx, double ly, double lz, double ka, double kd, double ks,
                         double shininess) {
    double ndl = (nx * lx + ny * ly) + nz * lz;
    double diff = kd * pymax0(ndl);
    double rv = 2.0 * ndl * ndl - 1.0;
    double spec = ks * SHADE_POW(pymax0(rv), shininess);
    *r = clampf(*r * (ka + diff) + spec, 0.0, 1.0);
    *g = clampf(*g * (ka + diff) + spec, 0.0, 1.0);
    *b = clampf(*b * (ka + diff) + spec, 0.0, 1.0);
}

/* ------------------------------------------------------ block attribution */

typedef struct {
    const int16_t *atlas;
    const uint8_t *rgba_atlas;
    const int64_t *offsets;
    const int64_t *org_x, *org_y, *org_z;
    const int64_t *ext_x, *ext_y, *ext_z;
    int64_t nbx, nby, nbz;
    int64_t stride;
} grid_t;

static inline int64_t owner(double x, int64_t stride, int64_t nb) {
    return clampi((int64_t)floor((x - 1.0) / (double)stride), 0, nb - 1);
}

/* _kernels.py:211-233 */
static inline double attr_sample(const grid_t *g, double x, double y, double z, int cubic) {
    int64_t bi = owner(x, g->stride, g->nbx);
    int64_t bj = owner(y, g->stride, g->nby);
    int64_t bk = owner(z, g->stride, g->nbz);
    int64_t b = (bk * g->nby + bj) * g->nbx + bi;
    return vro_sample(g->atlas, g->offsets[b], g->ext_x[bi], g->ext_y[bj], g->ext_z[bk],
                      x - (double)g->org_x[bi], y - (double)g->org_y[bj], z - (double)g->org_z[bk],
                      cubic);
}

/* _kernels.py:236-253 */
static inline void attr_grad(const grid_t *g, double x, double y, double z, int cubic,
                             double sx, double sy, double sz, double out[3]) {
    const double h = 0.5;
    double gx = attr_sample(g, x + h, y, z, cubic) - attr_sample(g, x - h, y, z, cubic);
    double gy = attr_sample(g, x, y + h, z, cubic) - attr_sample(g, x, y - h, z, cubic);
    double gz = attr_sample(g, x, y, z + h, cubic) - attr_sample(g, x, y, z - h, cubic);
    out[0] = gx / sx;
    out[1] = gy / sy;
    out[2] = gz / sz;
}

/* _kernels.py:256-276 */
static inline double attr_rgba(const grid_t *g, double x, double y, double z, int cubic, int ch) {
    int64_t bi = owner(x, g->stride, g->nbx);
    int64_t bj = owner(y, g->stride, g->nby);
    int64_t bk = owner(z, g->stride, g->nbz);
    int64_t b = (bk * g->nby + bj) * g->nbx + bi;
    int64_t ex = g->ext_x[bi], ey = g->ext_y[bj], ez = g->ext_z[bk];
    double v = vro_sample_u8(g->rgba_atlas, g->offsets[b] * 4 + ch * ex * ey * ez, ex, ey, ez,
                             x - (double)g->org_x[bi], y - (double)g->org_y[bj],
                             z - (double)g->org_z[bk], cubic);
    return clampf(v / 255.0, 0.0, 1.0);
}

/* ------------------------------------------------------------------ march */

/* _kernels.py:279-594, one pixel.  Outputs are written exactly as the
 * reference does (premultiplied float64 RGBA, depth only on an iso hit). */
static void march_pixel(int64_t p, const double *origins, const double *dirs,
                        const double *tmins, const double *tmaxs, double sx, double sy,
                        double sz, double step, double ref_step, int mode, int cubic,
                        int lighting, int classify, int skip_empty, const grid_t *g,
                        const double *vmin, const double *vmax, const uint8_t *empty,
                        const double *box_lo, const double *box_hi, const double *lut,
                        int64_t nlut, double lut_lo, double lut_inv_w, const double *table,
                        int64_t ntbl, double tbl_lo, double tbl_inv_w, double isovalue,
                        double term_alpha, double ka, double kd, double ks, double shininess,
                        double bg_r, double bg_g, double bg_b, double bg_a, double *out,
                        double *depth, int64_t *taken, int64_t *skipped, uint8_t *blocks_hit) {
    const double corr = step / ref_step;
    const int chained = (mode == MODE_ISO) || (classify == CLS_PREINT);
    double acc_r = 0.0, acc_g = 0.0, acc_b = 0.0, acc_a = 0.0;
    int64_t n_taken = 0, n_skip = 0;
    double t0 = tmins[p], t1 = tmaxs[p];
    if (t1 >= t0) {
        double ox = origins[3 * p], oy = origins[3 * p + 1], oz = origins[3 * p + 2];
        double dx = dirs[3 * p], dy = dirs[3 * p + 1], dz = dirs[3 * p + 2];
        int64_t nsteps = (int64_t)ceil((t1 - t0) / step);
        if (nsteps < 1) nsteps = 1;
        double prev_s = 0.0;
        int prev_valid = 0, prev_skippable = 0;
        for (int64_t n = 0; n < nsteps; ++n) {
            double t = t0 + ((double)n + 0.5) * step;
            if (t > t1) break;
            double x = (ox + t * dx) / sx;
            double y = (oy + t * dy) / sy;
            double z = (oz + t * dz) / sz;
            int64_t bi = owner(x, g->stride, g->nbx);
            int64_t bj = owner(y, g->stride, g->nby);
            int64_t bk = owner(z, g->stride, g->nbz);
            int64_t b = (bk * g->nby + bj) * g->nbx + bi;

            int skippable = 0;
            if (skip_empty) {
                if (mode == MODE_ISO) {
                    skippable = vmax[b] < isovalue || vmin[b] > isovalue;
                } else if (empty[b] == 1) {
                    skippable = 1;
                } else if (x < box_lo[3 * b] || x > box_hi[3 * b] || y < box_lo[3 * b + 1] ||
                           y > box_hi[3 * b + 1] || z < box_lo[3 * b + 2] ||
                           z > box_hi[3 * b + 2]) {
                    skippable = 1;
                }
            }
            if (skippable && (prev_skippable || !chained)) {
                n_skip += 1;
                prev_valid = 0;
                prev_skippable = 1;
                continue;
            }
            prev_skippable = skippable;
            blocks_hit[b] = 1;
            n_taken += 1;

            if (mode == MODE_ISO) {
                double s = attr_sample(g, x, y, z, cubic);
                if (!prev_valid && n > 0) {
                    double tp = t - step;
                    prev_s = attr_sample(g, (ox + tp * dx) / sx, (oy + tp * dy) / sy,
                                         (oz + tp * dz) / sz, cubic);
                    prev_valid = 1;
                }
                int hit = 0;
                double t_hit = t;
                if (prev_valid && (prev_s - isovalue) * (s - isovalue) < 0.0) {
                    double lo_t = t - step, hi_t = t, lo_s = prev_s;
                    for (int it = 0; it < 8; ++it) {
                        double mid = 0.5 * (lo_t + hi_t);
                        double ms = attr_sample(g, (ox + mid * dx) / sx, (oy + mid * dy) / sy,
                                                (oz + mid * dz) / sz, cubic);
                        if ((lo_s - isovalue) * (ms - isovalue) <= 0.0) {
                            hi_t = mid;
                        } else {
                            lo_t = mid;
                            lo_s = ms;
                        }
                    }
                    t_hit = 0.5 * (lo_t + hi_t);
                    hit = 1;
                } else if (s == isovalue) {
                    hit = 1;
                }
                if (hit) {
                    double hx = (ox + t_hit * dx) / sx;
                    double hy = (oy + t_hit * dy) / sy;
                    double hz = (oz + t_hit * dz) / sz;
                    int64_t ibin = lut_bin(isovalue, lut_lo, lut_inv_w, nlut);
                    double cr = lut[4 * ibin], cg = lut[4 * ibin + 1], cb = lut[4 * ibin + 2];
                    double gr[3];
                    attr_grad(g, hx, hy, hz, cubic, sx, sy, sz, gr);
                    double norm = sqrt((gr[0] * gr[0] + gr[1] * gr[1]) + gr[2] * gr[2]);
                    if (lighting && norm > 1e-12)
                        shade(&cr, &cg, &cb, -gr[0] / norm, -gr[1] / norm, -gr[2] / norm, -dx,
                              -dy, -dz, ka, kd, ks, shininess);
                    acc_r = cr;
                    acc_g = cg;
                    acc_b = cb;
                    acc_a = 1.0;
                    depth[p] = t_hit;
                    break;
                }
                prev_s = s;
                prev_valid = 1;
                continue;
            }

            if (classify == CLS_PRE) {
                double sa = attr_rgba(g, x, y, z, cubic, 3);
                if (sa > 0.0) {
                    double sr = attr_rgba(g, x, y, z, cubic, 0);
                    double sg = attr_rgba(g, x, y, z, cubic, 1);
                    double sb = attr_rgba(g, x, y, z, cubic, 2);
                    double ahat = 1.0 - pow(1.0 - sa, corr);
                    if (lighting) {
                        double gr[3];
                        attr_grad(g, x, y, z, cubic, sx, sy, sz, gr);
                        double norm = sqrt((gr[0] * gr[0] + gr[1] * gr[1]) + gr[2] * gr[2]);
                        if (norm > 1e-12)
                            shade(&sr, &sg, &sb, -gr[0] / norm, -gr[1] / norm, -gr[2] / norm,
                                  -dx, -dy, -dz, ka, kd, ks, shininess);
                    }
                    double w = (1.0 - acc_a) * ahat;
                    acc_r += w * sr;
                    acc_g += w * sg;
                    acc_b += w * sb;
                    acc_a += w;
                    if (acc_a >= term_alpha) break;
                }
            } else if (classify == CLS_POST) {
                double s = attr_sample(g, x, y, z, cubic);
                int64_t sbin = lut_bin(s, lut_lo, lut_inv_w, nlut);
                double sa = lut[4 * sbin + 3];
                if (sa > 0.0) {
                    double sr = lut[4 * sbin], sg = lut[4 * sbin + 1], sb = lut[4 * sbin + 2];
                    double ahat = 1.0 - pow(1.0 - sa, corr);
                    if (lighting) {
                        double gr[3];
                        attr_grad(g, x, y, z, cubic, sx, sy, sz, gr);
                        double norm = sqrt((gr[0] * gr[0] + gr[1] * gr[1]) + gr[2] * gr[2]);
                        if (norm > 1e-12)
                            shade(&sr, &sg, &sb, -gr[0] / norm, -gr[1] / norm, -gr[2] / norm,
                                  -dx, -dy, -dz, ka, kd, ks, shininess);
                    }
                    double w = (1.0 - acc_a) * ahat;
                    acc_r += w * sr;
                    acc_g += w * sg;
                    acc_b += w * sb;
                    acc_a += w;
                    if (acc_a >= term_alpha) break;
                }
            } else {
                double s = attr_sample(g, x, y, z, cubic);
                if (!prev_valid && n > 0) {
                    double tp = t - step;
                    prev_s = attr_sample(g, (ox + tp * dx) / sx, (oy + tp * dy) / sy,
                                         (oz + tp * dz) / sz, cubic);
                    prev_valid = 1;
                }
                double sf = prev_valid ? prev_s : s;
                int64_t fbin = lut_bin(sf, tbl_lo, tbl_inv_w, ntbl);
                int64_t bbin = lut_bin(s, tbl_lo, tbl_inv_w, ntbl);
                const double *cell = table + 4 * (fbin * ntbl + bbin);
                double seg_a = cell[3];
                if (seg_a > 0.0) {
                    double seg_r = cell[0], seg_g = cell[1], seg_b = cell[2];
                    if (lighting) {
                        double gr[3];
                        attr_grad(g, x, y, z, cubic, sx, sy, sz, gr);
                        double norm = sqrt((gr[0] * gr[0] + gr[1] * gr[1]) + gr[2] * gr[2]);
                        if (norm > 1e-12) {
                            double ndl = fabs(((gr[0] * -dx + gr[1] * -dy) + gr[2] * -dz) / norm);
                            double scale = ka + kd * ndl;
                            double spec = ks * pow(ndl, shininess) * seg_a;
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
                    if (acc_a >= term_alpha) break;
                }
                prev_s = s;
                prev_valid = 1;
            }
        }
    }
    double w = 1.0 - acc_a;
    acc_r += w * bg_r * bg_a;
    acc_g += w * bg_g * bg_a;
    acc_b += w * bg_b * bg_a;
    acc_a += w * bg_a;
    out[4 * p] = acc_r;
    out[4 * p + 1] = acc_g;
    out[4 * p + 2] = acc_b;
    out[4 * p + 3] = acc_a;
    taken[p] = n_taken;
    skipped[p] = n_skip;
}

int vro_num_threads(void) {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}

/* _kernels.py:279-594.  nthreads <= 0 uses every OpenMP thread. */
void vro_march(int64_t npix, const double *origins, const double *dirs, const double *tmins,
               const double *tmaxs, double sx, double sy, double sz, double step,
               double ref_step, int mode, int cubic, int lighting, int classify,
               int skip_empty, const int16_t *atlas, const uint8_t *rgba_atlas,
               const int64_t *offsets, const int64_t *org_x, const int64_t *org_y,
               const int64_t *org_z, const int64_t *ext_x, const int64_t *ext_y,
               const int64_t *ext_z, int64_t nbx, int64_t nby, int64_t nbz, int64_t stride,
               const double *vmin, const double *vmax, const uint8_t *empty,
               const double *box_lo, const double *box_hi, const double *lut, int64_t nlut,
               double lut_lo, double lut_inv_w, const double *table, int64_t ntbl,
               double tbl_lo, double tbl_inv_w, double isovalue, double term_alpha, double ka,
               double kd, double ks, double shininess, double bg_r, double bg_g, double bg_b,
               double bg_a, double *out, double *depth, int64_t *taken, int64_t *skipped,
               uint8_t *blocks_hit, int nthreads) {
    grid_t g = {atlas, rgba_atlas, offsets, org_x, org_y, org_z, ext_x, ext_y, ext_z,
                nbx, nby, nbz, stride};
#ifdef _OPENMP
    if (nthreads <= 0) nthreads = omp_get_max_threads();
#pragma omp parallel for schedule(dynamic, 64) num_threads(nthreads)
#endif
    for (int64_t p = 0; p < npix; ++p) {
        march_pixel(p, origins, dirs, tmins, tmaxs, sx, sy, sz, step, ref_step, mode, cubic,
                    lighting, classify, skip_empty, &g, vmin, vmax, empty, box_lo, box_hi, lut,
                    nlut, lut_lo, lut_inv_w, table, ntbl, tbl_lo, tbl_inv_w, isovalue,
                    term_alpha, ka, kd, ks, shininess, bg_r, bg_g, bg_b, bg_a, out, depth,
                    taken, skipped, blocks_hit);
    }
}

/* ------------------------------------------------------------------- rays */

/* render.py:125-144 restated per pixel: dirs = (fwd + u*right) + v*true_up,
 * then divided by sqrt((d0^2 + d1^2) + d2^2).  Rows [y0, y0+h), columns
 * [x0, x0+w) of a width x height frame, row-major. */
void vro_ray_grid(const double pos[3], const double fwd[3], const double right[3],
                  const double up[3], double half_w, double half_h, int64_t width,
                  int64_t height, int64_t x0, int64_t y0, int64_t w, int64_t h,
                  double *origins, double *dirs) {
    for (int64_t r = 0; r < h; ++r) {
        double py = (double)(y0 + r);
        double v = (1.0 - 2.0 * (py + 0.5) / (double)height) * half_h;
        for (int64_t c = 0; c < w; ++c) {
            double px = (double)(x0 + c);
            double u = (2.0 * (px + 0.5) / (double)width - 1.0) * half_w;
            int64_t p = r * w + c;
            double d[3];
            for (int a = 0; a < 3; ++a) d[a] = (fwd[a] + u * right[a]) + v * up[a];
            double nrm = sqrt((d[0] * d[0] + d[1] * d[1]) + d[2] * d[2]);
            for (int a = 0; a < 3; ++a) {
                dirs[3 * p + a] = d[a] / nrm;
                origins[3 * p + a] = pos[a];
            }
        }
    }
}

/* Orthographic rays (the reference has no orthographic camera; its
 * march is camera-agnostic).  Origin = (pos + u*right) + v*up with u, v in mm,
 * direction = fwd, for every pixel. */
void vro_ortho_rays(const double pos[3], const double fwd[3], const double right[3],
                    const double up[3], double half_w_mm, double half_h_mm, int64_t width,
                    int64_t height, int64_t x0, int64_t y0, int64_t w, int64_t h,
                    double *origins, double *dirs) {
    for (int64_t r = 0; r < h; ++r) {
        double py = (double)(y0 + r);
        double v = (1.0 - 2.0 * (py + 0.5) / (double)height) * half_h_mm;
        for (int64_t c = 0; c < w; ++c) {
            double px = (double)(x0 + c);
            double u = (2.0 * (px + 0.5) / (double)width - 1.0) * half_w_mm;
            int64_t p = r * w + c;
            for (int a = 0; a < 3; ++a) {
                origins[3 * p + a] = (pos[a] + u * right[a]) + v * up[a];
                dirs[3 * p + a] = fwd[a];
            }
        }
    }
}

/* render.py:147-156 */
void vro_clip_to_bounds(int64_t n, const double *origins, const double *dirs,
                        const double ext[3], double *tmin, double *tmax) {
    const double tiny = 1e-300;
    for (int64_t p = 0; p < n; ++p) {
        double lo_max = -INFINITY, hi_min = INFINITY;
        for (int a = 0; a < 3; ++a) {
            double d = dirs[3 * p + a];
            if (fabs(d) < tiny) d = (d < 0) ? -tiny : tiny;
            double lo = (0.0 - origins[3 * p + a]) / d;
            double hi = (ext[a] - origins[3 * p + a]) / d;
            double mn = lo < hi ? lo : hi;
            double mx = lo > hi ? lo : hi;
            if (a == 0 || mn > lo_max) lo_max = mn;
            if (a == 0 || mx < hi_min) hi_min = mx;
        }
        tmin[p] = lo_max > 0.0 ? lo_max : 0.0;
        tmax[p] = hi_min;
    }
}

/* ----------------------------------------------------------------- blocks */

/* blocks.py:100-107; returns the block count along one axis */
int64_t vro_axis_layout(int64_t n, int64_t block_size, int64_t stride, int64_t *origins,
                        int64_t *extents) {
    int64_t count;
    if (n <= block_size)
        count = 1;
    else
        count = (int64_t)ceil((double)(n - block_size) / (double)stride) + 1;
    if (origins) {
        for (int64_t i = 0; i < count; ++i) {
            origins[i] = i * stride;
            int64_t e = n - origins[i];
            extents[i] = e < block_size ? e : block_size;
        }
    }
    return count;
}

/* blocks.py:133-145: min/max over each block's region, overlap included;
 * outputs shaped (nbz, nby, nbx) */
void vro_block_minmax(const int16_t *vals, int64_t nx, int64_t ny, int64_t nz,
                      const int64_t *ox, const int64_t *ex, int64_t nbx, const int64_t *oy,
                      const int64_t *ey, int64_t nby, const int64_t *oz, const int64_t *ez,
                      int64_t nbz, int64_t *vmin, int64_t *vmax) {
    (void)nz;
    for (int64_t bk = 0; bk < nbz; ++bk)
        for (int64_t bj = 0; bj < nby; ++bj)
            for (int64_t bi = 0; bi < nbx; ++bi) {
                int64_t lo = INT64_MAX, hi = INT64_MIN;
                for (int64_t z = oz[bk]; z < oz[bk] + ez[bk]; ++z)
                    for (int64_t y = oy[bj]; y < oy[bj] + ey[bj]; ++y) {
                        const int16_t *row = vals + (z * ny + y) * nx;
                        for (int64_t x = ox[bi]; x < ox[bi] + ex[bi]; ++x) {
                            int64_t v = row[x];
                            if (v < lo) lo = v;
                            if (v > hi) hi = v;
                        }
                    }
                int64_t b = (bk * nby + bj) * nbx + bi;
                vmin[b] = lo;
                vmax[b] = hi;
            }
}

/* transfer.py:120-125 ClassifiedLUT.bin_index: floor((s - lo) / bin_width) clipped */
static inline int64_t classified_bin(double s, double lo, double bin_width, int64_t bins) {
    return clampi((int64_t)floor((s - lo) / bin_width), 0, bins - 1);
}

/* blocks.py:161-220.  alpha = lut column 3 (nbins entries).  empty shaped
 * (nbz,nby,nbx); aabb_lo/hi shaped (nbz,nby,nbx,3), (x,y,z) order, global
 * inclusive voxel indices, empty blocks keep the INT64_MAX//2 / -1 sentinel. */
void vro_visibility(const int16_t *vals, int64_t nx, int64_t ny, int64_t nz,
                    const int64_t *ox, const int64_t *ex, int64_t nbx, const int64_t *oy,
                    const int64_t *ey, int64_t nby, const int64_t *oz, const int64_t *ez,
                    int64_t nbz, const int64_t *vmin, const int64_t *vmax,
                    const double *lut_rgba, int64_t nbins, double lut_lo, double bin_width,
                    uint8_t *empty, int64_t *aabb_lo, int64_t *aabb_hi) {
    (void)nz;
    int64_t *prefix = (int64_t *)malloc((size_t)(nbins + 1) * sizeof(int64_t));
    prefix[0] = 0;
    for (int64_t i = 0; i < nbins; ++i) prefix[i + 1] = prefix[i] + (lut_rgba[4 * i + 3] > 0.0);
    for (int64_t bk = 0; bk < nbz; ++bk)
        for (int64_t bj = 0; bj < nby; ++bj)
            for (int64_t bi = 0; bi < nbx; ++bi) {
                int64_t b = (bk * nby + bj) * nbx + bi;
                int64_t lo = classified_bin((double)vmin[b], lut_lo, bin_width, nbins);
                int64_t hi = classified_bin((double)vmax[b], lut_lo, bin_width, nbins);
                int vis = (prefix[hi + 1] - prefix[lo]) > 0;
                empty[b] = (uint8_t)!vis;
                for (int a = 0; a < 3; ++a) {
                    aabb_lo[3 * b + a] = INT64_MAX / 2;
                    aabb_hi[3 * b + a] = -1;
                }
                if (!vis) continue;
                int64_t mn[3] = {INT64_MAX, INT64_MAX, INT64_MAX}, mx[3] = {-1, -1, -1};
                for (int64_t z = 0; z < ez[bk]; ++z)
                    for (int64_t y = 0; y < ey[bj]; ++y) {
                        const int16_t *row = vals + ((oz[bk] + z) * ny + (oy[bj] + y)) * nx + ox[bi];
                        for (int64_t x = 0; x < ex[bi]; ++x) {
                            int64_t k = classified_bin((double)row[x], lut_lo, bin_width, nbins);
                            if (lut_rgba[4 * k + 3] > 0.0) {
                                if (x < mn[0]) mn[0] = x;
                                if (x > mx[0]) mx[0] = x;
                                if (y < mn[1]) mn[1] = y;
                                if (y > mx[1]) mx[1] = y;
                                if (z < mn[2]) mn[2] = z;
                                if (z > mx[2]) mx[2] = z;
                            }
                        }
                    }
                if (mx[0] < 0) continue; /* reference raises EmptyBlock; cannot happen
                                            with monotone-prefix verdicts */
                int64_t org[3] = {ox[bi], oy[bj], oz[bk]}, ext[3] = {ex[bi], ey[bj], ez[bk]};
                for (int a = 0; a < 3; ++a) {
                    int64_t l = mn[a] - 1;
                    int64_t h = mx[a] + 1;
                    aabb_lo[3 * b + a] = org[a] + (l > 0 ? l : 0);
                    aabb_hi[3 * b + a] = org[a] + (h < ext[a] - 1 ? h : ext[a] - 1);
                }
            }
    free(prefix);
}

/* blocks.py:269-294; atlas must hold sum of block volumes; offsets per block */
void vro_build_atlas(const int16_t *vals, int64_t nx, int64_t ny, int64_t nz,
                     const int64_t *ox, const int64_t *ex, int64_t nbx, const int64_t *oy,
                     const int64_t *ey, int64_t nby, const int64_t *oz, const int64_t *ez,
                     int64_t nbz, int16_t *atlas, int64_t *offsets) {
    (void)nz;
    int64_t pos = 0;
    for (int64_t bk = 0; bk < nbz; ++bk)
        for (int64_t bj = 0; bj < nby; ++bj)
            for (int64_t bi = 0; bi < nbx; ++bi) {
                offsets[(bk * nby + bj) * nbx + bi] = pos;
                for (int64_t z = oz[bk]; z < oz[bk] + ez[bk]; ++z)
                    for (int64_t y = oy[bj]; y < oy[bj] + ey[bj]; ++y) {
                        memcpy(atlas + pos, vals + (z * ny + y) * nx + ox[bi],
                               (size_t)ex[bi] * sizeof(int16_t));
                        pos += ex[bi];
                    }
            }
}

/* -------------------------------------------------------- volume measure */

/* K4 (parity unpinned): number of voxels with value >= thr */
uint64_t vro_threshold_count(const int16_t *vals, int64_t n, int32_t thr) {
    uint64_t c = 0;
    for (int64_t i = 0; i < n; ++i) c += (vals[i] >= thr);
    return c;
}

/* K4 ball form: voxels with value >= thr whose centre (i*sx, j*sy, k*sz) mm
 * lies in the closed ball |p - c|^2 <= R^2, the squared distance summed as
 * ((dx^2 + dy^2) + dz^2) in float64. */
void vro_ball_counts(const int16_t *vals, int64_t nx, int64_t ny, int64_t nz, double sx,
                     double sy, double sz, int32_t thr, const double *centres,
                     const double *radii, int64_t nballs, uint64_t *counts) {
    for (int64_t q = 0; q < nballs; ++q) {
        double cx = centres[3 * q], cy = centres[3 * q + 1], cz = centres[3 * q + 2];
        double r2 = radii[q] * radii[q];
        uint64_t c = 0;
        for (int64_t k = 0; k < nz; ++k) {
            double dz = (double)k * sz - cz;
            for (int64_t j = 0; j < ny; ++j) {
                double dy = (double)j * sy - cy;
                const int16_t *row = vals + (k * ny + j) * nx;
                for (int64_t i = 0; i < nx; ++i) {
                    double dx = (double)i * sx - cx;
                    c += (row[i] >= thr && (dx * dx + dy * dy) + dz * dz <= r2);
                }
            }
        }
        counts[q] = c;
    }
}

/* K4 surface S of the method of spheres (the reference
 * measures it on triangle meshes, morphology.py:70-143 clipped_area).  On the
 * voxel grid the object {v >= thr} is bounded by the isosurface of the
 * trilinear-by-tetrahedra interpolant at level L = thr - 0.5 (integer voxels:
 * v >= thr <=> v > L, so the surface separates exactly the voxels V counts):
 *  - cells are the unit cubes between voxel centres, padded by one cell on
 *    every side with the outside value -32768 (the surface closes at the
 *    volume border);
 *  - each cell is split into the 6 Kuhn tetrahedra 000 -> e_a -> e_a+e_b -> 111
 *    (a, b, c a permutation of x, y, z; face-consistent between cells);
 *  - in a tetrahedron the linear interpolant's level set is a triangle (one
 *    corner inside or outside) or a planar quad (two and two), its vertices
 *    at t = f_in / (f_in - f_out) from the inside corner (f = v - L);
 *  - S sums the polygon areas (mm^2; corners at index * spacing), each rounded
 *    to a multiple of 2^-24 mm^2 so the sum is exact and order-free; the ball
 *    form keeps the polygons whose vertex centroid lies in the closed ball.
 * Bit-exactness with the CUDA kernel: same operations, same order, no FMA. */
#define VRO_AREA_SCALE 16777216.0 /* 2^24 */

static const int KUHN[6][3] = {{0, 1, 2}, {0, 2, 1}, {1, 0, 2}, {1, 2, 0}, {2, 0, 1}, {2, 1, 0}};

static inline double field_at(const int16_t *vals, int64_t nx, int64_t ny, int64_t nz, int64_t i, int64_t j,
                              int64_t k, double level) {
    if (i < 0 || j < 0 || k < 0 || i >= nx || j >= ny || k >= nz) return -32768.0 - level;
    return (double)vals[(k * ny + j) * nx + i] - level;
}

static inline void edge_point(const double *P, const double *Q, double fp, double fq, double *out) {
    double t = fp / (fp - fq);
    out[0] = P[0] + t * (Q[0] - P[0]);
    out[1] = P[1] + t * (Q[1] - P[1]);
    out[2] = P[2] + t * (Q[2] - P[2]);
}

static inline double cross_half_norm(double ux, double uy, double uz, double wx, double wy, double wz) {
    double cx = uy * wz - uz * wy;
    double cy = uz * wx - ux * wz;
    double cz = ux * wy - uy * wx;
    return 0.5 * sqrt((cx * cx + cy * cy) + cz * cz);
}

/* area (fixed point) of the cell's surface polygons; ball == NULL keeps all */
static uint64_t cell_area_fx(const double f[8], const double P[8][3], const double *ball, double r2) {
    uint64_t acc = 0;
    for (int t = 0; t < 6; ++t) {
        int v[4];
        v[0] = 0;
        v[1] = 1 << KUHN[t][0];
        v[2] = v[1] | (1 << KUHN[t][1]);
        v[3] = 7;
        int in[4], out[4], ni = 0, no = 0;
        for (int c = 0; c < 4; ++c) {
            if (f[v[c]] > 0.0) in[ni++] = v[c];
            else out[no++] = v[c];
        }
        if (ni == 0 || no == 0) continue;
        double a[3], b[3], c3[3], d[3], area, gx, gy, gz;
        if (ni == 1 || no == 1) {
            if (ni == 1) {
                edge_point(P[in[0]], P[out[0]], f[in[0]], f[out[0]], a);
                edge_point(P[in[0]], P[out[1]], f[in[0]], f[out[1]], b);
                edge_point(P[in[0]], P[out[2]], f[in[0]], f[out[2]], c3);
            } else {
                edge_point(P[in[0]], P[out[0]], f[in[0]], f[out[0]], a);
                edge_point(P[in[1]], P[out[0]], f[in[1]], f[out[0]], b);
                edge_point(P[in[2]], P[out[0]], f[in[2]], f[out[0]], c3);
            }
            area = cross_half_norm(b[0] - a[0], b[1] - a[1], b[2] - a[2], c3[0] - a[0], c3[1] - a[1], c3[2] - a[2]);
            gx = ((a[0] + b[0]) + c3[0]) / 3.0;
            gy = ((a[1] + b[1]) + c3[1]) / 3.0;
            gz = ((a[2] + b[2]) + c3[2]) / 3.0;
        } else {
            /* quad a=(i0,o0) b=(i0,o1) c=(i1,o1) d=(i1,o0): a cycle, planar */
            edge_point(P[in[0]], P[out[0]], f[in[0]], f[out[0]], a);
            edge_point(P[in[0]], P[out[1]], f[in[0]], f[out[1]], b);
            edge_point(P[in[1]], P[out[1]], f[in[1]], f[out[1]], c3);
            edge_point(P[in[1]], P[out[0]], f[in[1]], f[out[0]], d);
            area = cross_half_norm(c3[0] - a[0], c3[1] - a[1], c3[2] - a[2], d[0] - b[0], d[1] - b[1], d[2] - b[2]);
            gx = (((a[0] + b[0]) + c3[0]) + d[0]) * 0.25;
            gy = (((a[1] + b[1]) + c3[1]) + d[1]) * 0.25;
            gz = (((a[2] + b[2]) + c3[2]) + d[2]) * 0.25;
        }
        if (ball) {
            double dx = gx - ball[0], dy = gy - ball[1], dz = gz - ball[2];
            if (!((dx * dx + dy * dy) + dz * dz <= r2)) continue;
        }
        acc += (uint64_t)llrint(area * VRO_AREA_SCALE);
    }
    return acc;
}

static uint64_t cell_at(const int16_t *vals, int64_t nx, int64_t ny, int64_t nz, double sx, double sy,
                        double sz, double level, int64_t i, int64_t j, int64_t k, const double *ball,
                        double r2) {
    double f[8], P[8][3];
    int any_in = 0, any_out = 0;
    for (int c = 0; c < 8; ++c) {
        int64_t a = i + (c & 1), b = j + ((c >> 1) & 1), e = k + ((c >> 2) & 1);
        f[c] = field_at(vals, nx, ny, nz, a, b, e, level);
        P[c][0] = (double)a * sx;
        P[c][1] = (double)b * sy;
        P[c][2] = (double)e * sz;
        if (f[c] > 0.0) any_in = 1; else any_out = 1;
    }
    if (!any_in || !any_out) return 0;
    return cell_area_fx(f, P, ball, r2);
}

/* whole volume: out[0] = voxels >= thr, out[1] = surface area * 2^24 */
void vro_threshold_measure(const int16_t *vals, int64_t nx, int64_t ny, int64_t nz, double sx, double sy,
                           double sz, int32_t thr, uint64_t *out) {
    const double level = (double)thr - 0.5;
    uint64_t area = 0;
#pragma omp parallel for reduction(+ : area) schedule(dynamic, 1)
    for (int64_t k = -1; k < nz; ++k)
        for (int64_t j = -1; j < ny; ++j)
            for (int64_t i = -1; i < nx; ++i) area += cell_at(vals, nx, ny, nz, sx, sy, sz, level, i, j, k, NULL, 0.0);
    uint64_t c = 0;
    for (int64_t i = 0; i < nx * ny * nz; ++i) c += (vals[i] >= thr);
    out[0] = c;
    out[1] = area;
}

/* per ball: counts[q] = voxels >= thr with centre in the ball (vro_ball_counts),
 * area[q] = surface inside the ball * 2^24 (cells of the ball's bounding box
 * widened by one cell; the centroid test decides) */
void vro_ball_measure(const int16_t *vals, int64_t nx, int64_t ny, int64_t nz, double sx, double sy, double sz,
                      int32_t thr, const double *centres, const double *radii, int64_t nballs, uint64_t *counts,
                      uint64_t *area) {
    const double level = (double)thr - 0.5;
    vro_ball_counts(vals, nx, ny, nz, sx, sy, sz, thr, centres, radii, nballs, counts);
#pragma omp parallel for schedule(dynamic, 1)
    for (int64_t q = 0; q < nballs; ++q) {
        const double *c = centres + 3 * q;
        double rad = radii[q], r2 = rad * rad;
        int64_t i0 = (int64_t)floor((c[0] - rad) / sx) - 1, i1 = (int64_t)ceil((c[0] + rad) / sx) + 1;
        int64_t j0 = (int64_t)floor((c[1] - rad) / sy) - 1, j1 = (int64_t)ceil((c[1] + rad) / sy) + 1;
        int64_t k0 = (int64_t)floor((c[2] - rad) / sz) - 1, k1 = (int64_t)ceil((c[2] + rad) / sz) + 1;
        if (i0 < -1) i0 = -1;
        if (j0 < -1) j0 = -1;
        if (k0 < -1) k0 = -1;
        if (i1 > nx - 1) i1 = nx - 1;
        if (j1 > ny - 1) j1 = ny - 1;
        if (k1 > nz - 1) k1 = nz - 1;
        uint64_t a = 0;
        for (int64_t k = k0; k <= k1; ++k)
            for (int64_t j = j0; j <= j1; ++j)
                for (int64_t i = i0; i <= i1; ++i) a += cell_at(vals, nx, ny, nz, sx, sy, sz, level, i, j, k, c, r2);
        area[q] = a;
    }
}
