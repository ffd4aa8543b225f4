// vr_raycast.cuh -- arguments of the K3 ray-cast kernel (host + device view).
#pragma once
#include "vr_common.cuh"

namespace vr {

struct RenderArgs {
    // volume and its block layout (monolithic = one block spanning the volume)
    const int16_t *vol;
    BrickVol bv;  // the same voxels in 4^3 bricks (K1), read by every interpolation
    TexVol tv;    // VR_SAMPLER_TEX builds: the x-quad texture (sampling-path A/B)
    Layout L;
    Divisor dsx, dsy, dsz;  // spacing divisors (x = (o + t*d) / s)
    double ext_mm[3];       // (n-1)*s, volume.py:62-67

    // camera (render.py:125-156 or the orthographic variant)
    int projection, W, H, tx, ty, tw, th;
    int il_n, il_k;        // sort-first interleave: render cells c % il_n == il_k
    int il_packed;         // outputs packed slot after slot (else at row-major rectangle positions)
    int cells_x, ncells;   // 16x8 cells across the rectangle, total
    const int *cell_order; // persistent ray queue: slot -> cell (nullptr: row-major)
    int phase_cap;         // per-lane post-classified kernel: cheap steps per trip
    int slots;             // CTAs launched (cells rendered by this call)
    double pos[3], fwd[3], right[3], up[3];
    double half_w, half_h;
    // batched views (a turntable sweep): nviews frames of the same size, view
    // v's camera at views[14 v ..] = pos, fwd, right, up, half_w, half_h
    // (device; null: the one camera above).  Work items, outputs, totals and
    // blocks_hit are laid out view after view.
    int nviews;                // views in this launch (view0 .. view0 + nviews - 1)
    int view0;
    const double *views;
    long long items_per_view;  // slots * 128
    long long view_pix;        // output pixels per view
    int nblocks;               // blocks_hit entries per view

    // settings (render.py:361-425 resolved)
    double step, ref_step;
    PowSpec corr, shin;
    int mode, cubic, lighting, classify, skip_empty, chained;
    double isovalue, term_alpha, ka, kd, ks;
    double bg[4];
    const double *lut;
    int nlut;
    double lut_lo, lut_inv_w;
    const double *table;
    int ntbl;
    double tbl_lo, tbl_inv_w;
    const uint8_t *rgba;     // 4 planar (nz,ny,nx) uint8 channels (pre-classification)
    long long rgba_plane;    // elements per channel plane

    // block classification (K2 outputs; unused when skip_empty == 0)
    const uint8_t *empty;    // nblocks
    const float *box;        // nblocks x 8 (BlockRec): lo xyz - margin, empty, hi xyz + margin, 0
    const int *vmin, *vmax;  // nblocks (iso skip predicate)
    const int *uni;          // 6: union of the fitted global AABBs (lo xyz, hi xyz); lo > hi = none
    double margin;           // SKIP_MARGIN applied to every box
    double inv_step;         // 1 / step (leap estimates only; sample positions use step)

    // transparency culling (post-classification): dilated 4^3 cell min/max and
    // the LUT's first/last bins with nonzero opacity
    const short2 *cells;
    int ncx, ncy;
    const short2 *cubes;   // optional per unit cube interpolant bounds, 4^3 brick order (index as bv)
    const short2 *mcells;  // optional per 16^3 macro cell: union of its cells' bounds
    int nmx, nmy;
    const int *lut_range;
    int cull;
    // chained modes (iso, pre-integrated): transparency culling of runs whose
    // interpolated values provably produce no hit / no opacity.  Pre-integrated:
    // a (ntbl+1)^2 prefix count of table cells with alpha > 0 (square queries).
    const int *tbl_nz;
    // pre-classified: (first, last) int16 value whose alpha plane is non-zero;
    // cells / mcells then hold raw footprint bounds instead of interpolant bounds
    const int *pre_range;

    unsigned long long *work_counter;  // persistent kernel's ray queue head (zeroed per launch)
    unsigned long long *debug_times;   // VR_DEBUG_TIMES builds: per warp (start, end, smid, lanes used)

    // long rays handed over to the warp-cooperative kernel (HeavyRay records)
    void *heavy;
    unsigned long long *heavy_count;  // records pushed (zeroed per launch)
    unsigned long long *heavy_head;   // records claimed by the cooperative kernel
    unsigned long long *heavy_count_long;  // records pushed to the long-ray queue (stored after the short one)
    long long heavy_long;      // rays with at least this many samples left use the long queue
    long long heavy_cap;
    long long heavy_min_left;  // tail rays with at least this many samples left are handed over
    int heavy_after;           // ... and, before the queue drains, rays that took more steps than this
    int heavy_vis;             // ... or composited at least this many samples (dense rays)
    double heavy_vis_alpha;    // ... while still below this opacity (far from termination)

    // outputs (all optional)
    uint8_t *pixels;
    double *premult;
    double *depth;
    long long *taken, *skipped;
    uint8_t *blocks_hit;
    unsigned long long *totals;  // per view [5 v + 0] taken, [5 v + 1] skipped
    unsigned long long *work;    // [0] gradient evaluations, [1] interpolations, [2] loop iterations
};

// CTA = 16 x 8 pixels, four warps, each warp an 8 x 4 screen tile so that the
// rays of a warp stay spatially coherent (SIMT efficiency 0.80 for
// 8x4 tiles vs 0.59 for row-major warps).
constexpr int kTileW = 16;
constexpr int kTileH = 8;
constexpr int kThreads = 128;
#ifndef VR_PERSIST_THREADS
#define VR_PERSIST_THREADS 32  // one warp per CTA: resources free warp by warp (C3 +1 %)
#endif
constexpr int kPersistThreads = VR_PERSIST_THREADS;  // CTA size of the persistent ray casters
constexpr size_t kHeavyRayBytes = 128;  // sizeof(HeavyRay) in vr_raycast.cu
constexpr size_t kChainRecBytes = 144;  // sizeof(ChainRec): chained-mode hand-off record
// views per persistent launch pair of a batched sweep; measured at C5:
// 1 (901 views/s) > 4 (844) > 16 (831) -- each view's tail rays are best
// handed to the cooperative kernel as in a single frame
#ifndef VR_VIEW_CHUNK
#define VR_VIEW_CHUNK 1
#endif
constexpr int kViewChunk = VR_VIEW_CHUNK;

cudaError_t launch_raycast(const RenderArgs &a, cudaStream_t stream);

}  // namespace vr
