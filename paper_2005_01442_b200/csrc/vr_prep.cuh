// vr_prep.cuh -- K1/K2 kernels: volume statistics, synthetic phantoms, block
// min/max (decompose), transfer-function visibility (cull_empty +
// fit_bounding_box), preclassification, point sampling and the K4 volume
// measure.  Launchers return the launch error; all work is stream-ordered.
#pragma once
#include "vr_common.cuh"

namespace vr {

// value range of the whole volume (make_volume, volume.py:74-79); out[0]=min, out[1]=max
cudaError_t launch_value_range(const int16_t *vol, long long n, int *out, cudaStream_t s);

// phantoms.py:98-111 on the device
cudaError_t launch_phantom(int kind, int nx, int ny, int nz, int16_t *out, cudaStream_t s);

// decompose() min/max (blocks.py:133-145); vmin/vmax int32 [nblocks]
cudaError_t launch_block_minmax(const int16_t *vol, const Layout &L, int *vmin, int *vmax,
                                cudaStream_t s);

// Per-frame zeroing folded into the first kernel of a frame (instead of a
// memset launch each): up to three u64 ranges and one byte range.
struct ZeroSpec {
    unsigned long long *p[3];
    int n[3];
    uint8_t *b;
    int nb;
};

VR_D void zero_fill(const ZeroSpec &z) {
    for (int k = 0; k < 3; ++k)
        for (int i = threadIdx.x; i < z.n[k]; i += blockDim.x) z.p[k][i] = 0ull;
    for (int i = threadIdx.x; i < z.nb; i += blockDim.x) z.b[i] = 0;
}

// Visibility state for one LUT (blocks.py:161-220).
struct VisArgs {
    const double *lut;  // (nbins, 4)
    int nbins;
    double lut_lo, bin_width;
    const int *vmin, *vmax;
    int nblocks;
    // outputs
    unsigned int *visbits;   // 65536 bits: int16 value v visible <=> bit (v + 32768)
    uint8_t *empty;          // nblocks
    int *aabb;               // nblocks x 6 local min/max (x,y,z) of visible voxels
    float *box;              // nblocks x 8: box lo xyz - margin, empty flag, hi xyz + margin, 0 (BlockRec)
    long long *aabb_global;  // optional nblocks x 6 int64 inclusive global aabb (lo xyz, hi xyz)
    unsigned long long *counters;  // [0] empty blocks, [1] non-empty blocks without a visible voxel
    int *uni;                // 6: union of the fitted global AABBs (lo xyz, hi xyz)
    int *list;               // nblocks + 1: [0] = count, then the non-empty block ids (any order)
    int *visprefix;          // 2049: visible values in visbits words [0, w)
    const short2 *cells;     // the volume's 4^3 cell bounds (cover every voxel value of the cell)
    int ncx, ncy, ncz;
    const short2 *mcells;    // unions over 4^3 cells (16^3 voxels): whole layers of a block skipped at once
    int nmx, nmy;
    double margin;
    int *lut_range;          // optional out (4 ints): as launch_lut_range
    double lut_inv_w;        // the march's bin scale nbins / (hi - lo) (render.py:423)
    ZeroSpec zero;           // zeroed by the setup kernel (frame counters, totals, blocks_hit)
};
cudaError_t launch_visibility(const int16_t *bricks, const Layout &L, const VisArgs &v,
                              cudaStream_t s);

// K1 brick upload: re-lay the x-fastest volume into 4x4x4 bricks of 64 voxels
// (128 bytes, x fastest inside a brick, bricks x-fastest), padded with zeros
// to whole bricks; bn* = ceil(n*/4).
cudaError_t launch_brick_volume(const int16_t *vol, int nx, int ny, int nz, int16_t *bricks, cudaStream_t s);

constexpr int kCell = 4;  // culling cell = 4^3 unit cubes

// Interpolant bounds (TF-independent, once per volume).  cubes[g] (brick
// order, bnx/bny as the int16 bricks) = (lo, hi) such that every trilinear or
// Catmull-Rom value of a sample whose base index is g -- under any block-local
// clamping of its taps -- lies in [lo, hi]; a bound at the int16 limit is
// saturated and proves nothing on that side.  cells[c] = union over the 4^3
// cubes of cell c (ncx = ceil(nx/4), ...); mcells[m] = union over the 4^3
// cells of the 16^3 macro cell m (nmx = ceil(nx/16), ...).
cudaError_t launch_interp_bounds(const int16_t *vol, int nx, int ny, int nz, int bnx, int bny, short2 *cubes,
                                 int ncx, int ncy, int ncz, short2 *cells, int nmx, int nmy, int nmz, short2 *mcells,
                                 cudaStream_t s);

// range[0] = first LUT bin with nonzero opacity (nbins if none),
// range[1] = last such bin (-1 if none)
// range[0..1] as above, range[2..3] = the integer value thresholds of that bin range
// under the march's bin formula (visible_value_range, lut_inv_w = nbins / (hi - lo))
// 2-D prefix count of pre-integrated table cells with opacity > 0 ((n+1)^2 ints)
// pre-classified culling: raw footprint bounds per cell / macro cell (once per
// volume) and the per-frame non-zero-alpha value range
cudaError_t launch_raw_bounds(const int16_t *vol, int nx, int ny, int nz, int ncx, int ncy, int ncz, short2 *rcells,
                              int nmx, int nmy, int nmz, short2 *rmcells, cudaStream_t s);
cudaError_t launch_pre_range(const double *lut, int nbins, double lut_lo, double bin_width, int vmin, int vmax,
                             int *out, cudaStream_t s);
cudaError_t launch_tbl_nonzero(const double *table, int n, int *nz, cudaStream_t s);
cudaError_t launch_lut_range(const double *lut, int nbins, double lut_lo, double lut_inv_w, int *range,
                             const ZeroSpec &zero, cudaStream_t s);

// blocks_visited = sum(blocks_hit) -> *out (render.py:467)
// also copies the two visibility counters (blocks_empty, empty-block errors)
// to out[1..2] when vis_counters is given
cudaError_t launch_xquads(const int16_t *vol, int nx, int ny, int nz, unsigned long long surf, cudaStream_t s);
cudaError_t launch_count_hits(const uint8_t *hits, int n, int nviews, unsigned long long *totals,
                              const unsigned long long *vis_counters, cudaStream_t s);

// preclassify_volume (transfer.py:142-145): 4 planar uint8 channels
cudaError_t launch_preclassify(const int16_t *vol, long long n, const double *lut, int nbins,
                               double lut_lo, double bin_width, uint8_t *rgba, cudaStream_t s);

// sample_points / gradient_points (_kernels.py:169-187)
cudaError_t launch_sample_points(const int16_t *vol, int nx, int ny, int nz, const double *pts,
                                 long long n, int cubic, int gradient, double sx, double sy,
                                 double sz, double *out, cudaStream_t s);

// K0 ingest: samples as read from a raw file or DICOM slices -> int16 volume.
// format 0 = u8, 1 = i16, 2 = u16 (volume.py:85-109 load_raw: u16 values above
// 32767 clamped and counted), 3 = i32 (a DICOM series mixing signed and
// unsigned slices, widened on the host; calibrated only).  With calib (2 doubles per z-slice: slope,
// intercept) every sample is calibrated as in dicom.py:287-290 instead:
// slope * s + intercept in float64, counted when outside [-32768, 32767],
// rint(clip) -> int16.
constexpr int kFormatU8 = 0, kFormatI16 = 1, kFormatU16 = 2, kFormatI32 = 3;
cudaError_t launch_ingest(const void *src, int format, long long nxy, int nz, const double *calib,
                          int16_t *out, unsigned long long *clamped, cudaStream_t s);

// K4: voxels >= thr
cudaError_t launch_threshold_count(const int16_t *vol, long long n, int thr,
                                   unsigned long long *count, cudaStream_t s);
// K4 ball form
// K4 method of spheres (vr_measure.cu): whole-volume count + isosurface area
// (out[0..1], zeroed by the call), and per ball count + area (areas may be null)
cudaError_t launch_threshold_measure(const int16_t *vol, int nx, int ny, int nz, double sx, double sy,
                                     double sz, int thr, unsigned long long *out, cudaStream_t s);
cudaError_t launch_ball_measure(const int16_t *vol, int nx, int ny, int nz, double sx, double sy, double sz,
                                int thr, const double *centres, const double *radii, int nballs,
                                unsigned long long *counts, unsigned long long *areas, cudaStream_t s);

// image metrics (vr_quality.cu; quality.py:37-79): exact sum of squared RGB
// differences, and the sum of the SSIM map over the valid region
cudaError_t launch_image_sse(const uint8_t *a, const uint8_t *b, long long npix, int ca, int cb,
                             unsigned long long *sse, cudaStream_t s);
size_t image_ssim_scratch(int h, int w);
cudaError_t launch_image_ssim(const uint8_t *a, const uint8_t *b, int h, int w, int ca, int cb, const double *win_host,
                              void *scratch, double *out_sum, cudaStream_t s);

}  // namespace vr
