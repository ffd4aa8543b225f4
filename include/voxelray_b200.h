/*
 * voxelray_b200.h -- C ABI of the B200-native volume ray caster.
 *
 * Drop-in boundary for the reference's native hot path.  The reference
 * (Python package `voxelray`, /root/reference/pkg/src/voxelray) crosses into
 * native code at exactly one place, the numba kernel `_kernels.march`
 * (_kernels.py:279-331, called from render.py:438-452), with its block prep
 * done in numpy (blocks.py:110-220) and the point sampler in numba
 * (_kernels.py:169-187).  Each entry point below names the reference
 * interface it replaces.  Plain pointers and sizes only; no torch types.
 *
 * Conventions
 *  - Every function returns VR_OK (0) or a VR_E* status; vr_last_error()
 *    returns a thread-local message for the last failure on this thread.
 *    The Python host maps statuses to the reference's exception classes
 *    (errors.py:9-97): VR_EINVALID -> InvalidSettings, VR_EBLOCKSPEC ->
 *    InvalidBlockSpec, VR_EISO -> IsovalueOutOfRange.
 *  - Volumes are int16, (nz, ny, nx) C order, x fastest (volume.py:23-55).
 *  - `stream` is a cudaStream_t passed as void* (NULL = legacy default
 *    stream).  Calls are asynchronous on that stream unless documented as
 *    synchronous; distinct streams may be used concurrently (the reference's
 *    HTTP service renders from a thread pool, service.py:213-226).
 *  - Pointers documented as "device" must be device (or managed) memory on
 *    the volume's device; "host" pointers are ordinary host memory (pinned
 *    memory makes the copies asynchronous).
 */
#ifndef VOXELRAY_B200_H
#define VOXELRAY_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define VR_ABI_VERSION 1

enum vr_status {
    VR_OK = 0,
    VR_EINVALID = 1,   /* invalid argument / settings (InvalidSettings) */
    VR_EBLOCKSPEC = 2, /* block_size/overlap out of range (InvalidBlockSpec) */
    VR_EISO = 3,       /* isovalue outside the value range (IsovalueOutOfRange) */
    VR_ECUDA = 4,      /* CUDA runtime failure */
    VR_ENOMEM = 5      /* device allocation failed */
};

/* _kernels.py:24-31 */
enum vr_mode { VR_MODE_DVR = 0, VR_MODE_ISO = 1 };
enum vr_classify { VR_CLS_POST = 0, VR_CLS_PRE = 1, VR_CLS_PREINT = 2 };
enum vr_projection { VR_PINHOLE = 0, VR_ORTHOGRAPHIC = 1 };
enum vr_phantom { VR_PHANTOM_SPHERE = 0, VR_PHANTOM_SHELL = 1, VR_PHANTOM_TORSO = 2 };

typedef struct vr_volume vr_volume; /* device-resident int16 volume (+ cached min/max) */
typedef struct vr_grid vr_grid;     /* overlapping block decomposition of a volume */

/* Camera: a pinhole camera as render.py:56-144 defines it (basis from
 * Camera.basis(), half_h = tan(fov/2), half_w = half_h*W/H computed by the
 * caller exactly as the reference does), or the orthographic variant
 * (SURVEY G1): origin = (position + u*right) + v*up, direction = fwd, with
 * half_w/half_h in millimetres.  The rendered rectangle is columns
 * [tile_x, tile_x+tile_w) and rows [tile_y, tile_y+tile_h) of a
 * width x height frame (sub-rectangle == crop of the full frame).
 *
 * Sort-first interleaving (multi-GPU): with interleave_n > 1 the
 * rectangle is cut into 16x8-pixel cells, numbered row-major, and only cells
 * c with c % interleave_n == interleave_k are rendered; outputs are then
 * packed cell after cell (cell c at slot c / interleave_n, 128 pixels each,
 * row-major inside the cell), so equal-size buffers from every rank
 * reassemble the frame with one gather.  With interleave_frame = 1 the cells
 * are instead written at their row-major positions of the whole rectangle
 * (buffers sized tile_w * tile_h), so every rank can store straight into one
 * shared frame -- e.g. rank 0's, mapped into the others over NVLink (CUDA IPC)
 * -- and the gather disappears into the kernels' epilogue.  interleave_n <= 1
 * renders the rectangle with row-major outputs. */
typedef struct {
    int32_t projection; /* vr_projection */
    int32_t width, height;
    int32_t tile_x, tile_y, tile_w, tile_h;
    int32_t interleave_n, interleave_k;
    int32_t interleave_frame; /* 1: interleaved cells at full-frame positions */
    double position[3];
    double fwd[3], right[3], up[3];
    double half_w, half_h;
} vr_camera;

/* Everything about a render except camera and tables; the fields of
 * RenderSettings (render.py:159-181) after render.py:361-425 resolved them. */
typedef struct {
    double step, ref_step;
    int32_t mode, cubic, lighting, classify;
    double isovalue, term_alpha;
    double ka, kd, ks, shininess;
    double bg[4];
    double lut_lo, lut_hi; /* transfer-function domain; LUT bins = nlut */
    int32_t nlut, ntbl;    /* LUT bins (4096), pre-integration bins (256) */
    double margin;         /* SKIP_MARGIN (render.py:53): 2.0 trilinear, 3.0 tricubic */
} vr_render_params;

/* Render outputs; every pointer is optional (NULL = not written).
 * Device pointers, sized for the tile (tile_w*tile_h pixels, row-major). */
typedef struct {
    uint8_t *pixels;     /* tile_h*tile_w*4 straight RGBA (render.py:454-459) */
    double *premult;     /* tile_h*tile_w*4 premultiplied float64 (march `out`) */
    double *depth;       /* tile_h*tile_w, NaN where no iso hit */
    int64_t *taken;      /* per-pixel samples taken */
    int64_t *skipped;    /* per-pixel samples skipped */
    uint8_t *blocks_hit; /* grid block count (1 when monolithic) */
    uint64_t *totals;    /* [5]: samples_taken, samples_skipped,
                            blocks_visited, blocks_empty, and the number of
                            non-empty blocks without a visible voxel (the
                            reference raises EmptyBlock for those,
                            blocks.py:186-187) -- the last three written, and
                            blocks_visited only when blocks_hit is given */
    uint64_t *work;      /* [3] optional: gradient evaluations (shaded samples),
                            interpolated samples (taken minus culled), march-loop iterations.
                            totals, work and blocks_hit are zeroed by the call itself
                            (in its first kernel) */
    void *ev_start;      /* optional cudaEvent_t recorded just before the ray-cast kernel */
    void *ev_stop;       /* optional cudaEvent_t recorded just after it */
} vr_render_outputs;

/* cells per rank and pixels per rank buffer for an interleaved render */
int vr_interleave_size(const vr_camera *cam, int64_t *cells_per_rank, int64_t *pixels_per_rank);

const char *vr_last_error(void);
int vr_abi_version(void);

/* CUDA events for timing a launch on its own stream (bench / profiling). */
int vr_event_create(void **ev);
int vr_event_destroy(void *ev);
int vr_event_elapsed_ms(void *start, void *stop, float *ms); /* synchronizes on stop */

/* ---------------------------------------------------------------- volumes */

/* Upload an int16 (nz,ny,nx) volume (K1).  Replaces ScalarVolume construction
 * (volume.py:23-79) on the device side; value_range is computed on the GPU.
 * src is host memory when src_on_device == 0, else device memory. Synchronous. */
int vr_volume_create(int device, int64_t nx, int64_t ny, int64_t nz, double sx, double sy,
                     double sz, const int16_t *src, int src_on_device, void *stream,
                     vr_volume **out);
/* Ingest raw samples (host or device pointer) into a device volume, converting
 * on the device.  format: VR_SAMPLE_U8 / _I16 / _U16 / _I32, samples
 * little-endian (nz,ny,nx) x fastest.  Replaces volume.py:85-109 load_raw (u16
 * values > 32767 clamped and counted) and, with calib = nz (slope, intercept)
 * pairs, the calibration of dicom.py:254-295 assemble_volume (slope*s +
 * intercept in float64, counted when outside int16, rint(clip)); the geometry
 * checks and slice ordering stay on the host.  *clamp_count (optional) receives
 * the number of clamped samples.  Synchronous. */
#define VR_SAMPLE_U8 0
#define VR_SAMPLE_I16 1
#define VR_SAMPLE_U16 2
#define VR_SAMPLE_I32 3 /* calibrated only: a series mixing signed and unsigned slices */
int vr_volume_ingest(int device, int format, int64_t nx, int64_t ny, int64_t nz, double sx, double sy,
                     double sz, const void *src, int src_on_device, const double *calib, void *stream,
                     vr_volume **out, uint64_t *clamp_count);
/* Generate a synthetic CT phantom on the device, bit-identical to
 * phantoms.py:98-111 generate_phantom(kind, (nx,ny,nz), spacing).  Synchronous. */
int vr_phantom_create(int device, int kind, int64_t nx, int64_t ny, int64_t nz, double sx,
                      double sy, double sz, void *stream, vr_volume **out);
int vr_volume_destroy(vr_volume *vol);
/* Copy the transparency-culling tables K1 built (host buffers, synchronous):
 * cubes = ceil(nx/4)*ceil(ny/4)*ceil(nz/4)*64 (lo, hi) int16 pairs in 4^3 brick
 * order (entry of voxel g: brick (gz/4, gy/4, gx/4) x-fastest, then
 * (gz%4, gy%4, gx%4) x-fastest; padding entries undefined): every trilinear or
 * Catmull-Rom value of a sample whose base index is g lies in [lo, hi] unless
 * saturated at the int16 limit; cells = ceil(n/4)^3 pairs, the union over
 * each brick.  Either pointer may be NULL.  (Test / inspection entry point.) */
int vr_volume_culling_tables(const vr_volume *vol, int16_t *cubes, int16_t *cells);
/* dims = (nx, ny, nz), spacing = (sx, sy, sz), value_range = (min, max) */
int vr_volume_info(const vr_volume *vol, int64_t dims[3], double spacing[3],
                   int32_t value_range[2], int *device);
/* device pointer to the (nz,ny,nx) int16 values */
const int16_t *vr_volume_data(const vr_volume *vol);
/* copy values to host memory (synchronous) */
int vr_volume_download(const vr_volume *vol, int16_t *dst, void *stream);

/* ----------------------------------------------------------------- blocks */

/* decompose() (blocks.py:110-158): block layout + per-block min/max (K2a).
 * Raises VR_EBLOCKSPEC unless block_size >= 8 and 1 <= overlap < block_size.
 * Synchronous. */
int vr_grid_create(vr_volume *vol, int64_t block_size, int64_t overlap, void *stream,
                   vr_grid **out);
int vr_grid_destroy(vr_grid *grid);
/* shape = (nbx, nby, nbz) */
int vr_grid_shape(const vr_grid *grid, int64_t shape[3]);
/* vmin/vmax host arrays of nbz*nby*nbx int64 in (bk,bj,bi) order; synchronous */
int vr_grid_minmax(const vr_grid *grid, int64_t *vmin, int64_t *vmax, void *stream);
/* with_visibility() (blocks.py:161-220, K2b): classify the blocks against a
 * LUT (lut_rgba: host (nbins,4) float64 straight RGBA at bin centres, as
 * transfer.py:136-139 builds it, over domain [lut_lo, lut_hi]).  Writes host
 * arrays: empty (nblocks uint8), aabb_lo/aabb_hi (nblocks*3 int64, x,y,z,
 * global inclusive voxel indices; empty blocks keep INT64_MAX/2 and -1).
 * Synchronous. */
int vr_grid_visibility(const vr_grid *grid, const double *lut_rgba, int32_t nbins,
                       double lut_lo, double lut_hi, uint8_t *empty, int64_t *aabb_lo,
                       int64_t *aabb_hi, void *stream);

/* ----------------------------------------------------------------- render */

/* _kernels.march + its prep (render.py:361-459) on the device (K2b + K3).
 * grid == NULL renders the monolithic layout (use_blocks=False); otherwise
 * the block layout with empty-space leaping, TF visibility recomputed from
 * the LUT on every call.  Tables are DEVICE pointers:
 *   lut   (nlut,4) float64  -- always
 *   table (ntbl,ntbl,4) float64 pre-integrated (classify == PREINT), else NULL
 *   rgba  (nz,ny,nx,4) uint8 preclassified volume, RGBA interleaved per voxel (classify == PRE),
 *         as transfer.py:142-145 paints them (see vr_preclassify), else NULL.
 * Outputs as in vr_render_outputs (device).  Asynchronous on `stream`. */
int vr_render(vr_volume *vol, vr_grid *grid, const vr_camera *cam, const vr_render_params *prm,
              const double *lut, const double *table, const uint8_t *rgba,
              const vr_render_outputs *out, void *stream);

/* A batch of views in one submission -- the turntable sweep of BASELINE
 * configs[4] (the reference's viewer orbits the camera, frontend/src/camera.ts
 * :35-44, and renders each view with its own render() call, render.py:327).
 * Every view is the frame `frame` describes (size, tile, projection,
 * interleave) seen from views[14 v .. 14 v + 13] = position[3], fwd[3],
 * right[3], up[3], half_w, half_h (device float64, v < nviews).  The TF
 * visibility (K2b) runs once for the batch, then one persistent ray-cast pass
 * takes the rays of all views from one queue.  Outputs are laid out view after
 * view: pixels / premult / depth / taken / skipped at v * (pixels per view),
 * blocks_hit at v * nblocks, totals at 5 v (work: the whole batch).  Each
 * view's outputs equal vr_render's for that camera.  Asynchronous. */
int vr_render_views(vr_volume *vol, vr_grid *grid, const vr_camera *frame, const double *views,
                    int32_t nviews, const vr_render_params *prm, const double *lut,
                    const double *table, const uint8_t *rgba, const vr_render_outputs *out,
                    void *stream);

/* Reference-facing host entry: same as vr_render with HOST tables and HOST
 * outputs (pixels required, others optional; totals_host[5] required).  The
 * library stages tables/outputs through stream-ordered device memory; the
 * volume (and grid) are already resident.  Synchronous. */
int vr_render_to_host(vr_volume *vol, vr_grid *grid, const vr_camera *cam,
                      const vr_render_params *prm, const double *lut_host,
                      const double *table_host, uint8_t *pixels_host, double *premult_host,
                      double *depth_host, uint64_t *totals_host, void *stream);

/* preclassify_volume (transfer.py:142-145) on the device: rgba_out holds the
 * (nz,ny,nx,4) uint8 array the reference returns, rint(lut[bin(v)] * 255).  lut is a device
 * pointer.  Asynchronous. */
int vr_preclassify(const vr_volume *vol, const double *lut, int32_t nbins, double lut_lo,
                   double lut_hi, uint8_t *rgba_out, void *stream);

/* --------------------------------------------------------------- sampling */

/* sample_points / gradient_points (_kernels.py:169-187): pts (n,3) continuous
 * voxel coordinates (x,y,z), device pointers.  gradient out (n,3) per mm. */
int vr_sample_points(const vr_volume *vol, const double *pts, int64_t n, int cubic,
                     double *out, void *stream);
int vr_gradient_points(const vr_volume *vol, const double *pts, int64_t n, int cubic,
                       double *out, void *stream);

/* ------------------------------------------------------- volume measure K4 */

/* Number of voxels with value >= thr (builder-defined, no
 * reference function).  count: device uint64 (accumulated; zero it first). */
int vr_threshold_count(const vr_volume *vol, int32_t thr, uint64_t *count, void *stream);
/* The method of spheres on the voxel grid.  Replaces the
 * reference's mesh estimators morphology.py:70-143 clipped_area (S),
 * :238-267 clipped_volume (V) and :270-306 svr_at_point (SVR = S/V) for a CT
 * volume thresholded at thr:
 *   V = (voxels with value >= thr [and centre (i*sx, j*sy, k*sz) in the closed
 *       ball, ((dx^2 + dy^2) + dz^2) <= r^2]) * sx*sy*sz;
 *   S = area (mm^2) of the isosurface at level thr - 0.5 of the piecewise-
 *       linear interpolant over the 6 Kuhn tetrahedra of every cell (cells
 *       between voxel centres, the volume padded with -32768 so the surface
 *       closes at its border) [polygons with vertex centroid in the ball],
 *       each polygon rounded to a multiple of 2^-24 mm^2: area_fx = S * 2^24
 *       as an exact integer sum.
 * vr_threshold_measure: out[0] = count, out[1] = area_fx for the whole volume
 * (device uint64[2], overwritten).  vr_ball_measure: per ball q (centres
 * (nballs,3) mm, radii (nballs) mm, device float64) counts[q] and, unless
 * area_fx is NULL, area_fx[q] (device uint64, overwritten).  Asynchronous. */
#define VR_AREA_SCALE 16777216.0 /* 2^24 */
int vr_threshold_measure(const vr_volume *vol, int32_t thr, uint64_t *out, void *stream);
int vr_ball_measure(const vr_volume *vol, int32_t thr, const double *centres, const double *radii,
                    int64_t nballs, uint64_t *counts, uint64_t *area_fx, void *stream);

/* Let kernels running on `device` read and write `peer`'s memory (NVLink P2P),
 * e.g. a frame of rank 0 mapped into another rank with interleave_frame = 1.
 * Idempotent; VR_EINVALID when the pair has no peer access. */
int vr_enable_peer_access(int device, int peer);

/* ---- image metrics (quality.py:37-79), device pointers, stream-ordered ----
 * a, b: uint8 (h, w, ca|cb) images, ca/cb = 3 or 4 (alpha ignored).
 * vr_image_sse: *sse (device) = sum over pixels and RGB of (a - b)^2, exact;
 *   psnr = 10 log10(255^2 / (sse / (3 h w))) capped at 99 dB on the host.
 * vr_image_ssim: *sum (device) = sum of the SSIM map over the valid region of
 *   the Rec. 601 luma planes with the 11x11 window `window` (host, float64,
 *   quality.py:50-54); ssim = sum / ((h - 10) (w - 10)). */
int vr_image_sse(const uint8_t *a, const uint8_t *b, int64_t h, int64_t w, int ca, int cb, uint64_t *sse,
                 void *stream);
int vr_image_ssim(const uint8_t *a, const uint8_t *b, int64_t h, int64_t w, int ca, int cb, const double *window,
                  double *sum, void *stream);

#ifdef __cplusplus
}
#endif
#endif /* VOXELRAY_B200_H */
