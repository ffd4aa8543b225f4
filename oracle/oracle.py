"""CPU oracle for the voxelray hot path -- TEST INFRASTRUCTURE ONLY.

Only tests/, ``__graft_entry__.smoke()`` and bench.py's cpu_baseline / ``--impl
reference`` legs may import this module, and only as the checker or as the timed
CPU baseline.  The product package (paper_2005_01442_b200) never imports it.

It restates the reference's render orchestration (``render.py:340-471``) on top
of ``vr_oracle.c`` (a C restatement of ``_kernels.march`` and the block prep) and
numpy restatements of the table builders.  Every function cites the reference
file:line it follows (relative to /root/reference/pkg/src/voxelray/).

Pinned: tests/test_oracle_golden.py compares this module bit-for-bit with
golden vectors that tests/golden/make_golden.py produced from the unmodified
reference.  The volume measure (K4) has no reference function: its
restatement here is "parity unpinned".
"""

from __future__ import annotations

import ctypes
import math
import os
import subprocess
from dataclasses import dataclass
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
LIB_PATH = HERE / "libvr_oracle.so"

MODE_DVR, MODE_ISO = 0, 1
CLS_POST, CLS_PRE, CLS_PREINT = 0, 1, 2
LUT_BINS = 4096
PREINT_BINS = 256
PREINT_SUBSTEPS = 64
SKIP_MARGIN = {"trilinear": 2.0, "tricubic": 3.0}  # render.py:53

# transfer.py:207-228 presets as (value, r, g, b, a) control points over the
# CT domain (-1000, 2000): the oracle's own copy, so the CPU baseline and the
# tests never need the product package for their inputs.
CT_DOMAIN = (-1000.0, 2000.0)
PRESET_POINTS = {
    "bone": [(-1000.0, 0, 0, 0, 0.0), (550.0, .40, .28, .16, 0.0), (800.0, .85, .78, .62, .70),
             (1400.0, .98, .96, .90, .95), (2000.0, 1, 1, 1, 1.0)],
    "soft-tissue": [(-1000.0, 0, 0, 0, 0.0), (-350.0, .55, .25, .15, 0.0), (-50.0, .70, .40, .30, .05),
                    (100.0, .80, .45, .35, .12), (500.0, .90, .80, .70, .40),
                    (900.0, .98, .95, .90, .85), (2000.0, 1, 1, 1, .95)],
    "grayscale": [(-1000.0, 0, 0, 0, 0.0), (2000.0, 1, 1, 1, 1.0)],
}


def preset_arrays(name: str):
    """(values, rgba, domain) of a preset TF (transfer.py:207-228)."""
    pts = PRESET_POINTS[name]
    v = np.array([p[0] for p in pts], dtype=np.float64)
    c = np.array([p[1:] for p in pts], dtype=np.float64)
    return v, c, CT_DOMAIN


_lib = None


def build(force: bool = False) -> Path:
    """Compile vr_oracle.c into libvr_oracle.so (oracle/Makefile recipe)."""
    src = HERE / "vr_oracle.c"
    if force or not LIB_PATH.exists() or LIB_PATH.stat().st_mtime < src.stat().st_mtime:
        subprocess.run(["make", "-s", "-C", str(HERE)], check=True)
    return LIB_PATH


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(str(LIB_PATH))
        P = ctypes.c_void_p
        i64, f64, i32 = ctypes.c_int64, ctypes.c_double, ctypes.c_int
        L.vro_march.argtypes = (
            [i64, P, P, P, P, f64, f64, f64, f64, f64, i32, i32, i32, i32, i32,
             P, P, P, P, P, P, P, P, P, i64, i64, i64, i64,
             P, P, P, P, P, P, i64, f64, f64, P, i64, f64, f64,
             f64, f64, f64, f64, f64, f64, f64, f64, f64, f64,
             P, P, P, P, P, i32]
        )
        L.vro_march.restype = None
        L.vro_ray_grid.argtypes = [P, P, P, P, f64, f64, i64, i64, i64, i64, i64, i64, P, P]
        L.vro_ortho_rays.argtypes = [P, P, P, P, f64, f64, i64, i64, i64, i64, i64, i64, P, P]
        L.vro_clip_to_bounds.argtypes = [i64, P, P, P, P, P]
        L.vro_axis_layout.argtypes = [i64, i64, i64, P, P]
        L.vro_axis_layout.restype = i64
        L.vro_block_minmax.argtypes = [P, i64, i64, i64, P, P, i64, P, P, i64, P, P, i64, P, P]
        L.vro_visibility.argtypes = [P, i64, i64, i64, P, P, i64, P, P, i64, P, P, i64, P, P,
                                     P, i64, f64, f64, P, P, P]
        L.vro_build_atlas.argtypes = [P, i64, i64, i64, P, P, i64, P, P, i64, P, P, i64, P, P]
        L.vro_threshold_count.argtypes = [P, i64, ctypes.c_int32]
        L.vro_threshold_count.restype = ctypes.c_uint64
        L.vro_ball_counts.argtypes = [P, i64, i64, i64, f64, f64, f64, ctypes.c_int32, P, P, i64, P]
        L.vro_threshold_measure.argtypes = [P, i64, i64, i64, f64, f64, f64, ctypes.c_int32, P]
        L.vro_ball_measure.argtypes = [P, i64, i64, i64, f64, f64, f64, ctypes.c_int32, P, P, i64, P, P]
        L.vro_sample_points.argtypes = [P, i64, i64, i64, P, i64, i32, P]
        L.vro_gradient_points.argtypes = [P, i64, i64, i64, P, i64, i32, f64, f64, f64, P]
        L.vro_num_threads.restype = i32
        _lib = L
    return _lib


def _p(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p)


def num_threads() -> int:
    return int(lib().vro_num_threads())


# ------------------------------------------------------------------ phantoms


def _voxel_grid(dims):  # phantoms.py:21-29
    nx, ny, nz = dims
    z, y, x = np.meshgrid(
        np.arange(nz, dtype=np.float64), np.arange(ny, dtype=np.float64),
        np.arange(nx, dtype=np.float64), indexing="ij",
    )
    return x, y, z


def _ellipsoid_blend(x, y, z, center, semi, width):  # phantoms.py:32-42
    cx, cy, cz = center
    ax, ay, az = semi
    e = np.sqrt(((x - cx) / ax) ** 2 + ((y - cy) / ay) ** 2 + ((z - cz) / az) ** 2)
    s_min = min(ax, ay, az)
    return np.clip((1.0 - e) * s_min / width + 0.5, 0.0, 1.0)


def phantom(name: str, dims) -> np.ndarray:
    """phantoms.py:45-111 restated; returns int16 (nz, ny, nx)."""
    dims = tuple(int(d) for d in dims)
    x, y, z = _voxel_grid(dims)
    if name == "sphere":  # phantoms.py:45-50
        c = [d // 2 for d in dims]
        r = np.sqrt((x - c[0]) ** 2 + (y - c[1]) ** 2 + (z - c[2]) ** 2)
        radius = min(dims) // 2
        field = np.clip(1000 - 2 * 1000 * r / radius, -1000, 1000)
    elif name == "shell":  # phantoms.py:53-60
        c = [(d - 1) / 2.0 for d in dims]
        r = np.sqrt((x - c[0]) ** 2 + (y - c[1]) ** 2 + (z - c[2]) ** 2)
        radius = min(dims) / 2.0
        d = np.maximum(0.55 * radius - r, r - 0.80 * radius)
        band = np.clip(0.5 - d / 1.5, 0.0, 1.0)
        field = -1000 + (800 - -1000) * band
    elif name == "torso":  # phantoms.py:63-79
        nx, ny, nz = dims

        def c(fx, fy, fz):
            return fx * nx, fy * ny, fz * nz

        body = _ellipsoid_blend(x, y, z, c(0.50, 0.63, 0.63), c(0.46, 0.29, 0.29), 2.0)
        spine = _ellipsoid_blend(x, y, z, c(0.50, 0.63, 0.71), c(0.40, 0.065, 0.065), 1.5)
        blob_l = _ellipsoid_blend(x, y, z, c(0.34, 0.60, 0.55), c(0.17, 0.10, 0.08), 1.5)
        blob_r = _ellipsoid_blend(x, y, z, c(0.68, 0.66, 0.56), c(0.12, 0.11, 0.09), 1.5)
        bone = np.maximum(spine, np.maximum(blob_l, blob_r))
        field = -1000 + (40 - -1000) * body + (1200 - 40) * bone
    else:
        raise ValueError(name)
    return np.rint(field).astype(np.int16)


# ------------------------------------------------------------- transfer/LUT


def tf_evaluate(values, rgba, scalars):  # transfer.py:56-62
    s = np.asarray(scalars, dtype=np.float64)
    out = np.empty(s.shape + (4,))
    for ch in range(4):
        out[..., ch] = np.interp(s, values, rgba[:, ch])
    return out


def build_lut(values, rgba, domain, bins: int = LUT_BINS) -> np.ndarray:
    """transfer.py:136-139: (bins, 4) float64 at bin centres."""
    lo, hi = domain
    centres = lo + (np.arange(bins) + 0.5) * (hi - lo) / bins
    return tf_evaluate(values, rgba, centres)


def lut_bin_index(lut_rgba, domain, scalars):  # transfer.py:120-125
    s = np.asarray(scalars, dtype=np.float64)
    lo, hi = domain
    bw = (hi - lo) / lut_rgba.shape[0]
    idx = np.floor((s - lo) / bw).astype(np.int64)
    return np.clip(idx, 0, lut_rgba.shape[0] - 1)


def preclassify(values_zyx, lut_rgba, domain) -> np.ndarray:  # transfer.py:142-145
    rgba = lut_rgba[lut_bin_index(lut_rgba, domain, values_zyx)]
    return np.rint(rgba * 255.0).astype(np.uint8)


def preintegrated(lut_rgba, domain, length, ref_step=None, bins=PREINT_BINS,
                  substeps=PREINT_SUBSTEPS) -> np.ndarray:
    """transfer.py:166-202: (bins, bins, 4) premultiplied segment table."""
    if ref_step is None:
        ref_step = length
    lo, hi = domain
    centres = lo + (np.arange(bins) + 0.5) * (hi - lo) / bins
    front = centres[:, None, None]
    back = centres[None, :, None]
    frac = (np.arange(substeps) + 0.5)[None, None, :] / substeps
    scalars = front + (back - front) * frac
    slice_rgba = lut_rgba[lut_bin_index(lut_rgba, domain, scalars)]
    ds = length / substeps
    a_hat = 1.0 - (1.0 - slice_rgba[..., 3]) ** (ds / ref_step)
    out = np.zeros((bins, bins, 4))
    trans = 1.0 - out[..., 3]
    for i in range(substeps):
        w = trans * a_hat[..., i]
        out[..., 0] += w * slice_rgba[..., i, 0]
        out[..., 1] += w * slice_rgba[..., i, 1]
        out[..., 2] += w * slice_rgba[..., i, 2]
        out[..., 3] += w
        trans = 1.0 - out[..., 3]
    return out


# ------------------------------------------------------------------ camera


def camera_basis(position, look_at, up):  # render.py:78-85
    fwd = np.subtract(look_at, position, dtype=np.float64)
    fwd /= np.linalg.norm(fwd)
    right = np.cross(fwd, np.asarray(up, dtype=np.float64))
    right /= np.linalg.norm(right)
    true_up = np.cross(right, fwd)
    return fwd, right, true_up


def rays(camera, projection="pinhole", ortho_half_h=None, tile=None):
    """render.py:125-144 (pinhole) or the orthographic variant.

    tile = (x0, y0, w, h) sub-rectangle of the frame; None = full frame.
    """
    fwd, right, up = camera_basis(camera.position, camera.look_at, camera.up)
    W, H = camera.width, camera.height
    x0, y0, w, h = tile if tile is not None else (0, 0, W, H)
    pos = np.asarray(camera.position, dtype=np.float64)
    origins = np.empty((w * h, 3))
    dirs = np.empty((w * h, 3))
    L = lib()
    if projection == "pinhole":
        half_h = math.tan(math.radians(camera.vertical_fov_deg) / 2.0)
        half_w = half_h * camera.width / camera.height
        L.vro_ray_grid(_p(pos), _p(fwd), _p(right), _p(up), half_w, half_h, W, H, x0, y0, w, h,
                       _p(origins), _p(dirs))
    elif projection == "orthographic":
        half_h = float(ortho_half_h)
        half_w = half_h * camera.width / camera.height
        L.vro_ortho_rays(_p(pos), _p(fwd), _p(right), _p(up), half_w, half_h, W, H, x0, y0, w, h,
                         _p(origins), _p(dirs))
    else:
        raise ValueError(projection)
    return origins, dirs


def clip_to_bounds(origins, dirs, extent_mm):  # render.py:147-156
    n = origins.shape[0]
    tmin = np.empty(n)
    tmax = np.empty(n)
    ext = np.asarray(extent_mm, dtype=np.float64)
    lib().vro_clip_to_bounds(n, _p(origins), _p(dirs), _p(ext), _p(tmin), _p(tmax))
    return tmin, tmax


# ------------------------------------------------------------------ blocks


@dataclass
class OracleGrid:
    block_size: int
    overlap: int
    origins: tuple
    extents: tuple
    vmin: np.ndarray  # (nbz, nby, nbx) int64
    vmax: np.ndarray
    empty: np.ndarray | None = None  # (nbz, nby, nbx) bool
    aabb_lo: np.ndarray | None = None  # (nbz, nby, nbx, 3) int64
    aabb_hi: np.ndarray | None = None

    @property
    def shape(self):
        return tuple(len(o) for o in self.origins)

    @property
    def stride(self):
        return self.block_size - self.overlap

    @property
    def count(self):
        a, b, c = self.shape
        return a * b * c


def axis_layout(n, block_size, stride):  # blocks.py:100-107
    L = lib()
    cnt = L.vro_axis_layout(n, block_size, stride, None, None)
    o = np.empty(cnt, dtype=np.int64)
    e = np.empty(cnt, dtype=np.int64)
    L.vro_axis_layout(n, block_size, stride, _p(o), _p(e))
    return o, e


def decompose(values_zyx, block_size=64, overlap=3) -> OracleGrid:  # blocks.py:110-158
    vals = np.ascontiguousarray(values_zyx, dtype=np.int16)
    nz, ny, nx = vals.shape
    stride = block_size - overlap
    ox, ex = axis_layout(nx, block_size, stride)
    oy, ey = axis_layout(ny, block_size, stride)
    oz, ez = axis_layout(nz, block_size, stride)
    vmin = np.empty((len(oz), len(oy), len(ox)), dtype=np.int64)
    vmax = np.empty_like(vmin)
    lib().vro_block_minmax(_p(vals), nx, ny, nz, _p(ox), _p(ex), len(ox), _p(oy), _p(ey), len(oy),
                           _p(oz), _p(ez), len(oz), _p(vmin), _p(vmax))
    return OracleGrid(block_size, overlap, (ox, oy, oz), (ex, ey, ez), vmin, vmax)


def with_visibility(values_zyx, grid: OracleGrid, lut_rgba, domain) -> OracleGrid:
    """blocks.py:161-220 (cull_empty + fit_bounding_box per block)."""
    vals = np.ascontiguousarray(values_zyx, dtype=np.int16)
    nz, ny, nx = vals.shape
    (ox, oy, oz), (ex, ey, ez) = grid.origins, grid.extents
    nbz, nby, nbx = grid.vmin.shape
    empty = np.empty((nbz, nby, nbx), dtype=np.uint8)
    lo = np.empty((nbz, nby, nbx, 3), dtype=np.int64)
    hi = np.empty_like(lo)
    lut = np.ascontiguousarray(lut_rgba, dtype=np.float64)
    bw = (domain[1] - domain[0]) / lut.shape[0]
    lib().vro_visibility(_p(vals), nx, ny, nz, _p(ox), _p(ex), nbx, _p(oy), _p(ey), nby, _p(oz),
                         _p(ez), nbz, _p(grid.vmin), _p(grid.vmax), _p(lut), lut.shape[0],
                         float(domain[0]), bw, _p(empty), _p(lo), _p(hi))
    grid.empty = empty.astype(bool)
    grid.aabb_lo = lo
    grid.aabb_hi = hi
    return grid


def build_atlas(values_zyx, grid: OracleGrid):  # blocks.py:269-294
    vals = np.ascontiguousarray(values_zyx, dtype=np.int16)
    nz, ny, nx = vals.shape
    (ox, oy, oz), (ex, ey, ez) = grid.origins, grid.extents
    total = int(np.sum(ez[:, None, None] * ey[None, :, None] * ex[None, None, :]))
    atlas = np.empty(total, dtype=np.int16)
    offsets = np.empty(grid.count, dtype=np.int64)
    lib().vro_build_atlas(_p(vals), nx, ny, nz, _p(ox), _p(ex), len(ox), _p(oy), _p(ey), len(oy),
                          _p(oz), _p(ez), len(oz), _p(atlas), _p(offsets))
    return atlas, offsets


def build_rgba_atlas(grid: OracleGrid, rgba_volume):  # blocks.py:297-317
    (ox, oy, oz), (ex, ey, ez) = grid.origins, grid.extents
    parts = []
    nbx, nby, nbz = grid.shape
    for bk in range(nbz):
        for bj in range(nby):
            for bi in range(nbx):
                region = rgba_volume[oz[bk]:oz[bk] + ez[bk], oy[bj]:oy[bj] + ey[bj],
                                     ox[bi]:ox[bi] + ex[bi], :]
                for ch in range(4):
                    parts.append(np.ascontiguousarray(region[..., ch]).ravel())
    return np.concatenate(parts)


# ------------------------------------------------------------------ render


@dataclass
class OracleResult:
    out: np.ndarray  # (H*W, 4) premultiplied float64
    depth: np.ndarray  # (H*W,) float64, NaN where no iso hit
    taken: np.ndarray  # (H*W,) int64
    skipped: np.ndarray
    blocks_hit: np.ndarray  # (nblocks,) uint8
    pixels: np.ndarray  # (h, w, 4) uint8 straight RGBA
    blocks_total: int
    blocks_empty: int

    @property
    def samples_taken(self):
        return int(self.taken.sum())

    @property
    def samples_skipped(self):
        return int(self.skipped.sum())

    @property
    def blocks_visited(self):
        return int(self.blocks_hit.sum())


def to_pixels(out: np.ndarray, h: int, w: int) -> np.ndarray:
    """render.py:454-459: premultiplied float64 -> straight uint8."""
    premult = out.reshape(h, w, 4)
    alpha = premult[..., 3:4]
    straight = np.where(alpha > 0, premult[..., :3] / np.maximum(alpha, 1e-12), 0.0)
    pixels = np.empty((h, w, 4), dtype=np.uint8)
    pixels[..., :3] = np.rint(np.clip(straight, 0.0, 1.0) * 255.0)
    pixels[..., 3] = np.rint(np.clip(premult[..., 3], 0.0, 1.0) * 255.0)
    return pixels


def render(values_zyx, spacing, camera, tf_values, tf_rgba, tf_domain, settings, *,
           projection="pinhole", ortho_half_h=None, tile=None, nthreads=0,
           grid: OracleGrid | None = None) -> OracleResult:
    """render.py:340-471 restated over the C march.

    settings is any object with the RenderSettings fields (render.py:159-181).
    """
    vals = np.ascontiguousarray(values_zyx, dtype=np.int16)
    nz, ny, nx = vals.shape
    sx, sy, sz = (float(s) for s in spacing)
    extent = ((nx - 1) * sx, (ny - 1) * sy, (nz - 1) * sz)
    use_blocks = bool(settings.use_blocks) or grid is not None
    ref_step = 0.5 * min(spacing)
    step = settings.step if settings.step is not None else ref_step
    cubic = settings.interpolation == "tricubic"
    tf_values = np.asarray(tf_values, dtype=np.float64)
    tf_rgba = np.asarray(tf_rgba, dtype=np.float64)
    lut = build_lut(tf_values, tf_rgba, tf_domain)
    mode = MODE_ISO if settings.mode == "isosurface" else MODE_DVR
    classify = {"post": CLS_POST, "pre": CLS_PRE, "preintegrated": CLS_PREINT}[settings.classification]
    if mode == MODE_ISO:
        classify = CLS_POST
    vr_lo, vr_hi = int(vals.min()), int(vals.max())

    blocks_empty = 0
    if use_blocks:
        if grid is None:
            grid = decompose(vals, settings.block_size, settings.overlap)
        grid = with_visibility(vals, grid, lut, tf_domain)
        blocks_empty = int(np.count_nonzero(grid.empty))
        atlas, offsets = build_atlas(vals, grid)
        org_x, org_y, org_z = grid.origins
        ext_x, ext_y, ext_z = grid.extents
        stride = grid.stride
        vmin = grid.vmin.ravel().astype(np.float64)
        vmax = grid.vmax.ravel().astype(np.float64)
        empty = grid.empty.ravel().astype(np.uint8)
        margin = SKIP_MARGIN[settings.interpolation]
        box_lo = grid.aabb_lo.reshape(-1, 3).astype(np.float64) - margin
        box_hi = grid.aabb_hi.reshape(-1, 3).astype(np.float64) + margin
        skip_empty = 1
        blocks_total = grid.count
    else:
        atlas = vals.ravel()
        offsets = np.zeros(1, dtype=np.int64)
        org_x = org_y = org_z = np.zeros(1, dtype=np.int64)
        ext_x = np.array([nx], dtype=np.int64)
        ext_y = np.array([ny], dtype=np.int64)
        ext_z = np.array([nz], dtype=np.int64)
        stride = max(nx, ny, nz)
        vmin = np.array([float(vr_lo)])
        vmax = np.array([float(vr_hi)])
        empty = np.zeros(1, dtype=np.uint8)
        box_lo = np.full((1, 3), -1e30)
        box_hi = np.full((1, 3), 1e30)
        skip_empty = 0
        blocks_total = 1

    if classify == CLS_PRE:
        rgba_volume = preclassify(vals, lut, tf_domain)
        if use_blocks:
            rgba_atlas = build_rgba_atlas(grid, rgba_volume)
        else:
            rgba_atlas = np.concatenate(
                [np.ascontiguousarray(rgba_volume[..., ch]).ravel() for ch in range(4)])
    else:
        rgba_atlas = np.zeros(4, dtype=np.uint8)
    if classify == CLS_PREINT:
        table = preintegrated(lut, tf_domain, step, ref_step)
    else:
        table = np.zeros((1, 1, 4))

    lut_lo, lut_hi = tf_domain
    lut_inv_w = lut.shape[0] / (lut_hi - lut_lo)
    tbl_inv_w = table.shape[0] / (lut_hi - lut_lo)

    origins, dirs = rays(camera, projection, ortho_half_h, tile)
    tmins, tmaxs = clip_to_bounds(origins, dirs, extent)
    npix = origins.shape[0]
    out = np.empty((npix, 4))
    depth = np.full(npix, np.nan)
    taken = np.zeros(npix, dtype=np.int64)
    skipped = np.zeros(npix, dtype=np.int64)
    blocks_hit = np.zeros(offsets.shape[0], dtype=np.uint8)
    bg = settings.background
    c = np.ascontiguousarray
    a = [c(atlas), c(rgba_atlas), c(offsets), c(org_x), c(org_y), c(org_z), c(ext_x), c(ext_y),
         c(ext_z), c(vmin), c(vmax), c(empty), c(box_lo), c(box_hi), c(lut), c(table)]
    lib().vro_march(
        npix, _p(origins), _p(dirs), _p(tmins), _p(tmaxs), sx, sy, sz, float(step),
        float(ref_step), mode, int(cubic), int(bool(settings.lighting)), classify, skip_empty,
        _p(a[0]), _p(a[1]), _p(a[2]), _p(a[3]), _p(a[4]), _p(a[5]), _p(a[6]), _p(a[7]), _p(a[8]),
        len(org_x), len(org_y), len(org_z), int(stride),
        _p(a[9]), _p(a[10]), _p(a[11]), _p(a[12]), _p(a[13]), _p(a[14]), lut.shape[0],
        float(lut_lo), float(lut_inv_w), _p(a[15]), table.shape[0], float(lut_lo), float(tbl_inv_w),
        float(settings.isovalue if settings.isovalue is not None else 0.0),
        float(settings.early_termination_alpha),
        float(getattr(settings, "ambient", 0.1)), float(getattr(settings, "diffuse", 0.7)),
        float(getattr(settings, "specular", 0.2)), float(getattr(settings, "shininess", 32.0)),
        float(bg[0]), float(bg[1]), float(bg[2]), float(bg[3]),
        _p(out), _p(depth), _p(taken), _p(skipped), _p(blocks_hit), int(nthreads),
    )
    if tile is not None:
        h, w = tile[3], tile[2]
    else:
        h, w = camera.height, camera.width
    return OracleResult(out, depth, taken, skipped, blocks_hit, to_pixels(out, h, w),
                        blocks_total, blocks_empty)


# --------------------------------------------------------- sampling / K4


def sample_points(values_zyx, pts, cubic):  # _kernels.py:169-174
    vals = np.ascontiguousarray(values_zyx, dtype=np.int16)
    nz, ny, nx = vals.shape
    pts = np.ascontiguousarray(pts, dtype=np.float64).reshape(-1, 3)
    out = np.empty(pts.shape[0])
    lib().vro_sample_points(_p(vals), nx, ny, nz, _p(pts), pts.shape[0], int(cubic), _p(out))
    return out


def gradient_points(values_zyx, pts, cubic, spacing):  # _kernels.py:177-187
    vals = np.ascontiguousarray(values_zyx, dtype=np.int16)
    nz, ny, nx = vals.shape
    pts = np.ascontiguousarray(pts, dtype=np.float64).reshape(-1, 3)
    out = np.empty((pts.shape[0], 3))
    sx, sy, sz = spacing
    lib().vro_gradient_points(_p(vals), nx, ny, nz, _p(pts), pts.shape[0], int(cubic),
                              float(sx), float(sy), float(sz), _p(out))
    return out


def threshold_count(values_zyx, thr: int) -> int:
    """K4 restatement (parity unpinned): count of voxels >= thr."""
    vals = np.ascontiguousarray(values_zyx, dtype=np.int16)
    return int(lib().vro_threshold_count(_p(vals), vals.size, int(thr)))


AREA_SCALE = float(1 << 24)  # vr_oracle.c VRO_AREA_SCALE


def ball_counts(values_zyx, spacing, thr: int, centres, radii):
    """K4 ball form (parity unpinned): voxels >= thr with centre in each closed ball."""
    vals = np.ascontiguousarray(values_zyx, dtype=np.int16)
    nz, ny, nx = vals.shape
    centres = np.ascontiguousarray(centres, dtype=np.float64).reshape(-1, 3)
    radii = np.ascontiguousarray(radii, dtype=np.float64).reshape(-1)
    counts = np.empty(centres.shape[0], dtype=np.uint64)
    sx, sy, sz = spacing
    lib().vro_ball_counts(_p(vals), nx, ny, nz, float(sx), float(sy), float(sz), int(thr),
                          _p(centres), _p(radii), centres.shape[0], _p(counts))
    return counts


def threshold_measure(values_zyx, spacing, thr: int):
    """K4 whole volume: (voxels >= thr, isosurface area * 2^24) as ints
    (marching tetrahedra at thr - 0.5, vr_oracle.c)."""
    vals = np.ascontiguousarray(values_zyx, dtype=np.int16)
    nz, ny, nx = vals.shape
    out = np.zeros(2, dtype=np.uint64)
    sx, sy, sz = spacing
    lib().vro_threshold_measure(_p(vals), nx, ny, nz, float(sx), float(sy), float(sz), int(thr), _p(out))
    return int(out[0]), int(out[1])


def ball_measure(values_zyx, spacing, thr: int, centres, radii):
    """K4 per ball: (counts, area * 2^24) uint64 arrays -- V = count * voxel
    volume, S = area / 2^24 mm^2 of the isosurface with centroid in the ball."""
    vals = np.ascontiguousarray(values_zyx, dtype=np.int16)
    nz, ny, nx = vals.shape
    centres = np.ascontiguousarray(centres, dtype=np.float64).reshape(-1, 3)
    radii = np.ascontiguousarray(radii, dtype=np.float64).reshape(-1)
    counts = np.empty(centres.shape[0], dtype=np.uint64)
    area = np.empty(centres.shape[0], dtype=np.uint64)
    sx, sy, sz = spacing
    lib().vro_ball_measure(_p(vals), nx, ny, nz, float(sx), float(sy), float(sz), int(thr),
                           _p(centres), _p(radii), centres.shape[0], _p(counts), _p(area))
    return counts, area
