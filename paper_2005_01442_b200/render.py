"""Render entry points: the reference's ``render()`` API over the sm_100a kernels.

``render(target, camera, tf, settings) -> ImageRGBA`` keeps the signature,
validation, errors and outputs of voxelray.render.render (reference
render.py:327-471); the march itself -- ray generation, box clipping,
empty-space leaping, sampling, classification, shading, compositing, the
uint8 epilogue and the stats -- runs in K3 (csrc/vr_raycast.cu) behind the
C-ABI call ``vr_render_to_host``.  ``Renderer`` is the device-resident form
(torch CUDA tensors in and out, no host copies) used for frame loops and the
multi-GPU tile path.
"""

from __future__ import annotations

import ctypes
import math
import time
import weakref
from dataclasses import dataclass

import numpy as np

from . import _lib
from .blocks import DEFAULT_BLOCK_SIZE, DEFAULT_OVERLAP, BlockGrid, device_grid
from .errors import EmptyBlock, InvalidSettings, IsovalueOutOfRange
from .sampling import INTERPOLATIONS
from .transfer import ClassifiedLUT, TransferFunction, build_lut, build_preintegrated
from .volume import DeviceVolume, ScalarVolume

CLASSIFICATIONS = ("post", "pre", "preintegrated")
MODES = ("dvr", "isosurface")
PROJECTIONS = ("pinhole", "orthographic")

# voxels of slack around a visibility box (render.py:50-53): the reach of the
# interpolant plus the gradient's half-voxel offsets
SKIP_MARGIN = {"trilinear": 2.0, "tricubic": 3.0}


def _basis(position, look_at, up):
    """Orthonormal (forward, right, true_up), computed as render.py:78-85 does
    (numpy's own norm and cross, so the rays match the reference bit for bit);
    memoised per view because numpy's small-vector overhead is ~0.1 ms."""
    try:
        key = (tuple(map(float, position)), tuple(map(float, look_at)), tuple(map(float, up)))
    except TypeError:
        key = None
    if key is not None:
        hit = _basis_cache.get(key)
        if hit is not None:
            return tuple(v.copy() for v in hit)
    fwd = np.subtract(look_at, position, dtype=np.float64)
    fwd /= np.linalg.norm(fwd)
    right = np.cross(fwd, np.asarray(up, dtype=np.float64))
    right /= np.linalg.norm(right)
    out = (fwd, right, np.cross(right, fwd))
    if key is not None:
        if len(_basis_cache) > 4096:
            _basis_cache.clear()
        _basis_cache[key] = tuple(v.copy() for v in out)
    return out


_basis_cache: dict = {}


@dataclass(frozen=True)
class Camera:
    """Pinhole camera (render.py:56-95); millimetres and degrees."""

    position: tuple[float, float, float]
    look_at: tuple[float, float, float]
    up: tuple[float, float, float] = (0.0, 0.0, 1.0)
    vertical_fov_deg: float = 30.0
    width: int = 256
    height: int = 256

    def __post_init__(self):
        if self.width < 1 or self.height < 1:
            raise ValueError(f"image size must be positive, got {self.width}x{self.height}")
        if not 0.0 < self.vertical_fov_deg < 180.0:
            raise ValueError(f"vertical_fov_deg must be in (0, 180), got {self.vertical_fov_deg}")
        _check_view(self.position, self.look_at, self.up)

    def basis(self):
        return _basis(self.position, self.look_at, self.up)

    def half_extents(self):
        """(half_w, half_h) on the image plane at unit distance (render.py:128-129)."""
        half_h = math.tan(math.radians(self.vertical_fov_deg) / 2.0)
        return half_h * self.width / self.height, half_h

    projection = "pinhole"

    def to_dict(self) -> dict:
        return {"position": list(self.position), "look_at": list(self.look_at),
                "up": list(self.up), "vertical_fov_deg": self.vertical_fov_deg,
                "width": self.width, "height": self.height}


@dataclass(frozen=True)
class OrthographicCamera:
    """Parallel projection (the reference has only the pinhole):
    the ray of pixel (px, py) starts at (position + u*right) + v*true_up and
    travels along forward, u and v spanning +-half_width/height_mm."""

    position: tuple[float, float, float]
    look_at: tuple[float, float, float]
    up: tuple[float, float, float] = (0.0, 0.0, 1.0)
    half_height_mm: float = 32.0
    width: int = 256
    height: int = 256

    projection = "orthographic"

    def __post_init__(self):
        if self.width < 1 or self.height < 1:
            raise ValueError(f"image size must be positive, got {self.width}x{self.height}")
        if not self.half_height_mm > 0:
            raise ValueError(f"half_height_mm must be positive, got {self.half_height_mm}")
        _check_view(self.position, self.look_at, self.up)

    def basis(self):
        return _basis(self.position, self.look_at, self.up)

    def half_extents(self):
        half_h = float(self.half_height_mm)
        return half_h * self.width / self.height, half_h


def _check_view(position, look_at, up):
    fwd = np.subtract(look_at, position, dtype=np.float64)
    if np.linalg.norm(fwd) == 0:
        raise ValueError("camera position and look_at coincide")
    if np.linalg.norm(np.cross(fwd, np.asarray(up, dtype=np.float64))) == 0:
        raise ValueError("camera up vector is parallel to the view direction")


def camera_from_dict(data: dict) -> Camera:
    return Camera(position=tuple(data["position"]), look_at=tuple(data["look_at"]),
                  up=tuple(data.get("up", (0.0, 0.0, 1.0))),
                  vertical_fov_deg=float(data.get("vertical_fov_deg", 30.0)),
                  width=int(data.get("width", 256)), height=int(data.get("height", 256)))


def generate_ray(camera: Camera, pixel: tuple[int, int]):
    """Origin and unit direction of the ray through pixel (px, py) (render.py:109-122)."""
    px, py = pixel
    fwd, right, up = camera.basis()
    half_w, half_h = camera.half_extents()
    u = (2.0 * (px + 0.5) / camera.width - 1.0) * half_w
    v = (1.0 - 2.0 * (py + 0.5) / camera.height) * half_h
    d = fwd + u * right + v * up
    return np.asarray(camera.position, dtype=np.float64), d / np.linalg.norm(d)


@dataclass(frozen=True)
class RenderSettings:
    """Everything about a render except camera and TF (render.py:159-223)."""

    step: float | None = None
    interpolation: str = "trilinear"
    classification: str = "post"
    mode: str = "dvr"
    isovalue: float | None = None
    lighting: bool = True
    early_termination_alpha: float = 0.99
    use_blocks: bool = False
    block_size: int = DEFAULT_BLOCK_SIZE
    overlap: int = DEFAULT_OVERLAP
    background: tuple[float, float, float, float] = (0.0, 0.0, 0.0, 1.0)
    ambient: float = 0.1
    diffuse: float = 0.7
    specular: float = 0.2
    shininess: float = 32.0

    def validate(self) -> None:
        checks = (
            (self.step is not None and not self.step > 0, f"step must be positive, got {self.step}"),
            (self.interpolation not in INTERPOLATIONS,
             f"interpolation must be one of {INTERPOLATIONS}, got {self.interpolation!r}"),
            (self.classification not in CLASSIFICATIONS,
             f"classification must be one of {CLASSIFICATIONS}, got {self.classification!r}"),
            (self.mode not in MODES, f"mode must be one of {MODES}, got {self.mode!r}"),
            (self.mode == "isosurface" and self.isovalue is None,
             "isovalue is required when mode is 'isosurface'"),
            (not 0.0 < self.early_termination_alpha <= 1.0,
             f"early_termination_alpha must be in (0, 1], got {self.early_termination_alpha}"),
            (len(self.background) != 4 or any(not 0.0 <= c <= 1.0 for c in self.background),
             f"background must be four channels in [0, 1], got {self.background}"),
        )
        for bad, msg in checks:
            if bad:
                raise InvalidSettings(msg)

    def to_dict(self) -> dict:
        keys = ("step", "interpolation", "classification", "mode", "isovalue", "lighting",
                "early_termination_alpha", "use_blocks", "block_size", "overlap")
        d = {k: getattr(self, k) for k in keys}
        d["background"] = list(self.background)
        return d


def settings_from_dict(data: dict) -> RenderSettings:
    unknown = set(data) - set(RenderSettings.__dataclass_fields__)
    if unknown:
        raise InvalidSettings(f"unknown settings fields: {sorted(unknown)}")
    kw = dict(data)
    if kw.get("background") is not None:
        kw["background"] = tuple(kw["background"])
    return RenderSettings(**kw)


@dataclass(frozen=True)
class RenderStats:
    rays: int
    samples_taken: int
    samples_skipped: int
    blocks_total: int
    blocks_empty: int
    blocks_visited: int
    wall_time_s: float

    def to_dict(self) -> dict:
        return {k: getattr(self, k) for k in self.__dataclass_fields__}


@dataclass(frozen=True)
class ImageRGBA:
    """Straight (non-premultiplied) 8-bit RGBA (render.py:259-274)."""

    pixels: np.ndarray
    stats: RenderStats | None = None
    depth: np.ndarray | None = None

    @property
    def width(self) -> int:
        return self.pixels.shape[1]

    @property
    def height(self) -> int:
        return self.pixels.shape[0]


def composite_step(dst, src, step: float, ref_step: float):
    """One front-to-back step with the opacity correction (render.py:277-287)."""
    r, g, b, a = dst
    sr, sg, sb, sa = src
    w = (1.0 - a) * (1.0 - (1.0 - sa) ** (step / ref_step))
    return (r + w * sr, g + w * sg, b + w * sb, a + w)


def shade_headlight(rgb, grad, view_dir, ka=0.1, kd=0.7, ks=0.2, shininess=32.0):
    """Headlight Phong with r.v = 2(n.l)^2 - 1 (render.py:290-309)."""
    g = np.asarray(grad, dtype=np.float64)
    norm = np.linalg.norm(g)
    if norm < 1e-12:
        return tuple(float(c) for c in rgb)
    light = -np.asarray(view_dir, dtype=np.float64)
    ndl = float((-g / norm) @ (light / np.linalg.norm(light)))
    lit = ka + kd * max(ndl, 0.0)
    spec = ks * max(2.0 * ndl * ndl - 1.0, 0.0) ** shininess
    return tuple(min(1.0, max(0.0, c * lit + spec)) for c in rgb)


# ------------------------------------------------------------------ plumbing


@dataclass
class _Resolved:
    params: _lib.RenderParams
    lut: ClassifiedLUT
    table: np.ndarray | None


_lut_cache: dict = {}


def _lut_for(tf: TransferFunction):
    """build_lut(tf), memoised per TransferFunction object: its control-point
    arrays are read-only (transfer.py) so the LUT cannot go stale."""
    hit = _lut_cache.get(id(tf))
    if hit is not None and hit[0]() is tf:
        return hit[1]
    lut = build_lut(tf)
    if len(_lut_cache) > 64:
        _lut_cache.clear()
    _lut_cache[id(tf)] = (weakref.ref(tf), lut)
    return lut


_preint_cache: dict = {}


def _preint_for(lut, step, ref_step):
    """build_preintegrated(lut, step, ref_step).rgba, memoised per LUT object
    and step pair (the LUT is immutable, _lut_for), in page-locked memory: a
    frame loop with one TF pays the 256^2 x 64-substep table once."""
    key = (id(lut), float(step), float(ref_step))
    hit = _preint_cache.get(key)
    if hit is not None and hit[0]() is lut:
        return hit[1]
    rgba = build_preintegrated(lut, step, ref_step).rgba
    buf = _pinned_empty(rgba.shape, np.float64)
    buf[...] = rgba
    if len(_preint_cache) > 16:
        _preint_cache.clear()
    _preint_cache[key] = (weakref.ref(lut), buf)
    return buf


_lut_pinned: dict = {}


def _lut_host_copy(lut):
    """The LUT's float64 table in pinned memory (uploaded every frame), kept per LUT object."""
    hit = _lut_pinned.get(id(lut))
    if hit is not None and hit[0]() is lut:
        return hit[1]
    buf = _pinned_empty(lut.rgba.shape, np.float64)
    buf[...] = lut.rgba
    if len(_lut_pinned) > 64:
        _lut_pinned.clear()
    _lut_pinned[id(lut)] = (weakref.ref(lut), buf)
    return buf


def _pinned_empty(shape, dtype):
    """Host output buffer in page-locked memory (torch's caching host
    allocator), so the device-to-host copy of a frame is a full-speed DMA
    (4 MiB: 0.09 ms pinned vs 0.41 ms pageable on the B200 box)."""
    import torch

    n = int(np.prod(shape)) * np.dtype(dtype).itemsize
    buf = torch.empty(n, dtype=torch.uint8, pin_memory=True)
    return buf.numpy().view(dtype).reshape(shape)


def _resolve(volume_spacing, value_range, tf: TransferFunction, settings: RenderSettings) -> _Resolved:
    """render.py:354-425: step, ref_step, LUT, mode/classification, tables."""
    lo_v, hi_v = value_range
    if settings.mode == "isosurface" and not lo_v <= settings.isovalue <= hi_v:
        raise IsovalueOutOfRange(
            f"isovalue {settings.isovalue} outside value range [{lo_v}, {hi_v}]")
    ref_step = 0.5 * min(volume_spacing)
    step = settings.step if settings.step is not None else ref_step
    lut = _lut_for(tf)
    iso = settings.mode == "isosurface"
    classify = {"post": _lib.CLS_POST, "pre": _lib.CLS_PRE,
                "preintegrated": _lib.CLS_PREINT}[settings.classification]
    if iso:
        classify = _lib.CLS_POST
    table = None
    if classify == _lib.CLS_PREINT:
        table = _preint_for(lut, step, ref_step)
    p = _lib.RenderParams()
    p.step = float(step)
    p.ref_step = float(ref_step)
    p.mode = _lib.MODE_ISO if iso else _lib.MODE_DVR
    p.cubic = int(settings.interpolation == "tricubic")
    p.lighting = int(bool(settings.lighting))
    p.classify = classify
    p.isovalue = float(settings.isovalue if settings.isovalue is not None else 0.0)
    p.term_alpha = float(settings.early_termination_alpha)
    p.ka, p.kd, p.ks = float(settings.ambient), float(settings.diffuse), float(settings.specular)
    p.shininess = float(settings.shininess)
    for k in range(4):
        p.bg[k] = float(settings.background[k])
    p.lut_lo, p.lut_hi = float(lut.domain[0]), float(lut.domain[1])
    p.nlut = lut.bins
    p.ntbl = table.shape[0] if table is not None else 1
    p.margin = SKIP_MARGIN[settings.interpolation]
    return _Resolved(p, lut, table)


# ---------------------------------------------------- reference-typed inputs
# render() is a drop-in for voxelray.render.render: its callers (service.py:68-88
# prepare_render, store.py:131-143, quality.py:98-101) hand it the REFERENCE's
# own objects -- voxelray.volume.ScalarVolume, voxelray.blocks.BlockGrid,
# voxelray.render.Camera / RenderSettings, voxelray.transfer.TransferFunction.
# These adapters accept anything carrying the reference's attributes.

_foreign_volumes: dict = {}


def as_volume(obj) -> ScalarVolume:
    """A ScalarVolume for any object with the reference's ``values`` (int16
    (nz, ny, nx)), ``spacing`` and optional ``value_range`` / ``clamp_count``
    (volume.py:23-71).  The wrapper -- and with it the device upload and block
    grids -- is cached per source object for as long as that object lives, as
    the reference's store caches volumes by id (store.py:62-67)."""
    if isinstance(obj, ScalarVolume):
        return obj
    if not (hasattr(obj, "values") and hasattr(obj, "spacing")):
        raise TypeError(f"render target must be a volume or a block grid, got {type(obj).__name__}")
    hit = _foreign_volumes.get(id(obj))
    if hit is not None and hit[0]() is obj:
        return hit[1]
    vals = np.ascontiguousarray(obj.values, dtype=np.int16)
    vr_ = getattr(obj, "value_range", None)
    value_range = (int(vr_[0]), int(vr_[1])) if vr_ is not None else (int(vals.min()), int(vals.max()))
    sv = ScalarVolume(vals, tuple(float(x) for x in obj.spacing), value_range,
                      int(getattr(obj, "clamp_count", 0) or 0))
    try:
        ref = weakref.ref(obj, lambda _r, k=id(obj): _foreign_volumes.pop(k, None))
    except TypeError:  # not weak-referenceable: no caching
        return sv
    _foreign_volumes[id(obj)] = (ref, sv)
    return sv


def as_camera(cam):
    """The camera itself when it is one of ours; otherwise a Camera (pinhole,
    render.py:56-95) or OrthographicCamera built from the reference's
    attributes (position, look_at, up, vertical_fov_deg, width, height)."""
    if isinstance(cam, (Camera, OrthographicCamera)):
        return cam
    up = tuple(getattr(cam, "up", (0.0, 0.0, 1.0)))
    if getattr(cam, "projection", "pinhole") == "orthographic":
        return OrthographicCamera(position=tuple(cam.position), look_at=tuple(cam.look_at), up=up,
                                  half_height_mm=float(cam.half_height_mm), width=int(cam.width),
                                  height=int(cam.height))
    return Camera(position=tuple(cam.position), look_at=tuple(cam.look_at), up=up,
                  vertical_fov_deg=float(getattr(cam, "vertical_fov_deg", 30.0)), width=int(cam.width),
                  height=int(cam.height))


def as_settings(settings) -> "RenderSettings":
    """RenderSettings from any object with the reference's fields (render.py:159-181)."""
    if isinstance(settings, RenderSettings):
        return settings
    kw = {}
    for f in RenderSettings.__dataclass_fields__:
        if hasattr(settings, f):
            kw[f] = getattr(settings, f)
    if kw.get("background") is not None:
        kw["background"] = tuple(kw["background"])
    return RenderSettings(**kw)


def as_transfer(tf) -> TransferFunction:
    """TransferFunction from any object with ``values``, ``rgba`` and ``domain``
    (transfer.py:28-62); ours pass through."""
    if isinstance(tf, TransferFunction):
        return tf
    hit = _foreign_tfs.get(id(tf))
    if hit is not None and hit[0]() is tf:
        return hit[1]
    ours = TransferFunction(np.array(tf.values, dtype=np.float64), np.array(tf.rgba, dtype=np.float64),
                            (float(tf.domain[0]), float(tf.domain[1])))
    try:
        _foreign_tfs[id(tf)] = (weakref.ref(tf, lambda _r, k=id(tf): _foreign_tfs.pop(k, None)), ours)
    except TypeError:
        pass
    return ours


_foreign_tfs: dict = {}


def camera_struct(camera, tile=None, interleave=None) -> _lib.Camera:
    """C camera for the frame or the sub-rectangle tile=(x0, y0, w, h);
    interleave=(n, k) renders the k-th of n sort-first cell sets."""
    fwd, right, up = camera.basis()
    half_w, half_h = camera.half_extents()
    c = _lib.Camera()
    c.projection = _lib.ORTHOGRAPHIC if getattr(camera, "projection", "pinhole") == "orthographic" else _lib.PINHOLE
    c.width, c.height = int(camera.width), int(camera.height)
    x0, y0, w, h = tile if tile is not None else (0, 0, camera.width, camera.height)
    c.tile_x, c.tile_y, c.tile_w, c.tile_h = int(x0), int(y0), int(w), int(h)
    for k in range(3):
        c.position[k] = float(camera.position[k])
        c.fwd[k] = float(fwd[k])
        c.right[k] = float(right[k])
        c.up[k] = float(up[k])
    c.half_w, c.half_h = float(half_w), float(half_h)
    if interleave is not None and interleave[0] > 1:
        c.interleave_n, c.interleave_k = int(interleave[0]), int(interleave[1])
    return c


def output_pixels(cam: _lib.Camera) -> int:
    """Pixels one render call writes (rectangle, or the packed interleaved cells)."""
    npix = ctypes.c_int64()
    _lib.check(_lib.load().vr_interleave_size(ctypes.byref(cam), None, ctypes.byref(npix)))
    return int(npix.value)


def render(target, camera, tf: TransferFunction, settings: RenderSettings = RenderSettings(), *,
           device: int = 0, tile=None, return_premultiplied: bool = False) -> ImageRGBA:
    """Render a ScalarVolume or a BlockGrid to straight RGBA (render.py:327-471).

    tile=(x0, y0, w, h) renders that sub-rectangle of the frame (equal to the
    crop of the full render).  return_premultiplied attaches the
    float64 premultiplied buffer as ``image.premultiplied`` (parity checks).
    """
    t_start = time.perf_counter()
    settings = as_settings(settings)
    settings.validate()
    camera = as_camera(camera)
    tf = as_transfer(tf)
    if isinstance(target, BlockGrid) or (not hasattr(target, "values") and hasattr(target, "block_size")):
        # ours, or the reference's BlockGrid (blocks.py:73-97): only its volume
        # and layout are used -- visibility is recomputed from the LUT per frame
        grid, volume, use_blocks = target, as_volume(target.volume), True
        block_size, overlap = int(target.block_size), int(target.overlap)
    else:
        volume, grid, use_blocks = as_volume(target), None, settings.use_blocks
        block_size, overlap = settings.block_size, settings.overlap
        if use_blocks:
            from .blocks import _check_spec
            _check_spec(block_size, overlap)
    res = _resolve(volume.spacing, volume.value_range, tf, settings)
    dvol = volume.device(device)
    dgrid = device_grid(volume, block_size, overlap, device) if use_blocks else None
    cam = camera_struct(camera, tile)
    npix = cam.tile_w * cam.tile_h
    pixels = _pinned_empty((cam.tile_h, cam.tile_w, 4), np.uint8)
    premult = np.empty((npix, 4)) if return_premultiplied else None
    iso = settings.mode == "isosurface"
    depth = _pinned_empty((npix,), np.float64) if iso else None
    totals = np.zeros(8, dtype=np.uint64)
    lut = _lut_host_copy(res.lut)
    _lib.check(_lib.load().vr_render_to_host(
        dvol.handle, dgrid.handle if dgrid else None, ctypes.byref(cam), ctypes.byref(res.params),
        _lib.ptr(lut), _lib.ptr(res.table), _lib.ptr(pixels), _lib.ptr(premult), _lib.ptr(depth),
        _lib.ptr(totals), None))
    if use_blocks and int(totals[4]):
        raise EmptyBlock(f"{int(totals[4])} block(s) pass the interval test without a visible voxel")
    stats = RenderStats(
        rays=npix, samples_taken=int(totals[0]), samples_skipped=int(totals[1]),
        blocks_total=dgrid.count if dgrid else 1, blocks_empty=int(totals[3]),
        blocks_visited=int(totals[2]), wall_time_s=time.perf_counter() - t_start)
    img = ImageRGBA(pixels=pixels, stats=stats,
                    depth=depth.reshape(cam.tile_h, cam.tile_w) if iso else None)
    if return_premultiplied:
        object.__setattr__(img, "premultiplied", premult)
    return img


_views_cache: dict = {}


def render_views(target, cameras, tf: TransferFunction, settings: RenderSettings = RenderSettings(), *,
                 device: int = 0) -> list:
    """Render a batch of views -- e.g. the viewer's 360-view turntable
    (frontend/src/camera.ts:35-44) -- in one submission: the TF visibility is
    computed once and one persistent ray-cast pass serves every view.  Returns
    one ImageRGBA per camera, each equal to render(target, camera, tf, settings)."""
    cameras = list(cameras)
    t_start = time.perf_counter()
    settings = as_settings(settings)
    if isinstance(target, BlockGrid) or (not hasattr(target, "values") and hasattr(target, "block_size")):
        settings = RenderSettings(**{**settings.__dict__, "use_blocks": True, "block_size": int(target.block_size),
                                     "overlap": int(target.overlap)})
        target = target.volume
    vol = as_volume(target)
    tfo = as_transfer(tf)
    cams = [as_camera(c) for c in cameras]
    key = (id(vol), id(tfo), settings, len(cams), cams[0].width, cams[0].height, device)
    hit = _views_cache.get(key)
    if hit is not None and hit[0]() is vol and hit[1]() is tfo:
        r = hit[2]  # device buffers, LUT and grid kept across calls
    else:
        r = Renderer(vol, cams[0], tfo, settings, device=device, views=len(cams))
        if len(_views_cache) > 4:
            _views_cache.clear()
        _views_cache[key] = (weakref.ref(vol), weakref.ref(tfo), r)
    r.set_views(cams)
    r.render_async()
    # frames land in page-locked host memory (torch's caching host allocator):
    # a full-speed DMA instead of a pageable copy (360 views: 1.5 GB per sweep)
    pixels = _pinned_empty(tuple(r.pixels.shape), np.uint8)
    import torch

    torch.from_numpy(pixels).copy_(r.pixels)
    depth = r.depth.cpu().numpy() if r.depth is not None else None
    per_view = r.view_stats()
    errors = r.totals.cpu().tolist()[4::5][:len(cameras)]
    if settings.use_blocks and any(errors):
        raise EmptyBlock(f"{max(errors)} block(s) pass the interval test without a visible voxel")
    wall = time.perf_counter() - t_start
    H, W = r.cam.tile_h, r.cam.tile_w
    out = []
    for v, st in enumerate(per_view):
        px = pixels[v] if len(cameras) > 1 else pixels
        dv = (depth[v] if len(cameras) > 1 else depth).reshape(H, W) if depth is not None else None
        out.append(ImageRGBA(pixels=px, stats=RenderStats(wall_time_s=wall / len(cameras), **st), depth=dv))
    return out


class Renderer:
    """Device-resident renderer: volume and grid in HBM, tables and outputs
    as torch CUDA tensors, asynchronous on a CUDA stream.  One frame is one
    ``vr_render`` call: TF visibility (K2b) + the ray-cast kernel (K3) + the
    stats finalisation."""

    def __init__(self, volume, camera, tf: TransferFunction, settings: RenderSettings = RenderSettings(),
                 *, device: int = 0, tile=None, interleave=None, keep_premultiplied: bool = False,
                 per_pixel_counts: bool = False, time_kernel: bool = False, frame_out=None, views: int = 1):
        import torch

        settings = as_settings(settings)
        settings.validate()
        tf = as_transfer(tf)
        if not isinstance(volume, DeviceVolume):
            volume = as_volume(volume)
        self.torch = torch
        self.device = torch.device("cuda", device)
        if isinstance(volume, DeviceVolume):
            self.dvol = volume
            spacing, vrange = volume.spacing, volume.value_range
        else:
            self.dvol = volume.device(device)
            spacing, vrange = volume.spacing, volume.value_range
        self.settings = settings
        self.res = _resolve(spacing, vrange, tf, settings)
        if settings.use_blocks:
            from .blocks import DeviceGrid, _check_spec
            _check_spec(settings.block_size, settings.overlap)
            if isinstance(volume, DeviceVolume):
                self.dgrid = DeviceGrid(volume, settings.block_size, settings.overlap)
            else:
                self.dgrid = device_grid(volume, settings.block_size, settings.overlap, device)
        else:
            self.dgrid = None
        self.lut = torch.from_numpy(np.ascontiguousarray(self.res.lut.rgba)).to(self.device)
        self.table = (torch.from_numpy(self.res.table).to(self.device)
                      if self.res.table is not None else None)
        self.rgba = None
        if self.res.params.classify == _lib.CLS_PRE:
            nx, ny, nz = self.dvol.dims
            self.rgba = torch.empty(4 * nx * ny * nz, dtype=torch.uint8, device=self.device)
            p = self.res.params
            _lib.check(_lib.load().vr_preclassify(
                self.dvol.handle, _lib.ptr(self.lut), p.nlut, p.lut_lo, p.lut_hi, _lib.ptr(self.rgba),
                _lib.ptr_stream(torch.cuda.current_stream(self.device))))
        self.interleave = interleave
        # frame_out: a (tile_h, tile_w, 4) uint8 CUDA tensor -- possibly another
        # GPU's memory mapped here (distributed.SharedFrame) -- that this
        # rank's interleaved cells are stored into at their frame positions
        self.frame_out = frame_out
        # views > 1: a batch of views of the same frame size rendered by one
        # vr_render_views call (set_views); outputs gain a leading view axis
        self.nviews = int(views)
        if self.nviews < 1 or (self.nviews > 1 and frame_out is not None):
            raise ValueError("views must be >= 1 (and batched views cannot store into frame_out)")
        self.view_table = None
        self.set_camera(camera, tile)
        nblocks = self.dgrid.count if self.dgrid else 1
        n = output_pixels(self.cam)
        self.npix = n
        V = self.nviews
        if frame_out is not None:
            if tuple(frame_out.shape) != (self.cam.tile_h, self.cam.tile_w, 4) or frame_out.dtype != torch.uint8:
                raise ValueError(f"frame_out must be a ({self.cam.tile_h}, {self.cam.tile_w}, 4) uint8 tensor")
            self.pixels = frame_out
        else:
            shape = (self.cam.tile_h, self.cam.tile_w, 4) if n == self.cam.tile_h * self.cam.tile_w and not (
                interleave and interleave[0] > 1) else (n, 4)
            self.pixels = torch.empty(((V,) if V > 1 else ()) + shape, dtype=torch.uint8, device=self.device)
        lead = (V, n) if V > 1 else (n,)
        self.premult = torch.empty(lead + (4,), dtype=torch.float64, device=self.device) if keep_premultiplied else None
        self.depth = torch.empty(lead, dtype=torch.float64, device=self.device) if settings.mode == "isosurface" else None
        self.taken = torch.empty(lead, dtype=torch.int64, device=self.device) if per_pixel_counts else None
        self.skipped = torch.empty(lead, dtype=torch.int64, device=self.device) if per_pixel_counts else None
        self.blocks_hit = torch.empty(V * nblocks, dtype=torch.uint8, device=self.device)
        # per view [taken, skipped, blocks_visited, blocks_empty, empty-block errors], then work[3]
        self.totals = torch.zeros(5 * V + 3, dtype=torch.int64, device=self.device)
        self._events = None
        if time_kernel:
            evs = []
            for _ in range(2):
                e = ctypes.c_void_p()
                _lib.check(_lib.load().vr_event_create(ctypes.byref(e)))
                evs.append(e)
            self._events = evs

    def __del__(self):
        evs = getattr(self, "_events", None)
        if evs:
            try:
                L = _lib.load()
                for e in evs:
                    L.vr_event_destroy(e)
            except Exception:  # interpreter shutdown: module globals already torn down
                pass

    def set_camera(self, camera, tile=None):
        """Point at a new view (same rectangle size); buffers are reused."""
        camera = as_camera(camera)
        self.camera = camera
        self.cam = camera_struct(camera, tile, self.interleave)
        if getattr(self, "frame_out", None) is not None:
            self.cam.interleave_frame = 1

    def kernel_ms(self) -> float:
        """Duration of the last ray-cast kernel launch (CUDA events on its stream)."""
        ms = ctypes.c_float()
        _lib.check(_lib.load().vr_event_elapsed_ms(self._events[0], self._events[1], ctypes.byref(ms)))
        return float(ms.value)

    def outputs(self) -> _lib.RenderOutputs:
        o = _lib.RenderOutputs()
        o.pixels = _lib.ptr(self.pixels).value
        o.premult = _lib.ptr(self.premult).value
        o.depth = _lib.ptr(self.depth).value
        o.taken = _lib.ptr(self.taken).value
        o.skipped = _lib.ptr(self.skipped).value
        o.blocks_hit = _lib.ptr(self.blocks_hit).value
        o.totals = self.totals.data_ptr()
        o.work = self.totals.data_ptr() + 5 * self.nviews * 8
        if self._events:
            o.ev_start, o.ev_stop = self._events[0].value, self._events[1].value
        return o

    def render_async(self, stream=None):
        """Enqueue one frame on ``stream`` (default: torch's current stream)."""
        torch = self.torch
        s = stream if stream is not None else torch.cuda.current_stream(self.device)
        out = self.outputs()  # (totals / work / blocks_hit are zeroed by vr_render itself)
        if self.nviews > 1:
            if self.view_table is None:
                raise ValueError("batched Renderer: call set_views(cameras) first")
            _lib.check(_lib.load().vr_render_views(
                self.dvol.handle, self.dgrid.handle if self.dgrid else None, ctypes.byref(self.cam),
                _lib.ptr(self.view_table), self.nviews, ctypes.byref(self.res.params), _lib.ptr(self.lut),
                _lib.ptr(self.table), _lib.ptr(self.rgba), ctypes.byref(out), _lib.ptr_stream(s)))
            return
        _lib.check(_lib.load().vr_render(
            self.dvol.handle, self.dgrid.handle if self.dgrid else None, ctypes.byref(self.cam),
            ctypes.byref(self.res.params), _lib.ptr(self.lut), _lib.ptr(self.table), _lib.ptr(self.rgba),
            ctypes.byref(out), _lib.ptr_stream(s)))

    def set_views(self, cameras, tile=None):
        """The batch's cameras (len == views, all of the frame's size and
        projection): a (views, 14) float64 device table of position, basis and
        half extents, as vr_render_views reads it."""
        cams = [as_camera(c) for c in cameras]
        if len(cams) != self.nviews:
            raise ValueError(f"expected {self.nviews} cameras, got {len(cams)}")
        rows = []
        for c in cams:
            cs = camera_struct(c, tile, self.interleave)
            if (cs.width, cs.height, cs.projection) != (self.cam.width, self.cam.height, self.cam.projection):
                raise ValueError("every view must have the frame's size and projection")
            rows.append([*cs.position, *cs.fwd, *cs.right, *cs.up, cs.half_w, cs.half_h])
        table = self.torch.tensor(rows, dtype=self.torch.float64)
        self.view_table = table.to(self.device)
        self.cameras = cams

    def view_stats(self) -> list:
        """Per-view RenderStats fields of the last batch (synchronising)."""
        t = self.totals.cpu().tolist()
        nb = self.dgrid.count if self.dgrid else 1
        rays = self.cam.tile_w * self.cam.tile_h if not self.interleave else self.npix
        return [{"rays": rays, "samples_taken": t[5 * v], "samples_skipped": t[5 * v + 1],
                 "blocks_total": nb, "blocks_empty": t[5 * v + 3], "blocks_visited": t[5 * v + 2]}
                for v in range(self.nviews)]

    def stats(self) -> dict:
        t = self.totals.cpu().tolist()
        V = self.nviews
        if V > 1:  # the batch: sums over views; the last view's block counts
            w = t[5 * V:]
            t = [sum(t[5 * v] for v in range(V)), sum(t[5 * v + 1] for v in range(V)), t[5 * V - 3],
                 t[5 * V - 2], t[5 * V - 1], *w]
        return {"samples_taken": t[0], "samples_skipped": t[1], "blocks_visited": t[2],
                "blocks_empty": t[3], "empty_block_errors": t[4], "shaded": t[5],
                "interpolated": t[6], "march_iterations": t[7],
                "blocks_total": self.dgrid.count if self.dgrid else 1,
                "rays": self.cam.tile_w * self.cam.tile_h if not self.interleave else self.npix}


def _preclassify_device(volume: ScalarVolume, lut: ClassifiedLUT) -> np.ndarray:
    import torch

    dvol = volume.device(0)
    dev = torch.device("cuda", dvol.device)
    nx, ny, nz = dvol.dims
    lut_t = torch.from_numpy(np.ascontiguousarray(lut.rgba)).to(dev)
    out = torch.empty(4 * nx * ny * nz, dtype=torch.uint8, device=dev)
    _lib.check(_lib.load().vr_preclassify(dvol.handle, _lib.ptr(lut_t), lut.bins, float(lut.domain[0]),
                                          float(lut.domain[1]), _lib.ptr(out),
                                          _lib.ptr_stream(torch.cuda.current_stream(dev))))
    return out.cpu().numpy().reshape(nz, ny, nx, 4)
