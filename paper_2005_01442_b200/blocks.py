"""Block decomposition for empty-space leaping, computed on the GPU.

Same contract as voxelray.blocks (reference blocks.py:29-266): cubic blocks of
edge ``block_size`` on a stride of ``block_size - overlap``, the last block per
axis clipped to the volume; each block carries its value range (K2a, computed
on the device by ``vr_grid_create``) and, for a LUT, an emptiness verdict and
a tight visible AABB dilated by one voxel (K2b, ``vr_grid_visibility``).

There is no atlas: the renderer samples blocks in place in the volume, with
the reference's block-local clamping (see csrc/vr_raycast.cu), which reads
exactly the voxels ``build_atlas`` (blocks.py:269-294) would have copied.
"""

from __future__ import annotations

import ctypes
import threading
import weakref
from dataclasses import dataclass, replace

import numpy as np

from . import _lib
from .errors import InvalidBlockSpec
from .transfer import ClassifiedLUT
from .volume import ScalarVolume

DEFAULT_BLOCK_SIZE = 64
DEFAULT_OVERLAP = 3


def _destroy_grid(L, h, _volume):
    L.vr_grid_destroy(h)


class DeviceGrid:
    """``vr_grid`` handle: layout + per-block int32 min/max in HBM."""

    def __init__(self, dvol, block_size: int, overlap: int):
        h = ctypes.c_void_p()
        L = _lib.load()
        _lib.check(L.vr_grid_create(dvol.handle, int(block_size), int(overlap), None, ctypes.byref(h)))
        self._h = h
        self.volume = dvol  # keep the volume alive as long as the grid
        shape = (ctypes.c_int64 * 3)()
        _lib.check(L.vr_grid_shape(h, shape))
        self.shape = tuple(int(s) for s in shape)
        # the finalizer holds the volume: its handle outlives the grid's even
        # when both are collected in one cycle
        self._finalizer = weakref.finalize(self, _destroy_grid, L, h, dvol)

    @property
    def handle(self):
        return self._h

    @property
    def count(self) -> int:
        a, b, c = self.shape
        return a * b * c

    def minmax(self):
        n = self.count
        vmin = np.empty(n, dtype=np.int64)
        vmax = np.empty(n, dtype=np.int64)
        _lib.check(_lib.load().vr_grid_minmax(self._h, _lib.ptr(vmin), _lib.ptr(vmax), None))
        nbx, nby, nbz = self.shape
        return vmin.reshape(nbz, nby, nbx), vmax.reshape(nbz, nby, nbx)

    def visibility(self, lut: ClassifiedLUT, strict: bool = True):
        """(empty, aabb_lo, aabb_hi) for the LUT.  strict=False tolerates blocks
        that pass the interval test without a visible voxel (the verdicts stay
        valid; only their AABB fit is undefined and keeps the sentinel)."""
        n = self.count
        rgba = np.ascontiguousarray(lut.rgba, dtype=np.float64)
        empty = np.empty(n, dtype=np.uint8)
        lo = np.empty((n, 3), dtype=np.int64)
        hi = np.empty((n, 3), dtype=np.int64)
        L = _lib.load()
        status = L.vr_grid_visibility(
            self._h, _lib.ptr(rgba), rgba.shape[0], float(lut.domain[0]), float(lut.domain[1]),
            _lib.ptr(empty), _lib.ptr(lo), _lib.ptr(hi), None)
        if status != _lib.VR_OK:
            msg = (L.vr_last_error() or b"").decode()
            if strict or not msg.startswith("EmptyBlock"):
                _lib.check(status)
        nbx, nby, nbz = self.shape
        return (empty.reshape(nbz, nby, nbx).astype(bool), lo.reshape(nbz, nby, nbx, 3),
                hi.reshape(nbz, nby, nbx, 3))


@dataclass(frozen=True)
class Block:
    """One block; coordinates are global voxel indices (blocks.py:29-39)."""

    index: tuple[int, int, int]
    origin: tuple[int, int, int]
    extent: tuple[int, int, int]
    value_min: int
    value_max: int
    empty: bool | None = None
    tight_aabb: tuple[tuple[int, int, int], tuple[int, int, int]] | None = None


@dataclass(frozen=True)
class BlockGrid:
    """A decomposition (blocks.py:42-97); updates return a new grid sharing
    the same device handle."""

    volume: ScalarVolume
    block_size: int
    overlap: int
    shape: tuple[int, int, int]
    origins: tuple[np.ndarray, np.ndarray, np.ndarray]
    extents: tuple[np.ndarray, np.ndarray, np.ndarray]
    vmin: np.ndarray
    vmax: np.ndarray
    empty: np.ndarray | None = None
    aabb_lo: np.ndarray | None = None
    aabb_hi: np.ndarray | None = None
    device_grid: DeviceGrid | None = None

    @property
    def stride(self) -> int:
        return self.block_size - self.overlap

    @property
    def count(self) -> int:
        a, b, c = self.shape
        return a * b * c

    @property
    def empty_count(self) -> int:
        return 0 if self.empty is None else int(np.count_nonzero(self.empty))

    def block(self, bi: int, bj: int, bk: int) -> Block:
        empty = None if self.empty is None else bool(self.empty[bk, bj, bi])
        aabb = None
        if self.aabb_lo is not None and empty is False:
            aabb = (tuple(int(v) for v in self.aabb_lo[bk, bj, bi]),
                    tuple(int(v) for v in self.aabb_hi[bk, bj, bi]))
        return Block(
            index=(bi, bj, bk),
            origin=tuple(int(o[i]) for o, i in zip(self.origins, (bi, bj, bk))),
            extent=tuple(int(e[i]) for e, i in zip(self.extents, (bi, bj, bk))),
            value_min=int(self.vmin[bk, bj, bi]), value_max=int(self.vmax[bk, bj, bi]),
            empty=empty, tight_aabb=aabb)

    def iter_indices(self):
        nbx, nby, nbz = self.shape
        for bk in range(nbz):
            for bj in range(nby):
                for bi in range(nbx):
                    yield bi, bj, bk


def axis_layout(n: int, block_size: int, stride: int):
    """Origins i*stride and extents min(B, n - origin) along one axis (blocks.py:100-107)."""
    count = 1 if n <= block_size else int(np.ceil((n - block_size) / stride)) + 1
    origins = stride * np.arange(count, dtype=np.int64)
    return origins, np.minimum(block_size, n - origins)


_grid_lock = threading.Lock()


def device_grid(volume: ScalarVolume, block_size: int, overlap: int, device: int = 0) -> DeviceGrid:
    """The device decomposition of a volume, built once per (block_size, overlap)."""
    cache = volume.__dict__.get("_grid_cache")
    if cache is None:
        cache = {}
        object.__setattr__(volume, "_grid_cache", cache)
    key = (device, int(block_size), int(overlap))
    g = cache.get(key)
    if g is None:
        with _grid_lock:
            g = cache.get(key)
            if g is None:
                g = DeviceGrid(volume.device(device), block_size, overlap)
                cache[key] = g
    return g


def _check_spec(block_size: int, overlap: int) -> None:
    if block_size < 8:
        raise InvalidBlockSpec(f"block_size must be >= 8, got {block_size}")
    if not 1 <= overlap < block_size:
        raise InvalidBlockSpec(f"overlap must satisfy 1 <= overlap < block_size, got {overlap}")


def decompose(volume: ScalarVolume, block_size: int = DEFAULT_BLOCK_SIZE,
              overlap: int = DEFAULT_OVERLAP, device: int = 0) -> BlockGrid:
    """Overlapping blocks with per-block value ranges (blocks.py:110-158), min/max on the GPU."""
    _check_spec(block_size, overlap)
    stride = block_size - overlap
    nx, ny, nz = volume.dims
    layouts = [axis_layout(n, block_size, stride) for n in (nx, ny, nz)]
    g = device_grid(volume, block_size, overlap, device)
    vmin, vmax = g.minmax()
    origins = tuple(o for o, _ in layouts)
    extents = tuple(e for _, e in layouts)
    for arr in (*origins, *extents, vmin, vmax):
        arr.flags.writeable = False
    return BlockGrid(volume, block_size, overlap, g.shape, origins, extents, vmin, vmax,
                     device_grid=g)


def _device(grid: BlockGrid) -> DeviceGrid:
    return grid.device_grid or device_grid(grid.volume, grid.block_size, grid.overlap)


def cull_empty(grid: BlockGrid, lut: ClassifiedLUT) -> BlockGrid:
    """Blocks whose whole value interval maps to zero opacity (blocks.py:161-173)."""
    empty, _, _ = _device(grid).visibility(lut, strict=False)
    empty.flags.writeable = False
    return replace(grid, empty=empty)


def with_visibility(grid: BlockGrid, lut: ClassifiedLUT) -> BlockGrid:
    """Emptiness + tight AABBs for every non-empty block (blocks.py:202-220);
    raises EmptyBlock where the reference's fit_bounding_box would."""
    empty, lo, hi = _device(grid).visibility(lut, strict=True)
    for arr in (empty, lo, hi):
        arr.flags.writeable = False
    return replace(grid, empty=empty, aabb_lo=lo, aabb_hi=hi)


def traversal_order(grid: BlockGrid, camera) -> list[tuple[int, int, int]]:
    """Non-empty blocks sorted by (distance camera->block centre, index) (blocks.py:223-248)."""
    pos = np.asarray(getattr(camera, "position", camera), dtype=np.float64)
    sp = grid.volume.spacing
    keyed = []
    for bi, bj, bk in grid.iter_indices():
        if grid.empty is not None and grid.empty[bk, bj, bi]:
            continue
        idx = (bi, bj, bk)
        centre = np.array([(grid.origins[a][idx[a]] + (grid.extents[a][idx[a]] - 1) / 2.0) * sp[a]
                           for a in range(3)])
        keyed.append((float(np.linalg.norm(centre - pos)), idx))
    keyed.sort()
    return [idx for _, idx in keyed]


def block_stats(grid: BlockGrid) -> dict:
    """JSON-friendly summary (blocks.py:251-266)."""
    has = grid.empty is not None
    return {
        "block_size": grid.block_size,
        "overlap": grid.overlap,
        "stride": grid.stride,
        "shape": list(grid.shape),
        "count": grid.count,
        "empty": grid.empty_count if has else None,
        "empty_fraction": grid.empty_count / grid.count if has else None,
        "value_min": int(grid.vmin.min()),
        "value_max": int(grid.vmax.max()),
    }
