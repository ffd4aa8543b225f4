"""Scalar volume container, host side and device side.

``ScalarVolume`` / ``make_volume`` / ``load_raw`` keep the reference's contract
(voxelray/volume.py:23-109): int16 ``values[z, y, x]`` (x fastest), spacing in
mm, value range, immutable.  ``DeviceVolume`` is the B200 side: the same voxels
resident in HBM behind a ``vr_volume`` handle (K1 upload, include/voxelray_b200.h).
A ScalarVolume uploads itself once and keeps the handle, so repeated renders
of one volume pay the host-to-device copy once (the reference keys its
volume cache on content, store.py:62-67; identity is enough in-process).
"""

from __future__ import annotations

import ctypes
import threading
import weakref
from dataclasses import dataclass

import numpy as np

from . import _lib
from .errors import SizeMismatch

SAMPLE_FORMAT = "i16"
ENDIANNESS = "little"


class DeviceVolume:
    """An int16 volume resident on one GPU (``vr_volume`` handle)."""

    def __init__(self, handle: ctypes.c_void_p):
        self._h = handle
        L = _lib.load()
        dims = (ctypes.c_int64 * 3)()
        sp = (ctypes.c_double * 3)()
        vr = (ctypes.c_int32 * 2)()
        dev = ctypes.c_int()
        _lib.check(L.vr_volume_info(handle, dims, sp, vr, ctypes.byref(dev)))
        self.dims = tuple(int(d) for d in dims)
        self.spacing = tuple(float(s) for s in sp)
        self.value_range = (int(vr[0]), int(vr[1]))
        self.device = int(dev.value)
        self.clamp_count = 0  # samples clamped at ingest (ingest.py)
        self._finalizer = weakref.finalize(self, L.vr_volume_destroy, handle)

    @property
    def handle(self) -> ctypes.c_void_p:
        return self._h

    @property
    def data_ptr(self) -> int:
        return int(_lib.load().vr_volume_data(self._h) or 0)

    @classmethod
    def upload(cls, values: np.ndarray, spacing, device: int = 0, stream=None) -> "DeviceVolume":
        """Copy host int16 (nz, ny, nx) values to the device (K1)."""
        vals = np.ascontiguousarray(values, dtype=np.int16)
        nz, ny, nx = vals.shape
        h = ctypes.c_void_p()
        _lib.check(_lib.load().vr_volume_create(
            device, nx, ny, nz, float(spacing[0]), float(spacing[1]), float(spacing[2]),
            _lib.ptr(vals), 0, _stream_ptr(stream), ctypes.byref(h)))
        return cls(h)

    @classmethod
    def from_device(cls, tensor, spacing, stream=None) -> "DeviceVolume":
        """Adopt (copy) a CUDA int16 torch tensor of shape (nz, ny, nx)."""
        nz, ny, nx = tensor.shape
        t = tensor.contiguous()
        h = ctypes.c_void_p()
        _lib.check(_lib.load().vr_volume_create(
            t.device.index, nx, ny, nz, float(spacing[0]), float(spacing[1]), float(spacing[2]),
            ctypes.c_void_p(t.data_ptr()), 1, _stream_ptr(stream), ctypes.byref(h)))
        return cls(h)

    @classmethod
    def phantom(cls, name: str, dims, spacing=(1.0, 1.0, 1.0), device: int = 0,
                stream=None) -> "DeviceVolume":
        """generate_phantom (phantoms.py:98-111) computed on the device."""
        if name not in _lib.PHANTOM_KINDS:
            raise ValueError(f"unknown phantom {name!r}, expected one of {tuple(_lib.PHANTOM_KINDS)}")
        nx, ny, nz = (int(d) for d in dims)
        if min(nx, ny, nz) < 8:
            raise ValueError(f"phantom dims must be >= 8 per axis, got {tuple(dims)}")
        h = ctypes.c_void_p()
        _lib.check(_lib.load().vr_phantom_create(
            device, _lib.PHANTOM_KINDS[name], nx, ny, nz, float(spacing[0]), float(spacing[1]),
            float(spacing[2]), _stream_ptr(stream), ctypes.byref(h)))
        return cls(h)

    def culling_tables(self):
        """K1's transparency-culling tables as (nz, ny, nx, 2) per-cube and
        (ncz, ncy, ncx, 2) per-cell int16 (lo, hi) arrays (vr_volume_culling_tables)."""
        nx, ny, nz = self.dims
        bx, by, bz = (nx + 3) // 4, (ny + 3) // 4, (nz + 3) // 4
        cubes = np.empty((bz, by, bx, 4, 4, 4, 2), dtype=np.int16)
        cells = np.empty((bz, by, bx, 2), dtype=np.int16)
        _lib.check(_lib.load().vr_volume_culling_tables(self._h, _lib.ptr(cubes), _lib.ptr(cells)))
        lin = cubes.transpose(0, 3, 1, 4, 2, 5, 6).reshape(bz * 4, by * 4, bx * 4, 2)
        return np.ascontiguousarray(lin[:nz, :ny, :nx]), cells

    def download(self) -> np.ndarray:
        nx, ny, nz = self.dims
        out = np.empty((nz, ny, nx), dtype=np.int16)
        _lib.check(_lib.load().vr_volume_download(self._h, _lib.ptr(out), None))
        return out


def _stream_ptr(stream):
    if stream is None:
        return None
    if hasattr(stream, "cuda_stream"):
        return ctypes.c_void_p(stream.cuda_stream)
    return ctypes.c_void_p(int(stream))


_upload_lock = threading.Lock()


@dataclass(frozen=True)
class ScalarVolume:
    """Dense scalar field on a regular grid (volume.py:23-71).

    values: int16 (nz, ny, nx) C order; spacing (sx, sy, sz) mm;
    value_range (min, max); clamp_count samples clamped at calibration.
    """

    values: np.ndarray
    spacing: tuple[float, float, float]
    value_range: tuple[int, int]
    clamp_count: int = 0

    def __post_init__(self):
        v = self.values
        if v.ndim != 3:
            raise ValueError(f"values must be 3-d, got ndim={v.ndim}")
        if v.dtype != np.int16:
            raise ValueError(f"values must be int16, got {v.dtype}")
        if any(n < 2 for n in v.shape):
            raise ValueError(f"every dimension must be >= 2, got shape {v.shape}")
        if any(s <= 0 for s in self.spacing):
            raise ValueError(f"spacing must be positive, got {self.spacing}")
        v.flags.writeable = False

    @property
    def dims(self) -> tuple[int, int, int]:
        nz, ny, nx = self.values.shape
        return nx, ny, nz

    @property
    def extent_mm(self) -> tuple[float, float, float]:
        nx, ny, nz = self.dims
        sx, sy, sz = self.spacing
        return (nx - 1) * sx, (ny - 1) * sy, (nz - 1) * sz

    def voxel_bytes(self) -> bytes:
        return self.values.astype("<i2", copy=False).tobytes()

    def device(self, device: int = 0) -> DeviceVolume:
        """The device-resident copy (uploaded on first use, then cached)."""
        cache = self.__dict__.get("_device_cache")
        if cache is None:
            cache = {}
            object.__setattr__(self, "_device_cache", cache)
        dv = cache.get(device)
        if dv is None:
            with _upload_lock:
                dv = cache.get(device)
                if dv is None:
                    dv = DeviceVolume.upload(self.values, self.spacing, device)
                    cache[device] = dv
        return dv

    def _attach_device(self, dv: DeviceVolume) -> None:
        cache = self.__dict__.get("_device_cache")
        if cache is None:
            cache = {}
            object.__setattr__(self, "_device_cache", cache)
        cache[dv.device] = dv


def make_volume(values: np.ndarray, spacing, clamp_count: int = 0) -> ScalarVolume:
    """volume.py:74-79"""
    values = np.ascontiguousarray(values, dtype=np.int16)
    return ScalarVolume(values, tuple(float(s) for s in spacing),
                        (int(values.min()), int(values.max())), clamp_count)


_SAMPLE_DTYPES = {"u8": "u1", "i16": "<i2", "u16": "<u2"}


def load_raw(data: bytes, dims, spacing, sample_format: str = SAMPLE_FORMAT) -> ScalarVolume:
    """volume.py:85-109: headerless little-endian samples, x fastest."""
    if sample_format not in _SAMPLE_DTYPES:
        raise ValueError(f"unknown sample_format {sample_format!r}")
    dtype = np.dtype(_SAMPLE_DTYPES[sample_format])
    nx, ny, nz = (int(d) for d in dims)
    expected = nx * ny * nz * dtype.itemsize
    if len(data) != expected:
        raise SizeMismatch(
            f"raw payload is {len(data)} bytes, dims {nx}x{ny}x{nz} "
            f"{sample_format} require {expected}")
    arr = np.frombuffer(data, dtype=dtype).reshape(nz, ny, nx)
    clamped = 0
    if sample_format == "u16":
        clamped = int(np.count_nonzero(arr > 32767))
        arr = np.minimum(arr, 32767)
    return make_volume(arr.astype(np.int16), spacing, clamp_count=clamped)
