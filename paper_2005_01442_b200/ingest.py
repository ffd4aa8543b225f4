"""Volume ingest straight to the device.

The reference decodes volumes on the CPU and keeps them in a small LRU of
host arrays: ``load_raw`` widens u8/u16 samples to int16 (volume.py:85-109),
``assemble_volume`` calibrates DICOM slices (dicom.py:254-295), and
``VolumeStore`` keys decoded volumes by a content id (store.py:62-67,131-143).
Here the raw sample bytes are copied to HBM as they are (half the bytes for
u8) and converted there by ``vr_volume_ingest`` (K0), which then builds the
bricks and culling cells (K1) of the resident volume.  Validation, slice
ordering and the error classes stay on the host, message for message.
"""

from __future__ import annotations

import ctypes
import hashlib
import json
import threading
from collections import OrderedDict
from pathlib import Path

import numpy as np

from . import _lib
from .errors import (DuplicatePosition, InconsistentGeometry, NonUniformSpacing, SizeMismatch,
                     UnknownVolume)
from .volume import DeviceVolume, ScalarVolume, _stream_ptr

_SAMPLE_DTYPES = {"u8": "u1", "i16": "<i2", "u16": "<u2"}


def _ingest(samples: np.ndarray, fmt: str, dims, spacing, calib=None, device: int = 0,
            stream=None) -> DeviceVolume:
    nx, ny, nz = (int(d) for d in dims)
    buf = np.ascontiguousarray(samples)
    cal = None if calib is None else np.ascontiguousarray(calib, dtype=np.float64).reshape(nz, 2)
    h = ctypes.c_void_p()
    clamped = ctypes.c_uint64(0)
    _lib.check(_lib.load().vr_volume_ingest(
        device, _lib.SAMPLE_FORMATS[fmt], nx, ny, nz, float(spacing[0]), float(spacing[1]),
        float(spacing[2]), _lib.ptr(buf), 0, None if cal is None else _lib.ptr(cal),
        _stream_ptr(stream), ctypes.byref(h), ctypes.byref(clamped)))
    dv = DeviceVolume(h)
    dv.clamp_count = int(clamped.value)
    return dv


def ingest_raw(data: bytes, dims, spacing, sample_format: str = "i16", device: int = 0,
               stream=None) -> DeviceVolume:
    """``load_raw`` (volume.py:85-109) with the widening done on the device.

    Same arguments and errors; returns the resident volume, whose
    ``clamp_count`` is the number of u16 samples above 32767 (clamped).
    """
    if sample_format not in _SAMPLE_DTYPES:
        raise ValueError(f"unknown sample_format {sample_format!r}")
    dtype = np.dtype(_SAMPLE_DTYPES[sample_format])
    nx, ny, nz = (int(d) for d in dims)
    expected = nx * ny * nz * dtype.itemsize
    if len(data) != expected:
        raise SizeMismatch(
            f"raw payload is {len(data)} bytes, dims {nx}x{ny}x{nz} "
            f"{sample_format} require {expected}")
    arr = np.frombuffer(data, dtype=dtype)
    return _ingest(arr, sample_format, (nx, ny, nz), spacing, device=device, stream=stream)


def assemble_volume_device(slices, device: int = 0, stream=None) -> DeviceVolume:
    """``assemble_volume`` (dicom.py:254-295) with the calibration on the device.

    ``slices`` are parsed slices with the reference's ``SliceImage`` fields
    (rows, cols, pixel_spacing (row_mm, col_mm), position, rescale_slope,
    rescale_intercept, pixel_representation, samples).  Geometry checks,
    ordering and errors are the reference's; ``clamp_count`` of the result
    counts calibrated values outside int16.
    """
    if len(slices) < 2:
        raise InconsistentGeometry(f"need at least 2 slices, got {len(slices)}")
    first = slices[0]
    for s in slices[1:]:
        if (s.rows, s.cols) != (first.rows, first.cols):
            raise InconsistentGeometry(
                f"slice size {s.rows}x{s.cols} differs from {first.rows}x{first.cols}")
        if s.pixel_spacing != first.pixel_spacing:
            raise InconsistentGeometry(
                f"pixel spacing {s.pixel_spacing} differs from {first.pixel_spacing}")
    ordered = sorted(slices, key=lambda s: s.position)
    positions = np.array([s.position for s in ordered])
    gaps = np.diff(positions)
    if np.any(gaps == 0):
        at = positions[np.argmin(gaps)]
        raise DuplicatePosition(f"two slices share position {at}")
    median = float(np.median(gaps))
    if np.any(np.abs(gaps - median) > 0.10 * median):
        raise NonUniformSpacing(
            f"slice gaps {gaps.tolist()} deviate more than 10% from median {median}")
    kinds = {np.asarray(s.samples).dtype.kind for s in ordered}
    if kinds == {"i"} and all(np.asarray(s.samples).dtype.itemsize == 2 for s in ordered):
        fmt, dt = "i16", np.int16
    elif kinds == {"u"} and all(np.asarray(s.samples).dtype.itemsize == 2 for s in ordered):
        fmt, dt = "u16", np.uint16
    else:  # mixed signed / unsigned series: widen losslessly, calibrate on the device
        fmt, dt = "i32", np.int32
    stack = np.empty((len(ordered), first.rows, first.cols), dtype=dt)
    for i, s in enumerate(ordered):
        stack[i] = np.asarray(s.samples).astype(dt, copy=False)
    calib = np.array([[float(s.rescale_slope), float(s.rescale_intercept)] for s in ordered])
    row_mm, col_mm = first.pixel_spacing
    return _ingest(stack, fmt, (first.cols, first.rows, len(ordered)), (col_mm, row_mm, median),
                   calib=calib, device=device, stream=stream)


def volume_id(volume) -> str:
    """store.py:62-67: deterministic id from geometry and sample bytes."""
    h = hashlib.sha256()
    h.update(json.dumps([list(volume.dims), list(volume.spacing)]).encode())
    h.update(np.ascontiguousarray(volume.values, dtype="<i2").tobytes())
    return "v-" + h.hexdigest()[:16]


class DeviceVolumeCache:
    """Device-resident volumes of a reference ``VolumeStore`` directory.

    ``get(vid)`` reads ``<root>/<vid>/manifest.json`` + ``data.raw`` (the
    store's on-disk format, store.py:1-8) and ingests the bytes on the device
    on a miss; resident volumes are kept in LRU order within ``capacity_bytes``
    of HBM (the reference keeps ``DEFAULT_CACHE_SIZE = 4`` host arrays).
    ``put(volume)`` makes an in-memory ScalarVolume resident under its
    content id.  Thread-safe.
    """

    def __init__(self, root=None, capacity_bytes: int = 64 << 30, device: int = 0):
        self.root = Path(root) if root is not None else None
        self.capacity_bytes = int(capacity_bytes)
        self.device = device
        self._lock = threading.RLock()
        self._cache: OrderedDict[str, DeviceVolume] = OrderedDict()
        self.hits = 0
        self.misses = 0

    @staticmethod
    def _bytes(dv: DeviceVolume) -> int:
        nx, ny, nz = dv.dims
        return 2 * nx * ny * nz * 2  # linear + bricked copies (cells are < 4%)

    def _remember(self, vid: str, dv: DeviceVolume) -> DeviceVolume:
        self._cache[vid] = dv
        self._cache.move_to_end(vid)
        while len(self._cache) > 1 and sum(map(self._bytes, self._cache.values())) > self.capacity_bytes:
            self._cache.popitem(last=False)
        return dv

    def __contains__(self, vid: str) -> bool:
        with self._lock:
            return vid in self._cache

    def __len__(self) -> int:
        with self._lock:
            return len(self._cache)

    def put(self, volume: ScalarVolume) -> str:
        vid = volume_id(volume)
        with self._lock:
            if vid not in self._cache:
                dv = DeviceVolume.upload(volume.values, volume.spacing, device=self.device)
                dv.clamp_count = volume.clamp_count
                self._remember(vid, dv)
            return vid

    def get(self, vid: str) -> DeviceVolume:
        with self._lock:
            dv = self._cache.get(vid)
            if dv is not None:
                self._cache.move_to_end(vid)
                self.hits += 1
                return dv
            self.misses += 1
            if self.root is None or not (self.root / vid / "manifest.json").exists():
                raise UnknownVolume(f"no volume stored under id {vid!r}")
            m = json.loads((self.root / vid / "manifest.json").read_text())
            data = (self.root / vid / "data.raw").read_bytes()
            dv = ingest_raw(data, m["dims"], m["spacing"], "i16", device=self.device)
            return self._remember(vid, dv)
