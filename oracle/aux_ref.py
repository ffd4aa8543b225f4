"""CPU restatement of the §8(f) rows beside the render path (TEST INFRASTRUCTURE ONLY).

Only tests/ may import this module: it is the checker for the device ingest
(K0, csrc/vr_prep.cu) and image metrics (csrc/vr_quality.cu), never a
product path.  Each function follows the reference line by line and is pinned
by tests/golden/aux.npz, which tests/golden/make_golden_aux.py generated from
the unmodified reference.
"""

from __future__ import annotations

import hashlib
import json

import numpy as np
from scipy.signal import convolve2d

_SAMPLE_DTYPES = {"u8": "u1", "i16": "<i2", "u16": "<u2"}


def load_raw(data: bytes, dims, sample_format: str = "i16"):
    """voxelray/volume.py:85-109 -> (values int16 (nz,ny,nx), clamp_count, (vmin, vmax))."""
    dtype = np.dtype(_SAMPLE_DTYPES[sample_format])
    nx, ny, nz = (int(d) for d in dims)
    arr = np.frombuffer(data, dtype=dtype).reshape(nz, ny, nx)
    clamped = 0
    if sample_format == "u16":
        clamped = int(np.count_nonzero(arr > 32767))
        arr = np.minimum(arr, 32767)
    values = np.ascontiguousarray(arr.astype(np.int16))
    return values, clamped, (int(values.min()), int(values.max()))


def assemble(samples, positions, slopes, intercepts):
    """voxelray/dicom.py:276-295 (after the geometry checks): sort by position,
    calibrate slope * s + intercept in float64, count and clip to int16, rint.
    Returns (values, clamp_count, (vmin, vmax), z spacing)."""
    order = sorted(range(len(samples)), key=lambda i: positions[i])
    pos = np.array([positions[i] for i in order])
    median = float(np.median(np.diff(pos)))
    stack = np.empty((len(order),) + np.asarray(samples[0]).shape, dtype=np.int16)
    clamp = 0
    for k, i in enumerate(order):
        cal = slopes[i] * np.asarray(samples[i]).astype(np.float64) + intercepts[i]
        clamp += int(np.count_nonzero((cal < -32768) | (cal > 32767)))
        stack[k] = np.rint(np.clip(cal, -32768, 32767)).astype(np.int16)
    return stack, clamp, (int(stack.min()), int(stack.max())), median


def volume_id(values, dims, spacing) -> str:
    """voxelray/store.py:62-67."""
    h = hashlib.sha256()
    h.update(json.dumps([list(dims), list(spacing)]).encode())
    h.update(np.ascontiguousarray(values, dtype="<i2").tobytes())
    return "v-" + h.hexdigest()[:16]


def psnr(a, b) -> float:
    """voxelray/quality.py:37-43."""
    ra, rb = np.asarray(a)[..., :3].astype(np.float64), np.asarray(b)[..., :3].astype(np.float64)
    mse = float(np.mean((ra - rb) ** 2))
    if mse == 0.0:
        return 99.0
    return min(99.0, 10.0 * np.log10(255.0**2 / mse))


def ssim(a, b) -> float:
    """voxelray/quality.py:46-79."""
    ra, rb = np.asarray(a)[..., :3].astype(np.float64), np.asarray(b)[..., :3].astype(np.float64)

    def luma(rgb):
        return 0.299 * rgb[..., 0] + 0.587 * rgb[..., 1] + 0.114 * rgb[..., 2]

    offsets = np.arange(11) - 5.0
    w = np.exp(-(offsets**2) / (2.0 * 1.5**2))
    win = np.outer(w, w)
    win = win / win.sum()
    x, y = luma(ra), luma(rb)
    c1, c2 = (0.01 * 255.0) ** 2, (0.03 * 255.0) ** 2
    mu_x = convolve2d(x, win, mode="valid")
    mu_y = convolve2d(y, win, mode="valid")
    xx = convolve2d(x * x, win, mode="valid")
    yy = convolve2d(y * y, win, mode="valid")
    xy = convolve2d(x * y, win, mode="valid")
    var_x = xx - mu_x**2
    var_y = yy - mu_y**2
    cov = xy - mu_x * mu_y
    num = (2.0 * mu_x * mu_y + c1) * (2.0 * cov + c2)
    den = (mu_x**2 + mu_y**2 + c1) * (var_x + var_y + c2)
    return float(np.mean(num / den))
