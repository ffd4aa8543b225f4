"""Image metrics and step-size convergence studies on the device.

Mirrors voxelray/quality.py:1-109: ``psnr`` over 8-bit RGB (alpha ignored,
99 dB cap), ``ssim`` on the Rec. 601 luma plane with an 11x11 Gaussian window
(sigma 1.5) over the valid region, and ``convergence_study``, which renders
each step against a half-step reference.  The metrics run as CUDA kernels
(csrc/vr_quality.cu) on images wherever they live: host images (ImageRGBA /
numpy) are uploaded, device images (torch CUDA tensors, e.g. a Renderer's
``pixels``) are used in place, so a study never downloads its renders.
PSNR is bit-identical to the reference (exact integer squared error); SSIM
agrees to ~1e-15 (window sums in a different order than scipy's convolve2d).
"""

from __future__ import annotations

import ctypes

import numpy as np

from . import _lib
from .errors import DimensionMismatch
from .render import ImageRGBA, Renderer, RenderSettings

PSNR_CAP = 99.0


def _gaussian_window(size: int = 11, sigma: float = 1.5) -> np.ndarray:
    """quality.py:50-54 (the same float64 window)."""
    offsets = np.arange(size) - (size - 1) / 2.0
    w = np.exp(-(offsets**2) / (2.0 * sigma**2))
    kernel = np.outer(w, w)
    return kernel / kernel.sum()


_WINDOW = np.ascontiguousarray(_gaussian_window())


def _image_shape(image):
    if isinstance(image, ImageRGBA):
        image = image.pixels
    shape = tuple(image.shape) if hasattr(image, "shape") else np.asarray(image).shape
    if len(shape) != 3 or shape[2] not in (3, 4):
        raise DimensionMismatch(f"expected (h, w, 3|4) image, got shape {shape}")
    return shape


def _device_image(image, device):
    """(h, w, c) uint8 CUDA tensor for an ImageRGBA, numpy array or torch tensor."""
    import torch

    if isinstance(image, ImageRGBA):
        image = image.pixels
    if isinstance(image, torch.Tensor):
        t = image if image.is_cuda else image.to(torch.device("cuda", device))
    else:
        t = torch.from_numpy(np.ascontiguousarray(np.asarray(image), dtype=np.uint8)).to(
            torch.device("cuda", device))
    if t.dtype != torch.uint8:
        t = t.to(torch.uint8)
    return t.contiguous()


def _pair(a, b, device, min_hw=0):
    """Shapes checked as quality.py:23-34 does, before anything touches the device."""
    sa, sb = _image_shape(a), _image_shape(b)
    ra, rb = tuple(sa[:2]) + (3,), tuple(sb[:2]) + (3,)
    if ra != rb:
        raise DimensionMismatch(f"image shapes differ: {ra} vs {rb}")
    if sa[0] < min_hw or sa[1] < min_hw:
        raise DimensionMismatch(f"images must be at least {min_hw}x{min_hw} for SSIM, got {tuple(sa[:2])}")
    ta, tb = _device_image(a, device), _device_image(b, device)
    if tb.device != ta.device:
        tb = tb.to(ta.device)
    return ta, tb


def _stream(t):
    import torch

    return _lib.ptr_stream(torch.cuda.current_stream(t.device))


def psnr(a, b, *, device: int = 0) -> float:
    """Peak signal-to-noise ratio in dB over RGB; 99 dB when identical (quality.py:37-43)."""
    import torch

    ta, tb = _pair(a, b, device)
    h, w = ta.shape[:2]
    sse = torch.zeros(1, dtype=torch.int64, device=ta.device)
    _lib.check(_lib.load().vr_image_sse(_lib.ptr(ta), _lib.ptr(tb), h, w, ta.shape[2], tb.shape[2],
                                        _lib.ptr(sse), _stream(ta)))
    mse = float(int(sse.item())) / float(h * w * 3)
    if mse == 0.0:
        return PSNR_CAP
    return min(PSNR_CAP, 10.0 * np.log10(255.0**2 / mse))


def ssim(a, b, *, device: int = 0) -> float:
    """Mean structural similarity over the valid region of the luma plane (quality.py:57-79)."""
    import torch

    ta, tb = _pair(a, b, device, min_hw=_WINDOW.shape[0])
    h, w = ta.shape[:2]
    total = torch.zeros(1, dtype=torch.float64, device=ta.device)
    _lib.check(_lib.load().vr_image_ssim(_lib.ptr(ta), _lib.ptr(tb), h, w, ta.shape[2], tb.shape[2],
                                         _WINDOW.ctypes.data_as(ctypes.c_void_p), _lib.ptr(total),
                                         _stream(ta)))
    n = (h - _WINDOW.shape[0] + 1) * (w - _WINDOW.shape[1] + 1)
    return float(total.item()) / n


def convergence_study(target, camera, tf, settings: RenderSettings, steps, *, device: int = 0) -> list[dict]:
    """PSNR/SSIM of renders at each step against a half-step reference (quality.py:82-109).

    The reference uses half the smallest step in the list; all other settings
    are shared.  Returns one record per step, largest first.  Every render
    stays on the device; only the metric scalars come back.
    """
    steps = sorted(float(s) for s in steps)
    if not steps:
        raise ValueError("steps must not be empty")

    from .blocks import BlockGrid

    base = dict(settings.__dict__)
    volume = target
    if isinstance(target, BlockGrid):  # render(BlockGrid) renders with its blocks
        volume = target.volume
        base.update(use_blocks=True, block_size=target.block_size, overlap=target.overlap)

    def frame(step):
        r = Renderer(volume, camera, tf, RenderSettings(**{**base, "step": step}), device=device)
        r.render_async()
        return r.pixels

    reference = frame(steps[0] / 2.0)
    records = []
    for s in sorted(steps, reverse=True):
        image = frame(s)
        records.append({"step": s, "psnr_db": psnr(image, reference, device=device),
                        "ssim": ssim(image, reference, device=device)})
    return records


__all__ = ["PSNR_CAP", "psnr", "ssim", "convergence_study"]
