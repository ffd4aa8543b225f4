"""Voxel volume measure (K4) -- the paper's "method of spheres" on voxels.

The reference measures S (surface inside a probe ball) and V (object volume
inside it) on triangle meshes by Monte Carlo (morphology.py:70-143
clipped_area, :238-267 clipped_volume, :270-306 svr_at_point: SVR = S/V,
undefined where V == 0); it has no voxel form.  Here, on the CT
volume thresholded at ``thr`` (csrc/vr_measure.cu):

* V = number of voxels with value >= thr (centre in the closed ball for the
  ball form) times the voxel volume sx*sy*sz -- an exact integer count;
* S = area of the isosurface at thr - 0.5 of the piecewise-linear
  (Kuhn-tetrahedra) interpolant, which separates exactly the voxels V counts
  (polygons with centroid in the ball for the ball form), summed exactly in
  units of 2^-24 mm^2.

Both are bit-exact against the C restatement in oracle/ (parity unpinned:
there is no reference function); the definitions are pinned by the analytic
oracles of SPEC.md:472-473 in tests/test_measure.py.
"""

from __future__ import annotations

import numpy as np

from . import _lib

AREA_SCALE = float(1 << 24)  # include/voxelray_b200.h VR_AREA_SCALE


def _dev(volume, device):
    import torch

    if not hasattr(volume, "handle"):
        from .render import as_volume

        volume = as_volume(volume)
    dvol = volume.device(device) if hasattr(volume, "device") and callable(volume.device) else volume
    return torch, dvol, torch.device("cuda", dvol.device)


def _svr(V, S):
    with np.errstate(divide="ignore", invalid="ignore"):
        return np.where(V > 0, S / np.where(V > 0, V, 1.0), np.nan)


def threshold_count(volume, thr: int, device: int = 0) -> int:
    torch, dvol, dev = _dev(volume, device)
    count = torch.zeros(1, dtype=torch.int64, device=dev)
    _lib.check(_lib.load().vr_threshold_count(dvol.handle, int(thr), _lib.ptr(count),
                                              _lib.ptr_stream(torch.cuda.current_stream(dev))))
    return int(count.item())


def threshold_volume_mm3(volume, thr: int, device: int = 0) -> float:
    sx, sy, sz = volume.spacing
    return threshold_count(volume, thr, device) * (sx * sy * sz)


def threshold_measure(volume, thr: int, device: int = 0) -> dict:
    """Whole volume: count, area_fx (exact), V (mm^3), S (mm^2), SVR = S/V."""
    torch, dvol, dev = _dev(volume, device)
    out = torch.empty(2, dtype=torch.int64, device=dev)
    _lib.check(_lib.load().vr_threshold_measure(dvol.handle, int(thr), _lib.ptr(out),
                                                _lib.ptr_stream(torch.cuda.current_stream(dev))))
    count, area_fx = (int(x) for x in out.cpu().tolist())
    sx, sy, sz = volume.spacing
    V = count * (sx * sy * sz)
    S = area_fx / AREA_SCALE
    return {"count": count, "area_fx": area_fx, "V_mm3": V, "S_mm2": S, "svr": S / V if V > 0 else float("nan")}


def _balls(volume, thr, centres, radii, device, with_area):
    torch, dvol, dev = _dev(volume, device)
    c = np.ascontiguousarray(centres, dtype=np.float64).reshape(-1, 3)
    r = np.array(np.broadcast_to(np.asarray(radii, dtype=np.float64), (c.shape[0],)))
    n = c.shape[0]
    ct = torch.from_numpy(c).to(dev)
    rt = torch.from_numpy(r).to(dev)
    counts = torch.empty(n, dtype=torch.int64, device=dev)
    area = torch.empty(n, dtype=torch.int64, device=dev) if with_area else None
    _lib.check(_lib.load().vr_ball_measure(dvol.handle, int(thr), _lib.ptr(ct), _lib.ptr(rt), n,
                                           _lib.ptr(counts), _lib.ptr(area),
                                           _lib.ptr_stream(torch.cuda.current_stream(dev))))
    counts = counts.cpu().numpy().astype(np.uint64)
    return (counts, area.cpu().numpy().astype(np.uint64)) if with_area else counts


def ball_counts(volume, thr: int, centres, radii, device: int = 0) -> np.ndarray:
    """Voxels >= thr with centre in each closed ball B(X, R), uint64 (nballs,)."""
    return _balls(volume, thr, centres, radii, device, False)


def ball_measure(volume, thr: int, centres, radii, device: int = 0) -> dict:
    """Per ball: count, area_fx (exact), V (mm^3), S (mm^2) and SVR = S/V
    (NaN where V == 0: the reference's Undefined, morphology.py:296-306)."""
    counts, area = _balls(volume, thr, centres, radii, device, True)
    sx, sy, sz = volume.spacing
    V = counts.astype(np.float64) * (sx * sy * sz)
    S = area.astype(np.float64) / AREA_SCALE
    return {"count": counts, "area_fx": area, "V_mm3": V, "S_mm2": S, "svr": _svr(V, S)}
