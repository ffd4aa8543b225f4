"""Voxel volume measure (K4) -- the paper's "method of spheres" on voxels.

The reference measures S and V of a probe ball on triangle meshes by Monte
Carlo (morphology.py:238-306); it has no voxel form.  Here, on the
CT volume itself and exactly:

* ``threshold_count(volume, thr)``: number of voxels with value >= thr; the
  object volume is that count times the voxel volume sx*sy*sz.
* ``ball_measure(volume, thr, centres, radii)``: per probe ball B(X, R), the
  member voxels (value >= thr, centre (i*sx, j*sy, k*sz) inside the closed
  ball) -> V = count * voxel volume, and their exposed faces (6-neighbour
  below thr or outside the volume) -> S = sum of face areas; SVR = S / V
  (PAPER.md:150-172), undefined (None/NaN) where V == 0.

Integer results; the CPU restatement in oracle/ checks them bit-exactly
(parity unpinned: there is no reference function to pin against).
"""

from __future__ import annotations

import numpy as np

from . import _lib


def _dev(volume, device):
    import torch

    dvol = volume.device(device) if hasattr(volume, "device") and callable(volume.device) else volume
    return torch, dvol, torch.device("cuda", dvol.device)


def threshold_count(volume, thr: int, device: int = 0) -> int:
    torch, dvol, dev = _dev(volume, device)
    count = torch.zeros(1, dtype=torch.int64, device=dev)
    _lib.check(_lib.load().vr_threshold_count(dvol.handle, int(thr), _lib.ptr(count),
                                              _lib.ptr_stream(torch.cuda.current_stream(dev))))
    return int(count.item())


def threshold_volume_mm3(volume, thr: int, device: int = 0) -> float:
    sx, sy, sz = volume.spacing
    return threshold_count(volume, thr, device) * (sx * sy * sz)


def ball_counts(volume, thr: int, centres, radii, device: int = 0):
    """(counts (nballs,), faces (nballs, 3) exposed faces per axis) as uint64."""
    torch, dvol, dev = _dev(volume, device)
    c = np.ascontiguousarray(centres, dtype=np.float64).reshape(-1, 3)
    r = np.array(np.broadcast_to(np.asarray(radii, dtype=np.float64), (c.shape[0],)))
    n = c.shape[0]
    ct = torch.from_numpy(c).to(dev)
    rt = torch.from_numpy(r).to(dev)
    counts = torch.empty(n, dtype=torch.int64, device=dev)
    faces = torch.empty((n, 3), dtype=torch.int64, device=dev)
    _lib.check(_lib.load().vr_ball_counts(dvol.handle, int(thr), _lib.ptr(ct), _lib.ptr(rt), n,
                                          _lib.ptr(counts), _lib.ptr(faces),
                                          _lib.ptr_stream(torch.cuda.current_stream(dev))))
    return counts.cpu().numpy().astype(np.uint64), faces.cpu().numpy().astype(np.uint64)


def ball_measure(volume, thr: int, centres, radii, device: int = 0) -> dict:
    """V (mm^3), S (mm^2) and SVR = S/V per ball (NaN where V == 0)."""
    counts, faces = ball_counts(volume, thr, centres, radii, device)
    sx, sy, sz = volume.spacing
    V = counts.astype(np.float64) * (sx * sy * sz)
    f = faces.astype(np.float64)
    S = (f[:, 0] * (sy * sz) + f[:, 1] * (sx * sz)) + f[:, 2] * (sx * sy)
    with np.errstate(divide="ignore", invalid="ignore"):
        svr = np.where(V > 0, S / V, np.nan)
    return {"count": counts, "faces": faces, "V_mm3": V, "S_mm2": S, "svr": svr}
