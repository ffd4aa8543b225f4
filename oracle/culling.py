"""Restatement of K1's transparency-culling bounds (TEST INFRASTRUCTURE ONLY).

Only tests/ import this: it is the checker for ``cube_bound_kernel`` /
``cell_from_cubes_kernel`` (csrc/vr_prep.cu).  The reference has no such
table -- it evaluates every sample (``_kernels.py:508-537``) -- so what must
hold is rigor: every interpolated value the reference computes for a sample
based in cube g (``_cub_sample`` / ``_tri_sample``, ``_kernels.py:52-143``,
with block-local tap clamping) lies in the cube's bound.  tests/test_culling.py
checks both that and that the device table equals this float32 restatement.
"""

from __future__ import annotations

import numpy as np

F = np.float32


def _row_hull(a, b, c, d):
    k = F(1.0) / F(6.0)
    p1, p1c = b + (c - a) * k, b + (c - b) * k
    p2, p2c = c - (d - b) * k, c - (c - b) * k
    lo = np.minimum(np.minimum(np.minimum(b, c), np.minimum(p1, p1c)), np.minimum(p2, p2c))
    hi = np.maximum(np.maximum(np.maximum(b, c), np.maximum(p1, p1c)), np.maximum(p2, p2c))
    return lo, hi


def _span_hull(s0, s1, s2, s3):
    k = F(1.0) / F(6.0)
    l0, l3 = np.minimum(s0[0], s1[0]), np.minimum(s3[0], s2[0])
    h0, h3 = np.maximum(s0[1], s1[1]), np.maximum(s3[1], s2[1])
    hi = np.maximum(np.maximum(s1[1], s2[1]), np.maximum(s1[1] + (s2[1] - l0) * k, s2[1] - (l3 - s1[1]) * k))
    lo = np.minimum(np.minimum(s1[0], s2[0]), np.minimum(s1[0] + (s2[0] - h0) * k, s2[0] - (h3 - s1[0]) * k))
    return lo, hi


def cube_bounds(values: np.ndarray) -> np.ndarray:
    """(nz, ny, nx, 2) int16 bounds for an int16 (nz, ny, nx) volume."""
    v = values.astype(F)
    nz, ny, nx = v.shape
    iz, iy, ix = np.arange(nz), np.arange(ny), np.arange(nx)

    def tap(arr, axis, n, off):
        idx = np.clip(np.arange(n) + off, 0, n - 1)
        return np.take(arr, idx, axis=axis)

    planes = []
    for kz in range(4):
        vz = tap(v, 0, nz, kz - 1)
        rows = []
        for jy in range(4):
            vy = tap(vz, 1, ny, jy - 1)
            rows.append(_row_hull(tap(vy, 2, nx, -1), tap(vy, 2, nx, 0), tap(vy, 2, nx, 1), tap(vy, 2, nx, 2)))
        planes.append(_span_hull(*rows))
    lo, hi = _span_hull(*planes)
    lo = np.maximum(np.floor(lo) - F(1), F(-32768))
    hi = np.minimum(np.ceil(hi) + F(1), F(32767))
    del iz, iy, ix
    return np.stack([lo, hi], -1).astype(np.int16)


def cell_bounds(cubes: np.ndarray) -> np.ndarray:
    """Union over 4^3 cells of the per-cube bounds."""
    nz, ny, nx, _ = cubes.shape
    cz, cy, cx = -(-nz // 4), -(-ny // 4), -(-nx // 4)
    lo = np.full((cz * 4, cy * 4, cx * 4), 32767, np.int32)
    hi = np.full((cz * 4, cy * 4, cx * 4), -32768, np.int32)
    lo[:nz, :ny, :nx] = cubes[..., 0]
    hi[:nz, :ny, :nx] = cubes[..., 1]
    lo = lo.reshape(cz, 4, cy, 4, cx, 4).min(axis=(1, 3, 5))
    hi = hi.reshape(cz, 4, cy, 4, cx, 4).max(axis=(1, 3, 5))
    return np.stack([lo, hi], -1).astype(np.int16)


def cr_weights(t):
    """_kernels.py:83-91."""
    t2 = t * t
    t3 = t2 * t
    return (0.5 * ((-t3 + 2.0 * t2) - t), 0.5 * ((3.0 * t3 - 5.0 * t2) + 2.0),
            0.5 * ((-3.0 * t3 + 4.0 * t2) + t), 0.5 * (t3 - t2))
