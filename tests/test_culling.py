"""Transparency-culling bounds (K1 cube / cell tables).

The reference evaluates every sample; the product skips samples whose
interpolated value provably classifies transparent.  What must hold is
rigor: every value the reference computes for a sample based in unit cube g
-- Catmull-Rom or trilinear, with any block-local clamping of its taps --
lies in the cube's bound.  CPU tests check that on adversarial volumes for the
float32 restatement in oracle/culling.py; GPU tests check the device tables
equal that restatement exactly.
"""

from __future__ import annotations

import numpy as np
import pytest

from oracle import culling


def volumes():
    rng = np.random.default_rng(7)
    yield "random", rng.integers(-3000, 3000, (11, 13, 14)).astype(np.int16)
    z, y, x = np.indices((10, 12, 9))
    yield "checker", np.where((x + y + z) % 2 == 0, 32000, -32000).astype(np.int16)
    yield "step", np.where(x >= 5, 1200, 40).astype(np.int16)
    spikes = np.full((9, 10, 11), 40, np.int16)
    spikes[4, 5, 5] = 1200
    spikes[1, 2, 8] = -1000
    yield "spikes", spikes
    yield "extremes", rng.choice(np.array([-32768, 32767, 0], np.int16), (8, 9, 10))


def _axis_taps(n, g, variant):
    """Tap indices of a sample based at g along one axis: unclamped (volume
    edges clamp) or with block-local clamping on the left / right / both."""
    idx = np.stack([g - 1, g, g + 1, g + 2], -1)
    if variant in (1, 3):
        idx[..., 0] = g
    if variant in (2, 3):
        idx[..., 3] = g + 1
    return np.clip(idx, 0, n - 1)


def _cr_values(vol, t, variants):
    """Reference-order Catmull-Rom value (_kernels.py:94-143) at base g = every
    voxel, fractional offsets t (3, nz, ny, nx), per-axis clamp variants."""
    v = vol.astype(np.float64)
    nz, ny, nx = v.shape
    gz, gy, gx = np.indices(v.shape)
    ix = _axis_taps(nx, gx, variants[0])
    iy = _axis_taps(ny, gy, variants[1])
    iz = _axis_taps(nz, gz, variants[2])
    wx, wy, wz = culling.cr_weights(t[0]), culling.cr_weights(t[1]), culling.cr_weights(t[2])
    planes = []
    for c in range(4):
        rows = []
        for r in range(4):
            tap = [v[iz[..., c], iy[..., r], ix[..., i]] for i in range(4)]
            rows.append(((wx[0] * tap[0] + wx[1] * tap[1]) + wx[2] * tap[2]) + wx[3] * tap[3])
        planes.append(((wy[0] * rows[0] + wy[1] * rows[1]) + wy[2] * rows[2]) + wy[3] * rows[3])
    return ((wz[0] * planes[0] + wz[1] * planes[1]) + wz[2] * planes[2]) + wz[3] * planes[3]


def _tri_values(vol, t):
    v = vol.astype(np.float64)
    nz, ny, nx = v.shape
    gz, gy, gx = np.indices(v.shape)
    x1, y1, z1 = np.minimum(gx + 1, nx - 1), np.minimum(gy + 1, ny - 1), np.minimum(gz + 1, nz - 1)
    fx, fy, fz = t
    c00 = v[gz, gy, gx] + (v[gz, gy, x1] - v[gz, gy, gx]) * fx
    c10 = v[gz, y1, gx] + (v[gz, y1, x1] - v[gz, y1, gx]) * fx
    c01 = v[z1, gy, gx] + (v[z1, gy, x1] - v[z1, gy, gx]) * fx
    c11 = v[z1, y1, gx] + (v[z1, y1, x1] - v[z1, y1, gx]) * fx
    c0 = c00 + (c10 - c00) * fy
    c1 = c01 + (c11 - c01) * fy
    return c0 + (c1 - c0) * fz


@pytest.mark.parametrize("name,vol", list(volumes()))
def test_cube_bounds_contain_every_interpolated_value(name, vol):
    b = culling.cube_bounds(vol).astype(np.float64)
    lo = np.where(b[..., 0] <= -32768, -np.inf, b[..., 0])
    hi = np.where(b[..., 1] >= 32767, np.inf, b[..., 1])
    rng = np.random.default_rng(11)
    for draw in range(6):
        t = rng.random((3,) + vol.shape)
        if draw == 0:
            t[:] = 0.5  # maximal negative lobes
        if draw == 1:
            t[:] = 1.0 / 3.0
        for variants in ((0, 0, 0), (1, 2, 3), (3, 1, 2), (2, 3, 1)):
            val = _cr_values(vol, t, variants)
            assert np.all(val >= lo) and np.all(val <= hi), (name, draw, variants)
        tri = _tri_values(vol, t)
        assert np.all(tri >= lo) and np.all(tri <= hi), (name, draw)


def test_cell_bounds_are_the_union_of_their_cubes():
    vol = next(volumes())[1]
    cubes = culling.cube_bounds(vol)
    cells = culling.cell_bounds(cubes)
    nz, ny, nx = vol.shape
    for cz in range(cells.shape[0]):
        for cy in range(cells.shape[1]):
            for cx in range(cells.shape[2]):
                sub = cubes[4 * cz:4 * cz + 4, 4 * cy:4 * cy + 4, 4 * cx:4 * cx + 4]
                assert cells[cz, cy, cx, 0] == sub[..., 0].min()
                assert cells[cz, cy, cx, 1] == sub[..., 1].max()


def test_bounds_are_tight_enough_to_matter():
    """A flat region far from an edge is bounded by its own value (±1)."""
    vol = np.full((12, 12, 12), 40, np.int16)
    vol[:, :, 9:] = 1200
    b = culling.cube_bounds(vol)
    assert b[5, 5, 3, 1] <= 41 and b[5, 5, 3, 0] >= 39


@pytest.mark.gpu
@pytest.mark.parametrize("name,vol", list(volumes()))
def test_device_tables_equal_the_restatement(name, vol):
    import paper_2005_01442_b200 as vr

    dv = vr.DeviceVolume.upload(vol, (1.0, 1.0, 1.0))
    cubes, cells = dv.culling_tables()
    ref = culling.cube_bounds(vol)
    np.testing.assert_array_equal(cubes, ref)
    np.testing.assert_array_equal(cells, culling.cell_bounds(ref))


@pytest.mark.gpu
def test_device_tables_on_the_torso_phantom():
    import paper_2005_01442_b200 as vr

    vol = vr.generate_phantom("torso", (40, 36, 33)).values
    cubes, cells = vr.DeviceVolume.upload(vol, (1.0, 1.0, 1.0)).culling_tables()
    ref = culling.cube_bounds(vol)
    np.testing.assert_array_equal(cubes, ref)
    np.testing.assert_array_equal(cells, culling.cell_bounds(ref))
