"""K4 -- the method of spheres on voxels (csrc/vr_measure.cu).

V = count of voxels >= thr, S = area of the isosurface at thr - 0.5 of the
Kuhn-tetrahedra interpolant (exact fixed-point sum).  There is no reference
function for the voxel form, so the definition is pinned three
ways:

1. the C restatement (oracle/vr_oracle.c) equals an independent pure-Python
   marching-tetrahedra restatement on small volumes (CPU);
2. the analytic oracles of the reference spec (/root/reference/SPEC.md:472-473,
   the mesh estimators' own acceptance cases, morphology.py:270-306): a probe
   ball centred on a flat face -> SVR = 3/(2R), a ball enclosing a sphere of
   radius a -> SVR = 3/a, each within 3 %; plus S of a sphere -> 4 pi a^2
   and V -> 4/3 pi a^3 within 1 % (CPU, on the oracle);
3. the CUDA kernels equal the C restatement bit for bit (GPU).

Voxelisation: the test objects carry a linear partial-volume ramp across the
surface (100 HU per voxel, like CT's 1-2 voxel edges), and the flat face lies
between voxel centres; V counts whole voxels, so a face cutting through voxel
centres would add up to half a voxel of thickness (|dV|/V <= 0.75/R, checked).
"""

from __future__ import annotations

import math

import numpy as np
import pytest

from oracle import oracle as O

KUHN = ((0, 1, 2), (0, 2, 1), (1, 0, 2), (1, 2, 0), (2, 0, 1), (2, 1, 0))


def _py_measure(vals, spacing, thr, ball=None):
    """Independent restatement: numpy per tetrahedron, float64 area."""
    nz, ny, nx = vals.shape
    level = thr - 0.5
    pad = np.full((nz + 2, ny + 2, nx + 2), -32768.0)
    pad[1:-1, 1:-1, 1:-1] = vals
    f = pad - level
    sx, sy, sz = spacing
    total = 0.0
    for k in range(-1, nz):
        for j in range(-1, ny):
            for i in range(-1, nx):
                cube = f[k + 1:k + 3, j + 1:j + 3, i + 1:i + 3]
                if (cube > 0).all() or (cube <= 0).all():
                    continue
                for perm in KUHN:
                    corners = [np.zeros(3, int)]
                    for ax in perm:
                        c = corners[-1].copy()
                        c[ax] = 1
                        corners.append(c)
                    fv = [cube[c[2], c[1], c[0]] for c in corners]
                    P = [np.array([(i + c[0]) * sx, (j + c[1]) * sy, (k + c[2]) * sz]) for c in corners]
                    ins = [q for q in range(4) if fv[q] > 0]
                    outs = [q for q in range(4) if fv[q] <= 0]
                    if not ins or not outs:
                        continue

                    def ep(a, b):
                        t = fv[a] / (fv[a] - fv[b])
                        return P[a] + t * (P[b] - P[a])

                    if len(ins) == 1:
                        poly = [ep(ins[0], o) for o in outs]
                    elif len(outs) == 1:
                        poly = [ep(q, outs[0]) for q in ins]
                    else:
                        poly = [ep(ins[0], outs[0]), ep(ins[0], outs[1]), ep(ins[1], outs[1]), ep(ins[1], outs[0])]
                    if len(poly) == 3:
                        area = 0.5 * np.linalg.norm(np.cross(poly[1] - poly[0], poly[2] - poly[0]))
                    else:
                        area = 0.5 * np.linalg.norm(np.cross(poly[2] - poly[0], poly[3] - poly[1]))
                    if ball is not None:
                        g = np.mean(poly, axis=0)
                        if np.sum((g - ball[0]) ** 2) > ball[1] ** 2:
                            continue
                    total += area
    return total


def _sphere(a, spacing=(1.0, 1.0, 1.0), margin=6):
    n = [int(2 * a / s) + 2 * margin for s in spacing]
    c = [(n[q] - 1) * spacing[q] / 2 for q in range(3)]
    z, y, x = np.meshgrid(np.arange(n[2]) * spacing[2], np.arange(n[1]) * spacing[1],
                          np.arange(n[0]) * spacing[0], indexing="ij")
    r = np.sqrt((x - c[0]) ** 2 + (y - c[1]) ** 2 + (z - c[2]) ** 2)
    return np.clip(np.rint(100.0 * (a - r)), -1000, 1000).astype(np.int16), np.array(c)


def _half_space(R, xf):
    n = 3 * R + 10
    x = np.broadcast_to(np.arange(n, dtype=np.float64), (n, n, n))
    return np.clip(np.rint(100.0 * (xf - x)), -1000, 1000).astype(np.int16), np.array([xf, (n - 1) / 2, (n - 1) / 2])


@pytest.mark.parametrize("spacing", [(1.0, 1.0, 1.0), (0.8, 0.7, 1.5)])
def test_oracle_equals_python_restatement(spacing):
    vals = O.phantom("torso", (14, 12, 10))
    for thr in (-999, 40, 550, 1200):
        count, area = O.threshold_measure(vals, spacing, thr)
        assert count == int(np.count_nonzero(vals >= thr))
        assert abs(area / O.AREA_SCALE - _py_measure(vals, spacing, thr)) <= 1e-6 * max(1.0, area / O.AREA_SCALE)
    centre, rad = np.array([6.0, 5.0, 4.5]), 4.0
    counts, areas = O.ball_measure(vals, spacing, 40, centre[None], np.array([rad]))
    assert abs(areas[0] / O.AREA_SCALE - _py_measure(vals, spacing, 40, (centre, rad))) <= 1e-6 * max(
        1.0, areas[0] / O.AREA_SCALE)
    assert counts[0] == O.ball_counts(vals, spacing, 40, centre[None], np.array([rad]))[0]


@pytest.mark.parametrize("spacing", [(1.0, 1.0, 1.0), (0.8, 0.9, 1.2)])
@pytest.mark.parametrize("a", [8.0, 12.0, 20.0])
def test_sphere_area_volume_and_enclosing_ball(a, spacing):
    """S -> 4 pi a^2, V -> 4/3 pi a^3; a ball of radius > a centred on the
    sphere: SVR = 3/a within 3 %."""
    vals, c = _sphere(a, spacing)
    vox = spacing[0] * spacing[1] * spacing[2]
    count, area = O.threshold_measure(vals, spacing, 0)
    S, V = area / O.AREA_SCALE, count * vox
    assert abs(S / (4 * math.pi * a * a) - 1) < 0.01
    assert abs(V / (4 / 3 * math.pi * a ** 3) - 1) < 0.02
    counts, areas = O.ball_measure(vals, spacing, 0, c[None], np.array([a + 3.0]))
    svr = (areas[0] / O.AREA_SCALE) / (counts[0] * vox)
    assert abs(svr / (3.0 / a) - 1) < 0.03
    assert counts[0] == count and areas[0] == area  # the whole object is inside the ball


@pytest.mark.parametrize("R", [8, 12, 16])
def test_flat_face_svr(R):
    """Ball centred on a large flat face: S -> pi R^2, V -> 2/3 pi R^3,
    SVR -> 3/(2R) within 3 %."""
    n = 3 * R + 10
    vals, X = _half_space(R, n / 2 + 0.5)  # face between voxel centres
    counts, areas = O.ball_measure(vals, (1.0, 1.0, 1.0), 0, X[None], np.array([float(R)]))
    S, V = areas[0] / O.AREA_SCALE, float(counts[0])
    assert abs(S / (math.pi * R * R) - 1) < 0.015
    assert abs(V / (2 / 3 * math.pi * R ** 3) - 1) < 0.02
    assert abs((S / V) / (3.0 / (2 * R)) - 1) < 0.03
    # a face through voxel centres: S unchanged, V off by at most half a voxel slab
    for xf in (n / 2 + 0.25, n / 2):
        vals, X = _half_space(R, xf)
        counts, areas = O.ball_measure(vals, (1.0, 1.0, 1.0), 0, X[None], np.array([float(R)]))
        assert abs(areas[0] / O.AREA_SCALE / (math.pi * R * R) - 1) < 0.015
        assert abs(float(counts[0]) / (2 / 3 * math.pi * R ** 3) - 1) <= 0.75 / R + 0.02


def test_disjoint_ball_is_undefined():
    """Omega disjoint from G -> V = 0, SVR undefined (morphology.py:296-306)."""
    vals, c = _sphere(8.0)
    counts, areas = O.ball_measure(vals, (1.0, 1.0, 1.0), 0, np.array([[1.0, 1.0, 1.0], [-50.0, 9.0, 9.0]]),
                                   np.array([2.0, 5.0]))
    assert counts.tolist() == [0, 0] and areas.tolist() == [0, 0]


# ------------------------------------------------------------------ GPU


@pytest.mark.gpu
@pytest.mark.parametrize("dims,spacing", [((72, 60, 50), (0.8, 0.7, 1.5)), ((64, 64, 64), (1.0, 1.0, 1.0)),
                                          ((61, 37, 29), (1.0, 1.1, 0.9)), ((9, 8, 8), (1.0, 1.0, 1.0)),
                                          ((33, 8, 11), (0.5, 2.0, 1.0))])
def test_kernels_equal_restatement(dims, spacing):
    import paper_2005_01442_b200 as vr

    vol = vr.generate_phantom("torso", dims, spacing)
    for thr in (-1000, -999, 0, 40, 550, 1200, 1201, 32767, -32768):
        m = vr.threshold_measure(vol, thr)
        assert (m["count"], m["area_fx"]) == O.threshold_measure(vol.values, spacing, thr), thr
    rng = np.random.default_rng(0)
    centres = rng.uniform(-5, 60, size=(40, 3))
    radii = rng.uniform(0.5, 16.0, size=40)
    m = vr.ball_measure(vol, 550, centres, radii)
    want_c, want_a = O.ball_measure(vol.values, spacing, 550, centres, radii)
    assert np.array_equal(m["count"], want_c)
    assert np.array_equal(m["area_fx"], want_a)
    far = vr.ball_measure(vol, 550, np.array([[1e9, -1e9, 5.0]]), np.array([3.0]))
    assert far["count"].tolist() == [0] and far["area_fx"].tolist() == [0] and np.isnan(far["svr"][0])


@pytest.mark.gpu
def test_kernels_on_analytic_objects():
    import paper_2005_01442_b200 as vr

    vals, c = _sphere(12.0, (0.8, 0.9, 1.2))
    vol = vr.make_volume(vals, (0.8, 0.9, 1.2))
    m = vr.threshold_measure(vol, 0)
    assert (m["count"], m["area_fx"]) == O.threshold_measure(vals, (0.8, 0.9, 1.2), 0)
    b = vr.ball_measure(vol, 0, c[None], np.array([15.0]))
    assert abs(b["svr"][0] / (3.0 / 12.0) - 1) < 0.03
    vals, X = _half_space(12, 23.5)
    vol = vr.make_volume(vals, (1.0, 1.0, 1.0))
    b = vr.ball_measure(vol, 0, X[None], np.array([12.0]))
    assert abs(b["svr"][0] / (3.0 / 24.0) - 1) < 0.03


@pytest.mark.gpu
def test_kernels_on_noise_exercise_the_overflow_path():
    """A noise volume: almost every cell straddles the level, more than the
    straddling-cell list holds, so the one-pass fallback kernel computes S."""
    import paper_2005_01442_b200 as vr

    rng = np.random.default_rng(7)
    vals = rng.integers(-200, 200, size=(16, 20, 24)).astype(np.int16)
    vol = vr.make_volume(vals, (0.9, 1.1, 1.3))
    for thr in (0, 50, -150):
        m = vr.threshold_measure(vol, thr)
        assert (m["count"], m["area_fx"]) == O.threshold_measure(vals, (0.9, 1.1, 1.3), thr), thr
    centres = rng.uniform(0, 20, size=(12, 3))
    b = vr.ball_measure(vol, 0, centres, 4.0)
    want_c, want_a = O.ball_measure(vals, (0.9, 1.1, 1.3), 0, centres, np.full(12, 4.0))
    assert np.array_equal(b["count"], want_c) and np.array_equal(b["area_fx"], want_a)
