"""The CPU oracle against golden vectors produced by the unmodified reference.

This pins oracle/ (tests/golden/make_golden.py ran the reference's own
render(), decompose(), with_visibility(), sample(), gradient(),
build_lut(), build_preintegrated() and generate_phantom()).  Everything must
match bit for bit.
"""

from __future__ import annotations

import hashlib
from types import SimpleNamespace

import numpy as np
import pytest

from conftest import compare_render, settings_dict, tf_arrays
from oracle import oracle as O


def _cases(meta):
    return [c["name"] for c in meta["cases"]]


def test_every_render_case_bit_exact(golden_meta, golden_renders):
    worst = []
    for case in golden_meta["cases"]:
        vals = O.phantom(case["phantom"], case["dims"])
        v, c, dom = tf_arrays(case["tf"])
        r = O.render(vals, case["spacing"], SimpleNamespace(**case["camera"]), v, c, dom,
                     SimpleNamespace(**settings_dict(case)), projection=case["projection"],
                     ortho_half_h=case["ortho_half_h"])
        stats = [r.out.shape[0], r.samples_taken, r.samples_skipped, r.blocks_total,
                 r.blocks_empty, r.blocks_visited]
        d_out, d_px = compare_render(case["name"], golden_renders, r.out, r.pixels, stats,
                                     taken=r.taken, blocks_hit=r.blocks_hit)
        if case["settings"].get("mode") == "isosurface":
            g = golden_renders[case["name"] + "__depth"]
            assert np.array_equal(np.isnan(g), np.isnan(r.depth))
            assert np.array_equal(g[~np.isnan(g)], r.depth[~np.isnan(r.depth)])
        worst.append((d_out, d_px))
        assert d_out == 0.0 and d_px == 0, case["name"]
    assert len(worst) == len(golden_meta["cases"])


def test_tile_equals_crop(golden_meta, golden_renders):
    """a sub-rectangle render equals the crop of the full frame."""
    case = next(c for c in golden_meta["cases"] if c["name"] == "torso48_bone_cubic_blocks16")
    vals = O.phantom(case["phantom"], case["dims"])
    v, c, dom = tf_arrays(case["tf"])
    W = case["camera"]["width"]
    tile = (5, 9, 23, 17)
    r = O.render(vals, case["spacing"], SimpleNamespace(**case["camera"]), v, c, dom,
                 SimpleNamespace(**settings_dict(case)), tile=tile)
    full = golden_renders[case["name"] + "__out"].reshape(-1, W, 4)
    crop = full[tile[1]:tile[1] + tile[3], tile[0]:tile[0] + tile[2]].reshape(-1, 4)
    assert np.array_equal(r.out, crop)


def test_phantom_hashes(golden_meta):
    for key, digest in golden_meta["phantom_sha256"].items():
        name, dims = key.split("_")
        dims = tuple(int(d) for d in dims.split("x"))
        if np.prod(dims) > 300_000:
            continue  # the big ones are checked on the GPU (device generator)
        vals = O.phantom(name, dims)
        assert hashlib.sha256(vals.astype("<i2").tobytes()).hexdigest() == digest, key


@pytest.mark.parametrize("name,dims,bs,ov", [("torso64_16_3", (64, 64, 64), 16, 3),
                                             ("torso96x80x64_64_3", (96, 80, 64), 64, 3),
                                             ("torso48_10_1", (48, 48, 48), 10, 1)])
def test_block_prep(golden_prep, name, dims, bs, ov):
    vals = O.phantom("torso", dims)
    g = O.decompose(vals, bs, ov)
    assert np.array_equal(g.vmin, golden_prep[f"{name}_vmin"])
    assert np.array_equal(g.vmax, golden_prep[f"{name}_vmax"])
    for tfn, spec in (("bone", {"preset": "bone"}), ("soft-tissue", {"preset": "soft-tissue"}),
                      ("custom", {"points": [[-500.0, 0, 0, 0, 0.0], [300.0, 0.9, 0.5, 0.2, 0.0],
                                             [700.0, 1.0, 0.8, 0.6, 0.6], [1500.0, 1.0, 1.0, 1.0, 0.9]],
                                  "domain": [-600.0, 1400.0]})):
        v, c, dom = tf_arrays(spec)
        lut = O.build_lut(v, c, dom)
        gg = O.with_visibility(vals, O.decompose(vals, bs, ov), lut, dom)
        assert np.array_equal(gg.empty, golden_prep[f"{name}_{tfn}_empty"])
        assert np.array_equal(gg.aabb_lo, golden_prep[f"{name}_{tfn}_lo"])
        assert np.array_equal(gg.aabb_hi, golden_prep[f"{name}_{tfn}_hi"])


def test_luts_and_preintegration(golden_prep):
    for tfn in ("bone", "soft-tissue", "grayscale"):
        v, c, dom = tf_arrays({"preset": tfn})
        assert np.array_equal(O.build_lut(v, c, dom), golden_prep[f"lut_{tfn}"])
    v, c, dom = tf_arrays({"preset": "soft-tissue"})
    table = O.preintegrated(O.build_lut(v, c, dom), dom, 0.35, 0.5)
    assert np.array_equal(table[::17, ::13], golden_prep["preint_soft_0.35_strided"])
    digest = np.frombuffer(hashlib.sha256(np.ascontiguousarray(table).tobytes()).digest(), np.uint8)
    assert np.array_equal(digest, golden_prep["preint_soft_0.35_sha256"])


def test_point_sampling(golden_sampling):
    n = 16
    z, y, x = np.meshgrid(np.arange(n), np.arange(n), np.arange(n), indexing="ij")
    cub = np.asarray((x + 8.0) ** 3, dtype=np.int16)
    torso = O.phantom("torso", (24, 20, 16))
    pts = golden_sampling["pts"]
    for interp, cubic in (("trilinear", False), ("tricubic", True)):
        assert np.array_equal(O.sample_points(cub, pts, cubic), golden_sampling[f"cub_{interp}_sample"])
        assert np.array_equal(O.gradient_points(cub, pts, cubic, (1, 1, 1)), golden_sampling[f"cub_{interp}_grad"])
        assert np.array_equal(O.sample_points(torso, pts, cubic), golden_sampling[f"torso_{interp}_sample"])
        assert np.array_equal(O.gradient_points(torso, pts, cubic, (0.5, 1.0, 2.0)),
                              golden_sampling[f"torso_{interp}_grad"])


def test_threshold_restatement_matches_numpy():
    """K4 has no reference function (parity unpinned); check the C restatement
    against numpy on the same definition."""
    vals = O.phantom("torso", (40, 36, 32))
    for thr in (-1000, 0, 550, 1200, 1201):
        assert O.threshold_count(vals, thr) == int(np.count_nonzero(vals >= thr))
    sp = (0.8, 0.7, 1.5)
    centres = np.array([[15.0, 12.0, 20.0], [0.0, 0.0, 0.0], [31.2, 24.5, 46.5]])
    radii = np.array([6.0, 10.0, 3.3])
    got = O.ball_counts(vals, sp, 550, centres, radii)
    k, j, i = np.meshgrid(np.arange(32), np.arange(36), np.arange(40), indexing="ij")
    for q in range(3):
        d2 = ((i * sp[0] - centres[q, 0]) ** 2 + (j * sp[1] - centres[q, 1]) ** 2) + (k * sp[2] - centres[q, 2]) ** 2
        member = (d2 <= radii[q] ** 2) & (vals >= 550)
        assert got[q] == np.count_nonzero(member)

