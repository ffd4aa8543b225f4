"""Randomised parity: GPU render() vs the CPU oracle on seeded random scenes.

Covers the combinations the fixed goldens do not reach: oblique / grazing
cameras, anisotropic spacing, odd dimensions, random block sizes and
overlaps, custom transfer functions with narrow domains, all classification
modes, and step sizes whose opacity-correction exponent step/ref_step is 1,
1/2 or an integer.  Everything the leaps, culling tables, hand-off to the
cooperative kernel and block attribution decide must leave the result
bit-identical -- premultiplied float64 colours, uint8 pixels and the stats --
whatever the exponent: the device evaluates (1-a)^e and the Phong power with
glibc's own pow algorithm and tables (csrc/vr_glibc_pow.h), as the reference's
numba `**` does through libm.
"""

from __future__ import annotations

import math

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

N_CASES = 80


def _case(seed):
    rng = np.random.default_rng(1000 + seed)
    phantom = ["torso", "torso", "sphere", "shell"][seed % 4]
    dims = tuple(int(d) for d in rng.integers(24, 72, 3))
    spacing = tuple(float(s) for s in rng.choice([0.5, 0.8, 1.0, 1.0, 1.25, 1.6], 3))
    ext = [(d - 1) * s for d, s in zip(dims, spacing)]
    centre = np.array(ext) / 2.0
    direction = rng.normal(size=3)
    direction /= np.linalg.norm(direction)
    dist = float(rng.uniform(1.4, 3.0)) * max(ext)
    position = centre + dist * direction
    look_at = centre + rng.uniform(-0.15, 0.15, 3) * np.array(ext)
    up = rng.normal(size=3)
    fwd = (look_at - position) / np.linalg.norm(look_at - position)
    if abs(float(np.dot(up / np.linalg.norm(up), fwd))) > 0.95:
        up = np.cross(fwd, [1.0, 0.0, 0.0])
    w, h = int(rng.integers(24, 56)), int(rng.integers(20, 48))
    ortho = seed % 7 == 3
    mode = "isosurface" if seed % 11 == 5 else "dvr"
    classification = {9: "pre", 10: "preintegrated"}.get(seed % 12, "post")
    tf = ["bone", "soft-tissue", "grayscale", "custom"][int(rng.integers(0, 4))]
    custom = None
    if tf == "custom":
        lo = float(rng.uniform(-1200, 200))
        hi = lo + float(rng.uniform(150, 2500))
        xs = np.sort(rng.uniform(lo, hi, 4))
        custom = dict(points=[(float(x), *map(float, rng.uniform(0, 1, 3)), float(a))
                              for x, a in zip(xs, [0.0, rng.uniform(0, 0.6), rng.uniform(0.2, 1), 0.0])],
                      domain=(lo, hi))
    ref_step = 0.5 * min(spacing)
    factor = float(rng.choice([1.0, 1.0, 0.5, 2.0, 3.0]))
    settings = dict(
        interpolation="tricubic" if rng.random() < 0.7 else "trilinear",
        lighting=bool(rng.random() < 0.7),
        use_blocks=bool(rng.random() < 0.6),
        block_size=int(rng.integers(8, 33)),
        overlap=int(rng.integers(1, 4)),
        step=ref_step * factor,
        early_termination_alpha=float(rng.choice([0.95, 0.99, 1.0])),
        mode=mode, classification=classification)
    if mode == "isosurface":
        settings["isovalue"] = 600.0 if phantom == "torso" else 500.0
    return dict(phantom=phantom, dims=dims, spacing=spacing, position=tuple(position), look_at=tuple(look_at),
                up=tuple(up), fov=float(rng.uniform(20, 50)), w=w, h=h, ortho=ortho, ortho_half=0.6 * max(ext),
                tf=tf, custom=custom, settings=settings)


@pytest.mark.parametrize("seed", range(N_CASES))
def test_random_scene_matches_oracle(seed):
    import paper_2005_01442_b200 as vr
    from oracle import oracle as O

    c = _case(seed)
    vol = vr.generate_phantom(c["phantom"], c["dims"], c["spacing"])
    if c["ortho"]:
        cam = vr.OrthographicCamera(position=c["position"], look_at=c["look_at"], up=c["up"],
                                    half_height_mm=c["ortho_half"], width=c["w"], height=c["h"])
    else:
        cam = vr.Camera(position=c["position"], look_at=c["look_at"], up=c["up"], vertical_fov_deg=c["fov"],
                        width=c["w"], height=c["h"])
    if c["custom"]:
        tf = vr.transfer_from_points(c["custom"]["points"], domain=c["custom"]["domain"])
    else:
        tf = vr.get_preset(c["tf"])
    s = vr.RenderSettings(**c["settings"])
    if s.mode == "isosurface" and not (vol.value_range[0] <= s.isovalue <= vol.value_range[1]):
        pytest.skip("isovalue outside this phantom's range")
    try:
        img = vr.render(vol, cam, tf, s, return_premultiplied=True)
    except vr.EmptyBlock:
        pytest.skip("a block passes the interval test without a visible voxel: the reference raises "
                    "EmptyBlock here too (blocks.py:186-187)")
    ref = O.render(vol.values, vol.spacing, cam, tf.values, tf.rgba, tf.domain, s,
                   projection=getattr(cam, "projection", "pinhole"),
                   ortho_half_h=getattr(cam, "half_height_mm", None))
    d = float(np.abs(img.premultiplied - ref.out).max())
    assert np.array_equal(img.premultiplied, ref.out), (seed, c["settings"], d)
    assert np.array_equal(img.pixels, ref.pixels), seed
    assert img.stats.samples_taken == ref.samples_taken, seed
    assert img.stats.samples_skipped == ref.samples_skipped, seed
    if s.use_blocks:
        assert img.stats.blocks_visited == ref.blocks_visited, seed
        assert img.stats.blocks_empty == ref.blocks_empty, seed
    if s.mode == "isosurface":
        both = np.isnan(img.depth.ravel()) == np.isnan(ref.depth)
        assert both.all()
        ok = ~np.isnan(ref.depth)
        assert np.abs(img.depth.ravel()[ok] - ref.depth[ok]).max(initial=0.0) <= 1e-9
    assert math.isfinite(d)
