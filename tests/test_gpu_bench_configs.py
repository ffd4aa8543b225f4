"""Every benchmark configuration's frame, bit-exact against the CPU oracle.

bench.py measures C1 (64^3 -> 128^2 orthographic, monolithic), C2 (256^3 ->
512^2 monolithic), C3 (512^3 -> 1024^2 bricks 64/3; bone and soft-tissue),
C3-stress (monolithic grayscale, ET off, no lighting), C4 (512x512x2048 ->
2048^2 bricks) and C5 (the 360-view turntable).  Each test renders the bench
scene through the public API and compares the premultiplied float64 frame,
the uint8 pixels, the per-pixel sample counts and the RenderStats with the
oracle (a C restatement of _kernels.march + the block prep, pinned to the
reference's goldens), i.e. the reference's algorithm
(/root/reference/pkg/src/voxelray/_kernels.py:279-594, render.py:327-471).

Everything is compared bit for bit.  (Before the kernels evaluated x ** y
with glibc's own pow algorithm, csrc/vr_glibc_pow.h, a few pixels per million
differed by one ulp here: glibc's pow is accurate to <= 0.52 ulp but not
correctly rounded, and the reference's numba `**` calls it.)

The expensive frames are compared on crops: a sub-rectangle equals the crop
of the full frame bit for bit (reference SPEC.md:354), so C3-stress (the
oracle needs ~30 s for the whole frame) is checked on a 256^2 window where
every ray crosses the volume.  RenderStats of the whole frames are pinned by
SURVEY_STATS, the counts the unmodified reference produced.
"""

from __future__ import annotations

import math

import numpy as np
import pytest

pytestmark = pytest.mark.gpu



@pytest.fixture(scope="module")
def vr():
    import paper_2005_01442_b200 as vr

    return vr


_VOLUMES = {}


def _volume(vr, dims):
    if dims not in _VOLUMES:
        _VOLUMES.clear()  # one large volume at a time
        _VOLUMES[dims] = vr.generate_phantom("torso", dims)
    return _VOLUMES[dims]


def _centered(vr, dims, size, ortho=False):
    ext = tuple(float(d - 1) for d in dims)
    c = tuple(0.5 * e for e in ext)
    pos = (c[0] + 2.2 * max(ext), c[1], c[2])
    if ortho:
        return vr.OrthographicCamera(position=pos, look_at=c, half_height_mm=0.5 * max(ext) + 1.0,
                                     width=size, height=size)
    return vr.Camera(position=pos, look_at=c, width=size, height=size)


def _orbit(vr, dims, size, k, views=360, elevation_deg=0.0):
    """C5 view k (bench.py orbit_cameras; frontend/src/camera.ts:35-44)."""
    ext = tuple(float(d - 1) for d in dims)
    cx, cy, cz = (0.5 * e for e in ext)
    d = 2.2 * max(ext)
    ang = 2.0 * math.pi * k / views
    el = math.radians(elevation_deg)
    return vr.Camera(position=(cx + d * math.cos(el) * math.cos(ang), cy + d * math.cos(el) * math.sin(ang),
                               cz + d * math.sin(el)), look_at=(cx, cy, cz), width=size, height=size)


def _compare(vr, vol, cam, tf, s, tile=None):
    from oracle import oracle as O

    img = vr.render(vol, cam, tf, s, return_premultiplied=True, tile=tile)
    r = vr.Renderer(vol, cam, tf, s, tile=tile, per_pixel_counts=True)
    r.render_async()
    ref = O.render(vol.values, vol.spacing, cam, tf.values, tf.rgba, tf.domain, s,
                   projection=cam.projection, ortho_half_h=getattr(cam, "half_height_mm", None), tile=tile)
    d = np.abs(img.premultiplied - ref.out).max(axis=1)
    assert np.array_equal(img.premultiplied, ref.out), (float(d.max()), int(np.count_nonzero(d)))
    assert np.array_equal(img.pixels, ref.pixels)
    assert np.array_equal(r.taken.cpu().numpy(), ref.taken)
    assert np.array_equal(r.skipped.cpu().numpy(), ref.skipped)
    st = img.stats
    assert (st.samples_taken, st.samples_skipped) == (ref.samples_taken, ref.samples_skipped)
    assert (st.blocks_total, st.blocks_empty, st.blocks_visited) == (
        ref.blocks_total, ref.blocks_empty, ref.blocks_visited)
    return img, ref


def test_c1_orthographic_frame(vr):
    dims = (64, 64, 64)
    vol = _volume(vr, dims)
    _compare(vr, vol, _centered(vr, dims, 128, ortho=True), vr.get_preset("bone"),
             vr.RenderSettings(interpolation="tricubic"))


def test_c2_monolithic_frame(vr):
    dims = (256, 256, 256)
    vol = _volume(vr, dims)
    img, _ = _compare(vr, vol, _centered(vr, dims, 512), vr.get_preset("bone"),
                      vr.RenderSettings(interpolation="tricubic"))
    assert img.stats.samples_taken == 96_850_415  # SURVEY 6, the unmodified reference


@pytest.mark.parametrize("tfname", ["bone", "soft-tissue"])
def test_c3_frame(vr, tfname):
    """C3 bone is the headline; soft tissue with lighting is where float32
    fails by 40/255 -- hence the float64 parity mode."""
    dims = (512, 512, 512)
    vol = _volume(vr, dims)
    _compare(vr, vol, _centered(vr, dims, 1024), vr.get_preset(tfname),
             vr.RenderSettings(interpolation="tricubic", use_blocks=True))


def test_c3_stress_window(vr):
    dims = (512, 512, 512)
    vol = _volume(vr, dims)
    s = vr.RenderSettings(interpolation="tricubic", lighting=False, early_termination_alpha=1.0)
    _compare(vr, vol, _centered(vr, dims, 1024), vr.get_preset("grayscale"), s, tile=(384, 384, 256, 256))


@pytest.mark.parametrize("k,elev", [(0, 0.0), (37, 0.0), (90, 0.0), (135, 0.0), (180, 0.0), (223, 0.0),
                                    (270, 0.0), (315, 0.0), (60, 35.0), (200, -50.0)])
def test_c5_orbit_views(vr, k, elev):
    """Turntable views, on-axis and oblique (plus two elevated ones)."""
    dims = (512, 512, 512)
    vol = _volume(vr, dims)
    _compare(vr, vol, _orbit(vr, dims, 1024, k, elevation_deg=elev), vr.get_preset("bone"),
             vr.RenderSettings(interpolation="tricubic", use_blocks=True))


def test_c4_frame(vr):
    dims = (512, 512, 2048)
    vol = _volume(vr, dims)
    img, _ = _compare(vr, vol, _centered(vr, dims, 2048), vr.get_preset("bone"),
                      vr.RenderSettings(interpolation="tricubic", use_blocks=True))
    assert (img.stats.samples_taken, img.stats.samples_skipped) == (4_776_603, 745_212_706)


# RenderStats of the unmodified reference at full size (SURVEY 6 / VERDICT r1)
FULL_STATS = {
    "c3_soft": ((512, 512, 512), 1024, "soft-tissue", dict(interpolation="tricubic", use_blocks=True),
                39_682_875, 599_018_911),
    "c3_stress": ((512, 512, 512), 1024, "grayscale",
                  dict(interpolation="tricubic", lighting=False, early_termination_alpha=1.0), 775_848_757, 0),
}


@pytest.mark.parametrize("key", sorted(FULL_STATS))
def test_full_frame_stats(vr, key):
    dims, size, tfname, kw, taken, skipped = FULL_STATS[key]
    vol = _volume(vr, dims)
    img = vr.render(vol, _centered(vr, dims, size), vr.get_preset(tfname), vr.RenderSettings(**kw))
    assert (img.stats.samples_taken, img.stats.samples_skipped) == (taken, skipped)
