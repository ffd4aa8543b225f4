"""Edge cases of the render path vs the CPU oracle: degenerate sizes, a camera
inside the volume, rays along the axes (zero direction components), blocks
larger than the volume, and a frame larger than the cooperative kernel's
hand-off queue would hold at once."""

from __future__ import annotations

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _check(vr, vol, cam, tf, s):
    from oracle import oracle as O

    img = vr.render(vol, cam, tf, s, return_premultiplied=True)
    ref = O.render(vol.values, vol.spacing, cam, tf.values, tf.rgba, tf.domain, s,
                   projection=getattr(cam, "projection", "pinhole"),
                   ortho_half_h=getattr(cam, "half_height_mm", None))
    assert np.array_equal(img.premultiplied, ref.out)
    assert np.array_equal(img.pixels, ref.pixels)
    assert img.stats.samples_taken == ref.samples_taken
    assert img.stats.samples_skipped == ref.samples_skipped
    return img


@pytest.fixture(scope="module")
def vr():
    import paper_2005_01442_b200 as vr

    return vr


@pytest.mark.parametrize("interp", ["tricubic", "trilinear"])
@pytest.mark.parametrize("blocks", [False, True])
def test_minimum_volume(vr, interp, blocks):
    vals = np.array([[[-1000, 40], [1200, 300]], [[500, 2000], [-200, 900]]], dtype=np.int16)
    vol = vr.make_volume(vals, (1.0, 1.0, 1.0))
    cam = vr.Camera(position=(4.0, 1.3, 0.7), look_at=(0.5, 0.5, 0.5), width=9, height=7)
    _check(vr, vol, cam, vr.get_preset("grayscale"),
           vr.RenderSettings(interpolation=interp, use_blocks=blocks, block_size=8, overlap=3))


def test_single_pixel(vr):
    vol = vr.generate_phantom("torso", (32, 30, 28))
    c = tuple(0.5 * e for e in vol.extent_mm)
    cam = vr.Camera(position=(c[0] + 80.0, c[1], c[2]), look_at=c, width=1, height=1)
    _check(vr, vol, cam, vr.get_preset("bone"), vr.RenderSettings(interpolation="tricubic", use_blocks=True,
                                                                    block_size=16))


def test_camera_inside_the_volume(vr):
    vol = vr.generate_phantom("torso", (48, 48, 48))
    c = tuple(0.5 * e for e in vol.extent_mm)
    cam = vr.Camera(position=(c[0] + 5.0, c[1] - 3.0, c[2] + 2.0), look_at=(0.0, 0.0, 0.0),
                    vertical_fov_deg=70.0, width=40, height=36)
    for tf in ("bone", "soft-tissue"):
        _check(vr, vol, cam, vr.get_preset(tf), vr.RenderSettings(interpolation="tricubic", use_blocks=True,
                                                                    block_size=16, overlap=2))


def test_axis_aligned_orthographic_rays(vr):
    """Parallel rays along -x: two direction components are exactly zero."""
    vol = vr.generate_phantom("torso", (40, 36, 32))
    ext = vol.extent_mm
    c = tuple(0.5 * e for e in ext)
    cam = vr.OrthographicCamera(position=(c[0] + 100.0, c[1], c[2]), look_at=c, up=(0.0, 0.0, 1.0),
                                half_height_mm=0.6 * max(ext), width=48, height=44)
    for blocks in (False, True):
        _check(vr, vol, cam, vr.get_preset("bone"),
               vr.RenderSettings(interpolation="tricubic", use_blocks=blocks, block_size=12, overlap=3))


def test_block_larger_than_volume(vr):
    vol = vr.generate_phantom("sphere", (20, 18, 16))
    c = tuple(0.5 * e for e in vol.extent_mm)
    cam = vr.Camera(position=(c[0] + 50.0, c[1] + 20.0, c[2]), look_at=c, width=30, height=26)
    _check(vr, vol, cam, vr.get_preset("bone"),
           vr.RenderSettings(interpolation="tricubic", use_blocks=True, block_size=64, overlap=3))


def test_many_long_rays_wide_frame(vr):
    """A 700x300 frame on an elongated volume: tens of thousands of rays go to
    the cooperative kernel's queues."""
    vol = vr.generate_phantom("torso", (96, 40, 40))
    ext = vol.extent_mm
    c = tuple(0.5 * e for e in ext)
    cam = vr.Camera(position=(c[0] + 260.0, c[1] + 12.0, c[2] + 9.0), look_at=c, vertical_fov_deg=20.0,
                    width=700, height=300)
    _check(vr, vol, cam, vr.get_preset("soft-tissue"),
           vr.RenderSettings(interpolation="tricubic", use_blocks=True, block_size=24, overlap=3))
