"""Host-side API of the package, no GPU needed: the reference's pins for rays,
compositing, shading, settings, transfer functions and block specs
(reference pkg/tests/test_render.py, test_transfer.py, test_blocks.py) applied
to this package, plus bit-exactness of the host-built tables against the
reference's goldens."""

from __future__ import annotations

import hashlib
import math

import numpy as np
import pytest

import paper_2005_01442_b200 as vr
from paper_2005_01442_b200.errors import InvalidBlockSpec, InvalidSettings


# ------------------------------------------------------------------ rays


def test_center_pixel_ray_hits_look_at():
    cam = vr.Camera(position=(10.0, 3.0, -2.0), look_at=(1.0, 2.0, 5.0), width=97, height=97)
    origin, direction = vr.generate_ray(cam, (48, 48))
    fwd = np.subtract(cam.look_at, cam.position)
    assert np.allclose(origin, cam.position)
    assert np.allclose(direction, fwd / np.linalg.norm(fwd), atol=1e-6)


def test_vertical_subtense_matches_fov():
    h = 401
    cam = vr.Camera(position=(0.0, 0.0, 0.0), look_at=(0.0, 0.0, -50.0), up=(0, 1, 0),
                    vertical_fov_deg=40.0, width=401, height=h)
    _, top = vr.generate_ray(cam, (200, 0))
    _, bottom = vr.generate_ray(cam, (200, h - 1))
    angle = math.acos(float(np.clip(top @ bottom, -1.0, 1.0)))
    expected = 2.0 * math.atan(math.tan(math.radians(40.0) / 2.0) * (1.0 - 1.0 / h))
    assert abs(angle - expected) < 1e-9


def test_camera_validation():
    for kw in (dict(position=(0, 0, 0), look_at=(0, 0, 0)),
               dict(position=(0, 0, 0), look_at=(0, 0, 1), up=(0, 0, 2)),
               dict(position=(0, 0, 0), look_at=(1, 0, 0), vertical_fov_deg=180.0),
               dict(position=(0, 0, 0), look_at=(1, 0, 0), width=0)):
        with pytest.raises(ValueError):
            vr.Camera(**kw)
    with pytest.raises(ValueError):
        vr.OrthographicCamera(position=(0, 0, 0), look_at=(1, 0, 0), half_height_mm=0.0)


def test_camera_dict_round_trip():
    cam = vr.Camera(position=(1, 2, 3), look_at=(4, 5, 6), up=(0, 1, 0), vertical_fov_deg=25.0,
                    width=10, height=20)
    again = vr.camera_from_dict(cam.to_dict())
    assert tuple(again.position) == (1, 2, 3) and again.vertical_fov_deg == 25.0
    assert (again.width, again.height) == (10, 20)


def test_camera_struct_matches_reference_basis():
    """The C camera carries Camera.basis() and tan(fov/2) exactly as render.py:125-144 computes them."""
    from paper_2005_01442_b200.render import camera_struct

    cam = vr.Camera(position=(140.0, 31.5, 31.5), look_at=(31.5, 31.5, 31.5), up=(0.0, 0.3, 1.0),
                    vertical_fov_deg=41.0, width=36, height=28)
    c = camera_struct(cam, tile=(3, 4, 10, 11), interleave=(4, 1))
    fwd = np.subtract(cam.look_at, cam.position, dtype=np.float64)
    fwd /= np.linalg.norm(fwd)
    right = np.cross(fwd, np.asarray(cam.up, dtype=np.float64))
    right /= np.linalg.norm(right)
    up = np.cross(right, fwd)
    assert list(c.fwd) == list(fwd) and list(c.right) == list(right) and list(c.up) == list(up)
    half_h = math.tan(math.radians(41.0) / 2.0)
    assert c.half_h == half_h and c.half_w == half_h * 36 / 28
    assert (c.tile_x, c.tile_y, c.tile_w, c.tile_h, c.interleave_n, c.interleave_k) == (3, 4, 10, 11, 4, 1)


# ----------------------------------------------------------- compositing


def test_composite_hand_values():
    assert vr.composite_step((0.0, 0.0, 0.0, 0.0), (1.0, 0.0, 0.0, 1.0), 0.5, 0.5) == (1.0, 0.0, 0.0, 1.0)
    dst = (0.3, 0.2, 0.1, 0.6)
    assert vr.composite_step(dst, (1.0, 1.0, 1.0, 0.0), 0.5, 0.5) == dst
    d = vr.composite_step((0.0, 0.0, 0.0, 0.0), (1.0, 0.0, 0.0, 0.5), 1.0, 1.0)
    d = vr.composite_step(d, (0.0, 0.0, 1.0, 1.0), 1.0, 1.0)
    assert np.allclose(d, (0.5, 0.0, 0.5, 1.0))
    out = vr.composite_step((0.0, 0.0, 0.0, 0.0), (1.0, 1.0, 1.0, 0.75), 1.0, 0.5)
    assert math.isclose(out[3], 0.9375)


def test_shade_hand_values():
    assert np.allclose(vr.shade_headlight((0.5, 0.25, 0.0), (4.0, 0.0, 0.0), (1.0, 0.0, 0.0)),
                       (0.5 * 0.8 + 0.2, 0.25 * 0.8 + 0.2, 0.2))
    assert np.allclose(vr.shade_headlight((0.6, 0.6, 0.6), (0.0, 2.0, 0.0), (1.0, 0.0, 0.0)), (0.06,) * 3)
    assert vr.shade_headlight((0.4, 0.5, 0.6), (0.0, 0.0, 0.0), (1, 0, 0)) == (0.4, 0.5, 0.6)
    assert np.allclose(vr.shade_headlight((1.0, 0.0, 0.0), (-3.0, 0.0, 0.0), (1.0, 0.0, 0.0)), (0.3, 0.2, 0.2))
    assert vr.shade_headlight((1.0, 1.0, 1.0), (9.0, 0.0, 0.0), (1.0, 0.0, 0.0)) == (1.0, 1.0, 1.0)


# -------------------------------------------------------------- settings


def test_settings_validation():
    for kw in (dict(step=0.0), dict(interpolation="nearest"), dict(classification="mid"),
               dict(mode="mip"), dict(mode="isosurface"), dict(early_termination_alpha=0.0),
               dict(background=(2.0, 0.0, 0.0, 1.0))):
        with pytest.raises(InvalidSettings):
            vr.RenderSettings(**kw).validate()
    vr.RenderSettings(mode="isosurface", isovalue=100.0).validate()


def test_settings_dict_round_trip_and_unknown_keys():
    s = vr.RenderSettings(step=0.25, classification="preintegrated", use_blocks=True)
    again = vr.settings_from_dict(s.to_dict())
    assert again.step == 0.25 and again.classification == "preintegrated"
    with pytest.raises(InvalidSettings):
        vr.settings_from_dict({"stepp": 1.0})


def test_error_codes_are_class_names():
    assert InvalidSettings("x").code == "InvalidSettings"
    assert vr.IsovalueOutOfRange("x").code == "IsovalueOutOfRange"


# -------------------------------------------------------------- transfer


def ramp_tf():
    return vr.transfer_from_points([(0.0, 0.0, 0.0, 0.0, 0.0), (100.0, 1.0, 0.5, 0.0, 1.0)])


def test_evaluate_and_bins():
    tf = ramp_tf()
    assert np.allclose(tf.evaluate(50.0), [0.5, 0.25, 0.0, 0.5])
    lut = vr.build_lut(tf, bins=10)
    assert lut.bin_width == 10.0
    assert lut.bin_index(0.0) == 0 and lut.bin_index(9.999) == 0 and lut.bin_index(10.0) == 1
    assert lut.bin_index(-50.0) == 0 and lut.bin_index(1e9) == 9
    with pytest.raises(ValueError):
        vr.transfer_from_points([(0, 0, 0, 0, 0), (0, 1, 1, 1, 1)])
    with pytest.raises(ValueError):
        vr.transfer_from_points([(0, 0, 0, 0, 2.0)])


def test_transfer_round_trip_and_presets():
    tf = ramp_tf()
    back = vr.transfer_from_dict(tf.to_dict())
    assert np.array_equal(back.values, tf.values) and np.array_equal(back.rgba, tf.rgba)
    assert set(vr.transfer.PRESET_NAMES) == {"bone", "grayscale", "soft-tissue"}
    assert np.array_equal(vr.resolve_transfer("bone").rgba, vr.resolve_transfer({"preset": "bone"}).rgba)
    with pytest.raises(KeyError):
        vr.resolve_transfer({"preset": "marble"})


def test_luts_bit_exact_vs_reference(golden_prep):
    for name in ("bone", "soft-tissue", "grayscale"):
        assert np.array_equal(vr.build_lut(vr.get_preset(name)).rgba, golden_prep[f"lut_{name}"])
    custom = vr.transfer_from_points([(-500.0, 0, 0, 0, 0.0), (300.0, 0.9, 0.5, 0.2, 0.0),
                                      (700.0, 1.0, 0.8, 0.6, 0.6), (1500.0, 1.0, 1.0, 1.0, 0.9)],
                                     domain=(-600.0, 1400.0))
    assert np.array_equal(vr.build_lut(custom).rgba, golden_prep["lut_custom"])


def test_preintegrated_table_bit_exact_vs_reference(golden_prep):
    table = vr.build_preintegrated(vr.build_lut(vr.get_preset("soft-tissue")), 0.35, 0.5).rgba
    assert np.array_equal(table[::17, ::13], golden_prep["preint_soft_0.35_strided"])
    digest = np.frombuffer(hashlib.sha256(np.ascontiguousarray(table).tobytes()).digest(), np.uint8)
    assert np.array_equal(digest, golden_prep["preint_soft_0.35_sha256"])


# ---------------------------------------------------------------- blocks


def test_invalid_block_specs_raise_before_any_device_work():
    vol = vr.make_volume(np.zeros((16, 16, 16), dtype=np.int16), (1, 1, 1))
    for bs, ov in ((64, 64), (4, 1), (64, 0)):
        with pytest.raises(InvalidBlockSpec):
            vr.decompose(vol, bs, ov)


def test_axis_layout_matches_reference():
    from paper_2005_01442_b200.blocks import axis_layout

    o, e = axis_layout(512, 64, 61)
    assert len(o) == 9 and o[-1] == 488 and e[-1] == 24
    o, e = axis_layout(64, 64, 61)
    assert list(o) == [0] and list(e) == [64]
    covered = np.zeros(512, dtype=int)
    for a, b in zip(*axis_layout(512, 64, 61)):
        covered[a:a + b] += 1
    assert covered.min() >= 1


def test_volume_contract():
    with pytest.raises(ValueError):
        vr.ScalarVolume(np.zeros((4, 4), dtype=np.int16), (1, 1, 1), (0, 0))
    with pytest.raises(ValueError):
        vr.ScalarVolume(np.zeros((4, 4, 1), dtype=np.int16), (1, 1, 1), (0, 0))
    v = vr.make_volume(np.arange(24, dtype=np.int16).reshape(2, 3, 4), (0.5, 1.0, 2.0))
    assert v.dims == (4, 3, 2) and v.value_range == (0, 23)
    assert v.extent_mm == (1.5, 2.0, 2.0)
    raw = vr.load_raw(v.voxel_bytes(), (4, 3, 2), (0.5, 1.0, 2.0))
    assert np.array_equal(raw.values, v.values)
    with pytest.raises(vr.SizeMismatch):
        vr.load_raw(b"\x00" * 10, (4, 3, 2), (1, 1, 1))
