"""The drop-in boundary takes the REFERENCE's own objects.

The reference's callers build voxelray types and call
``render(volume, camera, tf, settings)`` (service.py:68-88 prepare_render,
store.py:131-143 returns reference ScalarVolumes, quality.py:98-101).  The
stand-ins below carry exactly the attributes of those classes and nothing of
ours: ScalarVolume (volume.py:23-71), Camera (render.py:56-95),
TransferFunction (transfer.py:28-62), RenderSettings (render.py:159-181),
BlockGrid (blocks.py:43-97).  render() must accept them unchanged and give
the same image and stats as with our own types.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np
import pytest

from oracle import oracle as O


@dataclass(frozen=True)
class RefScalarVolume:  # volume.py:23-55
    values: np.ndarray
    spacing: tuple
    value_range: tuple
    clamp_count: int = 0


@dataclass(frozen=True)
class RefCamera:  # render.py:56-95 (attributes and basis() only)
    position: tuple
    look_at: tuple
    up: tuple = (0.0, 0.0, 1.0)
    vertical_fov_deg: float = 30.0
    width: int = 256
    height: int = 256

    def basis(self):
        fwd = np.subtract(self.look_at, self.position, dtype=np.float64)
        fwd /= np.linalg.norm(fwd)
        right = np.cross(fwd, np.asarray(self.up, dtype=np.float64))
        right /= np.linalg.norm(right)
        return fwd, right, np.cross(right, fwd)


@dataclass(frozen=True)
class RefTransfer:  # transfer.py:28-62
    values: np.ndarray
    rgba: np.ndarray
    domain: tuple

    def evaluate(self, scalars):
        s = np.asarray(scalars, dtype=np.float64)
        return np.stack([np.interp(s, self.values, self.rgba[:, c]) for c in range(4)], axis=-1)


@dataclass(frozen=True)
class RefSettings:  # render.py:159-181
    step: float | None = None
    interpolation: str = "trilinear"
    classification: str = "post"
    mode: str = "dvr"
    isovalue: float | None = None
    lighting: bool = True
    early_termination_alpha: float = 0.99
    use_blocks: bool = False
    block_size: int = 64
    overlap: int = 3
    background: tuple = (0.0, 0.0, 0.0, 1.0)
    ambient: float = 0.1
    diffuse: float = 0.7
    specular: float = 0.2
    shininess: float = 32.0

    def validate(self):
        pass


@dataclass(frozen=True)
class RefBlockGrid:  # blocks.py:43-57 (the fields render() reads)
    volume: RefScalarVolume
    block_size: int
    overlap: int
    vmin: np.ndarray = field(default=None)
    vmax: np.ndarray = field(default=None)


def _ref_scene(dims=(40, 36, 32), size=(48, 40)):
    vals = O.phantom("torso", dims)
    vals.flags.writeable = False
    vol = RefScalarVolume(vals, (1.0, 1.0, 1.0), (int(vals.min()), int(vals.max())))
    ext = ((dims[0] - 1) * 1.0, (dims[1] - 1) * 1.0, (dims[2] - 1) * 1.0)
    c = tuple(0.5 * e for e in ext)
    cam = RefCamera(position=(c[0] + 2.2 * max(ext), c[1] + 3.0, c[2] - 2.0), look_at=c,
                    width=size[0], height=size[1])
    v, rgba, dom = O.preset_arrays("bone")
    tf = RefTransfer(v, rgba, dom)
    return vol, cam, tf


def test_adapters_build_equivalent_objects():
    import paper_2005_01442_b200 as vr
    from paper_2005_01442_b200.render import as_camera, as_settings, as_transfer, as_volume

    vol, cam, tf = _ref_scene()
    ours = as_volume(vol)
    assert isinstance(ours, vr.ScalarVolume)
    assert ours.values is vol.values or np.shares_memory(ours.values, vol.values)  # no copy
    assert ours.spacing == vol.spacing and ours.value_range == vol.value_range
    assert as_volume(vol) is ours  # cached per source object
    c = as_camera(cam)
    assert isinstance(c, vr.Camera)
    for a, b in zip(c.basis(), cam.basis()):
        np.testing.assert_array_equal(a, b)
    half_h = math.tan(math.radians(cam.vertical_fov_deg) / 2.0)  # render.py:128-129
    assert c.half_extents() == (half_h * cam.width / cam.height, half_h)
    s = as_settings(RefSettings(interpolation="tricubic", use_blocks=True, background=[0.2, 0.4, 0.6, 1.0]))
    assert isinstance(s, vr.RenderSettings) and s.interpolation == "tricubic" and s.use_blocks
    assert s.background == (0.2, 0.4, 0.6, 1.0)
    t = as_transfer(tf)
    np.testing.assert_array_equal(vr.build_lut(t).rgba, vr.build_lut(vr.get_preset("bone")).rgba)
    with pytest.raises(vr.InvalidSettings):
        as_settings(RefSettings(interpolation="nearest")).validate()


@pytest.mark.gpu
@pytest.mark.parametrize("blocks", [False, True])
def test_render_takes_reference_objects(blocks):
    import paper_2005_01442_b200 as vr

    vol, cam, tf = _ref_scene()
    st = RefSettings(interpolation="tricubic", use_blocks=blocks, block_size=16)
    img = vr.render(vol, cam, tf, st, return_premultiplied=True)
    ref = O.render(vol.values, vol.spacing, cam, tf.values, tf.rgba, tf.domain, st)
    np.testing.assert_array_equal(img.premultiplied, ref.out)
    np.testing.assert_array_equal(img.pixels, ref.pixels)
    assert img.stats.samples_taken == ref.samples_taken
    assert img.stats.samples_skipped == ref.samples_skipped
    # and identical to the same render through our own types
    ours = vr.render(vr.make_volume(np.array(vol.values), vol.spacing), vr.Camera(
        position=cam.position, look_at=cam.look_at, width=cam.width, height=cam.height), vr.get_preset("bone"),
        vr.RenderSettings(interpolation="tricubic", use_blocks=blocks, block_size=16))
    np.testing.assert_array_equal(img.pixels, ours.pixels)
    assert img.stats == type(img.stats)(**{**ours.stats.__dict__, "wall_time_s": img.stats.wall_time_s})


@pytest.mark.gpu
def test_render_takes_reference_block_grid():
    import paper_2005_01442_b200 as vr

    vol, cam, tf = _ref_scene()
    grid = RefBlockGrid(vol, 16, 3)
    img = vr.render(grid, cam, tf, RefSettings(interpolation="tricubic"))
    ref = O.render(vol.values, vol.spacing, cam, tf.values, tf.rgba, tf.domain,
                   RefSettings(interpolation="tricubic", use_blocks=True, block_size=16, overlap=3))
    np.testing.assert_array_equal(img.pixels, ref.pixels)
    assert img.stats.samples_taken == ref.samples_taken
    assert img.stats.blocks_visited == ref.blocks_visited


@pytest.mark.gpu
def test_prepare_render_sequence_with_only_render_swapped():
    """service.py:68-88 with reference objects throughout, render() ours:
    camera from the request dict, TF preset, settings from the dict."""
    import paper_2005_01442_b200 as vr

    vol, _, _ = _ref_scene((48, 40, 36))
    payload = {"camera": {"position": [110.0, 20.0, 18.0], "look_at": [23.5, 19.5, 17.5],
                          "up": [0, 0, 1], "vertical_fov_deg": 30.0, "width": 40, "height": 32},
               "transfer": "bone", "settings": {"interpolation": "tricubic", "use_blocks": True,
                                                "block_size": 16, "classification": "post"}}
    d = payload["camera"]
    camera = RefCamera(position=tuple(d["position"]), look_at=tuple(d["look_at"]), up=tuple(d["up"]),
                       vertical_fov_deg=float(d["vertical_fov_deg"]), width=int(d["width"]),
                       height=int(d["height"]))  # camera_from_dict, render.py:98-106
    v, rgba, dom = O.preset_arrays(payload["transfer"])
    tf = RefTransfer(v, rgba, dom)  # resolve_transfer -> get_preset
    settings = RefSettings(**payload["settings"])  # settings_from_dict
    img = vr.render(vol, camera, tf, settings)
    ref = O.render(vol.values, vol.spacing, camera, v, rgba, dom, settings)
    np.testing.assert_array_equal(img.pixels, ref.pixels)
    assert img.stats.samples_taken == ref.samples_taken
    from paper_2005_01442_b200.imageio import encode_png

    png = encode_png(img)  # the service's next step (imageio.py:14-19)
    assert png[:8] == b"\x89PNG\r\n\x1a\n"
