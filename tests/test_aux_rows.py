"""SURVEY §8(f) rows beside the render path: device ingest (row 2) and image
metrics / convergence studies (row 4).

CPU tests pin the oracle (oracle/aux_ref.py) to the reference's goldens
(tests/golden/aux.npz, made by make_golden_aux.py) and check the host-side
validation; GPU tests run the CUDA paths (vr_volume_ingest, vr_image_sse,
vr_image_ssim) against the same goldens.
"""

from __future__ import annotations

import json
from dataclasses import dataclass

import numpy as np
import pytest

from conftest import GOLDEN
from oracle import aux_ref


@pytest.fixture(scope="module")
def aux():
    return json.loads((GOLDEN / "aux.json").read_text()), dict(np.load(GOLDEN / "aux.npz"))


@dataclass(frozen=True)
class Slice:  # the reference's SliceImage fields (dicom.py:73-90)
    rows: int
    cols: int
    pixel_spacing: tuple
    position: float
    rescale_slope: float
    rescale_intercept: float
    pixel_representation: int
    samples: np.ndarray


def series_slices(case, arrays):
    return [Slice(case["rows"], case["cols"], tuple(case["pixel_spacing"]), case["positions"][i],
                  case["slopes"][i], case["icpts"][i], case["reps"][i], arrays[f"{case['name']}__s{i}"])
            for i in range(case["nslices"])]


# ---------------------------------------------------------------- oracle (CPU)

def test_oracle_load_raw_matches_reference(aux):
    meta, arrays = aux
    for case in meta["raw"]:
        data = arrays[f"{case['name']}__in"].tobytes()
        values, clamp, vrange = aux_ref.load_raw(data, case["dims"], case["fmt"])
        np.testing.assert_array_equal(values, arrays[f"{case['name']}__values"])
        assert clamp == case["clamp_count"] and list(vrange) == case["value_range"]
        assert aux_ref.volume_id(values, case["dims"], case["spacing"]) == case["volume_id"]


def test_oracle_assemble_matches_reference(aux):
    meta, arrays = aux
    for case in meta["series"]:
        sl = series_slices(case, arrays)
        values, clamp, vrange, dz = aux_ref.assemble([s.samples for s in sl], [s.position for s in sl],
                                                     [s.rescale_slope for s in sl],
                                                     [s.rescale_intercept for s in sl])
        np.testing.assert_array_equal(values, arrays[f"{case['name']}__values"])
        assert clamp == case["clamp_count"] and list(vrange) == case["value_range"]
        assert dz == case["spacing"][2]


def test_oracle_metrics_match_reference(aux):
    meta, arrays = aux
    for case in meta["quality"]:
        a, b = arrays[f"img_{case['a']}"], arrays[f"img_{case['b']}"]
        assert aux_ref.psnr(a, b) == case["psnr"]
        assert aux_ref.ssim(a, b) == case["ssim"]


# ------------------------------------------------- host validation (no device)

def test_ingest_validation_errors():
    import paper_2005_01442_b200 as vr

    with pytest.raises(vr.SizeMismatch):
        vr.ingest_raw(b"\x00" * 10, (2, 2, 2), (1, 1, 1), "i16")
    with pytest.raises(ValueError):
        vr.ingest_raw(b"\x00" * 8, (2, 2, 2), (1, 1, 1), "f32")
    s = np.zeros((4, 5), dtype=np.int16)
    mk = lambda pos, rows=4, sp=(1.0, 1.0): Slice(rows, 5, sp, pos, 1.0, 0.0, 1, s if rows == 4 else s[:3])  # noqa: E731
    with pytest.raises(vr.InconsistentGeometry):
        vr.assemble_volume_device([mk(0.0)])
    with pytest.raises(vr.InconsistentGeometry):
        vr.assemble_volume_device([mk(0.0), mk(1.0, rows=3)])
    with pytest.raises(vr.InconsistentGeometry):
        vr.assemble_volume_device([mk(0.0), mk(1.0, sp=(1.0, 0.5))])
    with pytest.raises(vr.DuplicatePosition):
        vr.assemble_volume_device([mk(0.0), mk(1.0), mk(1.0)])
    with pytest.raises(vr.NonUniformSpacing):
        vr.assemble_volume_device([mk(0.0), mk(1.0), mk(2.5)])
    assert vr.InconsistentGeometry("x").code == "InconsistentGeometry"


def test_metric_shape_errors():
    import paper_2005_01442_b200 as vr

    a = np.zeros((20, 20, 4), np.uint8)
    with pytest.raises(vr.DimensionMismatch, match="expected"):
        vr.psnr(a, np.zeros((20, 20), np.uint8))
    with pytest.raises(vr.DimensionMismatch, match="differ"):
        vr.psnr(a, np.zeros((20, 21, 4), np.uint8))
    with pytest.raises(vr.DimensionMismatch, match="at least 11x11"):
        vr.ssim(np.zeros((10, 20, 4), np.uint8), np.zeros((10, 20, 3), np.uint8))


# ------------------------------------------------------------------ GPU paths

@pytest.mark.gpu
def test_ingest_raw_on_device_matches_reference(aux):
    import paper_2005_01442_b200 as vr

    meta, arrays = aux
    for case in meta["raw"]:
        dv = vr.ingest_raw(arrays[f"{case['name']}__in"].tobytes(), case["dims"], case["spacing"], case["fmt"])
        np.testing.assert_array_equal(dv.download(), arrays[f"{case['name']}__values"])
        assert dv.clamp_count == case["clamp_count"]
        assert list(dv.value_range) == case["value_range"]
        assert dv.dims == tuple(case["dims"]) and dv.spacing == tuple(case["spacing"])


@pytest.mark.gpu
def test_assemble_on_device_matches_reference(aux):
    import paper_2005_01442_b200 as vr

    meta, arrays = aux
    for case in meta["series"]:
        dv = vr.assemble_volume_device(series_slices(case, arrays))
        np.testing.assert_array_equal(dv.download(), arrays[f"{case['name']}__values"])
        assert dv.clamp_count == case["clamp_count"], case["name"]
        assert list(dv.value_range) == case["value_range"]
        assert list(dv.spacing) == case["spacing"]


@pytest.mark.gpu
def test_ingested_volume_renders_like_an_uploaded_one():
    import paper_2005_01442_b200 as vr

    vals = vr.generate_phantom("torso", (40, 36, 32)).values
    dv = vr.ingest_raw(vals.astype("<i2").tobytes(), (40, 36, 32), (1.0, 1.0, 1.0), "i16")
    up = vr.DeviceVolume.upload(vals, (1.0, 1.0, 1.0))
    cam = vr.Camera(position=(120.0, 17.5, 15.5), look_at=(19.5, 17.5, 15.5), width=32, height=24)
    tf, st = vr.get_preset("bone"), vr.RenderSettings(interpolation="tricubic", use_blocks=True, block_size=16)
    frames = []
    for v in (dv, up):
        r = vr.Renderer(v, cam, tf, st)
        r.render_async()
        frames.append(r.pixels.cpu().numpy())
    np.testing.assert_array_equal(frames[0], frames[1])


@pytest.mark.gpu
def test_device_volume_cache_reads_a_store_directory(tmp_path):
    import paper_2005_01442_b200 as vr

    vals = vr.generate_phantom("sphere", (24, 20, 16)).values
    vol = vr.make_volume(vals, (0.5, 0.5, 1.0))
    vid = vr.volume_id(vol)
    d = tmp_path / vid
    d.mkdir()
    (d / "data.raw").write_bytes(vals.astype("<i2").tobytes())
    (d / "manifest.json").write_text(json.dumps({"id": vid, "dims": [24, 20, 16], "spacing": [0.5, 0.5, 1.0],
                                                 "value_range": list(vol.value_range), "source": "phantom",
                                                 "created_at": "2026-01-01T00:00:00+00:00"}))
    cache = vr.DeviceVolumeCache(tmp_path, capacity_bytes=1 << 30)
    dv = cache.get(vid)
    np.testing.assert_array_equal(dv.download(), vals)
    assert cache.get(vid) is dv and cache.hits == 1 and cache.misses == 1
    with pytest.raises(vr.UnknownVolume):
        cache.get("v-0000000000000000")
    other = vr.make_volume(vals[::-1].copy(), (1.0, 1.0, 1.0))
    assert cache.put(other) == vr.volume_id(other) and len(cache) == 2
    small = vr.DeviceVolumeCache(tmp_path, capacity_bytes=1)  # evicts down to the newest volume
    small.get(vid)
    small.put(other)
    assert len(small) == 1 and vr.volume_id(other) in small


@pytest.mark.gpu
def test_metrics_on_device_match_reference(aux):
    import torch

    import paper_2005_01442_b200 as vr

    meta, arrays = aux
    for case in meta["quality"]:
        a, b = arrays[f"img_{case['a']}"], arrays[f"img_{case['b']}"]
        assert vr.psnr(a, b) == case["psnr"]  # exact: integer squared error
        assert abs(vr.ssim(a, b) - case["ssim"]) <= 1e-12
        # device-resident inputs and RGB (3-channel) images take the same path
        ta, tb = torch.from_numpy(a).cuda(), torch.from_numpy(np.ascontiguousarray(b[..., :3])).cuda()
        assert vr.psnr(ta, tb) == case["psnr"]
        assert abs(vr.ssim(ta, tb) - case["ssim"]) <= 1e-12


@pytest.mark.gpu
def test_convergence_study_matches_reference(aux):
    import paper_2005_01442_b200 as vr

    study = aux[0]["convergence"]
    nx, ny, nz = study["dims"]
    vol = vr.generate_phantom("torso", (nx, ny, nz))
    ext = (nx - 1.0, ny - 1.0, nz - 1.0)
    cx, cy, cz = (0.5 * e for e in ext)
    d = 2.2 * max(ext)
    cam = vr.Camera(position=(cx + d, cy, cz), look_at=(cx, cy, cz), **study["camera"])
    rec = vr.convergence_study(vol, cam, vr.get_preset(study["tf"]), vr.RenderSettings(**study["settings"]),
                               study["steps"])
    assert [r["step"] for r in rec] == [r["step"] for r in study["records"]]
    for got, want in zip(rec, study["records"]):
        assert got["psnr_db"] == want["psnr_db"]
        assert abs(got["ssim"] - want["ssim"]) <= 1e-12


# ------------------------------------------------ service path (§8(f) row 3)

def test_request_validation_errors():
    from paper_2005_01442_b200 import errors, service

    with pytest.raises(errors.InvalidSettings, match="camera"):
        service.prepare_render(None, {"transfer": "bone"})
    with pytest.raises(errors.InvalidSettings, match="camera:"):
        service.prepare_render(None, {"camera": {"position": [0, 0, 1]}})
    with pytest.raises(errors.InvalidSettings, match="transfer:"):
        service.prepare_render(None, {"camera": {"position": [1, 0, 0], "look_at": [0, 0, 0], "width": 4,
                                                 "height": 4}, "transfer": "no-such-preset"})
    assert service.status_for(errors.UnknownVolume("x")) == 404
    assert service.status_for(errors.InvalidSettings("x")) == 422
    assert service.status_for(errors.SizeMismatch("x")) == 400


def test_ppm_encoding():
    from paper_2005_01442_b200 import imageio

    px = np.arange(2 * 3 * 4, dtype=np.uint8).reshape(2, 3, 4)
    ppm = imageio.encode_ppm(px)
    assert ppm.startswith(b"P6\n3 2\n255\n") and ppm[11:] == px[..., :3].tobytes()
    np.testing.assert_array_equal(imageio.decode_png(imageio.encode_png(px)), px)


@pytest.mark.gpu
def test_render_request_bytes_match_reference(aux):
    import paper_2005_01442_b200 as vr
    from paper_2005_01442_b200 import service

    meta, arrays = aux
    svc = meta["service"]
    vol = vr.generate_phantom("torso", tuple(svc["dims"]))
    for case in svc["cases"]:
        png, stats = service.render_request(vol, case["payload"])
        assert png == arrays[f"svc_{case['name']}"].tobytes(), case["name"]
        assert {k: v for k, v in stats.items() if k != "wall_time_s"} == case["stats"]
        assert json.loads(service.stats_header(stats)[service.STATS_HEADER]) == stats
