"""Golden vectors for the §8(f) rows next to the render path, from the UNMODIFIED
reference (run in the build container, never on the GPU box):

    python tests/golden/make_golden_aux.py

* ingest: ``volume.load_raw`` for u8 / i16 / u16 payloads, ``dicom.assemble_volume``
  for shuffled series with per-slice rescale (incl. clamping, half-way rounding
  and a mixed signed/unsigned series), ``store.volume_id``;
* quality: ``quality.psnr`` / ``quality.ssim`` on image pairs and
  ``quality.convergence_study`` on a small phantom render;
* service: ``service.render_request`` (PNG bytes + stats dict) for request
  bodies covering the render modes, on a small phantom.

Output: tests/golden/aux.npz + aux.json.
"""

from __future__ import annotations

import json
import os
import sys
from pathlib import Path

os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/vr_numba_cache")
sys.dont_write_bytecode = True
sys.pycache_prefix = "/tmp/vr_pycache"
REF = "/root/reference/pkg/src"
sys.path.insert(0, REF)

import numpy as np  # noqa: E402

from voxelray import quality  # noqa: E402
from voxelray.dicom import SliceImage, assemble_volume  # noqa: E402
from voxelray.service import render_request  # noqa: E402
from voxelray.phantoms import generate_phantom  # noqa: E402
from voxelray.render import Camera, RenderSettings  # noqa: E402
from voxelray.store import volume_id  # noqa: E402
from voxelray.transfer import get_preset  # noqa: E402
from voxelray.volume import load_raw  # noqa: E402

OUT = Path(__file__).resolve().parent


def raw_cases(rng):
    dims = (20, 18, 16)
    n = dims[0] * dims[1] * dims[2]
    payloads = {
        "u8": rng.integers(0, 256, n, dtype=np.uint8).tobytes(),
        "i16": rng.integers(-32768, 32768, n, dtype=np.int64).astype("<i2").tobytes(),
        "u16": rng.integers(0, 65536, n, dtype=np.int64).astype("<u2").tobytes(),
    }
    arrays, meta = {}, []
    for fmt, data in payloads.items():
        v = load_raw(data, dims, (0.7, 0.8, 1.5), fmt)
        arrays[f"raw_{fmt}__in"] = np.frombuffer(data, dtype=np.uint8)
        arrays[f"raw_{fmt}__values"] = v.values
        meta.append(dict(name=f"raw_{fmt}", fmt=fmt, dims=dims, spacing=[0.7, 0.8, 1.5],
                         value_range=list(v.value_range), clamp_count=v.clamp_count,
                         volume_id=volume_id(v)))
    return arrays, meta


def series_cases(rng):
    rows, cols, nz = 12, 10, 9
    arrays, meta = {}, []
    specs = {
        # signed samples, integer slope / intercept
        "series_i16": dict(kind="i2", lo=-2000, hi=3000, slopes=[1.0] * nz, icpts=[-1024.0] * nz),
        # unsigned samples, slope 2 pushes many values past int16 -> clamped
        "series_u16_clamp": dict(kind="u2", lo=0, hi=65536, slopes=[2.0] * nz, icpts=[-1024.0] * nz),
        # slope 0.5: half-way values exercise rint's round-half-even; per-slice intercepts
        "series_half": dict(kind="u2", lo=0, hi=5000, slopes=[0.5] * nz,
                            icpts=[-1000.0 + 0.5 * k for k in range(nz)]),
        # a series mixing signed and unsigned slices
        "series_mixed": dict(kind="mix", lo=0, hi=40000, slopes=[1.0 + 0.25 * (k % 3) for k in range(nz)],
                             icpts=[-1024.0] * nz),
    }
    for name, sp in specs.items():
        positions = [5.0 + 1.25 * k for k in range(nz)]
        order = rng.permutation(nz)
        slices = []
        for k in order:
            kind = sp["kind"] if sp["kind"] != "mix" else ("<i2" if k % 2 else "<u2")
            if kind in ("i2", "<i2"):
                s = rng.integers(max(sp["lo"], -32768), min(sp["hi"], 32768), (rows, cols)).astype("<i2")
                rep = 1
            else:
                s = rng.integers(sp["lo"], sp["hi"], (rows, cols)).astype("<u2")
                rep = 0
            slices.append(SliceImage(rows=rows, cols=cols, pixel_spacing=(0.6, 0.55), position=positions[k],
                                     rescale_slope=sp["slopes"][k], rescale_intercept=sp["icpts"][k],
                                     pixel_representation=rep, samples=s, sop_instance_uid=f"{name}.{k}"))
        v = assemble_volume(slices)
        for i, s in enumerate(slices):
            arrays[f"{name}__s{i}"] = s.samples
        arrays[f"{name}__values"] = v.values
        meta.append(dict(name=name, rows=rows, cols=cols, nslices=nz,
                         positions=[s.position for s in slices], slopes=[s.rescale_slope for s in slices],
                         icpts=[s.rescale_intercept for s in slices], reps=[s.pixel_representation for s in slices],
                         pixel_spacing=[0.6, 0.55], spacing=list(v.spacing), value_range=list(v.value_range),
                         clamp_count=v.clamp_count))
    return arrays, meta


def quality_cases(rng):
    arrays, meta = {}, []
    a = rng.integers(0, 256, (40, 36, 4), dtype=np.uint8)
    b = a.copy()
    b[5:20, 3:30, :3] = np.clip(b[5:20, 3:30, :3].astype(int) + rng.integers(-20, 21, (15, 27, 3)), 0, 255)
    c = rng.integers(0, 256, (40, 36, 4), dtype=np.uint8)
    arrays["img_a"], arrays["img_b"], arrays["img_c"] = a, b, c
    for x, y in (("a", "b"), ("a", "c"), ("a", "a"), ("b", "c")):
        ia, ib = arrays[f"img_{x}"], arrays[f"img_{y}"]
        meta.append(dict(name=f"{x}{y}", a=x, b=y, psnr=quality.psnr(ia, ib), ssim=quality.ssim(ia, ib)))
    # convergence study on a small render (the reference's own render path)
    vol = generate_phantom("torso", (40, 40, 40))
    nx, ny, nz = vol.dims
    ext = ((nx - 1.0), (ny - 1.0), (nz - 1.0))
    cx, cy, cz = (0.5 * e for e in ext)
    d = 2.2 * max(ext)
    cam = Camera(position=(cx + d, cy, cz), look_at=(cx, cy, cz), width=48, height=40)
    rec = quality.convergence_study(vol, cam, get_preset("bone"), RenderSettings(interpolation="tricubic"),
                                    [0.5, 1.0, 2.0])
    study = dict(dims=[40, 40, 40], camera=dict(width=48, height=40), tf="bone",
                 settings=dict(interpolation="tricubic"), steps=[0.5, 1.0, 2.0], records=rec)
    return arrays, meta, study


PAYLOADS = {
    "bone_tricubic": {"camera": {"position": [100.0, 18.0, 16.0], "look_at": [18.0, 17.0, 15.0], "width": 40,
                                 "height": 32}, "transfer": "bone",
                      "settings": {"interpolation": "tricubic", "use_blocks": True, "block_size": 16}},
    "soft_preint": {"camera": {"position": [18.0, 100.0, 20.0], "look_at": [18.0, 17.0, 15.0], "width": 36,
                               "height": 36}, "transfer": "soft-tissue",
                    "settings": {"classification": "preintegrated", "lighting": False}},
    "iso": {"camera": {"position": [100.0, 18.0, 16.0], "look_at": [18.0, 17.0, 15.0], "width": 32, "height": 30},
            "settings": {"mode": "isosurface", "isovalue": 600}},
}


def service_cases():
    vol = generate_phantom("torso", (36, 34, 30))
    arrays, meta = {}, []
    for name, body in PAYLOADS.items():
        png, stats = render_request(vol, body)
        arrays[f"svc_{name}"] = np.frombuffer(png, dtype=np.uint8)
        stats = {k: v for k, v in stats.items() if k != "wall_time_s"}
        meta.append(dict(name=name, payload=body, stats=stats))
    return arrays, dict(dims=[36, 34, 30], cases=meta)


def main():
    rng = np.random.default_rng(20260417)
    arrays, meta = {}, {}
    a, m = raw_cases(rng)
    arrays.update(a)
    meta["raw"] = m
    a, m = series_cases(rng)
    arrays.update(a)
    meta["series"] = m
    a, m, study = quality_cases(rng)
    arrays.update(a)
    meta["quality"] = m
    meta["convergence"] = study
    a, m = service_cases()
    arrays.update(a)
    meta["service"] = m
    np.savez_compressed(OUT / "aux.npz", **arrays)
    (OUT / "aux.json").write_text(json.dumps(meta, indent=1))
    print(json.dumps(meta["quality"], indent=1), json.dumps(study["records"], indent=1))


if __name__ == "__main__":
    main()
