"""Generate golden vectors from the UNMODIFIED reference (run in the build container).

    python tests/golden/make_golden.py

Imports voxelray from /root/reference/pkg/src (read-only; bytecode and numba
caches are redirected to /tmp) and records, for a matrix of render cases, the
float64 premultiplied ``out`` buffer, depth, per-pixel taken/skipped counts and
blocks_hit that ``_kernels.march`` filled, plus the uint8 image and RenderStats
that ``render()`` returned.  The march outputs are captured by wrapping the
reference's own ``_kernels.march`` (the wrapper calls it unchanged), so every
case goes through the reference's stock ``render()`` code path.  Orthographic
cases replace ``render._ray_grid`` by parallel rays; everything
else in ``render()`` still runs as shipped.

Also records block prep (decompose / with_visibility), LUTs, point sampling and
phantom hashes.  Output: tests/golden/*.npz + cases.json.  The GPU box never
runs this script (no /root/reference there); it only reads the fixtures.
"""

from __future__ import annotations

import hashlib
import json
import math
import os
import sys
from pathlib import Path

os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/vr_numba_cache")
sys.dont_write_bytecode = True
sys.pycache_prefix = "/tmp/vr_pycache"
REF = "/root/reference/pkg/src"
sys.path.insert(0, REF)

import numpy as np  # noqa: E402

import voxelray  # noqa: E402
from voxelray import _kernels  # noqa: E402
from voxelray.blocks import decompose, with_visibility  # noqa: E402
from voxelray.phantoms import generate_phantom  # noqa: E402
from voxelray.render import Camera, RenderSettings  # noqa: E402
from voxelray.sampling import gradient, sample  # noqa: E402
from voxelray.transfer import build_lut, build_preintegrated, get_preset, transfer_from_points  # noqa: E402

render_mod = sys.modules["voxelray.render"]
OUT = Path(__file__).resolve().parent

_captured = {}
_real_march = _kernels.march


def _march_spy(*args):
    _real_march(*args)
    out, depth, taken, skipped, blocks_hit = args[-5:]
    _captured.update(out=out.copy(), depth=depth.copy(), taken=taken.copy(),
                     skipped=skipped.copy(), blocks_hit=blocks_hit.copy())


_kernels.march = _march_spy


def centered_camera(extent, size, distance_factor=2.2, height=None):
    """tests/conftest.py:34-43 geometry."""
    cx, cy, cz = (0.5 * e for e in extent)
    d = distance_factor * max(extent)
    return dict(position=[cx + d, cy, cz], look_at=[cx, cy, cz], up=[0.0, 0.0, 1.0],
                vertical_fov_deg=30.0, width=size, height=height or size)


def tf_spec(name):
    if name == "custom":
        return dict(points=[[-500.0, 0, 0, 0, 0.0], [300.0, 0.9, 0.5, 0.2, 0.0],
                            [700.0, 1.0, 0.8, 0.6, 0.6], [1500.0, 1.0, 1.0, 1.0, 0.9]],
                    domain=[-600.0, 1400.0])
    if name == "clear":
        return dict(points=[[-2000.0, 0, 0, 0, 0.0], [2000.0, 0, 0, 0, 0.0]], domain=None)
    if name == "red":
        return dict(points=[[-1000.0, 1, 0, 0, 1.0], [3000.0, 1, 0, 0, 1.0]],
                    domain=[-1000.0, 3000.0])
    return dict(preset=name)


def make_tf(spec):
    if "preset" in spec:
        return get_preset(spec["preset"])
    return transfer_from_points([tuple(p) for p in spec["points"]], domain=spec["domain"])


def ortho_ray_grid(half_h):
    def ray_grid(camera):
        fwd, right, true_up = camera.basis()
        half_w = half_h * camera.width / camera.height
        px = np.arange(camera.width, dtype=np.float64)
        py = np.arange(camera.height, dtype=np.float64)
        u = (2.0 * (px + 0.5) / camera.width - 1.0) * half_w
        v = (1.0 - 2.0 * (py + 0.5) / camera.height) * half_h
        pos = np.asarray(camera.position, dtype=np.float64)
        origins = (pos[None, None, :] + u[None, :, None] * right[None, None, :]
                   + v[:, None, None] * true_up[None, None, :]).reshape(-1, 3)
        dirs = np.broadcast_to(fwd, origins.shape).copy()
        return np.ascontiguousarray(origins), np.ascontiguousarray(dirs)
    return ray_grid


def case_list():
    cases = []

    def add(name, phantom, dims, spacing=(1.0, 1.0, 1.0), camera=None, tf="bone",
            projection="pinhole", ortho_half_h=None, **settings):
        cases.append(dict(name=name, phantom=phantom, dims=list(dims), spacing=list(spacing),
                          camera=camera, tf=tf_spec(tf), projection=projection,
                          ortho_half_h=ortho_half_h, settings=settings))

    t48 = (47.0, 47.0, 47.0)
    add("torso48_bone_cubic_mono", "torso", (48, 48, 48), camera=centered_camera(t48, 40),
        interpolation="tricubic")
    add("torso48_bone_linear_mono", "torso", (48, 48, 48), camera=centered_camera(t48, 40))
    add("torso48_bone_cubic_blocks16", "torso", (48, 48, 48), camera=centered_camera(t48, 40),
        interpolation="tricubic", use_blocks=True, block_size=16, overlap=3)
    add("torso48_bone_linear_blocks16", "torso", (48, 48, 48), camera=centered_camera(t48, 40),
        use_blocks=True, block_size=16, overlap=3)
    add("torso48_soft_cubic_mono_light", "torso", (48, 48, 48), camera=centered_camera(t48, 40),
        tf="soft-tissue", interpolation="tricubic")
    add("torso48_soft_linear_blocks16_nolight", "torso", (48, 48, 48),
        camera=centered_camera(t48, 40), tf="soft-tissue", use_blocks=True, block_size=16,
        overlap=3, lighting=False)
    add("torso48_soft_cubic_blocks16_light", "torso", (48, 48, 48),
        camera=centered_camera(t48, 40), tf="soft-tissue", interpolation="tricubic",
        use_blocks=True, block_size=16, overlap=3)
    add("torso48_gray_stress", "torso", (48, 48, 48), camera=centered_camera(t48, 40),
        tf="grayscale", interpolation="tricubic", lighting=False, early_termination_alpha=1.0)
    aniso_ext = (39 * 0.8, 35 * 0.7, 31 * 1.5)
    cam = dict(position=[aniso_ext[0] * 0.5 - 40.0, aniso_ext[1] * 0.5 + 70.0, aniso_ext[2] * 0.5 + 25.0],
               look_at=[aniso_ext[0] * 0.5, aniso_ext[1] * 0.5, aniso_ext[2] * 0.5],
               up=[0.0, 0.3, 1.0], vertical_fov_deg=41.0, width=36, height=28)
    add("aniso_oblique_cubic_blocks12", "torso", (40, 36, 32), spacing=(0.8, 0.7, 1.5),
        camera=cam, interpolation="tricubic", use_blocks=True, block_size=12, overlap=3)
    add("aniso_oblique_linear_mono_soft", "torso", (40, 36, 32), spacing=(0.8, 0.7, 1.5),
        camera=cam, tf="soft-tissue")
    add("torso48_custom_tf_linear_blocks16", "torso", (48, 48, 48),
        camera=centered_camera(t48, 40), tf="custom", use_blocks=True, block_size=16, overlap=3)
    add("torso48_step035_cubic", "torso", (48, 48, 48), camera=centered_camera(t48, 32),
        interpolation="tricubic", step=0.35)
    add("torso48_step035_blocks_soft", "torso", (48, 48, 48), camera=centered_camera(t48, 32),
        tf="soft-tissue", step=0.35, use_blocks=True, block_size=16, overlap=3)
    add("torso48_bg_blocks", "torso", (48, 48, 48), camera=centered_camera(t48, 32),
        use_blocks=True, block_size=16, overlap=3, background=[0.2, 0.4, 0.6, 0.7])
    add("torso48_ortho_cubic_mono", "torso", (48, 48, 48), camera=centered_camera(t48, 40),
        projection="orthographic", ortho_half_h=24.5, interpolation="tricubic")
    add("torso48_ortho_cubic_blocks16", "torso", (48, 48, 48), camera=centered_camera(t48, 40),
        projection="orthographic", ortho_half_h=24.5, interpolation="tricubic",
        use_blocks=True, block_size=16, overlap=3)
    add("torso80_bone_cubic_blocks64", "torso", (80, 80, 80), camera=centered_camera((79.0,) * 3, 40),
        interpolation="tricubic", use_blocks=True)
    add("torso48_overlap1_linear", "torso", (48, 48, 48), camera=centered_camera(t48, 32),
        use_blocks=True, block_size=10, overlap=1)
    add("torso48_overlap2_cubic", "torso", (48, 48, 48), camera=centered_camera(t48, 32),
        interpolation="tricubic", use_blocks=True, block_size=12, overlap=2)
    add("torso48_clear_blocks", "torso", (48, 48, 48), camera=centered_camera(t48, 24),
        tf="clear", use_blocks=True, background=[0.2, 0.4, 0.6, 1.0])
    add("torso48_miss", "torso", (48, 48, 48),
        camera=dict(position=[300.0, 32.0, 32.0], look_at=[600.0, 32.0, 32.0], up=[0, 0, 1.0],
                    vertical_fov_deg=30.0, width=8, height=8))
    add("shell32_soft_et", "shell", (32, 32, 32), camera=centered_camera((31.0,) * 3, 32),
        tf="soft-tissue")
    add("sphere32_iso_cubic", "sphere", (32, 32, 32), camera=centered_camera((31.0,) * 3, 32),
        tf="red", mode="isosurface", isovalue=0.0, interpolation="tricubic")
    add("sphere32_iso_linear_blocks", "sphere", (32, 32, 32), camera=centered_camera((31.0,) * 3, 32),
        tf="bone", mode="isosurface", isovalue=300.0, use_blocks=True, block_size=12, overlap=3)
    add("torso32_pre_linear_light", "torso", (32, 32, 32), camera=centered_camera((31.0,) * 3, 32),
        classification="pre")
    add("torso32_pre_cubic_blocks", "torso", (32, 32, 32), camera=centered_camera((31.0,) * 3, 32),
        classification="pre", interpolation="tricubic", use_blocks=True, block_size=12, overlap=3)
    add("torso32_preint_linear_blocks", "torso", (32, 32, 32),
        camera=centered_camera((31.0,) * 3, 32), tf="soft-tissue",
        classification="preintegrated", use_blocks=True, block_size=12, overlap=3)
    add("torso32_preint_cubic_mono_step", "torso", (32, 32, 32),
        camera=centered_camera((31.0,) * 3, 32), classification="preintegrated",
        interpolation="tricubic", step=0.4)
    return cases


def run_case(case):
    vol = generate_phantom(case["phantom"], tuple(case["dims"]), tuple(case["spacing"]))
    cam = Camera(position=tuple(case["camera"]["position"]), look_at=tuple(case["camera"]["look_at"]),
                 up=tuple(case["camera"]["up"]), vertical_fov_deg=case["camera"]["vertical_fov_deg"],
                 width=case["camera"]["width"], height=case["camera"]["height"])
    s = dict(case["settings"])
    if "background" in s:
        s["background"] = tuple(s["background"])
    settings = RenderSettings(**s)
    tf = make_tf(case["tf"])
    real_grid = render_mod._ray_grid
    if case["projection"] == "orthographic":
        render_mod._ray_grid = ortho_ray_grid(case["ortho_half_h"])
    try:
        _captured.clear()
        img = voxelray.render(vol, cam, tf, settings)
    finally:
        render_mod._ray_grid = real_grid
    st = img.stats
    return dict(
        out=_captured["out"], depth=_captured["depth"], taken=_captured["taken"].astype(np.int32),
        skipped=_captured["skipped"].astype(np.int32), blocks_hit=_captured["blocks_hit"],
        pixels=img.pixels,
        stats=np.array([st.rays, st.samples_taken, st.samples_skipped, st.blocks_total,
                        st.blocks_empty, st.blocks_visited], dtype=np.int64),
    )


def prep_goldens():
    res = {}
    for name, dims, bs, ov in (("torso64_16_3", (64, 64, 64), 16, 3),
                               ("torso96x80x64_64_3", (96, 80, 64), 64, 3),
                               ("torso48_10_1", (48, 48, 48), 10, 1)):
        vol = generate_phantom("torso", dims)
        grid = decompose(vol, bs, ov)
        res[f"{name}_vmin"] = grid.vmin
        res[f"{name}_vmax"] = grid.vmax
        for tfn in ("bone", "soft-tissue", "custom"):
            lut = build_lut(make_tf(tf_spec(tfn)))
            g = with_visibility(grid, lut)
            res[f"{name}_{tfn}_empty"] = g.empty
            res[f"{name}_{tfn}_lo"] = g.aabb_lo
            res[f"{name}_{tfn}_hi"] = g.aabb_hi
    for tfn in ("bone", "soft-tissue", "grayscale", "custom"):
        res[f"lut_{tfn}"] = build_lut(make_tf(tf_spec(tfn))).rgba
    table = build_preintegrated(build_lut(get_preset("soft-tissue")), 0.35, 0.5).rgba
    res["preint_soft_0.35_strided"] = table[::17, ::13]
    res["preint_soft_0.35_sha256"] = np.frombuffer(
        hashlib.sha256(np.ascontiguousarray(table).tobytes()).digest(), dtype=np.uint8)
    return res


def sampling_goldens():
    res = {}
    rng = np.random.default_rng(0)
    n = 16
    z, y, x = np.meshgrid(np.arange(n), np.arange(n), np.arange(n), indexing="ij")
    cub = voxelray.make_volume(np.asarray((x + 8.0) ** 3, dtype=np.int16), (1, 1, 1))
    torso = generate_phantom("torso", (24, 20, 16), (0.5, 1.0, 2.0))
    pts = np.concatenate([rng.uniform(-2.0, 17.0, size=(300, 3)),
                          np.stack(np.meshgrid(np.arange(4.0), np.arange(4.0), np.arange(4.0)), -1).reshape(-1, 3)])
    res["pts"] = pts
    for interp in ("trilinear", "tricubic"):
        res[f"cub_{interp}_sample"] = sample(cub, pts, interp)
        res[f"cub_{interp}_grad"] = gradient(cub, pts, interp)
        res[f"torso_{interp}_sample"] = sample(torso, pts, interp)
        res[f"torso_{interp}_grad"] = gradient(torso, pts, interp)
    return res


def phantom_hashes():
    out = {}
    for name, dims in (("torso", (48, 48, 48)), ("torso", (40, 36, 32)), ("torso", (64, 64, 64)),
                       ("torso", (96, 80, 64)), ("sphere", (32, 32, 32)), ("shell", (32, 32, 32)),
                       ("torso", (128, 128, 128)), ("sphere", (48, 40, 33)), ("shell", (20, 24, 28))):
        v = generate_phantom(name, dims)
        out[f"{name}_{dims[0]}x{dims[1]}x{dims[2]}"] = hashlib.sha256(v.voxel_bytes()).hexdigest()
    return out


def main():
    cases = case_list()
    arrays = {}
    for c in cases:
        r = run_case(c)
        for k, v in r.items():
            if k == "depth" and c["settings"].get("mode") != "isosurface":
                continue
            arrays[f"{c['name']}__{k}"] = v
        print(c["name"], r["stats"].tolist(), flush=True)
    np.savez_compressed(OUT / "renders.npz", **arrays)
    np.savez_compressed(OUT / "prep.npz", **prep_goldens())
    np.savez_compressed(OUT / "sampling.npz", **sampling_goldens())
    meta = dict(cases=cases, phantom_sha256=phantom_hashes(), reference=REF,
                numpy=np.__version__, numba=__import__("numba").__version__)
    (OUT / "cases.json").write_text(json.dumps(meta, indent=1))
    print("wrote", sorted(p.name for p in OUT.glob("*.npz")))


if __name__ == "__main__":
    main()
