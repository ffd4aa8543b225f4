"""Where the end-to-end render() time goes at a bench config (GPU box).

    python tools/e2e_profile.py [c3]
"""
import cProfile
import pstats
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2005_01442_b200 as vr  # noqa: E402


def main(config="c3"):
    cfg = bench.CONFIGS[config]
    dvol = vr.device_phantom("torso", cfg["dims"])
    host = vr.ScalarVolume(dvol.download(), (1.0, 1.0, 1.0), dvol.value_range)
    host._attach_device(dvol)
    nx, ny, nz = dvol.dims
    cam = bench.make_camera(vr, cfg, (nx - 1.0, ny - 1.0, nz - 1.0))
    tf = vr.get_preset(cfg["tf"])
    st = vr.RenderSettings(**cfg["settings"])
    for _ in range(5):
        vr.render(host, cam, tf, st)
    torch.cuda.synchronize()
    n = 50
    t0 = time.perf_counter()
    for _ in range(n):
        vr.render(host, cam, tf, st)
    print(f"render(): {1e3 * (time.perf_counter() - t0) / n:.3f} ms/frame")
    pr = cProfile.Profile()
    pr.enable()
    for _ in range(n):
        vr.render(host, cam, tf, st)
    pr.disable()
    pstats.Stats(pr).sort_stats("tottime").print_stats(12)
    r = vr.Renderer(dvol, cam, tf, st, time_kernel=True)
    for _ in range(3):
        r.render_async()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(n):
        r.render_async()
    torch.cuda.synchronize()
    print(f"Renderer.render_async (device only): {1e3 * (time.perf_counter() - t0) / n:.3f} ms/frame, "
          f"kernel {r.kernel_ms():.3f} ms")
    pix = np.empty((cam.height, cam.width, 4), np.uint8)
    pinned = torch.empty((cam.height, cam.width, 4), dtype=torch.uint8, pin_memory=True)
    for name, dst in (("pageable", torch.from_numpy(pix)), ("pinned", pinned)):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(n):
            dst.copy_(r.pixels, non_blocking=False)
        torch.cuda.synchronize()
        print(f"D2H 4 MiB {name}: {1e3 * (time.perf_counter() - t0) / n:.3f} ms")
    lut = build = time.perf_counter()
    for _ in range(n):
        vr.build_lut(tf)
    print(f"build_lut: {1e3 * (time.perf_counter() - build) / n:.3f} ms")
    del lut




def host_overhead(config="c3"):
    """render() wall time vs the bare vr_render_to_host call it makes."""
    import ctypes

    from paper_2005_01442_b200 import _lib
    from paper_2005_01442_b200.render import _lut_host_copy, _pinned_empty, _resolve, camera_struct

    cfg = bench.CONFIGS[config]
    dvol = vr.device_phantom("torso", cfg["dims"])
    host = vr.ScalarVolume(dvol.download(), (1.0, 1.0, 1.0), dvol.value_range)
    host._attach_device(dvol)
    nx, ny, nz = dvol.dims
    cam = bench.make_camera(vr, cfg, (nx - 1.0, ny - 1.0, nz - 1.0))
    tf, st = vr.get_preset(cfg["tf"]), vr.RenderSettings(**cfg["settings"])
    for _ in range(5):
        vr.render(host, cam, tf, st)
    res = _resolve(host.spacing, host.value_range, tf, st)
    dgrid = vr.blocks.device_grid(host, st.block_size, st.overlap, 0)
    c = camera_struct(cam)
    pixels = _pinned_empty((c.tile_h, c.tile_w, 4), np.uint8)
    totals = np.zeros(8, dtype=np.uint64)
    lut = _lut_host_copy(res.lut)
    L = _lib.load()
    n = 100

    def bare():
        _lib.check(L.vr_render_to_host(dvol.handle, dgrid.handle, ctypes.byref(c), ctypes.byref(res.params),
                                       _lib.ptr(lut), None, _lib.ptr(pixels), None, None, _lib.ptr(totals), None))

    for f, name in ((bare, "vr_render_to_host"), (lambda: vr.render(host, cam, tf, st), "render()")):
        for _ in range(5):
            f()
        t0 = time.perf_counter()
        for _ in range(n):
            f()
        print(f"{name}: {1e3 * (time.perf_counter() - t0) / n:.3f} ms")
    pr = cProfile.Profile()
    pr.enable()
    for _ in range(n):
        vr.render(host, cam, tf, st)
    pr.disable()
    pstats.Stats(pr).sort_stats("tottime").print_stats(15)


if __name__ == "__main__":
    if sys.argv[1:2] == ["host"]:
        host_overhead(*sys.argv[2:])
    else:
        main(*sys.argv[1:])
