"""Per-warp timeline of the persistent ray-cast kernel (needs a library built
with -DVR_DEBUG_TIMES):

    python paper_2005_01442_b200/_build.py build_variants/dbg.so VR_DEBUG_TIMES [VR_DEBUG_STATS]
    VR_LIB=build_variants/dbg.so python tools/diag_warps.py c3
"""

import ctypes
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2005_01442_b200 as vr  # noqa: E402
from paper_2005_01442_b200 import _lib  # noqa: E402


def main(config="c3"):
    cfg = bench.CONFIGS[config]
    dvol = vr.device_phantom("torso", cfg["dims"])
    nx, ny, nz = dvol.dims
    cam = bench.make_camera(vr, cfg, (nx - 1.0, ny - 1.0, nz - 1.0))
    r = vr.Renderer(dvol, cam, vr.get_preset(cfg["tf"]), vr.RenderSettings(**cfg["settings"]), time_kernel=True)
    buf = torch.zeros(4 * 148 * 64 + 64, dtype=torch.int64, device="cuda")  # [0, 148*32) kernel 1 warps, rest kernel 2
    L = _lib.load()
    L.vr_debug_set_times.argtypes = [ctypes.c_void_p]
    L.vr_debug_set_times(ctypes.c_void_p(buf.data_ptr()))
    for _ in range(3):
        r.render_async()
    torch.cuda.synchronize()
    print("kernel ms", r.kernel_ms())
    host = buf.cpu().numpy()
    st = host[4 * 148 * 64:] // 3  # three frames rendered
    names = ["chunks", "chunks_cand", "cands", "contribs", "leaps", "leapt", "et_rays", "rays", "left",
             "h0", "h1-4", "h5-16", "h17-32"]
    print("heavy stats:", {n: int(v) for n, v in zip(names[:9], st[:9])},
          "cands/chunk hist:", {n: int(v) for n, v in zip(names[9:], st[10:14])},
          "visible/chunk hist:", {n: int(v) for n, v in zip(["1-2", "3-5", "6-10", "11-32"], st[14:18])})
    pst = host[4 * 148 * 64 + 20: 4 * 148 * 64 + 26] // 3
    print("post rays: no-sample", int(pst[0]), "work", int(pst[1]), "| sampled", int(pst[2]), "work", int(pst[3]),
          "| handed over", int(pst[4]), "work", int(pst[5]))
    allt = host[: 4 * 148 * 64].reshape(-1, 4)
    t = allt[: 148 * 32]
    t = t[t[:, 1] > 0]
    t0 = t[:, 0].min()
    h = allt[148 * 32:]
    h = h[h[:, 1] > 0]
    if len(h):
        hs, he = (h[:, 0] - t0) / 1e3, (h[:, 1] - t0) / 1e3
        print(f"cooperative kernel: {len(h)} warps, heavy rays {h[0, 2]}, rays/warp max {h[:, 3].max()} "
              f"mean {h[:, 3].mean():.1f}; start {hs.min():.1f}..{hs.max():.1f} us, end p50 "
              f"{np.percentile(he, 50):.1f} p90 {np.percentile(he, 90):.1f} max {he.max():.1f} us")
    start = (t[:, 0] - t0) / 1e3
    end = (t[:, 1] - t0) / 1e3
    print(f"warps {len(t)}  start max {start.max():.1f} us  end: min {end.min():.1f} "
          f"p10 {np.percentile(end, 10):.1f} p50 {np.percentile(end, 50):.1f} p90 {np.percentile(end, 90):.1f} "
          f"p99 {np.percentile(end, 99):.1f} max {end.max():.1f} us")
    dr = t[:, 2]
    has = dr > 0
    if has.any():
        tail = (t[has, 1] - dr[has]) / 1e3
        print(f"post warps: drained seen at {((dr[has] - t0) / 1e3).min():.1f}..{((dr[has] - t0) / 1e3).max():.1f} us; "
              f"end - drain p50 {np.percentile(tail, 50):.1f} p90 {np.percentile(tail, 90):.1f} max {tail.max():.1f} us; "
              f"trips after drain p50 {np.percentile(t[has, 3], 50):.0f} max {t[has, 3].max()}")
    busy = np.zeros(400)
    for e in end:
        busy[: int(e / (end.max() / 400)) + 0] += 1
    print("warps alive over time (10 buckets):", [int(busy[i * 40]) for i in range(10)])
    order = np.argsort(-end)[:10]
    print("latest warps (end us, trips after drain):", [(round(end[i], 1), int(t[i, 3])) for i in order])


if __name__ == "__main__":
    main(*sys.argv[1:])
