"""Diagnostics: time the heaviest 16x8 cell of a config warp by warp (8x4
tiles) and ray by ray.  Development tool."""

import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2005_01442_b200 as vr  # noqa: E402


def main(config="c3", cx=36, cy=48, reps=3, only_ray=0):
    reps, only_ray = int(reps), int(only_ray)
    cfg = bench.CONFIGS[config]
    dvol = vr.device_phantom("torso", cfg["dims"])
    nx, ny, nz = dvol.dims
    cam = bench.make_camera(vr, cfg, (nx - 1.0, ny - 1.0, nz - 1.0))
    tf = vr.get_preset(cfg["tf"])
    s = vr.RenderSettings(**cfg["settings"])

    def run(rect):
        r = vr.Renderer(dvol, cam, tf, s, tile=rect, time_kernel=True, per_pixel_counts=True)
        best = 1e9
        for _ in range(reps):
            r.render_async()
            torch.cuda.synchronize()
            best = min(best, r.kernel_ms())
        return best, r

    x0, y0 = int(cx) * 16, int(cy) * 8
    if only_ray:
        t, r = run((586, 384, 1, 1))
        print(f"ray (586,384): {t:.3f} ms {r.stats()}")
        return
    t, r = run((x0, y0, 16, 8))
    print(f"cell ({cx},{cy}) 16x8: {t:.3f} ms {r.stats()}")
    for wy in range(2):
        for wx in range(2):
            t, r = run((x0 + 8 * wx, y0 + 4 * wy, 8, 4))
            st = r.stats()
            print(f"  warp tile ({wx},{wy}) 8x4: {t:.3f} ms taken={st['samples_taken']} "
                  f"interp={st['interpolated']} iters={st['march_iterations']} "
                  f"max taken/ray={int(r.taken.max())}")
    # the single most expensive ray of the cell
    t, r = run((x0, y0, 16, 8))
    taken = r.taken.cpu().numpy().reshape(8, 16)
    py, px = np.unravel_index(np.argmax(taken), taken.shape)
    t1, r1 = run((x0 + int(px), y0 + int(py), 1, 1))
    print(f"  heaviest ray ({x0 + px},{y0 + py}) alone: {t1:.3f} ms {r1.stats()}")


if __name__ == "__main__":
    main(*sys.argv[1:])
