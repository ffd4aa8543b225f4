"""Diagnostics: where does a frame's time go?  Times the ray-cast kernel on
sub-rectangles of the C3 frame (CUDA events around the launch) and reports
the per-tile cost next to the full-frame cost.  Development tool."""

import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2005_01442_b200 as vr  # noqa: E402


def main(config="c3", tile=128):
    cfg = bench.CONFIGS[config]
    dvol = vr.device_phantom("torso", cfg["dims"])
    nx, ny, nz = dvol.dims
    cam = bench.make_camera(vr, cfg, (nx - 1.0, ny - 1.0, nz - 1.0))
    tf = vr.get_preset(cfg["tf"])
    s = vr.RenderSettings(**cfg["settings"])
    W = cam.width

    def kernel_ms(rect, reps=3):
        r = vr.Renderer(dvol, cam, tf, s, tile=rect, time_kernel=True, per_pixel_counts=True)
        best = 1e9
        for _ in range(reps):
            r.render_async()
            torch.cuda.synchronize()
            best = min(best, r.kernel_ms())
        return best, r

    full, rf = kernel_ms(None)
    taken = rf.taken.cpu().numpy().reshape(cam.height, W)
    st = rf.stats()
    print(f"full frame: {full:.3f} ms  {st}")
    grid = np.zeros((W // tile, W // tile))
    for ty in range(W // tile):
        for tx in range(W // tile):
            grid[ty, tx], _ = kernel_ms((tx * tile, ty * tile, tile, tile), reps=2)
    print(f"{tile}x{tile} tiles: sum {grid.sum():.3f} ms, max {grid.max():.3f} ms")
    print(np.array2string(grid, precision=2, max_line_width=200))
    # the heaviest 16x8 cell by taken samples
    cells = taken.reshape(cam.height // 8, 8, W // 16, 16).sum(axis=(1, 3))
    cy, cx = np.unravel_index(np.argmax(cells), cells.shape)
    one, r1 = kernel_ms((cx * 16, cy * 8, 16, 8))
    print(f"heaviest cell ({cx},{cy}) taken={cells[cy, cx]} max/ray={taken[cy*8:cy*8+8, cx*16:cx*16+16].max()}: "
          f"{one:.3f} ms alone; {r1.stats()}")


if __name__ == "__main__":
    main(*sys.argv[1:2])
