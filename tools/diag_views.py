"""Batched views in several chunks vs single renders (debug, with timings)."""
import math, sys, time
import numpy as np
sys.path.insert(0, '.')
import torch
import paper_2005_01442_b200 as vr
n = int(sys.argv[1]) if len(sys.argv) > 1 else 20
dims = tuple(int(x) for x in (sys.argv[2] if len(sys.argv) > 2 else "96,80,72").split(","))
size = int(sys.argv[3]) if len(sys.argv) > 3 else 64
vol = vr.generate_phantom("torso", dims)
ext = vol.extent_mm; c = [0.5 * e for e in ext]; d = 2.2 * max(ext)
cams = [vr.Camera(position=(c[0] + d * math.cos(2 * math.pi * k / n), c[1] + d * math.sin(2 * math.pi * k / n), c[2]),
                  look_at=tuple(c), width=size, height=size) for k in range(n)]
s = vr.RenderSettings(interpolation="tricubic", use_blocks=True, block_size=32)
tf = vr.get_preset("bone")
r = vr.Renderer(vol, cams[0], tf, s, views=n)
r.set_views(cams)
t0 = time.time(); r.render_async(); torch.cuda.synchronize(); print("batch", n, "views", round(time.time() - t0, 3), "s", flush=True)
pv = r.view_stats()
bad = 0
for v in range(n):
    one = vr.Renderer(vol, cams[v], tf, s); one.render_async()
    ok = np.array_equal(r.pixels[v].cpu().numpy(), one.pixels.cpu().numpy()) and pv[v]["samples_taken"] == one.stats()["samples_taken"]
    bad += not ok
print("views differing:", bad, flush=True)
