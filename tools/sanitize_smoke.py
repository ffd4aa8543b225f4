"""Small workload touching every kernel family, for compute-sanitizer:
K0 ingest, K1 volume/bricks/culling tables, K2 block min/max + visibility,
K3 persistent + cooperative ray casters (post), one-thread-per-ray kernels
(pre / preint / iso), batched views, K4 measures, point sampling, quality."""
import sys
import numpy as np
sys.path.insert(0, ".")
import torch
import paper_2005_01442_b200 as vr

vol = vr.generate_phantom("torso", (56, 48, 40), (0.9, 1.0, 1.2))
raw = vr.ingest_raw(vol.values.astype("<u2").tobytes(), (56, 48, 40), (0.9, 1.0, 1.2), "u16") \
    if hasattr(vr, "ingest_raw") else None
ext = vol.extent_mm
c = tuple(0.5 * e for e in ext)
cams = [vr.Camera(position=(c[0] + 2.2 * max(ext), c[1] + 5.0, c[2] - 3.0), look_at=c, width=48, height=40),
        vr.Camera(position=(c[0], c[1] - 2.2 * max(ext), c[2] + 9.0), look_at=c, width=48, height=40)]
tf = vr.get_preset("bone")
runs = [dict(interpolation="tricubic", use_blocks=True, block_size=16),
        dict(interpolation="tricubic"),
        dict(interpolation="trilinear", use_blocks=True, block_size=16, lighting=False, early_termination_alpha=1.0),
        dict(interpolation="tricubic", classification="pre", use_blocks=True, block_size=16),
        dict(interpolation="trilinear", classification="preintegrated", use_blocks=True, block_size=16),
        dict(interpolation="tricubic", mode="isosurface", isovalue=600.0, use_blocks=True, block_size=16)]
for kw in runs:
    s = vr.RenderSettings(**kw)
    img = vr.render(vol, cams[0], tf, s)
    print(kw, img.stats.samples_taken)
r = vr.Renderer(vol, cams[0], tf, vr.RenderSettings(**runs[0]), views=2, per_pixel_counts=True)
r.set_views(cams)
r.render_async()
torch.cuda.synchronize()
print("views", [v["samples_taken"] for v in r.view_stats()])
print("measure", vr.threshold_measure(vol, 550), vr.ball_measure(vol, 550, [[20.0, 20.0, 20.0]], 8.0)["count"])
print("sample", vr.sample(vol, np.array([[3.3, 4.4, 5.5]]), "tricubic"))
a = vr.render(vol, cams[0], tf, vr.RenderSettings(**runs[0])).pixels
print("psnr", vr.psnr(a, a), "ssim", vr.ssim(a, a))
