"""Per-call render() latency distribution at c3 (GPU box): spikes hunting."""
import gc
import sys
import time

sys.path.insert(0, '/root/repo')
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2005_01442_b200 as vr  # noqa: E402

cfg = bench.CONFIGS['c3']
dvol = vr.device_phantom("torso", cfg["dims"])
host = vr.ScalarVolume(dvol.download(), (1.0, 1.0, 1.0), dvol.value_range)
host._attach_device(dvol)
cam = bench.make_camera(vr, cfg, (511.0, 511.0, 511.0))
tf, st = vr.get_preset('bone'), vr.RenderSettings(**cfg['settings'])
for _ in range(3):
    vr.render(host, cam, tf, st)
torch.cuda.synchronize()
for label, disable_gc in (("gc on", False), ("gc off", True)):
    if disable_gc:
        gc.disable()
    ts = []
    for _ in range(300):
        t0 = time.perf_counter()
        px = vr.render(host, cam, tf, st).pixels
        ts.append(time.perf_counter() - t0)
    ts = np.array(ts) * 1e3
    print(label, "mean %.3f p50 %.3f p90 %.3f p99 %.3f max %.3f" % (ts.mean(), *np.percentile(ts, [50, 90, 99]), ts.max()),
          "slow calls:", np.nonzero(ts > 3)[0][:20].tolist())
    gc.enable()
