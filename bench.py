#!/usr/bin/env python
"""Benchmark of the volume ray-casting hot path (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config c3]

Metric: frames/s (and samples/s) rendering the torso phantom 512^3 int16 CT to
1024^2 with tricubic sampling, 64^3/overlap-3 bricks with empty-space leaping,
bone TF, headlight shading, ET 0.99.  One step = one
frame: TF visibility (K2b) + the ray-cast kernel (K3) + stats; for N > 1 the
frame is split sort-first into interleaved 16x8 cells across ranks and the
packed cells are gathered to rank 0 over NCCL (strong scaling).

``value`` is device time with the volume resident in HBM (CUDA events on the
render stream, L2 flushed between steps by writing a 512 MiB buffer, then
reading another 512 MiB so the flush's dirty lines are written back before the
timed frame starts; max over ranks).  ``e2e`` is the same metric through the public host API
``render(volume, camera, tf, settings)`` (LUT uploaded and the uint8 image +
stats downloaded every step; the volume stays cached on the device as the
reference's volume store caches it).  ``--impl reference`` times the CPU
oracle (oracle/, a C restatement of the reference's numba march pinned to the
reference's goldens) on all host threads.
"""

from __future__ import annotations

import argparse
import gc
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

CONFIGS = {
    # name: phantom dims, image size, settings overrides, tf
    "c1": dict(dims=(64, 64, 64), size=128, tf="bone", projection="orthographic",
               settings=dict(interpolation="tricubic"), desc="64^3 -> 128^2 orthographic, tricubic, monolithic"),
    "c2": dict(dims=(256, 256, 256), size=512, tf="bone", projection="pinhole",
               settings=dict(interpolation="tricubic"), desc="256^3 -> 512^2 pinhole, tricubic, monolithic"),
    "c3": dict(dims=(512, 512, 512), size=1024, tf="bone", projection="pinhole",
               settings=dict(interpolation="tricubic", use_blocks=True),
               desc="512^3 -> 1024^2 pinhole, tricubic, bricks 64/3 + empty-space leaping"),
    "c3soft": dict(dims=(512, 512, 512), size=1024, tf="soft-tissue", projection="pinhole",
                   settings=dict(interpolation="tricubic", use_blocks=True),
                   desc="C3 with the soft-tissue TF"),
    "c3stress": dict(dims=(512, 512, 512), size=1024, tf="grayscale", projection="pinhole",
                     settings=dict(interpolation="tricubic", lighting=False, early_termination_alpha=1.0),
                     desc="C3-stress: monolithic, grayscale, ET off, no lighting (every step sampled)"),
    "c3pre": dict(dims=(512, 512, 512), size=1024, tf="bone", projection="pinhole",
                  settings=dict(interpolation="tricubic", use_blocks=True, classification="pre"),
                  desc="C3, pre-classified (_kernels.py:471-507)"),
    "c3preint": dict(dims=(512, 512, 512), size=1024, tf="bone", projection="pinhole",
                     settings=dict(interpolation="tricubic", use_blocks=True, classification="preintegrated"),
                     desc="C3, pre-integrated (_kernels.py:538-581; the reference service's default)"),
    "c3iso": dict(dims=(512, 512, 512), size=1024, tf="bone", projection="pinhole",
                  settings=dict(interpolation="tricubic", use_blocks=True, mode="isosurface", isovalue=600.0),
                  desc="C3, isosurface at 600 HU (_kernels.py:405-468)"),
    "c4": dict(dims=(512, 512, 2048), size=2048, tf="bone", projection="pinhole",
               settings=dict(interpolation="tricubic", use_blocks=True),
               desc="512x512x2048 -> 2048^2, tricubic, bricks 64/3"),
    "c5": dict(dims=(512, 512, 512), size=1024, tf="bone", projection="pinhole", views=360,
               settings=dict(interpolation="tricubic", use_blocks=True),
               measure=dict(threshold=550, balls=360, radius=16.0),
               desc="turntable: 360 views/step (1 deg apart) of C3 in one batched submission + the method "
                    "of spheres (threshold 550: whole-volume V and S, 360 probe balls R=16 mm)"),
}

# standalone K4 line (`--config k4`): the method of spheres on the C3 volume
K4_CONFIG = dict(dims=(512, 512, 512), threshold=550, balls=360, radius=16.0,
                 desc="method of spheres on the 512^3 torso: whole-volume V (voxel count) and S (isosurface "
                      "area) at 550 HU + 360 probe balls R=16 mm")

L2_FLUSH_BYTES = 512 << 20


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=100)
    p.add_argument("--warmup", type=int, default=5)
    p.add_argument("--impl", choices=("ours", "reference"), default="ours")
    p.add_argument("--config", choices=sorted(CONFIGS) + ["k4"], default="c3")
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--dist-backend", choices=("nccl", "gloo"), default="nccl")
    p.add_argument("--transport", choices=("shared", "gather"), default=None,
                   help="N>1 frame exchange: one stream-ordered NCCL/gloo gather of the packed cells "
                        "(gather, default) or stores into rank 0's frame over NVLink (shared; host "
                        "barriers per frame)")
    p.add_argument("--set", action="append", default=[], metavar="KEY=VALUE",
                   help="override a RenderSettings field of the config (ablations)")
    args = p.parse_args()
    for kv in args.set if args.config != "k4" else []:
        key, val = kv.split("=", 1)
        try:
            CONFIGS[args.config]["settings"][key] = json.loads(val)
        except json.JSONDecodeError:
            CONFIGS[args.config]["settings"][key] = val
        CONFIGS[args.config]["desc"] += f" [{kv}]"
    return args


def centered_camera(cls, extent, size, **kw):
    """tests/conftest.py:34-43 of the reference: +x side at 2.2x the largest extent."""
    cx, cy, cz = (0.5 * e for e in extent)
    d = 2.2 * max(extent)
    return cls(position=(cx + d, cy, cz), look_at=(cx, cy, cz), width=size, height=size, **kw)


def make_camera(vr, cfg, extent):
    if cfg["projection"] == "orthographic":
        half = 0.5 * max(extent) + 1.0
        return centered_camera(vr.OrthographicCamera, extent, cfg["size"], half_height_mm=half)
    return centered_camera(vr.Camera, extent, cfg["size"])


class ClockSampler:
    """nvidia-smi clocks and throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "20"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
            t0 = time.time()
            while not self.lines and time.time() - t0 < 5.0:  # nvidia-smi is up and sampling
                time.sleep(0.01)
        except Exception:
            self.proc = None
        self.start = len(self.lines)
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *exc):
        t0 = time.time()
        while self.proc and len(self.lines) <= self.start and time.time() - t0 < 0.2:
            time.sleep(0.005)  # short runs: at least one sample taken after the timed region began
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], [], set()
        names = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
        for ln in self.lines[self.start:] if len(self.lines) > self.start else self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
            except ValueError:
                continue
            for name, val in zip(names, parts[3:7]):
                if val.lower().startswith("active"):
                    reasons.add(name)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(mx), "reasons": sorted(reasons),
                "samples": len(sm)}


def measured_peak():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        try:
            return float(json.loads(p.read_text())["hbm_gbs"]), "measured"
        except Exception:
            pass
    return 6650.0, "fallback"


def committed_traffic(config):
    """dram bytes per launch of the ray-cast kernel from the committed ncu capture."""
    p = ROOT / "profiles" / f"ncu_raycast_{config}.json"
    if p.exists():
        try:
            return float(json.loads(p.read_text())["dram_bytes_per_launch"])
        except Exception:
            return None
    return None


def committed_ncu(config):
    """Issue / pipe utilisation and memory traffic of the ray casters from the
    committed ncu --set full capture (profiles/ncu_raycast_<config>.json)."""
    p = ROOT / "profiles" / f"ncu_raycast_{config}.json"
    if not p.exists():
        return None
    try:
        d = json.loads(p.read_text())
    except Exception:
        return None
    return {k: d[k] for k in ("source", "kernels", "dram_bytes_per_launch", "issue_active_pct",
                              "fp64_pipe_pct", "l1_hit_pct", "l2_hit_pct", "warps_active_pct", "per_kernel")
            if k in d}


def dist_setup(n, backend):
    """One process per GPU (torchrun env); NCCL over NVLink by default.  gloo
    (CPU transport, several ranks may share one GPU) exists only to exercise
    the multi-rank code path where fewer GPUs than ranks are available."""
    if n <= 1:
        return 0, 1, 0
    import torch
    import torch.distributed as dist

    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    rank = int(os.environ["RANK"])
    world = int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    if backend == "nccl":
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    else:
        torch.cuda.set_device(local % torch.cuda.device_count())
        dist.init_process_group("gloo")
    return rank, world, local


def orbit_cameras(vr, extent, size, views):
    """Turntable (C5): azimuth k*360/views degrees in the z = centre plane at
    2.2x the largest extent (viewer orbit, frontend/src/camera.ts:35-44)."""
    import math

    cx, cy, cz = (0.5 * e for e in extent)
    d = 2.2 * max(extent)
    cams = []
    for k in range(views):
        ang = 2.0 * math.pi * k / views
        cams.append(vr.Camera(position=(cx + d * math.cos(ang), cy + d * math.sin(ang), cz),
                              look_at=(cx, cy, cz), width=size, height=size))
    return cams


ORACLE_DEFAULTS = dict(step=None, interpolation="trilinear", classification="post", mode="dvr",
                       isovalue=None, lighting=True, early_termination_alpha=0.99, use_blocks=False,
                       block_size=64, overlap=3, background=(0.0, 0.0, 0.0, 1.0), ambient=0.1,
                       diffuse=0.7, specular=0.2, shininess=32.0)  # RenderSettings defaults, render.py:159-181


def oracle_scene_args(cfg, extent):
    """Camera, TF arrays and settings of a config for the CPU oracle, built
    without the product package (the reference arm maps no product code)."""
    from types import SimpleNamespace

    from oracle import oracle as O

    cx, cy, cz = (0.5 * e for e in extent)
    d = 2.2 * max(extent)
    cam = SimpleNamespace(position=(cx + d, cy, cz), look_at=(cx, cy, cz), up=(0.0, 0.0, 1.0),
                          vertical_fov_deg=30.0, width=cfg["size"], height=cfg["size"],
                          projection=cfg["projection"],
                          half_height_mm=0.5 * max(extent) + 1.0 if cfg["projection"] == "orthographic" else None)
    settings = SimpleNamespace(**dict(ORACLE_DEFAULTS, **cfg["settings"]))
    return cam, O.preset_arrays(cfg["tf"]), settings


def cpu_oracle_frame(values, spacing, camera, tf, settings, nthreads=0):
    """One full frame through the CPU oracle (prep + march), like reference render().
    tf = (values, rgba, domain) arrays."""
    from oracle import oracle as O

    t0 = time.perf_counter()
    r = O.render(values, spacing, camera, tf[0], tf[1], tf[2], settings,
                 projection=getattr(camera, "projection", "pinhole"),
                 ortho_half_h=getattr(camera, "half_height_mm", None), nthreads=nthreads)
    return time.perf_counter() - t0, r


def bench_config(args, cfg):
    """The `config` object both arms print (identical, so the driver can pair them)."""
    return {"workload": args.config, "desc": cfg["desc"], "volume": list(cfg["dims"]),
            "image": [cfg["size"], cfg["size"]], "views_per_step": cfg.get("views", 1), "tf": cfg["tf"],
            "settings": {k: v for k, v in sorted(cfg["settings"].items())}}


def ball_centres(extent, n):
    """K4 probe-ball centres (seeded: default_rng(0))."""
    import numpy as np

    rng = np.random.default_rng(0)
    return rng.uniform(0.2, 0.8, size=(n, 3)) * np.array(extent)


def cpu_sweep_sample(cfg, values, spacing, extent, sample_views):
    """C5 on the CPU oracle, bounded: `sample_views` of the 360 views (evenly
    spaced) plus the full method-of-spheres measure; the sweep time is
    estimated as 360/sample_views x the views' time + the measure's."""
    from types import SimpleNamespace

    from oracle import oracle as O

    views = cfg["views"]
    cam0, tf, settings = oracle_scene_args(cfg, extent)
    cx, cy, cz = (0.5 * e for e in extent)
    d = 2.2 * max(extent)
    t_views = 0.0
    taken = 0
    for i in range(sample_views):
        k = i * views // sample_views
        ang = 2.0 * math.pi * k / views
        cam = SimpleNamespace(**{**cam0.__dict__, "position": (cx + d * math.cos(ang), cy + d * math.sin(ang), cz)})
        t, r = cpu_oracle_frame(values, spacing, cam, tf, settings)
        t_views += t
        taken += r.samples_taken
    m = cfg["measure"]
    t0 = time.perf_counter()
    O.threshold_measure(values, spacing, m["threshold"])
    O.ball_measure(values, spacing, m["threshold"], ball_centres(extent, m["balls"]), [m["radius"]] * m["balls"])
    t_k4 = time.perf_counter() - t0
    sweep = t_views * views / sample_views + t_k4
    return {"value": views / sweep, "unit": "frames/s", "cores": O.num_threads(), "kind": "port",
            "sample": f"{sample_views} of the {views} views via oracle.render ({t_views:.2f} s) + the full "
                      f"method-of-spheres measure via the oracle ({t_k4:.2f} s); sweep time estimated as "
                      f"{views}/{sample_views} x views + measure",
            "samples_taken_sampled_views": taken}


def run_reference(args):
    """--impl reference: the CPU oracle port (C restatement of the reference's
    numba march + numpy prep, pinned to the reference's goldens) on all host
    threads, rank 0 only.  Nothing from the product package is imported: the
    phantom is the oracle's numpy restatement of phantoms.py."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    from oracle import oracle as O

    cfg = CONFIGS[args.config]
    t_ph = time.perf_counter()
    values = O.phantom("torso", cfg["dims"])
    t_ph = time.perf_counter() - t_ph
    spacing = (1.0, 1.0, 1.0)
    nz, ny, nx = values.shape
    extent = ((nx - 1) * spacing[0], (ny - 1) * spacing[1], (nz - 1) * spacing[2])
    camera, tf, settings = oracle_scene_args(cfg, extent)
    threads = O.num_threads()
    if cfg.get("views", 1) > 1:
        # the sweep, sampled: each step renders 2 of the views + the full measure
        for _ in range(max(args.warmup, 0)):
            cpu_sweep_sample(cfg, values, spacing, extent, sample_views=2)
        est = [cpu_sweep_sample(cfg, values, spacing, extent, sample_views=2) for _ in range(args.steps)]
        sweep_s = [cfg["views"] / e["value"] for e in est]
        fps = args.steps * cfg["views"] / sum(sweep_s)
        line = {
            "impl": "reference", "metric": "frames/sec", "value": fps, "unit": "frames/s",
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": 1e3 * sum(sweep_s) / args.steps, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic", "config": bench_config(args, cfg),
            "parallelism": f"CPU, {threads} threads (rank 0 only)",
            "cpu_baseline": {"value": fps, "unit": "frames/s", "cores": threads, "kind": "port",
                             "sample": "per step: " + est[-1]["sample"]},
            "e2e": {"value": fps, "unit": "frames/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        }
        print(json.dumps(line), flush=True)
        return
    for _ in range(max(args.warmup, 0)):
        cpu_oracle_frame(values, spacing, camera, tf, settings)
    times, taken = [], 0
    for _ in range(args.steps):
        t, r = cpu_oracle_frame(values, spacing, camera, tf, settings)
        times.append(t)
        taken = r.samples_taken
    total = sum(times)
    fps = args.steps / total
    line = {
        "impl": "reference", "metric": "frames/sec", "value": fps, "unit": "frames/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * total / args.steps, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "samples_per_sec": taken * fps, "samples_taken": taken,
        "config": bench_config(args, cfg),
        "parallelism": f"CPU, {threads} threads (rank 0 only)",
        "cpu_baseline": {"value": fps, "unit": "frames/s", "cores": threads, "kind": "port",
                         "sample": f"{args.steps} full {args.config} frames via oracle.render "
                                   "(C restatement of _kernels.march, OpenMP over pixels, prep included; "
                                   f"phantom from the oracle's numpy generator, {t_ph:.1f} s, untimed)"},
        "e2e": {"value": fps, "unit": "frames/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def launches_per_frame(settings):
    """Kernels of ours in one single-view frame (vr_render): TF visibility (4
    on the block path: value bits, block intervals + LUT range + frame zeroing,
    AABB fit, boxes; the LUT range kernel on the monolithic post path), the
    mode's table kernel (pre-integrated: the non-zero prefix count; pre: the
    non-zero-alpha value range), the per-lane and cooperative ray casters
    (every mode, persistent), and the blocks_visited count."""
    post = settings.mode == "dvr" and settings.classification == "post"
    n = 4 if settings.use_blocks else (1 if post else 0)
    if settings.mode == "dvr" and settings.classification in ("pre", "preintegrated"):
        n += 1
    n += 2  # per-lane + cooperative ray casters
    return n + 1


def run_ours(args):
    import ctypes

    import torch

    import paper_2005_01442_b200 as vr
    from paper_2005_01442_b200 import _lib
    from paper_2005_01442_b200.distributed import gather_frame, render_sharded

    rank, world, local = dist_setup(args.gpus, args.dist_backend)
    if world == 1:
        torch.cuda.set_device(0)
    dev = torch.device("cuda", torch.cuda.current_device())
    cfg = CONFIGS[args.config]
    spacing = (1.0, 1.0, 1.0)
    dvol = vr.device_phantom("torso", cfg["dims"], spacing, device=dev.index)
    nx, ny, nz = dvol.dims
    extent = ((nx - 1) * spacing[0], (ny - 1) * spacing[1], (nz - 1) * spacing[2])
    views = cfg.get("views", 1)
    cameras = orbit_cameras(vr, extent, cfg["size"], views) if views > 1 else [make_camera(vr, cfg, extent)]
    my_views = list(range(rank, views, world)) if views > 1 else [0]  # view-parallel sweep: view v -> rank v % N
    tf = vr.get_preset(cfg["tf"])
    settings = vr.RenderSettings(**cfg["settings"])
    # the NCCL gather is stream-ordered (no host round trip per frame); the
    # CUDA-IPC shared frame needs host barriers per frame and is opt-in
    transport = args.transport or "gather"
    shared = None
    if world > 1 and views == 1 and transport == "shared":
        from paper_2005_01442_b200.distributed import SharedFrame

        try:
            shared = SharedFrame(cameras[0].height, cameras[0].width, device=dev.index)
        except Exception as exc:  # no peer access between these GPUs: fall back to the gather
            print(f"shared frame unavailable ({exc}); using the gather", file=sys.stderr)
            transport = "gather"
    if views > 1:
        # the sweep: one vr_render_views submission for all of this rank's views
        rend = vr.Renderer(dvol, cameras[my_views[0]], tf, settings, device=dev.index, time_kernel=True,
                           views=len(my_views))
        rend.set_views([cameras[v] for v in my_views])
    else:
        rend = vr.Renderer(dvol, cameras[0], tf, settings, device=dev.index,
                           interleave=(world, rank) if world > 1 else None, time_kernel=True,
                           frame_out=shared.frame if shared is not None else None)
    stream = torch.cuda.current_stream(dev)
    flush = torch.empty(L2_FLUSH_BYTES, dtype=torch.uint8, device=dev)
    # read after the write flush so L2 holds clean lines: the timed frame then
    # does not pay the write-back of the flush buffer's dirty lines
    clean = torch.ones(L2_FLUSH_BYTES // 4, dtype=torch.int32, device=dev)
    W, H = cameras[0].width, cameras[0].height
    measure = cfg.get("measure")
    L = _lib.load()
    if measure:
        # K4 batched with the sweep: whole-volume threshold count + ball counts
        import numpy as np

        centres = torch.from_numpy(ball_centres(extent, measure["balls"])).to(dev)
        radii = torch.full((measure["balls"],), float(measure["radius"]), dtype=torch.float64, device=dev)
        k4 = torch.zeros(2 + 2 * measure["balls"], dtype=torch.int64, device=dev)

    def frame():
        if views > 1:
            rend.render_async(stream)
        else:
            if shared is not None:
                shared.acquire()  # rank 0 is done with the previous frame
            rend.render_async(stream)
            if shared is not None:
                shared.publish()
            elif world > 1:
                packed = rend.pixels.reshape(-1, 4)
                gather_frame(packed if args.dist_backend == "nccl" else packed.cpu(), W, H)
        if measure and rank == 0:  # K4 on the sweep's stream (rank 0: it is whole-volume)
            s = _lib.ptr_stream(stream)
            _lib.check(L.vr_threshold_measure(dvol.handle, int(measure["threshold"]), _lib.ptr(k4), s))
            nb = measure["balls"]
            _lib.check(L.vr_ball_measure(dvol.handle, int(measure["threshold"]), _lib.ptr(centres), _lib.ptr(radii),
                                         nb, ctypes.c_void_p(k4.data_ptr() + 16),
                                         ctypes.c_void_p(k4.data_ptr() + 16 + 8 * nb), s))

    for _ in range(max(args.warmup, 3)):
        frame()
    torch.cuda.synchronize()
    st = rend.stats()  # this rank's frame share, or its whole batch of views
    st_local = dict(st)
    if world > 1:
        import torch.distributed as dist

        t = torch.tensor([st["samples_taken"], st["samples_skipped"], st["shaded"]], dtype=torch.int64)
        t = t if args.dist_backend == "gloo" else t.to(dev)
        dist.all_reduce(t)
        st["samples_taken"], st["samples_skipped"], st["shaded"] = (int(x) for x in t.tolist())
        dist.barrier()
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    step_ms, kern_ms = [], []
    torch.cuda.synchronize()
    with ClockSampler(dev.index) as clocks:
        for _ in range(args.steps):
            flush.fill_(1)  # evict the previous frame's working set from L2 (outside the timed pair)
            clean.amax()
            ev0.record(stream)
            frame()
            ev1.record(stream)
            ev1.synchronize()
            step_ms.append(ev0.elapsed_time(ev1))
            kern_ms.append(rend.kernel_ms())  # the ray-cast launch pair (all of a batch's views)
        torch.cuda.synchronize()
    total_ms = sum(step_ms)
    kern_total = sum(kern_ms)
    if world > 1:
        import torch.distributed as dist

        t = torch.tensor([total_ms, kern_total], dtype=torch.float64)
        t = t if args.dist_backend == "gloo" else t.to(dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total_ms, kern_total = t.tolist()
    fps = args.steps * views / (total_ms / 1e3)
    taken, shaded = st["samples_taken"], st["shaded"]
    kern_s = kern_total / args.steps / 1e3
    cubic = settings.interpolation == "tricubic"
    b_sample = 128 if cubic else 16
    b_grad = 768 if cubic else 96
    # Bytes the ray-cast launches actually gather (one rank's share of the
    # frame): every interpolation evaluated -- sample interpolations plus the
    # 6 gradient taps of each shaded sample -- reads its B_s-byte tap
    # neighbourhood; every march iteration reads its block's 32-byte skip
    # record; every pixel writes 4 bytes.  Culled samples (provably
    # transparent) are counted as taken but read nothing, so the survey's
    # taken-based model overstates the work; it is kept below
    # as `survey_model` for comparison.
    interp = int(st_local.get("interpolated") or 0)
    iters = int(st_local.get("march_iterations") or 0)
    pix_bytes = (W * H * len(my_views) if views > 1 else rend.npix) * 4
    gathered = (interp + 6 * st_local["shaded"]) * b_sample + iters * 32 + pix_bytes
    achieved = gathered / kern_s / 1e9
    survey_bytes = st_local["samples_taken"] * b_sample + st_local["shaded"] * b_grad + pix_bytes
    peak, peak_kind = measured_peak()

    e2e = None
    if not args.no_e2e and views > 1:
        # the sweep through the public host API: render_views (one submission,
        # frames copied to host memory) + the method of spheres on rank 0
        import numpy as np

        host_vol = vr.ScalarVolume(dvol.download(), spacing, dvol.value_range)
        host_vol._attach_device(dvol)
        mine = [cameras[v] for v in my_views]
        c_host = centres.cpu().numpy() if measure else None

        def call():
            imgs = vr.render_views(host_vol, mine, tf, settings)
            if measure and rank == 0:
                vr.threshold_measure(host_vol, measure["threshold"])
                vr.ball_measure(host_vol, measure["threshold"], c_host, measure["radius"])
            return imgs
        for _ in range(max(1, min(args.warmup, 2))):
            call()
        torch.cuda.synchronize()
        if world > 1:
            import torch.distributed as dist

            dist.barrier()
        gc.collect()
        gc.disable()
        t0 = time.perf_counter()
        for _ in range(args.steps):
            imgs = call()
        e2e_s = time.perf_counter() - t0
        gc.enable()
        del imgs
        if world > 1:
            t = torch.tensor([e2e_s], dtype=torch.float64)
            t = t if args.dist_backend == "gloo" else t.to(dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            e2e_s = float(t.item())
        nb = measure["balls"] if measure else 0
        e2e = {"value": args.steps * views / e2e_s, "unit": "frames/s",
               "h2d_bytes_per_step": 4096 * 4 * 8 + 14 * 8 * len(my_views) + (32 * nb if measure else 0),
               "d2h_bytes_per_step": W * H * 4 * len(my_views) + 8 * (5 * len(my_views) + 3)
               + (16 + 16 * nb if measure else 0),
               "api": ("paper_2005_01442_b200.render_views(volume, cameras, TF, settings) -> [ImageRGBA] "
                       "(vr_render_views: one submission for the sweep; frames copied to host) + "
                       "threshold_measure / ball_measure (vr_threshold_measure / vr_ball_measure)")}
    if not args.no_e2e and views == 1:
        host_vol = vr.ScalarVolume(dvol.download(), spacing, dvol.value_range)
        host_vol._attach_device(dvol)
        cam = cameras[0]
        api = ("paper_2005_01442_b200.render(ScalarVolume, Camera, TF, RenderSettings) -> ImageRGBA "
               "(C-ABI vr_render_to_host; volume cached on device; LUT uploaded and the uint8 frame "
               "written to page-locked host memory by the kernels over PCIe every step)")
        if world == 1:
            def call():
                return vr.render(host_vol, cam, tf, settings).pixels
        else:
            import torch.distributed as dist

            api = ("paper_2005_01442_b200.distributed.render_sharded(volume, camera, TF, settings) -> "
                   f"host frame on rank 0 (sort-first cells, {transport})")

            def call():
                return render_sharded(host_vol, cam, tf, settings, shared=shared)[0]
        for _ in range(max(args.warmup, 3)):  # the timed loop's pattern: the last frame stays alive
            px = call()
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        # as timeit does: no cyclic-GC pass inside the timed calls (a full
        # collection of this process's heap is tens of ms, one per ~20 calls)
        gc.collect()
        gc.disable()
        t0 = time.perf_counter()
        per_call = []
        for _ in range(args.steps):
            tc = time.perf_counter()
            px = call()
            per_call.append(time.perf_counter() - tc)
        torch.cuda.synchronize()
        e2e_s = time.perf_counter() - t0
        gc.enable()
        if os.environ.get("VR_E2E_DEBUG"):
            import numpy as np

            pc = np.array(per_call) * 1e3
            print(f"e2e per call ms: mean {pc.mean():.3f} p50 {np.median(pc):.3f} max {pc.max():.3f} "
                  f"first {pc[:5].round(3).tolist()}", file=sys.stderr)
        if world > 1:
            t = torch.tensor([e2e_s], dtype=torch.float64)
            t = t if args.dist_backend == "gloo" else t.to(dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            e2e_s = float(t.item())
        e2e = {"value": args.steps / e2e_s, "unit": "frames/s",
               "h2d_bytes_per_step": 4096 * 4 * 8,
               "d2h_bytes_per_step": W * H * 4 + (5 * 8 if world == 1 else 0),
               "api": api}

    cpu = None
    if rank == 0 and world == 1 and views > 1 and not args.no_cpu_baseline:
        cpu = cpu_sweep_sample(cfg, dvol.download(), spacing, extent, sample_views=2)
    if rank == 0 and world == 1 and views == 1 and not args.no_cpu_baseline:
        from oracle import oracle as O

        values = dvol.download()
        o_cam, o_tf, o_set = oracle_scene_args(cfg, extent)
        t, r = cpu_oracle_frame(values, spacing, o_cam, o_tf, o_set)
        cpu = {"value": 1.0 / t, "unit": "frames/s", "cores": O.num_threads(), "kind": "port",
               "sample": f"one full {args.config} frame via oracle.render (C restatement of "
                         "_kernels.march + block prep, OpenMP over pixels)",
               "samples_taken": r.samples_taken}
    if rank != 0:
        if world > 1:
            import torch.distributed as dist

            dist.destroy_process_group()
        return
    line = {
        "metric": "frames/sec", "value": fps, "unit": "frames/s", "n_gpus": world,
        "steps": args.steps, "warmup": max(args.warmup, 3), "ms_per_step": total_ms / args.steps,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (torso phantom generated on the device, bit-identical to the reference's)",
        "samples_per_sec": taken / (total_ms / args.steps / 1e3), "samples_taken": taken,
        "samples_skipped": st["samples_skipped"],
        "shaded_samples": shaded, "interpolated_samples": st.get("interpolated"),
        "march_iterations": st.get("march_iterations"),
        "config": bench_config(args, cfg),
        "parallelism": (f"sort-first x{world} ({args.dist_backend}, {transport})" if world > 1
                        else "single GPU"),
        "l2": "flushed between steps (512 MiB write, then 512 MiB read)",
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak, "peak_source": peak_kind,
                     "traffic": committed_traffic(args.config),
                     "kernel": "raycast_post_kernel + raycast_heavy_kernel (one vr_render launch pair)",
                     "kernel_ms": kern_s * 1e3,
                     "bytes_model": (f"gathered: (interpolations + 6*shaded)*{b_sample} + iterations*32 "
                                     "+ W*H*4 per launch (taps mostly served from L1; see profiles/ "
                                     "for DRAM bytes and issue utilisation)"),
                     "survey_model": {"bytes": survey_bytes, "achieved": survey_bytes / kern_s / 1e9,
                                      "formula": f"taken*{b_sample} + shaded*{b_grad} + W*H*4 (SURVEY 8(d))"},
                     "ncu": committed_ncu(args.config)},
        "clocks": clocks.summary(),
        "gpu_launches": (launches_per_frame(settings) + (2 if measure else 0)) * args.steps,
        "e2e": e2e,
        "cpu_baseline": cpu,
    }
    print(json.dumps(line), flush=True)
    if world > 1:
        import torch.distributed as dist

        dist.destroy_process_group()


def run_k4(args):
    """--config k4: K4 alone.  One step = whole-volume threshold measure (V
    count + isosurface S) + 360 probe balls, L2 flushed before each step.  The
    roofline is the whole-volume pass (HBM-bound: 2 bytes per voxel), timed
    per kernel with CUDA events on the launching stream; the count-only pass
    (vr_threshold_count) is reported beside it."""
    import ctypes

    import numpy as np
    import torch

    import paper_2005_01442_b200 as vr
    from paper_2005_01442_b200 import _lib

    rank, world, _ = dist_setup(args.gpus, args.dist_backend)
    if world == 1:
        torch.cuda.set_device(0)
    dev = torch.device("cuda", torch.cuda.current_device())
    c = K4_CONFIG
    spacing = (1.0, 1.0, 1.0)
    dvol = vr.device_phantom("torso", c["dims"], spacing, device=dev.index)
    nx, ny, nz = dvol.dims
    extent = ((nx - 1) * spacing[0], (ny - 1) * spacing[1], (nz - 1) * spacing[2])
    nb = c["balls"]
    centres = torch.from_numpy(ball_centres(extent, nb)).to(dev)
    radii = torch.full((nb,), float(c["radius"]), dtype=torch.float64, device=dev)
    out = torch.zeros(2 + 2 * nb, dtype=torch.int64, device=dev)
    cnt = torch.zeros(1, dtype=torch.int64, device=dev)
    L = _lib.load()
    stream = torch.cuda.current_stream(dev)
    s = _lib.ptr_stream(stream)
    thr = int(c["threshold"])
    flush = torch.empty(L2_FLUSH_BYTES, dtype=torch.uint8, device=dev)
    # a read pass after the flush's writes: L2 then holds clean lines, so the
    # timed kernels' reads do not also pay the flush's write-backs
    clean = torch.ones(L2_FLUSH_BYTES // 4, dtype=torch.int32, device=dev)
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(6)]

    def step(timed):
        if timed:
            ev[0].record(stream)
        _lib.check(L.vr_threshold_measure(dvol.handle, thr, _lib.ptr(out), s))
        if timed:
            ev[1].record(stream)
        _lib.check(L.vr_ball_measure(dvol.handle, thr, _lib.ptr(centres), _lib.ptr(radii), nb,
                                     ctypes.c_void_p(out.data_ptr() + 16),
                                     ctypes.c_void_p(out.data_ptr() + 16 + 8 * nb), s))
        if timed:
            ev[2].record(stream)

    for _ in range(max(args.warmup, 3)):
        step(False)
    torch.cuda.synchronize()
    t_step, t_whole, t_balls, t_count = [], [], [], []
    with ClockSampler(dev.index) as clocks:
        for _ in range(args.steps):
            flush.fill_(1)
            clean.amax()
            step(True)
            flush.fill_(2)
            cnt.zero_()
            clean.amax()
            ev[3].record(stream)
            _lib.check(L.vr_threshold_count(dvol.handle, thr, _lib.ptr(cnt), s))
            ev[4].record(stream)
            ev[4].synchronize()
            t_whole.append(ev[0].elapsed_time(ev[1]))
            t_balls.append(ev[1].elapsed_time(ev[2]))
            t_step.append(ev[0].elapsed_time(ev[2]))
            t_count.append(ev[3].elapsed_time(ev[4]))
    res = out.cpu().numpy()
    count, area_fx = int(res[0]), int(res[1])
    nvox = nx * ny * nz
    peak, peak_kind = measured_peak()
    whole_ms = float(np.mean(t_whole))
    count_ms = float(np.mean(t_count))
    achieved = 2 * nvox / (whole_ms / 1e3) / 1e9
    count_gbs = 2 * nvox / (count_ms / 1e3) / 1e9
    total_ms = sum(t_step)
    cpu = None
    if not args.no_cpu_baseline:
        from oracle import oracle as O

        values = dvol.download()
        t0 = time.perf_counter()
        want = O.threshold_measure(values, spacing, thr)
        t_cpu = time.perf_counter() - t0
        assert want == (count, area_fx), (want, count, area_fx)
        cpu = {"value": 1.0 / t_cpu, "unit": "whole-volume measures/s", "cores": O.num_threads(), "kind": "port",
               "sample": "one whole-volume measure (V count + marching-tetrahedra S) via oracle.threshold_measure "
                         "(equal to the GPU's, checked)"}
    line = {
        "metric": "method-of-spheres measures/sec", "value": args.steps / (total_ms / 1e3),
        "unit": "measures/s", "n_gpus": 1, "steps": args.steps, "warmup": max(args.warmup, 3),
        "ms_per_step": total_ms / args.steps, "higher_is_better": True, "scaling": "replicas",
        "vs_baseline": None, "dtype": "i16 -> u64 (S in f64, fixed-point sum)", "data": "synthetic",
        "config": {"workload": "k4", "desc": c["desc"], "volume": list(c["dims"]), "balls": nb,
                   "radius_mm": c["radius"], "threshold": thr},
        "l2": "flushed before every timed kernel (512 MiB write, then 512 MiB read)",
        "result": {"count": count, "V_mm3": count * 1.0, "S_mm2": area_fx / 2.0 ** 24,
                   "svr_per_mm": (area_fx / 2.0 ** 24) / count if count else None},
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                     "peak_source": peak_kind, "traffic": None,
                     "kernel": "threshold_measure_kernel (whole volume: V count + isosurface S)",
                     "kernel_ms": whole_ms, "bytes_model": "2 B per voxel (int16 read once)",
                     "count_only": {"kernel": "threshold_kernel (vr_threshold_count)", "kernel_ms": count_ms,
                                    "achieved": count_gbs, "frac": count_gbs / peak},
                     "balls_ms": float(np.mean(t_balls))},
        "clocks": clocks.summary(),
        "gpu_launches": 3 * args.steps,
        "e2e": None,
        "cpu_baseline": cpu,
    }
    print(json.dumps(line), flush=True)


def main():
    args = parse()
    if args.config == "k4":
        if args.impl == "reference":
            print(json.dumps({"impl": "reference", "unavailable": "k4 is an auxiliary line; the reference arm "
                              "times the headline configs"}))
            return
        run_k4(args)
    elif args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
