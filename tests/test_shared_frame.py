"""Sort-first rendering into one shared frame (no gather): the kernels store
each rank's interleaved cells at their frame positions (interleave_frame).

Single-process: all ranks' cell sets rendered into one buffer == the frame.
Two processes on one GPU (gloo for the barrier): rank 1 maps rank 0's frame
through CUDA IPC -- the same mapping peer GPUs use over NVLink -- and both
store into it; rank 0's frame == the single-GPU frame.  The ranks' kernels
never wait on each other (host barrier only).
"""

from __future__ import annotations

import os
import socket

import numpy as np
import pytest


def _scene(vr):
    vol = vr.generate_phantom("torso", (48, 44, 40))
    ext = vol.extent_mm
    c = tuple(0.5 * e for e in ext)
    cam = vr.Camera(position=(c[0] + 2.2 * max(ext), c[1] + 7.0, c[2] - 5.0), look_at=c, width=72, height=52)
    st = vr.RenderSettings(interpolation="tricubic", use_blocks=True, block_size=16)
    return vol, cam, vr.get_preset("bone"), st


@pytest.mark.gpu
@pytest.mark.parametrize("n", [2, 3, 8])
def test_interleaved_cells_at_frame_positions(n):
    import torch

    import paper_2005_01442_b200 as vr

    vol, cam, tf, st = _scene(vr)
    ref = vr.render(vol, cam, tf, st).pixels
    frame = torch.zeros((cam.height, cam.width, 4), dtype=torch.uint8, device="cuda")
    taken = 0
    for k in range(n):
        r = vr.Renderer(vol, cam, tf, st, interleave=(n, k), frame_out=frame)
        r.render_async()
        taken += r.stats()["samples_taken"]
    np.testing.assert_array_equal(frame.cpu().numpy(), ref)
    assert taken == vr.render(vol, cam, tf, st).stats.samples_taken


def _other_view(vr, vol, cam):
    ext = vol.extent_mm
    c = tuple(0.5 * e for e in ext)
    return vr.Camera(position=(c[0], c[1] - 2.2 * max(ext), c[2] + 9.0), look_at=c, width=cam.width,
                     height=cam.height)


def _worker(rank, world, port, out):
    import torch
    import torch.distributed as dist

    import paper_2005_01442_b200 as vr
    from paper_2005_01442_b200.distributed import SharedFrame, render_sharded

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    vol, cam, tf, st = _scene(vr)
    shared = SharedFrame(cam.height, cam.width)
    frame, stats = render_sharded(vol, cam, tf, st, shared=shared)
    # a different view straight after: the peers' stores of frame 2 must not
    # land in rank 0's frame before rank 0 has read frame 1 (write-after-read)
    frame2, _ = render_sharded(vol, _other_view(vr, vol, cam), tf, st, shared=shared)
    frame3, _ = render_sharded(vol, cam, tf, st, shared=shared)
    if rank == 0:
        np.save(out, np.stack([frame, frame2, frame3]))
        np.save(out + ".stats.npy", np.array(stats, dtype=np.int64))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.gpu
def test_two_processes_store_into_rank0_frame(tmp_path):
    import torch.multiprocessing as mp

    import paper_2005_01442_b200 as vr

    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    out = str(tmp_path / "frame.npy")
    mp.spawn(_worker, args=(2, port, out), nprocs=2, join=True)
    vol, cam, tf, st = _scene(vr)
    ref = vr.render(vol, cam, tf, st)
    frames = np.load(out)
    np.testing.assert_array_equal(frames[0], ref.pixels)
    np.testing.assert_array_equal(frames[1], vr.render(vol, _other_view(vr, vol, cam), tf, st).pixels)
    np.testing.assert_array_equal(frames[2], ref.pixels)
    stats = np.load(out + ".stats.npy")
    assert int(stats[0]) == ref.stats.samples_taken and int(stats[1]) == ref.stats.samples_skipped
