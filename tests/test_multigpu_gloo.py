"""Sort-first multi-GPU path on CPU: cell interleave, packing, gather, unpack.

Each rank renders its interleaved 16x8 cells with the CPU oracle (one tile
render per cell), packs them exactly as the kernel's interleave mode does,
and gathers to rank 0 over gloo; rank 0 unpacks and must obtain the
single-process frame bit for bit (pixel independence, reference SPEC.md:354).
The device kernels are covered by tests/test_gpu_parity.py.
"""

from __future__ import annotations

import os
import socket
from types import SimpleNamespace

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from conftest import DEFAULT_SETTINGS, tf_arrays
from paper_2005_01442_b200 import distributed as D


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _scene():
    from oracle import oracle as O

    vals = O.phantom("torso", (40, 36, 32))
    ext = (39.0, 35.0, 31.0)
    c = tuple(0.5 * e for e in ext)
    cam = SimpleNamespace(position=[c[0] + 2.2 * 39.0, c[1], c[2]], look_at=list(c), up=[0.0, 0.0, 1.0],
                          vertical_fov_deg=30.0, width=45, height=27)
    s = dict(DEFAULT_SETTINGS, interpolation="tricubic", use_blocks=True, block_size=12, overlap=3)
    return vals, cam, SimpleNamespace(**s)


def _render_cells(rank, world):
    from oracle import oracle as O

    vals, cam, s = _scene()
    v, col, dom = tf_arrays({"preset": "bone"})
    W, H = cam.width, cam.height
    packed = np.zeros((D.cells_per_rank(W, H, world) * 128, 4), dtype=np.uint8)
    taken = 0
    for slot, c in enumerate(D.rank_cells(W, H, world, rank)):
        x0, y0, w, h = D.cell_rect(W, H, c)
        r = O.render(vals, (1.0, 1.0, 1.0), cam, v, col, dom, s, tile=(x0, y0, w, h))
        cell = packed[slot * 128:(slot + 1) * 128].reshape(8, 16, 4)
        cell[:h, :w] = r.pixels
        taken += r.samples_taken
    return packed, taken


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        packed, taken = _render_cells(rank, world)
        _, cam, _ = _scene()
        frame = D.gather_frame(torch.from_numpy(packed), cam.width, cam.height)
        t = torch.tensor([taken], dtype=torch.int64)
        dist.all_reduce(t)
        if rank == 0:
            q.put((frame.numpy(), int(t.item())))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_gathered_frame_equals_single_process(world):
    from oracle import oracle as O

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    frame, taken = q.get(timeout=300)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    vals, cam, s = _scene()
    v, col, dom = tf_arrays({"preset": "bone"})
    full = O.render(vals, (1.0, 1.0, 1.0), cam, v, col, dom, s)
    assert np.array_equal(frame, full.pixels)
    assert taken == full.samples_taken


@pytest.mark.parametrize("W,H,n", [(1024, 1024, 8), (45, 27, 2), (45, 27, 3), (17, 9, 5), (16, 8, 1)])
def test_pack_unpack_round_trip(W, H, n):
    rng = np.random.default_rng(W * H + n)
    frame = torch.from_numpy(rng.integers(0, 255, size=(H, W, 4), dtype=np.uint8))
    packed = torch.stack([D.pack_cells(frame, n, k) for k in range(n)])
    assert packed.shape[1] == D.cells_per_rank(W, H, n) * 128
    assert torch.equal(D.unpack_cells(packed, W, H), frame)


def test_cells_partition_the_frame():
    W, H, n = 100, 37, 3
    cx, cy = D.cell_grid(W, H)
    seen = sorted(c for k in range(n) for c in D.rank_cells(W, H, n, k))
    assert seen == list(range(cx * cy))
    # interleaving balances the counts to within one cell
    counts = [len(D.rank_cells(W, H, n, k)) for k in range(n)]
    assert max(counts) - min(counts) <= 1
