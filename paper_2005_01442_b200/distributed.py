"""Sort-first multi-GPU rendering: interleaved 16x8 cells per rank, one gather
(or none: the cells stored straight into rank 0's frame over NVLink).

The frame is cut into 16x8-pixel cells numbered row-major; rank k of n renders
cells c with c % n == k (the kernel's interleave mode, include/voxelray_b200.h)
into a packed buffer of ceil(ncells / n) cells, identical in size on every
rank.  The volume is replicated (one copy per GPU; 1 GiB at the largest
config vs 180 GB of HBM).  The only exchange is the gather of the packed
uint8 cells to rank 0 (NCCL over NVLink on the GPU box, gloo in the CPU
tests), where ``unpack_cells`` restores the row-major frame.  Pixels are
independent (reference SPEC.md:354, _kernels.py:13-14), so the gathered frame
equals the single-GPU frame bit for bit.

``SharedFrame`` fuses the exchange into the render: rank 0's frame is mapped
into every rank (CUDA IPC, peer access over NVLink/NVSwitch) and each rank's
ray-cast kernels store their cells at their frame positions
(``interleave_frame``), so after a barrier rank 0 holds the frame with no
gather, no packing and no unpack pass.
"""

from __future__ import annotations

import math

CELL_W, CELL_H = 16, 8


def cell_grid(width: int, height: int):
    """(cells_x, cells_y) covering a width x height rectangle."""
    return math.ceil(width / CELL_W), math.ceil(height / CELL_H)


def cells_per_rank(width: int, height: int, n: int) -> int:
    cx, cy = cell_grid(width, height)
    return math.ceil(cx * cy / n)


def rank_cells(width: int, height: int, n: int, k: int) -> list[int]:
    """Cell indices rendered by rank k of n, in packed order."""
    cx, cy = cell_grid(width, height)
    return list(range(k, cx * cy, n))


def cell_rect(width: int, height: int, c: int):
    """(x0, y0, w, h) of cell c clipped to the frame."""
    cx, _ = cell_grid(width, height)
    x0, y0 = (c % cx) * CELL_W, (c // cx) * CELL_H
    return x0, y0, min(CELL_W, width - x0), min(CELL_H, height - y0)


def pack_cells(frame, n: int, k: int):
    """What rank k's packed buffer holds for a (H, W, C) frame (torch or numpy):
    shape (cells_per_rank * 128, C), cells beyond the frame left zero."""
    H, W, C = frame.shape
    slots = cells_per_rank(W, H, n)
    out = frame.new_zeros((slots * CELL_H * CELL_W, C)) if hasattr(frame, "new_zeros") else \
        __import__("numpy").zeros((slots * CELL_H * CELL_W, C), dtype=frame.dtype)
    for s, c in enumerate(rank_cells(W, H, n, k)):
        x0, y0, w, h = cell_rect(W, H, c)
        block = out[s * 128:(s + 1) * 128].reshape(CELL_H, CELL_W, C)
        block[:h, :w] = frame[y0:y0 + h, x0:x0 + w]
    return out


def unpack_cells(gathered, width: int, height: int):
    """Reassemble the frame from the n packed rank buffers.

    gathered: torch tensor (n, slots * 128, C) in rank order.  Returns (H, W, C).
    """
    n, per, C = gathered.shape
    slots = per // (CELL_W * CELL_H)
    cx, cy = cell_grid(width, height)
    # slot s of rank k holds cell s * n + k
    cells = gathered.reshape(n, slots, CELL_H, CELL_W, C).transpose(0, 1).reshape(n * slots, CELL_H, CELL_W, C)
    cells = cells[: cx * cy].reshape(cy, cx, CELL_H, CELL_W, C)
    frame = cells.permute(0, 2, 1, 3, 4).reshape(cy * CELL_H, cx * CELL_W, C)
    return frame[:height, :width]


def gather_frame(packed, width: int, height: int, group=None):
    """Gather every rank's packed cells to rank 0 and unpack there.

    packed: (slots * 128, C) tensor on this rank's device (CUDA for NCCL, CPU
    for gloo).  Returns the (H, W, C) frame on rank 0, None elsewhere.
    """
    import torch
    import torch.distributed as dist

    n = dist.get_world_size(group)
    rank = dist.get_rank(group)
    if n == 1:
        return unpack_cells(packed.unsqueeze(0), width, height)
    if rank == 0:
        bufs = [torch.empty_like(packed) for _ in range(n)]
        dist.gather(packed, gather_list=bufs, dst=0, group=group)
        return unpack_cells(torch.stack(bufs), width, height)
    dist.gather(packed, gather_list=None, dst=0, group=group)
    return None


class SharedFrame:
    """An (H, W, C) uint8 frame in rank 0's HBM that every rank of ``group``
    can store into.  Collective: every rank constructs it with the same size.
    Rank 0 allocates and exports a CUDA IPC handle (torch.multiprocessing's
    reduction); the others map it and enable peer access from their device.
    ``publish()`` (collective) orders every rank's stores before rank 0 reads.
    """

    def __init__(self, height: int, width: int, channels: int = 4, group=None, device=None):
        import torch
        import torch.distributed as dist
        from torch.multiprocessing.reductions import reduce_tensor

        from . import _lib

        self.group = group
        self.rank = dist.get_rank(group)
        dev = torch.cuda.current_device() if device is None else device
        if self.rank == 0:
            self.frame = torch.zeros((height, width, channels), dtype=torch.uint8, device=dev)
            msg = [reduce_tensor(self.frame)]
        else:
            msg = [None]
        dist.broadcast_object_list(msg, src=0, group=group)
        if self.rank != 0:
            rebuild, args = msg[0]
            self.frame = rebuild(*args)
            owner = self.frame.device.index
            if owner != dev:
                _lib.check(_lib.load().vr_enable_peer_access(dev, owner))

    def acquire(self):
        """Collective, before a frame's stores: rank 0 has finished reading the
        previous frame (its ``frame.cpu()`` returned before it entered this
        barrier), so no rank's next-frame stores can overwrite cells rank 0 is
        still copying (write-after-read across frames)."""
        import torch.distributed as dist

        dist.barrier(group=self.group)

    def publish(self):
        """Every rank's stores into the frame are complete and visible to rank 0."""
        import torch
        import torch.distributed as dist

        torch.cuda.synchronize()
        dist.barrier(group=self.group)


class ShardedRenderer:
    """One rank's share of sort-first multi-GPU rendering, kept across frames:
    the volume, block grid, LUT and output buffers stay resident (one
    ``Renderer`` per rank), so a frame is one camera update plus one
    ``vr_render`` call -- no allocation and no table upload per frame.

    ``render_async(camera)`` enqueues the frame on the current stream.  With
    the NCCL gather (``shared=None``) the exchange is stream-ordered as well:
    ``gather_async()`` enqueues ``dist.gather`` of the packed cells and the
    unpack on rank 0, and nothing in the frame waits on the host.  With a
    ``SharedFrame`` the cells land in rank 0's frame directly; ``gather_async()`` then
    publishes it and ``render_async`` first waits until rank 0 has read the
    previous frame (host barriers: the CUDA-IPC transport's only ordering).
    """

    def __init__(self, volume, camera, tf, settings, *, group=None, device=None,
                 shared: SharedFrame | None = None):
        import torch
        import torch.distributed as dist

        from .render import Renderer

        self.group = group
        self.n = dist.get_world_size(group) if dist.is_initialized() else 1
        self.k = dist.get_rank(group) if dist.is_initialized() else 0
        self.device = torch.cuda.current_device() if device is None else device
        self.shared = shared if self.n > 1 else None
        self.width, self.height = camera.width, camera.height
        self.renderer = Renderer(volume, camera, tf, settings, device=self.device,
                                 interleave=(self.n, self.k) if self.n > 1 else None,
                                 frame_out=self.shared.frame if self.shared is not None else None)

    def render_async(self, camera=None):
        if camera is not None:
            if (camera.width, camera.height) != (self.width, self.height):
                raise ValueError("ShardedRenderer: camera size differs from the one it was built for")
            self.renderer.set_camera(camera)
        if self.shared is not None:
            self.shared.acquire()
        self.renderer.render_async()

    def gather_async(self):
        """Stream-ordered exchange: rank 0 gets the (H, W, 4) device frame."""
        if self.shared is not None:
            self.shared.publish()
            return self.shared.frame if self.k == 0 else None
        if self.n == 1:
            return self.renderer.pixels
        return gather_frame(self.renderer.pixels.reshape(-1, 4), self.width, self.height, self.group)

    def stats(self):
        """[samples_taken, samples_skipped] summed over ranks (synchronising)."""
        import torch.distributed as dist

        totals = self.renderer.totals[:2].clone()
        if self.n > 1:
            if dist.get_backend(self.group) == "gloo":
                totals = totals.cpu()
            dist.all_reduce(totals, group=self.group)
        return totals.cpu().tolist()


_SHARDED: dict = {}


def render_sharded(volume, camera, tf, settings, *, group=None, device=None, shared: SharedFrame | None = None):
    """Multi-GPU render of one frame: every rank calls this with the same
    arguments; rank 0 returns the (H, W, 4) uint8 frame as a host array and
    the summed stats, other ranks return (None, stats).  With ``shared`` (a
    SharedFrame of the frame's size) the cells are stored straight into rank
    0's frame instead of gathered.  The per-rank renderer is cached across
    calls for the same volume, TF, settings, frame size and transport."""
    import torch

    dev = torch.cuda.current_device() if device is None else device
    key = (id(volume), id(tf), settings, camera.width, camera.height, id(group), dev, id(shared))
    sr = _SHARDED.get(key)
    if sr is None or sr[0] is not volume or sr[1] is not tf:
        if len(_SHARDED) > 8:
            _SHARDED.clear()
        sr = (volume, tf, ShardedRenderer(volume, camera, tf, settings, group=group, device=dev, shared=shared))
        _SHARDED[key] = sr
    r = sr[2]
    r.render_async(camera)
    frame = r.gather_async()
    stats = r.stats()
    if frame is None:
        return None, stats
    return frame.cpu().numpy(), stats
