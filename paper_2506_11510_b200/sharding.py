"""Image-space sharding for multi-GPU rendering.

The frame is cut into 16x16 tiles, numbered row-major; tile t belongs to rank
t % n_ranks. Every rank renders its tiles with the reference's per-pixel sample
order, so the assembled frame is bit-identical for any rank count. After the
render each rank packs its tiles into an equal-size block (ceil(tiles /
n_ranks) * 256 pixel slots), one all-gather moves the blocks, and every block
is scattered back. This module is the host-side mirror of the device pack /
unpack kernels (csrc/tv_tiles.cu), used by bench.py and by the CPU gloo tests.

PeerFrame is the fused alternative: rank 0's full-frame accumulators are mapped
into every rank (CUDA IPC), each rank's accumulate kernel stores its pixels
straight into them over NVLink, and a stream-ordered one-word all-reduce is the
only collective (a completion barrier, no pixel data).
"""
from __future__ import annotations

import numpy as np

TILE = 16


def n_tiles(width: int, height: int) -> tuple[int, int]:
    return (width + TILE - 1) // TILE, (height + TILE - 1) // TILE


def slots_per_rank(width: int, height: int, n_ranks: int) -> int:
    tx, ty = n_tiles(width, height)
    return (tx * ty + n_ranks - 1) // n_ranks * TILE * TILE


def rank_tiles(width: int, height: int, rank: int, n_ranks: int) -> np.ndarray:
    tx, ty = n_tiles(width, height)
    return np.arange(rank, tx * ty, n_ranks)


def slot_pixels(width: int, height: int, rank: int, n_ranks: int) -> np.ndarray:
    """Flat pixel index of every packed slot of `rank` (-1 for padding slots)."""
    tx, ty = n_tiles(width, height)
    slots = slots_per_rank(width, height, n_ranks)
    k = np.arange(slots) // (TILE * TILE)
    local = np.arange(slots) % (TILE * TILE)
    t = rank + k * n_ranks
    px = (t % tx) * TILE + local % TILE
    py = (t // tx) * TILE + local // TILE
    ok = (t < tx * ty) & (px < width) & (py < height)
    return np.where(ok, py * width + px, -1)


def pack(frame: np.ndarray, width: int, height: int, rank: int, n_ranks: int) -> np.ndarray:
    """frame: (W*H, E) -> (slots, E), zero in padding slots."""
    pix = slot_pixels(width, height, rank, n_ranks)
    out = np.zeros((len(pix),) + frame.shape[1:], frame.dtype)
    out[pix >= 0] = frame[pix[pix >= 0]]
    return out


def unpack(packed: np.ndarray, frame: np.ndarray, width: int, height: int, rank: int, n_ranks: int) -> None:
    pix = slot_pixels(width, height, rank, n_ranks)
    frame[pix[pix >= 0]] = packed[pix >= 0]


def owner_map(width: int, height: int, n_ranks: int) -> np.ndarray:
    """(H, W) rank owning each pixel."""
    tx, _ = n_tiles(width, height)
    y, x = np.mgrid[0:height, 0:width]
    return ((y // TILE) * tx + x // TILE) % n_ranks


class PeerFrame:
    """Rank 0's frame accumulators (sum, sum_sq: 3 doubles per pixel; counts: u32
    per pixel), mapped on every rank of `group` through tv_ipc_export /
    tv_ipc_open. `ptrs` are this rank's device pointers to them."""

    def __init__(self, width: int, height: int, rank: int, device: int, group=None):
        import torch
        import torch.distributed as dist

        import paper_2506_11510_b200 as tv

        npx = width * height
        self.rank, self.device, self.mapped = rank, device, []
        self.local = None
        handles = [None, None, None]
        if rank == 0:
            self.local = (torch.zeros(npx * 3, dtype=torch.float64, device=f"cuda:{device}"),
                          torch.zeros(npx * 3, dtype=torch.float64, device=f"cuda:{device}"),
                          torch.zeros(npx, dtype=torch.int32, device=f"cuda:{device}"))
            handles = [tv.ipc_export(t.data_ptr()) for t in self.local]
        box = [handles]
        dist.broadcast_object_list(box, src=0, group=group)
        if rank == 0:
            self.ptrs = tuple(t.data_ptr() for t in self.local)
        else:
            self.mapped = [(tv.ipc_open(h, device), h) for h in box[0]]
            self.ptrs = tuple(p for p, _ in self.mapped)

    def close(self):
        import paper_2506_11510_b200 as tv

        for p, h in self.mapped:
            tv.ipc_close(p, h)
        self.mapped = []
