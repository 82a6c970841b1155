"""Multi-GPU image-space sharding, host side, on CPU.

Each rank owns the interleaved 16x16 tiles t with t % n_ranks == rank, packs
them into an equal-size block, and one all-gather plus unpack rebuilds the
frame on every rank. Run here with world_size 2 over gloo:
every rank renders its OWN pixels with the CPU oracle (row-restricted renders
are cheap at this size), and the assembled frame must be bit-identical to a
single-rank render — the invariant the GPU path also holds for G = 1, 2, 4, 8.
"""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2506_11510_b200 import sharding

W, H, SPP = 50, 37, 3


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _frame(seed=4):
    import oracle as O

    g = O.fuzzed(O.c_oracle(), 120, 0x31)
    p = g.pools()
    rng = np.random.default_rng(seed)
    lm = p.leaf_mask
    p.tets["density"][lm] = rng.random(lm.sum()).astype(np.float32) * 4
    p.tets["mask"][lm] = 1
    g2 = O.from_pools(O.c_oracle(), p)
    cam = O.camera((0.5, 0.5, -1.6), (0, 0, 1), (0, 1, 0), 45, W, H)
    out = g2.render(cam, O.render_cfg(spp=SPP, max_bounces=8, seed=11), 1)
    return out["sum"].reshape(W * H, 3)


def _worker(rank, world, port, q):
    import torch

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    full = _frame()
    mine = sharding.owner_map(W, H, world).reshape(-1) == rank
    local = np.where(mine[:, None], full, 0.0)  # this rank rendered only its tiles
    packed = torch.from_numpy(sharding.pack(local, W, H, rank, world))
    bufs = [torch.zeros_like(packed) for _ in range(world)]
    dist.all_gather(bufs, packed)
    frame = np.zeros_like(full)
    for r in range(world):
        sharding.unpack(bufs[r].numpy(), frame, W, H, r, world)
    q.put((rank, bool(np.array_equal(frame.view(np.uint64), full.view(np.uint64)))))
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2])
def test_tile_gather_gloo_bit_identical(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    assert all(ok for _, ok in res), res


@pytest.mark.parametrize("world", [1, 2, 3, 4, 8])
def test_tiles_partition_the_frame(world):
    own = sharding.owner_map(W, H, world)
    counts = np.bincount(own.reshape(-1), minlength=world)
    assert counts.sum() == W * H
    covered = np.zeros(W * H, int)
    for r in range(world):
        pix = sharding.slot_pixels(W, H, r, world)
        covered[pix[pix >= 0]] += 1
        assert np.all(own.reshape(-1)[pix[pix >= 0]] == r)
    assert np.all(covered == 1)


@pytest.mark.parametrize("world", [1, 2, 4, 8])
def test_pack_size_matches_the_c_abi(world):
    import paper_2506_11510_b200 as tv

    for (w, h) in [(1024, 1024), (50, 37), (16, 16), (17, 1)]:
        for r in range(world):
            assert tv.tile_pack_words(w, h, r, world, 3) == sharding.slots_per_rank(w, h, world) * 3
