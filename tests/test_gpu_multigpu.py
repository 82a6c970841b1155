"""Multi-GPU frame assembly on one GPU: every rank's share is rendered with
tv_render_tiles, packed with tv_tile_pack into the equal-size block an NCCL
all-gather would move, and all blocks are unpacked with tv_tile_unpack. The
assembled frame must be bit-identical to a single-rank render.
The ranks run one after another, so no kernel waits on another."""
import numpy as np
import pytest

import oracle as O

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("n_ranks", [2, 3, 8])
def test_tile_share_pack_unpack_bit_identical(n_ranks):
    import torch

    import paper_2506_11510_b200 as tv

    g = O.fuzzed(O.c_oracle(), 250, 0x91)
    p = g.pools()
    rng = np.random.default_rng(2)
    lm = p.leaf_mask
    p.tets["density"][lm] = rng.random(lm.sum()).astype(np.float32) * 5
    p.tets["mask"][lm] = 1
    dg = tv.TetGrid.upload(p.vq, p.tets.view(tv.TET_DTYPE), p.roots, p.max_level)
    W, H = 100, 70
    cam = tv.PinholeCamera((0.5, 0.5, -1.4), (0, 0, 1), (0, 1, 0), 50, W, H)
    rc = tv.RenderConfig(spp=3, max_bounces=12, seed=4)
    full = tv.render(dg, cam, rc)

    words = tv.tile_pack_words(W, H, 0, n_ranks, 3)
    gathered = torch.zeros(words * n_ranks, dtype=torch.float64, device="cuda")
    stats = torch.zeros(3, dtype=torch.int64, device="cuda")
    for r in range(n_ranks):  # each "rank" on the same GPU, sequentially
        part = torch.zeros(W * H * 3, dtype=torch.float64, device="cuda")
        tv.render_tiles(dg, cam, rc, r, n_ranks, part.data_ptr(), None, None, stats.data_ptr(), 0)
        tv.tile_pack(part.data_ptr(), gathered[r * words:(r + 1) * words].data_ptr(), W, H, r, n_ranks, 3, 0)
    frame = torch.zeros(W * H * 3, dtype=torch.float64, device="cuda")
    for r in range(n_ranks):
        tv.tile_unpack(gathered[r * words:(r + 1) * words].data_ptr(), frame.data_ptr(), W, H, r, n_ranks, 3, 0)
    torch.cuda.synchronize()
    assert np.array_equal(frame.cpu().numpy().view(np.uint64), full.sum.view(np.uint64))
    assert int(stats[0]) == full.cells_visited


def test_renders_on_different_streams_share_the_workspace_safely():
    """Asynchronous tv_render_tiles calls on two non-blocking streams, with
    different rank splits (so different tile-order tables: 4 and 8 ranks use
    the outer-tiles-last schedule), followed at once by a synchronous tv_render
    on the library's own stream. Every call shares the device workspace; the
    frames must come out exactly as when run one by one (the
    workspace and the tile-order table are stream-ordered)."""
    import torch

    import paper_2506_11510_b200 as tv

    g = O.fuzzed(O.c_oracle(), 250, 0x92)
    p = g.pools()
    rng = np.random.default_rng(3)
    lm = p.leaf_mask
    p.tets["density"][lm] = rng.random(lm.sum()).astype(np.float32) * 6
    p.tets["mask"][lm] = 1
    dg = tv.TetGrid.upload(p.vq, p.tets.view(tv.TET_DTYPE), p.roots, p.max_level)
    W, H = 160, 144
    cam = tv.PinholeCamera((0.5, 0.5, -1.4), (0, 0, 1), (0, 1, 0), 50, W, H)
    rc = tv.RenderConfig(spp=4, max_bounces=16, seed=5)
    splits = [(1, 4), (5, 8), (2, 4), (0, 8)]

    def share(rank, n_ranks, stream):
        part = torch.zeros(W * H * 3, dtype=torch.float64, device="cuda")
        tv.render_tiles(dg, cam, rc, rank, n_ranks, part.data_ptr(), None, None, None, stream)
        return part

    ref = []
    for r, n in splits:  # one at a time
        ref.append(share(r, n, 0).cpu().numpy())
        torch.cuda.synchronize()
    full = tv.render(dg, cam, rc)
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    for _ in range(2):
        parts = [share(r, n, (s1 if i % 2 == 0 else s2).cuda_stream) for i, (r, n) in enumerate(splits)]
        again = tv.render(dg, cam, rc)  # issued while the tile renders may still run
        torch.cuda.synchronize()
        for a, b in zip(parts, ref):
            assert np.array_equal(a.cpu().numpy().view(np.uint64), b.view(np.uint64))
        assert np.array_equal(again.sum.view(np.uint64), full.sum.view(np.uint64))


def test_last_frame_timing_covers_every_batch():
    """last_frame_timing counts every batch of the last frame (it
    used to time only the first 8), and a rank without tiles reports zeros."""
    import torch

    import paper_2506_11510_b200 as tv

    g = O.fuzzed(O.c_oracle(), 120, 0x93)
    p = g.pools()
    dg = tv.TetGrid.upload(p.vq, p.tets.view(tv.TET_DTYPE), p.roots, p.max_level)
    cam = tv.PinholeCamera((0.5, 0.5, -1.4), (0, 0, 1), (0, 1, 0), 50, 64, 64)
    tv.render(dg, cam, tv.RenderConfig(spp=2, max_bounces=4, seed=1))
    t = tv.last_frame_timing(0)
    assert t["launches"] == 3 and t["trace_ms"] > 0
    # 16 tiles; rank 20 of 32 owns none
    buf = torch.zeros(64 * 64 * 3, dtype=torch.float64, device="cuda")
    tv.render_tiles(dg, cam, tv.RenderConfig(spp=2, max_bounces=4, seed=1), 20, 32, buf.data_ptr(), None, None,
                    None, 0)
    torch.cuda.synchronize()
    t = tv.last_frame_timing(0)
    assert t["launches"] == 0 and t["trace_ms"] == 0.0


def _p2p_worker(rank, world, port, q):
    import os

    import torch
    import torch.distributed as dist

    import paper_2506_11510_b200 as tv
    from paper_2506_11510_b200 import sharding

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    g = O.fuzzed(O.c_oracle(), 250, 0x94)
    p = g.pools()
    rng = np.random.default_rng(7)
    lm = p.leaf_mask
    p.tets["density"][lm] = rng.random(lm.sum()).astype(np.float32) * 5
    p.tets["mask"][lm] = 1
    dg = tv.TetGrid.upload(p.vq, p.tets.view(tv.TET_DTYPE), p.roots, p.max_level)
    W, H = 96, 80
    cam = tv.PinholeCamera((0.5, 0.5, -1.4), (0, 0, 1), (0, 1, 0), 50, W, H)
    rc = tv.RenderConfig(spp=3, max_bounces=12, seed=9)
    pf = sharding.PeerFrame(W, H, rank, 0)
    s, sq, cn = pf.ptrs
    tv.render_tiles(dg, cam, rc, rank, world, s, sq, cn, None, 0)  # this rank's pixels into rank 0's HBM
    torch.cuda.synchronize()
    dist.barrier()
    ok = True
    if rank == 0:
        full = tv.render(dg, cam, rc)
        ok = (np.array_equal(pf.local[0].cpu().numpy().view(np.uint64), full.sum.view(np.uint64)) and
              np.array_equal(pf.local[1].cpu().numpy().view(np.uint64), full.sum_sq.view(np.uint64)) and
              np.array_equal(pf.local[2].cpu().numpy().view(np.uint32), full.sample_counts))
    dist.barrier()
    pf.close()
    q.put((rank, bool(ok)))
    dist.destroy_process_group()


def test_peer_frame_direct_writes_two_processes():
    """The fused gather (tv_ipc_export / tv_ipc_open + tv_render_tiles into the
    mapped accumulators): two processes on this one GPU, each renders its tiles
    straight into rank 0's frame buffers; the frame must equal a one-rank
    render bit for bit. The processes only meet at host barriers, so no kernel
    waits on another."""
    import socket

    import torch.multiprocessing as mp

    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_p2p_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    assert all(ok for _, ok in res), res


@pytest.mark.parametrize("peer", ["1", "0"])
def test_render_multi_one_process_bit_identical(peer, monkeypatch):
    """tv_render_multi: one process, one host thread per rank.
    On this one-GPU box every rank's grid lives on device 0 (ranks sharing a
    device run one after another); TV_MULTI_PEER=0 sends every rank > 0
    through the private-frame + host-merge path that devices without peer
    access take. Each way the frame equals tv_render's bit for bit."""
    import paper_2506_11510_b200 as tv

    monkeypatch.setenv("TV_MULTI_PEER", peer)
    g = O.fuzzed(O.c_oracle(), 250, 0x93)
    p = g.pools()
    rng = np.random.default_rng(5)
    lm = p.leaf_mask
    p.tets["density"][lm] = rng.random(lm.sum()).astype(np.float32) * 5
    p.tets["mask"][lm] = 1
    dg = tv.TetGrid.upload(p.vq, p.tets.view(tv.TET_DTYPE), p.roots, p.max_level)
    dg2 = tv.TetGrid.upload(p.vq, p.tets.view(tv.TET_DTYPE), p.roots, p.max_level)
    W, H = 90, 75  # ragged last tile row / column
    cam = tv.PinholeCamera((0.5, 0.5, -1.4), (0, 0, 1), (0, 1, 0), 50, W, H)
    rc = tv.RenderConfig(spp=3, max_bounces=12, seed=6)
    full = tv.render(dg, cam, rc)
    for grids in ([dg], [dg, dg2], [dg, dg2, dg], [dg2] * 5):
        m = tv.render_multi(grids, cam, rc)
        assert np.array_equal(m.sum.view(np.uint64), full.sum.view(np.uint64)), len(grids)
        assert np.array_equal(m.sum_sq.view(np.uint64), full.sum_sq.view(np.uint64)), len(grids)
        assert np.array_equal(m.sample_counts, full.sample_counts), len(grids)
        assert m.cells_visited == full.cells_visited and m.paths_traced == full.paths_traced
        assert m.degenerate_paths == full.degenerate_paths
    with pytest.raises(ValueError, match="at least one grid"):
        tv.render_multi([], cam, rc)
