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
