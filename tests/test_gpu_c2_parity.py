"""Parity at the bench's full size: the GPU-built cloud
256^3 grid (12.1 M leaves), a 1024 x 1024 x 32 spp frame with up to 64
bounces, checked bit for bit against the C oracle on every 64th image row
(16 rows = 524,288 paths, about 100 M tet steps on the host), plus the frame's
size-independent invariants (sample counts, cells per path)."""
import numpy as np
import pytest

import oracle as O

pytestmark = pytest.mark.gpu

CAM = ((0.5, 0.5, -1.2), (0.0, 0.0, 1.0), (0.0, 1.0, 0.0), 40.0, 1024, 1024)


def test_c2_frame_rows_bit_exact():
    import torch

    import paper_2506_11510_b200 as tv

    assert tv.device_count() >= 1, "no CUDA device: the product has no CPU fallback"
    n = 256
    vol = torch.empty(n ** 3, dtype=torch.float32, device="cuda")
    tv.generate_volume_dev("cloud", n, vol.data_ptr())
    cam = tv.PinholeCamera(*CAM)
    grid, st = tv.build_adaptive_grid_dev(vol.data_ptr(), (n, n, n), tv.BuildConfig(0.15, 24, True, 1.0, 16.0), cam)
    assert st.leaf_count == 12086142  # SURVEY.md 8(d) C2, measured with the oracle
    img = tv.render(grid, cam, tv.RenderConfig(spp=32, max_bounces=64, seed=0))
    assert np.all(img.sample_counts == 32)
    assert img.degenerate_paths == 0
    assert abs(img.cells_visited / img.paths_traced - 196.749) < 0.01  # 196.74 cells/path

    v, t, r = grid.download()
    og = O.from_pools(O.c_oracle(), O.Pools(v, t.view(O.TET_DTYPE), r, 24))
    want = og.render(O.camera(*CAM), O.render_cfg(spp=32, max_bounces=64, seed=0), 0, 64, 7)
    rows = np.arange(7, 1024, 64)
    a = img.sum.reshape(1024, 1024, 3)[rows]
    b = want["sum"].reshape(1024, 1024, 3)[rows]
    assert np.array_equal(a.view(np.uint64), b.view(np.uint64))
    a2 = img.sum_sq.reshape(1024, 1024, 3)[rows]
    b2 = want["sum_sq"].reshape(1024, 1024, 3)[rows]
    assert np.array_equal(a2.view(np.uint64), b2.view(np.uint64))
    grid.close()
