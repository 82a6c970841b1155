"""Every selectable trace-kernel configuration (register cap, block size,
warp-batching thresholds, path order, locate jump-table resolution, 32-B hot
records; DESIGN.md §4 tuning knobs) renders the
same framebuffer bits: the knobs change scheduling, never results. Each
configuration runs in a subprocess because the library reads the knobs once
per process."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
HERE = os.path.dirname(os.path.abspath(__file__))

CONFIGS = [
    {},
    {"TV_TRACE_MAXREG": "128"},
    {"TV_TRACE_MAXREG": "96"},
    {"TV_TRACE_MAXREG": "80"},
    {"TV_TRACE_THREADS": "64"},
    {"TV_TRACE_THREADS": "64", "TV_TRACE_MAXREG": "88"},
    {"TV_REGEN_MIN": "1", "TV_SCATTER_MIN": "1"},
    {"TV_REGEN_MIN": "32", "TV_SCATTER_MIN": "32"},
    {"TV_ORDER": "0"},
    {"TV_CARVEOUT": "50"},
    {"TV_TILE_ORDER": "2"},
    {"TV_TILE_ORDER": "2", "TV_TILE_RADIUS_PCT": "30"},
    {"TV_TILE_ORDER": "4"},
    {"TV_JUMP_RES": "0"},
    {"TV_JUMP_RES": "32"},
    {"TV_JUMP_RES": "256"},
    {"TV_HOT": "1"},  # 32-B hot records (csrc/tv_grid.cu hot_kernel, exit_face_hot3)
    {"TV_HOT": "1", "TV_TRACE_MAXREG": "96"},
]


def _run(env_extra):
    env = dict(os.environ, **env_extra)
    out = subprocess.run([sys.executable, os.path.join(HERE, "_variant_render.py")], env=env, capture_output=True,
                         text=True, timeout=300)
    assert out.returncode == 0, out.stderr[-2000:]
    return out.stdout.strip().splitlines()[-1]


@pytest.fixture(scope="module")
def reference_line():
    return _run({})


@pytest.mark.parametrize("cfg", CONFIGS[1:], ids=lambda c: ",".join(f"{k}={v}" for k, v in c.items()))
def test_trace_kernel_configuration_is_bit_identical(reference_line, cfg):
    assert _run(cfg) == reference_line
