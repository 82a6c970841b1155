"""CPU checks of the drop-in boundary: the C-ABI library loads, exports every
entry point include/tetvol_b200.h declares, validates arguments with the
reference's rules before touching a device, and fails loudly (no CPU fallback)
when there is no GPU."""
import ctypes
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "tetvol_b200.h")
HEADERS = [os.path.join(ROOT, "include", h) for h in ("tetvol_b200.h", "tetvol_b200_diag.h")]


def declared_symbols():
    out = set()
    for h in HEADERS:
        text = open(h).read()
        text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
        out |= set(re.findall(r"\b(tv_[a-z_0-9]+)\s*\(", text))
    return sorted(out)


def test_library_exports_every_declared_symbol():
    import paper_2506_11510_b200 as tv

    lib = ctypes.CDLL(tv.LIB_PATH)
    syms = declared_symbols()
    assert len(syms) >= 22
    missing = [s for s in syms if not hasattr(lib, s)]
    assert not missing, missing
    assert "sm_100a" in tv.version()


def test_cuda_objects_target_sm100a():
    """The shipped .so carries sm_100a SASS (cuobjdump lists the ELF arch)."""
    import shutil
    import subprocess

    import paper_2506_11510_b200 as tv

    if not shutil.which("cuobjdump"):
        pytest.skip("cuobjdump not available")
    out = subprocess.run(["cuobjdump", "--list-elf", tv.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_config_and_camera_errors_before_device():
    """RenderConfig::validate / BuildConfig::validate / camera ctor rules
    (tracer.cpp:131-141, builder.cpp:12-17, camera.cpp:15-20) are enforced
    host-side with the reference's messages."""
    import paper_2506_11510_b200 as tv

    vol = np.zeros((4, 4, 4), np.float32)
    with pytest.raises(tv.ConfigError, match="maxLevel out of range"):
        tv.build_adaptive_grid(vol, tv.BuildConfig(max_level=49))
    with pytest.raises(tv.ConfigError, match="pixelThreshold"):
        tv.build_adaptive_grid(vol, tv.BuildConfig(pixel_threshold=0.0))
    with pytest.raises(tv.ConfigError, match="useCamera set but no camera given"):
        tv.build_adaptive_grid(vol, tv.BuildConfig(use_camera=True))
    with pytest.raises(tv.CameraError, match="vfov"):
        tv.build_adaptive_grid(vol, tv.BuildConfig(use_camera=True), tv.PinholeCamera(vfov_degrees=0.0))
    with pytest.raises(tv.CameraError, match="image dimensions"):
        tv.build_adaptive_grid(vol, tv.BuildConfig(use_camera=True), tv.PinholeCamera(width=0))


def test_no_cpu_fallback_without_gpu():
    import paper_2506_11510_b200 as tv

    if tv.device_count() > 0:
        pytest.skip("a GPU is present")
    tv.build_trim()
    assert tv.build_scratch_bytes() == 0
    vol = np.zeros((4, 4, 4), np.float32)
    with pytest.raises(tv.CudaError):
        tv.build_adaptive_grid(vol, tv.BuildConfig())
    v = np.zeros((15, 3), np.uint32)
    t = np.zeros(24, tv.TET_DTYPE)
    t["children"] = 0xFFFFFFFF
    with pytest.raises(tv.CudaError):
        tv.TetGrid.upload(v, t, np.arange(24, dtype=np.uint32))


def test_upload_rejects_corrupt_pools_like_load_grid():
    """builder.cpp:253-285 range checks (FormatError in the reference) -> GridError."""
    import oracle as O
    import paper_2506_11510_b200 as tv

    p = O.init_roots(O.c_oracle()).pools()
    bad = p.tets.copy().view(tv.TET_DTYPE)
    bad["verts"][3, 1] = 999
    with pytest.raises(tv.GridError, match="vertex id out of range"):
        tv.TetGrid.upload(p.vq, bad, p.roots)
    bad = p.tets.copy().view(tv.TET_DTYPE)
    bad["normal_ids"][0, 2] = 18
    with pytest.raises(tv.GridError, match="face normal id out of range"):
        tv.TetGrid.upload(p.vq, bad, p.roots)
    with pytest.raises(ValueError):
        tv.TetGrid.upload(p.vq, p.tets.view(tv.TET_DTYPE), p.roots[:23])


def test_tgrid_header_errors_before_device(tmp_path):
    """load_grid's header checks (builder.cpp:240-247) run before any device work."""
    import paper_2506_11510_b200 as tv

    cases = {"magic": b"TGRX" + bytes(12), "version": b"TGRD" + (2).to_bytes(4, "little") + bytes(8),
             "count": b"TGRD" + (1).to_bytes(4, "little") + (7).to_bytes(8, "little"), "empty": b""}
    want = {"magic": "not a TGRD file: ", "version": "unsupported TGRD version", "count": "bad vertex count",
            "empty": "not a TGRD file: "}
    for k, raw in cases.items():
        fn = tmp_path / f"{k}.tgrid"
        fn.write_bytes(raw)
        with pytest.raises(tv.FormatError) as e:
            tv.load_grid(fn)
        assert str(e.value).startswith(want[k])
    with pytest.raises(tv.IoError, match="cannot open"):
        tv.load_grid(tmp_path / "missing.tgrid")
    if tv.device_count() == 0:  # a valid file still needs the device: no CPU fallback
        import oracle as O
        from oracle.tgrid import tgrid_bytes

        p = O.init_roots(O.c_oracle()).pools()
        fn = tmp_path / "roots.tgrid"
        fn.write_bytes(tgrid_bytes(p.vq, p.tets, p.roots))
        with pytest.raises(tv.CudaError):
            tv.load_grid(fn)


def test_spot_rays_match_reference_cli():
    """cmd_validate's spot-check rays are generated on the host: bit-identical to cli.cpp:552-569."""
    import ctypes as C

    import oracle as O
    import paper_2506_11510_b200 as tv

    ref = O.ref_oracle()
    if ref is None:
        pytest.skip("oracle/_ref not built")
    for seed in (0, 7, 2**63 + 5):
        mine = tv.spot_rays(seed, 300)
        want = np.zeros((300, 8))
        ref.fn("spot_rays")(seed, 300, want.ctypes.data_as(C.POINTER(C.c_double)))
        assert np.array_equal(mine.view(np.uint64), want.view(np.uint64))


def test_ipc_and_diag_entry_points_fail_loudly_without_a_gpu():
    """The peer-write helpers and the diagnostic validate their arguments and,
    without a device, return TV_ERR_CUDA / TV_ERR_ARG instead of doing anything."""
    import ctypes as C

    import paper_2506_11510_b200 as tv

    lib = tv._lib
    h = (C.c_uint8 * 64)()
    off = C.c_uint64()
    assert lib.tv_ipc_export(None, h, C.byref(off)) != 0  # null pointer
    out = C.c_void_p()
    rc = lib.tv_ipc_open(h, 0, 0, C.byref(out))
    if tv.device_count() == 0:
        assert rc == 6  # TV_ERR_CUDA: no device, no fallback
    assert lib.tv_ipc_close(None, 0) == 0
    res = (C.c_double * 6)()
    assert lib.tv_diag_gather_ceiling(None, None, None, 1, res) == 8  # TV_ERR_ARG
