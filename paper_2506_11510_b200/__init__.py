"""tetvol_b200 — B200-native adaptive-tetrahedral-grid volumetric path tracer.

Host-side Python mirror of the reference ``tetvol`` C++ API for the hot path
(``render``, ``build_adaptive_grid``, ``march_segments``, ``PinholeCamera``,
``RenderConfig``, ``BuildConfig``, ``ImageAccumulator``; see
/root/reference/proj/include/tetvol/{tracer,builder,camera,image}.hpp), calling
the sm_100a CUDA library ``_lib/libtetvol_b200.so`` through its C ABI
(``include/tetvol_b200.h``). Errors map to the reference exception names.

There is no CPU fallback: importing this package without the built library
raises ImportError, and every compute call without a CUDA device raises
``CudaError``.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("TETVOL_B200_LIB") or os.path.join(_HERE, "_lib", "libtetvol_b200.so")
NO_TET = 0xFFFFFFFF

if not os.path.exists(LIB_PATH):
    raise ImportError(
        f"{LIB_PATH} is missing: build it with `make -C paper_2506_11510_b200/csrc` "
        "(or __graft_entry__.build()); there is no CPU fallback"
    )
_lib = C.CDLL(LIB_PATH)


# ---------------------------------------------------------------- errors ---
class TetvolError(RuntimeError):
    """Runtime failure (reference: std::runtime_error)."""


class ConfigError(TetvolError):
    """errors.hpp:7-9"""


class CameraError(TetvolError):
    """camera.hpp:10-12"""


class GridError(TetvolError):
    """tet_grid.hpp:24-26"""


class OutsideGrid(GridError):
    """tet_grid.hpp:33-35"""


class CudaError(TetvolError):
    """No usable CUDA device, or a launch/copy failed."""


class FormatError(TetvolError):
    """errors.hpp: malformed .tgrid (builder.cpp:184-293)"""


class IoError(TetvolError):
    """errors.hpp: a file cannot be opened or written"""


class VolumeError(TetvolError):
    """volume.hpp:13-18 (and UnknownChannel)"""


class ImageError(TetvolError):
    """image.hpp: PFM I/O"""


_ERRS = {1: TetvolError, 2: ConfigError, 3: CameraError, 4: GridError, 5: OutsideGrid, 6: CudaError,
         7: CudaError, 8: ValueError, 9: FormatError, 10: IoError, 11: VolumeError,
         12: ImageError}


def _check(rc: int):
    if rc:
        msg = _lib.tv_last_error().decode()
        raise _ERRS.get(rc, TetvolError)(msg)


# ------------------------------------------------------------- C structs ---
class _Camera(C.Structure):
    _fields_ = [("position", C.c_double * 3), ("forward", C.c_double * 3), ("up", C.c_double * 3),
                ("vfov_degrees", C.c_double), ("width", C.c_int32), ("height", C.c_int32),
                ("basis_final", C.c_int32), ("pad", C.c_int32)]


class _RenderConfig(C.Structure):
    _fields_ = [("spp", C.c_int32), ("max_bounces", C.c_int32), ("seed", C.c_uint64), ("hg_g", C.c_double),
                ("default_albedo", C.c_double), ("environment", C.c_double * 3), ("emission_scale", C.c_double),
                ("exposure", C.c_double), ("gamma", C.c_double)]


class _BuildConfig(C.Structure):
    _fields_ = [("variation_threshold", C.c_double), ("max_level", C.c_int32), ("use_camera", C.c_int32),
                ("pixel_threshold", C.c_double), ("density_scale", C.c_double)]


class _BuildStats(C.Structure):
    _fields_ = [("leaf_count", C.c_uint64), ("max_depth", C.c_int32), ("rounds", C.c_int32),
                ("seconds", C.c_double), ("criterion_splits", C.c_uint64), ("propagation_splits", C.c_uint64),
                ("closure_passes", C.c_uint64), ("voxel_visits", C.c_uint64)]


class _RenderStats(C.Structure):
    _fields_ = [("cells_visited", C.c_uint64), ("paths_traced", C.c_uint64), ("degenerate_paths", C.c_uint64),
                ("seconds", C.c_double)]


class _Framebuffer(C.Structure):
    _fields_ = [("sum", C.POINTER(C.c_double)), ("sum_sq", C.POINTER(C.c_double)),
                ("sample_counts", C.POINTER(C.c_uint32))]


class _ValidationReport(C.Structure):
    _fields_ = [("ok", C.c_int32), ("pad", C.c_int32), ("leaf_count", C.c_uint64), ("interior_faces", C.c_uint64),
                ("boundary_faces", C.c_uint64), ("first_violation", C.c_char * 128)]


class _GridInfo(C.Structure):
    _fields_ = [("n_vertices", C.c_uint64), ("n_tets", C.c_uint64), ("n_leaves", C.c_uint64),
                ("n_internal", C.c_uint64), ("max_level", C.c_int32), ("max_depth", C.c_int32),
                ("device", C.c_int32), ("pad", C.c_int32), ("device_bytes", C.c_uint64)]


_P = C.c_void_p
_D = C.POINTER(C.c_double)
_F = C.POINTER(C.c_float)
_U32 = C.POINTER(C.c_uint32)
_U64 = C.POINTER(C.c_uint64)


def _sig(name, res, *args):
    fn = getattr(_lib, name)
    fn.restype = res
    fn.argtypes = list(args)
    return fn


_sig("tv_last_error", C.c_char_p)
_sig("tv_version", C.c_char_p)
_sig("tv_device_count", C.c_int, C.POINTER(C.c_int))
_sig("tv_grid_upload", C.c_int, _P, C.c_uint64, _P, C.c_uint64, _U32, C.c_int32, C.c_int, C.POINTER(_P))
_sig("tv_grid_download", C.c_int, _P, _P, _P, _U32)
_sig("tv_grid_get_info", C.c_int, _P, C.POINTER(_GridInfo))
_sig("tv_grid_free", None, _P)
_sig("tv_grid_save", C.c_int, _P, C.c_char_p)
_sig("tv_grid_validate", C.c_int, _P, _P)
_sig("tv_validate_rays", C.c_int, _P, _P, C.c_int32, C.POINTER(C.c_int32), C.POINTER(C.c_int32))
_sig("tv_validate_spot_rays", C.c_int, C.c_uint64, C.c_int32, _P)
_sig("tv_grid_load", C.c_int, C.c_char_p, C.c_int, C.POINTER(_P))
_sig("tv_build", C.c_int, _F, _F, _F, C.c_int32, C.c_int32, C.c_int32, C.POINTER(_BuildConfig), C.POINTER(_Camera),
     C.c_int, C.POINTER(_P), C.POINTER(_BuildStats))
_sig("tv_build_dev", C.c_int, _P, _P, _P, C.c_int32, C.c_int32, C.c_int32, C.POINTER(_BuildConfig),
     C.POINTER(_Camera), C.c_int, C.POINTER(_P), C.POINTER(_BuildStats))
_sig("tv_build_trim", C.c_int, C.c_int)
_sig("tv_build_scratch_bytes", C.c_uint64, C.c_int)
_sig("tv_generate_volume_dev", C.c_int, C.c_int32, C.c_int32, C.c_int32, C.c_int32, C.c_double, _P, C.c_int)
_sig("tv_render_multi", C.c_int, C.POINTER(_P), C.c_int32, C.POINTER(_Camera), C.POINTER(_RenderConfig),
     C.POINTER(_Framebuffer), C.POINTER(_RenderStats))
_sig("tv_render", C.c_int, _P, C.POINTER(_Camera), C.POINTER(_RenderConfig), C.POINTER(_Framebuffer),
     C.POINTER(_RenderStats))
_sig("tv_render_tiles", C.c_int, _P, C.POINTER(_Camera), C.POINTER(_RenderConfig), C.c_int32, C.c_int32, _P, _P, _P,
     _P, _P)
_sig("tv_tile_pack_words", C.c_uint64, C.c_int32, C.c_int32, C.c_int32, C.c_int32, C.c_int32)
_sig("tv_last_frame_timing", C.c_int, C.c_int, C.POINTER(C.c_double))
_sig("tv_tile_pack", C.c_int, _P, _P, C.c_int32, C.c_int32, C.c_int32, C.c_int32, C.c_int32, _P)
_sig("tv_tile_unpack", C.c_int, _P, _P, C.c_int32, C.c_int32, C.c_int32, C.c_int32, C.c_int32, _P)
_sig("tv_march_segments", C.c_int, _P, _P, C.c_uint64, _P, _U64, C.c_uint64, _U64, _U64)
_sig("tv_locate_points", C.c_int, _P, _D, C.c_uint64, _U32)
_sig("tv_march_transmittance", C.c_int, _P, _P, C.c_uint64, _D, _D, _U64)
_sig("tv_trace_rays", C.c_int, _P, _P, C.c_uint64, C.POINTER(_RenderConfig), C.c_uint64, _U64, _U64, _D, _U64)
_sig("tv_sample_free_path", C.c_int, _P, _P, C.c_uint64, C.c_uint64, _U64, _U64, _P, _U64)
_sig("tv_render_tracking", C.c_int, _P, C.POINTER(_Camera), C.POINTER(_RenderConfig), C.c_int32, C.c_double,
     C.POINTER(_Framebuffer), C.POINTER(_RenderStats))
_sig("tv_transmittance_tracking", C.c_int, _P, _P, C.c_uint64, C.c_int32, C.c_double, C.c_uint64, _U64, _U64, _D,
     _U64)
_sig("tv_render_regular", C.c_int, _F, C.c_int32, C.c_int32, C.c_int32, C.c_double, C.POINTER(_Camera),
     C.POINTER(_RenderConfig), C.c_int, C.POINTER(_Framebuffer), C.POINTER(_RenderStats))
_sig("tv_render_regular_dev", C.c_int, _P, C.c_int32, C.c_int32, C.c_int32, C.c_double, C.POINTER(_Camera),
     C.POINTER(_RenderConfig), C.c_int, C.POINTER(_Framebuffer), C.POINTER(_RenderStats))

_sig("tv_ipc_export", C.c_int, _P, C.POINTER(C.c_uint8), C.POINTER(C.c_uint64))
_sig("tv_ipc_open", C.c_int, C.POINTER(C.c_uint8), C.c_uint64, C.c_int, C.POINTER(_P))
_sig("tv_ipc_close", C.c_int, _P, C.c_uint64)
_sig("tv_diag_gather_ceiling", C.c_int, _P, C.POINTER(_Camera), C.POINTER(_RenderConfig), C.c_int,
     C.POINTER(C.c_double))

# reference Tet layout (tet_grid.hpp:64-75; 68 bytes)
TET_DTYPE = np.dtype([("verts", "<u4", 4), ("children", "<u4", 2), ("parent", "<u4"), ("neighbors", "<u4", 4),
                      ("normal_ids", "u1", 4), ("level", "u1"), ("pad0", "u1", 3), ("density", "<f4"),
                      ("temperature", "<f4"), ("albedo", "<f4"), ("mask", "u1"), ("pad1", "u1", 3)])
SEGMENT_DTYPE = np.dtype([("cell", "<u4"), ("pad", "<u4"), ("t_enter", "<f8"), ("t_exit", "<f8")])


def version() -> str:
    return _lib.tv_version().decode()


def device_count() -> int:
    n = C.c_int()
    _check(_lib.tv_device_count(C.byref(n)))
    return n.value


# ------------------------------------------------------ config mirrors ---
@dataclass
class PinholeCamera:
    """camera.hpp:16-48 (validated by the library exactly as camera.cpp:15-20)."""

    position: tuple = (0.5, 0.5, -2.0)
    forward: tuple = (0.0, 0.0, 1.0)
    up: tuple = (0.0, 1.0, 0.0)
    vfov_degrees: float = 40.0
    width: int = 256
    height: int = 256

    def _c(self) -> _Camera:
        c = _Camera()
        c.position[:] = [float(x) for x in self.position]
        c.forward[:] = [float(x) for x in self.forward]
        c.up[:] = [float(x) for x in self.up]
        c.vfov_degrees = float(self.vfov_degrees)
        c.width, c.height = int(self.width), int(self.height)
        return c


@dataclass
class RenderConfig:
    """tracer.hpp:16-28"""

    spp: int = 32
    max_bounces: int = 64
    seed: int = 0
    hg_g: float = 0.0
    default_albedo: float = 0.8
    environment: tuple = (1.0, 1.0, 1.0)
    emission_scale: float = 1.0
    exposure: float = 1.0
    gamma: float = 2.2

    def _c(self) -> _RenderConfig:
        r = _RenderConfig()
        r.spp, r.max_bounces, r.seed = int(self.spp), int(self.max_bounces), int(self.seed)
        r.hg_g, r.default_albedo = float(self.hg_g), float(self.default_albedo)
        r.environment[:] = [float(x) for x in self.environment]
        r.emission_scale, r.exposure, r.gamma = float(self.emission_scale), float(self.exposure), float(self.gamma)
        return r


@dataclass
class BuildConfig:
    """builder.hpp:21-29"""

    variation_threshold: float = 0.1
    max_level: int = 24
    use_camera: bool = False
    pixel_threshold: float = 1.0
    density_scale: float = 1.0

    def _c(self) -> _BuildConfig:
        b = _BuildConfig()
        b.variation_threshold, b.max_level, b.use_camera = float(self.variation_threshold), int(self.max_level), int(
            bool(self.use_camera))
        b.pixel_threshold, b.density_scale = float(self.pixel_threshold), float(self.density_scale)
        return b


@dataclass
class BuildStats:
    """builder.hpp:31-38 plus GPU round counters."""

    leaf_count: int = 0
    max_depth: int = 0
    rounds: int = 0
    seconds: float = 0.0
    criterion_splits: int = 0
    propagation_splits: int = 0
    closure_passes: int = 0
    voxel_visits: int = 0


@dataclass
class ImageAccumulator:
    """image.hpp:18-70 (host copy of the framebuffer)."""

    width: int
    height: int
    sum: np.ndarray
    sum_sq: np.ndarray
    sample_counts: np.ndarray
    cells_visited: int = 0
    paths_traced: int = 0
    degenerate_paths: int = 0
    seconds: float = 0.0

    def mean(self) -> np.ndarray:
        n = self.sample_counts.reshape(-1, 1).astype(np.float64)
        m = np.zeros_like(self.sum.reshape(-1, 3))
        nz = n[:, 0] > 0
        m[nz] = self.sum.reshape(-1, 3)[nz] / n[nz]
        return m.reshape(self.height, self.width, 3)

    def variance_of_mean(self) -> np.ndarray:
        """image.hpp:56-69"""
        n = self.sample_counts.reshape(-1, 1).astype(np.float64)
        s = self.sum.reshape(-1, 3)
        q = self.sum_sq.reshape(-1, 3)
        out = np.zeros_like(s)
        ok = n[:, 0] >= 2
        m = s[ok] / n[ok]
        var = (q[ok] - n[ok] * m * m) / (n[ok] - 1.0)
        out[ok] = np.maximum(0.0, var) / n[ok]
        return out.reshape(self.height, self.width, 3)


# ------------------------------------------------------------------ grid ---
class TetGrid:
    """A tet grid resident in one GPU's HBM (opaque ``tv_grid`` handle)."""

    def __init__(self, handle):
        self._h = handle

    @classmethod
    def upload(cls, vertices: np.ndarray, tets: np.ndarray, roots, max_level: int = 48, device: int = 0):
        """From reference pools: vertices (nv,3) u32 fixed point, tets (nt,) TET_DTYPE, roots (24,) u32."""
        v = np.ascontiguousarray(vertices, np.uint32)
        t = np.ascontiguousarray(tets)
        if t.dtype != TET_DTYPE:
            raise ValueError("tets must use TET_DTYPE (the reference 68-byte Tet layout)")
        r = np.ascontiguousarray(roots, np.uint32)
        if r.shape != (24,):
            raise ValueError("roots must have 24 entries")
        h = _P()
        _check(_lib.tv_grid_upload(v.ctypes.data_as(_P), len(v), t.ctypes.data_as(_P), len(t), r.ctypes.data_as(_U32),
                                   int(max_level), int(device), C.byref(h)))
        return cls(h)

    @property
    def handle(self):
        if not self._h:
            raise ValueError("grid is closed")
        return self._h

    def info(self) -> dict:
        gi = _GridInfo()
        _check(_lib.tv_grid_get_info(self.handle, C.byref(gi)))
        return {k: getattr(gi, k) for k, _ in _GridInfo._fields_ if k != "pad"}

    def download(self):
        """-> (vertices (nv,3) u32, tets (nt,) TET_DTYPE, roots (24,) u32) in reference layout and ids."""
        i = self.info()
        v = np.zeros((i["n_vertices"], 3), np.uint32)
        t = np.zeros(i["n_tets"], TET_DTYPE)
        r = np.zeros(24, np.uint32)
        _check(_lib.tv_grid_download(self.handle, v.ctypes.data_as(_P), t.ctypes.data_as(_P), r.ctypes.data_as(_U32)))
        return v, t, r

    def validate(self) -> dict:
        """TetGrid::validate (tet_grid.cpp:474-636) on the GPU: the reference's report fields."""
        r = _ValidationReport()
        _check(_lib.tv_grid_validate(self.handle, C.byref(r)))
        return dict(ok=bool(r.ok), firstViolation=r.first_violation.decode() or None, leafCount=r.leaf_count,
                    interiorFaces=r.interior_faces, boundaryFaces=r.boundary_faces)

    def spot_check(self, rays: int = 100, seed: int = 0) -> tuple:
        """cmd_validate's traversal spot checks (cli.cpp:565-595) -> (failures, first failing ray or -1)."""
        r = spot_rays(seed, rays)
        f, first = C.c_int32(), C.c_int32()
        _check(_lib.tv_validate_rays(self.handle, r.ctypes.data_as(_P), len(r), C.byref(f), C.byref(first)))
        return f.value, first.value

    def save(self, path) -> None:
        """save_grid (builder.hpp:59): the reference's TGRD v1 file, packed on the device."""
        _check(_lib.tv_grid_save(self.handle, os.fsencode(path)))

    @classmethod
    def load(cls, path, device: int = 0) -> "TetGrid":
        """load_grid (builder.hpp:60): checks and messages as the reference, unpacked on the device."""
        h = _P()
        _check(_lib.tv_grid_load(os.fsencode(path), int(device), C.byref(h)))
        return cls(h)

    def close(self):
        if getattr(self, "_h", None):
            if _lib is not None:  # None only during interpreter shutdown
                _lib.tv_grid_free(self._h)
            self._h = None

    def __del__(self):
        self.close()

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()


# ---------------------------------------------------------------- calls ---
def render(grid: TetGrid, camera: PinholeCamera, cfg: RenderConfig, threads: int = 0) -> ImageAccumulator:
    """tracer.hpp:84-85. ``threads`` is accepted for signature parity and ignored."""
    del threads
    w, h = int(camera.width), int(camera.height)
    s = np.zeros(w * h * 3)
    sq = np.zeros(w * h * 3)
    cnt = np.zeros(w * h, np.uint32)
    fb = _Framebuffer(s.ctypes.data_as(_D), sq.ctypes.data_as(_D), cnt.ctypes.data_as(_U32))
    st = _RenderStats()
    cam, rc = camera._c(), cfg._c()
    _check(_lib.tv_render(grid.handle, C.byref(cam), C.byref(rc), C.byref(fb), C.byref(st)))
    return ImageAccumulator(w, h, s, sq, cnt, st.cells_visited, st.paths_traced, st.degenerate_paths, st.seconds)


def render_multi(grids, camera: PinholeCamera, cfg: RenderConfig) -> ImageAccumulator:
    """render() over several GPUs from one process: grids[r] (one per device,
    normally the same grid uploaded or built on each) renders the interleaved
    16x16 tiles t % len(grids) == r; the result equals render()'s bit for bit.
    ``seconds`` is the slowest rank's device time."""
    grids = list(grids)
    w, h = int(camera.width), int(camera.height)
    s = np.zeros(w * h * 3)
    sq = np.zeros(w * h * 3)
    cnt = np.zeros(w * h, np.uint32)
    fb = _Framebuffer(s.ctypes.data_as(_D), sq.ctypes.data_as(_D), cnt.ctypes.data_as(_U32))
    st = _RenderStats()
    cam, rc = camera._c(), cfg._c()
    hs = (_P * len(grids))(*[g.handle for g in grids])
    _check(_lib.tv_render_multi(hs, len(grids), C.byref(cam), C.byref(rc), C.byref(fb), C.byref(st)))
    return ImageAccumulator(w, h, s, sq, cnt, st.cells_visited, st.paths_traced, st.degenerate_paths, st.seconds)


def render_into(grid: TetGrid, camera: PinholeCamera, cfg: RenderConfig, sum_out: np.ndarray,
                sum_sq_out: np.ndarray | None = None, counts_out: np.ndarray | None = None) -> dict:
    """render() into caller-provided (e.g. pinned) host buffers; returns the stats."""
    fb = _Framebuffer(sum_out.ctypes.data_as(_D), None if sum_sq_out is None else sum_sq_out.ctypes.data_as(_D),
                      None if counts_out is None else counts_out.ctypes.data_as(_U32))
    st = _RenderStats()
    cam, rc = camera._c(), cfg._c()
    _check(_lib.tv_render(grid.handle, C.byref(cam), C.byref(rc), C.byref(fb), C.byref(st)))
    return dict(cells_visited=st.cells_visited, paths_traced=st.paths_traced, degenerate_paths=st.degenerate_paths,
                seconds=st.seconds)


def render_tiles(grid: TetGrid, camera: PinholeCamera, cfg: RenderConfig, rank: int, n_ranks: int, sum_dev: int,
                 sum_sq_dev: int | None, counts_dev: int | None, stats_dev: int | None, stream: int = 0):
    """Asynchronous per-rank share of a frame into device buffers (raw device pointers)."""
    cam, rc = camera._c(), cfg._c()
    _check(_lib.tv_render_tiles(grid.handle, C.byref(cam), C.byref(rc), int(rank), int(n_ranks), sum_dev, sum_sq_dev,
                                counts_dev, stats_dev, stream))


def last_frame_timing(device: int = 0) -> dict:
    """Device ms of the last frame's kernels (start, trace, accumulate) and its launch count."""
    out = (C.c_double * 4)()
    _check(_lib.tv_last_frame_timing(int(device), out))
    return dict(start_ms=out[0], trace_ms=out[1], accum_ms=out[2], launches=int(out[3]))


def diag_gather_ceiling(grid: TetGrid, camera: PinholeCamera, cfg: RenderConfig, reps: int = 3) -> dict:
    """Memory-latency ceiling of the trace kernel on this frame (include/tetvol_b200_diag.h):
    the recorded tet-step sequences of every path replayed as dependent 64-B record loads."""
    cam, rc = camera._c(), cfg._c()
    out = (C.c_double * 6)()
    _check(_lib.tv_diag_gather_ceiling(grid.handle, C.byref(cam), C.byref(rc), int(reps), out))
    return dict(steps_per_s=out[0], steps_per_s_full_occupancy=out[1], steps=int(out[2]), replay_ms=out[3],
                seq_bytes_per_step=out[4], warps_per_sm=int(out[5]))


def ipc_export(dev_ptr: int) -> bytes:
    """Handle (64 bytes) + byte offset (8) of a device pointer, for ipc_open in another process."""
    h = (C.c_uint8 * 64)()
    off = C.c_uint64()
    _check(_lib.tv_ipc_export(C.c_void_p(dev_ptr), h, C.byref(off)))
    return bytes(h) + int(off.value).to_bytes(8, "little")


def ipc_open(handle: bytes, device: int = 0) -> int:
    """Maps a peer process's pointer (ipc_export) on `device`; returns the device pointer."""
    h = (C.c_uint8 * 64).from_buffer_copy(handle[:64])
    out = C.c_void_p()
    _check(_lib.tv_ipc_open(h, int.from_bytes(handle[64:72], "little"), int(device), C.byref(out)))
    return int(out.value)


def ipc_close(dev_ptr: int, handle: bytes) -> None:
    _check(_lib.tv_ipc_close(C.c_void_p(dev_ptr), int.from_bytes(handle[64:72], "little")))


def tile_pack_words(width: int, height: int, rank: int, n_ranks: int, elem_words: int) -> int:
    return int(_lib.tv_tile_pack_words(width, height, rank, n_ranks, elem_words))


def tile_pack(frame_dev: int, packed_dev: int, width, height, rank, n_ranks, elem_words, stream: int = 0):
    _check(_lib.tv_tile_pack(frame_dev, packed_dev, width, height, rank, n_ranks, elem_words, stream))


def tile_unpack(packed_dev: int, frame_dev: int, width, height, rank, n_ranks, elem_words, stream: int = 0):
    _check(_lib.tv_tile_unpack(packed_dev, frame_dev, width, height, rank, n_ranks, elem_words, stream))


def march_segments(grid: TetGrid, rays: np.ndarray):
    """tracer.hpp:49 over a batch. rays: (n, 8) [origin, dir, t_min, t_max].

    Returns (segments: SEGMENT_DTYPE array, offsets: (n+1,) u64, degenerate_paths)."""
    r = np.ascontiguousarray(rays, np.float64)
    if r.ndim != 2 or r.shape[1] != 8:
        raise ValueError("rays must be (n, 8)")
    n = len(r)
    off = np.zeros(n + 1, np.uint64)
    total = C.c_uint64()
    deg = C.c_uint64()
    _check(_lib.tv_march_segments(grid.handle, r.ctypes.data_as(_P), n, None, off.ctypes.data_as(_U64), 0,
                                  C.byref(total), C.byref(deg)))
    seg = np.zeros(total.value, SEGMENT_DTYPE)
    _check(_lib.tv_march_segments(grid.handle, r.ctypes.data_as(_P), n, seg.ctypes.data_as(_P),
                                  off.ctypes.data_as(_U64), total.value, C.byref(total), C.byref(deg)))
    return seg, off, deg.value


FREE_PATH_DTYPE = np.dtype([("collided", "<i4"), ("cell", "<u4"), ("distance", "<f8"), ("position", "<f8", 3)])


def trace(grid: TetGrid, rays: np.ndarray, cfg: RenderConfig, seed: int, pixels, samples):
    """tracer.hpp:78-79 over a batch, RngStream(seed, pixels[i], samples[i]) per ray.
    -> ((n, 3) radiance, cells_visited, degenerate_paths)"""
    r = np.ascontiguousarray(rays, np.float64).reshape(-1, 8)
    px = np.ascontiguousarray(np.broadcast_to(pixels, len(r)), np.uint64)
    sm = np.ascontiguousarray(np.broadcast_to(samples, len(r)), np.uint64)
    out = np.zeros((len(r), 3))
    st = np.zeros(2, np.uint64)
    rc = cfg._c()
    _check(_lib.tv_trace_rays(grid.handle, r.ctypes.data_as(_P), len(r), C.byref(rc), int(seed),
                              px.ctypes.data_as(_U64), sm.ctypes.data_as(_U64), out.ctypes.data_as(_D),
                              st.ctypes.data_as(_U64)))
    return out, int(st[0]), int(st[1])


def march_transmittance(grid: TetGrid, rays: np.ndarray):
    """tracer.hpp:52 over a batch -> (tau (bit-exact optical depth), exp(-tau), cells_visited, degenerate_paths)."""
    r = np.ascontiguousarray(rays, np.float64).reshape(-1, 8)
    tau = np.zeros(len(r))
    tr = np.zeros(len(r))
    st = np.zeros(2, np.uint64)
    _check(_lib.tv_march_transmittance(grid.handle, r.ctypes.data_as(_P), len(r), tau.ctypes.data_as(_D),
                                       tr.ctypes.data_as(_D), st.ctypes.data_as(_U64)))
    return tau, tr, int(st[0]), int(st[1])


# free-flight estimators (include/tetvol_b200.h): regular tracking is the
# reference's and tv_render's; delta / ratio tracking over the per-tet majorant
# mu = majorant_scale * density are optional modes, equal in distribution
TRACK_REGULAR, TRACK_DELTA, TRACK_RATIO = 0, 1, 2


def render_tracking(grid: TetGrid, camera: PinholeCamera, cfg: RenderConfig, tracking: int = TRACK_DELTA,
                    majorant_scale: float = 1.0) -> ImageAccumulator:
    """render() with delta tracking over the per-tet majorant (TRACK_REGULAR is render())."""
    w, h = int(camera.width), int(camera.height)
    s = np.zeros(w * h * 3)
    sq = np.zeros(w * h * 3)
    cnt = np.zeros(w * h, np.uint32)
    fb = _Framebuffer(s.ctypes.data_as(_D), sq.ctypes.data_as(_D), cnt.ctypes.data_as(_U32))
    st = _RenderStats()
    cam, rc = camera._c(), cfg._c()
    _check(_lib.tv_render_tracking(grid.handle, C.byref(cam), C.byref(rc), int(tracking), float(majorant_scale),
                                   C.byref(fb), C.byref(st)))
    return ImageAccumulator(w, h, s, sq, cnt, st.cells_visited, st.paths_traced, st.degenerate_paths, st.seconds)


def transmittance_tracking(grid: TetGrid, rays: np.ndarray, tracking: int, majorant_scale: float = 1.0,
                           seed: int = 0, pixels=0, samples=0):
    """One transmittance estimate per ray -> (estimates, cells_visited, degenerate_paths)."""
    r = np.ascontiguousarray(rays, np.float64).reshape(-1, 8)
    px = np.ascontiguousarray(np.broadcast_to(pixels, len(r)), np.uint64)
    sm = np.ascontiguousarray(np.broadcast_to(samples, len(r)), np.uint64)
    out = np.zeros(len(r))
    st = np.zeros(2, np.uint64)
    _check(_lib.tv_transmittance_tracking(grid.handle, r.ctypes.data_as(_P), len(r), int(tracking),
                                          float(majorant_scale), int(seed), px.ctypes.data_as(_U64),
                                          sm.ctypes.data_as(_U64), out.ctypes.data_as(_D), st.ctypes.data_as(_U64)))
    return out, int(st[0]), int(st[1])


def sample_free_path(grid: TetGrid, rays: np.ndarray, seed: int, pixels, samples):
    """tracer.hpp:63 over a batch with RngStream(seed, pixels[i], samples[i]) -> FREE_PATH_DTYPE records."""
    r = np.ascontiguousarray(rays, np.float64).reshape(-1, 8)
    px = np.ascontiguousarray(np.broadcast_to(pixels, len(r)), np.uint64)
    sm = np.ascontiguousarray(np.broadcast_to(samples, len(r)), np.uint64)
    out = np.zeros(len(r), FREE_PATH_DTYPE)
    _check(_lib.tv_sample_free_path(grid.handle, r.ctypes.data_as(_P), len(r), int(seed), px.ctypes.data_as(_U64),
                                    sm.ctypes.data_as(_U64), out.ctypes.data_as(_P), None))
    return out


def locate_points(grid: TetGrid, points: np.ndarray) -> np.ndarray:
    """TetGrid::locate_point over a batch (tet_grid.hpp:166); NO_TET outside the cube."""
    p = np.ascontiguousarray(points, np.float64).reshape(-1, 3)
    out = np.zeros(len(p), np.uint32)
    _check(_lib.tv_locate_points(grid.handle, p.ctypes.data_as(_D), len(p), out.ctypes.data_as(_U32)))
    return out


def _vol_ptrs(volume, temperature=None, albedo=None):
    v = np.ascontiguousarray(volume, np.float32)
    if v.ndim != 3:
        raise ValueError("volume must be (nz, ny, nx) float32, x fastest")
    t = None if temperature is None else np.ascontiguousarray(temperature, np.float32)
    a = None if albedo is None else np.ascontiguousarray(albedo, np.float32)
    return v, t, a


def build_adaptive_grid(volume: np.ndarray, cfg: BuildConfig, camera: PinholeCamera | None = None,
                        temperature: np.ndarray | None = None, albedo: np.ndarray | None = None,
                        device: int = 0):
    """builder.hpp:51-52 on the GPU. volume: (nz, ny, nx) float32 density. -> (TetGrid, BuildStats)."""
    v, t, a = _vol_ptrs(volume, temperature, albedo)
    nz, ny, nx = v.shape
    h = _P()
    st = _BuildStats()
    bc = cfg._c()
    cam = camera._c() if camera is not None else None
    _check(_lib.tv_build(v.ctypes.data_as(_F), None if t is None else t.ctypes.data_as(_F),
                         None if a is None else a.ctypes.data_as(_F), nx, ny, nz, C.byref(bc),
                         C.byref(cam) if cam is not None else None, int(device), C.byref(h), C.byref(st)))
    return TetGrid(h), BuildStats(**{k: getattr(st, k) for k, _ in _BuildStats._fields_})


def build_adaptive_grid_dev(density_dev: int, shape, cfg: BuildConfig, camera: PinholeCamera | None = None,
                            device: int = 0, temperature_dev: int | None = None, albedo_dev: int | None = None):
    """Same, with the density already in HBM (raw device pointer; shape = (nz, ny, nx))."""
    nz, ny, nx = shape
    h = _P()
    st = _BuildStats()
    bc = cfg._c()
    cam = camera._c() if camera is not None else None
    _check(_lib.tv_build_dev(density_dev, temperature_dev, albedo_dev, nx, ny, nz, C.byref(bc),
                             C.byref(cam) if cam is not None else None, int(device), C.byref(h), C.byref(st)))
    return TetGrid(h), BuildStats(**{k: getattr(st, k) for k, _ in _BuildStats._fields_})


def build_trim(device: int = -1) -> None:
    """Release the build scratch kept on `device` (-1: all devices) for the next build."""
    _check(_lib.tv_build_trim(int(device)))


def build_scratch_bytes(device: int = -1) -> int:
    """Device bytes of build scratch currently held (see tv_build_trim)."""
    return int(_lib.tv_build_scratch_bytes(int(device)))


VOLUME_KINDS = {"constant": 0, "ramp": 1, "blob": 2, "step": 3, "noise": 4, "cloud": 5}


def generate_volume_dev(kind: str, n: int, out_dev: int, device: int = 0, value: float = 1.0):
    """Procedural density field written into HBM (n^3 float32 at out_dev)."""
    _check(_lib.tv_generate_volume_dev(VOLUME_KINDS[kind], n, n, n, float(value), out_dev, int(device)))


def render_reference(volume: np.ndarray, density_scale: float, camera: PinholeCamera, cfg: RenderConfig,
                     device: int = 0) -> ImageAccumulator:
    """regular_grid.hpp:66-67: RegularGrid::from_volume + render_reference on the GPU."""
    v, _, _ = _vol_ptrs(volume)
    nz, ny, nx = v.shape
    w, h = int(camera.width), int(camera.height)
    s = np.zeros(w * h * 3)
    sq = np.zeros(w * h * 3)
    cnt = np.zeros(w * h, np.uint32)
    fb = _Framebuffer(s.ctypes.data_as(_D), sq.ctypes.data_as(_D), cnt.ctypes.data_as(_U32))
    st = _RenderStats()
    cam, rc = camera._c(), cfg._c()
    _check(_lib.tv_render_regular(v.ctypes.data_as(_F), nx, ny, nz, float(density_scale), C.byref(cam), C.byref(rc),
                                  int(device), C.byref(fb), C.byref(st)))
    return ImageAccumulator(w, h, s, sq, cnt, st.cells_visited, st.paths_traced, st.degenerate_paths, st.seconds)


def render_reference_dev(density_dev: int, shape, density_scale: float, camera: PinholeCamera, cfg: RenderConfig,
                         device: int = 0) -> ImageAccumulator:
    """render_reference with the density already in HBM (raw device pointer, shape = (nz, ny, nx))."""
    nz, ny, nx = shape
    w, h = int(camera.width), int(camera.height)
    s = np.zeros(w * h * 3)
    sq = np.zeros(w * h * 3)
    cnt = np.zeros(w * h, np.uint32)
    fb = _Framebuffer(s.ctypes.data_as(_D), sq.ctypes.data_as(_D), cnt.ctypes.data_as(_U32))
    st = _RenderStats()
    cam, rc = camera._c(), cfg._c()
    _check(_lib.tv_render_regular_dev(density_dev, nx, ny, nz, float(density_scale), C.byref(cam), C.byref(rc),
                                      int(device), C.byref(fb), C.byref(st)))
    return ImageAccumulator(w, h, s, sq, cnt, st.cells_visited, st.paths_traced, st.degenerate_paths, st.seconds)


def spot_rays(seed: int, n: int) -> np.ndarray:
    """cmd_validate's spot-check rays (cli.cpp:552-569), (n, 8) float64 [origin, dir, t_min, t_max]."""
    out = np.zeros((n, 8), np.float64)
    _check(_lib.tv_validate_spot_rays(int(seed), int(n), out.ctypes.data_as(_P)))
    return out


def save_grid(grid: TetGrid, path) -> None:
    """builder.hpp:59"""
    grid.save(path)


def load_grid(path, device: int = 0) -> TetGrid:
    """builder.hpp:60"""
    return TetGrid.load(path, device)


from .image import (FloatImage, compare_images, pfm_pixels, read_pfm, render_accumulate,  # noqa: E402
                    write_pfm, write_variance_pfm)
from .volume import DenseVolume, build_adaptive_grid_volume  # noqa: E402

__all__ = [
    "BuildConfig", "BuildStats", "CameraError", "ConfigError", "CudaError", "DenseVolume", "FloatImage",
    "FormatError", "GridError", "ImageError", "VolumeError", "build_adaptive_grid_volume", "compare_images",
    "pfm_pixels", "read_pfm", "render_accumulate", "write_pfm", "write_variance_pfm",
    "ImageAccumulator", "IoError", "load_grid", "save_grid", "spot_rays",
    "OutsideGrid", "PinholeCamera", "RenderConfig", "TET_DTYPE", "SEGMENT_DTYPE", "TetGrid", "TetvolError",
    "build_adaptive_grid", "build_adaptive_grid_dev", "build_scratch_bytes", "build_trim", "device_count", "generate_volume_dev", "locate_points",
    "march_segments", "march_transmittance", "trace", "sample_free_path", "FREE_PATH_DTYPE", "render", "render_into", "render_multi", "render_reference", "render_tiles", "tile_pack", "tile_pack_words",
    "tile_unpack", "version",
]
