"""TEST INFRASTRUCTURE ONLY — ctypes bindings to the two CPU checkers.

* ``C``   — ``oracle/liboracle.so``: the C restatement of the reference path
  (``oracle/tvo.c``), built by ``oracle/Makefile``.
* ``REF`` — ``oracle/_ref/libtetvol_ref.so``: the unmodified reference library
  compiled from ``/root/reference/proj/src`` plus ``oracle/ref_shim.cpp``.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU legs import
this package. The product (``paper_2506_11510_b200``) never does.

Both libraries export the same entry points (``tvo_*`` / ``ref_*``) with the
same argument structs, so a test can run one workload through either checker
and compare bit patterns.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
NO_TET = 0xFFFFFFFF

# reference Tet layout (tet_grid.hpp:64-75), 68 bytes
TET_DTYPE = np.dtype(
    [
        ("verts", "<u4", 4),
        ("children", "<u4", 2),
        ("parent", "<u4"),
        ("neighbors", "<u4", 4),
        ("normal_ids", "u1", 4),
        ("level", "u1"),
        ("pad0", "u1", 3),
        ("density", "<f4"),
        ("temperature", "<f4"),
        ("albedo", "<f4"),
        ("mask", "u1"),
        ("pad1", "u1", 3),
    ]
)
assert TET_DTYPE.itemsize == 68


class Camera(C.Structure):
    _fields_ = [
        ("pos", C.c_double * 3),
        ("fwd", C.c_double * 3),
        ("up", C.c_double * 3),
        ("vfov", C.c_double),
        ("width", C.c_int32),
        ("height", C.c_int32),
    ]


class RenderCfg(C.Structure):
    _fields_ = [
        ("spp", C.c_int32),
        ("max_bounces", C.c_int32),
        ("seed", C.c_uint64),
        ("hg_g", C.c_double),
        ("default_albedo", C.c_double),
        ("env", C.c_double * 3),
        ("emission_scale", C.c_double),
    ]


class BuildCfg(C.Structure):
    _fields_ = [
        ("variation_threshold", C.c_double),
        ("max_level", C.c_int32),
        ("use_camera", C.c_int32),
        ("pixel_threshold", C.c_double),
        ("density_scale", C.c_double),
    ]


class BuildStats(C.Structure):
    _fields_ = [
        ("leaf_count", C.c_uint64),
        ("max_depth", C.c_int32),
        ("pad", C.c_int32),
        ("seconds", C.c_double),
        ("criterion_splits", C.c_uint64),
        ("propagation_splits", C.c_uint64),
    ]


def camera(pos=(0.5, 0.5, -2.0), fwd=(0, 0, 1), up=(0, 1, 0), vfov=40.0, width=256, height=256) -> Camera:
    c = Camera()
    c.pos[:] = pos
    c.fwd[:] = fwd
    c.up[:] = up
    c.vfov = vfov
    c.width = width
    c.height = height
    return c


def render_cfg(spp=32, max_bounces=64, seed=0, hg_g=0.0, default_albedo=0.8, env=(1.0, 1.0, 1.0), emission_scale=1.0):
    r = RenderCfg()
    r.spp, r.max_bounces, r.seed, r.hg_g, r.default_albedo = spp, max_bounces, seed, hg_g, default_albedo
    r.env[:] = env
    r.emission_scale = emission_scale
    return r


def build_cfg(variation_threshold=0.1, max_level=24, use_camera=False, pixel_threshold=1.0, density_scale=1.0):
    b = BuildCfg()
    b.variation_threshold, b.max_level, b.use_camera = variation_threshold, max_level, int(use_camera)
    b.pixel_threshold, b.density_scale = pixel_threshold, density_scale
    return b


_P = C.c_void_p
_D = C.POINTER(C.c_double)
_U32 = C.POINTER(C.c_uint32)
_U64 = C.POINTER(C.c_uint64)
_F = C.POINTER(C.c_float)


def _ptr(a, t):
    return None if a is None else a.ctypes.data_as(t)


@dataclass
class Pools:
    """Host pools of a TetGrid: vertices (nv,3) u32, tets (nt,) TET_DTYPE, roots (24,) u32."""

    vq: np.ndarray
    tets: np.ndarray
    roots: np.ndarray
    max_level: int

    @property
    def leaf_mask(self):
        return self.tets["children"][:, 0] == NO_TET


class Checker:
    """One CPU checker library (prefix 'tvo' = C restatement, 'ref' = reference)."""

    def __init__(self, path: str, prefix: str):
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} missing: run `make -f oracle/Makefile`")
        self.lib = C.CDLL(path)
        self.prefix = prefix
        L, p = self.lib, prefix

        def f(name, res, *args):
            fn = getattr(L, f"{p}_{name}")
            fn.restype = res
            fn.argtypes = list(args)
            return fn

        f("last_error", C.c_char_p)
        f("grid_free", None, _P)
        f("grid_init_roots", _P, C.c_int)
        f("grid_fuzzed", _P, C.c_int, C.c_uint64, C.c_int)
        f("grid_counts", None, _P, _U64)
        f("grid_export", None, _P, _U32, _P, _U32)
        f("grid_refine_conforming", C.c_int, _P, C.c_uint32)
        f("grid_fill_density", None, _P, C.c_float)
        f("grid_build", _P, _F, _F, _F, C.c_int, C.c_int, C.c_int, C.POINTER(BuildCfg), C.POINTER(Camera),
          C.POINTER(BuildStats))
        f("locate_point", C.c_int, _P, _D, _U32)
        f("exit_face", C.c_int, _P, C.c_uint32, _D, _D, _D)
        f("march_segments", C.c_int64, _P, _D, C.c_uint64, _U32, _D, _D, _U64, C.c_uint64, _U64)
        f("march_transmittance", C.c_double, _P, _D)
        f("sample_free_path", None, _P, _D, C.c_uint64, C.c_uint64, C.c_uint64, _D)
        f("hg_sample_cos", C.c_double, C.c_double, C.c_double)
        f("sample_phase_hg", None, _D, C.c_double, C.c_uint64, C.c_uint64, C.c_uint64, _D)
        f("emission_color", None, C.c_double, _D)
        f("rng_draws", None, C.c_uint64, C.c_uint64, C.c_uint64, C.c_int, _D)
        f("mix64", C.c_uint64, C.c_uint64)
        f("primary_ray", C.c_int, C.POINTER(Camera), C.c_int, C.c_int, C.c_double, C.c_double, _D)
        f("camera_tet_tests", C.c_int, C.POINTER(Camera), _D, _D)
        f("density_stats", None, _P, _F, C.c_int, C.c_int, C.c_int, C.c_uint32, _D)
        f("dda_segments", C.c_int64, _F, C.c_int, C.c_int, C.c_int, C.c_double, _D, C.c_uint64, _U32, _D, _D,
          _U64, C.c_uint64)
        f("random_cube_rays", None, C.c_uint64, C.c_uint64, C.c_uint64, _D)
        f("render_regular", C.c_int, _F, C.c_int, C.c_int, C.c_int, C.c_double, C.POINTER(Camera),
          C.POINTER(RenderCfg), C.c_int, _D, _D, _U32, _U64, _D)
        if prefix == "tvo":
            f("grid_from_pools", _P, _U32, C.c_uint64, _P, C.c_uint64, _U32, C.c_int)
            f("render", C.c_int, _P, C.POINTER(Camera), C.POINTER(RenderCfg), C.c_int, C.c_int, C.c_int, _D, _D,
              _U32, _U64, _D)
            f("gen_volume", None, C.c_int, C.c_int, C.c_int, C.c_int, C.c_double, _F)
            f("fnv64_doubles", C.c_uint64, _D, C.c_uint64)
        else:
            f("grid_assemble", _P, _U32, C.c_uint64, _P, C.c_uint64, _U32, C.c_int)
            f("render", C.c_int, _P, C.POINTER(Camera), C.POINTER(RenderCfg), C.c_int, _D, _D, _U32, _U64, _D)
            f("grid_validate", C.c_int, _P, C.c_char_p, C.c_int, _U64)
            f("grid_uniform", _P, C.c_int)
            f("grid_load", _P, C.c_char_p)
            f("grid_save", C.c_int, _P, C.c_char_p)
            f("grid_set_payload", None, _P, C.c_uint32, C.c_float, C.c_float, C.c_float, C.c_uint32)
            f("dvol_save", C.c_int, C.c_char_p, C.c_int, C.c_int, C.c_int, C.c_int, C.POINTER(C.c_char_p),
              C.POINTER(_F))
            f("dvol_load", C.c_int, C.c_char_p, C.POINTER(C.c_int), C.POINTER(C.c_int), C.POINTER(C.c_char_p),
              C.POINTER(_F))
            f("write_pfm", C.c_int, C.c_char_p, C.c_int, C.c_int, _D, _D, _U32, C.c_int)
            f("spot_rays", None, C.c_uint64, C.c_int, _D)
            f("trace_ray", None, _P, _D, C.POINTER(RenderCfg), C.c_uint64, C.c_uint64, C.c_uint64, _D, _U64)
            f("spot_checks", None, _P, C.c_int, C.c_uint64, C.POINTER(C.c_int), C.POINTER(C.c_int))
            f("read_pfm", C.c_int, C.c_char_p, C.POINTER(C.c_int), C.POINTER(C.c_int), _F)
            f("trace_sample", None, _P, C.POINTER(Camera), C.POINTER(RenderCfg), C.c_int, C.c_int, C.c_int, _D, _U64)

    def fn(self, name):
        return getattr(self.lib, f"{self.prefix}_{name}")

    def err(self) -> str:
        return self.fn("last_error")().decode()


class Grid:
    """Owning handle to a grid inside one checker."""

    def __init__(self, chk: Checker, handle):
        if not handle:
            raise RuntimeError(f"{chk.prefix}: {chk.err()}")
        self.chk, self.h = chk, handle

    def __del__(self):
        if getattr(self, "h", None):
            self.chk.fn("grid_free")(self.h)
            self.h = None

    def counts(self):
        out = np.zeros(4, np.uint64)
        self.chk.fn("grid_counts")(self.h, _ptr(out, _U64))
        return dict(n_verts=int(out[0]), n_tets=int(out[1]), n_leaves=int(out[2]), max_level=int(out[3]))

    def pools(self) -> Pools:
        c = self.counts()
        vq = np.zeros((c["n_verts"], 3), np.uint32)
        tets = np.zeros(c["n_tets"], TET_DTYPE)
        roots = np.zeros(24, np.uint32)
        self.chk.fn("grid_export")(self.h, _ptr(vq, _U32), tets.ctypes.data_as(_P), _ptr(roots, _U32))
        return Pools(vq, tets, roots, c["max_level"])

    def fill_density(self, lam: float):
        self.chk.fn("grid_fill_density")(self.h, lam)

    def refine_conforming(self, t: int):
        if self.chk.fn("grid_refine_conforming")(self.h, t):
            raise RuntimeError(self.chk.err())

    def locate(self, p):
        p = np.ascontiguousarray(p, np.float64)
        out = C.c_uint32()
        rc = self.chk.fn("locate_point")(self.h, _ptr(p, _D), C.byref(out))
        return None if rc else int(out.value)

    def exit_face(self, cell, pos, d):
        pos = np.ascontiguousarray(pos, np.float64)
        d = np.ascontiguousarray(d, np.float64)
        t = C.c_double()
        slot = self.chk.fn("exit_face")(self.h, cell, _ptr(pos, _D), _ptr(d, _D), C.byref(t))
        return slot, t.value

    def march_segments(self, rays: np.ndarray, cap: int | None = None):
        """rays: (n, 8) float64 [o, d, tmin, tmax]. Returns (cells, t0, t1, offsets, stats)."""
        rays = np.ascontiguousarray(rays, np.float64)
        n = rays.shape[0]
        offsets = np.zeros(n + 1, np.uint64)
        stats = np.zeros(2, np.uint64)
        fn = self.chk.fn("march_segments")
        if cap is None:
            total = fn(self.h, _ptr(rays, _D), n, None, None, None, _ptr(offsets, _U64), 0, _ptr(stats, _U64))
            cap = int(total)
        cells = np.zeros(cap, np.uint32)
        t0 = np.zeros(cap, np.float64)
        t1 = np.zeros(cap, np.float64)
        fn(self.h, _ptr(rays, _D), n, _ptr(cells, _U32), _ptr(t0, _D), _ptr(t1, _D), _ptr(offsets, _U64), cap,
           _ptr(stats, _U64))
        return cells, t0, t1, offsets, stats

    def render(self, cam: Camera, rc: RenderCfg, threads: int = 0, row_stride: int = 1, row_offset: int = 0):
        w, h = cam.width, cam.height
        s = np.zeros(w * h * 3)
        sq = np.zeros(w * h * 3)
        cnt = np.zeros(w * h, np.uint32)
        st = np.zeros(3, np.uint64)
        sec = C.c_double()
        if self.chk.prefix == "tvo":
            r = self.chk.fn("render")(self.h, C.byref(cam), C.byref(rc), threads, row_stride, row_offset, _ptr(s, _D),
                                      _ptr(sq, _D), _ptr(cnt, _U32), _ptr(st, _U64), C.byref(sec))
        else:
            assert row_stride == 1 and row_offset == 0
            r = self.chk.fn("render")(self.h, C.byref(cam), C.byref(rc), threads, _ptr(s, _D), _ptr(sq, _D),
                                      _ptr(cnt, _U32), _ptr(st, _U64), C.byref(sec))
        if r:
            raise RuntimeError(self.chk.err())
        return dict(sum=s, sum_sq=sq, counts=cnt, cells_visited=int(st[0]), paths_traced=int(st[1]),
                    degenerate_paths=int(st[2]), seconds=sec.value)

    def density_stats(self, vol: np.ndarray, leaf: int):
        vol = np.ascontiguousarray(vol, np.float32)
        nz, ny, nx = vol.shape
        out = np.zeros(4)
        self.chk.fn("density_stats")(self.h, _ptr(vol, _F), nx, ny, nz, leaf, _ptr(out, _D))
        return out


def _lib_or_none(path, prefix):
    try:
        return Checker(path, prefix)
    except (FileNotFoundError, OSError):
        return None


_C = None
_REF = None


def c_oracle() -> Checker:
    global _C
    if _C is None:
        _C = Checker(os.path.join(HERE, "liboracle.so"), "tvo")
    return _C


def ref_oracle() -> Checker | None:
    """The compiled reference, or None when oracle/_ref was never built."""
    global _REF
    if _REF is None:
        _REF = _lib_or_none(os.path.join(HERE, "_ref", "libtetvol_ref.so"), "ref")
    return _REF


_REF_PAD = None


def ref_pad_oracle() -> Checker | None:
    """The reference built with ``struct alignas(64) TraceStats``,
    or None when it was never built. Used only for bench.py's cpu_baseline."""
    global _REF_PAD
    if _REF_PAD is None:
        _REF_PAD = _lib_or_none(os.path.join(HERE, "_ref", "pad", "libtetvol_ref_pad.so"), "ref")
    return _REF_PAD


def gen_volume(kind: str, n: int, value: float = 1.0) -> np.ndarray:
    kinds = {"constant": 0, "ramp": 1, "blob": 2, "step": 3, "noise": 4, "cloud": 5}
    out = np.zeros((n, n, n), np.float32)
    c_oracle().fn("gen_volume")(kinds[kind], n, n, n, value, _ptr(out, _F))
    return out


def build(chk: Checker, vol: np.ndarray, bc: BuildCfg, cam: Camera | None = None, temperature=None, albedo=None):
    vol = np.ascontiguousarray(vol, np.float32)
    nz, ny, nx = vol.shape
    st = BuildStats()
    h = chk.fn("grid_build")(_ptr(vol, _F), _ptr(temperature, _F), _ptr(albedo, _F), nx, ny, nz, C.byref(bc),
                             C.byref(cam) if cam is not None else None, C.byref(st))
    g = Grid(chk, h)
    return g, dict(leaf_count=st.leaf_count, max_depth=st.max_depth, seconds=st.seconds,
                   criterion_splits=st.criterion_splits, propagation_splits=st.propagation_splits)


def fuzzed(chk: Checker, steps: int, seed: int, max_level: int = 48) -> Grid:
    return Grid(chk, chk.fn("grid_fuzzed")(steps, seed, max_level))


def init_roots(chk: Checker, max_level: int = 48) -> Grid:
    return Grid(chk, chk.fn("grid_init_roots")(max_level))


def from_pools(chk: Checker, p: Pools) -> Grid:
    vq = np.ascontiguousarray(p.vq, np.uint32)
    tets = np.ascontiguousarray(p.tets)
    roots = np.ascontiguousarray(p.roots, np.uint32)
    name = "grid_from_pools" if chk.prefix == "tvo" else "grid_assemble"
    return Grid(chk, chk.fn(name)(_ptr(vq, _U32), len(vq), tets.ctypes.data_as(_P), len(tets), _ptr(roots, _U32),
                                  p.max_level))


def fnv64(v: np.ndarray) -> int:
    v = np.ascontiguousarray(v, np.float64)
    return int(c_oracle().fn("fnv64_doubles")(_ptr(v, _D), v.size))


def rng_draws(chk: Checker, seed, pixel, sample, n):
    out = np.zeros(n)
    chk.fn("rng_draws")(seed, pixel, sample, n, _ptr(out, _D))
    return out


def random_cube_rays(seed: int, salt: int, n: int, chk: Checker | None = None) -> np.ndarray:
    """acceptance.cpp:49-61 random_cube_ray(seed, salt, i) for i in [0, n), as (n, 8) rays."""
    out = np.zeros((n, 8))
    (chk or c_oracle()).fn("random_cube_rays")(seed, salt, n, _ptr(out, _D))
    return out
