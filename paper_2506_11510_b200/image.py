"""PFM output and image compare (image.cpp:33-101, cli.cpp:487-531) with the
per-pixel work on the GPU, and progressive device accumulation."""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np

from . import (ImageAccumulator, PinholeCamera, RenderConfig, TetGrid, _Framebuffer, _check, _lib, _sig, _D, _F, _P,
               _U32)


class _CompareStats(C.Structure):
    _fields_ = [("rmse", C.c_double), ("max_abs_diff", C.c_double), ("outlier_fraction", C.c_double),
                ("outliers", C.c_uint64)]


_I32P = C.POINTER(C.c_int32)
_sig("tv_image_pfm_pixels", C.c_int, _D, _D, _U32, C.c_int32, C.c_int32, C.c_int32, C.c_int32, C.c_int, _F)
_sig("tv_image_write_pfm", C.c_int, C.c_char_p, C.POINTER(_Framebuffer), C.c_int32, C.c_int32, C.c_int32, C.c_int32,
     C.c_int)
_sig("tv_pfm_write", C.c_int, C.c_char_p, _F, C.c_int32, C.c_int32)
_sig("tv_pfm_read", C.c_int, C.c_char_p, _I32P, _I32P, _F)
_sig("tv_image_compare", C.c_int, _F, _F, _F, _F, C.c_uint64, C.c_int, C.POINTER(_CompareStats))
_sig("tv_render_accumulate", C.c_int, _P, _P, _P, C.c_int32, C.c_int32, C.c_int32, _P, _P, _P, _P, _P)


@dataclass
class FloatImage:
    """image.hpp: linear RGB f32, rgb is (height, width, 3), row 0 = top."""

    width: int
    height: int
    rgb: np.ndarray


def _fb(img: ImageAccumulator) -> _Framebuffer:
    fb = _Framebuffer()
    fb.sum = img.sum.ctypes.data_as(_D)
    fb.sum_sq = img.sum_sq.ctypes.data_as(_D)
    fb.sample_counts = img.sample_counts.ctypes.data_as(_U32)
    return fb


def pfm_pixels(img: ImageAccumulator, variance: bool = False, device: int = 0) -> np.ndarray:
    """ImageAccumulator::mean / variance_of_mean rounded to f32 (what the PFM writers store), on the GPU."""
    out = np.empty((img.height, img.width, 3), np.float32)
    for a in (img.sum, img.sum_sq, img.sample_counts):
        assert a.flags.c_contiguous
    _check(_lib.tv_image_pfm_pixels(img.sum.ctypes.data_as(_D), img.sum_sq.ctypes.data_as(_D),
                                    img.sample_counts.ctypes.data_as(_U32), img.width, img.height, int(variance), 0,
                                    int(device), out.ctypes.data_as(_F)))
    return out


def write_pfm(path, img, device: int = 0) -> None:
    """write_pfm (image.cpp:49-81) of an ImageAccumulator or a FloatImage; byte-identical files."""
    if isinstance(img, FloatImage):
        rgb = np.ascontiguousarray(img.rgb, np.float32)
        _check(_lib.tv_pfm_write(os.fsencode(path), rgb.ctypes.data_as(_F), img.width, img.height))
        return
    fb = _fb(img)
    _check(_lib.tv_image_write_pfm(os.fsencode(path), C.byref(fb), img.width, img.height, 0, 0, int(device)))


def write_variance_pfm(path, img: ImageAccumulator, device: int = 0) -> None:
    """write_variance_pfm (image.cpp:66-77)"""
    fb = _fb(img)
    _check(_lib.tv_image_write_pfm(os.fsencode(path), C.byref(fb), img.width, img.height, 1, 0, int(device)))


def read_pfm(path) -> FloatImage:
    """read_pfm (image.cpp:83-101), with its ImageError messages."""
    w, h = C.c_int32(), C.c_int32()
    _check(_lib.tv_pfm_read(os.fsencode(path), C.byref(w), C.byref(h), None))
    rgb = np.empty((h.value, w.value, 3), np.float32)
    _check(_lib.tv_pfm_read(os.fsencode(path), C.byref(w), C.byref(h), rgb.ctypes.data_as(_F)))
    return FloatImage(w.value, h.value, rgb)


def compare_images(a: FloatImage, b: FloatImage, var_a: FloatImage | None = None, var_b: FloatImage | None = None,
                   device: int = 0) -> dict:
    """cmd_compare's metrics (cli.cpp:493-531): rmse, maxAbsDiff, outlierFraction (None without variances)."""
    from . import ConfigError, FormatError

    if a.width != b.width or a.height != b.height:
        raise FormatError(f"image dimensions differ: {a.width}x{a.height} vs {b.width}x{b.height}")
    if (var_a is None) != (var_b is None):
        raise ConfigError("--var-a and --var-b must be given together")
    if var_a is not None:
        for v in (var_a, var_b):
            if v.width != a.width or v.height != a.height:
                raise FormatError("variance image dimensions do not match the images")
    arrs = [np.ascontiguousarray(x.rgb, np.float32) for x in (a, b)]
    vs = [np.ascontiguousarray(x.rgb, np.float32) for x in (var_a, var_b)] if var_a is not None else [None, None]
    st = _CompareStats()
    _check(_lib.tv_image_compare(arrs[0].ctypes.data_as(_F), arrs[1].ctypes.data_as(_F),
                                 None if vs[0] is None else vs[0].ctypes.data_as(_F),
                                 None if vs[1] is None else vs[1].ctypes.data_as(_F), a.width * a.height, int(device),
                                 C.byref(st)))
    return dict(width=a.width, height=a.height, rmse=st.rmse, maxAbsDiff=st.max_abs_diff,
                outlierFraction=None if var_a is None else st.outlier_fraction, outliers=int(st.outliers))


def render_accumulate(grid: TetGrid, camera: PinholeCamera, cfg: RenderConfig, first_sample: int, sum_dev: int,
                      sum_sq_dev: int | None = None, counts_dev: int | None = None, stats_dev: int | None = None,
                      rank: int = 0, n_ranks: int = 1, stream: int = 0) -> None:
    """Progressive frames: adds samples [first_sample, first_sample + cfg.spp) into device accumulators in sample
    order; frames covering [0, N) equal one N-spp render bit for bit (raw device pointers, asynchronous)."""
    cam, rc = camera._c(), cfg._c()
    _check(_lib.tv_render_accumulate(grid.handle, C.addressof(cam), C.addressof(rc), int(first_sample), int(rank),
                                     int(n_ranks), sum_dev, sum_sq_dev, counts_dev, stats_dev, stream))
