"""DenseVolume in HBM (volume.hpp:19-58) and its .dvol file (volume.cpp:84-138).

Channels are named f32 arrays (x fastest, shape (nz, ny, nx) on the host side)
held by the library on one GPU; ``generate`` / ``add_temperature`` /
``add_albedo`` are the reference CLI's ``gen`` (cli.cpp:349-380) on the device.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

from . import (BuildConfig, BuildStats, PinholeCamera, TetGrid, _BuildStats, _check, _lib, _sig, _F, _P)

KINDS = {"constant": 0, "ramp": 1, "blob": 2, "step": 3, "noise": 4, "cloud": 5}

_I3 = C.c_int32 * 3
_sig("tv_volume_create", C.c_int, C.c_int32, C.c_int32, C.c_int32, C.c_int, C.POINTER(_P))
_sig("tv_volume_load", C.c_int, C.c_char_p, C.c_int, C.POINTER(_P))
_sig("tv_volume_save", C.c_int, _P, C.c_char_p)
_sig("tv_volume_free", None, _P)
_sig("tv_volume_get_info", C.c_int, _P, C.POINTER(C.c_int32), C.POINTER(C.c_int32))
_sig("tv_volume_channel_name", C.c_int, _P, C.c_int32, C.c_char_p, C.c_int32)
_sig("tv_volume_channel_dev", C.c_int, _P, C.c_char_p, C.POINTER(_P))
_sig("tv_volume_add_channel", C.c_int, _P, C.c_char_p)
_sig("tv_volume_upload", C.c_int, _P, C.c_char_p, _F)
_sig("tv_volume_download", C.c_int, _P, C.c_char_p, _F)
_sig("tv_volume_generate", C.c_int, _P, C.c_int32, C.c_double)
_sig("tv_volume_add_temperature", C.c_int, _P)
_sig("tv_volume_add_albedo", C.c_int, _P, C.c_double)
_sig("tv_build_volume", C.c_int, _P, C.c_void_p, C.c_void_p, C.POINTER(_P), C.POINTER(_BuildStats))


class DenseVolume:
    """A DenseVolume resident in one GPU's HBM (opaque ``tv_volume`` handle)."""

    def __init__(self, handle):
        self._h = handle

    @classmethod
    def create(cls, nx: int, ny: int, nz: int, device: int = 0) -> "DenseVolume":
        """volume.hpp:25: a zero-filled "density" channel."""
        h = _P()
        _check(_lib.tv_volume_create(int(nx), int(ny), int(nz), int(device), C.byref(h)))
        return cls(h)

    @classmethod
    def load(cls, path, device: int = 0) -> "DenseVolume":
        """DenseVolume::load_dvol, streamed file -> HBM."""
        h = _P()
        _check(_lib.tv_volume_load(os.fsencode(path), int(device), C.byref(h)))
        return cls(h)

    @classmethod
    def generate(cls, kind: str, dims, value: float = 1.0, with_temperature: bool = False,
                 albedo: float | None = None, device: int = 0) -> "DenseVolume":
        """cmd_gen (cli.cpp:349-380) on the device; kind adds 'cloud'."""
        if kind not in KINDS:
            from . import ConfigError
            raise ConfigError(f"unknown kind '{kind}' (constant|ramp|blob|step|noise|cloud)")
        nx, ny, nz = dims
        v = cls.create(nx, ny, nz, device)
        _check(_lib.tv_volume_generate(v.handle, KINDS[kind], float(value)))
        if with_temperature:
            v.add_temperature()
        if albedo is not None:
            v.add_albedo(albedo)
        return v

    @property
    def handle(self):
        if not self._h:
            raise ValueError("volume is closed")
        return self._h

    @property
    def dims(self):
        d = _I3()
        _check(_lib.tv_volume_get_info(self.handle, d, None))
        return int(d[0]), int(d[1]), int(d[2])

    def channel_names(self) -> list:
        n = C.c_int32()
        _check(_lib.tv_volume_get_info(self.handle, None, C.byref(n)))
        out = []
        buf = C.create_string_buffer(256)
        for i in range(n.value):
            _check(_lib.tv_volume_channel_name(self.handle, i, buf, 256))
            out.append(buf.value.decode())
        return out

    def has_channel(self, name: str) -> bool:
        return name in self.channel_names()

    def channel_dev(self, name: str = "density") -> int:
        p = _P()
        _check(_lib.tv_volume_channel_dev(self.handle, name.encode(), C.byref(p)))
        return p.value

    def channel(self, name: str = "density") -> np.ndarray:
        nx, ny, nz = self.dims
        out = np.empty((nz, ny, nx), np.float32)
        _check(_lib.tv_volume_download(self.handle, name.encode(), out.ctypes.data_as(_F)))
        return out

    def add_channel(self, name: str, data: np.ndarray | None = None):
        _check(_lib.tv_volume_add_channel(self.handle, name.encode()))
        if data is not None:
            self.set_channel(name, data)

    def set_channel(self, name: str, data: np.ndarray):
        nx, ny, nz = self.dims
        a = np.ascontiguousarray(data, np.float32)
        if a.size != nx * ny * nz:
            raise ValueError("channel size does not match the volume")
        _check(_lib.tv_volume_upload(self.handle, name.encode(), a.ctypes.data_as(_F)))

    def add_temperature(self):
        """temperature = clamp(density, 0, 1) (cli.cpp:370-375)"""
        _check(_lib.tv_volume_add_temperature(self.handle))

    def add_albedo(self, value: float):
        """constant albedo channel (cli.cpp:376-380)"""
        _check(_lib.tv_volume_add_albedo(self.handle, float(value)))

    def save(self, path):
        """DenseVolume::save_dvol"""
        _check(_lib.tv_volume_save(self.handle, os.fsencode(path)))

    def close(self):
        if getattr(self, "_h", None):
            _lib.tv_volume_free(self._h)
            self._h = None

    def __del__(self):
        self.close()

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()


def build_adaptive_grid_volume(vol: DenseVolume, cfg: BuildConfig, camera: PinholeCamera | None = None):
    """build_adaptive_grid(DenseVolume, cfg, camera) (builder.hpp:51-52): density plus the optional
    temperature / albedo channels. -> (TetGrid, BuildStats)"""
    h = _P()
    st = _BuildStats()
    bc = cfg._c()
    cam = camera._c() if camera is not None else None
    _check(_lib.tv_build_volume(vol.handle, C.addressof(bc), C.addressof(cam) if cam is not None else None, C.byref(h),
                                C.byref(st)))
    return TetGrid(h), BuildStats(**{k: getattr(st, k) for k, _ in _BuildStats._fields_})
