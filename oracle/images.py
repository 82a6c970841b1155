"""Test infrastructure (checker only, never shipped): numpy restatements of the
reference's output formats and compare metrics, pinned to the compiled
reference by tests/test_oracle.py:

  * write_pfm / write_variance_pfm / read_pfm (image.cpp:33-101) with
    ImageAccumulator::mean / variance_of_mean (image.hpp:47-69);
  * DenseVolume::save_dvol (volume.cpp:84-100);
  * cmd_compare's rmse / maxAbsDiff / outlierFraction (cli.cpp:493-531), with
    the squared differences summed sequentially as the reference does.
"""
from __future__ import annotations

import numpy as np


def mean_f32(s: np.ndarray, counts: np.ndarray) -> np.ndarray:
    """flat (W*H, 3) f32 of ImageAccumulator::mean."""
    n = counts.reshape(-1, 1).astype(np.float64)
    out = np.zeros((n.shape[0], 3))
    nz = n[:, 0] > 0
    out[nz] = s.reshape(-1, 3)[nz] / n[nz]
    return out.astype(np.float32)


def variance_f32(s: np.ndarray, q: np.ndarray, counts: np.ndarray) -> np.ndarray:
    n = counts.reshape(-1, 1).astype(np.float64)
    out = np.zeros((n.shape[0], 3))
    ok = n[:, 0] >= 2
    m = s.reshape(-1, 3)[ok] / n[ok]
    var = (q.reshape(-1, 3)[ok] - n[ok] * m * m) / (n[ok] - 1.0)
    out[ok] = np.where(0.0 < var, var, 0.0) / n[ok]
    return out.astype(np.float32)


def pfm_bytes(rgb_top_down: np.ndarray, w: int, h: int) -> bytes:
    """image.cpp:35-45: header, rows bottom to top, little-endian f32."""
    rows = np.ascontiguousarray(rgb_top_down, "<f4").reshape(h, w * 3)[::-1]
    return f"PF\n{w} {h}\n-1.000000\n".encode() + rows.tobytes()


def dvol_bytes(dims, channels: dict) -> bytes:
    """volume.cpp:84-100; channels in insertion order, each (nz, ny, nx) f32."""
    nx, ny, nz = dims
    out = [b"DVOL", np.array([1, nx, ny, nz, len(channels)], "<u4").tobytes()]
    for name in channels:
        out += [bytes([len(name)]), name.encode()]
    for a in channels.values():
        out.append(np.ascontiguousarray(a, "<f4").tobytes())
    return b"".join(out)


def compare(a: np.ndarray, b: np.ndarray, va: np.ndarray | None = None, vb: np.ndarray | None = None) -> dict:
    """cli.cpp:499-528 on flat f32 arrays (3 values per pixel)."""
    d = a.astype(np.float64).ravel() - b.astype(np.float64).ravel()
    sq = np.cumsum(d * d)[-1] if d.size else 0.0  # sequential left-to-right, as the reference loop
    out = dict(rmse=float(np.sqrt(sq / d.size)), maxAbsDiff=float(np.abs(d).max()) if d.size else 0.0,
               outlierFraction=None)
    if va is not None:
        s = va.astype(np.float64).ravel() + vb.astype(np.float64).ravel()
        sigma = np.sqrt(np.where(0.0 < s, s, 0.0))
        bad = (np.abs(d) > 3.0 * sigma).reshape(-1, 3).any(axis=1)
        out["outlierFraction"] = float(bad.sum()) / bad.size
        out["outliers"] = int(bad.sum())
    return out
