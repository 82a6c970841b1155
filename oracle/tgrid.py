"""Test infrastructure (checker only, never shipped): a numpy restatement of the
reference's TGRD v1 grid file (save_grid / load_grid, builder.cpp:184-293).

Pinned against the compiled reference's own save_grid bytes by
tests/test_oracle.py::test_tgrid_restatement_matches_reference.
"""
from __future__ import annotations

import numpy as np

SENTINEL = 0xFFFFFFFFFFFFFFFF  # builder.cpp:186
NO_TET = 0xFFFFFFFF

# builder.cpp:219-232, packed little endian (90 bytes)
TET_RECORD = np.dtype([("verts", "<u4", 4), ("level", "u1"), ("children", "<u8", 2), ("parent", "<u8"),
                       ("neighbors", "<u8", 4), ("normal_ids", "u1", 4), ("mask", "u1"), ("density", "<f4"),
                       ("temperature", "<f4"), ("albedo", "<f4")])
assert TET_RECORD.itemsize == 90


def _id_out(a: np.ndarray) -> np.ndarray:  # builder.cpp:201
    a = a.astype(np.uint64)
    return np.where(a == NO_TET, np.uint64(SENTINEL), a)


def tgrid_bytes(vq: np.ndarray, tets: np.ndarray, roots: np.ndarray) -> bytes:
    """save_grid (builder.cpp:210-235) of reference pools (TET_DTYPE tets)."""
    rec = np.zeros(len(tets), TET_RECORD)
    rec["verts"] = tets["verts"]
    rec["level"] = tets["level"]
    rec["children"] = _id_out(tets["children"])
    rec["parent"] = _id_out(tets["parent"])
    rec["neighbors"] = _id_out(tets["neighbors"])
    rec["normal_ids"] = tets["normal_ids"]
    rec["mask"] = tets["mask"]
    for k in ("density", "temperature", "albedo"):
        rec[k] = tets[k]
    out = [b"TGRD", np.uint32(1).tobytes(), np.uint64(len(vq)).tobytes(),
           np.ascontiguousarray(vq, "<u4").tobytes(), np.uint64(len(tets)).tobytes(), rec.tobytes(),
           _id_out(np.asarray(roots, np.uint32)).astype("<u8").tobytes()]
    return b"".join(out)
