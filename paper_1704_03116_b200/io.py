"""Run outputs in the reference's file formats.

``write_trace`` writes the per-iteration trace CSV of io.py:214-224 (columns
iter, mu, energy, residual, max_block_residual, ms; floats as ``repr``),
``write_report`` the sorted-key JSON report (io.py:227-230), and
``write_labels`` a binary label map as PGM (2D, 0/255) or raw uint8 with a
descriptor (3D) -- so ``dope compare``-style tooling can read B200 runs.
"""
from __future__ import annotations

import csv
import json

import numpy as np

from .grid import GridShape

TRACE_FIELDS = ("iter", "mu", "energy", "residual", "max_block_residual", "ms")


def write_trace(path, trace) -> None:
    with open(path, "w", encoding="utf-8", newline="") as f:
        out = csv.writer(f)
        out.writerow(TRACE_FIELDS)
        for t in trace:
            out.writerow([t.iteration, repr(float(t.mu)), repr(float(t.energy)), repr(float(t.residual_sq)),
                          repr(float(t.max_block_residual)), repr(float(t.wall_ms))])


def write_report(path, report: dict) -> None:
    """Sorted-key JSON with a trailing newline, byte for byte the reference's format."""
    with open(path, "w", encoding="utf-8") as f:
        json.dump(report, f, sort_keys=True, indent=2)
        f.write("\n")


def write_labels(path_base, labels, shape: GridShape) -> str:
    """PGM (P5, maxval 255) for 2D label maps; raw uint8 + JSON descriptor for 3D."""
    lab = (np.asarray(labels).ravel() != 0).astype(np.uint8) * 255
    if shape.ndim == 2:
        h, w = shape.dims
        path = str(path_base) + ".pgm"
        with open(path, "wb") as f:
            f.write(f"P5\n{w} {h}\n255\n".encode("ascii"))
            f.write(lab.tobytes())
        return path
    path = str(path_base) + ".raw"
    lab.tofile(path)
    with open(path + ".json", "w", encoding="utf-8") as f:
        json.dump({"dims": [int(d) for d in shape.dims], "channels": 1, "dtype": "uint8"}, f, sort_keys=True)
        f.write("\n")
    return path
