"""Trace / report / label files in the reference's formats (CPU only)."""
import csv
import json

import numpy as np

import paper_1704_03116_b200 as dope
from paper_1704_03116_b200 import io as dio


def test_trace_csv_schema(tmp_path):
    tr = [dope.TraceRecord(1, 1.0, -12.5, 3.0, 1.7320508075688772, 0.25, False),
          dope.TraceRecord(2, 1.05, -13.0, 0.0, 0.0, 0.5, True)]
    p = tmp_path / "trace.csv"
    dio.write_trace(p, tr)
    rows = list(csv.reader(open(p)))
    assert tuple(rows[0]) == ("iter", "mu", "energy", "residual", "max_block_residual", "ms")
    assert rows[1] == ["1", "1.0", "-12.5", "3.0", "1.7320508075688772", "0.25"]
    assert float(rows[2][1]) == 1.05


def test_report_and_labels(tmp_path):
    dio.write_report(tmp_path / "r.json", {"b": 1, "a": [1, 2]})
    assert list(json.load(open(tmp_path / "r.json")).keys()) == ["a", "b"]
    # byte-identical to the reference writer (io.py:227-231: json.dump then "\n")
    assert open(tmp_path / "r.json", "rb").read() == b'{\n  "a": [\n    1,\n    2\n  ],\n  "b": 1\n}\n'
    lab = np.array([0, 1, 1, 0, 1, 0], dtype=np.int8)
    path = dio.write_labels(tmp_path / "lab", lab, dope.GridShape((2, 3)))
    data = open(path, "rb").read()
    assert data.startswith(b"P5\n3 2\n255\n")
    assert list(data[-6:]) == [0, 255, 255, 0, 255, 0]
    p3 = dio.write_labels(tmp_path / "vol", np.ones(8), dope.GridShape((2, 2, 2)))
    assert np.fromfile(p3, dtype=np.uint8).tolist() == [255] * 8
