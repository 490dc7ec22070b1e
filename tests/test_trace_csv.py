"""Trace writers: format_double (text.hpp:12-19) and
write_run_csv (harness.cpp:246-261).  format_double is checked against
std::to_chars itself (g++, tests/cpp/to_chars_check.cpp) on random and edge
values, and against every number string of the reference's golden CSVs
(parse -> format reproduces the reference's bytes)."""
import csv
import json
import os
import struct
import subprocess

import numpy as np
import pytest

HERE = os.path.dirname(os.path.abspath(__file__))
GOLD = json.load(open(os.path.join(HERE, "golden", "regression_floor.json")))


def test_format_double_matches_to_chars(tmp_path):
    from paper_1803_03383_b200.halp import format_double

    exe = tmp_path / "to_chars"
    r = subprocess.run(["g++", "-std=c++17", "-O1", "-o", str(exe), os.path.join(HERE, "cpp", "to_chars_check.cpp")],
                       capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    rng = np.random.default_rng(0)
    vals = list(rng.standard_normal(4000) * 10.0 ** rng.integers(-30, 30, 4000))
    vals += list(rng.integers(0, 2**62, 3000).astype(np.float64))
    vals += list(np.frombuffer(rng.integers(0, 2**63, 3000, dtype=np.uint64).tobytes(), dtype=np.float64))
    vals += [0.0, -0.0, 1.0, 100.0, 1e5, 1e-5, 1e15, 1e16, 1e17, 1e21, 1e22, 5e-324, 2.2250738585072014e-308,
             1.7976931348623157e308, 0.1, 0.5, 123456.0, 1234567.0, 0.001, 0.0001, 2.5e-06, 1e12]
    vals = [v for v in vals if np.isfinite(v)]
    inp = "\n".join("%016x" % struct.unpack("<Q", struct.pack("<d", v))[0] for v in vals) + "\n"
    out = subprocess.run([str(exe)], input=inp, capture_output=True, text=True).stdout.splitlines()
    assert len(out) == len(vals)
    bad = [(v, a, format_double(v)) for v, a in zip(vals, out) if a != format_double(v)]
    assert not bad, bad[:5]


def test_format_double_reproduces_golden_csv_strings():
    from paper_1803_03383_b200.halp import format_double

    n = 0
    for rows in GOLD["traces"].values():
        for row in rows:
            for k in ("pass", "seconds", "loss", "grad_norm", "delta"):
                assert format_double(float(row[k])) == row[k], (k, row[k])
                n += 1
    assert n >= 25 * 26 * 5


def test_write_run_csv_layout(tmp_path):
    import paper_1803_03383_b200 as H

    gold = GOLD["traces"]["halp-8_seed1"]
    rec = H.RunRecord(rows=[H.MetricRow(float(r["pass"]), float(r["seconds"]), float(r["loss"]),
                                        float(r["grad_norm"]), float(r["delta"])) for r in gold])
    path = tmp_path / "halp-8_seed1.csv"
    H.write_run_csv(str(path), rec)
    text = path.read_text()
    lines = text.splitlines()
    assert lines[0] == "pass,seconds,loss,grad_norm,delta" and text.endswith("\n")
    assert [dict(zip(lines[0].split(","), l.split(","))) for l in lines[1:]] == gold
