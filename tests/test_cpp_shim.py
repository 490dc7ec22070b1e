"""The C++ drop-in header include/halp_lpopt.hpp compiles against the C ABI
(CPU) and, on a B200, reproduces the Python API's run bit for bit on the
reference's golden problem (halp-8, seed 1, 4 epochs)."""
import os
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
EXE = os.path.join(ROOT, "build", "shim_example")


def _build():
    from paper_1803_03383_b200 import build

    build.build()
    os.makedirs(os.path.join(ROOT, "build"), exist_ok=True)
    subprocess.run(["g++", "-O2", "-std=c++17", "-I", os.path.join(ROOT, "include"),
                    os.path.join(ROOT, "tests", "cpp", "shim_example.cpp"), "-o", EXE,
                    "-L", os.path.join(ROOT, "paper_1803_03383_b200"), "-lhalp_b200",
                    "-Wl,-rpath," + os.path.join(ROOT, "paper_1803_03383_b200")], check=True)


def test_shim_compiles():
    _build()
    assert os.path.exists(EXE)


@pytest.mark.gpu
def test_shim_matches_python_api(oracle, tmp_path):
    _build()
    import paper_1803_03383_b200 as H

    X, y = oracle.make_regression(1000, 100, 0.0, 42)
    f = tmp_path / "prob.bin"
    with open(f, "wb") as fh:
        fh.write(np.int64(1000).tobytes() + np.int32(100).tobytes() + X.tobytes() + y.tobytes())
    out = subprocess.run([EXE, str(f)], capture_output=True, text=True)
    assert out.returncode == 0, out.stderr
    lines = out.stdout.strip().splitlines()
    lm_line = [l.split() for l in lines if l.startswith("lm ")]
    cpp_rows = [line.split() for line in lines if not line.startswith("lm ")]
    # the C++ run_prepared(LmHalp, data_seed 7) equals the Python one
    ds = H.Dataset(X, targets=y)
    H.quantize_dataset(ds, 8, 7)
    lrec = H.run_lm_halp(H.Objective(ds, H.LossFamily.Squared, 0.0),
                         H.OptimizerConfig(algorithm=H.Algorithm.LmHalp, alpha=5e-3, epochs=2, inner_steps=2000,
                                           bits=8, mu=3.0, seed=1))
    assert len(lm_line) == 1 and float(lm_line[0][1]) == lrec.rows[-1].loss
    assert float(lm_line[0][2]) == lrec.rows[-1].delta_inner and float(lm_line[0][3]) == lrec.rows[-1].delta_aux
    g = H.Objective(H.Dataset(X, targets=y), H.LossFamily.Squared, 0.0)
    rec = H.run_halp(g, H.OptimizerConfig(algorithm=H.Algorithm.Halp, alpha=5e-3, epochs=4, inner_steps=2000,
                                          bits=8, mu=3.0, seed=1))
    assert len(cpp_rows) == len(rec.rows) == 5
    for c, r in zip(cpp_rows, rec.rows):
        assert float(c[1]) == r.loss and float(c[2]) == r.grad_norm and float(c[3]) == r.delta
        assert int(c[4]) == r.iterate_hash
