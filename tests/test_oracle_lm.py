"""LM-HALP in the CPU oracle (optimizers.cpp:461-627, objectives.cpp:110-133):
the reference's own LM unit tests restated (tests/test_optimizers.cpp:303-329,
469-500; tests/test_objectives.cpp:310-356; acceptance check 8), plus the
host quantizer of the library against the oracle's (CPU only)."""
import math

import numpy as np
import pytest

import paper_1803_03383_b200 as H


def cls_data(oracle):
    ds = H.harness.make_classification(60, 5, 3, 2.0, 4)
    return ds.X, ds.labels


def test_quantize_dataset(oracle):
    X, _ = oracle.make_regression(40, 6, 0.0, 13)
    q = oracle.quantize_dataset(X, 8, 99)
    assert q.delta == pytest.approx(np.abs(X).max() / 127.0, rel=1e-15)
    err = np.abs(q.codes * q.delta - X)
    assert err.max() <= q.delta * (1 + 1e-12) and err.mean() <= q.delta / 2
    q2 = oracle.quantize_dataset(X, 8, 99)
    assert np.array_equal(q.codes, q2.codes)
    z = oracle.quantize_dataset(np.zeros((3, 2)), 8, 1)
    assert z.delta == 1.0 and (z.codes == 0).all()
    # the library's host quantizer (run_prepared / quantize_dataset) is the same restatement
    ds = H.Dataset(X, targets=np.zeros(40))
    H.quantize_dataset(ds, 8, 99)
    assert np.array_equal(ds.quantized.codes, q.codes) and ds.quantized.delta == q.delta
    assert H.data_scale(np.zeros((2, 2)), 8) == 1.0


@pytest.mark.parametrize("mirror", [False, True])
def test_integer_purity_and_scale_chain(oracle, mirror):
    X, lab = cls_data(oracle)
    q = oracle.quantize_dataset(X, 8, 9)
    o = oracle.OracleObjective(X, labels=lab, num_classes=3)
    cfg = oracle.OracleConfig(alpha=0.05, epochs=2, bits=8, mu=3.0, seed=11)
    rec = oracle.run_lm_halp(o, q, cfg, plan={"fg_splits": 4} if mirror else None)
    assert rec.status == "ok" and rec.inner_fp_vector_ops == 0 and rec.inner_lp_vector_ops > 0
    assert rec.rows[-1]["loss"] < rec.rows[0]["loss"]
    for row in rec.rows:
        if row["grad_norm"] == 0.0:
            continue
        assert row["delta_aux"] > 0.0
        assert row["delta_inner"] == row["delta_aux"] * q.delta
        assert row["delta"] == math.ldexp(row["delta_inner"], 8)
        target = max(oracle.halp_scale(row["grad_norm"], 3.0, 8), cfg.delta_min)
        assert abs(row["delta"] - target) <= 1e-12 * target


def test_converged_at_exact_optimum(oracle):
    X, y = oracle.make_regression(30, 4, 0.0, 8)
    q = oracle.quantize_dataset(X, 8, 5)
    o = oracle.OracleObjective(X, y=np.zeros(30))
    rec = oracle.run_lm_halp(o, q, oracle.OracleConfig(alpha=0.02, epochs=3, bits=8, mu=3.0, seed=11))
    assert rec.status == "converged" and rec.steps_taken == 0 and len(rec.rows) == 1


def test_determinism_and_seed(oracle):
    X, y = oracle.make_regression(80, 6, 0.2, 5)
    q = oracle.quantize_dataset(X, 8, 21)
    o = oracle.OracleObjective(X, y=y)
    c = oracle.OracleConfig(alpha=0.02, epochs=3, inner_steps=40, bits=8, mu=3.0, seed=11)
    a, b = oracle.run_lm_halp(o, q, c), oracle.run_lm_halp(o, q, c)
    assert [r["iterate_hash"] for r in a.rows] == [r["iterate_hash"] for r in b.rows]
    c.seed = 12
    assert not np.array_equal(oracle.run_lm_halp(o, q, c).final_iterate, a.final_iterate)


def test_validation(oracle):
    X, y = oracle.make_regression(30, 4, 0.1, 2)
    o = oracle.OracleObjective(X, y=y)
    q = oracle.quantize_dataset(X, 8, 1)
    with pytest.raises(oracle.OracleInvalidInput, match="no quantized"):
        oracle.run_lm_halp(o, None, oracle.OracleConfig(epochs=1, bits=8, mu=3.0))
    with pytest.raises(oracle.OracleInvalidInput, match="different width"):
        oracle.run_lm_halp(o, q, oracle.OracleConfig(epochs=1, bits=16, mu=3.0))
    with pytest.raises(oracle.OracleInvalidInput, match="last-iterate"):
        oracle.run_lm_halp(o, q, oracle.OracleConfig(epochs=1, bits=8, mu=3.0, option=1))
    with pytest.raises(oracle.OracleInvalidInput, match="<= 32"):
        oracle.run_lm_halp(o, oracle.quantize_dataset(X, 40, 1), oracle.OracleConfig(epochs=1, bits=40, mu=3.0))
