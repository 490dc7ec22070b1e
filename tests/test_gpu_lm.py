"""LM-HALP on the B200 (k_lm.cu: K7 epoch stats + K8 integer inner loop)
against the oracle (optimizers.cpp:461-627).  MIRROR order: rows (loss, grad
norm, the three scales, iterate hash), final iterate and every z code of the
first inner steps bit-identical.  REF order: the number of inner steps whose
codes differ (the inner loop is integer arithmetic; only the fp64 logits at
w~ and the link derivative depend on the order) must be 0."""
import math

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def H():
    import paper_1803_03383_b200 as H
    from paper_1803_03383_b200 import build

    build.build()
    return H


def rows_equal(grows, orows):
    assert len(grows) == len(orows)
    for a, b in zip(grows, orows):
        assert a.pass_ == b["pass_"]
        for f in ("loss", "grad_norm", "delta", "delta_inner", "delta_aux"):
            assert getattr(a, f) == b[f], (f, a, b)
        assert a.iterate_hash == b["iterate_hash"], (a, b)


CASES = [
    # (kind, n, d, C, bits, alpha, mu, T, epochs)
    ("squared", 800, 24, 1, 8, 0.02, 3.0, 1600, 4),
    ("squared", 3000, 100, 1, 16, 5e-3, 3.0, 2000, 3),
    ("softmax", 600, 5, 3, 8, 0.05, 3.0, 1200, 3),
    ("softmax", 2000, 64, 10, 8, 0.02, 2.5, 2000, 2),
    ("softmax", 1500, 300, 10, 16, 0.01, 2.5, 1000, 2),  # D = 3000: 12 coordinates per thread
]


@pytest.mark.parametrize("case", CASES)
def test_lm_bitexact_vs_mirror(H, oracle, case):
    kind, n, d, C, bits, alpha, mu, T, K = case
    if kind == "squared":
        X, y = oracle.make_regression(n, d, 0.1, 7)
        ds = H.Dataset(X, targets=y)
        o = oracle.OracleObjective(X, y=y, l2=1e-4)
        loss = H.LossFamily.Squared
    else:
        ds = H.harness.make_classification(n, d, C, 3.0, 4)
        X, y = ds.X, ds.labels
        o = oracle.OracleObjective(X, labels=y, num_classes=C, l2=1e-4)
        loss = H.LossFamily.Softmax
    H.quantize_dataset(ds, bits, 9)
    q = oracle.OracleQuantized(ds.quantized.codes, ds.quantized.delta, bits)
    g = H.Objective(ds, loss, 1e-4)
    cfg = H.OptimizerConfig(algorithm=H.Algorithm.LmHalp, alpha=alpha, epochs=K, inner_steps=T, bits=bits, mu=mu,
                            seed=6)
    D = d * C
    steps = 300
    tr = np.zeros(steps * D, dtype=np.int64)
    rec = H.run_lm_halp(g, cfg, trace=tr)
    ocfg = oracle.OracleConfig(alpha=alpha, epochs=K, inner_steps=T, bits=bits, mu=mu, seed=6)
    mir = oracle.run_lm_halp(o, q, ocfg, plan=g.oracle_plan(), trace_steps=steps, hash_steps=K * T)
    rows_equal(rec.rows, mir.rows)
    assert np.array_equal(rec.final_iterate, mir.final_iterate)
    assert np.array_equal(tr.reshape(steps, D), mir.trace)
    assert rec.inner_fp_vector_ops == 0 and rec.inner_lp_vector_ops == mir.inner_lp_vector_ops > 0
    assert rec.steps_taken == K * T and rec.status == "ok"
    ref = oracle.run_lm_halp(o, q, ocfg, hash_steps=K * T)
    mism = int((ref.step_hash != mir.step_hash).sum())
    assert mism == 0, mism
    for a, b in zip(rec.rows, ref.rows):
        assert abs(a.loss - b["loss"]) <= 1e-9 * max(abs(b["loss"]), abs(ref.rows[0]["loss"]))
    assert rec.rows[-1].loss < rec.rows[0].loss


def test_lm_converged_and_validation(H, oracle):
    X, _ = oracle.make_regression(30, 4, 0.0, 8)
    ds = H.Dataset(X, targets=np.zeros(30))
    H.quantize_dataset(ds, 8, 5)
    g = H.Objective(ds, H.LossFamily.Squared, 0.0)
    rec = H.run_lm_halp(g, H.OptimizerConfig(algorithm=H.Algorithm.LmHalp, alpha=0.02, epochs=3, bits=8, mu=3.0,
                                             seed=11))
    assert rec.status == "converged" and rec.steps_taken == 0 and len(rec.rows) == 1
    X, y = oracle.make_regression(30, 4, 0.1, 2)
    plain = H.Objective(H.Dataset(X, targets=y), H.LossFamily.Squared, 0.0)
    lm = H.OptimizerConfig(algorithm=H.Algorithm.LmHalp, alpha=0.02, epochs=1, bits=8, mu=3.0)
    with pytest.raises(H.InvalidInputError, match="no quantized"):
        H.run(plain, lm)
    ds = H.Dataset(X, targets=y)
    H.quantize_dataset(ds, 8, 1)
    qobj = H.Objective(ds, H.LossFamily.Squared, 0.0)
    bad = H.OptimizerConfig(algorithm=H.Algorithm.LmHalp, alpha=0.02, epochs=1, bits=16, mu=3.0)
    with pytest.raises(H.InvalidInputError, match="different width"):
        H.run(qobj, bad)
    with pytest.raises(H.InvalidInputError, match="last-iterate"):
        H.run(qobj, H.OptimizerConfig(algorithm=H.Algorithm.LmHalp, alpha=0.02, epochs=1, bits=8, mu=3.0,
                                      option=H.EpochOption.SampledIterate))
    # run_prepared quantizes a copy with the data seed (harness.cpp:299-306)
    r = H.run_prepared(plain, H.OptimizerConfig(algorithm=H.Algorithm.LmHalp, alpha=0.02, epochs=2, bits=8, mu=3.0,
                                                seed=3), data_seed=4)
    assert r.status == "ok" and r.rows[-1].loss < r.rows[0].loss


def test_lm_in_experiment(H, tmp_path):
    """tests/test_harness.cpp:270-295: an LM-HALP config and a diverging SGD
    config in one run_experiment"""
    from paper_1803_03383_b200 import harness as HR

    spec = HR.experiment_from_json({
        "dataset": {"kind": "regression", "n": 60, "d": 5, "noise_sd": 0.1, "seed": 3},
        "configs": [{"name": "lm-halp-8", "algo": "lm-halp", "alpha": 0.02, "epochs": 2, "bits": 8, "mu": 3.0},
                    {"name": "sgd-hot", "algo": "sgd", "alpha": 1e6, "epochs": 2, "divergence_limit": 1e8}],
        "seeds": [3], "out": str(tmp_path)})
    res = HR.run_experiment(spec)
    assert res.runs[0].status == "ok" and res.runs[0].final_loss < 1e6
    assert res.runs[1].status == "diverged"
    rows = HR.read_run_csv(str(tmp_path / res.runs[1].csv_path))
    assert not math.isfinite(rows[-1].loss) or rows[-1].loss > 1e8


def test_lm_device_resident_dataset(H, oracle):
    """X already in HBM (torch): the codes stay host arrays; same run as host X"""
    import torch

    X, y = oracle.make_regression(500, 16, 0.1, 3)
    ds_h = H.Dataset(X, targets=y)
    H.quantize_dataset(ds_h, 8, 2)
    ds_d = H.Dataset(torch.as_tensor(X, device="cuda"), targets=torch.as_tensor(y, device="cuda"))
    H.quantize_dataset(ds_d, 8, 2)
    assert np.array_equal(ds_d.quantized.codes, ds_h.quantized.codes)
    cfg = H.OptimizerConfig(algorithm=H.Algorithm.LmHalp, alpha=0.02, epochs=2, inner_steps=600, bits=8, mu=3.0, seed=1)
    a = H.run_lm_halp(H.Objective(ds_h, H.LossFamily.Squared, 0.0), cfg)
    b = H.run_lm_halp(H.Objective(ds_d, H.LossFamily.Squared, 0.0), cfg)
    assert [r.iterate_hash for r in a.rows] == [r.iterate_hash for r in b.rows]
    assert np.array_equal(a.final_iterate, b.final_iterate)
