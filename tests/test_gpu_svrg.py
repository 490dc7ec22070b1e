"""SVRG / LP-SVRG / SGD / LP-SGD (optimizers.cpp:229-385) on the HALP kernels:
K1 at the snapshot, K3 in mode 2 (fp64 iterate, no rounding) / mode 1 (the
iterate itself quantized at the fixed scale).  Bit-identical to the oracle's
MIRROR runs (rows, hashes, final iterates, LP codes of every step), and
against the reference's own golden traces svrg / lp-svrg-{8,16}_seed*.csv:
every row within 1e-9 (SVRG) / 1e-14 (LP-SVRG)."""
import json
import math
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "regression_floor.json")))


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
        for f in ("loss", "grad_norm", "delta"):
            va, vb = getattr(a, f), b[f]
            assert va == vb or (math.isnan(va) and math.isnan(vb)), (f, a, b)
        assert a.iterate_hash == b["iterate_hash"], (a, b)


ALGOS = {"svrg": (1, dict(alpha=5e-3), 1e-9), "lp-svrg-8": (3, dict(alpha=5e-3, delta=0.7, bits=8), 1e-14),
         "lp-svrg-16": (3, dict(alpha=5e-3, delta=0.003, bits=16), 1e-14), "sgd": (0, dict(alpha=2.5e-6), 1e-12),
         "lp-sgd-8": (2, dict(alpha=2.5e-6, delta=0.7, bits=8), 1e-14),
         "lp-sgd-16": (2, dict(alpha=2.5e-6, delta=0.003, bits=16), 1e-14)}
OPS = {0: 3, 1: 5, 2: 5, 3: 7}


@pytest.mark.parametrize("name", list(ALGOS))
@pytest.mark.parametrize("seed", [1, 3])
def test_golden_traces(H, oracle, name, seed):
    algo, kw, tol = ALGOS[name]
    X, y = oracle.make_regression(1000, 100, 0.0, 42)
    g = H.Objective(H.Dataset(X, targets=y), H.LossFamily.Squared, 0.0)
    cfg = H.OptimizerConfig(algorithm=H.Algorithm(algo), epochs=25, inner_steps=2000, seed=seed, **kw)
    rec = H.run(g, cfg)
    gold = GOLD["traces"][f"{name}_seed{seed}"]
    assert len(rec.rows) == 26 and rec.status == "ok" and rec.steps_taken == 50000
    assert rec.inner_fp_vector_ops == OPS[algo] * 50000
    for k, (a, b) in enumerate(zip(rec.rows, gold)):
        assert a.pass_ == float(b["pass"])
        for f in ("loss", "grad_norm", "delta"):
            bv = float(b[f])
            assert abs(getattr(a, f) - bv) <= tol * abs(bv), (k, f, getattr(a, f), bv)
    o = oracle.OracleObjective(X, y=y)
    orec = oracle.run(o, oracle.OracleConfig(epochs=25, inner_steps=2000, seed=seed, algorithm=algo, **kw),
                      plan=g.oracle_plan())
    rows_equal(rec.rows, orec.rows)
    assert np.array_equal(rec.final_iterate, orec.final_iterate)


@pytest.mark.parametrize("algo,kw", [(1, {}), (3, dict(delta=0.05, bits=8)), (3, dict(delta=1e-3, bits=16)), (0, {}),
                                     (2, dict(delta=0.05, bits=8))])
@pytest.mark.parametrize("option", [0, 1])
def test_bitexact_vs_mirror(H, oracle, algo, kw, option):
    X, y = oracle.make_regression(700, 37, 0.3, 5)
    X32 = X.astype(np.float32)
    g = H.Objective(H.Dataset(X32, targets=y), H.LossFamily.Squared, 1e-3)
    init = np.random.default_rng(1).standard_normal(37) * 0.1
    cfg = H.OptimizerConfig(algorithm=H.Algorithm(algo), alpha=4e-3, epochs=4, inner_steps=900, seed=11,
                            option=H.EpochOption(option), init=init, **kw)
    steps = 300
    tr = np.zeros(steps * 37, dtype=np.int64) if algo in (2, 3) else None
    rec = {0: H.run_sgd, 1: H.run_svrg}[algo](g, cfg) if tr is None else \
        {2: H.run_lp_sgd, 3: H.run_lp_svrg}[algo](g, cfg, trace=tr)
    o = oracle.OracleObjective(X32, y=y, l2=1e-3)
    orec = oracle.run(o, oracle.OracleConfig(alpha=4e-3, epochs=4, inner_steps=900, seed=11, option=option,
                                             init=init, algorithm=algo, **kw),
                      plan=g.oracle_plan(), trace_steps=steps if tr is not None else 0)
    rows_equal(rec.rows, orec.rows)
    assert np.array_equal(rec.final_iterate, orec.final_iterate)
    if tr is not None:
        assert np.array_equal(tr.reshape(steps, -1), orec.trace)


@pytest.mark.parametrize("algo,kw", [(1, {}), (3, dict(delta=0.01, bits=8)), (0, {}), (2, dict(delta=0.01, bits=8))])
def test_softmax_bitexact(H, oracle, algo, kw):
    rng = np.random.default_rng(4)
    n, d, C = 800, 30, 4
    X = (rng.random((n, d)) * (rng.random((n, d)) < 0.4)).astype(np.float32)
    lab = rng.integers(0, C, n).astype(np.int32)
    g = H.Objective(H.Dataset(X, labels=lab, num_classes=C), H.LossFamily.Softmax, 1e-4)
    cfg = H.OptimizerConfig(algorithm=H.Algorithm(algo), alpha=0.05, epochs=3, inner_steps=n, seed=2, **kw)
    rec = H.run(g, cfg)
    o = oracle.OracleObjective(X, labels=lab, num_classes=C, l2=1e-4)
    orec = oracle.run(o, oracle.OracleConfig(alpha=0.05, epochs=3, inner_steps=n, seed=2, algorithm=algo, **kw),
                      plan=g.oracle_plan())
    rows_equal(rec.rows, orec.rows)
    assert np.array_equal(rec.final_iterate, orec.final_iterate)
    assert rec.rows[-1].loss < rec.rows[0].loss


def test_lp_svrg_blowup_and_svrg_divergence(H, oracle):
    X, y = oracle.make_regression(200, 8, 0.1, 2)
    g = H.Objective(H.Dataset(X, targets=y), H.LossFamily.Squared, 0.0)
    o = oracle.OracleObjective(X, y=y)
    for algo, kw in ((3, dict(delta=0.1, bits=8)), (1, {}), (2, dict(delta=0.1, bits=8)), (0, {})):
        cfg = H.OptimizerConfig(algorithm=H.Algorithm(algo), alpha=1e306, epochs=3, inner_steps=200, seed=1, **kw)
        rec = H.run_prepared(g, cfg)
        orec = oracle.run(o, oracle.OracleConfig(alpha=1e306, epochs=3, inner_steps=200, seed=1, algorithm=algo, **kw),
                          plan=g.oracle_plan())
        assert rec.status == orec.status == "diverged"
        rows_equal(rec.rows, orec.rows)
        assert rec.steps_taken == 0
        with pytest.raises(H.DivergenceError):
            H.run(g, cfg)


def test_validation(H, oracle):
    X, y = oracle.make_regression(50, 4, 0.1, 2)
    g = H.Objective(H.Dataset(X, targets=y), H.LossFamily.Squared, 0.0)
    with pytest.raises(H.InvalidInputError, match="delta must be positive for fixed-scale runs"):
        H.run(g, H.OptimizerConfig(algorithm=H.Algorithm.LpSvrg, delta=0.0))
    with pytest.raises(H.InvalidInputError, match="bits must be in"):
        H.run(g, H.OptimizerConfig(algorithm=H.Algorithm.LpSvrg, delta=0.1, bits=1))
    H.run(g, H.OptimizerConfig(algorithm=H.Algorithm.Svrg, mu=0.0, bits=1))  # SVRG checks neither
    # LmHalp is bit-centred: validate_config rejects mu = 0 first (optimizers.cpp:69-75)
    with pytest.raises(H.InvalidInputError, match="mu must be positive"):
        H.run(g, H.OptimizerConfig(algorithm=H.Algorithm.LmHalp))
