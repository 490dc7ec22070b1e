"""run_halp semantics restated from proj/tests/test_optimizers.cpp, checked
on the oracle (the same cases run on the GPU in test_gpu_halp.py)."""
import math

import numpy as np
import pytest


def small_regression(oracle, seed=5, l2=0.0):
    X, y = oracle.make_regression(80, 6, 0.2, seed)
    return oracle.OracleObjective(X, y=y, l2=l2)


def base(oracle, **kw):
    c = oracle.OracleConfig(alpha=0.02, epochs=3, inner_steps=0, seed=11, mu=3.0)
    for k, v in kw.items():
        setattr(c, k, v)
    return c


def test_converged_at_exact_optimum(oracle):
    # test_optimizers.cpp:303-329
    X, y = oracle.make_regression(30, 4, 0.0, 8)
    obj = oracle.OracleObjective(X, y=np.zeros(30))
    rec = oracle.run_halp(obj, base(oracle))
    assert rec.status == "converged" and rec.steps_taken == 0
    assert len(rec.rows) == 1 and rec.rows[0]["grad_norm"] == 0.0 and rec.rows[0]["delta"] == 0.0


def test_delta_tracks_grad_norm(oracle):
    # test_optimizers.cpp:331-370
    obj = oracle.OracleObjective(np.ones((1, 1)), y=np.array([2.0]))
    cfg = base(oracle, bits=8, alpha=0.5, epochs=1, inner_steps=4)
    rec = oracle.run_halp(obj, cfg)
    assert rec.rows[0]["grad_norm"] == 2.0
    assert rec.rows[0]["delta"] == oracle.halp_scale(2.0, 3.0, 8)
    cfg.delta_min = 1.0
    assert oracle.run_halp(obj, cfg).rows[0]["delta"] == 1.0
    X, y = oracle.make_regression(200, 10, 0.0, 14)
    reg = oracle.OracleObjective(X, y=y)
    rows = oracle.run_halp(reg, base(oracle, alpha=0.05, epochs=6)).rows
    assert len(rows) >= 3 and rows[-1]["delta"] < 0.1 * rows[0]["delta"]
    for a, b in zip(rows, rows[1:]):
        assert b["delta"] <= a["delta"] * 1.5


def test_zero_epochs(oracle):
    obj = small_regression(oracle)
    rec = oracle.run_halp(obj, base(oracle, epochs=0))
    assert len(rec.rows) == 1 and rec.rows[0]["pass_"] == 0.0 and rec.steps_taken == 0
    assert np.all(rec.final_iterate == 0)


def test_deterministic_in_seed(oracle):
    obj = small_regression(oracle, 7)
    cfg = base(oracle, bits=8, inner_steps=40)
    r1, r2 = oracle.run_halp(obj, cfg), oracle.run_halp(obj, cfg)
    assert [(a["loss"], a["iterate_hash"]) for a in r1.rows] == [(a["loss"], a["iterate_hash"]) for a in r2.rows]
    assert np.array_equal(r1.final_iterate, r2.final_iterate)
    cfg.seed = 12
    assert not np.array_equal(oracle.run_halp(obj, cfg).final_iterate, r1.final_iterate)
    passes = [r["pass_"] for r in r1.rows]
    assert all(b > a for a, b in zip(passes, passes[1:]))


def test_sampled_iterate_option(oracle):
    obj = small_regression(oracle)
    rec = oracle.run_halp(obj, base(oracle, option=1))
    assert rec.rows[-1]["loss"] < rec.rows[0]["loss"]


def test_metric_gating(oracle):
    obj = small_regression(oracle)
    rec = oracle.run_halp(obj, base(oracle, inner_steps=80, epochs=3, metric_every_passes=2.0))
    assert [r["pass_"] for r in rec.rows] == [0.0, 2.0, 3.0]


def test_divergence_blowup(oracle):
    # mid-epoch non-finite update -> blowup row (inf, inf, delta), status diverged
    obj = oracle.OracleObjective(np.array([[2.0]]), y=np.array([3.0]))
    rec = oracle.run_halp(obj, base(oracle, alpha=1e308, epochs=2, inner_steps=3))
    assert rec.rc == 2 and rec.status == "diverged"
    assert math.isinf(rec.rows[-1]["loss"]) and math.isinf(rec.rows[-1]["grad_norm"])
    assert rec.rows[-1]["pass_"] == 1.0  # (steps + t + 1) / n with t = 0


def test_validation(oracle):
    obj = small_regression(oracle)
    for bad in (dict(alpha=-1.0), dict(epochs=-1), dict(mu=0.0), dict(bits=1), dict(bits=65),
                dict(delta_min=0.0), dict(divergence_limit=float("inf"))):
        with pytest.raises(oracle.OracleInvalidInput):
            oracle.run_halp(obj, base(oracle, **bad))


def test_fullgrad_thread_invariance(oracle):
    # test_objectives.cpp:230-238
    X, y = oracle.make_regression(3000, 9, 0.5, 77)
    obj = oracle.OracleObjective(X, y=y, l2=1e-4)
    w = np.random.default_rng(6).standard_normal(9)
    g1 = obj.full_gradient(w, 1)
    for t in (2, 3, 8):
        assert np.array_equal(g1, obj.full_gradient(w, t))


def test_fullgrad_is_mean_of_components_softmax(oracle):
    # test_objectives.cpp:194-204
    rng = np.random.default_rng(23)
    X = rng.standard_normal((50, 5))
    lab = rng.integers(0, 3, 50)
    obj = oracle.OracleObjective(X, labels=lab, num_classes=3, l2=1e-3)
    w = rng.standard_normal(15)
    mean = sum(obj.component_gradient(i, w) for i in range(50)) / 50
    g = obj.full_gradient(w)
    assert np.linalg.norm(g - mean) / np.linalg.norm(g) < 1e-12
    # uniform logits at w = 0: loss is ln C (test_objectives.cpp:279-284)
    assert obj.loss_value(np.zeros(15)) == pytest.approx(math.log(3.0), rel=1e-12)


def test_fd_gradients(oracle):
    # test_objectives.cpp:171-192
    rng = np.random.default_rng(2)
    X, y = oracle.make_regression(40, 6, 0.3, 17)
    objs = [oracle.OracleObjective(X, y=y, l2=1e-2),
            oracle.OracleObjective(rng.standard_normal((40, 4)), labels=rng.integers(0, 3, 40), num_classes=3, l2=1e-2)]
    for o in objs:
        w = rng.standard_normal(o.dim)
        g = o.full_gradient(w)
        fd = np.zeros_like(g)
        for k in range(o.dim):
            e = np.zeros_like(w)
            e[k] = 1e-6
            fd[k] = (o.loss_value(w + e) - o.loss_value(w - e)) / 2e-6
        assert np.linalg.norm(g - fd) / max(1.0, np.linalg.norm(fd)) <= 1e-5
