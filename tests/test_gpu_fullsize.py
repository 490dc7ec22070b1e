"""Parity at BASELINE's full row counts: C3's N = 4,194,304 (the maximum
split grid, S = 4096, and 1024-row splits) and C4's N = 16,777,216 (bf16, two
classes), with narrow rows so the CPU oracle finishes in seconds.  The
full-gradient pass, its loss and a short HALP run are bit-identical to the
oracle's MIRROR order; the split count, rows per split and row-tile tails are
the full-size ones."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def H():
    import paper_1803_03383_b200 as H
    from paper_1803_03383_b200 import build

    build.build()
    return H


def bf16_bits(a):
    u = np.ascontiguousarray(a, dtype=np.float32).view(np.uint32)
    return ((u + 0x7FFF + ((u >> 16) & 1)) >> 16).astype(np.uint16)


def test_c3_rows_least_squares(H, oracle):
    n, d = 4194304, 64
    rng = np.random.default_rng(3)
    X = rng.standard_normal((n, d), dtype=np.float32)
    wstar = rng.standard_normal(d)
    y = X.astype(np.float64) @ wstar + 0.1 * rng.standard_normal(n)
    g = H.Objective(H.Dataset(X, targets=y), H.LossFamily.Squared, 1e-5)
    plan = g.oracle_plan()
    assert plan["fg_splits"] == 4096
    o = oracle.OracleObjective(X, y=y, l2=1e-5)
    w = rng.standard_normal(d) * 0.5
    gg, gl = g._fullpass(w)
    assert np.array_equal(gg, o.full_gradient(w, plan=plan))
    assert gl == o.loss_value(w, plan=plan)
    cfg = H.OptimizerConfig(algorithm=H.Algorithm.Halp, alpha=2e-3, epochs=2, inner_steps=3000, bits=16, mu=1.0,
                            seed=5)
    rec = H.run_halp(g, cfg)
    orec = oracle.run_halp(o, oracle.OracleConfig(alpha=2e-3, epochs=2, inner_steps=3000, bits=16, mu=1.0, seed=5),
                           plan=plan)
    assert [(r.loss, r.grad_norm, r.delta, r.iterate_hash) for r in rec.rows] == \
        [(r["loss"], r["grad_norm"], r["delta"], r["iterate_hash"]) for r in orec.rows]
    assert np.array_equal(rec.final_iterate, orec.final_iterate)


def test_c4_rows_two_class_bf16(H, oracle):
    n, d = 16777216, 16
    rng = np.random.default_rng(4)
    X = rng.standard_normal((n, d), dtype=np.float32) / 4.0
    wstar = rng.standard_normal(d)
    lab = (rng.random(n) < 1.0 / (1.0 + np.exp(-(X @ wstar)))).astype(np.int32)
    Xb = bf16_bits(X)
    g = H.Objective(H.Dataset(Xb, labels=lab, num_classes=2), H.LossFamily.Softmax, 1e-5)
    plan = g.oracle_plan()
    o = oracle.OracleObjective(Xb, labels=lab, num_classes=2, l2=1e-5)
    for w in (rng.standard_normal(2 * d), np.zeros(2 * d)):
        gg, gl = g._fullpass(w)
        assert np.array_equal(gg, o.full_gradient(w, plan=plan))
        assert gl == o.loss_value(w, plan=plan)
