"""K5 (batched independent problems, BASELINE C5) against the oracle's MIRROR
order, problem by problem: rows, hashes and final iterates bit-identical."""
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
        for f in ("loss", "grad_norm", "delta"):
            va, vb = getattr(a, f), b[f]
            assert va == vb or (math.isinf(va) and math.isinf(vb)), (f, a, b)
        assert a.iterate_hash == b["iterate_hash"]


@pytest.mark.parametrize("warps", ["", "1", "2", "4"])
@pytest.mark.parametrize("dtype,d", [("f32", 128), ("f64", 100), ("f32", 64), ("f32", 256)])
def test_batch_bitexact_vs_mirror(H, oracle, dtype, d, warps, monkeypatch):
    """every K5 plan (1, 2 or 4 warps per problem; "" = the library's choice)"""
    if warps:
        monkeypatch.setenv("HALP_K5_WARPS", warps)
    P, n = 12, 512
    rng = np.random.default_rng(d)
    X = rng.standard_normal((P, n, d))
    wstar = rng.standard_normal((P, d))
    y = np.einsum("pnd,pd->pn", X, wstar) + 0.1 * rng.standard_normal((P, n))
    Xs = X.astype(np.float32) if dtype == "f32" else X
    b = H.BatchProblems(Xs, y, l2=1e-4)
    alphas = 10 ** rng.uniform(-4, -2, P)
    cfgs = []
    for p in range(P):
        cfgs.append(H.OptimizerConfig(algorithm=H.Algorithm.Halp, alpha=float(alphas[p]), epochs=3,
                                      inner_steps=300 + 7 * p, bits=(8 if p % 2 == 0 else 16), mu=3.0, seed=100 + p,
                                      option=H.EpochOption(1 if p % 3 == 0 else 0)))
    cfgs[5].alpha = 1e308  # blows up in the first epoch
    recs = b.run(cfgs)
    plan = b.oracle_plan()
    for p in range(P):
        o = oracle.OracleObjective(Xs[p], y=y[p], l2=1e-4)
        c = cfgs[p]
        orec = oracle.run_halp(o, oracle.OracleConfig(alpha=c.alpha, epochs=c.epochs, inner_steps=c.inner_steps,
                                                      bits=c.bits, mu=c.mu, seed=c.seed, option=int(c.option)),
                               plan=plan)
        rows_equal(recs[p].rows, orec.rows)
        assert np.array_equal(recs[p].final_iterate, orec.final_iterate), p
        assert recs[p].status == orec.status
        assert recs[p].steps_taken == orec.steps_taken
    assert recs[5].status == "diverged" and math.isinf(recs[5].rows[-1].loss)
    assert b.device_ms > 0


def test_batch_converged_and_gating(H, oracle):
    P, n, d = 4, 64, 8
    rng = np.random.default_rng(3)
    X = rng.standard_normal((P, n, d))
    y = np.zeros((P, n))  # w = 0 is the exact optimum: converged at the first boundary
    y[2:] = rng.standard_normal((2, n))
    b = H.BatchProblems(X, y)
    cfgs = [H.OptimizerConfig(algorithm=H.Algorithm.Halp, alpha=0.01, epochs=4, inner_steps=64, mu=3.0, seed=p,
                              metric_every_passes=2.0 if p == 3 else 0.0) for p in range(P)]
    recs = b.run(cfgs)
    assert recs[0].status == "converged" and len(recs[0].rows) == 1 and recs[0].steps_taken == 0
    for p in (2, 3):
        o = oracle.OracleObjective(X[p], y=y[p])
        c = cfgs[p]
        orec = oracle.run_halp(o, oracle.OracleConfig(alpha=c.alpha, epochs=c.epochs, inner_steps=c.inner_steps,
                                                      mu=c.mu, seed=c.seed, metric_every_passes=c.metric_every_passes),
                               plan=b.oracle_plan())
        rows_equal(recs[p].rows, orec.rows)
    assert len(recs[3].rows) < len(recs[2].rows)
