"""lpopt::grid_search (harness.cpp:379-447) on the B200: every (point, seed)
run of a least-squares grid goes through ONE K5 launch over the shared
dataset.  Each run is bit-identical to the oracle's MIRROR run_halp with the
batch plan, so the grid's per-seed metrics, means, statuses and the selected
point are the reference's own grid logic applied to reference-identical runs.
A softmax objective (not batchable) takes the sequential run_prepared path."""
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


def oracle_grid(oracle, o, base, axes, seeds, plan, metric="grad_norm"):
    """the reference's grid loop (harness.cpp:400-444) over oracle runs"""
    import itertools

    axes = sorted(axes, key=lambda a: a[0])
    pts, best, best_i = [], math.inf, 0
    for pi, combo in enumerate(itertools.product(*[v for _, v in axes])):
        kw = dict(base)
        for (name, _), v in zip(axes, combo):
            kw[{"inner": "inner_steps"}.get(name, name)] = int(round(v)) if name in ("bits", "inner", "epochs") else v
        per = []
        for sd in seeds:
            kw["seed"] = sd
            rec = oracle.run_halp(o, oracle.OracleConfig(**kw), plan=plan)
            m = rec.rows[-1]["loss" if metric == "loss" else "grad_norm"] if rec.rows else math.inf
            if rec.status == "diverged" or not math.isfinite(m):
                m = math.inf
            per.append(m)
        mean = sum(per) / len(per)
        if pi == 0 or mean < best:
            best, best_i = mean, pi
        pts.append(per)
    return pts, best_i


@pytest.mark.parametrize("dtype", ["f64", "f32"])
def test_grid_search_batched_matches_oracle(H, oracle, dtype):
    n, d = 400, 24
    X, y = oracle.make_regression(n, d, 0.2, 9)
    Xs = X.astype(np.float32) if dtype == "f32" else X
    obj = H.Objective(H.Dataset(Xs, targets=y), H.LossFamily.Squared, 1e-4)
    base = H.OptimizerConfig(algorithm=H.Algorithm.Halp, alpha=1e-3, epochs=3, inner_steps=500, bits=8, mu=3.0, seed=77)
    axes = [H.GridAxis("mu", [1.0, 3.0, 10.0]), H.GridAxis("alpha", [2e-3, 2e-2, 1e308])]  # 1e308 blows up
    seeds = [1, 2, 3]
    res = H.grid_search(obj, base, axes, seeds)
    assert len(res.points) == 9
    # axes are visited in name order: alpha outer, mu inner (last axis fastest)
    assert [p.params for p in res.points[:3]] == [{"alpha": 2e-3, "mu": m} for m in (1.0, 3.0, 10.0)]
    plan = H.BatchProblems(Xs, y, l2=1e-4, nprob=1).oracle_plan()
    o = oracle.OracleObjective(Xs, y=y, l2=1e-4)
    pts, best_i = oracle_grid(oracle, o, dict(alpha=1e-3, epochs=3, inner_steps=500, bits=8, mu=3.0),
                              [("mu", [1.0, 3.0, 10.0]), ("alpha", [2e-3, 2e-2, 1e308])], seeds, plan)
    for p, per in zip(res.points, pts):
        assert p.per_seed == per
    assert res.best_index == best_i
    assert res.points[-1].status == "diverged" and math.isinf(res.points[-1].mean_metric)
    assert res.best_config.seed == 77 and res.best_config.alpha == res.points[best_i].params["alpha"]


def test_grid_search_loss_metric_and_bits_axis(H, oracle):
    n, d = 300, 10
    X, y = oracle.make_regression(n, d, 0.1, 4)
    obj = H.Objective(H.Dataset(X, targets=y), H.LossFamily.Squared, 0.0)
    base = H.OptimizerConfig(algorithm=H.Algorithm.Halp, alpha=5e-3, epochs=2, inner_steps=300, mu=3.0, seed=0)
    res = H.grid_search(obj, base, [H.GridAxis("bits", [8, 16]), H.GridAxis("inner", [100, 600])], [5], metric="loss")
    plan = H.BatchProblems(X, y, nprob=1).oracle_plan()
    o = oracle.OracleObjective(X, y=y)
    pts, best_i = oracle_grid(oracle, o, dict(alpha=5e-3, epochs=2, inner_steps=300, mu=3.0),
                              [("bits", [8, 16]), ("inner", [100, 600])], [5], plan, metric="loss")
    assert [p.per_seed for p in res.points] == pts and res.best_index == best_i


def test_grid_search_softmax_sequential(H, oracle):
    rng = np.random.default_rng(2)
    n, d, C = 300, 12, 3
    X = rng.standard_normal((n, d)).astype(np.float32)
    lab = rng.integers(0, C, n).astype(np.int32)
    obj = H.Objective(H.Dataset(X, labels=lab, num_classes=C), H.LossFamily.Softmax, 1e-4)
    base = H.OptimizerConfig(algorithm=H.Algorithm.Halp, alpha=0.05, epochs=2, inner_steps=200, mu=2.5, seed=3)
    res = H.grid_search(obj, base, [H.GridAxis("alpha", [0.01, 0.05])], [1, 2])
    o = oracle.OracleObjective(X, labels=lab, num_classes=C, l2=1e-4)
    pts, best_i = oracle_grid(oracle, o, dict(alpha=0.05, epochs=2, inner_steps=200, mu=2.5),
                              [("alpha", [0.01, 0.05])], [1, 2], obj.oracle_plan())
    assert [p.per_seed for p in res.points] == pts and res.best_index == best_i
