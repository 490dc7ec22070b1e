"""Small workloads for compute-sanitizer (memcheck / racecheck / synccheck):

    compute-sanitizer --tool racecheck python tools/sanitize_run.py k3

k1: K1 streaming pass (least squares f32, two-class bf16), split tree, finalize
k3: K3 inner loop: single CTA, 4- and 16-CTA clusters, softmax, a mid-epoch blow-up
k5: K5 batch (one-warp and four-warp plans) incl. a diverging problem
lm: LM-HALP K7 + K8
Each case is checked against the oracle so a sanitizer run also proves the
instrumented kernels still compute the right answer."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1803_03383_b200 as H  # noqa: E402
from oracle import oracle as O  # noqa: E402


def bitexact(rec, orec):
    assert [(r.loss, r.grad_norm, r.iterate_hash) for r in rec.rows] == \
        [(r["loss"], r["grad_norm"], r["iterate_hash"]) for r in orec.rows]


def k1():
    X, y = O.generate("regression", 4096, 256, dtype="f32", noise_sd=0.1, seed=3)
    g = H.Objective(H.Dataset(X, targets=y), H.LossFamily.Squared, 1e-4)
    w = np.random.default_rng(0).standard_normal(256)
    gg, _ = g._fullpass(w)
    assert np.array_equal(gg, O.OracleObjective(X, y=y, l2=1e-4).full_gradient(w, plan=g.oracle_plan()))
    Xb, lb = O.generate("logistic", 4096, 1024, dtype="bf16", x_scale=1 / 32, seed=4)
    g2 = H.Objective(H.Dataset(Xb, labels=lb, num_classes=2), H.LossFamily.Softmax, 1e-5)
    w2 = np.random.default_rng(1).standard_normal(2048)
    gg2, _ = g2._fullpass(w2)
    o2 = O.OracleObjective(Xb, labels=lb, num_classes=2, l2=1e-5)
    assert np.array_equal(gg2, o2.full_gradient(w2, plan=g2.oracle_plan()))
    print("k1 ok")


def k3():
    X, y = O.make_regression(1000, 100, 0.0, 42)
    for nc in (0, 4, 16):
        os.environ["HALP_IN_NC"] = str(nc)
        g = H.Objective(H.Dataset(X, targets=y), H.LossFamily.Squared, 0.0)
        cfg = H.OptimizerConfig(algorithm=H.Algorithm.Halp, alpha=5e-3, epochs=2, inner_steps=300, bits=8, mu=3.0,
                                seed=1)
        rec = H.run_halp(g, cfg)
        bitexact(rec, O.run_halp(O.OracleObjective(X, y=y), O.OracleConfig(alpha=5e-3, epochs=2, inner_steps=300,
                                                                           bits=8, mu=3.0, seed=1),
                                 plan=g.oracle_plan()))
        # mid-epoch blow-up: the early-exit paths of every CTA of the cluster
        bad = H.OptimizerConfig(algorithm=H.Algorithm.Halp, alpha=1e300, epochs=2, inner_steps=300, bits=8, mu=3.0,
                                seed=1)
        try:
            H.run_halp(g, bad)
            raise AssertionError("expected a blow-up")
        except H.DivergenceError as e:
            assert math_isinf(e.partial.rows[-1].loss)
    os.environ.pop("HALP_IN_NC")
    Xs, ls = O.generate("softmax", 500, 100, num_classes=10, density=0.3, seed=2)
    g = H.Objective(H.Dataset(Xs, labels=ls, num_classes=10), H.LossFamily.Softmax, 1e-4)
    rec = H.run_halp(g, H.OptimizerConfig(algorithm=H.Algorithm.Halp, alpha=0.01, epochs=1, inner_steps=200, bits=8,
                                          mu=2.5, seed=2))
    o = O.OracleObjective(Xs, labels=ls, num_classes=10, l2=1e-4)
    bitexact(rec, O.run_halp(o, O.OracleConfig(alpha=0.01, epochs=1, inner_steps=200, bits=8, mu=2.5, seed=2),
                             plan=g.oracle_plan()))
    print("k3 ok")


def math_isinf(v):
    return v == float("inf")


def k5():
    P, n, d = 6, 512, 128
    rng = np.random.default_rng(0)
    X = rng.standard_normal((P, n, d)).astype(np.float32)
    y = rng.standard_normal((P, n))
    for w in ("1", "4"):
        os.environ["HALP_K5_WARPS"] = w
        b = H.BatchProblems(X, y, l2=1e-4)
        cfgs = [H.OptimizerConfig(algorithm=H.Algorithm.Halp, alpha=1e-3, epochs=2, inner_steps=200, bits=8, mu=3.0,
                                  seed=p) for p in range(P)]
        cfgs[2].alpha = 1e300
        recs = b.run(cfgs)
        for p in (0, 2):
            o = O.OracleObjective(X[p], y=y[p], l2=1e-4)
            c = cfgs[p]
            orec = O.run_halp(o, O.OracleConfig(alpha=c.alpha, epochs=2, inner_steps=200, bits=8, mu=3.0, seed=p),
                              plan=b.oracle_plan())
            assert [r.iterate_hash for r in recs[p].rows] == [r["iterate_hash"] for r in orec.rows]
    os.environ.pop("HALP_K5_WARPS")
    print("k5 ok")


def lm():
    ds = H.harness.make_classification(300, 20, 3, 3.0, 4)
    H.quantize_dataset(ds, 8, 9)
    g = H.Objective(ds, H.LossFamily.Softmax, 1e-4)
    cfg = H.OptimizerConfig(algorithm=H.Algorithm.LmHalp, alpha=0.05, epochs=2, inner_steps=200, bits=8, mu=3.0,
                            seed=6)
    rec = H.run_lm_halp(g, cfg)
    q = O.OracleQuantized(ds.quantized.codes, ds.quantized.delta, 8)
    o = O.OracleObjective(ds.X, labels=ds.labels, num_classes=3, l2=1e-4)
    orec = O.run_lm_halp(o, q, O.OracleConfig(alpha=0.05, epochs=2, inner_steps=200, bits=8, mu=3.0, seed=6),
                         plan=g.oracle_plan())
    bitexact(rec, orec)
    print("lm ok")


if __name__ == "__main__":
    for which in sys.argv[1:]:
        {"k1": k1, "k3": k3, "k5": k5, "lm": lm}[which]()
