"""Race / ordering stress in place of compute-sanitizer (which this GPU pool
refuses to run: profiles/r02_sanitizer/compute_sanitizer_refused.log).  A
shared-memory race, a missing mbarrier wait, a DSMEM store landing after its
reader, or an early-exit path leaving a CTA behind shows up as run-to-run
differences: every kernel family is run repeatedly -- back to back and
interleaved with other problems on the same device -- and must reproduce
its first result bit for bit (and the oracle's)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu
REPS = 12


@pytest.fixture(scope="module")
def H():
    import paper_1803_03383_b200 as H
    from paper_1803_03383_b200 import build

    build.build()
    return H


def sig(rec):
    return [(r.loss, r.grad_norm, r.delta, r.iterate_hash) for r in rec.rows], rec.final_iterate.tobytes()


@pytest.mark.parametrize("plan", ["0:0:1", "4:2:1", "16:2:1", "16:2:2", "8:4:2", "16:2:3", "8:4:3"])
def test_k1_k3_repeatable(H, oracle, monkeypatch, plan):
    nc, m, lv = plan.split(":")
    monkeypatch.setenv("HALP_IN_NC", nc)
    monkeypatch.setenv("HALP_IN_M", m)
    monkeypatch.setenv("HALP_IN_LEVELS", lv)
    X, y = oracle.generate("regression", 20000, 2048, dtype="f32", noise_sd=0.1, seed=5)
    g = H.Objective(H.Dataset(X, targets=y), H.LossFamily.Squared, 1e-5)
    cfg = H.OptimizerConfig(algorithm=H.Algorithm.Halp, alpha=2e-4, epochs=2, inner_steps=3000, bits=8, mu=2.0,
                            seed=3)
    first = sig(H.run_halp(g, cfg))
    other = H.Objective(H.Dataset(X[:5000], targets=y[:5000]), H.LossFamily.Squared, 0.0)
    for i in range(REPS):
        if i % 3 == 1:
            H.run_halp(other, cfg)  # interleave another problem's launches
        assert sig(H.run_halp(g, cfg)) == first, i
    orec = oracle.run_halp(oracle.OracleObjective(X, y=y, l2=1e-5),
                           oracle.OracleConfig(alpha=2e-4, epochs=2, inner_steps=3000, bits=8, mu=2.0, seed=3),
                           plan=g.oracle_plan())
    assert first[0] == [(r["loss"], r["grad_norm"], r["delta"], r["iterate_hash"]) for r in orec.rows]


def test_softmax_cluster_and_blowup_repeatable(H, oracle, monkeypatch):
    monkeypatch.setenv("HALP_IN_NC", "4")
    monkeypatch.setenv("HALP_IN_M", "2")
    rng = np.random.default_rng(5)
    X = (rng.random((400, 300)) * 4.0).astype(np.float32)
    lab = rng.integers(0, 3, 400).astype(np.int32)
    g = H.Objective(H.Dataset(X, labels=lab, num_classes=3), H.LossFamily.Softmax, 1e-4)
    cfg = H.OptimizerConfig(algorithm=H.Algorithm.Halp, alpha=0.01, epochs=2, inner_steps=500, bits=8, mu=2.0, seed=4)
    bad = H.OptimizerConfig(algorithm=H.Algorithm.Halp, alpha=1.5e308, epochs=2, inner_steps=50, bits=8, mu=2.0,
                            seed=4)
    first = sig(H.run_halp(g, cfg))
    blow = None
    for i in range(REPS):
        assert sig(H.run_halp(g, cfg)) == first, i
        with pytest.raises(H.DivergenceError) as e:  # every CTA leaves through the blow-up path
            H.run_halp(g, bad)
        b = [(r.pass_, r.iterate_hash) for r in e.value.partial.rows]
        blow = blow or b
        assert b == blow, i


def test_k1_bf16_two_class_repeatable(H, oracle):
    X, lab = oracle.generate("logistic", 200000, 1024, dtype="bf16", x_scale=1 / 32, seed=4)
    g = H.Objective(H.Dataset(X, labels=lab, num_classes=2), H.LossFamily.Softmax, 1e-5)
    w = np.random.default_rng(0).standard_normal(2048)
    g0, l0 = g._fullpass(w)
    for i in range(REPS):
        gi, li = g._fullpass(w)
        assert np.array_equal(gi, g0) and li == l0, i
        g.bench_full_gradient(1)


def test_k5_and_lm_repeatable(H, oracle):
    rng = np.random.default_rng(0)
    P, n, d = 40, 512, 128
    X = rng.standard_normal((P, n, d)).astype(np.float32)
    y = rng.standard_normal((P, n))
    cfgs = [H.OptimizerConfig(algorithm=H.Algorithm.Halp, alpha=1e-3, epochs=2, inner_steps=300, bits=8, mu=3.0,
                              seed=p) for p in range(P)]
    cfgs[3].alpha = 1e300
    for warps in ("1", "2", "4"):
        import os

        os.environ["HALP_K5_WARPS"] = warps
        b = H.BatchProblems(X, y, l2=1e-4)
        first = [sig(r) for r in b.run(cfgs)]
        for i in range(REPS // 2):
            assert [sig(r) for r in b.run(cfgs)] == first, (warps, i)
    os.environ.pop("HALP_K5_WARPS")
    ds = H.harness.make_classification(500, 64, 10, 3.0, 4)
    H.quantize_dataset(ds, 8, 9)
    g = H.Objective(ds, H.LossFamily.Softmax, 1e-4)
    cfg = H.OptimizerConfig(algorithm=H.Algorithm.LmHalp, alpha=0.02, epochs=2, inner_steps=500, bits=8, mu=2.5, seed=6)
    first = sig(H.run_lm_halp(g, cfg))
    for i in range(REPS):
        assert sig(H.run_lm_halp(g, cfg)) == first, i
