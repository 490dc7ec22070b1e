"""K3's alternative exchanges for squared loss on a cluster, each bit-identical
to the oracle's MIRROR order for its plan, including a mid-epoch blow-up:
in_levels = 2: each CTA's warps pre-reduced in shared memory, one DSMEM
record per CTA (the in-band flag survives the CTA combine);
in_levels = 3: fixed point -- thread partials rounded to integers at 2^S,
warp sums by REDUX, remote integer reductions (red.async) into running
totals, so the sum is exact and order-free."""
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def H():
    import paper_1803_03383_b200 as H
    from paper_1803_03383_b200 import build

    build.build()
    return H


@pytest.mark.parametrize("lv", [2, 3])
@pytest.mark.parametrize("nc,m", [(16, 2), (8, 4), (4, 4)])
def test_two_level_bitexact(H, oracle, monkeypatch, nc, m, lv):
    monkeypatch.setenv("HALP_IN_LEVELS", str(lv))
    monkeypatch.setenv("HALP_IN_NC", str(nc))
    monkeypatch.setenv("HALP_IN_M", str(m))
    X, y = oracle.generate("regression", 4096, 4096, dtype="f32", noise_sd=0.1, seed=3)
    g = H.Objective(H.Dataset(X, targets=y), H.LossFamily.Squared, 1e-5)
    plan = g.oracle_plan()
    assert plan["in_levels"] == lv and plan["in_ctas"] == nc
    cfg = dict(alpha=2e-4, epochs=2, inner_steps=1500, bits=16, mu=1.0, seed=7)
    steps = 300
    tr = np.zeros(steps * 4096, dtype=np.int64)
    rec = H.run_halp(g, H.OptimizerConfig(algorithm=H.Algorithm.Halp, **cfg), trace=tr)
    o = oracle.OracleObjective(X, y=y, l2=1e-5)
    orec = oracle.run_halp(o, oracle.OracleConfig(**cfg), plan=plan, trace_steps=steps)
    assert [(r.loss, r.grad_norm, r.delta, r.iterate_hash) for r in rec.rows] == \
        [(r["loss"], r["grad_norm"], r["delta"], r["iterate_hash"]) for r in orec.rows]
    assert np.array_equal(rec.final_iterate, orec.final_iterate)
    assert np.array_equal(tr.reshape(steps, 4096), orec.trace)
    # blow-up mid-epoch: same partial record as the oracle
    bad = dict(cfg, alpha=1e308)  # |alpha g~| overflows at step 0
    with pytest.raises(H.DivergenceError) as e:
        H.run_halp(g, H.OptimizerConfig(algorithm=H.Algorithm.Halp, **bad))
    orec = oracle.run_halp(o, oracle.OracleConfig(**bad), plan=plan)
    assert [(r.pass_, r.iterate_hash) for r in e.value.partial.rows] == \
        [(r["pass_"], r["iterate_hash"]) for r in orec.rows]


def test_fixed_point_nan_data_blows_up_like_oracle(H, oracle, monkeypatch):
    """a non-finite x makes the reference's dot NaN: same blow-up row"""
    monkeypatch.setenv("HALP_IN_LEVELS", "3")
    monkeypatch.setenv("HALP_IN_NC", "4")
    monkeypatch.setenv("HALP_IN_M", "2")
    X, y = oracle.generate("regression", 2000, 1024, dtype="f32", noise_sd=0.1, seed=5)
    X[777, 5] = np.inf
    g = H.Objective(H.Dataset(X, targets=y), H.LossFamily.Squared, 0.0)
    cfg = dict(alpha=1e-4, epochs=1, inner_steps=3000, bits=8, mu=1.0, seed=2)
    o = oracle.OracleObjective(X, y=y)
    orec = oracle.run_halp(o, oracle.OracleConfig(**cfg), plan=g.oracle_plan())
    with pytest.raises(H.DivergenceError) as e:
        H.run_halp(g, H.OptimizerConfig(algorithm=H.Algorithm.Halp, **cfg))
    # float.hex: NaN rows compare equal (nan != nan as floats)
    assert [(r.pass_, float(r.loss).hex(), r.iterate_hash) for r in e.value.partial.rows] == \
        [(r["pass_"], float(r["loss"]).hex(), r["iterate_hash"]) for r in orec.rows]


def test_fixed_point_one_cta(H, oracle, monkeypatch):
    """in_levels = 3 on a single CTA (records through shared memory + __syncthreads)"""
    monkeypatch.setenv("HALP_IN_LEVELS", "3")
    monkeypatch.setenv("HALP_IN_NC", "1")
    monkeypatch.setenv("HALP_IN_M", "2")
    X, y = oracle.generate("regression", 4096, 256, dtype="f32", noise_sd=0.01, seed=11)
    g = H.Objective(H.Dataset(X, targets=y), H.LossFamily.Squared, 0.0)
    plan = g.oracle_plan()
    assert plan["in_levels"] == 3 and plan["in_ctas"] == 1
    cfg = dict(alpha=1e-3, epochs=2, inner_steps=2000, bits=8, mu=10.0, seed=3)
    steps = 400
    tr = np.zeros(steps * 256, dtype=np.int64)
    rec = H.run_halp(g, H.OptimizerConfig(algorithm=H.Algorithm.Halp, **cfg), trace=tr)
    o = oracle.OracleObjective(X, y=y)
    orec = oracle.run_halp(o, oracle.OracleConfig(**cfg), plan=plan, trace_steps=steps)
    assert [(r.loss, r.grad_norm, r.delta, r.iterate_hash) for r in rec.rows] == \
        [(r["loss"], r["grad_norm"], r["delta"], r["iterate_hash"]) for r in orec.rows]
    assert np.array_equal(tr.reshape(steps, 256), orec.trace)


@pytest.mark.parametrize("d,nc,m", [(4096, 16, 2), (4096, 8, 4), (256, 1, 2), (250, 1, 2)])
def test_untraced_launch_equals_traced(H, oracle, monkeypatch, d, nc, m):
    """The launch without a code trace (the specialised FAST instantiation when
    every coordinate slot is real: d = 4096 / 256; d = 250 leaves dead slots and
    stays on the general kernel) gives the rows, hashes and iterate of the traced
    launch and of the oracle, including a mid-epoch blow-up."""
    monkeypatch.setenv("HALP_IN_NC", str(nc))
    monkeypatch.setenv("HALP_IN_M", str(m))
    X, y = oracle.generate("regression", 3000, d, dtype="f32", noise_sd=0.1, seed=5)
    g = H.Objective(H.Dataset(X, targets=y), H.LossFamily.Squared, 1e-6)
    plan = g.oracle_plan()
    assert plan["in_ctas"] == nc and plan["in_per"] == m
    cfg = dict(alpha=0.3 / d, epochs=3, inner_steps=1200, bits=16, mu=2.0, seed=9)
    tr = np.zeros(50 * d, dtype=np.int64)
    traced = H.run_halp(g, H.OptimizerConfig(algorithm=H.Algorithm.Halp, **cfg), trace=tr)
    plain = H.run_halp(g, H.OptimizerConfig(algorithm=H.Algorithm.Halp, **cfg))
    o = oracle.OracleObjective(X, y=y, l2=1e-6)
    orec = oracle.run_halp(o, oracle.OracleConfig(**cfg), plan=plan)
    key = lambda r: (r.loss, r.grad_norm, r.delta, r.iterate_hash)
    assert [key(r) for r in plain.rows] == [key(r) for r in traced.rows]
    assert [key(r) for r in plain.rows] == [(r["loss"], r["grad_norm"], r["delta"], r["iterate_hash"]) for r in orec.rows]
    assert np.array_equal(plain.final_iterate, traced.final_iterate)
    assert np.array_equal(plain.final_iterate, orec.final_iterate)
    bad = dict(cfg, alpha=1e308)
    with pytest.raises(H.DivergenceError) as e:
        H.run_halp(g, H.OptimizerConfig(algorithm=H.Algorithm.Halp, **bad))
    orec = oracle.run_halp(o, oracle.OracleConfig(**bad), plan=plan)
    assert [(r.pass_, r.iterate_hash) for r in e.value.partial.rows] == \
        [(r["pass_"], r["iterate_hash"]) for r in orec.rows]
