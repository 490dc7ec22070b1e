"""Oracle (REF order) pinned against the reference's golden HALP traces.

Fixture: tests/golden/regression_floor.json, extracted by
tests/golden/make_fixtures.py from proj/out/regression_floor/*.csv (the
output of `lpopt run --spec specs/regression_floor.json`, spec rows
halp-8 / halp-16: make_regression(1000,100,0,42), alpha 5e-3, mu 3,
T 2000, 25 epochs, seeds 1..5).

The reference's reduction order lives in Eigen (not available here); the
oracle's REF order reproduces the traces bit for bit for the first epochs
and to <= 1e-9 relative on every row of 8 of the 10 traces.  halp-16 seeds
3 and 4 take a different stochastic-rounding decision late in the run (one
code flip, caused by an ulp-level difference in g~ near delta ~ 1e-9..1e-10);
their rows are compared up to that point and their end state statistically.
"""
import json
import os

import numpy as np
import pytest

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "regression_floor.json")))
# epochs checked at 1e-9 per trace (all 26 rows unless a late flip is known)
ROWS_1E9 = {("halp-16", 3): 12, ("halp-16", 4): 22}


@pytest.fixture(scope="module")
def obj(oracle):
    X, y = oracle.make_regression(1000, 100, 0.0, 42)
    return oracle.OracleObjective(X, y=y)


@pytest.mark.parametrize("name,bits", [("halp-8", 8), ("halp-16", 16)])
@pytest.mark.parametrize("seed", [1, 2, 3, 4, 5])
def test_golden_trace(oracle, obj, name, bits, seed):
    cfg = oracle.OracleConfig(alpha=5e-3, epochs=25, inner_steps=2000, bits=bits, mu=3.0, seed=seed)
    rec = oracle.run_halp(obj, cfg)
    gold = GOLD["traces"][f"{name}_seed{seed}"]
    assert len(rec.rows) == len(gold) == 26
    assert rec.status == "ok" and rec.steps_taken == 50000
    assert rec.inner_fp_vector_ops == 8 * 2000 * 25
    nrow = ROWS_1E9.get((name, seed), 26)
    exact = 0
    for k, (a, b) in enumerate(zip(rec.rows, gold)):
        assert a["pass_"] == float(b["pass"])
        for f in ("loss", "grad_norm", "delta"):
            bv = float(b[f])
            if k < nrow:
                assert abs(a[f] - bv) <= 1e-9 * abs(bv), (k, f, a[f], bv)
            exact += a[f] == bv
    # the first epochs are reproduced bit for bit
    for f in ("loss", "grad_norm", "delta"):
        assert rec.rows[0][f] == float(gold[0][f])
    assert exact >= 15
    man = GOLD["manifest"][f"{name}_seed{seed}"]
    if nrow == 26:
        assert rec.rows[-1]["loss"] == pytest.approx(man["final_loss"], rel=1e-9)
    else:
        # after the flip both runs keep converging to the same floor
        assert 0.1 < rec.rows[-1]["grad_norm"] / man["final_grad_norm"] < 10


def test_golden_packet_width_is_sse2(oracle, obj):
    """REF's Eigen packet width (2 doubles, SSE2) is the one that makes the
    most golden rows bit-exact; 1 (scalar) and 4 (AVX) do worse."""
    L = oracle.lib()
    counts = {}
    try:
        for lanes in (1, 2, 4):
            L.oq_set_ref_lanes(lanes)
            n = 0
            for seed in (1, 2):
                cfg = oracle.OracleConfig(alpha=5e-3, epochs=6, inner_steps=2000, bits=8, mu=3.0, seed=seed)
                rec = oracle.run_halp(obj, cfg)
                gold = GOLD["traces"][f"halp-8_seed{seed}"]
                n += sum(a["grad_norm"] == float(b["grad_norm"]) for a, b in zip(rec.rows[:6], gold[:6]))
            counts[lanes] = n
    finally:
        L.oq_set_ref_lanes(2)
    assert counts[2] == 12 and counts[2] > counts[1] and counts[2] > counts[4], counts


OPS = {0: 3, 1: 5, 2: 5, 3: 7}  # instr fp vector ops per inner step (objectives.cpp:249, optimizers.cpp, fixed_point.cpp)


@pytest.mark.parametrize("name,algo,kw,tol", [("svrg", 1, dict(alpha=5e-3), 1e-9),
                                              ("lp-svrg-8", 3, dict(alpha=5e-3, delta=0.7, bits=8), 1e-15),
                                              ("lp-svrg-16", 3, dict(alpha=5e-3, delta=0.003, bits=16), 1e-15),
                                              ("sgd", 0, dict(alpha=2.5e-6), 0.0),
                                              ("lp-sgd-8", 2, dict(alpha=2.5e-6, delta=0.7, bits=8), 0.0),
                                              ("lp-sgd-16", 2, dict(alpha=2.5e-6, delta=0.003, bits=16), 1e-15)])
@pytest.mark.parametrize("seed", [1, 2, 3, 4, 5])
def test_golden_svrg_family(oracle, obj, name, algo, kw, tol, seed):
    """run_svrg / run_lp_svrg / run_sgd / run_lp_sgd (optimizers.cpp:229-385)
    restated, against the golden traces {svrg, lp-svrg-{8,16}, sgd,
    lp-sgd-{8,16}}_seed{1..5}.csv (spec rows specs/regression_floor.json:7-12):
    every row within 1e-9 (SVRG), 1e-15 (LP-SVRG) and bit for bit (SGD,
    LP-SGD-8; LP-SGD-16 to 1e-15)."""
    cfg = oracle.OracleConfig(epochs=25, inner_steps=2000, seed=seed, algorithm=algo, **kw)
    rec = oracle.run(obj, cfg)
    gold = GOLD["traces"][f"{name}_seed{seed}"]
    assert len(rec.rows) == len(gold) == 26 and rec.status == "ok" and rec.steps_taken == 50000
    assert rec.inner_fp_vector_ops == OPS[algo] * 2000 * 25
    for k, (a, b) in enumerate(zip(rec.rows, gold)):
        assert a["pass_"] == float(b["pass"])
        for f in ("loss", "grad_norm", "delta"):
            bv = float(b[f])
            assert abs(a[f] - bv) <= tol * abs(bv), (k, f, a[f], bv)
    man = GOLD["manifest"][f"{name}_seed{seed}"]
    assert rec.rows[-1]["grad_norm"] == pytest.approx(man["final_grad_norm"], rel=max(tol, 1e-12))
