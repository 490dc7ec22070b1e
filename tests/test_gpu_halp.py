"""GPU parity: the B200 kernels against the CPU oracle.

MIRROR mode reproduces the kernels' floating-point order, so every number
must be bit-identical (losses, gradient norms, deltas, iterate hashes, final
iterates, every z code).  REF mode is the reference's own order (pinned to
the golden traces); against it the z trajectory must still be identical and
losses / gradients agree to <= 1e-9 relative (north-star bar: 1e-5 for fp32).
"""
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


def objs(H, oracle, X, y=None, labels=None, C=0, l2=0.0):
    if labels is None:
        g = H.Objective(H.Dataset(X, targets=y), H.LossFamily.Squared, l2)
        o = oracle.OracleObjective(X, y=y, l2=l2)
    else:
        g = H.Objective(H.Dataset(X, labels=labels, num_classes=C), H.LossFamily.Softmax, l2)
        o = oracle.OracleObjective(X, labels=labels, num_classes=C, l2=l2)
    return g, o


def bf16_bits(a):
    u = np.ascontiguousarray(a, dtype=np.float32).view(np.uint32)
    # round to nearest even
    u = (u + 0x7FFF + ((u >> 16) & 1)) >> 16
    return u.astype(np.uint16)


@pytest.mark.parametrize("dtype", ["f64", "f32", "bf16"])
@pytest.mark.parametrize("shape", [(1000, 100), (777, 37), (5000, 256), (64, 8)])
def test_fullgrad_squared_bitexact(H, oracle, dtype, shape):
    n, d = shape
    X, y = oracle.make_regression(n, d, 0.3, 11)
    Xd = {"f64": X, "f32": X.astype(np.float32), "bf16": bf16_bits(X)}[dtype]
    g, o = objs(H, oracle, Xd, y, l2=1e-3)
    w = np.random.default_rng(1).standard_normal(d)
    gg, gl = g._fullpass(w)
    plan = g.oracle_plan()
    og = o.full_gradient(w, plan=plan)
    ol = o.loss_value(w, plan=plan)
    assert np.array_equal(gg, og)
    assert gl == ol
    rg = o.full_gradient(w)
    assert np.max(np.abs(gg - rg)) <= 1e-12 * np.max(np.abs(rg))
    assert abs(gl - o.loss_value(w)) <= 1e-12 * abs(gl)


@pytest.mark.parametrize("dtype,n,d", [("f32", 1501, 4096), ("f32", 1111, 3500), ("f64", 900, 2048), ("bf16", 700, 4096)])
def test_fullgrad_squared_wide_rows(H, oracle, dtype, n, d):
    """Rows of 16 KB (BASELINE C3's d = 4096 fp32): K1 streams them as 4-row, 64 KB
    tiles through a 3-deep ring (halp_capi.cpp plan_stream); bit-identical to the
    oracle, including a partial last tile and rows narrower than the thread tile."""
    X, y = oracle.make_regression(n, d, 0.1, 13)
    Xd = {"f64": X, "f32": X.astype(np.float32), "bf16": bf16_bits(X)}[dtype]
    g, o = objs(H, oracle, Xd, y, l2=1e-4)
    pl = g.plan()
    if dtype in ("f32", "f64"):
        assert pl["fg_rows_per_stage"] == 4 and pl["fg_stages"] == 3, pl
    w = np.random.default_rng(2).standard_normal(d)
    gg, gl = g._fullpass(w)
    plan = g.oracle_plan()
    assert np.array_equal(gg, o.full_gradient(w, plan=plan))
    assert gl == o.loss_value(w, plan=plan)


@pytest.mark.parametrize("C,d,n", [(2, 40, 3000), (3, 17, 500), (10, 784, 2000), (15, 33, 700)])
def test_fullgrad_softmax_bitexact(H, oracle, C, d, n):
    rng = np.random.default_rng(C)
    X = rng.random((n, d)).astype(np.float32) * (rng.random((n, d)) < 0.2)
    lab = rng.integers(0, C, n).astype(np.int32)
    g, o = objs(H, oracle, X, labels=lab, C=C, l2=1e-4)
    w = rng.standard_normal(d * C) * 0.1
    gg, gl = g._fullpass(w)
    plan = g.oracle_plan()
    assert np.array_equal(gg, o.full_gradient(w, plan=plan))
    assert gl == o.loss_value(w, plan=plan)
    rg = o.full_gradient(w)
    assert np.max(np.abs(gg - rg)) <= 1e-12 * max(1e-300, np.max(np.abs(rg)))
    assert abs(gl - o.loss_value(w)) <= 1e-12 * abs(gl)


@pytest.mark.parametrize("d,n", [(1024, 4096), (200, 3001), (24, 517)])
def test_fullgrad_two_class_bf16_integer_conversion(H, oracle, d, n):
    """bf16 two-class sweeps convert x with integer ops in the 2^-896-scaled
    domain (k_fullgrad_stream.cu load_group_scaled).  Bit-identical to the
    oracle's exact upcast on data that exercises every bf16 class: zeros of
    both signs, subnormals, the smallest / largest normal exponents."""
    rng = np.random.default_rng(d)
    X = rng.standard_normal((n, d)) / np.sqrt(d)
    X[rng.random((n, d)) < 0.1] = 0.0
    X[rng.random((n, d)) < 0.02] *= 2.0 ** -130  # bf16 subnormals
    X[rng.random((n, d)) < 0.01] *= 2.0 ** 100
    Xb = bf16_bits(X)
    Xb[0, 0] = 0x8000  # -0.0
    Xb[1, 1] = 0x0001  # smallest subnormal
    Xb[2, 2] = 0x7F7F  # largest finite
    lab = rng.integers(0, 2, n).astype(np.int32)
    g, o = objs(H, oracle, Xb, labels=lab, C=2, l2=1e-5)
    plan = g.oracle_plan()
    for w in (rng.standard_normal(2 * d) * 1e-3, np.zeros(2 * d), rng.standard_normal(2 * d) * 1e30):
        gg, gl = g._fullpass(w)
        assert np.array_equal(gg, o.full_gradient(w, plan=plan))
        assert gl == o.loss_value(w, plan=plan)


@pytest.mark.parametrize("dtype,d", [("bf16", 512), ("bf16", 1024), ("bf16", 2048), ("f32", 300), ("f32", 1024),
                                     ("f32", 2048), ("f64", 512)])
def test_fullgrad_two_class_warp_counts(H, oracle, dtype, d):
    """Two-class K1 on 2, 4, 8 and 16 warps per CTA: one rotating warp evaluates the
    tile's softmax derivative and another its loss terms behind a second barrier
    (k_fullgrad_stream.cu DW), 16-row tiles fill their dot slots in a lane-dependent row
    order (RL).  Partial last tiles (n not a multiple of the tile) are included (CTAs
    walking several splits: test_gpu_baseline_configs C4); loss and gradient
    bit-identical to the oracle."""
    rng = np.random.default_rng(d)
    n = 20011
    X = rng.standard_normal((n, d)) / np.sqrt(d)
    Xd = {"f64": X, "f32": X.astype(np.float32), "bf16": bf16_bits(X)}[dtype]
    lab = rng.integers(0, 2, n).astype(np.int32)
    g, o = objs(H, oracle, Xd, labels=lab, C=2, l2=1e-5)
    plan = g.oracle_plan()
    assert g.plan()["fg_threads"] >= 64
    for w in (rng.standard_normal(2 * d) * 0.5, rng.standard_normal(2 * d) * 20.0):
        gg, gl = g._fullpass(w)
        assert np.array_equal(gg, o.full_gradient(w, plan=plan))
        assert gl == o.loss_value(w, plan=plan)


@pytest.mark.parametrize("dtype,n,d", [("bf16", 150001, 512), ("f32", 60001, 1024)])
def test_fullgrad_two_class_multi_split(H, oracle, dtype, n, d):
    """More splits than resident CTAs on 2 and 8 warps per CTA: every CTA walks several
    splits, so the two-class window's loss-term / loss-sum pipeline is drained and
    restarted at split boundaries while the copy ring runs across them."""
    rng = np.random.default_rng(n)
    X = (rng.standard_normal((n, d), dtype=np.float32) / np.float32(np.sqrt(d))).astype(np.float32)
    Xd = X if dtype == "f32" else bf16_bits(X)
    lab = rng.integers(0, 2, n).astype(np.int32)
    g, o = objs(H, oracle, Xd, labels=lab, C=2, l2=1e-5)
    pl = g.plan()
    assert pl["fg_splits"] >= 1024 and pl["fg_threads"] in (64, 256), pl
    w = rng.standard_normal(2 * d) * 0.7
    gg, gl = g._fullpass(w)
    plan = g.oracle_plan()
    assert np.array_equal(gg, o.full_gradient(w, plan=plan))
    assert gl == o.loss_value(w, plan=plan)


def test_fullgrad_two_class_bf16_nonfinite_x(H, oracle):
    """A non-finite x disables the integer conversion (checked at creation):
    results follow IEEE arithmetic exactly like the oracle's (NaN / inf)."""
    rng = np.random.default_rng(3)
    n, d = 600, 64
    X = rng.standard_normal((n, d))
    Xb = bf16_bits(X)
    Xb[5, 7] = 0x7F80  # +inf
    lab = rng.integers(0, 2, n).astype(np.int32)
    g, o = objs(H, oracle, Xb, labels=lab, C=2, l2=0.0)
    w = rng.standard_normal(2 * d)
    gg, gl = g._fullpass(w)
    og = o.full_gradient(w, plan=g.oracle_plan())
    assert np.array_equal(gg, og, equal_nan=True)
    ol = o.loss_value(w, plan=g.oracle_plan())
    assert gl == ol or (math.isnan(gl) and math.isnan(ol))


def rows_equal(grows, orows):
    assert len(grows) == len(orows)
    for a, b in zip(grows, orows):
        assert a.pass_ == b["pass_"]
        assert a.loss == b["loss"] or (math.isnan(a.loss) and math.isnan(b["loss"])), (a, b)
        assert a.grad_norm == b["grad_norm"], (a, b)
        assert a.delta == b["delta"], (a, b)
        assert a.iterate_hash == b["iterate_hash"], (a, b)


@pytest.mark.parametrize("bits,seed", [(8, 1), (16, 4)])
def test_golden_problem_bitexact_vs_mirror(H, oracle, bits, seed):
    X, y = oracle.make_regression(1000, 100, 0.0, 42)
    g, o = objs(H, oracle, X, y)
    cfg = H.OptimizerConfig(algorithm=H.Algorithm.Halp, alpha=5e-3, epochs=25, inner_steps=2000, bits=bits, mu=3.0,
                            seed=seed)
    steps = 2000
    tr = np.zeros(steps * 100, dtype=np.int64)
    rec = H.run_halp(g, cfg, trace=tr)
    orec = oracle.run_halp(o, oracle.OracleConfig(alpha=5e-3, epochs=25, inner_steps=2000, bits=bits, mu=3.0,
                                                  seed=seed), plan=g.oracle_plan(), trace_steps=steps)
    rows_equal(rec.rows, orec.rows)
    assert np.array_equal(rec.final_iterate, orec.final_iterate)
    assert np.array_equal(tr.reshape(steps, 100), orec.trace)
    assert rec.steps_taken == 50000 and rec.inner_fp_vector_ops == 400000 and rec.status == "ok"


@pytest.mark.parametrize("name,bits", [("halp-8", 8), ("halp-16", 16)])
def test_golden_traces_gpu(H, oracle, name, bits):
    """The GPU reproduces the reference's own golden traces."""
    X, y = oracle.make_regression(1000, 100, 0.0, 42)
    g = H.Objective(H.Dataset(X, targets=y), H.LossFamily.Squared, 0.0)
    for seed in (1, 2, 5):
        cfg = H.OptimizerConfig(algorithm=H.Algorithm.Halp, alpha=5e-3, epochs=25, inner_steps=2000, bits=bits,
                                mu=3.0, seed=seed)
        rec = H.run_halp(g, cfg)
        gold = GOLD["traces"][f"{name}_seed{seed}"]
        assert len(rec.rows) == len(gold)
        for a, b in zip(rec.rows, gold):
            for f, gf in (("loss", "loss"), ("grad_norm", "grad_norm"), ("delta", "delta")):
                assert abs(getattr(a, f) - float(b[gf])) <= 1e-9 * abs(float(b[gf])), (seed, a, b)


def test_codes_match_reference_order(H, oracle):
    """Against the REF (reference-order) oracle the z trajectory is identical."""
    X, y = oracle.make_regression(1000, 100, 0.0, 42)
    g, o = objs(H, oracle, X, y)
    steps = 2000 * 3
    tr = np.zeros(steps * 100, dtype=np.int64)
    H.run_halp(g, H.OptimizerConfig(algorithm=H.Algorithm.Halp, alpha=5e-3, epochs=3, inner_steps=2000, bits=8,
                                    mu=3.0, seed=3), trace=tr)
    orec = oracle.run_halp(o, oracle.OracleConfig(alpha=5e-3, epochs=3, inner_steps=2000, bits=8, mu=3.0, seed=3),
                           trace_steps=steps)
    assert np.count_nonzero(tr.reshape(steps, 100) != orec.trace) == 0


@pytest.mark.parametrize("every", [0.0, 0.5, 2.0, 5.0])
def test_halp_init_and_metric_gating(H, oracle, every):
    """run_halp from a caller-supplied initial iterate (initial_iterate,
    optimizers.cpp:209-216) with the Recorder's metric_every_passes gating
    (optimizers.cpp:104-167) through halp_run: the same rows (count, pass
    values, losses, hashes) and final iterate as the oracle."""
    X, y = oracle.make_regression(800, 96, 0.05, 17)
    g, o = objs(H, oracle, X.astype(np.float32), y, l2=1e-4)
    init = np.random.default_rng(5).standard_normal(96) * 0.3
    kw = dict(alpha=4e-3, epochs=6, inner_steps=800, bits=8, mu=2.0, seed=11, metric_every_passes=every)
    rec = H.run_halp(g, H.OptimizerConfig(algorithm=H.Algorithm.Halp, init=init, **kw))
    orec = oracle.run_halp(o, oracle.OracleConfig(init=init, **kw), plan=g.oracle_plan())
    rows_equal(rec.rows, orec.rows)
    assert np.array_equal(rec.final_iterate, orec.final_iterate)
    assert rec.steps_taken == orec.steps_taken == 4800
    # the first row is the initial iterate's: its loss is f(init), not f(0)
    g0, l0 = g._fullpass(init)
    assert rec.rows[0].loss == l0
    if every >= 2.0:
        assert len(rec.rows) < 7
    with pytest.raises(H.InvalidInputError):
        H.run_halp(g, H.OptimizerConfig(algorithm=H.Algorithm.Halp, init=init[:-1], **kw))


@pytest.mark.parametrize("nc,m", [(1, 1), (2, 2), (4, 1), (3, 4), (16, 1), (8, 4), (1, 8), (16, 2)])
def test_cluster_plans_bitexact(H, oracle, nc, m, monkeypatch):
    monkeypatch.setenv("HALP_IN_NC", str(nc))
    monkeypatch.setenv("HALP_IN_M", str(m))
    X, y = oracle.make_regression(600, 150, 0.1, 5)
    Xf = X.astype(np.float32)
    g, o = objs(H, oracle, Xf, y, l2=1e-3)
    assert g.plan()["in_ctas"] == nc
    cfg = H.OptimizerConfig(algorithm=H.Algorithm.Halp, alpha=3e-3, epochs=3, inner_steps=700, bits=8, mu=2.0, seed=9)
    rec = H.run_halp(g, cfg)
    orec = oracle.run_halp(o, oracle.OracleConfig(alpha=3e-3, epochs=3, inner_steps=700, bits=8, mu=2.0, seed=9),
                           plan=g.oracle_plan())
    rows_equal(rec.rows, orec.rows)
    assert np.array_equal(rec.final_iterate, orec.final_iterate)


@pytest.mark.parametrize("C,nc", [(2, 1), (10, 0), (3, 2), (10, 8), (10, 16), (15, 4)])
def test_softmax_run_bitexact(H, oracle, C, nc, monkeypatch):
    if nc:
        monkeypatch.setenv("HALP_IN_NC", str(nc))
    rng = np.random.default_rng(7 + C)
    n, d = 1500, 64
    X = (rng.random((n, d)) * (rng.random((n, d)) < 0.3)).astype(np.float32)
    W = rng.standard_normal((d, C))
    lab = np.argmax(X @ W + rng.gumbel(size=(n, C)), axis=1).astype(np.int32)
    g, o = objs(H, oracle, X, labels=lab, C=C, l2=1e-4)
    cfg = H.OptimizerConfig(algorithm=H.Algorithm.Halp, alpha=0.05, epochs=3, inner_steps=n, bits=8, mu=2.5, seed=2)
    steps = 200
    tr = np.zeros(steps * d * C, dtype=np.int64)
    rec = H.run_halp(g, cfg, trace=tr)
    orec = oracle.run_halp(o, oracle.OracleConfig(alpha=0.05, epochs=3, inner_steps=n, bits=8, mu=2.5, seed=2),
                           plan=g.oracle_plan(), trace_steps=steps)
    rows_equal(rec.rows, orec.rows)
    assert np.array_equal(rec.final_iterate, orec.final_iterate)
    assert np.array_equal(tr.reshape(steps, -1), orec.trace)
    assert rec.rows[-1].loss < rec.rows[0].loss


def test_option_ii_and_wide_bits(H, oracle):
    X, y = oracle.make_regression(300, 20, 0.2, 5)
    g, o = objs(H, oracle, X, y)
    for bits, opt in ((8, 1), (40, 0), (64, 1)):
        cfg = H.OptimizerConfig(algorithm=H.Algorithm.Halp, alpha=0.02, epochs=4, bits=bits, mu=3.0, seed=11,
                                option=H.EpochOption(opt))
        rec = H.run_halp(g, cfg)
        orec = oracle.run_halp(o, oracle.OracleConfig(alpha=0.02, epochs=4, bits=bits, mu=3.0, seed=11, option=opt),
                               plan=g.oracle_plan())
        rows_equal(rec.rows, orec.rows)
        assert np.array_equal(rec.final_iterate, orec.final_iterate)


def test_converged_at_optimum(H, oracle):
    # test_optimizers.cpp:303-329
    X, _ = oracle.make_regression(30, 4, 0.0, 8)
    g = H.Objective(H.Dataset(X, targets=np.zeros(30)), H.LossFamily.Squared, 0.0)
    rec = H.run_halp(g, H.OptimizerConfig(algorithm=H.Algorithm.Halp, alpha=0.02, epochs=3, mu=3.0, seed=11))
    assert rec.status == "converged" and rec.steps_taken == 0
    assert len(rec.rows) == 1 and rec.rows[0].grad_norm == 0.0 and rec.rows[0].delta == 0.0


def test_delta_tracks_gradient(H):
    # test_optimizers.cpp:331-350
    g = H.Objective(H.Dataset(np.ones((1, 1)), targets=np.array([2.0])), H.LossFamily.Squared, 0.0)
    cfg = H.OptimizerConfig(algorithm=H.Algorithm.Halp, alpha=0.5, epochs=1, inner_steps=4, bits=8, mu=3.0, seed=11)
    rec = H.run_halp(g, cfg)
    assert rec.rows[0].grad_norm == 2.0 and rec.rows[0].delta == H.halp_scale(2.0, 3.0, 8)
    cfg.delta_min = 1.0
    assert H.run_halp(g, cfg).rows[0].delta == 1.0


def test_blowup_and_divergence(H, oracle):
    g = H.Objective(H.Dataset(np.array([[2.0]]), targets=np.array([3.0])), H.LossFamily.Squared, 0.0)
    cfg = H.OptimizerConfig(algorithm=H.Algorithm.Halp, alpha=1e308, epochs=2, inner_steps=3, mu=3.0, seed=11)
    with pytest.raises(H.DivergenceError) as ei:
        H.run_halp(g, cfg)
    part = ei.value.partial
    assert part.status == "diverged" and math.isinf(part.rows[-1].loss) and part.rows[-1].pass_ == 1.0
    o = oracle.OracleObjective(np.array([[2.0]]), y=np.array([3.0]))
    orec = oracle.run_halp(o, oracle.OracleConfig(alpha=1e308, epochs=2, inner_steps=3, mu=3.0, seed=11),
                           plan=g.oracle_plan())
    rows_equal(part.rows, orec.rows)
    assert np.array_equal(part.final_iterate, orec.final_iterate)
    assert H.run_prepared(g, H.OptimizerConfig(algorithm=H.Algorithm.Halp, alpha=1e308, epochs=2, inner_steps=3,
                                               mu=3.0, seed=11)).status == "diverged"
    # boundary divergence guard
    X, y = oracle.make_regression(80, 6, 0.2, 5)
    g2 = H.Objective(H.Dataset(X, targets=y), H.LossFamily.Squared, 0.0)
    with pytest.raises(H.DivergenceError):
        H.run_halp(g2, H.OptimizerConfig(algorithm=H.Algorithm.Halp, alpha=0.02, epochs=2, mu=3.0,
                                         divergence_limit=1e-3))


def test_validation_errors(H, oracle):
    X, y = oracle.make_regression(80, 6, 0.2, 5)
    g = H.Objective(H.Dataset(X, targets=y), H.LossFamily.Squared, 0.0)
    for bad in (dict(alpha=-1.0), dict(epochs=-1), dict(mu=0.0), dict(bits=1), dict(delta_min=0.0)):
        cfg = H.OptimizerConfig(algorithm=H.Algorithm.Halp, mu=3.0)
        for k, v in bad.items():
            setattr(cfg, k, v)
        with pytest.raises(H.InvalidInputError):
            H.run_halp(g, cfg)
    with pytest.raises(H.InvalidInputError):
        H.Objective(H.Dataset(X, labels=np.full(80, 7), num_classes=3), H.LossFamily.Softmax, 0.0)
    with pytest.raises(H.InvalidInputError):
        H.Objective(H.Dataset(X, targets=y), H.LossFamily.Squared, -1.0)
    rec = H.run_halp(g, H.OptimizerConfig(algorithm=H.Algorithm.Halp, epochs=0, mu=3.0))
    assert len(rec.rows) == 1 and rec.steps_taken == 0 and np.all(rec.final_iterate == 0)


def test_device_resident_inputs_and_datagen(H, oracle):
    import torch

    X, y = H.generate("regression", 4096, 128, dtype="f32", noise_sd=0.1, seed=3)
    assert X.is_cuda and torch.isfinite(X).all()
    g = H.Objective(H.Dataset(X, targets=y), H.LossFamily.Squared, 0.0)
    Xh, yh = X.cpu().numpy(), y.cpu().numpy()
    o = oracle.OracleObjective(Xh, y=yh)
    w = np.random.default_rng(0).standard_normal(128)
    gg, gl = g._fullpass(w)
    assert np.array_equal(gg, o.full_gradient(w, plan=g.oracle_plan()))
    # labels for the softmax / logistic generators
    Xs, lab = H.generate("softmax", 2000, 784, num_classes=10, dtype="f32", density=0.2, seed=1)
    labh = lab.cpu().numpy()
    assert labh.min() >= 0 and labh.max() <= 9 and len(np.unique(labh)) == 10
    assert 0.15 < float((Xs != 0).float().mean()) < 0.25
    Xb, lb = H.generate("logistic", 4096, 1024, dtype="bf16", x_scale=1 / 32, seed=2)
    assert Xb.dtype == torch.bfloat16 and set(np.unique(lb.cpu().numpy())) <= {0, 1}


@pytest.mark.parametrize("kind,nc,m", [("sq", 1, 2), ("sq", 4, 1), ("sq", 16, 2), ("sm1", 4, 2), ("sm1", 1, 4),
                                       ("sm2", 0, 0), ("sm2", 2, 1)])
def test_blowup_mid_epoch_bitexact(H, oracle, kind, nc, m, monkeypatch):
    """Blowups after a few inner steps, on single-CTA and cluster plans of all
    three inner-loop kinds: same step, same partial record, same iterate."""
    if nc:
        monkeypatch.setenv("HALP_IN_NC", str(nc))
        monkeypatch.setenv("HALP_IN_M", str(m))
    rng = np.random.default_rng(5)
    if kind == "sq":
        X, y = oracle.make_regression(300, 150, 0.5, 3)
        g, o = objs(H, oracle, X.astype(np.float32), y, l2=1e-3)
        alpha = 3e305
    else:
        d, C = (300, 3) if kind == "sm1" else (20, 10)
        X = (rng.random((400, d)) * 4.0).astype(np.float32)
        lab = rng.integers(0, C, 400).astype(np.int32)
        g, o = objs(H, oracle, X, labels=lab, C=C, l2=1e-4)
        alpha = 1.5e308 if kind == "sm1" else 5e307
    cfg = dict(alpha=alpha, epochs=3, inner_steps=50, bits=8, mu=2.0, seed=4)
    oc = oracle.OracleConfig(**cfg)
    orec = oracle.run_halp(o, oc, plan=g.oracle_plan())
    assert orec.status == "diverged"
    with pytest.raises(H.DivergenceError) as ei:
        H.run_halp(g, H.OptimizerConfig(algorithm=H.Algorithm.Halp, **cfg))
    part = ei.value.partial
    rows_equal(part.rows, orec.rows)
    assert np.array_equal(part.final_iterate, orec.final_iterate)
    assert part.steps_taken == orec.steps_taken
