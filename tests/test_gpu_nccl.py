"""The NCCL route of the row-sharded full gradient, executed on one B200.

At world_size 1 with collective=True the library creates a 1-rank NCCL
communicator, all-gathers its (D+1)-double subtree root and runs the
rank-tree finalize (k_finalize) -- the same code path every rank takes at
G = 2/4/8 (halp_capi.cpp gather_finalize).  Results must be bit-identical
to the direct path: the reduction tree is the same for any power-of-two G
(tests/test_multirank.py checks the G > 1 host logic)."""
import ctypes
import os
import subprocess
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def H():
    import torch  # noqa: F401  (loads torch's libnccl.so.2, which the library dlopens)

    import paper_1803_03383_b200 as H
    from paper_1803_03383_b200 import build

    build.build()
    return H


def unique_id():
    nccl = ctypes.CDLL("libnccl.so.2")
    idb = ctypes.create_string_buffer(128)
    assert nccl.ncclGetUniqueId(idb) == 0
    return idb.raw


@pytest.mark.parametrize("kind", ["squared", "softmax"])
def test_nccl_route_bit_identical(H, oracle, kind):
    if kind == "squared":
        X, y = oracle.generate("regression", 20000, 256, dtype="f32", noise_sd=0.1, seed=3)
        ds = H.Dataset(X, targets=y)
        loss, l2 = H.LossFamily.Squared, 1e-4
    else:
        X, y = oracle.generate("softmax", 20000, 100, num_classes=10, dtype="f32", density=0.3, seed=2)
        ds = H.Dataset(X, labels=y, num_classes=10)
        loss, l2 = H.LossFamily.Softmax, 1e-4
    direct = H.Objective(ds, loss, l2)
    viaccl = H.Objective(ds, loss, l2, world_size=1, rank=0, nccl_id=unique_id(), collective=True)
    w = np.random.default_rng(1).standard_normal(direct.dim()) * 0.1
    g0, l0 = direct._fullpass(w)
    g1, l1 = viaccl._fullpass(w)
    assert np.array_equal(g0, g1) and l0 == l1
    cfg = H.OptimizerConfig(algorithm=H.Algorithm.Halp, alpha=1e-3, epochs=3, inner_steps=2000, bits=8, mu=2.0, seed=4)
    r0, r1 = H.run_halp(direct, cfg), H.run_halp(viaccl, cfg)
    assert [(r.loss, r.grad_norm, r.delta, r.iterate_hash) for r in r0.rows] == \
        [(r.loss, r.grad_norm, r.delta, r.iterate_hash) for r in r1.rows]
    assert np.array_equal(r0.final_iterate, r1.final_iterate)
    # the benchmark helper includes the all-gather + finalize on the NCCL route
    assert viaccl.bench_full_gradient(2) > 0
    t = viaccl.timing()
    assert t["finalize_ms"] > 0


def test_nccl_route_needs_an_id(H, oracle):
    X, y = oracle.generate("regression", 1000, 16, dtype="f32", seed=1)
    with pytest.raises(H.InvalidInputError):
        H.Objective(H.Dataset(X, targets=y), H.LossFamily.Squared, 0.0, collective=True)


CHILD = r"""
import sys, ctypes
sys.path.insert(0, sys.argv[1])
import torch
import numpy as np
import paper_1803_03383_b200 as H
X = np.ones((64, 8), dtype=np.float32); y = np.ones(64)
bad = bytes([0xAB]) * 128   # not a bootstrap handle any root listens on
try:
    H.Objective(H.Dataset(X, targets=y), H.LossFamily.Squared, 0.0, world_size=1, rank=0, nccl_id=bad, collective=True)
    print("NO_ERROR")
except H.HalpCudaError as e:
    print("NCCL_ERROR" if "nccl" in str(e).lower() else "OTHER", e)
"""


def test_bad_nccl_id_is_an_nccl_error(H):
    env = dict(os.environ, NCCL_SOCKET_RETRY_CNT="2", NCCL_SOCKET_RETRY_SLEEP_MSEC="50")
    try:
        r = subprocess.run([sys.executable, "-c", CHILD, ROOT], capture_output=True, text=True, timeout=240, env=env)
    except subprocess.TimeoutExpired:
        pytest.fail("ncclCommInitRank with a bogus id did not return within 240 s")
    assert "NCCL_ERROR" in r.stdout, r.stdout + r.stderr[-2000:]


@pytest.mark.parametrize("G", [2, 4, 8])
@pytest.mark.parametrize("kind", ["squared", "two_class_bf16", "softmax10"])
def test_rank_plumbing_g_ranks(H, oracle, G, kind):
    """G ranks of the library on one GPU (collective="host"): each rank's K1
    over its own aligned split block + split tree, the caller concatenates the
    roots (what ncclAllGather does), every rank finalizes -- bit-identical to
    the single-GPU pass and to the oracle's split_subtree / finalize."""
    if kind == "squared":
        X, y = oracle.generate("regression", 50000, 300, dtype="f32", noise_sd=0.1, seed=6)
        ds, loss, l2, C = H.Dataset(X, targets=y), H.LossFamily.Squared, 1e-4, 1
        o = oracle.OracleObjective(X, y=y, l2=l2)
    elif kind == "two_class_bf16":
        X, y = oracle.generate("logistic", 40000, 256, dtype="bf16", x_scale=1 / 16, seed=7)
        ds, loss, l2, C = H.Dataset(X, labels=y, num_classes=2), H.LossFamily.Softmax, 1e-5, 2
        o = oracle.OracleObjective(X, labels=y, num_classes=2, l2=l2)
    else:
        X, y = oracle.generate("softmax", 30000, 64, num_classes=10, dtype="f32", density=0.3, seed=8)
        ds, loss, l2, C = H.Dataset(X, labels=y, num_classes=10), H.LossFamily.Softmax, 1e-4, 10
        o = oracle.OracleObjective(X, labels=y, num_classes=10, l2=l2)
    single = H.Objective(ds, loss, l2)
    w = np.random.default_rng(G).standard_normal(single.dim()) * 0.2
    g1, l1 = single._fullpass(w)
    ranks = [H.Objective(ds, loss, l2, world_size=G, rank=r, collective="host") for r in range(G)]
    roots = np.stack([rk.rank_partial(w) for rk in ranks])
    for r, rk in enumerate(ranks):
        pl = rk.plan()
        assert pl["fg_split_end"] - pl["fg_split_begin"] == pl["fg_splits"] // G
        assert pl["fg_split_begin"] == r * pl["fg_splits"] // G
        # the oracle's subtree of the same split block
        ref_root = o.split_subtree(w, rk.oracle_plan(), pl["fg_split_begin"], pl["fg_split_end"])
        assert np.array_equal(roots[r], ref_root), r
        g, l = rk.finalize_gathered(w, roots)
        assert np.array_equal(g, g1) and l == l1, r
    og, ol = o.finalize(w, roots)
    assert np.array_equal(og, g1) and ol == l1
    with pytest.raises(H.InvalidInputError):
        H.run_halp(ranks[0], H.OptimizerConfig(algorithm=H.Algorithm.Halp, epochs=1, inner_steps=10, mu=1.0))
