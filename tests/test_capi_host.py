"""CPU-side checks of the product library: it loads, exports every symbol
include/halp.h declares, and its host logic (kernel plan, shard plan, GF(2)
RNG jump-ahead) is right.  No compute call needs a GPU here."""
import re
import os

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def H():
    from paper_1803_03383_b200 import build

    build.build()
    import paper_1803_03383_b200 as H

    return H


def test_exports_every_declared_symbol(H):
    from paper_1803_03383_b200 import _capi

    hdr = open(os.path.join(ROOT, "include", "halp.h")).read()
    declared = set(re.findall(r"\b(halp_[a-z_0-9]+)\s*\(", hdr))
    assert declared == set(_capi.SYMBOLS), declared ^ set(_capi.SYMBOLS)
    L = _capi.lib()
    for s in declared:
        assert getattr(L, s) is not None
    assert L.halp_abi_version() == 4


def test_no_cpu_fallback(H):
    # without a B200 every compute entry point fails loudly
    import torch

    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(H.HalpCudaError):
        H.Objective(H.Dataset(np.zeros((4, 3)), targets=np.zeros(4)))


def test_rng_jump_matches_sequential(H, oracle):
    for seed, stream, count in [(0, 0, 0), (42, 1, 1), (7, 0, 12345), (3, 1, 10**6 + 17)]:
        r = oracle.QuantRng(seed, stream)
        for _ in range(count):
            r.next_u64()
        assert H.rng_state_after(seed, stream, count) == r.state


def test_shard_plan_partitions_rows(H):
    for n, d, C, dt in [(4194304, 4096, 1, 1), (16777216, 1024, 2, 2), (60000, 784, 10, 1), (1000, 100, 1, 0)]:
        for world in (1, 2, 4, 8):
            plans = [H.shard_plan(n, d, C, dt, world, r) for r in range(world)]
            S = plans[0]["splits"]
            assert S & (S - 1) == 0 and S >= world
            assert plans[0]["row_begin"] == 0 and plans[-1]["row_end"] == n
            for a, b in zip(plans, plans[1:]):
                assert a["row_end"] == b["row_begin"] and a["split_end"] == b["split_begin"]
            # every rank owns an aligned subtree of the split tree
            for p in plans:
                assert p["split_end"] - p["split_begin"] == S // world
            # the split count does not depend on the GPU count (G-invariant order)
            assert S == H.shard_plan(n, d, C, dt, 1, 0)["splits"] or world > S


def test_plan_for_configs(H):
    p = H.plan_for(4194304, 4096, 1, "f32")
    assert p["fg_threads"] in (256, 512) and p["fg_vec"] == 4 and p["fg_splits"] == 4096
    # C3's 16 KB rows: 4-row 64 KB tiles in a 3-deep ring (measured)
    assert (p["fg_rows_per_stage"], p["fg_stages"]) == (4, 3)
    p = H.plan_for(16777216, 1024, 2, "bf16")  # C4: 16-row tiles re-read from shared memory
    assert (p["fg_threads"], p["fg_rows_per_stage"], p["fg_stages"]) == (128, 16, 2)
    # streaming plans (up to 4 feature groups per thread): a tile never exceeds 64 KB, a ring never 220 KB
    for dt, es in (("f32", 4), ("f64", 8), ("bf16", 2)):
        for d in (24, 256, 1000, 1024, 2048, 3500, 4096):
            if (d * es + 15) // 16 > 4 * 256:
                continue  # wider rows take the generic kernel
            q = H.plan_for(100000, d, 1, dt)
            row = (d * es + 15) // 16 * 16
            assert q["fg_rows_per_stage"] * row <= 64 * 1024, (dt, d, q)
            assert q["fg_rows_per_stage"] * row * q["fg_stages"] <= 220 * 1024, (dt, d, q)
    p = H.plan_for(60000, 784, 10, "f32")
    assert p["in_ctas"] * p["in_threads"] * p["in_per"] >= 7840
    with pytest.raises(H.UnsupportedError):
        H.plan_for(1000, 100000, 1, "f32")
    with pytest.raises(H.InvalidInputError):
        H.plan_for(1000, 100, 1, "f32", world=3)
