"""Oracle pinned against the reference's own known-answer tests.

RNG: proj/tests/test_rng.cpp:10-32,99-105 (frozen outputs, Box-Muller draw count).
Quantizer: proj/tests/test_fixed_point.cpp:78-100,121-130,144-176.
halp_scale: proj/tests/test_optimizers.cpp:331-350 and theory.cpp:93-102.
"""
import json
import math
import os

import numpy as np
import pytest

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def test_rng_frozen_outputs(oracle):
    kats = json.load(open(os.path.join(GOLD, "rng_kats.json")))["kats"]
    assert len(kats) == 4
    for k in kats:
        r = oracle.QuantRng(k["seed"], k["stream"])
        for v in k["u64"]:
            assert r.next_u64() == v
        for v in k["uniform"]:
            assert r.next_uniform() == pytest.approx(v, rel=1e-15)


def test_rng_streams_and_seeds_decorrelate(oracle):
    a, b, c, d = (oracle.QuantRng(123, 0), oracle.QuantRng(123, 0), oracle.QuantRng(123, 1), oracle.QuantRng(124, 0))
    ds = dd = 0
    for _ in range(64):
        va = a.next_u64()
        assert va == b.next_u64()
        ds += va != c.next_u64()
        dd += va != d.next_u64()
    assert ds > 60 and dd > 60


def test_normal_consumes_two_uniforms(oracle):
    a, b = oracle.QuantRng(31), oracle.QuantRng(31)
    a.next_normal()
    b.next_uniform()
    b.next_uniform()
    assert a.next_u64() == b.next_u64()


def test_next_index_range(oracle):
    r = oracle.QuantRng(5)
    assert r.next_index(1) == 0
    hist = np.zeros(10, int)
    for _ in range(20000):
        k = r.next_index(10)
        assert 0 <= k < 10
        hist[k] += 1
    assert np.all(np.abs(hist - 2000) < 5 * math.sqrt(2000 * 0.9))


def test_quantizer_deterministic_branches(oracle):
    q = oracle.quantize_code
    # test_fixed_point.cpp:82-99 (delta 0.5, 8 bits)
    assert q(0.0, 0.5, 8, 0.999) == 0
    assert q(3.5, 0.5, 8, 0.999) == 7
    assert q(-3.0, 0.5, 8, 0.999) == -6
    assert q(63.5 + 5 * 0.5, 0.5, 8, 0.3) == 127
    assert q(-1e9, 0.5, 8, 0.3) == -128
    assert q(1.7, 1.0, 2, 0.0) == 1  # tiny lattice {-2,-1,0,1}
    with pytest.raises(oracle.OracleInvalidInput):
        q(float("nan"), 0.5, 8, 0.1)
    with pytest.raises(oracle.OracleInvalidInput):
        q(float("inf"), 0.5, 8, 0.1)


def test_quantizer_rounding_probability(oracle):
    # test_fixed_point.cpp:121-130: 5.3 at delta 1 rounds up with p = 0.3
    r = oracle.QuantRng(99)
    n = 50000
    up = sum(oracle.quantize_code(5.3, 1.0, 8, r.next_uniform()) == 6 for _ in range(n))
    assert up / n == pytest.approx(0.3, rel=0.05)


def test_quantizer_idempotent(oracle):
    # test_fixed_point.cpp:144-155
    rng, seq = oracle.QuantRng(7), oracle.QuantRng(8)
    for b in (4, 8, 16, 32, 50):
        for _ in range(200):
            x = (seq.next_uniform() - 0.5) * 2e3
            c = oracle.quantize_code(x, 0.013, b, rng.next_uniform())
            c2 = oracle.quantize_code(c * 0.013, 0.013, b, rng.next_uniform())
            assert c2 == c


def test_halp_scale(oracle):
    assert oracle.halp_scale(2.0, 3.0, 8) == 2.0 / (3.0 * 127.0)
    assert oracle.halp_scale(1.0, 1.0, 16) == 1.0 / 32767.0


def test_mirror_exp_log_accuracy(oracle):
    xs = np.concatenate([np.linspace(-740, 709, 4001), np.linspace(-1, 1, 2001), [-1e-300, 0.0, 1e-300]])
    for x in xs:
        e = oracle.mexp(float(x))
        ref = math.exp(float(x))
        assert abs(e - ref) <= 2 * np.spacing(ref) + 1e-320
    for x in np.concatenate([np.geomspace(1e-300, 1e300, 3001), np.linspace(0.5, 2.0, 2001)]):
        l = oracle.mlog(float(x))
        ref = math.log(float(x))
        assert abs(l - ref) <= 2 * np.spacing(abs(ref)) + 1e-300
