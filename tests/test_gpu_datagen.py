"""K6 (the device generator of the BASELINE configs' synthetic data) against
its host restatement oracle/datagen.c: identical bytes for every kind and
dtype, including row ranges deep into a large dataset (64-bit element
indices), so the CPU arms of bench.py build exactly the GPU arm's inputs."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def H():
    import paper_1803_03383_b200 as H
    from paper_1803_03383_b200 import build

    build.build()
    return H


def as_host(t):
    import torch

    if t.dtype == torch.bfloat16:
        return t.view(torch.int16).cpu().numpy().view(np.uint16)
    return t.cpu().numpy()


CASES = [
    ("regression", dict(n=3000, d=256, dtype="f32", noise_sd=0.1, seed=3)),
    ("regression", dict(n=1000, d=100, dtype="f64", noise_sd=0.0, seed=42)),
    ("regression", dict(n=777, d=37, dtype="bf16", noise_sd=0.5, x_scale=0.25, seed=9)),
    ("softmax", dict(n=2000, d=784, num_classes=10, dtype="f32", density=0.2, seed=0)),
    ("softmax", dict(n=500, d=33, num_classes=15, dtype="bf16", density=0.5, seed=1)),
    ("logistic", dict(n=4096, d=1024, dtype="bf16", x_scale=1 / 32, seed=4)),
    ("logistic", dict(n=999, d=64, dtype="f32", x_scale=0.125, seed=5)),
]


@pytest.mark.parametrize("kind,kw", CASES)
def test_k6_matches_host(H, oracle, kind, kw):
    Xg, yg = H.generate(kind, **kw)
    Xh, yh = oracle.generate(kind, **kw)
    assert np.array_equal(as_host(Xg), Xh)
    assert np.array_equal(as_host(yg), yh)


def test_k6_row_range_large(H, oracle):
    """the last rows of a 4,194,304-row dataset (C3's row count; e = i*d + j > 2^32)"""
    n, d = 4194304, 1024
    Xg, yg = H.generate("regression", n, d, dtype="f32", noise_sd=0.1, seed=3)
    r0, r1 = n - 300, n
    Xh, yh = oracle.generate("regression", n, d, dtype="f32", noise_sd=0.1, seed=3, rows=(r0, r1))
    assert np.array_equal(as_host(Xg[r0:r1]), Xh)
    assert np.array_equal(as_host(yg[r0:r1]), yh)
    Xh0, yh0 = oracle.generate("regression", n, d, dtype="f32", noise_sd=0.1, seed=3, rows=(0, 64))
    assert np.array_equal(as_host(Xg[:64]), Xh0)
    assert np.array_equal(as_host(yg[:64]), yh0)
