"""Host restatement of the K6 generator (oracle/datagen.c): row ranges are
slices of the full dataset, thread count does not change the bytes, and the
distributions are the ones BASELINE.json names (CPU only; the byte-equality
with K6 itself is tests/test_gpu_datagen.py)."""
import numpy as np


def test_row_range_and_threads(oracle):
    X, y = oracle.generate("regression", 500, 70, dtype="f32", noise_sd=0.1, seed=3, threads=1)
    X2, y2 = oracle.generate("regression", 500, 70, dtype="f32", noise_sd=0.1, seed=3, rows=(123, 456), threads=7)
    assert np.array_equal(X[123:456], X2) and np.array_equal(y[123:456], y2)
    L, lab = oracle.generate("softmax", 300, 50, num_classes=10, density=0.2, seed=1, threads=3)
    L2, lab2 = oracle.generate("softmax", 300, 50, num_classes=10, density=0.2, seed=1, rows=(100, 300))
    assert np.array_equal(L[100:], L2) and np.array_equal(lab[100:], lab2)


def test_distributions(oracle):
    X, y = oracle.generate("regression", 2000, 500, dtype="f64", noise_sd=0.0, seed=1)
    assert abs(X.mean()) < 5e-3 and abs(X.std() - 1.0) < 5e-3
    # y = x.w* exactly when noise_sd = 0: var(y) ~ d
    assert 0.8 * 500 < y.var() < 1.2 * 500
    S, lab = oracle.generate("softmax", 20000, 784, num_classes=10, dtype="f32", density=0.2, seed=0)
    assert abs((S > 0).mean() - 0.2) < 2e-3 and S.max() < 1.0 and S.min() >= 0.0
    assert len(np.unique(lab)) == 10
    B, bl = oracle.generate("logistic", 20000, 1024, dtype="bf16", x_scale=1 / 32, seed=4)
    assert B.dtype == np.uint16 and 0.45 < bl.mean() < 0.55
    f = (B.astype(np.uint32) << 16).view(np.float32)
    assert abs(f.std() - 1 / 32) < 1e-3
