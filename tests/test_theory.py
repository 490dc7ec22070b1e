"""lpopt::theory restated (paper_1803_03383_b200/theory.py) against the
reference's frozen expectations (proj/tests/test_theory.cpp:12-96), and the
clipping-variant config rule (optimizers.cpp:641-656)."""
import math

import pytest


@pytest.fixture(scope="module")
def th():
    from paper_1803_03383_b200 import theory

    return theory


def test_step_size(th):
    import paper_1803_03383_b200 as H

    assert th.step_size(0.5, 1.0) == pytest.approx(1.0 / 12.0, rel=1e-15)
    assert th.step_size(0.5, 4.0) == pytest.approx(1.0 / 48.0, rel=1e-15)
    a = th.step_size(0.9, 7.0)
    assert a * 4.0 * 7.0 * 1.9 == pytest.approx(0.9, rel=1e-15)
    for args in ((0.0, 1.0), (1.0, 1.0), (0.5, 0.0)):
        with pytest.raises(H.InvalidInputError):
            th.step_size(*args)


def test_epoch_lengths_and_bits(th):
    import paper_1803_03383_b200 as H

    assert th.epoch_length_lpsvrg(0.5, 1.0) == 48 and th.epoch_length_lpsvrg(0.5, 10.0) == 480
    prev = 0
    for k in (1.0, 2.0, 5.0, 17.0, 300.0):
        t = th.epoch_length_lpsvrg(0.5, k)
        assert t >= prev
        prev = t
    with pytest.raises(H.InvalidInputError):
        th.epoch_length_lpsvrg(1.0, 2.0)
    with pytest.raises(H.InvalidInputError):
        th.epoch_length_lpsvrg(0.5, 0.5)
    assert [th.min_bits_halp(0.5, k, dm) for k, dm in ((1.0, 1.0), (32.0, 1.0), (64.0, 1.0), (4.0, 64.0))] == \
        [4, 8, 9, 8]
    for k in (2.0, 8.0, 128.0):
        assert 0 <= th.min_bits_halp(0.5, 2 * k, 16.0) - th.min_bits_halp(0.5, k, 16.0) <= 2
    assert th.epoch_length_halp(0.5, 1.0, 1.0, 8) == 49
    assert th.epoch_length_halp(0.5, 4.0, 64.0, 8) == 807
    assert th.epoch_length_halp(0.5, 1.0, 1.0, 4) == 64
    with pytest.raises(th.InfeasiblePrecisionError):
        th.epoch_length_halp(0.5, 1.0, 1.0, 3)
    assert th.epoch_length_halp(0.3, 1.0, 1.0, 64) == th.epoch_length_lpsvrg(0.3, 1.0)
    for kappa in (1.0, 3.0, 10.0, 100.0):
        for dim in (1.0, 16.0, 1000.0):
            bmin = th.min_bits_halp(0.5, kappa, dim)
            th.epoch_length_halp(0.5, kappa, dim, bmin)
            if bmin > 2:
                with pytest.raises(th.InfeasiblePrecisionError):
                    th.epoch_length_halp(0.5, kappa, dim, bmin - 1)


def test_accuracy_floor_and_scale(th):
    import paper_1803_03383_b200 as H

    assert th.accuracy_floor(1.0, 1.0, 1.0, 0.5) == pytest.approx(8.0, rel=1e-15)
    assert th.accuracy_floor(100.0, 0.7, 1.0, 0.5) == pytest.approx(392.0, rel=1e-12)
    f1, f2 = th.accuracy_floor(17.0, 0.3, 2.5, 0.25), th.accuracy_floor(17.0, 0.6, 2.5, 0.25)
    assert f2 == pytest.approx(4.0 * f1, rel=1e-12)
    for args in ((1.0, 0.0, 1.0, 0.5), (1.0, 1.0, 1.0, 1.0)):
        with pytest.raises(H.InvalidInputError):
            th.accuracy_floor(*args)
    assert th.halp_scale(1.0, 1.0, 8) == pytest.approx(1.0 / 127.0, rel=1e-15)
    assert th.halp_scale(0.0, 3.0, 8) == 0.0
    assert th.halp_scale(2.5, 0.7, 8) * 127.0 == pytest.approx(2.5 / 0.7, rel=1e-15)
    for args in ((-1.0, 1.0, 8), (1.0, 0.0, 8), (1.0, 1.0, 65)):
        with pytest.raises(H.InvalidInputError):
            th.halp_scale(*args)


def test_clipping_variant_config():
    import paper_1803_03383_b200 as H

    base = H.OptimizerConfig(algorithm=H.Algorithm.Halp, bits=8, mu=3.0)
    c = H.clipping_variant_config(base, H.ClipMode.Clip)
    assert c.bits == 16 and c.mu == 3.0 and base.bits == 8
    s = H.clipping_variant_config(base, H.ClipMode.Scale)
    assert s.bits == 16 and s.mu == 3.0 * 127.0 / 32767.0
    with pytest.raises(H.InvalidInputError, match="bit-centered runs only"):
        H.clipping_variant_config(H.OptimizerConfig(algorithm=H.Algorithm.Svrg, bits=8), H.ClipMode.Clip)
    with pytest.raises(H.InvalidInputError, match="base must be narrower"):
        H.clipping_variant_config(H.OptimizerConfig(algorithm=H.Algorithm.Halp, bits=16), H.ClipMode.Clip)
    assert math.isclose(s.mu * (2**15 - 1), base.mu * 127.0)
