"""grid_search input validation (harness.cpp:383-398, :45-61): raised before
any run, so no GPU is involved."""
import pytest


def test_grid_validation():
    import paper_1803_03383_b200 as H

    base = H.OptimizerConfig(algorithm=H.Algorithm.Halp)
    with pytest.raises(H.InvalidInputError, match="metric must be grad_norm or loss"):
        H.grid_search(None, base, [H.GridAxis("alpha", [1e-3])], [1], metric="acc")
    with pytest.raises(H.InvalidInputError, match="need at least one seed"):
        H.grid_search(None, base, [H.GridAxis("alpha", [1e-3])], [])
    with pytest.raises(H.InvalidInputError, match="axis 'mu' has no values"):
        H.grid_search(None, base, [H.GridAxis("mu", [])], [1])
    with pytest.raises(H.InvalidInputError, match="duplicate axis 'alpha'"):
        H.grid_search(None, base, [H.GridAxis("alpha", [1.0]), H.GridAxis("alpha", [2.0])], [1])
    with pytest.raises(H.InvalidInputError, match="unknown parameter 'gamma'"):
        H.grid_search(None, base, [H.GridAxis("gamma", [1.0])], [1])


def test_llround_matches_std():
    from paper_1803_03383_b200.halp import _llround

    assert [_llround(v) for v in (2.5, -2.5, 7.49, 16.0, 0.5)] == [3, -3, 7, 16, 1]
