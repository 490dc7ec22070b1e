"""Host-side harness logic (no GPU): the reference's dataset generators,
the experiment spec / manifest JSON (checked byte for byte against the
reference's own manifest, proj/out/regression_floor/manifest.json), trace
CSV reading, and the conditioned generator's advertised spectrum
(tests/test_objectives.cpp:141-157 restated)."""
import json
import math
import os

import numpy as np
import pytest

import paper_1803_03383_b200 as H
from paper_1803_03383_b200 import harness as HR

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def test_make_regression_matches_oracle(oracle):
    ds = HR.make_regression(300, 17, 0.25, 9)
    X, y = oracle.make_regression(300, 17, 0.25, 9)
    assert np.array_equal(ds.X, X) and np.array_equal(ds.targets, y)
    with pytest.raises(H.InvalidInputError):
        HR.make_regression(0, 3, 0.0, 1)


def test_make_classification_shape():
    ds = HR.make_classification(60, 5, 3, 12.0, 11)
    assert ds.X.shape == (60, 5) and list(ds.labels[:6]) == [0, 1, 2, 0, 1, 2] and ds.num_classes == 3
    # well separated: each row is nearest to its own class mean
    means = np.stack([ds.X[ds.labels == c].mean(0) for c in range(3)])
    pred = np.argmin(((ds.X[:, None, :] - means[None]) ** 2).sum(-1), axis=1)
    assert (pred == ds.labels).mean() > 0.9


@pytest.mark.parametrize("kappa", [1.0, 16.0, 1024.0])
def test_conditioned_spectrum(kappa):
    ds = HR.make_conditioned_regression(kappa, 5)
    assert ds.X.shape == (1000, 64)
    ev = np.linalg.eigvalsh(ds.X.T @ ds.X / 1000.0)
    assert ev[0] == pytest.approx(1.0, rel=1e-6) and ev[-1] == pytest.approx(kappa, rel=1e-6)
    w = np.linalg.lstsq(ds.X, ds.targets, rcond=None)[0]
    loss = 0.5 * np.mean((ds.X @ w - ds.targets) ** 2)
    assert loss < 1e-15 * kappa
    a, b = HR.make_conditioned_regression(4.0, 7), HR.make_conditioned_regression(4.0, 7)
    assert np.array_equal(a.X, b.X)
    with pytest.raises(H.InvalidInputError):
        HR.make_conditioned_regression(0.5, 1)


def test_manifest_json_byte_identical_to_reference():
    """spec -> experiment_to_json + the reference's own run summaries -> the
    reference's manifest text, byte for byte (key order, indent, numbers)"""
    gold_text = open(os.path.join(GOLD, "regression_floor_manifest.json")).read()
    gold = json.loads(gold_text)
    spec = HR.experiment_from_json(json.load(open(os.path.join(GOLD, "regression_floor.json")))["spec"])
    m = HR.experiment_to_json(spec)
    m["runs"] = gold["runs"]
    assert HR.dump_json(m) + "\n" == gold_text
    # and the manifest is itself a runnable spec
    again = HR.experiment_from_json(gold)
    assert HR.experiment_to_json(again) == HR.experiment_to_json(spec)


def test_spec_validation():
    with pytest.raises(H.InvalidInputError):
        HR.experiment_from_json({"configs": []})
    with pytest.raises(H.InvalidInputError):
        HR.experiment_from_json({"configs": [{"algo": "halp", "alpha": 1e-3}, {"algo": "halp", "alpha": 1e-2}]})
    with pytest.raises(H.InvalidInputError):
        HR.experiment_from_json({"configs": [{"algo": "adam", "alpha": 1e-3}]})
    with pytest.raises(H.InvalidInputError):
        HR.experiment_from_json({"configs": [{"algo": "halp"}]})
    s = HR.experiment_from_json({"configs": [{"algo": "lp_svrg", "alpha": 1, "option": "II"}], "repetitions": 3,
                                 "seed_base": 10})
    assert s.seeds == [10, 11, 12] and s.configs[0].name == "lp-svrg"
    assert s.configs[0].config.option == H.EpochOption.SampledIterate and s.configs[0].config.alpha == 1.0
    with pytest.raises(H.UnsupportedError):
        HR.build_dataset(HR.DatasetSpec(kind="idx"))
    with pytest.raises(H.InvalidInputError):
        HR.build_dataset(HR.DatasetSpec(kind="parquet"))
    with pytest.raises(H.InvalidInputError):
        HR.resolve_loss(HR.ObjectiveSpec("hinge", 0.0), HR.make_regression(5, 2, 0.0, 1))
    assert HR.sanitize_name("halp 8/x") == "halp-8-x"
    with pytest.raises(H.InvalidInputError):
        HR.conditioning_sweep([], [8], 100, 1, 3)
    with pytest.raises(H.InvalidInputError):
        HR.conditioning_sweep([4.0], [8], 0, 1, 3)


def test_read_run_csv(tmp_path):
    rec = H.RunRecord(rows=[H.MetricRow(0.0, 0.5, 2.0, 1.5, 0.25), H.MetricRow(2.0, 1.0, 1.0, 0.5, 0.125)])
    p = str(tmp_path / "t.csv")
    H.write_run_csv(p, rec)
    back = HR.read_run_csv(p)
    assert [(r.pass_, r.seconds, r.loss, r.grad_norm, r.delta) for r in back] == \
        [(r.pass_, r.seconds, r.loss, r.grad_norm, r.delta) for r in rec.rows]
    with pytest.raises(HR.IoError):
        HR.read_run_csv(str(tmp_path / "absent.csv"))
    (tmp_path / "bad.csv").write_text("pass,loss\n0,1\n")
    with pytest.raises(HR.IoError):
        HR.read_run_csv(str(tmp_path / "bad.csv"))
    (tmp_path / "ragged.csv").write_text("pass,seconds,loss,grad_norm,delta\n1,2,3\n")
    with pytest.raises(HR.IoError):
        HR.read_run_csv(str(tmp_path / "ragged.csv"))


def test_sweep_grids():
    a, m = HR.sweep_alphas(), HR.sweep_mus()
    assert len(a) == 17 and a[0] == 1e-10 and a[-1] == pytest.approx(1e-2)
    assert len(m) == 13 and m[0] == pytest.approx(0.5) and m[-1] == pytest.approx(2000.0)
