"""The reference's experiment harness around the B200 solver (SURVEY.md 8f,
rows 1 and 4): datasets from a spec, run_experiment with its trace CSVs and
runnable manifest, and the conditioning sweep.  Mirrors
proj/include/lpopt/harness.hpp + proj/src/harness.cpp (same names, fields,
file formats and error behaviour); every solve runs on the B200 through
halp.run_prepared / grid_search (the HALP grids as one K5 launch each).

  reference (harness.cpp)                  here
  ---------------------------------------  ---------------------------------
  DatasetSpec / ObjectiveSpec / NamedConfig /  same dataclasses
  ExperimentSpec / RunOutput / ExperimentResult
  build_dataset (:70-93)                   build_dataset
  resolve_loss (:95-103)                   resolve_loss
  *_from_json / config_to_json /           experiment_from_json, load_experiment_file,
  experiment_to_json (:105-244)            config_to_json, experiment_to_json
  read_run_csv (:263-294)                  read_run_csv (write_run_csv: halp.py)
  run_experiment (:314-377)                run_experiment
  make_conditioned_regression              make_conditioned_regression
    (objectives.cpp:79-108)
  conditioning_sweep / write_sweep_csv     conditioning_sweep / write_sweep_csv
    (:449-539)

Dataset files (kind "csv" / "idx", dataset_io.cpp) are outside the B200 hot
path: build_dataset raises UnsupportedError for them.
"""
from __future__ import annotations

import copy
import ctypes as C
import json
import math
import os
from dataclasses import dataclass, field
from typing import List, Optional

import numpy as np

from . import _capi as A
from .halp import (Algorithm, Dataset, DivergenceError, EpochOption, GridAxis, InvalidInputError, LossFamily,  # noqa: F401
                   Objective, OptimizerConfig, RunRecord, UnsupportedError, format_double, grid_search, run_prepared,
                   write_run_csv, MetricRow)


class IoError(RuntimeError):
    """lpopt::IoError (errors.hpp)."""


# ---------------------------------------------------------------- specs (harness.hpp:15-60)
@dataclass
class DatasetSpec:
    kind: str = "regression"  # regression | classification | conditioned | csv | idx
    n: int = 1000
    d: int = 100
    noise_sd: float = 0.0
    classes: int = 10
    separation: float = 1.0
    kappa: float = 1.0
    seed: int = 0
    path: str = ""
    task: str = "regression"
    images: str = ""
    labels: str = ""


@dataclass
class ObjectiveSpec:
    loss: str = "auto"  # auto | squared | softmax
    l2: float = 0.0


@dataclass
class NamedConfig:
    name: str
    config: OptimizerConfig


@dataclass
class ExperimentSpec:
    dataset: DatasetSpec = field(default_factory=DatasetSpec)
    objective: ObjectiveSpec = field(default_factory=ObjectiveSpec)
    configs: List[NamedConfig] = field(default_factory=list)
    seeds: List[int] = field(default_factory=lambda: [0])
    out_dir: str = "out"


@dataclass
class RunOutput:
    name: str = ""
    seed: int = 0
    csv_path: str = ""
    status: str = ""
    final_loss: float = 0.0
    final_grad_norm: float = 0.0
    rows: int = 0
    steps: int = 0


@dataclass
class ExperimentResult:
    runs: List[RunOutput] = field(default_factory=list)
    records: List[RunRecord] = field(default_factory=list)
    manifest_path: str = ""


# ---------------------------------------------------------------- names (optimizers.cpp:171-201)
_ALGO_NAMES = {Algorithm.Sgd: "sgd", Algorithm.Svrg: "svrg", Algorithm.LpSgd: "lp-sgd", Algorithm.LpSvrg: "lp-svrg",
               Algorithm.Halp: "halp", Algorithm.LmHalp: "lm-halp"}


def algorithm_from_string(s: str) -> Algorithm:
    for a, name in _ALGO_NAMES.items():
        if s == name or s == name.replace("-", "_"):
            return a
    raise InvalidInputError(f"unknown algorithm '{s}'")


def algorithm_to_string(a) -> str:
    return _ALGO_NAMES[Algorithm(a)]


def epoch_option_from_string(s: str) -> EpochOption:
    if s in ("I", "i", "last"):
        return EpochOption.LastIterate
    if s in ("II", "ii", "sampled"):
        return EpochOption.SampledIterate
    raise InvalidInputError(f"unknown epoch option '{s}' (use I or II)")


def epoch_option_to_string(o) -> str:
    return "I" if EpochOption(o) == EpochOption.LastIterate else "II"


# ---------------------------------------------------------------- datasets
def make_regression(n: int, d: int, noise_sd: float, seed: int) -> Dataset:
    """objectives.cpp:27-45 (host generator in libhalp_b200.so, the reference's draw order)"""
    if n < 1 or d < 1:
        raise InvalidInputError("make_regression: n and d must be positive")
    if not (math.isfinite(noise_sd) and noise_sd >= 0.0):
        raise InvalidInputError("make_regression: noise_sd must be finite and >= 0")
    X = np.empty((n, d), dtype=np.float64)
    y = np.empty(n, dtype=np.float64)
    A.lib().halp_make_regression(n, d, float(noise_sd), int(seed) & (2**64 - 1), X.ctypes.data, y.ctypes.data)
    return Dataset(X, targets=y)


def make_classification(n: int, d: int, num_classes: int, separation: float, seed: int) -> Dataset:
    """objectives.cpp:46-76"""
    if n < 1 or d < 1:
        raise InvalidInputError("make_classification: n and d must be positive")
    if num_classes < 2:
        raise InvalidInputError("make_classification: need at least two classes")
    if not (math.isfinite(separation) and separation >= 0.0):
        raise InvalidInputError("make_classification: separation must be finite and >= 0")
    X = np.empty((n, d), dtype=np.float64)
    lab = np.empty(n, dtype=np.int32)
    A.lib().halp_make_classification(n, d, num_classes, float(separation), int(seed) & (2**64 - 1), X.ctypes.data,
                                     lab.ctypes.data)
    return Dataset(X, labels=lab, num_classes=num_classes)


def _normals(seed: int, stream: int, count: int) -> np.ndarray:
    out = np.empty(count, dtype=np.float64)
    A.lib().halp_normals(int(seed) & (2**64 - 1), stream, count, out.ctypes.data)
    return out


def make_conditioned_regression(kappa: float, seed: int) -> Dataset:
    """objectives.cpp:79-108: X = U diag(sigma) V^T with orthonormal U (1000 x 64)
    and V (64 x 64) from Householder QR of Gaussian matrices drawn row-wise
    from one QuantRng(seed) stream (then w_true from the same stream), sigma_j =
    sqrt(n kappa^(j/(d-1))) so the Hessian X^T X / n has eigenvalues
    kappa^(j/(d-1)) from exactly 1 to kappa; noiseless targets y = X w_true.
    The QR factorisations are LAPACK's (numpy) instead of Eigen's
    HouseholderQR: the same construction and spectrum, not the same bits
    (the reference pins this generator only by its spectrum, determinism and
    zero-loss optimum, tests/test_objectives.cpp:141-157)."""
    if not (math.isfinite(kappa) and kappa >= 1.0):
        raise InvalidInputError("make_conditioned_regression: kappa must be >= 1")
    n, d = 1000, 64
    g = _normals(seed, 0, n * d + d * d + d)
    a = g[: n * d].reshape(n, d)
    b = g[n * d: n * d + d * d].reshape(d, d)
    w_true = g[n * d + d * d:]
    u = np.linalg.qr(a, mode="reduced")[0]
    v = np.linalg.qr(b, mode="reduced")[0]
    sigma = np.array([math.sqrt(float(n) * math.pow(kappa, j / (d - 1))) for j in range(d)])
    X = (u * sigma) @ v.T
    return Dataset(np.ascontiguousarray(X), targets=X @ w_true)


def build_dataset(spec: DatasetSpec) -> Dataset:
    """harness.cpp:70-93"""
    if spec.kind == "regression":
        return make_regression(spec.n, spec.d, spec.noise_sd, spec.seed)
    if spec.kind == "classification":
        return make_classification(spec.n, spec.d, spec.classes, spec.separation, spec.seed)
    if spec.kind == "conditioned":
        return make_conditioned_regression(spec.kappa, spec.seed)
    if spec.kind in ("csv", "idx"):
        raise UnsupportedError(f"dataset: '{spec.kind}' files are outside the B200 hot path (load them yourself and "
                               "pass a Dataset)")
    raise InvalidInputError(f"dataset: unknown kind '{spec.kind}'")


def resolve_loss(ospec: ObjectiveSpec, ds: Dataset) -> LossFamily:
    """harness.cpp:95-103"""
    if ospec.loss == "auto":
        return LossFamily.Softmax if ds.is_classification() else LossFamily.Squared
    if ospec.loss == "squared":
        return LossFamily.Squared
    if ospec.loss == "softmax":
        return LossFamily.Softmax
    raise InvalidInputError(f"objective: unknown loss '{ospec.loss}'")


# ---------------------------------------------------------------- json (harness.cpp:105-244)
def _get(j: dict, key: str, default, typ):
    if key not in j:
        return default
    v = j[key]
    ok = isinstance(v, typ) and not (typ in (int, float) and isinstance(v, bool))
    if typ is float and isinstance(v, int) and not isinstance(v, bool):
        ok = True
    if not ok:
        raise InvalidInputError(f"json: '{key}' has the wrong type")
    return typ(v) if typ is float else v


def dataset_from_json(j: dict) -> DatasetSpec:
    s = DatasetSpec()
    s.kind = _get(j, "kind", s.kind, str)
    s.n = _get(j, "n", s.n, int)
    s.d = _get(j, "d", s.d, int)
    s.noise_sd = _get(j, "noise_sd", s.noise_sd, float)
    s.classes = _get(j, "classes", s.classes, int)
    s.separation = _get(j, "separation", s.separation, float)
    s.kappa = _get(j, "kappa", s.kappa, float)
    s.seed = _get(j, "seed", s.seed, int)
    s.path = _get(j, "path", s.path, str)
    s.task = _get(j, "task", s.task, str)
    s.images = _get(j, "images", s.images, str)
    s.labels = _get(j, "labels", s.labels, str)
    return s


def config_from_json(j: dict) -> OptimizerConfig:
    c = OptimizerConfig()
    if "algo" not in j or "alpha" not in j:
        raise InvalidInputError("config json: 'algo' and 'alpha' are required")
    c.algorithm = algorithm_from_string(_get(j, "algo", "", str))
    c.alpha = _get(j, "alpha", c.alpha, float)
    c.epochs = _get(j, "epochs", c.epochs, int)
    c.inner_steps = _get(j, "inner", c.inner_steps, int)
    c.bits = _get(j, "bits", c.bits, int)
    c.delta = _get(j, "delta", c.delta, float)
    c.mu = _get(j, "mu", c.mu, float)
    c.option = epoch_option_from_string(_get(j, "option", "I", str))
    c.full_grad_period = _get(j, "full_grad_period", c.full_grad_period, int)
    c.seed = _get(j, "seed", c.seed, int)
    c.metric_every_passes = _get(j, "metric_every_passes", c.metric_every_passes, float)
    c.delta_min = _get(j, "delta_min", c.delta_min, float)
    c.divergence_limit = _get(j, "divergence_limit", c.divergence_limit, float)
    return c


def experiment_from_json(j: dict) -> ExperimentSpec:
    s = ExperimentSpec()
    if "dataset" in j:
        s.dataset = dataset_from_json(j["dataset"])
    if "objective" in j:
        s.objective.loss = _get(j["objective"], "loss", s.objective.loss, str)
        s.objective.l2 = _get(j["objective"], "l2", s.objective.l2, float)
    if not isinstance(j.get("configs"), list) or not j["configs"]:
        raise InvalidInputError("experiment json: 'configs' must be a non-empty array")
    names = set()
    for item in j["configs"]:
        cfg = config_from_json(item)
        name = _get(item, "name", algorithm_to_string(cfg.algorithm), str)
        if name in names:
            raise InvalidInputError(f"experiment json: duplicate config name '{name}'")
        names.add(name)
        s.configs.append(NamedConfig(name, cfg))
    if "seeds" in j:
        s.seeds = [int(v) for v in j["seeds"]]
    elif "repetitions" in j:
        reps = int(j["repetitions"])
        if reps < 1:
            raise InvalidInputError("experiment json: repetitions must be >= 1")
        base = int(j.get("seed_base", 0))
        s.seeds = [base + r for r in range(reps)]
    if not s.seeds:
        raise InvalidInputError("experiment json: need at least one seed")
    s.out_dir = _get(j, "out", s.out_dir, str)
    return s


def load_experiment_file(path: str) -> ExperimentSpec:
    try:
        with open(path) as f:
            j = json.load(f)
    except OSError:
        raise IoError(f"cannot open experiment spec {path}")
    except json.JSONDecodeError as e:
        raise IoError(f"experiment spec {path}: {e}")
    return experiment_from_json(j)


def config_to_json(cfg: OptimizerConfig) -> dict:
    return {"algo": algorithm_to_string(cfg.algorithm), "alpha": float(cfg.alpha), "epochs": int(cfg.epochs),
            "inner": int(cfg.inner_steps), "bits": int(cfg.bits), "delta": float(cfg.delta), "mu": float(cfg.mu),
            "option": epoch_option_to_string(cfg.option), "full_grad_period": int(cfg.full_grad_period),
            "seed": int(cfg.seed), "metric_every_passes": float(cfg.metric_every_passes),
            "delta_min": float(cfg.delta_min), "divergence_limit": float(cfg.divergence_limit)}


def experiment_to_json(spec: ExperimentSpec) -> dict:
    ds = spec.dataset
    d = {"kind": ds.kind, "n": int(ds.n), "d": int(ds.d), "noise_sd": float(ds.noise_sd), "classes": int(ds.classes),
         "separation": float(ds.separation), "kappa": float(ds.kappa), "seed": int(ds.seed), "task": ds.task}
    if ds.path:
        d["path"] = ds.path
    if ds.images:
        d["images"] = ds.images
    if ds.labels:
        d["labels"] = ds.labels
    configs = []
    for nc in spec.configs:
        c = config_to_json(nc.config)
        c["name"] = nc.name
        configs.append(c)
    return {"dataset": d, "objective": {"loss": spec.objective.loss, "l2": float(spec.objective.l2)},
            "seeds": [int(v) for v in spec.seeds], "out": spec.out_dir, "configs": configs}


def dump_json(j: dict) -> str:
    """nlohmann::json::dump(2): keys sorted (std::map), 2-space indent, shortest
    round-trip doubles with a trailing '.0' on integral values -- the same
    text Python's json module produces for these value types."""
    return json.dumps(j, indent=2, sort_keys=True)


def _write_text_atomic(path: str, content: str) -> None:
    d = os.path.dirname(path)
    if d:
        os.makedirs(d, exist_ok=True)
    tmp = path + ".tmp"
    with open(tmp, "w", newline="") as f:
        f.write(content)
    os.replace(tmp, path)


# ---------------------------------------------------------------- traces
def read_run_csv(path: str) -> List[MetricRow]:
    """harness.cpp:263-294"""
    try:
        f = open(path)
    except OSError:
        raise IoError(f"cannot open trace {path}")
    with f:
        lines = f.read().split("\n")
    if not lines or lines[0] != "pass,seconds,loss,grad_norm,delta":
        raise IoError(f"trace {path}: unexpected header")
    rows = []
    for line in lines[1:]:
        if not line:
            continue
        fs = line.split(",")
        if len(fs) != 5:
            raise IoError(f"trace {path}: malformed row")
        try:
            v = [float(x) for x in fs]
        except ValueError:
            raise IoError(f"trace {path}: malformed number")
        rows.append(MetricRow(v[0], v[1], v[2], v[3], v[4]))
    return rows


def sanitize_name(name: str) -> str:
    """harness.cpp:33-42"""
    if not name:
        raise InvalidInputError("config name must not be empty")
    return "".join(c if (c.isascii() and (c.isalnum() or c in "-_.")) else "-" for c in name)


# ---------------------------------------------------------------- run_experiment (harness.cpp:314-377)
def run_experiment(spec: ExperimentSpec) -> ExperimentResult:
    """Executes every (config, seed) pair on the B200 (run_prepared), writes one
    trace CSV per run plus a manifest echoing the resolved spec (itself a
    runnable spec), and returns the per-run summaries."""
    if not spec.configs:
        raise InvalidInputError("experiment: no configs")
    if not spec.seeds:
        raise InvalidInputError("experiment: no seeds")
    names = set()
    for nc in spec.configs:
        if nc.name in names:
            raise InvalidInputError(f"experiment: duplicate config name '{nc.name}'")
        names.add(nc.name)
    os.makedirs(spec.out_dir, exist_ok=True)
    ds = build_dataset(spec.dataset)
    lf = resolve_loss(spec.objective, ds)
    base = Objective(ds, lf, spec.objective.l2)
    result = ExperimentResult()
    for nc in spec.configs:
        for seed in spec.seeds:
            cfg = copy.deepcopy(nc.config)
            cfg.seed = int(seed)
            rec = run_prepared(base, cfg, spec.dataset.seed)
            fname = sanitize_name(nc.name) + "_seed" + str(int(seed)) + ".csv"
            write_run_csv(os.path.join(spec.out_dir, fname), rec)
            ro = RunOutput(name=nc.name, seed=int(seed), csv_path=fname, status=rec.status,
                           final_loss=rec.rows[-1].loss if rec.rows else 0.0,
                           final_grad_norm=rec.rows[-1].grad_norm if rec.rows else 0.0, rows=len(rec.rows),
                           steps=int(rec.steps_taken))
            result.runs.append(ro)
            result.records.append(rec)
    manifest = experiment_to_json(spec)
    manifest["runs"] = [{"name": ro.name, "seed": ro.seed, "csv": ro.csv_path, "status": ro.status, "rows": ro.rows,
                         "steps": ro.steps, "final_loss": ro.final_loss, "final_grad_norm": ro.final_grad_norm}
                        for ro in result.runs]
    mpath = os.path.join(spec.out_dir, "manifest.json")
    _write_text_atomic(mpath, dump_json(manifest) + "\n")
    result.manifest_path = mpath
    return result


# ---------------------------------------------------------------- conditioning sweep (harness.cpp:449-539)
@dataclass
class SweepRow:
    kappa: float = 1.0
    algorithm: str = ""
    bits: int = 0  # 0 for full precision
    alpha: float = 0.0
    mu: float = 0.0
    grad_norm: float = 0.0
    status: str = ""


@dataclass
class SweepResult:
    rows: List[SweepRow] = field(default_factory=list)
    device_ms: float = 0.0  # K5 time of the batched HALP grids (not in the reference's struct)


def sweep_alphas() -> List[float]:
    """half-decade step sizes 1e-10 .. 1e-2 (harness.cpp:461-465)"""
    return [math.pow(10.0, -10.0 + 0.5 * i) for i in range(17)]


def sweep_mus() -> List[float]:
    """13 log-spaced scales 0.5 .. 2000 (harness.cpp:466-470)"""
    return [math.exp(math.log(0.5) + i * (math.log(2000.0) - math.log(0.5)) / 12.0) for i in range(13)]


def conditioning_sweep(kappas, bit_widths, inner_steps: int, epochs: int, seed: int) -> SweepResult:
    """For each condition number: tune full-precision SVRG over the step sizes
    and HALP over (step size, scale) at each width on make_conditioned_regression
    (kappa, seed), and report each winner's final gradient norm.  Every HALP
    grid (17 x 13 runs) is ONE K5 launch over the shared 1000 x 64 dataset;
    the SVRG grid runs its 17 points through run_prepared on K1/K3."""
    kappas = list(kappas)
    if not kappas:
        raise InvalidInputError("sweep: need at least one kappa")
    if inner_steps < 1 or epochs < 1:
        raise InvalidInputError("sweep: inner_steps and epochs must be >= 1")
    alphas, mus = sweep_alphas(), sweep_mus()
    res = SweepResult()
    for kappa in kappas:
        ds = make_conditioned_regression(float(kappa), seed)
        obj = Objective(ds, LossFamily.Squared, 0.0)
        base = OptimizerConfig(epochs=epochs, inner_steps=inner_steps, seed=seed)
        svrg = copy.deepcopy(base)
        svrg.algorithm = Algorithm.Svrg
        g = grid_search(obj, svrg, [GridAxis("alpha", alphas)], [seed], "grad_norm", seed)
        won = g.points[g.best_index]
        res.rows.append(SweepRow(float(kappa), "svrg", 0, won.params["alpha"], 0.0, won.mean_metric, won.status))
        for bits in bit_widths:
            halp = copy.deepcopy(base)
            halp.algorithm = Algorithm.Halp
            halp.bits = int(bits)
            halp.mu = 1.0
            g = grid_search(obj, halp, [GridAxis("alpha", alphas), GridAxis("mu", mus)], [seed], "grad_norm", seed)
            res.device_ms += g.device_ms
            won = g.points[g.best_index]
            res.rows.append(SweepRow(float(kappa), "halp", int(bits), won.params["alpha"], won.params["mu"],
                                     won.mean_metric, won.status))
    return res


def write_sweep_csv(path: str, res: SweepResult) -> None:
    """harness.cpp:520-539"""
    s = "kappa,algorithm,bits,alpha,mu,grad_norm,status\n"
    for r in res.rows:
        s += ",".join([format_double(r.kappa), r.algorithm, str(int(r.bits)), format_double(r.alpha),
                       format_double(r.mu), format_double(r.grad_norm), r.status]) + "\n"
    _write_text_atomic(path, s)
