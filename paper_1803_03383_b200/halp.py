"""lpopt-compatible host API over the B200 C ABI.

Mirrors the reference's solver interface for the HALP path so that callers
and tests read like the reference's own (proj/include/lpopt/*.hpp):

  reference (C++)                              here
  -------------------------------------------  ------------------------------------
  lpopt::LossFamily {Squared, Softmax}          LossFamily.Squared / .Softmax
  lpopt::Dataset {X, targets, labels, C}        Dataset(X, targets=, labels=, num_classes=)
  lpopt::Objective(ds, loss, l2)                Objective(ds, loss, l2, device=0)
    .full_gradient(w) / .loss(w)                  .full_gradient(w) / .loss(w)  (one fused pass)
  lpopt::OptimizerConfig                        OptimizerConfig (same fields and defaults)
  lpopt::MetricRow / RunRecord                  MetricRow / RunRecord
  lpopt::run_halp(obj, cfg)                     run_halp(obj, cfg)
  lpopt::run(obj, cfg) (Halp branch)            run(obj, cfg)
  lpopt::run_prepared (harness.cpp:296-312)     run_prepared(obj, cfg)
  InvalidInputError / DivergenceError           InvalidInputError / DivergenceError(.partial)

X may be a numpy array (float64 / float32 / bf16 bits as uint16) on the
host, or a CUDA torch tensor (float64 / float32 / bfloat16) already in HBM.
Every computation runs in libhalp_b200.so on the GPU; there is no CPU path.
"""
from __future__ import annotations

import ctypes as C
import enum
import math
from dataclasses import dataclass, field
from typing import List, Optional

import numpy as np

from . import _capi as A


class Error(RuntimeError):
    """lpopt::Error (errors.hpp:8-10)."""


class InvalidInputError(Error):
    """lpopt::InvalidInputError (errors.hpp:13-15)."""


class UnsupportedError(Error):
    """Shape or algorithm outside the B200 hot path."""


class HalpCudaError(Error):
    pass


class LossFamily(enum.IntEnum):
    Squared = 0
    Softmax = 1


class Algorithm(enum.IntEnum):
    Sgd = 0
    Svrg = 1
    LpSgd = 2
    LpSvrg = 3
    Halp = 4
    LmHalp = 5


class EpochOption(enum.IntEnum):
    LastIterate = 0
    SampledIterate = 1


@dataclass
class MetricRow:
    pass_: float = 0.0
    seconds: float = 0.0
    loss: float = 0.0
    grad_norm: float = 0.0
    delta: float = 0.0
    iterate_hash: int = 0
    delta_inner: float = 0.0
    delta_aux: float = 0.0


@dataclass
class RunRecord:
    rows: List[MetricRow] = field(default_factory=list)
    final_iterate: Optional[np.ndarray] = None
    status: str = "ok"
    inner_fp_vector_ops: int = 0
    inner_lp_vector_ops: int = 0
    steps_taken: int = 0


class DivergenceError(Error):
    """lpopt::DivergenceError (optimizers.hpp:71-75): carries the partial record."""

    def __init__(self, msg: str, partial: RunRecord):
        super().__init__(msg)
        self.partial = partial


_STATUS = {0: "ok", 1: "converged", 2: "diverged"}


def _raise(rc: int, partial: Optional[RunRecord] = None):
    msg = A.last_error()
    if rc == A.HALP_INVALID_INPUT:
        raise InvalidInputError(msg)
    if rc == A.HALP_DIVERGED:
        raise DivergenceError(msg, partial)
    if rc == A.HALP_UNSUPPORTED:
        raise UnsupportedError(msg)
    if rc in (A.HALP_CUDA_ERROR, A.HALP_NCCL_ERROR):
        raise HalpCudaError(msg)
    raise Error(f"halp rc={rc}: {msg}")


@dataclass
class QuantizedExamples:
    """lpopt::QuantizedExamples (objectives.hpp): the rows of X quantized once
    for LM-HALP -- int64 codes [n][d] at one scale `delta` and width `bits`,
    drawn with `seed` on RNG stream 2 (objectives.cpp:110-133)."""

    codes: np.ndarray
    delta: float
    bits: int
    seed: int = 0


@dataclass
class Dataset:
    """lpopt::Dataset (objectives.hpp:23-33); X row-major n x d."""

    X: object
    targets: Optional[object] = None
    labels: Optional[object] = None
    num_classes: int = 0
    quantized: Optional[QuantizedExamples] = None

    def n(self) -> int:
        return int(self.X.shape[0])

    def dim(self) -> int:
        return int(self.X.shape[1])

    def is_classification(self) -> bool:
        return self.num_classes > 0


def _is_torch_cuda(a) -> bool:
    return hasattr(a, "is_cuda") and bool(a.is_cuda)


def _x_dtype(X) -> int:
    if _is_torch_cuda(X):
        import torch

        return {torch.float64: A.F64, torch.float32: A.F32, torch.bfloat16: A.BF16}[X.dtype]
    return {np.dtype(np.float64): A.F64, np.dtype(np.float32): A.F32, np.dtype(np.uint16): A.BF16}[X.dtype]


class Objective:
    """lpopt::Objective (objectives.hpp:59-91) backed by a device problem.

    world_size / rank / nccl_id: multi-GPU problem (row-sharded full gradient,
    one NCCL all-gather per epoch).  collective=True runs that NCCL route even
    at world_size 1 (nccl_id required), so it can be exercised on one GPU;
    collective="host" leaves the exchange to the caller (rank_partial /
    finalize_gathered: the rank plumbing of G ranks checked on one GPU)."""

    def __init__(self, ds: Dataset, loss: LossFamily = LossFamily.Squared, l2: float = 0.0, device: int = 0,
                 world_size: int = 1, rank: int = 0, nccl_id: Optional[bytes] = None, collective=False):
        self.ds = ds
        self._loss = LossFamily(loss)
        self._l2 = float(l2)
        self.device = device
        self._keep = []
        X = ds.X
        dev = _is_torch_cuda(X)
        if dev:
            X = X.contiguous()
            xptr = X.data_ptr()
        else:
            X = np.ascontiguousarray(X)
            xptr = X.ctypes.data
        self._keep.append(X)
        dtype = _x_dtype(X)
        yptr = lptr = None
        C_ = 0
        if self._loss == LossFamily.Squared:
            if ds.targets is None:
                raise InvalidInputError("Objective: squared loss needs one target per row")
            y = ds.targets
            if dev:
                import torch

                y = torch.as_tensor(y, dtype=torch.float64, device=X.device).contiguous()
                yptr = y.data_ptr()
            else:
                y = np.ascontiguousarray(y, dtype=np.float64)
                if y.shape[0] != X.shape[0]:
                    raise InvalidInputError("Objective: squared loss needs one target per row")
                yptr = y.ctypes.data
            self._keep.append(y)
        else:
            if ds.labels is None or ds.num_classes < 2:
                raise InvalidInputError("Objective: softmax loss needs labels and classes")
            lab = ds.labels
            if dev:
                import torch

                lab = torch.as_tensor(lab, dtype=torch.int32, device=X.device).contiguous()
                lptr = lab.data_ptr()
            else:
                lab = np.ascontiguousarray(lab, dtype=np.int32)
                lptr = lab.ctypes.data
            self._keep.append(lab)
            C_ = int(ds.num_classes)
        if dev:
            # HALP_MEM_DEVICE readiness contract (halp.h): the library reads X / y /
            # labels on its own stream, so whatever produced them (and the
            # conversions above) must have finished
            import torch

            torch.cuda.current_stream(X.device).synchronize()
        idbuf = None
        if nccl_id is not None:
            idbuf = C.create_string_buffer(bytes(nccl_id), 128)
        qptr, qbits, qdelta = None, 0, 0.0
        if ds.quantized is not None:
            qc = np.ascontiguousarray(ds.quantized.codes, dtype=np.int64)
            if qc.shape != (int(X.shape[0]), int(X.shape[1])):
                raise InvalidInputError("lm_halp: quantized rows do not match the dataset shape")
            self._keep.append(qc)
            qptr, qbits, qdelta = qc.ctypes.data, int(ds.quantized.bits), float(ds.quantized.delta)
        desc = A.ProblemDesc(xptr, dtype, A.MEM_DEVICE if dev else A.MEM_HOST, int(X.shape[0]), int(X.shape[1]),
                             int(self._loss), C_, yptr, lptr, self._l2, device, world_size, rank,
                             C.cast(idbuf, C.c_void_p) if idbuf is not None else None,
                             2 if collective == "host" else 1 if collective else 0, qptr, qbits, qdelta)
        h = C.c_void_p()
        rc = A.lib().halp_problem_create(C.byref(desc), C.byref(h))
        if rc:
            _raise(rc)
        self._h = h
        self._n = int(X.shape[0])
        self._d = int(X.shape[1])
        self._C = C_ if C_ else 1

    def __del__(self):
        h = getattr(self, "_h", None)
        if h:
            try:
                A.lib().halp_problem_destroy(h)
            except Exception:  # interpreter shutdown: the module globals may be gone
                pass
            self._h = None

    # ---- lpopt::Objective accessors ----
    def num_components(self) -> int:
        return self._n

    def feature_dim(self) -> int:
        return self._d

    def num_outputs(self) -> int:
        return self._C

    def dim(self) -> int:
        return self._d * self._C

    def loss_family(self) -> LossFamily:
        return self._loss

    def l2(self) -> float:
        return self._l2

    def dataset(self) -> Dataset:
        return self.ds

    def _fullpass(self, w):
        w = np.ascontiguousarray(w, dtype=np.float64)
        if w.size != self.dim():
            raise InvalidInputError("full_gradient: parameter length mismatch")
        g = np.empty(self.dim(), dtype=np.float64)
        loss = C.c_double()
        rc = A.lib().halp_full_gradient(self._h, w.ctypes.data, g.ctypes.data, C.byref(loss))
        if rc:
            _raise(rc)
        return g, loss.value

    def full_gradient(self, w, num_threads: int = 1) -> np.ndarray:
        """objectives.cpp:258-311; num_threads is accepted for API parity (the
        device result is independent of it, like the reference's)."""
        if num_threads < 1:
            raise InvalidInputError("full_gradient: num_threads must be >= 1")
        return self._fullpass(w)[0]

    def loss(self, w) -> float:
        """objectives.cpp:193-223 (computed in the same fused device pass)."""
        if np.asarray(w).size != self.dim():
            raise InvalidInputError("loss: parameter length mismatch")
        return self._fullpass(w)[1]

    def rank_partial(self, w) -> np.ndarray:
        """this rank's subtree root of the sharded full gradient (D+1: gradient sums, loss sum)"""
        w = np.ascontiguousarray(w, dtype=np.float64)
        out = np.empty(self.dim() + 1, dtype=np.float64)
        rc = A.lib().halp_rank_partial(self._h, w.ctypes.data, out.ctypes.data)
        if rc:
            _raise(rc)
        return out

    def finalize_gathered(self, w, gathered):
        """(g, loss) from the all ranks' roots [world][D+1] (the exchange step's consumer)"""
        w = np.ascontiguousarray(w, dtype=np.float64)
        gat = np.ascontiguousarray(gathered, dtype=np.float64)
        g = np.empty(self.dim(), dtype=np.float64)
        loss = C.c_double()
        rc = A.lib().halp_finalize_gathered(self._h, w.ctypes.data, gat.ctypes.data, g.ctypes.data, C.byref(loss))
        if rc:
            _raise(rc)
        return g, loss.value

    def plan(self) -> dict:
        pl = A.Plan()
        rc = A.lib().halp_problem_plan(self._h, C.byref(pl))
        if rc:
            _raise(rc)
        return {k: getattr(pl, k) for k, _ in A.Plan._fields_}

    def oracle_plan(self) -> dict:
        p = self.plan()
        return {k: p[k] for k in ("fg_threads", "fg_vec", "fg_splits", "in_ctas", "in_threads", "in_per", "in_levels")}

    def timing(self) -> dict:
        t = A.Timing()
        rc = A.lib().halp_last_timing(self._h, C.byref(t))
        if rc:
            _raise(rc)
        return {k: getattr(t, k) for k, _ in A.Timing._fields_}

    def bench_full_gradient(self, reps: int = 10) -> float:
        ms = C.c_double()
        rc = A.lib().halp_bench_full_gradient(self._h, reps, C.byref(ms))
        if rc:
            _raise(rc)
        return ms.value


@dataclass
class OptimizerConfig:
    """lpopt::OptimizerConfig (optimizers.hpp:31-47), same defaults."""

    algorithm: Algorithm = Algorithm.Svrg
    alpha: float = 1e-3
    epochs: int = 1
    inner_steps: int = 0
    bits: int = 8
    delta: float = 0.0
    mu: float = 0.0
    option: EpochOption = EpochOption.LastIterate
    full_grad_period: int = 2
    seed: int = 0
    metric_every_passes: float = 0.0
    delta_min: float = 1e-300
    divergence_limit: float = 1e12
    lm_bypass_aux_quant: bool = False
    init: Optional[np.ndarray] = None


def _to_c_config(cfg: OptimizerConfig, keep: list) -> A.Config:
    init = None
    if cfg.init is not None and np.asarray(cfg.init).size:
        init = np.ascontiguousarray(cfg.init, dtype=np.float64)
        keep.append(init)
    return A.Config(float(cfg.alpha), int(cfg.epochs), int(cfg.inner_steps), int(cfg.bits), float(cfg.mu),
                    int(cfg.option), int(cfg.full_grad_period), int(cfg.seed) & (2**64 - 1),
                    float(cfg.metric_every_passes), float(cfg.delta_min), float(cfg.divergence_limit),
                    init.ctypes.data if init is not None else None, float(cfg.delta), int(cfg.algorithm))


def _record(rec: A.Record, rows, fin: np.ndarray) -> RunRecord:
    out = RunRecord()
    out.rows = [MetricRow(r.pass_, r.seconds, r.loss, r.grad_norm, r.delta, r.iterate_hash, r.delta_inner, r.delta_aux)
                for r in rows[: rec.rows_n]]
    out.final_iterate = fin
    out.status = _STATUS[rec.status]
    out.inner_fp_vector_ops = rec.inner_fp_vector_ops
    out.inner_lp_vector_ops = rec.inner_lp_vector_ops
    out.steps_taken = rec.steps_taken
    return out


def resolve_inner_steps(cfg: OptimizerConfig, n: int) -> int:
    """optimizers.cpp:209-216"""
    t = cfg.inner_steps if cfg.inner_steps > 0 else cfg.full_grad_period * n
    if t < 1:
        raise InvalidInputError("optimizer: epoch length must be >= 1")
    return t


def hash_vector(v) -> int:
    """optimizers.cpp:218-227 (FNV-1a over the double bytes)."""
    h = 1469598103934665603
    for b in np.ascontiguousarray(v, dtype=np.float64).tobytes():
        h ^= b
        h = (h * 1099511628211) & 0xFFFFFFFFFFFFFFFF
    return h


def run_halp(obj: Objective, cfg: OptimizerConfig, trace: Optional[np.ndarray] = None) -> RunRecord:
    """lpopt::run_halp (optimizers.cpp:387-459) on the B200.  `trace`, an
    int64 array, receives the z codes of every inner step (test hook)."""
    return _run_algo(obj, cfg, Algorithm.Halp, trace)


def run_svrg(obj: Objective, cfg: OptimizerConfig) -> RunRecord:
    """lpopt::run_svrg (optimizers.cpp:258-296) on the same kernels: K1 at the
    snapshot, K3 in full precision (z holds the fp64 iterate, no rounding)."""
    return _run_algo(obj, cfg, Algorithm.Svrg, None)


def run_lp_svrg(obj: Objective, cfg: OptimizerConfig, trace: Optional[np.ndarray] = None) -> RunRecord:
    """lpopt::run_lp_svrg (optimizers.cpp:336-385): K3 with the iterate itself
    quantized at the fixed scale cfg.delta (codes traced like HALP's z)."""
    return _run_algo(obj, cfg, Algorithm.LpSvrg, trace)


def run_sgd(obj: Objective, cfg: OptimizerConfig) -> RunRecord:
    """lpopt::run_sgd (optimizers.cpp:229-256): K3 with the fp64 iterate and
    u = w - alpha*g (no snapshot gradient); K1 only for the boundary rows."""
    return _run_algo(obj, cfg, Algorithm.Sgd, None)


def run_lp_sgd(obj: Objective, cfg: OptimizerConfig, trace: Optional[np.ndarray] = None) -> RunRecord:
    """lpopt::run_lp_sgd (optimizers.cpp:297-334): the iterate quantized at the
    fixed scale cfg.delta after every step."""
    return _run_algo(obj, cfg, Algorithm.LpSgd, trace)


def run_lm_halp(obj: Objective, cfg: OptimizerConfig, trace: Optional[np.ndarray] = None) -> RunRecord:
    """lpopt::run_lm_halp (optimizers.cpp:461-627): HALP's linear-model form
    with an integer-only inner loop over the dataset's quantized rows
    (obj.dataset().quantized, see quantize_dataset) -- K7 epoch stats + K8
    integer inner loop (k_lm.cu).  `trace` receives the z codes per step."""
    return _run_algo(obj, cfg, Algorithm.LmHalp, trace)


def data_scale(X, bits: int) -> float:
    """objectives.cpp:112-122: max|X| / (2^(bits-1) - 1), 1 for an all-zero X"""
    if bits < 2 or bits > 64:
        raise InvalidInputError("data_scale: bits must be in [2, 64]")
    X = np.asarray(X, dtype=np.float64)
    m = float(np.max(np.abs(X))) if X.size else 0.0
    if not math.isfinite(m):
        raise InvalidInputError("data_scale: matrix has non-finite entries")
    return 1.0 if m == 0.0 else m / (math.ldexp(1.0, bits - 1) - 1.0)


def quantize_dataset(ds: Dataset, bits: int, seed: int) -> None:
    """objectives.cpp:124-133: quantize every row of ds.X once (stream 2 of
    `seed`, row-major draws) and attach the codes as ds.quantized (host, the
    library's restatement of the reference's quantize_code)."""
    X = ds.X
    if _is_torch_cuda(X):
        X = X.double().cpu().numpy()
    elif np.asarray(X).dtype == np.uint16:  # bf16 bits
        X = (np.asarray(X, dtype=np.uint32) << 16).view(np.float32)
    X = np.ascontiguousarray(X, dtype=np.float64)
    data_scale(X, bits)  # the reference's checks and messages
    codes = np.empty(X.shape, dtype=np.int64)
    dl = C.c_double()
    rc = A.lib().halp_quantize_dataset(X.ctypes.data, X.shape[0], X.shape[1], bits, int(seed) & (2**64 - 1),
                                       codes.ctypes.data, C.byref(dl))
    if rc:
        raise InvalidInputError("quantize_dataset: invalid input")
    ds.quantized = QuantizedExamples(codes, dl.value, int(bits), int(seed))


def _run_algo(obj: Objective, cfg: OptimizerConfig, algo: Algorithm, trace) -> RunRecord:
    if cfg.init is not None and np.asarray(cfg.init).size not in (0, obj.dim()):
        raise InvalidInputError("optimizer: init length does not match objective")
    import copy

    cfg = copy.copy(cfg)
    cfg.algorithm = algo
    keep: list = []
    c = _to_c_config(cfg, keep)
    cap = max(cfg.epochs, 0) + 2
    if cfg.metric_every_passes <= 0:
        cap = max(cfg.epochs, 0) + 2
    rows = (A.Row * cap)()
    fin = np.zeros(obj.dim(), dtype=np.float64)
    rec = A.Record(rows, cap, 0, fin.ctypes.data, 0, 0, 0, 0)
    if trace is not None:
        assert trace.dtype == np.int64 and trace.flags.c_contiguous
        A.lib().halp_set_trace(obj._h, trace.ctypes.data, trace.size)
    try:
        rc = A.lib().halp_run(obj._h, C.byref(c), C.byref(rec))
    finally:
        if trace is not None:
            A.lib().halp_set_trace(obj._h, None, 0)
    if rc == A.HALP_DIVERGED:
        _raise(rc, _record(rec, rows, fin))
    if rc:
        _raise(rc)
    return _record(rec, rows, fin)


def run(obj: Objective, cfg: OptimizerConfig) -> RunRecord:
    """lpopt::run (optimizers.cpp:629-639): every algorithm of the reference
    runs on the B200 (LmHalp needs the dataset's quantized rows)."""
    fns = {Algorithm.Halp: run_halp, Algorithm.Svrg: run_svrg, Algorithm.LpSvrg: run_lp_svrg,
           Algorithm.Sgd: run_sgd, Algorithm.LpSgd: run_lp_sgd, Algorithm.LmHalp: run_lm_halp}
    if cfg.algorithm in fns:
        return fns[Algorithm(cfg.algorithm)](obj, cfg)
    raise UnsupportedError(f"algorithm {Algorithm(cfg.algorithm).name} is not on the B200 path")


def run_prepared(obj: Objective, cfg: OptimizerConfig, data_seed: int = 0) -> RunRecord:
    """harness.cpp:296-312: a diverged run is returned, not raised; LM-HALP on a
    dataset without codes of the config's width first quantizes a copy with
    data_seed."""
    try:
        if cfg.algorithm == Algorithm.LmHalp:
            q = obj.ds.quantized
            if q is None or q.bits != cfg.bits:
                import copy as _copy

                ds = _copy.copy(obj.ds)
                quantize_dataset(ds, cfg.bits, data_seed)
                prepared = Objective(ds, obj.loss_family(), obj.l2(), device=obj.device)
                return run(prepared, cfg)
        return run(obj, cfg)
    except DivergenceError as e:
        return e.partial


# ---------------------------------------------------------------- clipping variants
class ClipMode(enum.IntEnum):
    """lpopt::ClipMode (optimizers.hpp:23): how the 16-bit variant of a narrow
    bit-centered run keeps its dynamic range."""

    Scale = 0
    Clip = 1


def clipping_variant_config(base: OptimizerConfig, mode: ClipMode) -> OptimizerConfig:
    """optimizers.cpp:641-656: the same run at 16 bits; ClipMode.Scale also
    rescales mu so the representable range (mu * span) is unchanged."""
    import copy

    if base.algorithm not in (Algorithm.Halp, Algorithm.LmHalp):
        raise InvalidInputError("clipping variant applies to bit-centered runs only")
    if base.bits >= 16:
        raise InvalidInputError("clipping variant derives a 16-bit run; base must be narrower")
    out = copy.deepcopy(base)
    out.bits = 16
    if mode == ClipMode.Scale:
        span_base = math.ldexp(1.0, base.bits - 1) - 1.0
        span16 = math.ldexp(1.0, 15) - 1.0
        out.mu = base.mu * span_base / span16
    return out


def run_clipping_variant(obj: Objective, base: OptimizerConfig, mode: ClipMode) -> RunRecord:
    """optimizers.cpp:658-661"""
    return run(obj, clipping_variant_config(base, mode))


# ---------------------------------------------------------------- traces
def format_double(x: float) -> str:
    """lpopt::format_double (text.hpp:12-19): std::to_chars' shortest
    round-trip form -- the fewest significant digits that read back to x, in
    fixed or scientific notation, whichever is shorter (fixed on a tie);
    exponents carry a sign and at least two digits (printf's %e); integral
    values in fixed notation print their exact digits."""
    x = float(x)
    if math.isnan(x):
        return "-nan" if math.copysign(1.0, x) < 0 else "nan"
    if math.isinf(x):
        return "-inf" if x < 0 else "inf"
    sign = "-" if math.copysign(1.0, x) < 0 else ""
    if x == 0.0:
        return sign + "0"
    # shortest round-trip digits (Python's repr is shortest round-trip too)
    r = repr(abs(x))
    mant, _, ex = r.partition("e")
    e10 = int(ex) if ex else 0
    ip, _, fp = mant.partition(".")
    digits = (ip + fp).lstrip("0")
    # decimal exponent of the first significant digit
    if ip.strip("0"):
        point = len(ip.lstrip("0")) + e10  # digits before the decimal point
    else:
        point = -(len(fp) - len(fp.lstrip("0"))) + e10
    digits = digits.rstrip("0") or "0"
    n = len(digits)
    # scientific: d[.ddd]e+XX
    sci_exp = point - 1
    sci = digits[0] + ("." + digits[1:] if n > 1 else "") + ("e%+03d" % sci_exp)
    # fixed
    if point <= 0:
        fixed = "0." + "0" * (-point) + digits
    elif point >= n:
        fixed = str(int(abs(x)))  # an integer: to_chars prints its exact digits
    else:
        fixed = digits[:point] + "." + digits[point:]
    return sign + (fixed if len(fixed) <= len(sci) else sci)


def write_run_csv(path: str, rec: RunRecord) -> None:
    """lpopt::write_run_csv (harness.cpp:246-261): one row per MetricRow,
    `pass,seconds,loss,grad_norm,delta`, every number by format_double."""
    s = "pass,seconds,loss,grad_norm,delta\n"
    for r in rec.rows:
        s += ",".join(format_double(v) for v in (r.pass_, r.seconds, r.loss, r.grad_norm, r.delta)) + "\n"
    import os

    tmp = path + ".tmp"
    with open(tmp, "w", newline="") as f:  # write_text_atomic: write then rename
        f.write(s)
    os.replace(tmp, path)


# ---------------------------------------------------------------- grid search
@dataclass
class GridAxis:
    """lpopt::GridAxis (harness.hpp:92-95)."""

    param: str
    values: List[float]


@dataclass
class GridOutcome:
    """lpopt::GridOutcome (harness.hpp:97-102)."""

    params: dict = field(default_factory=dict)
    per_seed: List[float] = field(default_factory=list)  # +inf for diverged seeds
    mean_metric: float = 0.0
    status: str = "ok"


@dataclass
class GridResult:
    """lpopt::GridResult (harness.hpp:104-108)."""

    points: List[GridOutcome] = field(default_factory=list)
    best_index: int = 0
    best_config: Optional[OptimizerConfig] = None
    device_ms: float = 0.0  # K5 kernel time of a batched grid (not in the reference's struct)


def _apply_param(cfg: OptimizerConfig, param: str, v: float) -> None:
    """harness.cpp:45-61"""
    if param == "alpha":
        cfg.alpha = v
    elif param == "delta":
        cfg.delta = v
    elif param == "mu":
        cfg.mu = v
    elif param == "bits":
        cfg.bits = int(_llround(v))
    elif param == "epochs":
        cfg.epochs = int(_llround(v))
    elif param == "inner":
        cfg.inner_steps = int(_llround(v))
    else:
        raise InvalidInputError(f"grid: unknown parameter '{param}'")


def _llround(v: float) -> int:
    """std::llround: halves away from zero"""
    return int(math.floor(v + 0.5)) if v >= 0 else -int(math.floor(-v + 0.5))


def _final_metric(rec: RunRecord, metric: str) -> float:
    """harness.cpp:63-66"""
    if not rec.rows:
        return math.inf
    return rec.rows[-1].loss if metric == "loss" else rec.rows[-1].grad_norm


def _batchable(obj: Objective, cfgs) -> bool:
    return (obj.loss_family() == LossFamily.Squared and obj.dim() <= 256 and obj.ds.X is not None
            and all(c.algorithm == Algorithm.Halp for c in cfgs))


def grid_search(obj: Objective, base: OptimizerConfig, axes, seeds, metric: str = "grad_norm",
                data_seed: int = 0) -> GridResult:
    """lpopt::grid_search (harness.cpp:379-447): exhaustive Cartesian search,
    axes in name order with the listed value order (last axis fastest), the
    seed-mean of the final metric per point, diverged seeds count as +inf, and
    the first point reaching the minimum wins.  Every (point, seed) run is an
    independent run_prepared; on the B200 they all run at once -- one K5
    launch over the objective's dataset shared by every run (least squares,
    d <= 256) -- or one after another through run_prepared otherwise.  The
    records are the reference's per run (bit-identical to the oracle's MIRROR
    runs with the batch plan), so the outcome is."""
    if metric not in ("grad_norm", "loss"):
        raise InvalidInputError("grid: metric must be grad_norm or loss")
    seeds = [int(s) for s in seeds]
    if not seeds:
        raise InvalidInputError("grid: need at least one seed")
    axes = sorted((GridAxis(a.param, list(a.values)) for a in axes), key=lambda a: a.param)
    for i, a in enumerate(axes):
        if not a.values:
            raise InvalidInputError(f"grid: axis '{a.param}' has no values")
        if i > 0 and a.param == axes[i - 1].param:
            raise InvalidInputError(f"grid: duplicate axis '{a.param}'")
    # enumerate the points (odometer, last axis fastest) and their per-seed configs
    import copy
    import itertools

    points, cfgs = [], []
    for combo in itertools.product(*[a.values for a in axes]):
        cfg = copy.deepcopy(base)
        params = {}
        for a, v in zip(axes, combo):
            _apply_param(cfg, a.param, float(v))
            params[a.param] = float(v)
        points.append((params, cfg))
        for sd in seeds:
            c = copy.deepcopy(cfg)
            c.seed = sd
            cfgs.append(c)
    if _batchable(obj, cfgs):
        ds = obj.ds
        b = BatchProblems(ds.X, ds.targets, l2=obj.l2(), device=obj.device, nprob=len(cfgs))
        recs = b.run(cfgs)
        device_ms = b.device_ms
    else:
        recs = [run_prepared(obj, c, data_seed) for c in cfgs]
        device_ms = 0.0
    res = GridResult(device_ms=device_ms)
    best = math.inf
    for pi, (params, cfg) in enumerate(points):
        out = GridOutcome(params=params, status="ok")
        total = 0.0
        for si in range(len(seeds)):
            rec = recs[pi * len(seeds) + si]
            m = _final_metric(rec, metric)
            if rec.status == "diverged" or not math.isfinite(m):
                m = math.inf
                out.status = "diverged"
            out.per_seed.append(m)
            total += m
        out.mean_metric = total / float(len(seeds))
        if pi == 0 or out.mean_metric < best:
            best = out.mean_metric
            res.best_index = pi
            res.best_config = copy.deepcopy(cfg)
            res.best_config.seed = base.seed
        res.points.append(out)
    return res


def halp_scale(grad_norm: float, mu: float, bits: int) -> float:
    """theory.cpp:93-102"""
    if not (math.isfinite(grad_norm) and grad_norm >= 0.0):
        raise InvalidInputError("grad_norm must be finite and nonnegative")
    if not (math.isfinite(mu) and mu > 0.0):
        raise InvalidInputError("mu must be positive and finite")
    if bits < 2 or bits > 64:
        raise InvalidInputError("bits must be in [2, 64]")
    return grad_norm / (mu * (math.ldexp(1.0, bits - 1) - 1.0))


class BatchProblems:
    """Many independent least-squares problems of one shape (BASELINE C5 and the
    reference's grid / conditioning sweeps, harness.cpp:379-518) solved by the
    batched kernel K5: one CTA per problem runs the whole run_halp.

    X: [nprob, n, d] (numpy float64/float32/bf16-as-uint16, or a CUDA tensor),
    y: [nprob, n]; or X: [n, d], y: [n] with `nprob` given -- one dataset
    shared by every problem (each with its own config: grid searches).
    run(cfgs) returns one RunRecord per problem; a problem that diverges gets
    status "diverged" and its partial record (run_prepared semantics,
    harness.cpp:309-311) instead of an exception."""

    def __init__(self, X, y, l2: float = 0.0, device: int = 0, nprob: Optional[int] = None):
        dev = _is_torch_cuda(X)
        if dev:
            import torch

            X = X.contiguous()
            y = torch.as_tensor(y, dtype=torch.float64, device=X.device).contiguous()
            xptr, yptr = X.data_ptr(), y.data_ptr()
            torch.cuda.current_stream(X.device).synchronize()  # readiness contract (halp.h)
        else:
            X = np.ascontiguousarray(X)
            y = np.ascontiguousarray(y, dtype=np.float64)
            xptr, yptr = X.ctypes.data, y.ctypes.data
        self._keep = [X, y]
        shared = len(X.shape) == 2
        if shared:
            if nprob is None or nprob < 1:
                raise InvalidInputError("BatchProblems: a shared dataset needs nprob >= 1")
            n, d = (int(v) for v in X.shape)
        else:
            nprob, n, d = (int(v) for v in X.shape)
        if tuple(int(v) for v in y.shape) != ((n,) if shared else (nprob, n)):
            raise InvalidInputError("Objective: squared loss needs one target per row")
        self.nprob, self.n, self.d, self.shared = int(nprob), n, d, shared
        desc = A.BatchDesc(xptr, _x_dtype(X), A.MEM_DEVICE if dev else A.MEM_HOST, n, d, self.nprob, yptr, float(l2),
                           device, 1 if shared else 0)
        h = C.c_void_p()
        rc = A.lib().halp_batch_create(C.byref(desc), C.byref(h))
        if rc:
            _raise(rc)
        self._h = h
        self.device_ms = 0.0

    def __del__(self):
        h = getattr(self, "_h", None)
        if h:
            try:
                A.lib().halp_batch_destroy(h)
            except Exception:
                pass
            self._h = None

    def plan(self) -> dict:
        pl = A.Plan()
        rc = A.lib().halp_batch_plan(self._h, C.byref(pl))
        if rc:
            _raise(rc)
        return {k: getattr(pl, k) for k, _ in A.Plan._fields_}

    def oracle_plan(self) -> dict:
        p = self.plan()
        return {k: p[k] for k in ("fg_threads", "fg_vec", "fg_splits", "in_ctas", "in_threads", "in_per", "in_levels")}

    def run(self, cfgs) -> list:
        if len(cfgs) != self.nprob:
            raise InvalidInputError("halp_batch_run: one config per problem")
        keep: list = []
        carr = (A.Config * self.nprob)(*[_to_c_config(c, keep) for c in cfgs])
        caps = [max(c.epochs, 0) + 2 for c in cfgs]
        rows = [(A.Row * cap)() for cap in caps]
        fins = [np.zeros(self.d, dtype=np.float64) for _ in cfgs]
        recs = (A.Record * self.nprob)(*[A.Record(rows[i], caps[i], 0, fins[i].ctypes.data, 0, 0, 0, 0)
                                         for i in range(self.nprob)])
        ms = C.c_double()
        rc = A.lib().halp_batch_run(self._h, carr, recs, C.byref(ms))
        if rc:
            _raise(rc)
        self.device_ms = ms.value
        return [_record(recs[i], rows[i], fins[i]) for i in range(self.nprob)]


def generate(kind: str, n: int, d: int, *, num_classes: int = 0, dtype: str = "f32", noise_sd: float = 0.0,
             x_scale: float = 1.0, density: float = 1.0, seed: int = 0, device: int = 0):
    """K6 device generator for the BASELINE synthetic configs; returns torch
    CUDA tensors (X, y) for 'regression' or (X, labels) for 'softmax' /
    'logistic'."""
    import torch

    kinds = {"regression": 0, "softmax": 1, "logistic": 2}
    tdt = {"f64": torch.float64, "f32": torch.float32, "bf16": torch.bfloat16}[dtype]
    cdt = {"f64": A.F64, "f32": A.F32, "bf16": A.BF16}[dtype]
    dev = torch.device("cuda", device)
    X = torch.empty((n, d), dtype=tdt, device=dev)
    y = lab = None
    if kinds[kind] == 0:
        y = torch.empty(n, dtype=torch.float64, device=dev)
    else:
        lab = torch.empty(n, dtype=torch.int32, device=dev)
    desc = A.DatagenDesc(kinds[kind], n, d, num_classes, cdt, noise_sd, x_scale, density, seed)
    rc = A.lib().halp_datagen(C.byref(desc), device, X.data_ptr(), y.data_ptr() if y is not None else None,
                              lab.data_ptr() if lab is not None else None)
    if rc:
        _raise(rc)
    return (X, y) if y is not None else (X, lab)


def shard_plan(n: int, d: int, C_: int, dtype: int, world: int, rank: int) -> dict:
    """Host-side row/split plan of the multi-GPU full gradient (CPU-callable)."""
    vals = [C.c_int64() for _ in range(5)]
    rc = A.lib().halp_shard_plan(n, d, C_, dtype, world, rank, *[C.byref(v) for v in vals])
    if rc:
        _raise(rc)
    return dict(zip(("split_begin", "split_end", "splits", "row_begin", "row_end"), [v.value for v in vals]))


def plan_for(n: int, d: int, C_: int = 1, dtype: str = "f64", world: int = 1, rank: int = 0) -> dict:
    """Kernel plan for a problem shape, without a GPU (used by the CPU tests
    to put the oracle's MIRROR mode into the device's reduction order)."""
    pl = A.Plan()
    rc = A.lib().halp_plan_for(n, d, C_, {"f64": A.F64, "f32": A.F32, "bf16": A.BF16}[dtype], world, rank,
                               C.byref(pl))
    if rc:
        _raise(rc)
    return {k: getattr(pl, k) for k, _ in A.Plan._fields_}


def oracle_plan_for(n: int, d: int, C_: int = 1, dtype: str = "f64") -> dict:
    p = plan_for(n, d, C_, dtype)
    return {k: p[k] for k in ("fg_threads", "fg_vec", "fg_splits", "in_ctas", "in_threads", "in_per", "in_levels")}


def rng_state_after(seed: int, stream: int, count: int) -> int:
    return A.lib().halp_rng_state_after(seed, stream, count)
