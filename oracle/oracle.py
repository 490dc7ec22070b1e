"""ctypes wrapper of the CPU oracle (oracle/liboracle.so).

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and
bench.py's cpu_baseline / --impl reference legs.  The product package
(paper_1803_03383_b200) never imports this module.

The oracle restates the reference lpopt HALP path (see halp_oracle.h for
the reference file:line map).  ``plan=None`` selects REF order (pinned by
the reference's golden traces); an ``OraclePlan`` selects MIRROR order,
the exact operation order of the B200 kernels.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass, field
from typing import Optional

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "liboracle.so")

F64, F32, BF16 = 0, 1, 2
SQUARED, SOFTMAX = 0, 1
STATUS = {0: "ok", 1: "converged", 2: "diverged"}


def build(force: bool = False) -> str:
    if force or not os.path.exists(LIB_PATH) or os.path.getmtime(LIB_PATH) < max(
        os.path.getmtime(os.path.join(HERE, f)) for f in ("halp_oracle.c", "halp_oracle.h", "datagen.c")
    ):
        subprocess.run(["make", "-s", "-C", HERE, "-B" if force else "all"], check=True)
    return LIB_PATH


class _Objective(C.Structure):
    _fields_ = [
        ("X", C.c_void_p), ("dtype", C.c_int), ("n", C.c_int64), ("d", C.c_int), ("C", C.c_int),
        ("loss", C.c_int), ("y", C.c_void_p), ("labels", C.c_void_p), ("l2", C.c_double),
    ]


class _Plan(C.Structure):
    _fields_ = [(k, C.c_int) for k in ("fg_threads", "fg_vec", "fg_splits", "in_ctas", "in_threads", "in_per",
                                       "in_levels")]


class _Config(C.Structure):
    _fields_ = [
        ("alpha", C.c_double), ("epochs", C.c_int32), ("inner_steps", C.c_int64), ("bits", C.c_int32),
        ("mu", C.c_double), ("option", C.c_int32), ("full_grad_period", C.c_int32), ("seed", C.c_uint64),
        ("metric_every_passes", C.c_double), ("delta_min", C.c_double), ("divergence_limit", C.c_double),
        ("init", C.c_void_p), ("delta", C.c_double), ("algorithm", C.c_int32),
    ]


class _Row(C.Structure):
    _fields_ = [(k, C.c_double) for k in ("pass_", "seconds", "loss", "grad_norm", "delta")] + [
        ("iterate_hash", C.c_uint64), ("delta_inner", C.c_double), ("delta_aux", C.c_double)
    ]


class _Record(C.Structure):
    _fields_ = [
        ("rows", C.POINTER(_Row)), ("rows_cap", C.c_int32), ("rows_n", C.c_int32),
        ("final_iterate", C.c_void_p), ("status", C.c_int32), ("steps_taken", C.c_int64),
        ("inner_fp_vector_ops", C.c_uint64), ("trace_codes", C.c_void_p), ("trace_cap", C.c_int64),
        ("fullgrad_seconds", C.c_double), ("inner_seconds", C.c_double), ("fullgrad_threads", C.c_int),
        ("step_hash", C.c_void_p), ("step_hash_cap", C.c_int64), ("inner_lp_vector_ops", C.c_uint64),
    ]


class _Quantized(C.Structure):
    _fields_ = [("codes", C.c_void_p), ("delta", C.c_double), ("bits", C.c_int)]


class _Datagen(C.Structure):
    _fields_ = [("kind", C.c_int32), ("n", C.c_int64), ("d", C.c_int32), ("num_classes", C.c_int32),
                ("dtype", C.c_int32), ("noise_sd", C.c_double), ("x_scale", C.c_double), ("density", C.c_double),
                ("seed", C.c_uint64)]


_lib = None


def lib():
    global _lib
    if _lib is None:
        build()
        L = C.CDLL(LIB_PATH)
        L.oq_rng_init.argtypes = [C.c_void_p, C.c_uint64, C.c_uint64]
        L.oq_next_u64.restype = C.c_uint64
        L.oq_next_u64.argtypes = [C.c_void_p]
        L.oq_next_uniform.restype = C.c_double
        L.oq_next_uniform.argtypes = [C.c_void_p]
        L.oq_next_index.restype = C.c_uint64
        L.oq_next_index.argtypes = [C.c_void_p, C.c_uint64]
        L.oq_next_normal.restype = C.c_double
        L.oq_next_normal.argtypes = [C.c_void_p]
        L.oq_fill_u64.argtypes = [C.c_uint64, C.c_uint64, C.c_uint64, C.c_void_p, C.c_int64]
        L.oq_quantize_code.restype = C.c_int64
        L.oq_quantize_code.argtypes = [C.c_double, C.c_double, C.c_int, C.c_double, C.POINTER(C.c_int)]
        L.oq_halp_scale.restype = C.c_double
        L.oq_halp_scale.argtypes = [C.c_double, C.c_double, C.c_int]
        L.oq_make_regression.argtypes = [C.c_int64, C.c_int, C.c_double, C.c_uint64, C.c_void_p, C.c_void_p]
        L.oq_loss.argtypes = [C.POINTER(_Objective), C.c_void_p, C.POINTER(_Plan), C.POINTER(C.c_double)]
        L.oq_full_gradient.argtypes = [C.POINTER(_Objective), C.c_void_p, C.c_int, C.POINTER(_Plan), C.c_void_p]
        L.oq_component_gradient.argtypes = [C.POINTER(_Objective), C.c_int64, C.c_void_p, C.POINTER(_Plan), C.c_void_p]
        L.oq_run_halp.argtypes = [C.POINTER(_Objective), C.POINTER(_Config), C.POINTER(_Plan), C.POINTER(_Record)]
        L.oq_run.argtypes = [C.POINTER(_Objective), C.POINTER(_Config), C.POINTER(_Plan), C.POINTER(_Record)]
        L.oq_datagen.argtypes = [C.POINTER(_Datagen), C.c_int64, C.c_int64, C.c_int, C.c_void_p, C.c_void_p,
                                 C.c_void_p]
        L.oq_quantize_dataset.argtypes = [C.c_void_p, C.c_int64, C.c_int, C.c_int, C.c_uint64, C.c_void_p,
                                          C.POINTER(C.c_double)]
        L.oq_run_lm_halp.argtypes = [C.POINTER(_Objective), C.c_void_p, C.POINTER(_Config), C.POINTER(_Plan),
                                     C.POINTER(_Record)]
        L.oq_code_hash.restype = C.c_uint64
        L.oq_code_hash.argtypes = [C.c_void_p, C.c_int64]
        L.oq_hash_vector.restype = C.c_uint64
        L.oq_hash_vector.argtypes = [C.c_void_p, C.c_int64]
        L.oq_last_error.restype = C.c_char_p
        L.oq_mexp.restype = C.c_double
        L.oq_mexp.argtypes = [C.c_double]
        L.oq_mlog.restype = C.c_double
        L.oq_mlog.argtypes = [C.c_double]
        L.oq_split_subtree.argtypes = [C.POINTER(_Objective), C.c_void_p, C.POINTER(_Plan), C.c_int64, C.c_int64,
                                       C.c_void_p]
        L.oq_finalize.argtypes = [C.POINTER(_Objective), C.c_void_p, C.c_void_p, C.c_int, C.c_void_p,
                                  C.POINTER(C.c_double)]
        L.oq_resolve_inner_steps.restype = C.c_int64
        L.oq_resolve_inner_steps.argtypes = [C.POINTER(_Config), C.c_int64]
        _lib = L
    return _lib


class OracleError(RuntimeError):
    pass


class OracleInvalidInput(OracleError):
    pass


def _check(rc):
    if rc == 0:
        return
    msg = lib().oq_last_error().decode()
    if rc == 1:
        raise OracleInvalidInput(msg)
    raise OracleError(f"oracle rc={rc}: {msg}")


class QuantRng:
    """rng.hpp:27-64 (xorshift64*, splitmix-seeded)."""

    def __init__(self, seed: int, stream: int = 0):
        self._s = C.c_uint64(0)
        lib().oq_rng_init(C.byref(self._s), seed, stream)

    def next_u64(self) -> int:
        return lib().oq_next_u64(C.byref(self._s))

    def next_uniform(self) -> float:
        return lib().oq_next_uniform(C.byref(self._s))

    def next_index(self, n: int) -> int:
        return lib().oq_next_index(C.byref(self._s), n)

    def next_normal(self) -> float:
        return lib().oq_next_normal(C.byref(self._s))

    @property
    def state(self) -> int:
        return self._s.value


def fill_u64(seed: int, stream: int, skip: int, count: int) -> np.ndarray:
    out = np.empty(count, dtype=np.uint64)
    lib().oq_fill_u64(seed, stream, skip, out.ctypes.data, count)
    return out


def quantize_code(x: float, delta: float, bits: int, u: float) -> int:
    err = C.c_int(0)
    c = lib().oq_quantize_code(x, delta, bits, u, C.byref(err))
    if err.value:
        raise OracleInvalidInput("quantize: input must be finite")
    return c


def halp_scale(gn: float, mu: float, bits: int) -> float:
    return lib().oq_halp_scale(gn, mu, bits)


def make_regression(n: int, d: int, noise_sd: float, seed: int):
    X = np.empty((n, d), dtype=np.float64)
    y = np.empty(n, dtype=np.float64)
    _check(lib().oq_make_regression(n, d, noise_sd, seed, X.ctypes.data, y.ctypes.data))
    return X, y


@dataclass
class OracleObjective:
    """Mirror of lpopt::Objective (objectives.hpp:59-91).  X row-major:
    float64, float32, or bf16 given as a uint16 array of raw bits."""

    X: np.ndarray
    y: Optional[np.ndarray] = None
    labels: Optional[np.ndarray] = None
    num_classes: int = 0
    l2: float = 0.0

    def __post_init__(self):
        self.X = np.ascontiguousarray(self.X)
        if self.X.dtype == np.float64:
            self.dtype = F64
        elif self.X.dtype == np.float32:
            self.dtype = F32
        elif self.X.dtype == np.uint16:
            self.dtype = BF16
        else:
            raise TypeError(f"unsupported X dtype {self.X.dtype}")
        if self.labels is not None:
            self.labels = np.ascontiguousarray(self.labels, dtype=np.int32)
            self.loss = SOFTMAX
            self.C = int(self.num_classes)
        else:
            self.y = np.ascontiguousarray(self.y, dtype=np.float64)
            self.loss = SQUARED
            self.C = 1
        self.n, self.d = self.X.shape
        self._s = _Objective(
            self.X.ctypes.data, self.dtype, self.n, self.d, self.C, self.loss,
            self.y.ctypes.data if self.y is not None else None,
            self.labels.ctypes.data if self.labels is not None else None, float(self.l2),
        )

    @property
    def dim(self) -> int:
        return self.d * self.C

    def loss_value(self, w, plan=None) -> float:
        w = np.ascontiguousarray(w, dtype=np.float64)
        out = C.c_double()
        _check(lib().oq_loss(C.byref(self._s), w.ctypes.data, _plan(plan), C.byref(out)))
        return out.value

    def full_gradient(self, w, num_threads: int = 1, plan=None) -> np.ndarray:
        w = np.ascontiguousarray(w, dtype=np.float64)
        g = np.empty(self.dim, dtype=np.float64)
        _check(lib().oq_full_gradient(C.byref(self._s), w.ctypes.data, num_threads, _plan(plan), g.ctypes.data))
        return g

    def split_subtree(self, w, plan, s0: int, s1: int) -> np.ndarray:
        w = np.ascontiguousarray(w, dtype=np.float64)
        out = np.empty(self.dim + 1, dtype=np.float64)
        _check(lib().oq_split_subtree(C.byref(self._s), w.ctypes.data, _plan(plan), s0, s1, out.ctypes.data))
        return out

    def finalize(self, w, rank_sums: np.ndarray):
        w = np.ascontiguousarray(w, dtype=np.float64)
        rs = np.ascontiguousarray(rank_sums, dtype=np.float64)
        g = np.empty(self.dim, dtype=np.float64)
        loss = C.c_double()
        _check(lib().oq_finalize(C.byref(self._s), w.ctypes.data, rs.ctypes.data, rs.shape[0], g.ctypes.data,
                                 C.byref(loss)))
        return g, loss.value

    def component_gradient(self, i: int, w) -> np.ndarray:
        w = np.ascontiguousarray(w, dtype=np.float64)
        g = np.empty(self.dim, dtype=np.float64)
        _check(lib().oq_component_gradient(C.byref(self._s), i, w.ctypes.data, None, g.ctypes.data))
        return g


@dataclass
class OraclePlan:
    fg_threads: int = 256
    fg_vec: int = 4
    fg_splits: int = 1
    in_ctas: int = 1
    in_threads: int = 32
    in_per: int = 1
    in_levels: int = 1


def _plan(p):
    if p is None:
        return None
    if isinstance(p, dict):
        p = OraclePlan(**p)
    return C.byref(_Plan(p.fg_threads, p.fg_vec, p.fg_splits, p.in_ctas, p.in_threads, p.in_per, p.in_levels))


@dataclass
class OracleConfig:
    """lpopt::OptimizerConfig fields of the restated algorithms (optimizers.hpp:31-47);
    algorithm: 0 Sgd, 1 Svrg, 2 LpSgd, 3 LpSvrg, 4 Halp (run() dispatches, run_halp forces 4)."""

    alpha: float = 1e-3
    epochs: int = 1
    inner_steps: int = 0
    bits: int = 8
    mu: float = 0.0
    option: int = 0
    full_grad_period: int = 2
    seed: int = 0
    metric_every_passes: float = 0.0
    delta_min: float = 1e-300
    divergence_limit: float = 1e12
    init: Optional[np.ndarray] = None
    delta: float = 0.0
    algorithm: int = 4


@dataclass
class OracleRecord:
    rows: list = field(default_factory=list)
    final_iterate: Optional[np.ndarray] = None
    status: str = "ok"
    steps_taken: int = 0
    inner_fp_vector_ops: int = 0
    inner_lp_vector_ops: int = 0
    trace: Optional[np.ndarray] = None
    step_hash: Optional[np.ndarray] = None
    fullgrad_seconds: float = 0.0
    inner_seconds: float = 0.0
    rc: int = 0


def run_halp(obj: OracleObjective, cfg: OracleConfig, plan=None, trace_steps: int = 0,
             fullgrad_threads: int = 1, rows_cap: int = 0, hash_steps: int = 0) -> OracleRecord:
    """optimizers.cpp:387-459.  hash_steps > 0: OracleRecord.step_hash holds
    oq_code_hash of the codes after each of the first hash_steps inner steps
    (over all epochs), for REF-vs-MIRROR rounding-decision comparisons."""
    return _run(obj, cfg, plan, trace_steps, fullgrad_threads, rows_cap, 4, hash_steps)


def run(obj: OracleObjective, cfg: OracleConfig, plan=None, trace_steps: int = 0, fullgrad_threads: int = 1,
        rows_cap: int = 0) -> OracleRecord:
    """lpopt::run (optimizers.cpp:629-639) over Sgd (0), Svrg (1), LpSgd (2), LpSvrg (3), Halp (4)"""
    return _run(obj, cfg, plan, trace_steps, fullgrad_threads, rows_cap, int(cfg.algorithm))


def _run(obj, cfg, plan, trace_steps, fullgrad_threads, rows_cap, algorithm, hash_steps=0, quantized=None) -> OracleRecord:
    init = None
    if cfg.init is not None:
        init = np.ascontiguousarray(cfg.init, dtype=np.float64)
    c = _Config(cfg.alpha, cfg.epochs, cfg.inner_steps, cfg.bits, cfg.mu, cfg.option, cfg.full_grad_period,
                cfg.seed, cfg.metric_every_passes, cfg.delta_min, cfg.divergence_limit,
                init.ctypes.data if init is not None else None, cfg.delta, algorithm)
    cap = rows_cap or (cfg.epochs + 2)
    rows = (_Row * cap)()
    fin = np.zeros(obj.dim, dtype=np.float64)
    tr = np.zeros(trace_steps * obj.dim, dtype=np.int64) if trace_steps else None
    sh = np.zeros(hash_steps, dtype=np.uint64) if hash_steps else None
    rec = _Record(rows, cap, 0, fin.ctypes.data, 0, 0, 0, tr.ctypes.data if tr is not None else None,
                  tr.size if tr is not None else 0, 0.0, 0.0, fullgrad_threads,
                  sh.ctypes.data if sh is not None else None, hash_steps)
    if algorithm == 5:
        qs = None
        if quantized is not None:
            qs = _Quantized(quantized.codes.ctypes.data, quantized.delta, quantized.bits)
        rc = lib().oq_run_lm_halp(C.byref(obj._s), C.byref(qs) if qs is not None else None, C.byref(c), _plan(plan),
                                  C.byref(rec))
    else:
        rc = lib().oq_run(C.byref(obj._s), C.byref(c), _plan(plan), C.byref(rec))
    if rc not in (0, 2):
        _check(rc)
    out = OracleRecord()
    out.rc = rc
    out.rows = [
        dict(pass_=r.pass_, seconds=r.seconds, loss=r.loss, grad_norm=r.grad_norm, delta=r.delta,
             iterate_hash=r.iterate_hash, delta_inner=r.delta_inner, delta_aux=r.delta_aux)
        for r in rows[: rec.rows_n]
    ]
    out.final_iterate = fin
    out.status = STATUS[rec.status]
    out.steps_taken = rec.steps_taken
    out.inner_fp_vector_ops = rec.inner_fp_vector_ops
    out.inner_lp_vector_ops = rec.inner_lp_vector_ops
    out.fullgrad_seconds = rec.fullgrad_seconds
    out.inner_seconds = rec.inner_seconds
    if tr is not None:
        out.trace = tr.reshape(-1, obj.dim)
    out.step_hash = sh
    return out


def code_hash(codes) -> int:
    c = np.ascontiguousarray(codes, dtype=np.int64)
    return lib().oq_code_hash(c.ctypes.data, c.size)


def hash_vector(v) -> int:
    v = np.ascontiguousarray(v, dtype=np.float64)
    return lib().oq_hash_vector(v.ctypes.data, v.size)


def mexp(x: float) -> float:
    return lib().oq_mexp(x)


def mlog(x: float) -> float:
    return lib().oq_mlog(x)


_KINDS = {"regression": 0, "softmax": 1, "logistic": 2}
_DTYPES = {"f64": (F64, np.float64), "f32": (F32, np.float32), "bf16": (BF16, np.uint16)}


def generate(kind: str, n: int, d: int, *, num_classes: int = 0, dtype: str = "f32", noise_sd: float = 0.0,
             x_scale: float = 1.0, density: float = 1.0, seed: int = 0, rows=None, threads: int = 0):
    """Host restatement of the K6 generator (oracle/datagen.c): the same bytes
    as paper_1803_03383_b200.generate for the same arguments.  rows=(r0, r1)
    generates only that row range of the n-row dataset (bf16 as uint16 bits).
    Returns (X, y) for 'regression', (X, labels) otherwise."""
    code, npdt = _DTYPES[dtype]
    r0, r1 = rows if rows is not None else (0, n)
    g = _Datagen(_KINDS[kind], n, d, num_classes, code, noise_sd, x_scale, density, seed)
    X = np.empty((r1 - r0, d), dtype=npdt)
    y = lab = None
    if _KINDS[kind] == 0:
        y = np.empty(r1 - r0, dtype=np.float64)
    else:
        lab = np.empty(r1 - r0, dtype=np.int32)
    th = threads or (os.cpu_count() or 1)
    _check(lib().oq_datagen(C.byref(g), r0, r1 - r0, th, X.ctypes.data, y.ctypes.data if y is not None else None,
                            lab.ctypes.data if lab is not None else None))
    return (X, y) if y is not None else (X, lab)


@dataclass
class OracleQuantized:
    """lpopt::QuantizedExamples (objectives.hpp): int64 codes [n][d] at one scale"""

    codes: np.ndarray
    delta: float
    bits: int


def quantize_dataset(X, bits: int, seed: int) -> OracleQuantized:
    """objectives.cpp:110-133 (data_scale + stream-2 stochastic rounding, row-major)"""
    X = np.ascontiguousarray(X, dtype=np.float64)
    codes = np.empty(X.shape, dtype=np.int64)
    dl = C.c_double()
    _check(lib().oq_quantize_dataset(X.ctypes.data, X.shape[0], X.shape[1], bits, seed, codes.ctypes.data,
                                     C.byref(dl)))
    return OracleQuantized(codes, dl.value, bits)


def run_lm_halp(obj: OracleObjective, q: Optional[OracleQuantized], cfg: OracleConfig, plan=None,
                trace_steps: int = 0, hash_steps: int = 0) -> OracleRecord:
    """optimizers.cpp:461-627 (the non-bypass integer inner loop).  obj's X is
    not read: every pass uses the dequantized codes of q."""
    return _run(obj, cfg, plan, trace_steps, 1, 0, 5, hash_steps, q)
