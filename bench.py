"""Benchmark of the B200 HALP solver (driver contract: one JSON line on rank 0).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference]

Headline workload = BASELINE.json configs[2] ("C3"), the largest config
that fits one GPU: least-squares regression, N = 4,194,304, d = 4096, fp32
Gaussian x and w*, noise sd 0.1, HALP b = 16, T = N/8 = 524,288; alpha and
mu are unspecified in BASELINE and recorded in `config` (alpha = 5e-5 ~
0.2/|x|^2, mu = 1).  X is 68.7 GB (> the 126 MB L2).  The
data is synthetic: the counter-based generator K6 (device) / oracle/datagen.c
(host, byte-identical, tests/test_gpu_datagen.py).

One step = one HALP epoch of lpopt::run_halp (optimizers.cpp:387-459): the
full-gradient + loss pass at w~ (K1), centering (K2), sample indices (K4)
and the T-step b-bit inner loop (K3).  `value` = epochs/s of the whole job.
At N > 1 the same single problem runs on N GPUs: the full-gradient pass is
row-sharded (one NCCL all-gather per epoch), the sequential inner loop is
replicated -- total work fixed, so scaling is "strong".

Extra keys: `e2e` (the same epoch through the public API from pinned host
buffers, X uploaded every step), `roofline` (K1 at C3 against measured
HBM bandwidth, from the K1 time inside the timed region), `inner_loop` (K3,
the latency-bound stage that dominates the epoch), `fullgrad` (K1 at C3 and
C4), `c2` (the MNIST-shaped softmax epoch), `batch` (C5 via K5), `grid`,
`cpu_baseline` (the oracle's reference-order restatement on the host cores,
bounded sample, extrapolation stated).

--impl reference times the reference algorithm on the CPU.  The reference
(proj/, C++ + Eigen) cannot be built in this image (Eigen3 and vendor/ are
absent), so its restatement oracle/liboracle.so in REF order
(pinned to the reference's golden traces) runs the same C3 workload on a
bounded row / step sample per step, full gradient on all host threads (the
reference's blocked scheme, objectives.cpp:289-301), sequential inner loop;
its data comes from oracle/datagen.c.  That arm never loads libhalp_b200.so.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

C3 = dict(n=4194304, d=4096, dtype="f32", noise_sd=0.1, seed=3, bits=16, T=4194304 // 8, alpha=5e-5, mu=1.0, l2=0.0)
C2 = dict(n=60000, d=784, C=10, density=0.2, l2=1e-4, bits=8, alpha=0.01, mu=2.5)
C4 = dict(n=16777216, d=1024, dtype="bf16", epochs=3)
C5 = dict(nprob=512, n=4096, d=128, epochs=10, mu=3.0)  # per GPU; T = 2N (reference default)
# CPU sample of the C3 epoch: rows / steps divisors (the epoch cost is linear in both)
CPU_ROWS_DIV, CPU_STEPS_DIV = 64, 64

METRIC, UNIT = "HALP epochs/sec", "epochs/s"


def headline_config(world: int) -> dict:
    """identical in both arms (the driver compares them)"""
    return {
        "workload": "C3: least squares N=4194304 d=4096 fp32 Gaussian x and w*, noise 0.1; HALP b=16, "
                    "T=N/8=524288, alpha=5e-5, mu=1 (alpha, mu unspecified in BASELINE), option I, seed 0",
        "N": C3["n"], "d": C3["d"], "bits": C3["bits"], "T": C3["T"], "alpha": C3["alpha"], "mu": C3["mu"],
        "l2": C3["l2"], "x_dtype": "f32", "data_seed": C3["seed"],
        "l2_cache": "inputs (68.7 GB) larger than L2 (126 MB)",
        "parallelism": "single GPU" if world == 1 else
        f"full-gradient rows sharded x{world} + one NCCL all-gather per epoch; inner loop replicated",
    }


def peaks():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        return {"hbm_gbs": 6650.0, "_fallback": True}


class Clocks:
    """nvidia-smi sampler running during the timed region."""

    def __init__(self, device: int):
        self.f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
        q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")
        try:
            self.p = subprocess.Popen(["nvidia-smi", "-i", str(device), f"--query-gpu={q}", "--format=csv,noheader,nounits",
                                       "-lms", "200"], stdout=self.f, stderr=subprocess.DEVNULL)
        except Exception:
            self.p = None

    def stop(self):
        if self.p is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.p.terminate()
        self.p.wait()
        self.f.flush()
        rows = []
        for line in open(self.f.name):
            parts = [x.strip() for x in line.split(",")]
            if len(parts) >= 7:
                try:
                    rows.append((float(parts[0]), float(parts[1]), parts[3:7]))
                except ValueError:
                    pass
        os.unlink(self.f.name)
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no samples"]}
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for _, _, r in rows for i, v in enumerate(r) if v.lower() == "active"})
        return {"sm_mhz": statistics.median(r[0] for r in rows), "sm_max_mhz": max(r[1] for r in rows),
                "samples": len(rows), "reasons": reasons}


def dist_env():
    return int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)), int(os.environ.get("LOCAL_RANK", 0))


# ----------------------------------------------------------------------------- CPU (oracle) legs
def cpu_c3_sample(O, threads: int, rows_div: int = CPU_ROWS_DIV, steps_div: int = CPU_STEPS_DIV, data=None):
    """One bounded sample of the C3 epoch on the host: the REF-order oracle's
    run_halp (1 epoch) on the first N/rows_div rows of the C3 dataset with
    T/steps_div inner steps; full gradient on `threads` threads.  The epoch
    is one full-gradient + loss pass over N rows plus T sequential inner
    steps, both linear in their count, so
        epoch_s = (fullgrad_s / 2 passes) * rows_div + inner_s * steps_div
    (a 1-epoch run makes 2 passes: the epoch start and the final boundary).
    Returns (epoch_s, measured_s, data)."""
    ns = C3["n"] // rows_div
    if data is None:
        X, y = O.generate("regression", C3["n"], C3["d"], dtype="f32", noise_sd=C3["noise_sd"], seed=C3["seed"],
                          rows=(0, ns), threads=threads)
        data = O.OracleObjective(X, y=y, l2=C3["l2"])
    cfg = O.OracleConfig(alpha=C3["alpha"], epochs=1, inner_steps=C3["T"] // steps_div, bits=C3["bits"], mu=C3["mu"],
                         seed=0)
    t = time.perf_counter()
    rec = O.run_halp(data, cfg, fullgrad_threads=threads)
    measured = time.perf_counter() - t
    epoch_s = rec.fullgrad_seconds / 2.0 * rows_div + rec.inner_seconds * steps_div
    return epoch_s, measured, data


def cpu_c4_fullgrad(O, threads: int, rows_div: int = 256):
    """C4's full-gradient + loss pass on the host: the REF-order oracle (the
    reference's 1024-row blocks on `threads` threads, objectives.cpp:289-301) over
    the first N/rows_div rows of the C4 dataset, extrapolated linearly in rows."""
    n, d = C4["n"], C4["d"]
    ns = n // rows_div
    X, lab = O.generate("logistic", n, d, dtype="bf16", x_scale=d ** -0.5, seed=4, rows=(0, ns), threads=threads)
    o = O.OracleObjective(X, labels=lab, num_classes=2, l2=1e-5)
    w = np.random.default_rng(7).standard_normal(2 * d)
    o.full_gradient(w, num_threads=threads)
    t = time.perf_counter()
    reps = 3
    for _ in range(reps):
        o.full_gradient(w, num_threads=threads)
        o.loss_value(w)
    s = (time.perf_counter() - t) / reps
    return {"ms_per_pass": 1000.0 * s * rows_div, "cores": threads, "kind": "port",
            "sample": f"REF-order oracle full_gradient + loss on rows [0, N/{rows_div}) = {ns} rows of the C4 dataset, "
                      f"{threads} threads, x{rows_div} (linear in rows)", "measured_seconds": s * reps}


def cpu_c5_batch(O, threads: int):
    """C5 on the host: `threads` of the batch's problems solved concurrently, one
    REF-order oracle run_halp (K = 10, T = 2N) per thread; problems are independent,
    so the batch of 512 costs 512 / threads such rounds."""
    import concurrent.futures as cf

    n, d = C5["n"], C5["d"]
    rng = np.random.default_rng(0)
    probs = []
    for q in range(threads):
        X, y = O.generate("regression", n, d, dtype="f32", noise_sd=0.1, seed=10_000 + q)
        probs.append((O.OracleObjective(X, y=y, l2=0.0),
                      O.OracleConfig(alpha=float(10 ** rng.uniform(-4, -2)), epochs=C5["epochs"],
                                     bits=8 if q % 2 == 0 else 16, mu=C5["mu"], seed=q)))
    t = time.perf_counter()
    with cf.ThreadPoolExecutor(threads) as ex:
        list(ex.map(lambda pc: O.run_halp(pc[0], pc[1]), probs))
    s = time.perf_counter() - t
    per_batch = s * C5["nprob"] / threads
    return {"ms_per_batch": 1000.0 * per_batch, "problem_epochs_per_s": C5["nprob"] * C5["epochs"] / per_batch,
            "cores": threads, "kind": "port",
            "sample": f"{threads} of the 512 problems, one REF-order oracle run_halp per host thread concurrently; "
                      f"batch = measured x 512/{threads}", "measured_seconds": s}


def cpu_sample_text(threads):
    return (f"REF-order oracle run_halp, 1 epoch on rows [0, N/{CPU_ROWS_DIV}) of the C3 dataset with "
            f"T/{CPU_STEPS_DIV} = {C3['T'] // CPU_STEPS_DIV} inner steps, full gradient on {threads} threads "
            f"(objectives.cpp:289-301 blocks), inner loop sequential; epoch = (fullgrad_s/2)*{CPU_ROWS_DIV} + "
            f"inner_s*{CPU_STEPS_DIV}")


def run_reference(args, rank, world):
    """--impl reference: rank 0 only; the oracle restatement on all host threads.
    Imports nothing from the product package (no libhalp_b200.so)."""
    if rank != 0:
        return
    from oracle import oracle as O

    O.build()
    threads = os.cpu_count() or 1
    data = None
    for _ in range(args.warmup):
        _, _, data = cpu_c3_sample(O, threads, data=data)
    eps, meas = [], []
    for _ in range(args.steps):
        e, m, data = cpu_c3_sample(O, threads, data=data)
        eps.append(e)
        meas.append(m)
    ms = 1000.0 * sum(eps) / len(eps)
    v = 1000.0 / ms
    line = {
        "impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (oracle/datagen.c = K6 bytes, seeded)", "config": headline_config(world),
        "cpu_baseline": {"value": v, "unit": UNIT, "cores": threads, "kind": "port", "sample": cpu_sample_text(threads),
                         "measured_seconds_per_step": sum(meas) / len(meas)},
        "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "note": "reference proj/ cannot be built here (Eigen3, vendor/ absent); oracle/liboracle.so REF order "
                "restates it and reproduces its golden traces",
    }
    print(json.dumps(line), flush=True)


# ----------------------------------------------------------------------------- GPU legs
def c3_objective(H, device, world, rank, nccl_id):
    X, y = H.generate("regression", C3["n"], C3["d"], dtype="f32", noise_sd=C3["noise_sd"], x_scale=1.0,
                      seed=C3["seed"], device=device)
    obj = H.Objective(H.Dataset(X, targets=y), H.LossFamily.Squared, C3["l2"], device=device, world_size=world,
                      rank=rank, nccl_id=nccl_id)
    return obj, X, y


def c3_config(H, epochs):
    return H.OptimizerConfig(algorithm=H.Algorithm.Halp, alpha=C3["alpha"], epochs=epochs, inner_steps=C3["T"],
                             bits=C3["bits"], mu=C3["mu"], seed=0)


def fullgrad_c4(H, device, reps, world, rank, nccl_id):
    """K1 at C4: binary logistic as softmax C=2, bf16 x ~ N(0, 1/d), l2 1e-5"""
    n, d = C4["n"], C4["d"]
    X, y = H.generate("logistic", n, d, dtype="bf16", x_scale=d ** -0.5, seed=4, device=device)
    obj = H.Objective(H.Dataset(X, labels=y, num_classes=2), H.LossFamily.Softmax, 1e-5, device=device,
                      world_size=world, rank=rank, nccl_id=nccl_id)
    wgen = np.random.default_rng(7).standard_normal(obj.dim())
    obj.full_gradient(wgen)
    obj.bench_full_gradient(2)
    ms = obj.bench_full_gradient(reps)
    pl = obj.plan()
    rows = int(n * (pl["fg_split_end"] - pl["fg_split_begin"]) // pl["fg_splits"])
    # the same pass as it runs in the solver: K1 once per HALP epoch, the inner loop between
    # two passes (b = 8, alpha = 0.05, mu = 2.5 as in tests/test_gpu_baseline_configs.py; T = N/64)
    cfg = H.OptimizerConfig(algorithm=H.Algorithm.Halp, alpha=0.05, epochs=C4["epochs"], inner_steps=n // 64, bits=8,
                            mu=2.5, seed=0)
    rec = H.run_halp(obj, cfg)
    tim = obj.timing()
    in_epoch = {"ms_per_pass": tim["fullgrad_ms"] / (C4["epochs"] + 1),
                "inner_ns_per_step": 1e6 * tim["inner_ms"] / (C4["epochs"] * (n // 64)),
                "epochs": C4["epochs"], "T": n // 64, "loss_first_last": [rec.rows[0].loss, rec.rows[-1].loss]}
    return ms, rows * d * 2 + rows * 4, pl, in_epoch


def c2_epochs(H, device, rank, epochs):
    """the MNIST-shaped softmax epoch (BASELINE C2), inputs resident"""
    import torch

    X, lab = H.generate("softmax", C2["n"], C2["d"], num_classes=C2["C"], dtype="f32", density=C2["density"],
                        seed=rank, device=device)
    obj = H.Objective(H.Dataset(X, labels=lab, num_classes=C2["C"]), H.LossFamily.Softmax, C2["l2"], device=device)
    cfg = lambda k: H.OptimizerConfig(algorithm=H.Algorithm.Halp, alpha=C2["alpha"], epochs=k, inner_steps=C2["n"],
                                      bits=C2["bits"], mu=C2["mu"], seed=rank)
    H.run_halp(obj, cfg(1))
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    rec = H.run_halp(obj, cfg(epochs))
    e1.record()
    torch.cuda.synchronize()
    tim = obj.timing()
    ms = e0.elapsed_time(e1)
    return {"workload": "C2: softmax N=60000 d=784 C=10 fp32 (80% zeros), l2=1e-4, HALP b=8, alpha=0.01, T=N, "
                        "mu=2.5", "epochs_per_s": epochs / (ms / 1000.0), "ms_per_epoch": ms / epochs,
            "inner_ns_per_step": 1e6 * tim["inner_ms"] / (epochs * C2["n"]),
            "fullgrad_ms_per_pass": tim["fullgrad_ms"] / (epochs + 1),
            "loss_first_last": [rec.rows[0].loss, rec.rows[-1].loss]}


GRID = dict(n=1000, d=64, alphas=17, mus=13, seeds=(1, 2, 3), epochs=10, T=2000)


def grid_configs(H):
    """the reference's conditioning-sweep grid (harness.cpp:462-468: 17 step
    sizes x 13 scales per width) on one 1000 x 64 least-squares problem"""
    alphas = [float(a) for a in np.logspace(-4, -1, GRID["alphas"])]
    mus = [float(m) for m in np.logspace(-1, 2, GRID["mus"])]
    base = H.OptimizerConfig(algorithm=H.Algorithm.Halp, alpha=1e-3, epochs=GRID["epochs"], inner_steps=GRID["T"],
                             bits=8, mu=1.0, seed=0)
    return base, [H.GridAxis("alpha", alphas), H.GridAxis("mu", mus)]


def grid_bench(H, device):
    """grid_search over the shared dataset: every (alpha, mu, seed) run in one K5 launch"""
    import torch

    X, y = H.generate("regression", GRID["n"], GRID["d"], dtype="f64", noise_sd=0.1, seed=42, device=device)
    obj = H.Objective(H.Dataset(X, targets=y), H.LossFamily.Squared, 0.0, device=device)
    base, axes = grid_configs(H)
    H.grid_search(obj, base, [H.GridAxis("alpha", axes[0].values[:2]), H.GridAxis("mu", axes[1].values[:2])], [1])
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    res = H.grid_search(obj, base, axes, GRID["seeds"])
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    runs = len(res.points) * len(GRID["seeds"])
    return {"workload": "grid_search (harness.cpp:379-447): 17 alpha x 13 mu x 3 seeds on one 1000x64 f64 "
                        "least-squares problem, HALP b=8, T=2000, K=10; all runs in one K5 launch",
            "runs": runs, "wall_ms": 1000.0 * dt, "runs_per_s": runs / dt, "device_ms": res.device_ms,
            "best": {"alpha": res.best_config.alpha, "mu": res.best_config.mu,
                     "grad_norm": res.points[res.best_index].mean_metric}}


def c5_batch(H, device, rank, reps=2):
    """BASELINE C5: 512 independent least-squares HALP problems per GPU (4096 x 128
    fp32 Gaussian, per-problem seeds, alpha log-uniform [1e-4, 1e-2], b in {8, 16}
    alternating, T = 2N, K = 10, mu = 3 (unspecified in BASELINE; the golden value)),
    solved by K5 in one launch.  Returns device ms of the batch run."""
    import torch

    P, n, d = C5["nprob"], C5["n"], C5["d"]
    X = torch.empty((P, n, d), dtype=torch.float32, device=f"cuda:{device}")
    Y = torch.empty((P, n), dtype=torch.float64, device=f"cuda:{device}")
    for q in range(P):
        x1, y1 = H.generate("regression", n, d, dtype="f32", noise_sd=0.1, seed=10_000 * (rank + 1) + q, device=device)
        X[q].copy_(x1)
        Y[q].copy_(y1)
    b = H.BatchProblems(X, Y, l2=0.0, device=device)
    rng = np.random.default_rng(rank)
    cfgs = [H.OptimizerConfig(algorithm=H.Algorithm.Halp, alpha=float(10 ** rng.uniform(-4, -2)), epochs=C5["epochs"],
                              inner_steps=0, bits=8 if q % 2 == 0 else 16, mu=C5["mu"], seed=q) for q in range(P)]
    b.run([H.OptimizerConfig(algorithm=H.Algorithm.Halp, alpha=c.alpha, epochs=1, inner_steps=64, bits=c.bits,
                             mu=c.mu, seed=c.seed) for c in cfgs])
    ms = []
    for _ in range(reps):
        recs = b.run(cfgs)
        ms.append(b.device_ms)
    n_div = sum(r.status == "diverged" for r in recs)
    return min(ms), n_div, P * C5["epochs"] * 2 * n


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--no-extras", action="store_true", help="headline + e2e + cpu only")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--fg-reps", type=int, default=10)
    args = ap.parse_args()
    rank, world, local = dist_env()
    if args.impl == "reference":
        run_reference(args, rank, world)
        return
    if args.warmup < 3:
        args.warmup = 3

    import torch

    torch.cuda.set_device(local)
    pg = None
    if world > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        pg = dist

    import paper_1803_03383_b200 as H

    pk = peaks()

    def barrier():
        torch.cuda.synchronize()
        if pg:
            pg.barrier()
        torch.cuda.synchronize()

    def max_over_ranks(v):
        if not pg:
            return v
        t = torch.tensor([v], dtype=torch.float64, device="cuda")
        pg.all_reduce(t, op=pg.ReduceOp.MAX)
        return float(t.item())

    nccl_id = None
    if world > 1:
        import ctypes

        nccl = ctypes.CDLL("libnccl.so.2")
        idb = ctypes.create_string_buffer(128)
        if rank == 0:
            nccl.ncclGetUniqueId(idb)
        t = torch.tensor(list(idb.raw), dtype=torch.uint8, device="cuda")
        pg.broadcast(t, 0)
        nccl_id = bytes(t.cpu().tolist())

    # ---------------- headline: C3 HALP epochs, inputs resident in HBM ----------------
    obj, X, y = c3_objective(H, local, world, rank, nccl_id)
    H.run_halp(obj, c3_config(H, args.warmup))
    barrier()
    clk = Clocks(local)
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record()
    rec = H.run_halp(obj, c3_config(H, args.steps))
    ev1.record()
    barrier()
    clocks = clk.stop()
    ms_total = max_over_ranks(ev0.elapsed_time(ev1))
    tim = obj.timing()
    plan = obj.plan()
    ms_step = ms_total / args.steps
    value = args.steps / (ms_total / 1000.0)
    inner_ns = 1e6 * tim["inner_ms"] / (args.steps * C3["T"])
    fg_passes = args.steps + 1
    fg_ms = tim["fullgrad_ms"] / fg_passes  # K1 + split tree, CUDA events on the solver stream
    rows_local = int(C3["n"] * (plan["fg_split_end"] - plan["fg_split_begin"]) // plan["fg_splits"])
    algo_bytes = rows_local * C3["d"] * 4 + rows_local * 8
    achieved = algo_bytes / (fg_ms / 1000.0) / 1e9
    traffic = None
    try:
        tj = json.load(open(os.path.join(ROOT, "profiles", "k1_traffic.json")))["C3"]
        traffic = tj["dram_read_bytes_per_launch"] + tj["dram_write_bytes_per_launch"]
    except Exception:
        pass
    roofline = {"kernel": "k1_stream (+k1_tree_pass): the C3 full-gradient + loss pass (north star: >= 70% of HBM)",
                "bound": "hbm", "achieved": achieved, "peak": pk["hbm_gbs"], "unit": "GB/s",
                "frac": achieved / pk["hbm_gbs"], "traffic": traffic,
                "traffic_source": "profiles/k1_traffic.json (ncu dram__bytes_read+write per launch)",
                "peak_source": "MEASURED_PEAKS.json hbm_gbs" if "_fallback" not in pk else "fallback 6650 GB/s",
                "algorithmic_bytes_per_launch": algo_bytes, "launch_ms": fg_ms,
                "bytes_model": "rows*d*4 (x, fp32) + rows*8 (y, fp64) per pass; rows = this rank's row shard",
                "timed": f"K1 time inside the timed region ({fg_passes} passes, CUDA events on the solver stream)",
                "frac_of_nominal_8000": achieved / 8000.0,
                "note": "K1 is the HBM-bound kernel; the epoch's dominant kernel is K3 (latency-bound serial "
                        "chain, see inner_loop).  peak is a torch copy (read + write) figure: a read-only "
                        "stream can exceed it, so frac may pass 1; frac_of_nominal_8000 is against HBM3e's "
                        "nominal 8 TB/s"}
    inner = {"kernel": "k3_inner", "bound": "latency (one serial chain per step)", "ns_per_step": inner_ns,
             "steps_per_s": 1e9 / inner_ns, "cycles_per_step_at_sm_clock": inner_ns * (clocks.get("sm_mhz") or 0) / 1e3,
             "share_of_epoch": tim["inner_ms"] / ms_total if world == 1 else None,
             "plan": {k: plan[k] for k in ("in_ctas", "in_threads", "in_per")}}
    gpu_launches = int(tim["kernel_launches"])
    loss_fl = [rec.rows[0].loss, rec.rows[-1].loss]

    # ---------------- e2e: the same epoch through the public API from pinned host buffers ----------------
    e2e = None
    if not args.no_e2e and world == 1:
        Xh = torch.empty(X.shape, dtype=X.dtype, pin_memory=True)
        Xh.copy_(X)
        yh = y.cpu().numpy()
        Xn = Xh.numpy()
        del obj, X, y
        torch.cuda.empty_cache()
        e_steps = max(1, min(args.steps, 6))  # streamed solves: the first upload is not overlapped, amortise it
        mk = lambda: H.Objective(H.Dataset(Xn, targets=yh), H.LossFamily.Squared, C3["l2"], device=local)
        # untimed warm-up: the first problems grow the device pool by two 68.7 GB
        # copies of X (later problems reuse them), like the headline's warm-up epochs
        o_a, o_b = mk(), mk()
        H.run_halp(o_a, c3_config(H, 1))
        del o_a, o_b
        barrier()

        def account(o, r, acc):
            tt = o.timing()
            acc[0] += tt["h2d_bytes"] + Xn.nbytes + yh.nbytes
            acc[1] += tt["d2h_bytes"] + r.final_iterate.nbytes

        # (1) serial: create (upload) -> run_halp -> record, one solve after another
        acc_s = [0, 0]
        t0 = time.perf_counter()
        for _ in range(2):
            o2 = mk()
            r2 = H.run_halp(o2, c3_config(H, 1))
            account(o2, r2, acc_s)
            del o2
        torch.cuda.synchronize()
        serial_ms = 1000.0 * (time.perf_counter() - t0) / 2
        # (2) streamed: the next solve's Objective (its 68.7 GB upload, on its own
        # stream) is created by a second host thread while the current epoch runs --
        # independent runs may overlap; every step still uploads its X
        import threading

        acc = [0, 0]
        barrier()
        t0 = time.perf_counter()
        nxt = [mk()]
        for s_ in range(e_steps):
            cur = nxt[0]
            th = None
            if s_ + 1 < e_steps:
                th = threading.Thread(target=lambda: nxt.__setitem__(0, mk()))
                th.start()
            r2 = H.run_halp(cur, c3_config(H, 1))
            account(cur, r2, acc)
            if th is not None:
                th.join()
            del cur
        torch.cuda.synchronize()
        e_ms = 1000.0 * (time.perf_counter() - t0)
        del nxt
        barrier()
        # (3) for reference only: what a K-epoch solve costs end to end when X is uploaded
        # once, as one run_halp call does (the headline e2e above re-uploads X every epoch)
        WR_EPOCHS = 8
        t0 = time.perf_counter()
        o3 = mk()
        r3 = H.run_halp(o3, c3_config(H, WR_EPOCHS))
        torch.cuda.synchronize()
        wr_s = time.perf_counter() - t0
        wr_rows = len(r3.rows)
        del o3, r3
        e2e = {"value": e_steps / (e_ms / 1000.0), "unit": UNIT, "h2d_bytes_per_step": int(acc[0] // e_steps),
               "d2h_bytes_per_step": int(acc[1] // e_steps), "ms_per_step": e_ms / e_steps,
               "serial_ms_per_step": serial_ms, "serial_value": 1000.0 / serial_ms,
               "whole_run": {"epochs": WR_EPOCHS, "epochs_per_s": WR_EPOCHS / wr_s, "seconds": wr_s, "rows": wr_rows,
                             "what": "Objective(pinned host X, y) + ONE run_halp(epochs=8): one 68.7 GB upload "
                                     "amortised over the run, host wall clock; not the headline e2e"},
               "path": "Objective(pinned host numpy X, y) -> run_halp(epochs=1) -> RunRecord per step, 68.7 GB "
                       "upload of X inside every step; the next step's Objective is created (uploaded) by a second "
                       "host thread while the current epoch runs (serial_*: one after another); host wall clock"}
        del Xh, Xn
    else:
        if world > 1:
            e2e = {"value": None, "unit": UNIT, "h2d_bytes_per_step": None, "d2h_bytes_per_step": None,
                   "note": "not measured at N>1: every rank needs the full 68.7 GB X pinned on one host "
                           "(196 GB RAM)"}
        del obj, X, y
    torch.cuda.empty_cache()

    extras = {}
    if not args.no_extras:
        # ---------------- K1 full-gradient sweeps (C3 via a fresh problem, C4) ----------------
        barrier()
        o3, X3, y3 = c3_objective(H, local, world, rank, nccl_id)
        o3.full_gradient(np.random.default_rng(7).standard_normal(o3.dim()) * 0.5)
        o3.bench_full_gradient(2)
        ms3 = max_over_ranks(o3.bench_full_gradient(args.fg_reps))
        gbs3 = algo_bytes * world / (ms3 / 1000.0) / 1e9
        del o3, X3, y3
        torch.cuda.empty_cache()
        barrier()
        ms4, b4, _, c4_epoch = fullgrad_c4(H, local, args.fg_reps, world, rank, nccl_id)
        ms4 = max_over_ranks(ms4)
        gbs4 = b4 * world / (ms4 / 1000.0) / 1e9
        c4_epoch["ms_per_pass"] = max_over_ranks(c4_epoch["ms_per_pass"])
        c4_epoch["GB_per_s"] = b4 * world / (c4_epoch["ms_per_pass"] / 1000.0) / 1e9
        c4_epoch["frac_of_hbm_peak"] = c4_epoch["GB_per_s"] / world / pk["hbm_gbs"]
        c4_epoch["what"] = ("K1 (+ split tree) timed by CUDA events inside a C4 HALP run (b=8, T=N/64, alpha=0.05, "
                            "mu=2.5): one pass per epoch between inner loops, as the solver runs it")
        torch.cuda.empty_cache()
        extras["fullgrad"] = {
            "C3": {"shape": "4194304x4096 f32", "ms_per_pass": ms3, "GB_per_s": gbs3,
                   "frac_of_hbm_peak": gbs3 / world / pk["hbm_gbs"], "algorithmic_bytes_per_gpu": algo_bytes,
                   "includes": "K1 + split tree" + (" + NCCL all-gather + finalize" if world > 1 else "")},
            "C4": {"shape": "16777216x1024 bf16 (softmax C=2)", "ms_per_pass": ms4, "GB_per_s": gbs4,
                   "frac_of_hbm_peak": gbs4 / world / pk["hbm_gbs"], "algorithmic_bytes_per_gpu": b4,
                   "timed": f"{args.fg_reps} passes back to back", "in_epoch": c4_epoch}}
        # ---------------- C2 epochs (MNIST-shaped softmax) ----------------
        barrier()
        extras["c2"] = c2_epochs(H, local, rank, 5)
        torch.cuda.empty_cache()
        # ---------------- C5: batched independent problems (K5) ----------------
        barrier()
        bms, ndiv, inner_steps = c5_batch(H, local, rank)
        bms = max_over_ranks(bms)
        extras["batch"] = {"workload": "C5: 512 least-squares problems/GPU, 4096x128 fp32, T=2N=8192, K=10, b 8/16, "
                                       "mu 3", "problems": C5["nprob"] * world, "ms_per_batch": bms,
                           "problem_epochs_per_s": C5["nprob"] * world * C5["epochs"] / (bms / 1000.0),
                           "inner_steps_per_s": inner_steps * world / (bms / 1000.0), "diverged": ndiv,
                           "scaling": "weak (problems sharded, no collective)"}
        torch.cuda.empty_cache()
        barrier()
        extras["grid"] = grid_bench(H, local)
        torch.cuda.empty_cache()

    # ---------------- CPU baseline (rank 0, N=1 only) ----------------
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        from oracle import oracle as O

        O.build()
        threads = os.cpu_count() or 1
        ep, meas, data = cpu_c3_sample(O, threads)
        ep2, meas2, _ = cpu_c3_sample(O, threads, data=data)
        cpu = {"value": 2.0 / (ep + ep2), "unit": UNIT, "cores": threads, "kind": "port",
               "sample": cpu_sample_text(threads) + " (mean of 2 samples)", "measured_seconds": meas + meas2}
        if not args.no_extras:
            del data
            if "fullgrad" in extras:
                extras["fullgrad"]["C4"]["cpu_baseline"] = cpu_c4_fullgrad(O, threads)
            if "batch" in extras:
                extras["batch"]["cpu_baseline"] = cpu_c5_batch(O, threads)

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (K6 device generator, seeded; byte-identical host restatement in oracle/datagen.c)",
            "config": headline_config(world),
            "loss_first_last": loss_fl, "roofline": roofline, "inner_loop": inner, "cpu_baseline": cpu, "e2e": e2e,
            "gpu_launches": gpu_launches, "clocks": clocks,
            "plan": {k: plan[k] for k in ("fg_threads", "fg_splits", "in_ctas", "in_threads", "in_per")},
        }
        line.update(extras)
        print(json.dumps(line), flush=True)
    if pg:
        pg.barrier()
        pg.destroy_process_group()


if __name__ == "__main__":
    main()
