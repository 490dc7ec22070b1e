"""Time the bench's grid search pieces (BatchProblems creation, the K5 run)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1803_03383_b200 as H
import bench

X, y = H.generate("regression", 1000, 64, dtype="f64", noise_sd=0.1, seed=42, device=0)
base, axes = bench.grid_configs(H)
import itertools, copy
cfgs = []
for a, m in itertools.product(axes[0].values, axes[1].values):
    for sd in (1, 2, 3):
        c = copy.deepcopy(base); c.alpha = a; c.mu = m; c.seed = sd; cfgs.append(c)
for it in range(3):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    b = H.BatchProblems(X, y, l2=0.0, nprob=len(cfgs))
    torch.cuda.synchronize(); t1 = time.perf_counter()
    recs = b.run(cfgs)
    t2 = time.perf_counter()
    print(f"create {1e3*(t1-t0):.1f} ms  run {1e3*(t2-t1):.1f} ms  device {b.device_ms:.1f} ms", flush=True)
    del b
