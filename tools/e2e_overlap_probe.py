"""Probe: does creating the next C3 problem (68.7 GB H2D) overlap the current epoch?"""
import os, sys, threading, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import bench
import paper_1803_03383_b200 as H

X, y = H.generate("regression", 4194304, 4096, dtype="f32", noise_sd=0.1, seed=3)
Xh = torch.empty(X.shape, dtype=X.dtype, pin_memory=True)
Xh.copy_(X)
yh = y.cpu().numpy()
Xn = Xh.numpy()
del X, y
torch.cuda.empty_cache()
mk = lambda: H.Objective(H.Dataset(Xn, targets=yh), H.LossFamily.Squared, 0.0)
a, b = mk(), mk()
H.run_halp(a, bench.c3_config(H, 1))
del a, b
T0 = time.perf_counter()
log = []
def stamp(tag):
    log.append((tag, time.perf_counter() - T0))
stamp("create0 start"); o = mk(); stamp("create0 end")
stamp("run0 start"); H.run_halp(o, bench.c3_config(H, 1)); stamp("run0 end")
nxt = [None]
def bg():
    stamp("bg create start"); nxt[0] = mk(); stamp("bg create end")
th = threading.Thread(target=bg)
stamp("run1 start + bg"); th.start(); H.run_halp(o, bench.c3_config(H, 1)); stamp("run1 end"); th.join(); stamp("joined")
for t, v in log:
    print(f"{v:8.3f}  {t}")
