"""Break the bench's e2e step (Objective from pinned host numpy -> run_halp(1 epoch) -> destroy) into parts."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_1803_03383_b200 as H

X, lab = H.generate("softmax", 60000, 784, num_classes=10, dtype="f32", density=0.2, seed=0, device=0)
Xh = torch.empty(X.shape, dtype=X.dtype, pin_memory=True); Xh.copy_(X)
lh = torch.empty(lab.shape, dtype=lab.dtype, pin_memory=True); lh.copy_(lab)
Xn, ln = Xh.numpy(), lh.numpy()
cfg = H.OptimizerConfig(algorithm=H.Algorithm.Halp, alpha=0.01, epochs=1, inner_steps=60000, bits=8, mu=2.5, seed=0)
for it in range(4):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    o = H.Objective(H.Dataset(Xn, labels=ln, num_classes=10), H.LossFamily.Softmax, 1e-4, device=0)
    t1 = time.perf_counter()
    r = H.run_halp(o, cfg)
    t2 = time.perf_counter()
    tt = o.timing()
    del o
    t3 = time.perf_counter()
    print(f"create {1e3*(t1-t0):.1f} ms  run {1e3*(t2-t1):.1f} ms  destroy {1e3*(t3-t2):.1f} ms  timing {tt}", flush=True)
