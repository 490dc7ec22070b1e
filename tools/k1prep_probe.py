import sys; sys.path.insert(0, "/root/repo")
import numpy as np, paper_1803_03383_b200 as H
for n, d in [(600, 4096), (5000, 4096), (600, 2048), (300, 4096), (4194304 // 64, 4096)]:
    X = np.random.default_rng(0).standard_normal((n, d)).astype(np.float32)
    y = np.zeros(n)
    try:
        g = H.Objective(H.Dataset(X, targets=y), H.LossFamily.Squared, 0.0)
        print(n, d, "ok", g.plan())
    except Exception as e:
        print(n, d, "FAIL", e, H.plan_for(n, d, 1, "f32"))
