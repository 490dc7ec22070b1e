"""K1 full-gradient GB/s at BASELINE C3 / C4 (full size) under env variants.

    python tools/fg_sweep.py c3|c4 [VAR=VAL,VAR=VAL ...] ...
Each variant runs in a child process (the plan reads the environment)."""
import os, subprocess, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
CHILD = r'''
import os, sys
sys.path.insert(0, os.environ["ROOT"])
import paper_1803_03383_b200 as H
w = sys.argv[1]
if w == "c3":
    n, d = 4194304, 4096
    X, y = H.generate("regression", n, d, dtype="f32", noise_sd=0.1, seed=3)
    obj = H.Objective(H.Dataset(X, targets=y), H.LossFamily.Squared, 0.0); b = n * d * 4 + n * 8
elif w.startswith("sq:"):  # sq:<n>:<d>:<dtype>  least squares of any shape
    _, n, d, dt = w.split(":"); n, d = int(n), int(d)
    X, y = H.generate("regression", n, d, dtype=dt, noise_sd=0.1, seed=3)
    obj = H.Objective(H.Dataset(X, targets=y), H.LossFamily.Squared, 0.0); b = n * d * {"f32": 4, "f64": 8, "bf16": 2}[dt] + n * 8
elif w == "c1":
    n, d = 8192, 256
    X, y = H.generate("regression", n, d, dtype="f32", noise_sd=0.01, seed=0)
    obj = H.Objective(H.Dataset(X, targets=y), H.LossFamily.Squared, 0.0); b = n * d * 4 + n * 8
else:
    n, d = 16777216, 1024
    X, y = H.generate("logistic", n, d, dtype="bf16", x_scale=d ** -0.5, seed=4)
    obj = H.Objective(H.Dataset(X, labels=y, num_classes=2), H.LossFamily.Softmax, 1e-5); b = n * d * 2 + n * 4
if os.environ.get("FG_WRAND"):  # generic iterate instead of w = 0
    import hashlib
    import numpy as np
    wv = np.random.default_rng(7).standard_normal(obj.dim()) * 0.5
    g = obj.full_gradient(wv)
    print("RESULT_HASH", hashlib.sha1(g.tobytes()).hexdigest()[:16], repr(obj.loss(wv)))
obj.bench_full_gradient(2)
ms = obj.bench_full_gradient(10 if w != "c1" else 200)
p = obj.plan()
print("RESULT %s %.3f ms %.1f GB/s frac %.3f plan thr=%d rows=%d stages=%d splits=%d" % (
    w, ms, b / ms / 1e6, b / ms / 1e6 / 6553.3, p["fg_threads"], p["fg_rows_per_stage"], p["fg_stages"], p["fg_splits"]))
'''
w = sys.argv[1]
for v in (sys.argv[2:] or [""]):
    env = dict(os.environ, ROOT=os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    for kv in filter(None, v.split(",")):
        k, val = kv.split("=")
        env[k] = val
    r = subprocess.run([sys.executable, "-c", CHILD, w], env=env, capture_output=True, text=True, timeout=600)
    out = [l for l in r.stdout.splitlines() if l.startswith("RESULT")]
    print(v or "default", out[-1] if out else ("FAILED " + r.stderr[-800:]), " ".join(out[:-1]), flush=True)
