"""Inner-loop (K3) plan sweep: us/step for cluster size NC and coords/thread M.

    python tools/sweep_inner.py c2|c3|c4|c1 [T] [NC:M,NC:M,...] [VAR=VALUE ...]
"""
import itertools
import os
import subprocess
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

CHILD = r'''
import os, sys
sys.path.insert(0, os.environ["ROOT"])
import paper_1803_03383_b200 as H
which, T = sys.argv[1], int(sys.argv[2])
if which == "c2":
    X, lab = H.generate("softmax", 60000, 784, num_classes=10, dtype="f32", density=0.2, seed=0)
    obj = H.Objective(H.Dataset(X, labels=lab, num_classes=10), H.LossFamily.Softmax, 1e-4)
    cfg = dict(alpha=0.01, mu=2.5, bits=8)
elif which == "c3":
    X, y = H.generate("regression", 65536, 4096, dtype="f32", noise_sd=0.1, seed=3)
    obj = H.Objective(H.Dataset(X, targets=y), H.LossFamily.Squared, 0.0)
    cfg = dict(alpha=5e-5, mu=1.0, bits=16)
elif which == "c4":  # two-class bf16 d = 1024 on a 1 Mi-row slice of C4's generator (2 GiB > L2)
    X, lab = H.generate("logistic", 1048576, 1024, dtype="bf16", x_scale=1024 ** -0.5, seed=4)
    obj = H.Objective(H.Dataset(X, labels=lab, num_classes=2), H.LossFamily.Softmax, 1e-5)
    cfg = dict(alpha=0.05, mu=2.5, bits=8)
elif which.startswith("r"):
    X, y = H.generate("regression", 8192, int(which[1:]), dtype="f32", noise_sd=0.01, seed=0)
    obj = H.Objective(H.Dataset(X, targets=y), H.LossFamily.Squared, 0.0)
    cfg = dict(alpha=1e-4, mu=1e3, bits=8)
else:
    X, y = H.generate("regression", 8192, 256, dtype="f32", noise_sd=0.01, seed=0)
    obj = H.Objective(H.Dataset(X, targets=y), H.LossFamily.Squared, 0.0)
    cfg = dict(alpha=1e-3, mu=1e3, bits=8)
H.run_halp(obj, H.OptimizerConfig(algorithm=H.Algorithm.Halp, epochs=1, inner_steps=min(T, 1000), seed=0, **cfg))
H.run_halp(obj, H.OptimizerConfig(algorithm=H.Algorithm.Halp, epochs=1, inner_steps=T, seed=0, **cfg))
t = obj.timing(); p = obj.plan()
print("RESULT", p["in_ctas"], p["in_threads"], p["in_per"], "%.3f" % (1000 * t["inner_ms"] / T))
'''


def main():
    which = sys.argv[1]
    T = int(sys.argv[2]) if len(sys.argv) > 2 else 5000
    rgrid = [(0, 0)] + [(1, m) for m in (1, 2, 4, 8)] + [(nc, m) for nc in (2, 4, 8, 16) for m in (1, 2, 4)]
    grids = {"c2": [(nc, m) for nc in (4, 8, 16) for m in (1, 2, 4, 8)],
             "c3": [(nc, m) for nc in (1, 2, 4, 8, 16) for m in (1, 2, 4, 8)],
             "c4": [(0, 0)] + [(nc, m) for nc in (2, 4, 8, 16) for m in (1, 2, 4, 8) if 2048 <= nc * 256 * m <= 8192 * 2],
             "c1": [(nc, m) for nc in (1, 2, 4) for m in (1, 2, 4, 8)]}.get(which, rgrid)
    env = dict(os.environ, ROOT=os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    tag = ""
    for a in sys.argv[3:]:
        if "=" in a:
            k, v = a.split("=", 1)
            env[k] = v
            tag += " " + a
        else:
            grids = [tuple(int(x) for x in g.split(":")) for g in a.split(",")]
    for nc, m in grids:
        env["HALP_IN_NC"], env["HALP_IN_M"] = str(nc), str(m)  # 0 = the library's own plan
        r = subprocess.run([sys.executable, "-c", CHILD, which, str(T)], env=env, capture_output=True, text=True)
        line = [l for l in r.stdout.splitlines() if l.startswith("RESULT")]
        profs = [l for l in r.stdout.splitlines() if l.startswith("K3PROF")]  # -DHALP_K3_PROF builds
        for l in profs[-2:]:
            print("   ", l)
        print(which + tag, "NC", nc, "M", m, line[0] if line else ("ERR " + r.stderr.strip().splitlines()[-1][:150] if r.stderr.strip() else "ERR"), flush=True)


if __name__ == "__main__":
    main()
