"""Small fixed workloads for ncu captures (one launch of each hot kernel).

    python tools/prof_run.py c2      # C2 epoch: k1_fullgrad x2, k_finalize, k_samples, k3_inner (T=60000)
    python tools/prof_run.py c3      # K1 on a C3-shaped slice: 524288 x 4096 f32 (8 GiB > L2)
    python tools/prof_run.py c4      # K1 on a C4-shaped slice: 2097152 x 1024 bf16 as softmax C=2
    python tools/prof_run.py c5      # K5 on the C5 batch (512 problems 4096 x 128, T=8192, K=10)
    python tools/prof_run.py c3k3    # K3 at C3's D = 4096 on a 65536-row slice (T=20000)
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1803_03383_b200 as H  # noqa: E402


def main(which):
    import torch

    if which == "c2":
        X, lab = H.generate("softmax", 60000, 784, num_classes=10, dtype="f32", density=0.2, seed=0)
        obj = H.Objective(H.Dataset(X, labels=lab, num_classes=10), H.LossFamily.Softmax, 1e-4)
        steps = int(os.environ.get("PROF_T", 60000))
        rec = H.run_halp(obj, H.OptimizerConfig(algorithm=H.Algorithm.Halp, alpha=0.01, epochs=1, inner_steps=steps,
                                                bits=8, mu=2.5, seed=0))
        t = obj.timing()
        print("c2", rec.rows[-1].loss, "inner us/step", 1000 * t["inner_ms"] / steps, obj.plan(), t)
    elif which == "c3":
        X, y = H.generate("regression", 524288, 4096, dtype="f32", noise_sd=0.1, seed=3)
        obj = H.Objective(H.Dataset(X, targets=y), H.LossFamily.Squared, 0.0)
        obj.bench_full_gradient(2)
        ms = obj.bench_full_gradient(5)
        print("c3 slice ms", ms, "GB/s", 524288 * 4096 * 4 / ms / 1e6)
    elif which == "c4":
        X, lab = H.generate("logistic", 2097152, 1024, dtype="bf16", x_scale=1 / 32, seed=4)
        obj = H.Objective(H.Dataset(X, labels=lab, num_classes=2), H.LossFamily.Softmax, 1e-5)
        obj.bench_full_gradient(2)
        ms = obj.bench_full_gradient(5)
        print("c4 slice ms", ms, "GB/s", 2097152 * 1024 * 2 / ms / 1e6)
    elif which == "c5":
        import bench
        ms, nd, _ = bench.c5_batch(H, 0, 0, reps=1)
        print("c5 ms", ms, "diverged", nd)
    elif which == "c3k3":
        X, y = H.generate("regression", 65536, 4096, dtype="f32", noise_sd=0.1, seed=3)
        obj = H.Objective(H.Dataset(X, targets=y), H.LossFamily.Squared, 0.0)
        T = int(os.environ.get("PROF_T", 20000))
        H.run_halp(obj, H.OptimizerConfig(algorithm=H.Algorithm.Halp, alpha=5e-5, epochs=1, inner_steps=T, bits=16,
                                          mu=1.0, seed=0))
        t = obj.timing()
        print("c3k3 inner us/step", 1000 * t["inner_ms"] / T, obj.plan())
    torch.cuda.synchronize()


if __name__ == "__main__" and sys.argv[1] != "c1":
    main(sys.argv[1])


def c1(T=20000):
    X, y = H.generate("regression", 8192, 256, dtype="f32", noise_sd=0.01, seed=0)
    obj = H.Objective(H.Dataset(X, targets=y), H.LossFamily.Squared, 0.0)
    H.run_halp(obj, H.OptimizerConfig(algorithm=H.Algorithm.Halp, alpha=1e-3, epochs=1, inner_steps=T, bits=8,
                                      mu=1e3, seed=0))
    t = obj.timing()
    print("c1 inner us/step", 1000 * t["inner_ms"] / T, obj.plan())


if __name__ == "__main__" and sys.argv[1] == "c1":
    c1()
