"""Regenerate tests/golden/*.json from the reference tree (run in the build
container only; /root/reference does not exist on the GPU box).

Sources (reference outputs and known-answer tests, not source code):
  proj/out/regression_floor/{halp-8,halp-16,svrg,lp-svrg-8,lp-svrg-16,sgd,lp-sgd-8,lp-sgd-16}_seed{1..5}.csv  golden traces
  proj/out/regression_floor/manifest.json                        final values (+ verbatim copy)
  proj/specs/regression_floor.json                               their spec
  proj/tests/test_rng.cpp:14-31                                  RNG KATs
"""
import csv
import json
import os
import re

REF = "/root/reference/proj"
OUT = os.path.dirname(os.path.abspath(__file__))


def traces():
    spec = json.load(open(f"{REF}/specs/regression_floor.json"))
    man = json.load(open(f"{REF}/out/regression_floor/manifest.json"))
    runs = {}
    for name in ("halp-8", "halp-16", "svrg", "lp-svrg-8", "lp-svrg-16", "sgd", "lp-sgd-8", "lp-sgd-16"):
        for seed in range(1, 6):
            fn = f"{REF}/out/regression_floor/{name}_seed{seed}.csv"
            rows = list(csv.DictReader(open(fn)))
            # keep the exact decimal strings (shortest round-trip, text.hpp:12-19)
            runs[f"{name}_seed{seed}"] = rows
    finals = {f"{r['name']}_seed{r['seed']}": r for r in man["runs"] if r["name"] in ("halp-8", "halp-16", "svrg", "lp-svrg-8", "lp-svrg-16", "sgd", "lp-sgd-8", "lp-sgd-16")}
    json.dump({"source": "proj/out/regression_floor (lpopt run --spec specs/regression_floor.json)",
               "spec": spec, "traces": runs, "manifest": finals},
              open(os.path.join(OUT, "regression_floor.json"), "w"), indent=1)


def rng_kats():
    src = open(f"{REF}/tests/test_rng.cpp").read()
    block = src[src.index('TEST_CASE("generator output is frozen")'):src.index('TEST_CASE("equal seeds')]
    kats = []
    cur = None
    for line in block.splitlines():
        m = re.search(r"QuantRng (\w)\((\d+), (\d+)\)", line)
        if m:
            cur = {"var": m.group(1), "seed": int(m.group(2)), "stream": int(m.group(3)), "u64": [], "uniform": []}
            kats.append(cur)
            continue
        m = re.search(r"next_u64\(\) == (\d+)ULL", line)
        if m:
            cur["u64"].append(int(m.group(1)))
        m = re.search(r"next_uniform\(\) == doctest::Approx\(([0-9.e-]+)\)", line)
        if m:
            cur["uniform"].append(float(m.group(1)))
    json.dump({"source": "proj/tests/test_rng.cpp:14-31", "kats": kats},
              open(os.path.join(OUT, "rng_kats.json"), "w"), indent=1)


def manifest_copy():
    """the reference's run_experiment manifest, byte for byte (harness.cpp:358-375)"""
    src = open(f"{REF}/out/regression_floor/manifest.json").read()
    with open(os.path.join(OUT, "regression_floor_manifest.json"), "w") as f:
        f.write(src)


if __name__ == "__main__":
    traces()
    manifest_copy()
    rng_kats()
    print("fixtures written to", OUT)
