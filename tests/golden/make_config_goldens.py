"""Cached goldens for the BASELINE.json configs 2-5, from the UNMODIFIED reference.

Run in the build container (needs oracle/_ref/libbfly_ref.so, built by `make -C oracle`
from /root/reference/proj/src with the reference's Release flags). Each stage writes one
small JSON file under tests/golden/configs/, which tests/test_gpu_configs.py compares the
CUDA path against with `==` (integers and doubles alike). The edge lists are regenerated on
both sides from the same seeded synthetic generator (paper_1801_00338_b200/synth), so only
the outputs are committed.

  python tests/golden/make_config_goldens.py --stage c3_exact      # ~1 h, 1 core
  python tests/golden/make_config_goldens.py --stage c2_exact      # minutes, 1 core
  python tests/golden/make_config_goldens.py --stage c3_edges      # 8 threads
  python tests/golden/make_config_goldens.py --stage c4            # 8 threads
  python tests/golden/make_config_goldens.py --stage c5            # ~40 GB host RAM

Stages and the reference functions that produce them:
  c2_exact  exact_count (exact.cpp:45-47), single core, timed: config 2's CPU anchor
  c3_exact  exact_count on config 3, single core, timed
  c3_edges  count_per_edge (local.cpp:23-44) on 2^14 seeded canonical edge ids of config 3
  c4        run_estimator (sampling.cpp:206-278): WSamp with 2^20 iterations, VSamp / ESamp
            with 2^16 iterations (seed 4) + the first 1024 per-iteration values of each
  c5        edge_sparsify_estimate p in {0.01, 0.05, 0.1} and color_sparsify_estimate
            N in {10, 100} (sparsify.cpp:57-71), seed 5, on the 300M-edge config 5; the
            C restatement adds the retained butterfly and edge counts of each case
"""
import argparse
import json
import os
import platform
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

from oracle import oracle as O  # noqa: E402
import paper_1801_00338_b200 as B  # noqa: E402  (synthetic generators only)

OUT = os.path.join(ROOT, "tests", "golden", "configs")

CONFIGS = {
    2: dict(U=2_000_000, V=5_000_000, m=50_000_000, gu=2.1, gv=2.5, seed=2, cap=0),
    3: dict(U=1_000_000, V=1_000_000, m=20_000_000, gu=2.0, gv=2.0, seed=3, cap=500_000),
    5: dict(U=30_000_000, V=60_000_000, m=300_000_000, gu=2.2, gv=2.4, seed=5, cap=0),
}
C3_EDGE_SUBSET = 1 << 14
C4_ITERS = {0: 1 << 16, 1: 1 << 16, 2: 1 << 20}
C4_VALUES = 1024


def edges(cfg):
    c = CONFIGS[cfg]
    return B.synth_chung_lu(c["U"], c["V"], c["m"], c["gu"], c["gv"], c["seed"],
                            max_degree=c["cap"])


def c3_edge_ids(m):
    """2^14 canonical edge ids from the reference's own Rng (rng.hpp:36-58), seed 3."""
    rng = O.Rng(O.derive_seed(3, 0xE0))
    return np.array([rng.uniform_index(m) for _ in range(C3_EDGE_SUBSET)], np.uint64)


def host():
    model = ""
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    model = line.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    return {"cpu": model, "nproc": os.cpu_count(), "machine": platform.node()}


def write(stage, obj):
    os.makedirs(OUT, exist_ok=True)
    obj["generated_by"] = "tests/golden/make_config_goldens.py --stage " + stage
    obj["reference_build"] = "oracle/_ref/libbfly_ref.so (g++ -O3 -DNDEBUG)"
    with open(os.path.join(OUT, stage + ".json"), "w") as f:
        json.dump(obj, f, indent=1)
    print(json.dumps(obj)[:2000], flush=True)


def stage_exact(cfg):
    l, r = edges(cfg)
    t0 = time.perf_counter()
    ref = O.Ref(l, r)
    t_build = time.perf_counter() - t0
    st = ref.compute_stats()
    side, cl, cr = ref.choose_side()
    t0 = time.perf_counter()
    c = ref.exact_count()
    t_count = time.perf_counter() - t0
    write(f"c{cfg}_exact", {
        "config": cfg, "edges": int(len(l)), "sizes": list(ref.sizes()), "stats": st,
        "side": side, "cost_left": cl, "cost_right": cr, "butterflies": c,
        "from_edges_s": t_build, "exact_count_s": t_count, "threads": 1, "host": host()})


def stage_c3_edges():
    l, r = edges(3)
    ref = O.Ref(l, r)
    _, _, m = ref.sizes()
    ks = c3_edge_ids(m)
    t0 = time.perf_counter()
    got = ref.count_edges(ks, threads=os.cpu_count())
    write("c3_edges", {"config": 3, "edge_ids": [int(x) for x in ks],
                       "counts": [int(x) for x in got], "s": time.perf_counter() - t0,
                       "threads": os.cpu_count(), "host": host()})


def stage_c4():
    l, r = edges(2)
    ref = O.Ref(l, r)
    out = {"config": 4, "graph": "config 2", "seed": 4, "host": host(), "threads": os.cpu_count()}
    for method, name in ((2, "wsamp"), (1, "esamp"), (0, "vsamp")):
        it = C4_ITERS[method]
        t0 = time.perf_counter()
        est = ref.run_estimator(method, it, 4, threads=os.cpu_count())
        dt = time.perf_counter() - t0
        vals = [ref.iteration(method, 4, i) for i in range(C4_VALUES)]
        out[name] = {"iterations": it, "value": est["value"], "values_prefix": vals, "s": dt}
        print(name, it, est["value"], dt, flush=True)
    write("c4", out)


def stage_c5():
    l, r = edges(5)
    out = {"config": 5, "seed": 5, "edges": int(len(l)), "host": host()}
    t0 = time.perf_counter()
    ref = O.Ref(l, r)
    out["from_edges_s"] = time.perf_counter() - t0
    out["sizes"] = list(ref.sizes())
    for p in (0.01, 0.05, 0.1):
        t0 = time.perf_counter()
        out[f"espar_{p}"] = {"estimate": ref.edge_sparsify_estimate(p, 5),
                             "s": time.perf_counter() - t0}
        print(p, out[f"espar_{p}"], flush=True)
    for n in (10, 100):
        t0 = time.perf_counter()
        out[f"cspar_{n}"] = {"estimate": ref.color_sparsify_estimate(n, 5),
                             "s": time.perf_counter() - t0}
        print(n, out[f"cspar_{n}"], flush=True)
    del ref
    # the C restatement (pinned to the reference on the golden suites) adds the integer
    # retained counts; its estimate must equal the reference's
    o = O.Oracle(l, r)
    for p in (0.01, 0.05, 0.1):
        v, c, k = o.edge_sparsify_estimate(p, 5)
        assert v == out[f"espar_{p}"]["estimate"], (p, v, out[f"espar_{p}"])
        out[f"espar_{p}"].update(count=c, kept=k)
    for n in (10, 100):
        v, c, k = o.color_sparsify_estimate(n, 5)
        assert v == out[f"cspar_{n}"]["estimate"], (n, v, out[f"cspar_{n}"])
        out[f"cspar_{n}"].update(count=c, kept=k)
    write("c5", out)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--stage", required=True,
                    choices=["c2_exact", "c3_exact", "c3_edges", "c4", "c5"])
    a = ap.parse_args()
    if not O.ref_available():
        sys.exit("oracle/_ref/libbfly_ref.so missing: make -C oracle")
    if a.stage == "c2_exact":
        stage_exact(2)
    elif a.stage == "c3_exact":
        stage_exact(3)
    elif a.stage == "c3_edges":
        stage_c3_edges()
    elif a.stage == "c4":
        stage_c4()
    else:
        stage_c5()


if __name__ == "__main__":
    main()
