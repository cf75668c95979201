"""Run the BASELINE.json configs 1-5 on one B200 and check them (prints one JSON line per
config). Checks: the oracle (CPU restatement, host threads) where it finishes in seconds
to minutes, and size-independent identities everywhere (sum_v = sum_e = 4*bfly, sample
subsets against oracle per-sample values, sparsify counts against oracle counts).

  python tools/run_configs.py [--configs 1,2,3,4,5] [--oracle-exact-config2]
"""
import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_1801_00338_b200 as B  # noqa: E402
from oracle import oracle as O  # noqa: E402


def timed(f, reps=1):
    f()  # warm
    t = time.perf_counter()
    for _ in range(reps):
        out = f()
    return out, (time.perf_counter() - t) / reps


def config1():
    l, r = B.synth_uniform(10000, 5000, 100000, 1)
    g = B.BipartiteGraph.from_edges(l, r)
    o = O.Oracle(l, r)
    c, t = timed(lambda: B.exact_count(g), 5)
    v, tv = timed(lambda: B.count_all_vertices(g), 3)
    want = o.exact_count()
    return {"config": 1, "edges": len(l), "butterflies": c, "oracle": want, "exact_ok": c == want,
            "vertex_ok": bool(np.array_equal(v, o.count_all_vertices())),
            "sum_v_ok": int(v.sum()) == 4 * c, "exact_s": t, "all_vertices_s": tv}


def config2(oracle_exact):
    l, r = B.synth_chung_lu(2_000_000, 5_000_000, 50_000_000, 2.1, 2.5, 2)
    g = B.BipartiteGraph.from_edges(l, r)
    c, t = timed(lambda: B.exact_count(g), 3)
    res = {"config": 2, "edges": len(l), "butterflies": c, "exact_s": t,
           "exact_left": B.exact_count_side(g, B.Side.Left),
           "exact_right": B.exact_count_side(g, B.Side.Right)}
    if oracle_exact:
        t0 = time.perf_counter()
        o = O.Oracle(l, r)
        res["oracle"] = o.exact_count()
        res["oracle_s"] = time.perf_counter() - t0
        res["exact_ok"] = res["oracle"] == c
    return res, g, l, r


def config3():
    l, r = B.synth_chung_lu(1_000_000, 1_000_000, 20_000_000, 2.0, 2.0, 3, max_degree=500_000)
    g = B.BipartiteGraph.from_edges(l, r)
    c, t = timed(lambda: B.exact_count(g), 2)
    # all-edge local counts are cached per graph: time the first call on a fresh handle
    # (priority CSR with edge ids + the LOCAL pass + the 160 MB copy back)
    g2 = B.BipartiteGraph.from_edges(l, r)
    t0 = time.perf_counter()
    e = B.count_all_edges(g2)
    te = time.perf_counter() - t0
    g2.close()
    v = B.count_all_vertices(g)
    o = O.Oracle(l, r)
    ks = np.random.default_rng(3).integers(0, o.m, 4096).astype(np.uint64)
    t0 = time.perf_counter()
    want = o.count_edges_subset(ks)
    to = time.perf_counter() - t0
    return {"config": 3, "edges": len(l), "max_degree": int(max(np.bincount(l).max(),
                                                                 np.bincount(r).max())),
            "butterflies": c, "exact_s": t, "all_edges_s": te,
            "sum_e_ok": int(e.sum(dtype=np.uint64)) == 4 * c,
            "sum_v_ok": int(v.sum(dtype=np.uint64)) == 4 * c,
            "edge_subset_ok": bool(np.array_equal(e[ks], want)), "oracle_subset_s": to,
            "edge_subset_n": len(ks)}


def config4(g, l, r):
    out = {"config": 4}
    o = O.Oracle(l, r)
    prefix, total = o.build_wedge_index()
    for method, name in ((0, "vsamp"), (1, "esamp"), (2, "wsamp")):
        t0 = time.perf_counter()
        est = B.run_estimator(g, B.Method(method), iterations=1 << 20, seed=4, threads=16)
        dt = time.perf_counter() - t0
        out[f"{name}_estimate"] = est.value
        out[f"{name}_s"] = dt
        out[f"{name}_samples_per_s"] = (1 << 20) / dt
        out[f"{name}_path"] = B.last_sample_path(g) if method < 2 else "per-sample"
        # sample-by-sample parity on the first 512 iterations against the oracle
        ids, ii, jj = B.sample_ids(g, B.Method(method), 4, 0, 512)
        oid, oii, ojj = o.sample_draws(method, 4, 512, prefix, total)
        same_ids = bool(np.array_equal(ids, oid) and np.array_equal(ii, oii) and
                        np.array_equal(jj, ojj))
        if method == 0:
            got, want = B.count_vertices(g, ids), o.count_vertices_subset(ids)
        elif method == 1:
            got, want = B.count_edges(g, ids), o.count_edges_subset(ids)
        else:
            got = B.wedge_common_minus_1(g, ids, ii, jj)
            loff, ladj, roff, radj = o.csr()[:4]
            want = []
            for q in range(len(ids)):
                cg = int(ids[q])
                s = 0 if cg < o.L else 1
                ci = cg if s == 0 else cg - o.L
                adj = ladj[loff[ci]:loff[ci + 1]] if s == 0 else radj[roff[ci]:roff[ci + 1]]
                want.append(o.wedge_common_minus_1(s, int(adj[ii[q]]), int(adj[jj[q]])))
            want = np.array(want, np.uint64)
        out[f"{name}_ids_ok"] = same_ids
        out[f"{name}_counts_ok"] = bool(np.array_equal(got, want))
    return out


def config5(oracle):
    t0 = time.perf_counter()
    l, r = B.synth_chung_lu(30_000_000, 60_000_000, 300_000_000, 2.2, 2.4, 5)
    gen = time.perf_counter() - t0
    g = B.BipartiteGraph.from_edges(l, r)
    out = {"config": 5, "edges": len(l), "gen_s": gen}
    o = O.Oracle(l, r) if oracle else None
    for p in (0.01, 0.05, 0.1):
        (c, k), t = timed(lambda: B.espar_count(g, p, 5), 1)
        inv = 1.0 / p
        out[f"espar_{p}"] = {"count": c, "kept": k, "estimate": float(c) * inv * inv * inv * inv,
                             "s": t}
        if o is not None and p == 0.01:
            _, oc, ok = o.edge_sparsify_estimate(p, 5)
            out[f"espar_{p}"]["oracle_ok"] = (oc, ok) == (c, k)
    for n in (10, 100):
        (c, k), t = timed(lambda: B.cspar_count(g, n, 5), 1)
        out[f"cspar_{n}"] = {"count": c, "kept": k, "estimate": float(c) * n * n * n, "s": t}
        if o is not None and n == 100:
            _, oc, ok = o.color_sparsify_estimate(n, 5)
            out[f"cspar_{n}"]["oracle_ok"] = (oc, ok) == (c, k)
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="1,2,3,4,5")
    ap.add_argument("--oracle-exact-config2", action="store_true")
    ap.add_argument("--oracle-config5", action="store_true")
    a = ap.parse_args()
    want = {int(x) for x in a.configs.split(",")}
    g2 = None
    if 1 in want:
        print(json.dumps(config1()), flush=True)
    if 2 in want or 4 in want:
        res, g2, l2, r2 = config2(a.oracle_exact_config2)
        if 2 in want:
            print(json.dumps(res), flush=True)
    if 3 in want:
        print(json.dumps(config3()), flush=True)
    if 4 in want:
        print(json.dumps(config4(g2, l2, r2)), flush=True)
    if 5 in want:
        g2 = None
        print(json.dumps(config5(a.oracle_config5)), flush=True)


if __name__ == "__main__":
    main()
