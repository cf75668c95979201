"""Time the pair-type pass (pairs.cu: classify_pairs_at_scale) on growing graphs, with the
per-kernel device time of the moment pass; prints one JSON line per graph.

  python tools/profile_pairs.py [max_config]     (1: config 1 only ... 3: up to config 3)
"""
import json
import sys
import time

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
import paper_1801_00338_b200 as B  # noqa: E402

GRAPHS = [
    ("config1", lambda: B.synth_uniform(10_000, 5_000, 100_000, 1), 1),
    ("chung_lu_2M", lambda: B.synth_chung_lu(200_000, 500_000, 2_000_000, 2.1, 2.5, 7), 2),
    ("config3", lambda: B.synth_chung_lu(1_000_000, 1_000_000, 20_000_000, 2.0, 2.0, 3,
                                         max_degree=500_000), 3),
    ("config2", lambda: B.synth_chung_lu(2_000_000, 5_000_000, 50_000_000, 2.1, 2.5, 2), 4),
]


def main():
    top = int(sys.argv[1]) if len(sys.argv) > 1 else 3
    for name, gen, lvl in GRAPHS:
        if lvl > top:
            continue
        l, r = gen()
        g = B.BipartiteGraph.from_edges(l, r)
        st = B.compute_stats(g)
        B.exact_count(g)
        B.count_all_edges(g)  # the LOCAL pass is cached on the handle; time the pair pass alone
        B.profile_reset()
        B.profile_enable(True)
        t0 = time.perf_counter()
        c = B.classify_pairs_at_scale(g)
        dt = time.perf_counter() - t0
        B.profile_enable(False)
        snap = B.profile_snapshot()
        top_k = sorted(snap.items(), key=lambda kv: -kv[1][0])[:8]
        print(json.dumps({"graph": name, "edges": int(st.m), "wedge_count": int(st.wedge_count),
                          "seconds": dt, "wedges_per_s": st.wedge_count / dt,
                          "counts": [str(x) for x in c.as_tuple()],
                          "kernels_ms": {k: round(v[0], 3) for k, v in top_k}}), flush=True)
        g.close()


if __name__ == "__main__":
    main()
