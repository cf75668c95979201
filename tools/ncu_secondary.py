"""Drivers for the ncu captures of the secondary paths (SURVEY 8(d) "local / sampling /
sparsify"): run ONE of them under ncu with a kernel filter (tools/gpu/r2_ncu_secondary.sh).

  python tools/ncu_secondary.py local    # config 3: all-subject LOCAL pass (count_all_edges)
  python tools/ncu_secondary.py samples  # config 2: VSamp / ESamp per-sample kernels, WSamp
  python tools/ncu_secondary.py spar     # config 5: ESpar p = 0.01 and CSpar N = 100
"""
import os
import sys

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
import paper_1801_00338_b200 as B  # noqa: E402


def main():
    mode = sys.argv[1]
    if mode == "local":
        l, r = B.synth_chung_lu(1_000_000, 1_000_000, 20_000_000, 2.0, 2.0, 3, max_degree=500_000)
        g = B.BipartiteGraph.from_edges(l, r)
        e = B.count_all_edges(g)
        print("config 3 sum_e", int(e.sum(dtype="uint64")))
    elif mode == "samples":
        l, r = B.synth_chung_lu(2_000_000, 5_000_000, 50_000_000, 2.1, 2.5, 2)
        g = B.BipartiteGraph.from_edges(l, r)
        os.environ["BFLY_SAMPLE_PATH"] = "direct"
        for m, n in ((B.Method.Vertex, 1 << 12), (B.Method.Edge, 1 << 12), (B.Method.Wedge, 1 << 16)):
            c, _, _, _ = B.sample_batch(g, m, 4, 0, n)
            print(int(m), n, int(c.sum(dtype="uint64")))
    elif mode == "spar":
        l, r = B.synth_chung_lu(30_000_000, 60_000_000, 300_000_000, 2.2, 2.4, 5)
        g = B.BipartiteGraph.from_edges(l, r)
        del l, r
        print("espar 0.01", B.espar_count(g, 0.01, 5))
        print("cspar 100", B.cspar_count(g, 100, 5))
    else:
        raise SystemExit("mode: local | samples | spar")


if __name__ == "__main__":
    main()
