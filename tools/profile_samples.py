"""Per-sample kernel timing on the config-2 graph (BFLY_SAMPLE_PATH=direct): wall time and the
per-kernel device time of VSamp / ESamp batches of growing size, to find slow paths.

  python tools/profile_samples.py [max_log2]
"""
import json
import os
import sys
import time

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
import paper_1801_00338_b200 as B  # noqa: E402


def main():
    top = int(sys.argv[1]) if len(sys.argv) > 1 else 12
    os.environ["BFLY_SAMPLE_PATH"] = "direct"
    l, r = B.synth_chung_lu(2_000_000, 5_000_000, 50_000_000, 2.1, 2.5, 2)
    g = B.BipartiteGraph.from_edges(l, r)
    for meth in (B.Method.Vertex, B.Method.Edge):
        for lg in range(8, top + 1, 2):
            n = 1 << lg
            B.sample_batch(g, meth, 4, 0, 64)  # warm
            B.profile_reset()
            B.profile_enable(True)
            t0 = time.perf_counter()
            B.sample_batch(g, meth, 4, 0, n)
            dt = time.perf_counter() - t0
            B.profile_enable(False)
            snap = B.profile_snapshot()
            top_k = sorted(snap.items(), key=lambda kv: -kv[1][0])[:10]
            print(json.dumps({"method": int(meth), "samples": n, "seconds": dt,
                              "path": B.last_sample_path(g),
                              "kernels": {k: [round(v[0], 3), v[1]] for k, v in top_k}}),
                  flush=True)
            if dt > 60:
                break
    g.close()


if __name__ == "__main__":
    main()
