# vertex-only LOCAL pass: parity + timing of count_all_vertices / VSamp cold on config 2
mkdir -p gpurun_out
echo skip-tests

python - <<'PY'
import time, numpy as np
import paper_1801_00338_b200 as B
l, r = B.synth_chung_lu(2_000_000, 5_000_000, 50_000_000, 2.1, 2.5, 2)
for rep in range(2):
    g = B.BipartiteGraph.from_edges(l, r)
    t = time.perf_counter(); v = B.count_all_vertices(g); tv = time.perf_counter() - t
    t = time.perf_counter(); e = B.count_all_edges(g); te = time.perf_counter() - t
    print("vertices-only", round(tv, 4), "edges after", round(te, 4), int(v.sum(dtype=np.uint64)), int(e.sum(dtype=np.uint64)))
    g.close()
    g = B.BipartiteGraph.from_edges(l, r)
    t = time.perf_counter(); res = B.run_estimator(g, B.Method.Vertex, iterations=1 << 20, seed=4); tc = time.perf_counter() - t
    print("vsamp cold", round(tc, 4), res.value, B.last_sample_path(g))
    g.close()
g = B.BipartiteGraph.from_edges(l, r)
B.profile_reset(); B.profile_enable(True)
B.count_all_vertices(g)
B.profile_enable(False)
snap = B.profile_snapshot()
for k, (ms, n) in sorted(snap.items(), key=lambda kv: -kv[1][0])[:14]:
    print(f"  {k:28s} {ms:8.3f} ms  x{n}")
PY
