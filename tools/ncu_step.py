"""One config-2 graph build + exact count (cold), for ncu captures of single kernels:
  ncu --set full -k regex:<kernel> -c 1 python tools/ncu_step.py
"""
import sys

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
import paper_1801_00338_b200 as B  # noqa: E402

l, r = B.synth_chung_lu(2_000_000, 5_000_000, 50_000_000, 2.1, 2.5, 2)
g = B.BipartiteGraph.from_edges(l, r)
print(B.exact_count(g))
g.close()
