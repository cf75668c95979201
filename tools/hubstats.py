import sys; sys.path.insert(0, '.')
import paper_1801_00338_b200 as B
import torch
l, r = B.synth_chung_lu(2_000_000, 5_000_000, 50_000_000, 2.1, 2.5, 2)
g = B.BipartiteGraph.from_edges(l, r)
print(B.exact_count(g))
