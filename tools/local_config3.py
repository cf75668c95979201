import sys; sys.path.insert(0,'/root/repo')
import paper_1801_00338_b200 as B
l, r = B.synth_chung_lu(1_000_000, 1_000_000, 20_000_000, 2.0, 2.0, 3, max_degree=500_000)
g = B.BipartiteGraph.from_edges(l, r)
B.count_all_edges(g)
