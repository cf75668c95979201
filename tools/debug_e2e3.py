"""Debug: which phase of the host-buffer path spikes (BFLY_TRACE=1 marks, 12 iterations)."""
import sys, time
import numpy as np
import torch
sys.path.insert(0, ".")
import paper_1801_00338_b200 as B

l, r = B.synth_chung_lu(2_000_000, 5_000_000, 50_000_000, 2.1, 2.5, 2)
stream = torch.cuda.Stream()
B.set_stream(stream.cuda_stream)
hl = torch.from_numpy(l.view(np.int32)).pin_memory()
hr = torch.from_numpy(r.view(np.int32)).pin_memory()
hl_np, hr_np = hl.numpy().view(np.uint32), hr.numpy().view(np.uint32)
for it in range(12):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    print(f"=== iter {it}", file=sys.stderr, flush=True)
    g = B.BipartiteGraph.from_edges(hl_np, hr_np)
    c = B.exact_count(g)
    g.close()
    torch.cuda.synchronize()
    print(f"iter {it}: {1e3*(time.perf_counter()-t0):.1f} ms", flush=True)
