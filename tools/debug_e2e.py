"""Debug: host-timed phases of the e2e path (from_edges on pinned host buffers + count)."""
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
print("pinned:", hl.is_pinned(), hr.is_pinned())
hl_np, hr_np = hl.numpy().view(np.uint32), hr.numpy().view(np.uint32)
dl = torch.from_numpy(l.view(np.int32)).cuda(); dr = torch.from_numpy(r.view(np.int32)).cuda()
for it in range(4):
    for mode in ("host", "device"):
        torch.cuda.synchronize(); t0 = time.perf_counter()
        g = (B.BipartiteGraph.from_edges(hl_np, hr_np) if mode == "host"
             else B.BipartiteGraph.from_device(dl.data_ptr(), dr.data_ptr(), len(l)))
        torch.cuda.synchronize(); t1 = time.perf_counter()
        c = B.exact_count(g)
        torch.cuda.synchronize(); t2 = time.perf_counter()
        g.close()
        torch.cuda.synchronize(); t3 = time.perf_counter()
        print(f"{mode:6s} build {1e3*(t1-t0):7.1f} ms  count {1e3*(t2-t1):7.1f} ms  free {1e3*(t3-t2):6.1f} ms  c={c}")
free, total = torch.cuda.mem_get_info(); print("free GB", free/1e9)
