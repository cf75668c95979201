"""CPU (gloo, world_size 2): the multi-process plumbing bench.py uses for N>1 -- barrier
and max-over-ranks of the per-rank step time; ranks run independent replicas and only
exchange the 8-byte timing scalar."""
import os
import socket

import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, ws, port, out):
    import sys
    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE=str(ws), LOCAL_RANK=str(rank))
    import bench
    d = bench.Dist(ws, rank, rank, "gloo")
    d.barrier()
    out[rank] = d.max(10.0 + rank)
    d.close()


def test_dist_max_over_ranks():
    port = _free_port()
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(2, port, out), nprocs=2, join=True)
    assert out[0] == out[1] == 11.0
