#!/usr/bin/env python
"""Benchmark: exact butterfly count on the BASELINE.json config-2 power-law graph on B200.

One STEP = the whole exact-count job on the synthetic edge list: device graph build
(first-seen dense ids, dedup, both CSRs, degree statistics, priority relabel) + the exact
wedge-aggregation kernels. Inputs: seeded synthetic Chung-Lu graph with the config-2
shape (|U|=2M, |V|=5M, 50M distinct edges, gamma 2.1 / 2.5, seed 2) -- a stand-in for the
paper's KONECT graphs, which are not in this container.

  value   : inputs resident in HBM (device edge list), device-timed with CUDA events.
  e2e     : through the public C-ABI with pinned HOST buffers: H2D of the edge list +
            build + count + D2H of the 8-byte result inside the timed region.
  unit    : wedges/s in the reference's work unit W_C = sum over the reference's centre
            side of C(d,2); the reference arm reports the same unit.
  roofline: dominant kernel, algorithmic bytes = 4 B per wedge element + 24 B per adjacency
            segment it processes, over its event-timed duration.

`--impl reference` times the reference CPU implementation (oracle/_ref, the unmodified
reference sources compiled here with their Release flags) on a bounded prefix sample of the
same edge list, with one replica per host core.

Secondary legs (SURVEY 8(d) "local / sampling / sparsify"), each with its own roofline and
reference CPU baseline:
  config4  VSamp / ESamp / WSamp on the config-2 graph: cold (first call on a fresh handle),
           warm, and the per-sample kernels forced (BFLY_SAMPLE_PATH=direct)
  config3  exact + all-subject per-edge counts (the LOCAL pass: 2 * B_exact bytes)
  config5  ESpar p in {0.01, 0.05, 0.1} and CSpar N in {10, 100} on the 300M-edge graph
           (8 m + 8 m' + B_exact(G') bytes)
  pairs    e2e through the reference signature: from_edges(const vector<pair<u64,u64>>&)
           + exact_count in the C++ facade
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CONFIG2 = dict(U=2_000_000, V=5_000_000, m=50_000_000, gamma_u=2.1, gamma_v=2.5, seed=2)
METRIC = "exact-count wedges/sec (reference work unit W_C) on the config-2 power-law graph"
UNIT = "wedges/s"
PEAKS_PATH = os.path.join(ROOT, "MEASURED_PEAKS.json")
BYTES_PER_WEDGE = 4
BYTES_PER_ENTRY = 24


_T0 = time.perf_counter()


def log(msg):
    """progress line on stderr (the JSON line alone goes to stdout)"""
    print(f"[bench {time.perf_counter() - _T0:7.1f}s] {msg}", file=sys.stderr, flush=True)


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true", help="profiling runs: skip the e2e leg")
    ap.add_argument("--no-samples", action="store_true", help="skip the config-4 estimator leg")
    ap.add_argument("--no-config3", action="store_true", help="skip the config-3 LOCAL leg")
    ap.add_argument("--no-config5", action="store_true", help="skip the config-5 sparsify leg")
    ap.add_argument("--no-pairs", action="store_true", help="skip the pair-types leg")
    ap.add_argument("--cpu-full", action="store_true",
                    help="also time the reference exact_count on the FULL config-2 graph on one "
                         "core (about 100 s; cached into profiles/)")
    ap.add_argument("--cpu-target-wedges", type=float, default=1.5e9,
                    help="reference wedges per CPU replica step (bounded sample size)")
    ap.add_argument("--scale", type=float, default=1.0, help="debug: shrink the config")
    return ap.parse_args()


def config(scale):
    c = dict(CONFIG2)
    if scale != 1.0:
        for k in ("U", "V", "m"):
            c[k] = max(16, int(c[k] * scale))
    return c


def gen_edges(c):
    import paper_1801_00338_b200 as B
    return B.synth_chung_lu(c["U"], c["V"], c["m"], c["gamma_u"], c["gamma_v"], c["seed"])


def ref_wedges(l, r):
    """W_C of the reference's exact_count on this edge list (exact.cpp:9-21, 23-43)."""
    dl = np.bincount(l).astype(np.float64)
    dr = np.bincount(r).astype(np.float64)
    dl, dr = dl[dl > 0], dr[dr > 0]
    cost_l, cost_r = float((dl * dl).sum()), float((dr * dr).sum())
    centre = dl if cost_l < cost_r else dr  # anchors Right iff cost_l < cost_r
    return int((centre * (centre - 1) / 2).sum()), ("right" if cost_l < cost_r else "left")


def traffic_path():
    """ncu DRAM bytes per kernel of the newest committed capture."""
    for name in ("r2_ncu_traffic.json", os.path.join("r1", "ncu_traffic.json")):
        p = os.path.join(ROOT, "profiles", name)
        if os.path.exists(p):
            return p
    return os.path.join(ROOT, "profiles", "ncu_traffic.json")


def peaks():
    try:
        with open(PEAKS_PATH) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured (MEASURED_PEAKS.json)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


# ---- distributed plumbing (one process per GPU; replicas of the single-GPU job) ----------
def dist_setup():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


class Dist:
    def __init__(self, ws, rank, local, backend):
        self.ws, self.rank, self.local = ws, rank, local
        self.dist = None
        if ws > 1:
            import torch.distributed as dist
            dist.init_process_group(backend)
            self.dist = dist

    def barrier(self):
        if self.dist:
            self.dist.barrier()

    def max(self, x):
        if not self.dist:
            return x
        import torch
        t = torch.tensor([x], dtype=torch.float64,
                         device="cuda" if self.dist.get_backend() == "nccl" else "cpu")
        self.dist.all_reduce(t, op=self.dist.ReduceOp.MAX)
        return float(t.item())

    def close(self):
        if self.dist:
            self.dist.destroy_process_group()


# ---- clocks sampler ------------------------------------------------------------------------
class Clocks:
    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu):
        self.gpu = gpu
        self.f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
        self.p = None

    def start(self):
        try:
            self.p = subprocess.Popen(["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.FIELDS}",
                                       "--format=csv,noheader,nounits", "-lms", "100"],
                                      stdout=self.f, stderr=subprocess.DEVNULL)
        except Exception:
            self.p = None

    def stop(self):
        if self.p:
            self.p.terminate()
            try:
                self.p.wait(timeout=5)
            except Exception:
                self.p.kill()
        self.f.flush()
        rows = []
        with open(self.f.name) as fh:
            for line in fh:
                parts = [x.strip() for x in line.split(",")]
                if len(parts) >= 9:
                    rows.append(parts)
        os.unlink(self.f.name)
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        sm = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in rows if r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[5 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons, "samples": len(rows)}


# ---- CPU reference arm --------------------------------------------------------------------
def cpu_sample(l, r, target):
    """Largest prefix of the (draw-ordered, deduped) edge list with W_C <= target."""
    lo, hi = 1000, len(l)
    while lo < hi:
        mid = (lo + hi + 1) // 2
        w, _ = ref_wedges(l[:mid], r[:mid])
        if w <= target:
            lo = mid
        else:
            hi = mid - 1
    return lo


def run_reference_steps(l, r, steps, warmup, target):
    """Reference exact_count (oracle/_ref) on a prefix sample; one replica per host core."""
    from oracle import oracle as O
    if not O.ref_available():
        raise RuntimeError("oracle/_ref/libbfly_ref.so missing")
    m_s = cpu_sample(l, r, target)
    ls, rs = np.ascontiguousarray(l[:m_s]), np.ascontiguousarray(r[:m_s])
    wc, side = ref_wedges(ls, rs)
    ref = O.Ref(ls, rs)
    cores = os.cpu_count() or 1
    times = []
    results = []
    for it in range(warmup + steps):
        out = [None] * cores
        t_end = [0.0] * cores

        def work(i):
            out[i] = ref.exact_count()
            t_end[i] = time.perf_counter()

        ths = [threading.Thread(target=work, args=(i,)) for i in range(cores)]
        t0 = time.perf_counter()
        for t in ths:
            t.start()
        for t in ths:
            t.join()
        dt = max(t_end) - t0
        if it >= warmup:
            times.append(dt)
        results.append(out[0])
    ms = 1e3 * statistics.mean(times)
    value = cores * wc / (ms / 1e3)
    sample = (f"prefix of the config-2 edge list: {m_s} edges, W_C={wc} reference wedges "
              f"(anchor side {('left' if side == 'left' else 'right')}), "
              f"{cores} concurrent exact_count replicas per step")
    return dict(value=value, ms=ms, cores=cores, sample=sample, count=results[-1], m=m_s, wc=wc)


# ---- secondary legs (SURVEY 8(d) local / sampling / sparsify) -------------------------------
WORKLOAD = "config2: exact butterfly count, build + count per step"


def workload_config(c):
    """The `config` both arms print (identical: same workload, same graph)."""
    return {"workload": WORKLOAD, "graph": c}


def host_cpu():
    model = ""
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    model = line.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    return {"cpu": model, "nproc": os.cpu_count()}


def b_exact(wc, m, n):
    """B_exact = 4 (W_C + 2m) + 8 (n + 2) bytes."""
    return 4 * (wc + 2 * m) + 8 * (n + 2)


def roof(byts, seconds, hbm, peak_kind, **kw):
    ach = byts / seconds / 1e9 if seconds > 0 else 0.0
    out = {"bound": "hbm", "achieved": ach, "peak": hbm, "unit": "GB/s", "frac": ach / hbm,
           "traffic": None, "algorithmic_bytes": int(byts), "seconds": seconds,
           "peak_kind": peak_kind}
    out.update(kw)
    return out


def timed_wall(f, reps):
    best, out = float("inf"), None
    for _ in range(reps):
        t0 = time.perf_counter()
        out = f()
        best = min(best, time.perf_counter() - t0)
    return out, best


def degrees_two_hop(g):
    """Degrees of both sides and two_hop[v] = sum of the degrees of N(v) (global order)."""
    loff, ladj, roff, radj = g.export()[:4]
    dl = np.diff(loff).astype(np.int64)
    dr = np.diff(roff).astype(np.int64)

    def seg_sum(vals, off):
        cs = np.concatenate([[0], np.cumsum(vals, dtype=np.int64)])
        return cs[off[1:].astype(np.int64)] - cs[off[:-1].astype(np.int64)]
    th = np.concatenate([seg_sum(dr[ladj.astype(np.int64)], loff),
                         seg_sum(dl[radj.astype(np.int64)], roff)])
    return loff, ladj, roff, radj, dl, dr, th


def sample_bytes(method, ids, ii, jj, csr):
    """SURVEY 8(d) per-sample algorithmic bytes of the reference algorithm, + 16 B offsets per
    list touched: VSamp 4 (d_v + sum_{u in N(v)} d_u); ESamp 4 (d_b + d_a + sum_{w in N(a)}
    d_w) with a the lower-degree endpoint (local.cpp:27-30); WSamp 4 (d_v + d_w) + 8
    ceil(log2(n+1)) prefix probes."""
    loff, ladj, roff, radj, dl, dr, th = csr
    L = len(dl)
    deg = np.concatenate([dl, dr])
    ids = ids.astype(np.int64)
    if method == 0:
        return int((4 * (deg[ids] + th[ids]) + 16 * (1 + deg[ids])).sum())
    if method == 1:
        lv = np.searchsorted(loff, ids, side="right") - 1
        rv = ladj[ids].astype(np.int64)
        da, db = dl[lv], dr[rv]
        swap = da > db  # a = lower-degree endpoint
        a_deg = np.where(swap, db, da)
        b_deg = np.where(swap, da, db)
        a_th = np.where(swap, th[L + rv], th[lv])
        return int((4 * (b_deg + a_deg + a_th) + 16 * (2 + a_deg)).sum())
    n = len(deg)
    c = ids
    left = c < L
    off = np.where(left, loff[np.minimum(c, L - 1)].astype(np.int64),
                   roff[np.maximum(c - L, 0)].astype(np.int64))
    v = np.where(left, L + ladj[off + ii], radj[off + ii])
    w = np.where(left, L + ladj[off + jj], radj[off + jj])
    probes = 8 * int(np.ceil(np.log2(n + 1)))
    return int((4 * (deg[v] + deg[w]) + probes + 32).sum())


def leg_config4(B, make_graph, hbm, peak_kind, ref, cores):
    """VSamp / ESamp / WSamp with 2^20 iterations on the config-2 graph (BASELINE config 4)."""
    out = {}
    ns = 1 << 20
    nd = 1 << 16
    cpu_iters = {0: 1 << 12, 1: 1 << 12, 2: 1 << 20}
    csr = None
    # process warm-up on a small graph: every estimator and the all-subject passes once, so the
    # "cold" figures below are the first call on a fresh HANDLE (what it has to build), not the
    # first call in the process (lazy kernel loading, the first growth of the row scratch)
    wl, wr = B.synth_chung_lu(60_000, 150_000, 1_000_000, 2.1, 2.5, 7)
    wg = B.BipartiteGraph.from_edges(wl, wr)
    for meth in (B.Method.Vertex, B.Method.Edge, B.Method.Wedge):
        B.run_estimator(wg, meth, iterations=1 << 12, seed=1)
    B.count_all_vertices(wg)
    B.count_all_edges(wg)
    wg.close()
    wg = B.BipartiteGraph.from_edges(wl, wr)
    B.count_all_vertices(wg)
    wg.close()
    for meth, name in ((B.Method.Vertex, "vsamp"), (B.Method.Edge, "esamp"),
                       (B.Method.Wedge, "wsamp")):
        log(f"config4 {name}: device legs")
        g = make_graph()
        t0 = time.perf_counter()
        est = B.run_estimator(g, meth, iterations=ns, seed=4)  # cold: builds what it needs
        cold = time.perf_counter() - t0
        path_cold = B.last_sample_path(g) if name != "wsamp" else "per-sample"
        _, warm = timed_wall(lambda: B.run_estimator(g, meth, iterations=ns, seed=4), 2)
        if csr is None:
            csr = degrees_two_hop(g)
        g.close()
        leg = {"samples": ns, "estimate": est.value, "cold_seconds": cold,
               "cold_samples_per_s": ns / cold, "cold_path": path_cold,
               "warm_seconds": warm, "warm_samples_per_s": ns / warm}
        # the per-sample kernels forced (BFLY_SAMPLE_PATH=direct), 2^16 iterations (all 2^20
        # for WSamp): one cold call on a fresh handle, then warm; roofline of the warm call
        nit = nd if name != "wsamp" else ns
        os.environ["BFLY_SAMPLE_PATH"] = "direct"
        try:
            g = make_graph()
            t0 = time.perf_counter()
            B.run_estimator(g, meth, iterations=nit, seed=4)
            dcold = time.perf_counter() - t0
            _, dwarm = timed_wall(lambda: B.run_estimator(g, meth, iterations=nit, seed=4), 2)
            _, ids, ii, jj = B.sample_batch(g, meth, 4, 0, nit)
            g.close()
        finally:
            del os.environ["BFLY_SAMPLE_PATH"]
        byts = sample_bytes(int(meth), ids, ii, jj, csr)
        leg.update({"direct_samples": nit, "direct_cold_seconds": dcold,
                    "direct_warm_seconds": dwarm, "direct_samples_per_s": nit / dwarm})
        leg["roofline"] = roof(byts, dwarm, hbm, peak_kind,
                               kernel=f"{name} per-sample kernels (BFLY_SAMPLE_PATH=direct)",
                               bytes_formula="SURVEY 8(d) per-sample bytes + 16 B per list")
        if ref is not None:
            it = cpu_iters[int(meth)]
            log(f"config4 {name}: reference run_estimator, {it} iterations")
            t0 = time.perf_counter()
            ref.run_estimator(int(meth), it, 4, threads=cores)
            dt = time.perf_counter() - t0
            leg["cpu_baseline"] = {"value": it / dt, "unit": "samples/s", "cores": cores,
                                   "kind": "reference",
                                   "sample": f"run_estimator({name}, iterations={it}, seed=4, "
                                             f"threads={cores}) on the full config-2 graph"}
        out[name] = leg
    return out


def leg_config3(B, hbm, peak_kind, cores, with_cpu):
    """BASELINE config 3: exact + per-edge counts of every edge (the LOCAL pass)."""
    t0 = time.perf_counter()
    l, r = B.synth_chung_lu(1_000_000, 1_000_000, 20_000_000, 2.0, 2.0, 3, max_degree=500_000)
    gen = time.perf_counter() - t0
    g = B.BipartiteGraph.from_edges(l, r)
    cnt, t_exact = timed_wall(lambda: B.exact_count(g), 3)
    st = B.compute_stats(g)
    est = B.last_exact_stats(g)
    g.close()
    # the GPU's own algorithmic bytes for the LOCAL pass: both walks over the wedges and
    # segments the priority kernels process (per-unit figures of DESIGN.md section 4)
    own_bytes = 2 * sum(BYTES_PER_WEDGE * est.bucket_wedges[q] + (24 if q < 6 else 14) *
                        est.bucket_entries[q] for q in range(12))
    wc, _ = ref_wedges(l, r)
    # LOCAL pass on a fresh handle (priority CSR with edge ids + the counting phase + copy)
    g = B.BipartiteGraph.from_edges(l, r)
    B.profile_reset()
    B.profile_enable(True)
    t0 = time.perf_counter()
    e = B.count_all_edges(g)
    t_local = time.perf_counter() - t0
    B.profile_enable(False)
    prof = B.profile_snapshot()
    g.close()
    assert int(e.sum(dtype=np.uint64)) == 4 * cnt
    phase = prof.get("count_phase", (0.0, 0))[0] / 1e3
    byts = 2 * b_exact(wc, st.m, st.n)
    leg = {"edges": int(st.m), "butterflies": cnt, "ref_wedges_W_C": wc, "gen_s": gen,
           "exact_seconds": t_exact, "exact_W_C_wedges_per_s": wc / t_exact,
           "all_edges_seconds": t_local, "all_edges_per_s": st.m / t_local,
           "local_phase_seconds": phase,
           "wedges_processed": est.wedges_processed,
           "roofline": roof(own_bytes, phase, hbm, peak_kind, kernel="LOCAL counting phase "
                            "(all-subject per-vertex + per-edge pass)",
                            bytes_formula="2 x (4 B per processed wedge + 24 / 14 B per start / "
                                          "hub segment): the kernels' own work"),
           "roofline_s8d_accounting": roof(byts, phase, hbm, peak_kind,
                                           kernel="LOCAL counting phase",
                                           bytes_formula="2 * B_exact (SURVEY 8(d)): the "
                                                         "reference's bytes for its W_C wedges "
                                                         "-- accounting, not bandwidth")}
    try:
        with open(os.path.join(ROOT, "tests", "golden", "configs", "c3_exact.json")) as f:
            gold = json.load(f)
        leg["reference_exact_single_core_cached"] = {
            "seconds": gold["exact_count_s"], "from_edges_seconds": gold["from_edges_s"],
            "host": gold["host"], "butterflies": gold["butterflies"],
            "note": "cached: tests/golden/make_config_goldens.py --stage c3_exact"}
    except (OSError, ValueError, KeyError):
        pass
    log("config3: device legs done")
    if with_cpu:
        from oracle import oracle as O
        log("config3: reference count_per_edge sample")
        ref = O.Ref(l, r)
        ks = np.random.default_rng(3).integers(0, st.m, 1 << 10).astype(np.uint64)
        t0 = time.perf_counter()
        want = ref.count_edges(ks, threads=cores)
        dt = time.perf_counter() - t0
        assert np.array_equal(want, e[ks])
        leg["cpu_baseline"] = {"value": len(ks) / dt, "unit": "edges/s", "cores": cores,
                               "kind": "reference",
                               "sample": f"count_per_edge on {len(ks)} seeded edges of config 3, "
                                         f"{cores} threads (all {st.m} edges on the GPU); "
                                         "counts equal"}
        del ref
    return leg


def leg_pairs(B, hbm, peak_kind):
    """butterfly pair types at scale (classify_pairs_at_scale) on configs
    1 and 3; the reference's classify_pairs enumerates all C(bfly, 2) pairs (config 3: about
    2.8e23) and is guarded to desk-size graphs, so there is no CPU figure at these sizes."""
    out = {}
    for name, gen in (("config1", lambda: B.synth_uniform(10_000, 5_000, 100_000, 1)),
                      ("config3", lambda: B.synth_chung_lu(1_000_000, 1_000_000, 20_000_000, 2.0,
                                                           2.0, 3, max_degree=500_000))):
        l, r = gen()
        g = B.BipartiteGraph.from_edges(l, r)
        st = B.compute_stats(g)
        B.count_all_edges(g)  # the LOCAL pass is cached on the handle; time the pair pass
        B.profile_reset()
        B.profile_enable(True)
        t0 = time.perf_counter()
        c = B.classify_pairs_at_scale(g)
        dt = time.perf_counter() - t0
        B.profile_enable(False)
        prof = B.profile_snapshot()
        g.close()
        # algorithmic bytes: every wedge of the pair pass reads one 4-byte key (plus 16 B per
        # adjacency segment, ~ 2 m segments): the wedge count is sum over vertices C(d, 2)
        byts = 4 * st.wedge_count + 16 * 2 * st.m
        out[name] = {"edges": int(st.m), "wedge_count": int(st.wedge_count), "seconds": dt,
                     "wedges_per_s": st.wedge_count / dt, "butterflies": c.bfly,
                     "pair_counts": {k: str(getattr(c, k)) for k in
                                     ("p_0v", "p_1v", "p_2v", "p_1e", "p_1w")},
                     "heavy_ms": prof.get("pair_heavy", (0.0, 0))[0],
                     "roofline": roof(byts, dt, hbm, peak_kind, kernel="pair-moment pass (wall)",
                                      bytes_formula="4 B per wedge + 16 B per segment")}
    return out


def leg_config5(B, hbm, peak_kind, with_cpu):
    """BASELINE config 5: ESpar / CSpar estimates on the 300M-edge graph."""
    t0 = time.perf_counter()
    l, r = B.synth_chung_lu(30_000_000, 60_000_000, 300_000_000, 2.2, 2.4, 5)
    gen = time.perf_counter() - t0
    log(f"config5: generated in {gen:.1f} s")
    t0 = time.perf_counter()
    g = B.BipartiteGraph.from_edges(l, r)
    build = time.perf_counter() - t0
    m = g.edge_count()
    B.sparsify_stats(g, collect=1)
    out = {"edges": m, "gen_s": gen, "build_seconds": build}
    cases = [("espar", 0.01), ("espar", 0.05), ("espar", 0.1), ("cspar", 10), ("cspar", 100)]
    for kind, a in cases:
        run = (lambda: B.espar_count(g, a, 5)) if kind == "espar" else \
              (lambda: B.cspar_count(g, a, 5))
        run()
        stt = B.sparsify_stats(g)  # collected on the warm call
        B.sparsify_stats(g, collect=0)
        (cnt, kept), wall = timed_wall(run, 3)
        B.sparsify_stats(g, collect=1)
        if kind == "espar":  # sparsify.cpp:36-41 / 43-55 (multiplication order kept)
            inv = 1.0 / a
            est = float(cnt) * inv * inv * inv * inv
        else:
            nf = float(a)
            est = float(cnt) * nf * nf * nf
        byts = 8 * m + 8 * kept + b_exact(stt["retained_wc"], kept, stt["retained_n"])
        out[f"{kind}_{a}"] = {
            "count": cnt, "kept": kept, "estimate": est, "seconds": wall,
            "input_edges_per_s": m / wall, "peeled_edges": stt["peeled_edges"],
            "sub_graph": [stt["sub_left"], stt["sub_right"]],
            "retained_W_C": stt["retained_wc"],
            "roofline": roof(byts, wall, hbm, peak_kind, kernel="sparsify-then-count (wall)",
                             bytes_formula="8 m + 8 m' + B_exact(G') (SURVEY 8(d))")}
    g.close()
    log("config5: device legs done")
    if with_cpu:
        from oracle import oracle as O
        log("config5: reference sparsifiers on a prefix")
        ms = 10_000_000  # bounded sample: a prefix of the config-5 edge list
        ref = O.Ref(np.ascontiguousarray(l[:ms]), np.ascontiguousarray(r[:ms]))
        for kind, a in (("espar", 0.01), ("cspar", 100)):
            t0 = time.perf_counter()
            (ref.edge_sparsify_estimate(a, 5) if kind == "espar"
             else ref.color_sparsify_estimate(a, 5))
            dt = time.perf_counter() - t0
            out[f"{kind}_{a}"]["cpu_baseline"] = {
                "value": ms / dt, "unit": "input edges/s", "cores": 1, "kind": "reference",
                "sample": f"{kind} {a} seed 5 on a {ms}-edge prefix of the config-5 list "
                          "(the reference sparsifiers are single-threaded)"}
        del ref
    return out


def cpu_full_config2(l, r):
    """Reference exact_count on the FULL config-2 graph, one core."""
    from oracle import oracle as O
    t0 = time.perf_counter()
    ref = O.Ref(l, r)
    t_build = time.perf_counter() - t0
    t0 = time.perf_counter()
    c = ref.exact_count()
    t_count = time.perf_counter() - t0
    return {"butterflies": c, "from_edges_seconds": t_build, "exact_count_seconds": t_count,
            "cores": 1, "host": host_cpu()}


# ---- main ----------------------------------------------------------------------------------
def main():
    a = parse()
    ws, rank, local = dist_setup()
    c = config(a.scale)
    if a.impl == "reference":
        return main_reference(a, ws, rank, local, c)
    return main_b200(a, ws, rank, local, c)


def main_reference(a, ws, rank, local, c):
    if rank != 0:
        return 0
    l, r = gen_edges(c)
    res = run_reference_steps(l, r, a.steps, a.warmup, a.cpu_target_wedges)
    line = {
        "metric": METRIC, "value": res["value"], "unit": UNIT, "n_gpus": a.gpus,
        "steps": a.steps, "warmup": a.warmup, "ms_per_step": res["ms"],
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "u32/u64",
        "data": "synthetic (seeded Chung-Lu, config-2 shape; prefix sample for the CPU)",
        "impl": "reference",
        "config": workload_config(c),
        "workload_stats": {"sample_edges": res["m"], "sample_ref_wedges": res["wc"],
                           "reference_build": "g++ -O3 -DNDEBUG (proj/CMakeLists.txt Release)",
                           "host": host_cpu()},
        "cpu_baseline": {"value": res["value"], "unit": UNIT, "cores": res["cores"],
                         "kind": "reference", "sample": res["sample"]},
        "e2e": {"value": res["value"], "unit": UNIT, "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line))
    return 0


def main_b200(a, ws, rank, local, c):
    import torch
    import paper_1801_00338_b200 as B

    torch.cuda.set_device(local)
    dist = Dist(ws, rank, local, "nccl")
    if not B.device_ok():
        raise SystemExit("CUDA device unusable: " + B._abi.last_error())
    t0 = time.time()
    l, r = gen_edges(c)
    gen_s = time.time() - t0
    m_in = len(l)
    wc, anchor = ref_wedges(l, r)

    stream = torch.cuda.Stream()
    B.set_stream(stream.cuda_stream)
    dl = torch.from_numpy(l.view(np.int32)).to("cuda")
    dr = torch.from_numpy(r.view(np.int32)).to("cuda")
    torch.cuda.synchronize()

    def step_device(stats=False):
        # one step = the user's calls: from_edges (device-resident ids) + exact_count. The work
        # statistics of the count (bucket sizes, W_C) are read outside the timed region
        g = B.BipartiteGraph.from_device(dl.data_ptr(), dr.data_ptr(), m_in)
        cnt = B.exact_count(g)
        st = None
        if stats:
            st = B.last_exact_stats(g)
            st.n, st.m = g.vertex_count(), g.edge_count()
            st.dense = B.last_dense_stats(g)
        g.close()
        return cnt, st

    # warm-up (also the parity reference value for this run)
    for _ in range(max(a.warmup, 3)):
        count, est = step_device(stats=True)
    dist.barrier()
    torch.cuda.synchronize()
    B.profile_reset()
    B.profile_enable(True)
    launches0 = B.launch_count()
    clk = Clocks(local)
    clk.start()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    counts = []
    for _ in range(a.steps):
        cnt, _ = step_device()
        counts.append(cnt)
    e1.record(stream)
    torch.cuda.synchronize()
    clocks = clk.stop()
    B.profile_enable(False)
    prof = B.profile_snapshot()
    launches = (B.launch_count() - launches0) // a.steps
    ms = e0.elapsed_time(e1) / a.steps
    dist.barrier()
    ms = dist.max(ms)
    assert all(x == count for x in counts), "count changed between steps"

    # end to end through the C-ABI with pinned host buffers
    e2e_ms = float("nan")
    if not a.no_e2e:
        hl = torch.from_numpy(l.view(np.int32)).pin_memory()
        hr = torch.from_numpy(r.view(np.int32)).pin_memory()
        hl_np, hr_np = hl.numpy().view(np.uint32), hr.numpy().view(np.uint32)
        for _ in range(2):
            g = B.BipartiteGraph.from_edges(hl_np, hr_np)
            B.exact_count(g)
            g.close()
        dist.barrier()
        torch.cuda.synchronize()
        f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        per_step = []
        f0.record(stream)
        for _ in range(a.steps):
            t0 = time.perf_counter()
            g = B.BipartiteGraph.from_edges(hl_np, hr_np)  # H2D of both id arrays inside
            cnt = B.exact_count(g)                          # D2H of the 8-byte count
            g.close()
            per_step.append(1e3 * (time.perf_counter() - t0))
            assert cnt == count
        f1.record(stream)
        torch.cuda.synchronize()
        e2e_ms = dist.max(f0.elapsed_time(f1) / a.steps)
        print(f"e2e host ms per step: {[round(x, 1) for x in per_step]}", file=sys.stderr)

    # e2e through the reference signature: from_edges(const vector<pair<u64,u64>>&) +
    # exact_count in the C++ facade (pageable 16-byte pairs; wall clock per call)
    e2e_pairs = None
    if not a.no_e2e:
        pms, pcnt = B.time_from_pairs(l, r, reps=max(3, min(a.steps, 5)))
        assert pcnt == count
        pm = statistics.median(pms[1:]) if len(pms) > 1 else pms[0]
        e2e_pairs = {"value": ws * wc / (pm / 1e3), "unit": UNIT, "ms_per_step": pm,
                     "ms_all": pms, "h2d_bytes_per_step": 8 * m_in, "d2h_bytes_per_step": 8,
                     "host_input_bytes": 16 * m_in,
                     "call": "bfly::BipartiteGraph::from_edges(const std::vector<std::pair<"
                             "uint64_t, uint64_t>>&) + bfly::exact_count (wall clock)"}

    hbm, peak_kind = peaks()
    cores = os.cpu_count() or 1
    secondary = {}
    with_cpu = rank == 0 and ws == 1 and not a.no_cpu_baseline
    if not a.no_samples:
        ref2 = None
        if with_cpu:
            from oracle import oracle as O
            log("config4: reference from_edges (config 2)")
            ref2 = O.Ref(l, r)
        secondary["config4_estimators"] = leg_config4(
            B, lambda: B.BipartiteGraph.from_device(dl.data_ptr(), dr.data_ptr(), m_in), hbm,
            peak_kind, ref2, cores)
        del ref2
        g = B.BipartiteGraph.from_device(dl.data_ptr(), dr.data_ptr(), m_in)
        # Method::FastEdge: 2^16 iterations x the default 1000 probes
        nf = 1 << 16
        B.run_estimator(g, B.Method.FastEdge, iterations=nf, seed=4)
        res, dt = timed_wall(lambda: B.run_estimator(g, B.Method.FastEdge, iterations=nf, seed=4), 2)
        secondary["fastedge"] = {"samples_per_s": nf / dt, "seconds": dt, "estimate": res.value,
                                 "samples": nf, "repeats": 1000, "ids": "device",
                                 "probes_per_s": nf * 1000 / dt}
        # edge-list text: serialise the config-2 graph, parse it back
        t0 = time.perf_counter()
        text = g.serialize()
        t_ser = time.perf_counter() - t0
        t0 = time.perf_counter()
        h = B.BipartiteGraph.from_text(text)
        t_load = time.perf_counter() - t0
        assert B.exact_count(h) == count
        secondary["edge_list_text"] = {"bytes": len(text), "serialize_s": t_ser,
                                       "load_s": t_load,
                                       "load_gb_per_s": len(text) / t_load / 1e9,
                                       "note": "load = host->device copy + parse + from_edges"}
        h.close()
        del text
        g.close()
    log("fastedge / text legs done")
    if not a.no_config3:
        log("config3 leg")
        secondary["config3_local"] = leg_config3(B, hbm, peak_kind, cores, with_cpu)
    if not a.no_pairs:
        log("pair-types leg")
        secondary["pair_types"] = leg_pairs(B, hbm, peak_kind)
    if not a.no_config5:
        log("config5 leg")
        del dl, dr
        torch.cuda.empty_cache()
        secondary["config5_sparsify"] = leg_config5(B, hbm, peak_kind, with_cpu)

    # roofline of the dominant counting kernel
    # bucket index, bytes per adjacency segment (start path: padj + (start, length) = 12 B
    # + 8 B task offsets amortised -> 24 B; hub path: hlen + hpst + offset = 14 B); every key
    # element is 4 B
    # (buckets of aggregate.cuh: tiny, small-A, small-B, medium, medium-wide, heavy/split;
    # [0,6) start path, [6,12) hub path)
    kern = {"exact_tiny": ((0,), 24), "exact_small": ((1,), 24), "exact_small_b": ((2,), 24),
            "exact_medium": ((3,), 24), "exact_medium_wide": ((4,), 24),
            "exact_heavy": ((5,), 24), "hub_tiny": ((6,), 14), "hub_small": ((7,), 14),
            "hub_small_b": ((8,), 14),
            "hub_medium": ((9,), 14), "hub_medium_wide": ((10,), 14), "hub_heavy": ((11,), 14)}
    per_kernel = {}
    for name, (qs, bpe) in kern.items():
        if name in prof:
            tot_ms, n_launch = prof[name]
            byts = sum(BYTES_PER_WEDGE * est.bucket_wedges[q] + bpe * est.bucket_entries[q]
                       for q in qs)
            per_kernel[name] = dict(ms_per_step=tot_ms / a.steps, launches_per_step=n_launch / a.steps,
                                    bytes_per_step=byts,
                                    gbs=byts / (tot_ms / a.steps / 1e3) / 1e9 if tot_ms else 0.0)
    # dense top-hub kernels (csrc/hubdense.cuh): per adjacency entry of a task one 4-byte
    # neighbour id and that neighbour's mask row (4 * words bytes); their wedges are counted
    # from the masks, so they add no key bytes
    dn = est.dense
    for name, ents in (("hub_dense_small", dn["entries"] - dn["big_entries"]),
                       ("hub_dense_big", dn["big_entries"])):
        if name in prof and dn["words"]:
            tot_ms, n_launch = prof[name]
            byts = ents * (4 + 4 * dn["words"])
            per_kernel[name] = dict(ms_per_step=tot_ms / a.steps, launches_per_step=n_launch / a.steps,
                                    bytes_per_step=byts,
                                    gbs=byts / (tot_ms / a.steps / 1e3) / 1e9 if tot_ms else 0.0)
    dom = max(per_kernel, key=lambda k: per_kernel[k]["ms_per_step"]) if per_kernel else None
    roof = None
    if "count_phase" in prof and per_kernel:
        # The bucket kernels of both counting paths run concurrently on side streams (one
        # counting phase), so each kernel's own event span overlaps the others'; the dominant
        # unit of work is the phase: its algorithmic bytes (sum over the buckets, per-unit
        # figures of DESIGN.md section 4) over its wall time.
        ph_ms = prof["count_phase"][0] / a.steps
        byts = sum(v["bytes_per_step"] for v in per_kernel.values())
        traffic, tsrc = None, None
        try:
            tj = json.load(open(traffic_path()))
            tb = tj["dram_bytes_per_step"]
            if all(k in tb for k in per_kernel):
                traffic = sum(tb[k] for k in per_kernel)
            tsrc = os.path.relpath(traffic_path(), ROOT) + " (" + tj.get("source", "?") + \
                "), summed over the phase's kernels"
        except (OSError, ValueError, KeyError):
            pass
        ach = byts / (ph_ms / 1e3) / 1e9
        roof = {"bound": "hbm", "achieved": ach, "peak": hbm, "unit": "GB/s", "frac": ach / hbm,
                "physical_frac": (traffic / (ph_ms / 1e3) / 1e9 / hbm) if traffic else None,
                "physical_note": "ncu DRAM bytes of the phase's kernels over the phase time",
                "traffic": traffic, "traffic_unit": "bytes per step (DRAM read+write, ncu)",
                "traffic_source": tsrc, "algorithmic_bytes": byts,
                "kernel": "count_phase (" + ", ".join(sorted(per_kernel)) + ")",
                "peak_kind": peak_kind, "kernel_ms_per_step": ph_ms,
                "kernel_share_of_step": ph_ms / ms,
                "note": "bucket kernels overlap on side streams; per-kernel spans in 'kernels'"}
        dom = None
    if dom:
        d = per_kernel[dom]
        ach = d["gbs"]
        traffic, tsrc = None, None
        try:  # DRAM bytes of this kernel from a committed ncu --set full capture
            tj = json.load(open(traffic_path()))
            traffic = tj["dram_bytes_per_step"].get(dom)
            tsrc = os.path.relpath(traffic_path(), ROOT) + " (" + tj.get("source", "?") + ")"
        except (OSError, ValueError, KeyError):
            pass
        roof = {"bound": "hbm", "achieved": ach, "peak": hbm, "unit": "GB/s", "frac": ach / hbm,
                "traffic": traffic, "traffic_unit": "bytes per launch (DRAM read+write, ncu)",
                "traffic_source": tsrc, "algorithmic_bytes": d["bytes_per_step"],
                "kernel": dom, "peak_kind": peak_kind,
                "kernel_ms_per_step": d["ms_per_step"],
                "kernel_share_of_step": d["ms_per_step"] / ms}
    # SURVEY 8(d)'s whole-count figure: the reference's algorithmic bytes for this graph,
    # B_exact = 4 (W_C + 2m) + 8 (n + 2), over the wedge-aggregation kernels' time per step
    # (wall time of the two counting phases -- the bucket kernels of a phase overlap on side
    # streams, so the sum of their own durations overstates it -- else that sum)
    kern_sum_ms = sum(v["ms_per_step"] for v in per_kernel.values())
    phases = [prof["count_phase"]] if "count_phase" in prof else \
        [prof[p] for p in ("hub_phase", "exact_phase") if p in prof]
    agg_ms = sum(p[0] for p in phases) / a.steps if phases else kern_sum_ms
    b_exact = 4 * (wc + 2 * est.m) + 8 * (est.n + 2)
    roof_s8d = {"formula": "B_exact = 4*(W_C + 2m) + 8*(n + 2) bytes (SURVEY 8(d))",
                "note": "ACCOUNTING, not bandwidth: the reference's bytes for its own W_C "
                        "wedges; the GPU processes wedges_processed of them",
                "bytes": b_exact, "aggregation_ms_per_step": agg_ms,
                "achieved": b_exact / (agg_ms / 1e3) / 1e9 if agg_ms else 0.0, "peak": hbm,
                "unit": "GB/s",
                "frac": b_exact / (agg_ms / 1e3) / 1e9 / hbm if agg_ms else 0.0,
                "frac_of_whole_step": b_exact / (ms / 1e3) / 1e9 / hbm,
                "time_source": "counting-phase wall time (events around both paths' kernels)" if phases
                               else "sum of kernel durations",
                "kernel_duration_sum_ms_per_step": kern_sum_ms,
                "kernels": sorted(per_kernel)}
    all_kernels = {k: {"ms_per_step": v[0] / a.steps, "launches_per_step": v[1] / a.steps}
                   for k, v in sorted(prof.items(), key=lambda kv: -kv[1][0])}

    value = ws * wc / (ms / 1e3)
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws, "steps": a.steps,
        "warmup": a.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "u32 ids / u64 counts",
        "data": "synthetic (seeded Chung-Lu, BASELINE config-2 shape)",
        "config": workload_config(c),
        "workload_stats": {"edges": m_in, "butterflies": count,
                   "ref_wedges_W_C": wc, "reference_anchor_side": anchor,
                   "wedges_processed": est.wedges_processed,
                   "hub_starts_k": est.bucket_starts[12],
                   "dense_top_hubs": est.dense,
                   "buckets": "[0:6] start path tiny/small-A/small-B/medium/medium-wide/heavy, "
                              "[6:12] hub path (heavy = entry-range split)",
                   "bucket_tasks": est.bucket_starts[:12], "bucket_wedges": est.bucket_wedges,
                   "bucket_entries": est.bucket_entries,
                   "l2_policy": "inputs (400 MB edge list, >1 GB CSRs) exceed the 126 MB L2",
                   "parallelism": f"replicas x{ws}", "host_gen_s": round(gen_s, 2)},
        "e2e": {"value": ws * wc / (e2e_ms / 1e3), "unit": UNIT, "ms_per_step": e2e_ms,
                "h2d_bytes_per_step": 8 * m_in, "d2h_bytes_per_step": 8,
                "call": "Python API: BipartiteGraph.from_edges(pinned u32 arrays) + exact_count"},
        "e2e_reference_signature": e2e_pairs,
        "roofline": roof,
        "roofline_exact_s8d": roof_s8d,
        "secondary": secondary,
        "kernels": all_kernels,
        "gpu_launches": int(launches),
        "clocks": clocks,
    }
    if rank == 0 and ws == 1 and not a.no_cpu_baseline:
        try:
            res = run_reference_steps(l, r, 1, 0, a.cpu_target_wedges)
            line["cpu_baseline"] = {"value": res["value"], "unit": UNIT, "cores": res["cores"],
                                    "kind": "reference", "sample": res["sample"],
                                    "host": host_cpu()}
        except Exception as ex:  # reported, not fatal
            line["cpu_baseline"] = {"value": None, "unit": UNIT, "cores": 0, "kind": "reference",
                                    "sample": f"unavailable: {ex}"}
        # the same-config anchor (exact on 1 core): the reference exact_count on
        # the FULL config-2 graph, one core -- measured here with --cpu-full (about 100 s),
        # else the cached measurement
        full = None
        cache = os.path.join(ROOT, "profiles", "r2_cpu_full_config2.json")
        if a.cpu_full:
            full = cpu_full_config2(l, r)
            full["cached"] = False
            with open(cache, "w") as f:
                json.dump(full, f, indent=1)
        else:
            for path in (cache, os.path.join(ROOT, "tests", "golden", "configs", "c2_exact.json")):
                try:
                    with open(path) as f:
                        d = json.load(f)
                    full = {"butterflies": d["butterflies"],
                            "from_edges_seconds": d.get("from_edges_seconds", d.get("from_edges_s")),
                            "exact_count_seconds": d.get("exact_count_seconds",
                                                         d.get("exact_count_s")),
                            "cores": 1, "host": d["host"], "cached": os.path.relpath(path, ROOT)}
                    break
                except (OSError, ValueError, KeyError):
                    continue
        if full:
            assert full["butterflies"] == count
            full["value"] = wc / full["exact_count_seconds"]
            full["unit"] = UNIT
            full["e2e_value"] = wc / (full["exact_count_seconds"] + full["from_edges_seconds"])
            full["note"] = ("reference exact_count on the full config-2 graph, single core "
                            "(the reference is single-threaded, exact.cpp:23-43)")
            line["cpu_baseline_full_single_core"] = full
    if rank == 0:
        print(json.dumps(line))
    B.set_stream(0)
    dist.close()
    return 0


if __name__ == "__main__":
    sys.exit(main())
