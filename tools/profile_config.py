"""Per-kernel device time (library profiling registry) of one graph build, exact count and
all-subject local counts on a BASELINE config graph; for finding the next hot kernel.

  python tools/profile_config.py [2|3|5]     (5: the sparsify-then-count cases of config 5)
"""
import sys
import time

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
import paper_1801_00338_b200 as B  # noqa: E402

SHAPES = {2: (2_000_000, 5_000_000, 50_000_000, 2.1, 2.5, 2, 0),
          3: (1_000_000, 1_000_000, 20_000_000, 2.0, 2.0, 3, 500_000),
          5: (30_000_000, 60_000_000, 300_000_000, 2.2, 2.4, 5, 0)}


def sparsify_cases(l, r):
    g = B.BipartiteGraph.from_edges(l, r)
    cases = [("espar", 0.01), ("espar", 0.05), ("espar", 0.1), ("cspar", 10), ("cspar", 100)]
    run = {"espar": lambda a: B.espar_count(g, a, 5), "cspar": lambda a: B.cspar_count(g, a, 5)}
    for kind, a in cases:  # warm: reid, pool growth
        run[kind](a)
    B.profile_reset()
    for kind, a in cases:
        best = 1e9
        for _ in range(3):
            t = time.perf_counter()
            out = run[kind](a)
            best = min(best, time.perf_counter() - t)
        B.profile_reset()
        B.profile_enable(True)
        run[kind](a)
        B.profile_enable(False)
        show(f"{kind} {a}: {out} best wall {best * 1e3:.2f} ms")


def show(tag):
    snap = B.profile_snapshot()
    tot = sum(v[0] for v in snap.values())
    print(f"== {tag}: {tot:.2f} ms in {len(snap)} kernel names")
    for k, (ms, n) in sorted(snap.items(), key=lambda kv: -kv[1][0])[:25]:
        print(f"  {k:28s} {ms:8.3f} ms  x{n}")
    B.profile_reset()


def main():
    cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 3
    U, V, m, gu, gv, seed, cap = SHAPES[cfg]
    l, r = B.synth_chung_lu(U, V, m, gu, gv, seed, max_degree=cap) if cap else \
        B.synth_chung_lu(U, V, m, gu, gv, seed)
    if cfg == 5:
        return sparsify_cases(l, r)
    for rep in range(2):  # second round is warm
        g = B.BipartiteGraph.from_edges(l, r)
        B.exact_count(g)
        B.count_all_edges(g)
        g.close()
    B.profile_reset()
    B.profile_enable(True)
    t = time.perf_counter()
    g = B.BipartiteGraph.from_edges(l, r)
    show(f"config {cfg} build")
    c = B.exact_count(g)
    show(f"config {cfg} exact ({c})")
    B.count_all_edges(g)
    show(f"config {cfg} all-subject local")
    print("wall", time.perf_counter() - t)


if __name__ == "__main__":
    main()
