"""Generate tests/golden/golden.npz from the UNMODIFIED reference compiled here.

Run in the build container (needs oracle/_ref/libbfly_ref.so, built by `make -C oracle`
from /root/reference/proj/src). The output pins both the C restatement (oracle/) and the
CUDA path (tests/test_gpu_*.py) to the reference's own results on the same inputs:

  python tests/golden/make_golden.py
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

from oracle import oracle as O  # noqa: E402
import paper_1801_00338_b200 as B  # noqa: E402  (synthetic generators only)

out = {}


def put(key, arr):
    if isinstance(arr, list) and arr and all(isinstance(x, (int, np.integer)) for x in arr):
        out[key] = np.array([int(x) for x in arr], dtype=np.uint64)
    else:
        out[key] = np.asarray(arr)


def graph_case(tag, l, r, local=True, samples=True):
    ref = O.Ref(l, r)
    L, R, m = ref.sizes()
    st = ref.compute_stats()
    put(f"{tag}/edges", np.stack([l.astype(np.uint64), r.astype(np.uint64)]))
    put(f"{tag}/sizes", [L, R, m])
    put(f"{tag}/exact", [ref.exact_count(), ref.exact_count_side(0), ref.exact_count_side(1)])
    side, cl, cr = ref.choose_side()
    put(f"{tag}/side", [side])
    put(f"{tag}/costs", [cl, cr])
    put(f"{tag}/stats_u64", [st["n"], st["left"], st["right"], st["m"], st["wedge_count"],
                             st["max_degree"]])
    loff, ladj, roff, radj, lids, rids = ref.csr()
    put(f"{tag}/loff", loff)
    put(f"{tag}/ladj", ladj)
    put(f"{tag}/roff", roff)
    put(f"{tag}/radj", radj)
    put(f"{tag}/lids", lids)
    put(f"{tag}/rids", rids)
    if local:
        put(f"{tag}/vertex", ref.count_all_vertices())
        put(f"{tag}/edge", ref.count_edges())
    if samples:
        for method in (0, 1, 2):
            vals = [ref.iteration(method, 7, i) for i in range(64)]
            put(f"{tag}/iter{method}", vals)
            est = ref.run_estimator(method, 257, 99, threads=4)
            put(f"{tag}/est{method}", [est["value"]])
            mom = ref.run_estimator(method, 0, 7, groups=5, group_size=20, threads=2)
            put(f"{tag}/mom{method}", [mom["value"]] + mom["per_group_means"])
        # Method::FastEdge (sampling.cpp:125-147), fewer repeats than the default 1000
        put(f"{tag}/fast_iter", [ref.fast_iteration(50, 7, i) for i in range(64)])
        put(f"{tag}/est3", [ref.run_estimator(3, 257, 99, threads=4, repeats=100)["value"]])
        mom = ref.run_estimator(3, 0, 7, groups=5, group_size=20, threads=2, repeats=30)
        put(f"{tag}/mom3", [mom["value"]] + mom["per_group_means"])
        for seed in (0, 1, 42):
            put(f"{tag}/espar{seed}", [ref.edge_sparsify_estimate(0.5, seed),
                                       ref.edge_sparsify_estimate(0.3, seed)])
            put(f"{tag}/cspar{seed}", [ref.color_sparsify_estimate(2, seed),
                                       ref.color_sparsify_estimate(3, seed)])
        run = ref.sparsify_run(0, p=0.4, seed=99, trials=8)
        put(f"{tag}/sprun_edge", [run["value"]] + run["per_group_means"])
        run = ref.sparsify_run(1, colors=2, seed=99, trials=8)
        put(f"{tag}/sprun_color", [run["value"]] + run["per_group_means"])


def text_cases():
    """Crafted edge-list texts (comments, blanks, CR/LF, tabs, extra tokens, leading zeros,
    overflow, signs, vertical tab) plus a noisy text of a seeded power-law graph."""
    cases = [b"% bip\n1 2\n2 3\n\n# c\n  3 1 extra tokens\n\t4\t5\r\n", b"1 2\n3\n",
             b"1 2\n  \n x 5\n", b"% only\n\n", b"",
             b"18446744073709551615 0\n18446744073709551616 1\n", b"1 2\n\x0b\n", b"5 -3\n",
             b"+5 3\n", b"007 8\n1 2", b"\r\n1 2\r\n", b"1 2 \x0c 3\n", b"1\t\t2\n#\n%\n3 4",
             b"1 2\n2 1\n1 2\n2 2\n1 1\n", b"4294967296 7\n7 4294967296\n", b"1 2x\n", b"1 2\n\n\n9"]
    rng = np.random.default_rng(5)
    l, r = B.synth_chung_lu(3000, 4000, 20000, 2.1, 2.4, 6)
    parts = [b"% bip generated\n"]
    for a, b in zip(l.tolist(), r.tolist()):
        c = rng.integers(0, 40)
        if c == 0:
            parts.append(b"# comment\n")
        elif c == 1:
            parts.append(b"   \t\r\n")
        sep = [b" ", b"\t", b" \t "][rng.integers(0, 3)]
        end = [b"\n", b"\r\n", b" trailing\n"][rng.integers(0, 3)]
        lead = b"0" * int(rng.integers(0, 2))
        parts.append(lead + str(a * 7 + 1).encode() + sep + str(b * 3 + 5).encode() + end)
    cases.append(b"".join(parts))
    return cases


def main():
    # reference fixture graphs (tests/support/fixtures.hpp:31-85)
    from tests import helpers as H
    for name, (l, r) in zip(["k22", "k32", "k24", "k33", "two_k22", "cycle6", "star15", "path4"],
                            H.named_suite()):
        graph_case(f"named_{name}", l, r)
    for idx, (l, r) in enumerate(O.random_suite_edges(12, 12, 12, [0.2, 0.5, 0.8], 5000)):
        graph_case(f"rand5000_{idx}", l, r)
    # random_bipartite(40, 40, 0.2, 21) of tests/test_sampling.cpp:141-161
    l, r = O.random_bipartite_edges(40, 40, 0.2, 21)
    graph_case("rb40", l, r)
    # uniform config-1-shaped graph at reduced size (per-vertex and per-edge pinned)
    l, r = B.synth_uniform(1000, 500, 8000, 1)
    graph_case("uniform_small", l, r)
    # power-law (Chung-Lu) graph at reduced size, exact + local
    l, r = B.synth_chung_lu(3000, 6000, 30000, 2.1, 2.5, 2)
    graph_case("chunglu_small", l, r, samples=True)
    l, r = B.synth_chung_lu(2000, 2000, 20000, 2.0, 2.0, 3, max_degree=500)
    graph_case("chunglu_cap", l, r, samples=False)
    # config 1 exactly (exact count + all per-vertex counts; edges regenerated by synth)
    l, r = B.synth_uniform(10000, 5000, 100000, 1)
    ref = O.Ref(l, r)
    put("config1/exact", [ref.exact_count()])
    put("config1/vertex", ref.count_all_vertices())
    put("config1/edge_sum", [int(ref.count_edges().sum(dtype=np.uint64))])
    put("config1/edges_sha", [np.frombuffer(
        __import__("hashlib").sha256(l.tobytes() + r.tobytes()).digest(), np.uint8)])
    # edge-list text (graph.cpp:75-112): reference outcome for crafted and noisy texts
    for i, t in enumerate(text_cases()):
        put(f"text{i}/bytes", np.frombuffer(t, np.uint8) if t else np.zeros(0, np.uint8))
        res = O.Ref.load_text(t)
        if res[0] == "ok":
            put(f"text{i}/serialized", np.frombuffer(res[1].serialize(), np.uint8))
            put(f"text{i}/exact", [res[1].exact_count()])
        elif res[0] == "parse":
            put(f"text{i}/parse", np.frombuffer(res[1].encode(), np.uint8))
            put(f"text{i}/line", [res[2]])
        else:
            put(f"text{i}/empty", np.frombuffer(res[1].encode(), np.uint8))
    # rng pins: mix64 / derive_seed / first draw of Rng::stream(seed, i)
    xs = [0, 1, 2, 3, 42, 2 ** 63, 2 ** 64 - 1]
    lib = O.ref_lib()
    put("rng/mix64", [lib.ref_mix64(x) for x in xs])
    put("rng/derive", [lib.ref_derive_seed(x, y) for x in xs for y in xs])
    put("rng/stream_first", [lib.ref_rng_stream_first(s, i) for s in (0, 4, 99) for i in range(16)])
    path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden.npz")
    np.savez_compressed(path, **out)
    print("wrote", path, len(out), "arrays", os.path.getsize(path), "bytes")


if __name__ == "__main__":
    main()
