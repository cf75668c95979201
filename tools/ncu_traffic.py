"""Per-step DRAM traffic (dram__bytes_read.sum + dram__bytes_write.sum) of the counting
kernels from one `ncu --set full` capture, keyed by bench.py's kernel names; bench.py puts
the dominant kernel's figure in roofline.traffic.

  python tools/ncu_traffic.py gpurun_out/prof.ncu-rep > profiles/ncu_traffic.json
The capture must hold one step's launches of each kernel it reports (e.g. -k regex:... -c N
on the first exact count).
"""
import csv
import io
import json
import subprocess
import sys


def bench_name(kernel):
    if "k_dense_small" in kernel:
        return "hub_dense_small"
    if "k_dense_big" in kernel:
        return "hub_dense_big"
    src = "hub" if "HubSrc" in kernel else "exact" if "ExactSrc" in kernel else None
    if src is None:
        return None
    base = kernel.split("<")[0].split("::")[-1].replace("void ", "").strip()
    if base == "k_medium":
        wide = (src == "hub" and "DirectSplit" in kernel) or (src == "exact" and "Hash<14" in kernel)
        return f"{src}_medium_wide" if wide else f"{src}_medium"
    if base == "k_split":
        return f"{src}_heavy"
    if base == "k_small":  # small-A / small-B tables
        b = "BitHash<9>" in kernel or "Hash<10>" in kernel or "Hash<10," in kernel
        return f"{src}_small_b" if b else f"{src}_small"
    return {"k_tiny": f"{src}_tiny", "k_heavy": f"{src}_heavy"}.get(base)


def main():
    if sys.argv[1].endswith(".csv"):  # a raw page exported on the GPU box (--set full capture)
        out = open(sys.argv[1]).read()
    else:
        out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv", "--metrics",
                              "dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum"],
                             capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    res, cnt = {}, {}
    for r in rows[2:]:
        name = bench_name(r[hdr.index("Kernel Name")])
        if not name:
            continue
        b = 0.0
        for mname in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
            i = hdr.index(mname)
            b += float(r[i].replace(",", "")) * scale.get(units[i], 1)
        res[name] = res.get(name, 0.0) + b
        cnt[name] = cnt.get(name, 0) + 1
    # each bucket kernel launches once per count: a capture that ran into a second count
    # holds some names twice -> per-launch average
    res = {k: v / cnt[k] for k, v in res.items()}
    json.dump({"source": sys.argv[1].split("/")[-1], "dram_bytes_per_step": res,
               "launches_captured": cnt}, sys.stdout, indent=1)
    print()


if __name__ == "__main__":
    main()
