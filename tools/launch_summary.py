"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv) per kernel name.

  python tools/launch_summary.py gpurun_out/launches.csv > profiles/rNN_launches.md
Shows launches, total and mean duration and share of the summed kernel time. The launches
are serialised and cold-cache under ncu, so shares (not absolute times) are what compare
with bench.py's live per-kernel CUDA-event times.
"""
import csv
import io
import sys


def main():
    text = open(sys.argv[1]).read()
    start = text.find('"ID"')
    rows = list(csv.reader(io.StringIO(text[start:])))
    hdr = rows[0]
    kn, mn, mv, mu = (hdr.index(x) for x in ("Kernel Name", "Metric Name", "Metric Value",
                                             "Metric Unit"))
    agg = {}
    for r in rows[1:]:
        if len(r) != len(hdr) or r[mn] != "gpu__time_duration.sum":
            continue
        v = float(r[mv].replace(",", ""))
        v *= {"nsecond": 1e-6, "ns": 1e-6, "usecond": 1e-3, "us": 1e-3, "msecond": 1.0, "ms": 1.0,
              "second": 1e3, "s": 1e3}.get(r[mu], 1.0)
        name = r[kn].split("(")[0].replace("void ", "")
        a = agg.setdefault(name, [0, 0.0])
        a[0] += 1
        a[1] += v
    tot = sum(a[1] for a in agg.values()) or 1.0
    print(f"| kernel | launches | total ms | mean us | share |")
    print("|---|---|---|---|---|")
    for name, (n, t) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        print(f"| `{name[:90]}` | {n} | {t:.3f} | {1e3 * t / n:.1f} | {100 * t / tot:.1f}% |")
    print(f"\n{sum(a[0] for a in agg.values())} launches, {tot:.3f} ms summed kernel time")


if __name__ == "__main__":
    main()
