"""Aggregate an ncu source page (cuda,sass) to per-source-line instructions and stall samples.

  ncu -i rep --page source --csv --print-source cuda,sass > page.csv
  python tools/ncu_lines.py page.csv [top]
"""
import csv
import sys


def main():
    rows = list(csv.reader(open(sys.argv[1])))
    top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
    agg, hdr, cur_file = {}, None, ""
    for r in rows:
        if not r:
            continue
        if r[0] == "File Path":
            cur_file = r[1].split("/")[-1]
            continue
        if r[0] == "Line No":
            hdr = r
            continue
        if hdr is None or not r[0].isdigit():
            continue
        try:
            ie = hdr.index("Instructions Executed")
            st = hdr.index("Warp Stall Sampling (All Samples)")
        except ValueError:
            continue
        if len(r) != len(hdr):
            continue  # source text with unescaped quotes
        key = (cur_file, int(r[0]), r[1].strip()[:90])
        a = agg.setdefault(key, [0.0, 0.0])
        a[0] += float(r[ie]) if r[ie] not in ("", "-") else 0.0
        a[1] += float(r[st]) if r[st] not in ("", "-") else 0.0
    ti = sum(v[0] for v in agg.values()) or 1
    ts = sum(v[1] for v in agg.values()) or 1
    print(f"total warp instructions {ti:.3e}, stall samples {ts:.0f}")
    for k, v in sorted(agg.items(), key=lambda kv: -kv[1][1])[:top]:
        print(f"{100 * v[1] / ts:5.1f}% samp {100 * v[0] / ti:5.1f}% inst  {k[0]}:{k[1]}  {k[2]}")


if __name__ == "__main__":
    main()
