"""Summarise ncu reports (.ncu-rep) into a markdown table for profiles/.

Per kernel: duration, DRAM bytes and throughput (vs the measured HBM peak), L2 hit rate,
L1 hit rate, shared-memory atomics (count, per-SM rate), warps active, issue active and the
top stall reasons -- the counters the north star asks every design choice to cite.

  python tools/ncu_summary.py gpurun_out/prof_*.ncu-rep > profiles/r1_ncu_summary.md
  python tools/ncu_summary.py gpurun_out/r2_local.raw.csv ...   (raw pages exported on the box)
"""
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
METRICS = {
    "dur_ms": "gpu__time_duration.sum",
    "dram_rd": "dram__bytes_read.sum",
    "dram_wr": "dram__bytes_write.sum",
    "dram_pct": "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "l2_hit": "lts__t_sector_hit_rate.pct",
    "l1_hit": "l1tex__t_sector_hit_rate.pct",
    "smem_atom": "l1tex__data_pipe_lsu_wavefronts_mem_shared_op_atom.sum",
    "warps": "sm__warps_active.avg.pct_of_peak_sustained_active",
    "issue": "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "inst": "smsp__inst_executed.sum",
    "regs": "launch__registers_per_thread",
    "smem_limit": "launch__occupancy_limit_shared_mem",
}
STALLS = ["long_scoreboard", "short_scoreboard", "barrier", "wait", "mio_throttle",
          "lg_throttle", "math_pipe_throttle", "no_instruction", "branch_resolving", "membar"]


def to_bytes(v, unit):
    f = float(v)
    return f * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "B": 1, "KB": 1e3,
                "MB": 1e6, "GB": 1e9}.get(unit, 1)


def rows(rep):
    if rep.endswith(".csv"):  # a raw page exported on the GPU box (ncu -i rep --page raw --csv)
        out = open(rep).read()
    else:
        out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                             text=True).stdout
    r = list(csv.reader(io.StringIO(out)))
    return r[0], r[1], r[2:]


def main():
    peak = 6535.7
    try:
        peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"]
    except Exception:
        pass
    print("| report | kernel | ms | DRAM GB (rd+wr) | DRAM GB/s (%% of %.0f) | L2 hit | L1 hit | "
          "smem atomics (G/s) | warps active | issue active | top stalls (cycles/issue) |" % peak)
    print("|---|---|---|---|---|---|---|---|---|---|---|")
    for rep in sys.argv[1:]:
        hdr, units, data = rows(rep)
        col = {k: hdr.index(v) for k, v in METRICS.items() if v in hdr}
        for r in data:
            name = r[hdr.index("Kernel Name")]
            short = name.split("(")[0].replace("void ", "").replace("bflyd::agg::", "")[:60]
            ms = float(r[col["dur_ms"]]) * {"usecond": 1e-3, "us": 1e-3, "nsecond": 1e-6,
                                             "ns": 1e-6}.get(units[col["dur_ms"]], 1.0)
            rd = to_bytes(r[col["dram_rd"]], units[col["dram_rd"]])
            wr = to_bytes(r[col["dram_wr"]], units[col["dram_wr"]])
            gbs = (rd + wr) / (ms * 1e-3) / 1e9 if ms else 0.0
            atom = float(r[col["smem_atom"]]) if "smem_atom" in col else 0.0
            stalls = []
            for s in STALLS:
                key = f"smsp__average_warps_issue_stalled_{s}_per_issue_active.ratio"
                if key in hdr:
                    stalls.append((float(r[hdr.index(key)] or 0), s))
            stalls.sort(reverse=True)
            top = ", ".join(f"{s} {v:.1f}" for v, s in stalls[:3])
            print(f"| {os.path.basename(rep)} | `{short}` | {ms:.3f} | {(rd + wr) / 1e9:.2f} | "
                  f"{gbs:.0f} ({100 * gbs / peak:.1f}%) | {float(r[col['l2_hit']]):.1f}% | "
                  f"{float(r[col['l1_hit']]):.1f}% | {atom / (ms * 1e-3) / 1e9 if ms else 0:.1f} | "
                  f"{float(r[col['warps']]):.1f}% | {float(r[col['issue']]):.1f}% | {top} |")


if __name__ == "__main__":
    main()
