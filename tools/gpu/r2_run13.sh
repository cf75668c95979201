# Dense top-hub kernels timed alone (BFLY_AGG_CONCURRENT=0: bucket kernels serialised).
mkdir -p gpurun_out
for spec in off:BFLY_HUB_DENSE=0 w1:BFLY_HUB_DENSE_W=1 w4:BFLY_HUB_DENSE_W=4 w8:BFLY_HUB_DENSE_W=8 w32:BFLY_HUB_DENSE_W=32; do
  name="${spec%%:*}"; kv="${spec#*:}"
  env BFLY_AGG_CONCURRENT=0 "$kv" python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-samples --no-config3 --no-config5 --no-e2e --no-pairs > gpurun_out/r13_$name.json 2> gpurun_out/r13_$name.err || { echo "$name failed"; tail -5 gpurun_out/r13_$name.err; continue; }
  python - "$name" <<'PY'
import json, sys
n = sys.argv[1]
d = json.load(open(f"gpurun_out/r13_{n}.json"))
ks = sorted(d["kernels"].items(), key=lambda x: -x[1]["ms_per_step"])[:24]
print(n, "step", round(d["ms_per_step"], 3), "agg", round(d["roofline_exact_s8d"]["aggregation_ms_per_step"], 3),
      {k: round(v["ms_per_step"], 3) for k, v in ks if k.startswith(("hub_", "exact_", "count"))})
print("   keys", d["workload_stats"]["bucket_wedges"][6:], "tasks", d["workload_stats"]["bucket_tasks"][6:])
PY
done 2>&1 | tee gpurun_out/r13_ab.txt
