#!/bin/bash
# A/B of environment variants on the GPU box: tools/ab_env.sh "NAME=VAR=value" ...
# (NAME=- for no extra variable). Prints the step time and the top kernels of each.
mkdir -p gpurun_out
for spec in "$@"; do
  name="${spec%%=*}"; kv="${spec#*=}"
  if [ "$kv" = "-" ]; then envs=(); else envs=("$kv"); fi
  env "${envs[@]}" python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-samples > gpurun_out/ab_$name.json 2> gpurun_out/ab_$name.err || { echo "$name failed"; tail -5 gpurun_out/ab_$name.err; continue; }
  python - "$name" <<'PY'
import json, sys
n = sys.argv[1]
d = json.load(open(f"gpurun_out/ab_{n}.json"))
ks = sorted(d["kernels"].items(), key=lambda x: -x[1]["ms_per_step"])[:18]
print(n, "step", round(d["ms_per_step"], 3), "e2e", round(d["e2e"]["ms_per_step"], 3), "agg", round(d["roofline_exact_s8d"]["aggregation_ms_per_step"], 3),
      {k: round(v["ms_per_step"], 3) for k, v in ks})
PY
done
