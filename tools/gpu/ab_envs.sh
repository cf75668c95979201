#!/bin/bash
# A/B of environment settings on the config-2 bench: tools/gpu/ab_envs.sh TAG "name:VAR=1 VAR2=2" ...
# (name:- for no variable). Prints step / counting-phase time and the counting kernels.
TAG=$1; shift
mkdir -p gpurun_out
for spec in "$@"; do
  name="${spec%%:*}"; kv="${spec#*:}"
  [ "$kv" = "-" ] && kv="BFLY_NOP=1"
  env $kv python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-samples --no-config3 --no-config5 --no-e2e --no-pairs > gpurun_out/${TAG}_$name.json 2> gpurun_out/${TAG}_$name.err || { echo "$name failed"; tail -5 gpurun_out/${TAG}_$name.err; continue; }
  python - "$TAG" "$name" <<'PY'
import json, sys
t, n = sys.argv[1:3]
d = json.load(open(f"gpurun_out/{t}_{n}.json"))
ks = sorted(d["kernels"].items(), key=lambda x: -x[1]["ms_per_step"])[:40]
print(n, "step", round(d["ms_per_step"], 3), "agg", round(d["roofline_exact_s8d"]["aggregation_ms_per_step"], 3), "bfly", d["workload_stats"]["butterflies"],
      {k: round(v["ms_per_step"], 3) for k, v in ks if k.startswith(("hub_", "exact_"))})
PY
done 2>&1 | tee -a gpurun_out/${TAG}_ab.txt
