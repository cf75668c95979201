#!/bin/bash
# A/B of compile-time variants on the GPU box: tools/ab.sh "NAME=-DFLAG=1" "NAME2=-DFLAG=2" ...
# Each variant rebuilds the engine with EXTRA flags, runs the config-2 bench (no CPU baseline,
# no estimator leg) and prints the step time and the top kernels.
mkdir -p gpurun_out
for spec in "$@"; do
  name="${spec%%=*}"; flags="${spec#*=}"
  [ "$flags" = "-" ] && flags=""  # (a bare "-" would make nvcc read its source from stdin)
  touch paper_1801_00338_b200/csrc/*.cuh
  make lib -j32 EXTRA="$flags" < /dev/null > gpurun_out/ab_build_$name.log 2>&1 || { echo "build $name failed"; continue; }
  python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-samples --no-config3 --no-config5 --no-e2e --no-pairs > gpurun_out/ab_$name.json 2> gpurun_out/ab_$name.err
  python - "$name" <<'PY'
import json, sys
n = sys.argv[1]
d = json.load(open(f"gpurun_out/ab_{n}.json"))
ks = sorted(d["kernels"].items(), key=lambda x: -x[1]["ms_per_step"])[:16]
print(n, "step", round(d["ms_per_step"], 3), "agg", round(d["roofline_exact_s8d"]["aggregation_ms_per_step"], 3),
      {k: round(v["ms_per_step"], 3) for k, v in ks})
PY
done
