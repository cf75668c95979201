# Dense top-hub path (hubdense.cuh): parity first, then the config-2 bench for several mask widths.
mkdir -p gpurun_out
date
timeout 1200 python -m pytest -x -q -p no:cacheprovider tests/test_gpu_exact.py tests/test_gpu_local.py tests/test_gpu_estimators.py > gpurun_out/r12_tests.log 2>&1
echo "tests rc=$?"; tail -5 gpurun_out/r12_tests.log; date
for spec in off:BFLY_HUB_DENSE=0 w1:BFLY_HUB_DENSE_W=1 w2:BFLY_HUB_DENSE_W=2 w4:BFLY_HUB_DENSE_W=4 w8:BFLY_HUB_DENSE_W=8 w16:BFLY_HUB_DENSE_W=16 w32:BFLY_HUB_DENSE_W=32; do
  name="${spec%%:*}"; kv="${spec#*:}"
  env "$kv" python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-samples --no-config3 --no-config5 --no-e2e --no-pairs > gpurun_out/r12_$name.json 2> gpurun_out/r12_$name.err || { echo "$name failed"; tail -5 gpurun_out/r12_$name.err; continue; }
  python - "$name" <<'PY'
import json, sys
n = sys.argv[1]
d = json.load(open(f"gpurun_out/r12_{n}.json"))
ks = sorted(d["kernels"].items(), key=lambda x: -x[1]["ms_per_step"])[:22]
print(n, "step", round(d["ms_per_step"], 3), "agg", round(d["roofline_exact_s8d"]["aggregation_ms_per_step"], 3), "bfly", d["workload_stats"]["butterflies"], "wedges", d["workload_stats"]["wedges_processed"],
      {k: round(v["ms_per_step"], 3) for k, v in ks})
PY
done 2>&1 | tee gpurun_out/r12_ab.txt
date
timeout 1500 python -m pytest -x -q -p no:cacheprovider tests/test_gpu_configs.py > gpurun_out/r12_configs.log 2>&1
echo "configs rc=$?"; tail -5 gpurun_out/r12_configs.log; date
