# Dense top-hub path with the chunked big-task kernel: parity, then widths, concurrent and serial.
mkdir -p gpurun_out
timeout 1200 python -m pytest -x -q -p no:cacheprovider tests/test_gpu_exact.py tests/test_gpu_local.py > gpurun_out/r14_tests.log 2>&1
echo "tests rc=$?"; tail -3 gpurun_out/r14_tests.log
for conc in 1 0; do
for spec in off:BFLY_HUB_DENSE=0 w2:BFLY_HUB_DENSE_W=2 w4:BFLY_HUB_DENSE_W=4 w8:BFLY_HUB_DENSE_W=8 w16:BFLY_HUB_DENSE_W=16 w32:BFLY_HUB_DENSE_W=32; do
  name="${spec%%:*}_c$conc"; kv="${spec#*:}"
  env BFLY_AGG_CONCURRENT=$conc "$kv" python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-samples --no-config3 --no-config5 --no-e2e --no-pairs > gpurun_out/r14_$name.json 2> gpurun_out/r14_$name.err || { echo "$name failed"; tail -5 gpurun_out/r14_$name.err; continue; }
  python - "$name" <<'PY'
import json, sys
n = sys.argv[1]
d = json.load(open(f"gpurun_out/r14_{n}.json"))
ks = sorted(d["kernels"].items(), key=lambda x: -x[1]["ms_per_step"])[:30]
print(n, "step", round(d["ms_per_step"], 3), "agg", round(d["roofline_exact_s8d"]["aggregation_ms_per_step"], 3), "bfly", d["workload_stats"]["butterflies"],
      {k: round(v["ms_per_step"], 3) for k, v in ks if k.startswith(("hub_", "exact_"))})
PY
done
done 2>&1 | tee gpurun_out/r14_ab.txt
