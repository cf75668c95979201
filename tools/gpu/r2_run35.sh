# bench with the config-4 warm-up: samples leg only + the main line (traffic file check)
mkdir -p gpurun_out
timeout 1200 python bench.py --no-cpu-baseline --no-config3 --no-config5 --no-pairs > gpurun_out/r35_bench.json 2> gpurun_out/r35_bench.err; echo "bench rc=$?"
python - <<'PY'
import json
d = json.load(open("gpurun_out/r35_bench.json"))
print(d["ms_per_step"], d["roofline"]["physical_frac"], d["roofline"]["frac"])
c4 = d["secondary"]["config4_estimators"]
for m in ("vsamp", "esamp", "wsamp"):
    print(m, round(c4[m]["cold_seconds"], 4), c4[m]["cold_path"], c4[m]["estimate"], round(c4[m]["warm_samples_per_s"] / 1e6, 1))
PY
