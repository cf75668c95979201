# Two tasks per warp in the hub small-A bucket (k_small_pair) + the dense-path gate: parity,
# then A/B concurrent and serial, and the config-5 legs (small sub-graphs: gate off).
mkdir -p gpurun_out
timeout 1200 python -m pytest -x -q -p no:cacheprovider tests/test_gpu_exact.py tests/test_gpu_local.py tests/test_gpu_configs.py -k "not config5" > gpurun_out/r19_tests.log 2>&1
echo "tests rc=$?"; tail -3 gpurun_out/r19_tests.log
bash tools/gpu/ab_envs.sh r19 "pair:-" "nopair:BFLY_SMALL_PAIR=0" "pair_ser:BFLY_AGG_CONCURRENT=0" "nopair_ser:BFLY_SMALL_PAIR=0 BFLY_AGG_CONCURRENT=0"
BFLY_HUB_STATS=1 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-samples --no-config3 --no-e2e --no-pairs > gpurun_out/r19_c5.json 2> gpurun_out/r19_c5.err
grep "^\[hub\] k=" gpurun_out/r19_c5.err | sort | uniq -c
python - <<'PY'
import json
d = json.load(open("gpurun_out/r19_c5.json"))
c5 = d["secondary"]["config5_sparsify"]
print({k: round(v["seconds"] * 1e3, 3) for k, v in c5.items() if isinstance(v, dict) and "seconds" in v})
PY
