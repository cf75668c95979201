# Compact hub-prefix array for counting plans: parity + A/B
mkdir -p gpurun_out
timeout 1500 python -m pytest -x -q -p no:cacheprovider tests/test_gpu_exact.py tests/test_gpu_local.py tests/test_gpu_configs.py tests/test_gpu_estimators.py -k "not config5" > gpurun_out/r30_tests.log 2>&1
echo "tests rc=$?"; tail -3 gpurun_out/r30_tests.log
bash tools/gpu/ab_envs.sh r30 "compact:-" "plain:BFLY_HUB_COMPACT=0" "compact_ser:BFLY_AGG_CONCURRENT=0" "plain_ser:BFLY_HUB_COMPACT=0 BFLY_AGG_CONCURRENT=0"
python - <<'PY'
import json
for n in ("compact", "plain"):
    d = json.load(open(f"gpurun_out/r30_{n}.json"))
    print(n, {k: round(v["ms_per_step"], 3) for k, v in d["kernels"].items() if k.startswith(("hub_plan", "hub_mask", "hub_vprep", "hub_compact"))})
PY
