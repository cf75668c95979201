# hub plan without fseg reads for non-hub tasks, thread-per-vertex masks, keys-only priority rows
mkdir -p gpurun_out
timeout 1500 python -m pytest -x -q -p no:cacheprovider tests/test_gpu_exact.py tests/test_gpu_local.py tests/test_gpu_build.py tests/test_gpu_configs.py tests/test_gpu_estimators.py -k "not config5" > gpurun_out/r22_tests.log 2>&1
echo "tests rc=$?"; tail -3 gpurun_out/r22_tests.log
bash tools/gpu/ab_envs.sh r22 "new:-" "new_ser:BFLY_AGG_CONCURRENT=0"
python - <<'PY'
import json
for n in ("new", "new_ser"):
    d = json.load(open(f"gpurun_out/r22_{n}.json"))
    print(n, {k: round(v["ms_per_step"], 3) for k, v in d["kernels"].items() if k.startswith(("prio_", "hub_plan", "hub_mask", "hub_vprep", "sort_prio"))})
PY
