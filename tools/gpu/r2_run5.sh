# Validate element-balanced heavy parts + the 512-thread radix sweep; A/B against CUB; profile
# the per-sample path and the pair pass again.
mkdir -p gpurun_out
date
timeout 900 python tools/profile_samples.py 12 > gpurun_out/r5_samples.jsonl 2> gpurun_out/r5_samples.err; echo "samples rc=$?"
date
timeout 1800 python -m pytest -x -q -p no:cacheprovider tests/test_gpu_build.py tests/test_gpu_exact.py tests/test_gpu_local.py \
  tests/test_gpu_pairs.py tests/test_gpu_estimators.py tests/test_gpu_sampler.py tests/test_gpu_configs.py --durations=15 > gpurun_out/r5_tests.log 2>&1
echo "tests rc=$?"; tail -20 gpurun_out/r5_tests.log; date
timeout 900 python tools/profile_pairs.py 3 > gpurun_out/r5_pairs.jsonl 2> gpurun_out/r5_pairs.err; echo "pairs rc=$?"
date
bash tools/ab.sh "cub=-DBFLY_HAND_SORT=0" "hand=-" 2>&1 | tee gpurun_out/r5_ab.txt
date
