mkdir -p gpurun_out
date
timeout 1200 python -m pytest -x -q -p no:cacheprovider tests/test_gpu_pairs.py tests/test_gpu_local.py tests/test_gpu_exact.py tests/test_gpu_configs.py > gpurun_out/r9_tests.log 2>&1
echo "tests rc=$?"; tail -3 gpurun_out/r9_tests.log; date
timeout 600 python tools/profile_samples.py 12 > gpurun_out/r9_samples.jsonl 2> gpurun_out/r9_samples.err; echo "samples rc=$?"
timeout 900 python tools/profile_pairs.py 4 > gpurun_out/r9_pairs.jsonl 2> gpurun_out/r9_pairs.err; echo "pairs rc=$?"
date
