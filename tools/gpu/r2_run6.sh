# reduce-then-scan radix vs CUB; ESamp jobs; build tests
mkdir -p gpurun_out
date
timeout 900 python -m pytest -x -q -p no:cacheprovider tests/test_gpu_build.py tests/test_gpu_exact.py tests/test_gpu_local.py > gpurun_out/r6_tests.log 2>&1
echo "tests rc=$?"; tail -3 gpurun_out/r6_tests.log; date
timeout 600 python tools/profile_samples.py 12 > gpurun_out/r6_samples.jsonl 2> gpurun_out/r6_samples.err; echo "samples rc=$?"
bash tools/ab.sh "cub=-DBFLY_HAND_SORT=0" "hand=-" 2>&1 | tee gpurun_out/r6_ab.txt
date
