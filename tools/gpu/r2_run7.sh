mkdir -p gpurun_out
date
timeout 900 python -m pytest -x -q -p no:cacheprovider tests/test_gpu_build.py tests/test_gpu_exact.py tests/test_gpu_local.py > gpurun_out/r7_tests.log 2>&1
echo "tests rc=$?"; tail -2 gpurun_out/r7_tests.log
bash tools/ab.sh "cub=-DBFLY_HAND_SORT=0" "hand=-" "cub_noprefetch=-DBFLY_HAND_SORT=0 -DBFLY_SMALL_PREFETCH=0" 2>&1 | tee gpurun_out/r7_ab.txt
date
touch paper_1801_00338_b200/csrc/*.cuh; make lib -j32 EXTRA=-DBFLY_HAND_SORT=0 > /dev/null 2>&1
bash tools/gpu/r2_ncu_secondary.sh
ls -la gpurun_out; du -sh gpurun_out
date
