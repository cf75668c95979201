# A/B of the grouped walks (BFLY_GROUP_WALK) on the config-2 bench + parity of the variant.
mkdir -p gpurun_out
date
bash tools/ab.sh "base=-" "group=-DBFLY_GROUP_WALK=1" 2>&1 | tee gpurun_out/r11_ab.txt
date
timeout 900 python -m pytest -x -q -p no:cacheprovider tests/test_gpu_exact.py > gpurun_out/r11_tests_group.log 2>&1
echo "tests(group) rc=$?"; tail -3 gpurun_out/r11_tests_group.log; date
