# Validate the hand-written radix sort, striped hub tables and the pair-type pass on the GPU,
# then A/B the compile-time variants on the config-2 bench and capture the hub kernels.
mkdir -p gpurun_out
date
timeout 1500 python -m pytest -x -q -p no:cacheprovider tests/test_gpu_build.py tests/test_gpu_exact.py \
  tests/test_gpu_pairs.py tests/test_gpu_refsuite.py tests/test_gpu_local.py > gpurun_out/r3_tests.log 2>&1
echo "tests rc=$?"; tail -3 gpurun_out/r3_tests.log; date
bash tools/ab.sh "cub_nostripe=-DBFLY_HAND_SORT=0 -DBFLY_HUB_STRIPE=0" "hand_nostripe=-DBFLY_HUB_STRIPE=0" \
  "hand_stripe=-" "hand_stripe_match=-DBFLY_HUB_MATCH=1" "hand_nostripe_match=-DBFLY_HUB_STRIPE=0 -DBFLY_HUB_MATCH=1" 2>&1 | tee gpurun_out/r3_ab.txt
date
touch paper_1801_00338_b200/csrc/*.cuh; STRIPES="0 1" bash tools/gpu/r2_ncu_hub.sh
date
make lib -j32 > /dev/null 2>&1
timeout 1800 python bench.py > gpurun_out/r3_bench.json 2> gpurun_out/r3_bench.err; echo "bench rc=$?"
date
