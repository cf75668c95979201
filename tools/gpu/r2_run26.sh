# Dense mask kernels really overlapped with the walks (join waits deferred): parity + A/B
mkdir -p gpurun_out
timeout 1500 python -m pytest -x -q -p no:cacheprovider tests/test_gpu_exact.py tests/test_gpu_local.py tests/test_gpu_configs.py -k "not config5" > gpurun_out/r27_tests.log 2>&1
echo "tests rc=$?"; tail -3 gpurun_out/r27_tests.log
bash tools/gpu/ab_envs.sh r27 "first:-" "last:BFLY_DENSE_FIRST=0" "first_d44:BFLY_DENSE_GRID_S=4 BFLY_DENSE_GRID_B=4" "first_d63:BFLY_DENSE_GRID_S=6 BFLY_DENSE_GRID_B=3" "first_w16:BFLY_HUB_DENSE_W=16" "ser:BFLY_AGG_CONCURRENT=0"
  "first_d44:BFLY_DENSE_GRID_S=4 BFLY_DENSE_GRID_B=4" "first_d22:BFLY_DENSE_GRID_S=2 BFLY_DENSE_GRID_B=2" "first_d32:BFLY_DENSE_GRID_S=3 BFLY_DENSE_GRID_B=2" \
  "first_d63:BFLY_DENSE_GRID_S=6 BFLY_DENSE_GRID_B=3" "last_d44:BFLY_DENSE_FIRST=0 BFLY_DENSE_GRID_S=4 BFLY_DENSE_GRID_B=4" \
  "first_w16:BFLY_HUB_DENSE_W=16" "first_w16_d44:BFLY_HUB_DENSE_W=16 BFLY_DENSE_GRID_S=4 BFLY_DENSE_GRID_B=4" "first_w1024:BFLY_EXACT_WIDE_BLOCK=1024"
