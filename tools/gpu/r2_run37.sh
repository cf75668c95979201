# bulk asynchronous copy (cp.async.bulk + mbarrier) staging of the entry ids in k_dense_big: parity + A/B
mkdir -p gpurun_out
timeout 600 python -m pytest -x -q -p no:cacheprovider tests/test_gpu_exact.py tests/test_gpu_configs.py -k "not config5 and not config4" > gpurun_out/r37_tests.log 2>&1
echo "tests rc=$?"; tail -3 gpurun_out/r37_tests.log
bash tools/gpu/ab_envs.sh r37 "bulk:-" "bulk_ser:BFLY_AGG_CONCURRENT=0" "bulk_b4:BFLY_DENSE_GRID_B=4" "bulk_b3:BFLY_DENSE_GRID_B=3"
touch paper_1801_00338_b200/csrc/*.cuh
make lib -j32 EXTRA="-DBFLY_DENSE_BULK=0" > gpurun_out/r37_build.log 2>&1 || echo "build failed"
bash tools/gpu/ab_envs.sh r37 "ldg:-" "ldg_ser:BFLY_AGG_CONCURRENT=0"
