# Vectorised (uint4) segment walks of the counting runs: parity, then A/B against the scalar
# walks and the variants (one chunk round per iteration, start path included).
mkdir -p gpurun_out
timeout 1200 python -m pytest -x -q -p no:cacheprovider tests/test_gpu_exact.py tests/test_gpu_local.py tests/test_gpu_configs.py -k "not config5" > gpurun_out/r20_tests.log 2>&1
echo "tests rc=$?"; tail -3 gpurun_out/r20_tests.log
bash tools/gpu/ab_envs.sh r20 "v4:-" "v4_ser:BFLY_AGG_CONCURRENT=0"
for v in "ku1:-DBFLY_VEC4_KU=1" "ex1:-DBFLY_VEC4_EXACT=1" "off:-DBFLY_VEC4=0"; do
  name="${v%%:*}"; fl="${v#*:}"
  touch paper_1801_00338_b200/csrc/*.cuh
  make lib -j32 EXTRA="$fl" > gpurun_out/r20_build_$name.log 2>&1 || { echo "build $name failed"; continue; }
  bash tools/gpu/ab_envs.sh r20 "$name:-" "${name}_ser:BFLY_AGG_CONCURRENT=0"
done
