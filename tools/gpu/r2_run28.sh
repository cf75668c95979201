# hub warp-table kernels: 6 resident CTAs per SM (40 registers), task prefetch
mkdir -p gpurun_out
for v in "minb6:-DBFLY_SMALL_MINB=6" "minb6_pf:-DBFLY_SMALL_MINB=6 -DBFLY_SMALL_PREFETCH=1" "pf:-DBFLY_SMALL_PREFETCH=1" "ku8:-DBFLY_SMALL_KU=8" "base:-DBFLY_NOP=1"; do
  name="${v%%:*}"; fl="${v#*:}"
  touch paper_1801_00338_b200/csrc/*.cuh
  make lib -j32 EXTRA="$fl" > gpurun_out/r28_build_$name.log 2>&1 || { echo "build $name failed"; tail -3 gpurun_out/r28_build_$name.log; continue; }
  bash tools/gpu/ab_envs.sh r28 "$name:-" "${name}_ser:BFLY_AGG_CONCURRENT=0"
done
