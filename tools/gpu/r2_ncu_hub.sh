# A/B of the striped hub-table layout (BFLY_HUB_STRIPE) on the config-2 bench, plus one
# ncu --set full capture of the hub-path counting kernels of each variant (serialised buckets).
mkdir -p gpurun_out
export BFLY_AGG_CONCURRENT=0
for v in ${STRIPES:-0 1}; do
  touch paper_1801_00338_b200/csrc/*.cuh
  make lib -j32 EXTRA="-DBFLY_HUB_STRIPE=$v" > gpurun_out/r2_build_stripe$v.log 2>&1 || { echo "build $v failed"; continue; }
  BFLY_AGG_CONCURRENT=1 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-samples --no-config3 --no-config5 --no-e2e --no-pairs > gpurun_out/r2_stripe$v.json 2> gpurun_out/r2_stripe$v.err
  echo "stripe $v rc=$?"
  timeout 900 ncu --set full --import-source on --clock-control none --kernel-name-base demangled \
    -k regex:"HubSrc" -c 8 -f -o gpurun_out/r2_hub_stripe$v \
    python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-samples --no-config3 --no-config5 --no-e2e --no-pairs > gpurun_out/r2_ncu_stripe$v.log 2>&1
  echo "ncu $v rc=$?"
done
