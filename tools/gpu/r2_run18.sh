# Dense top-hub path: hub/start split re-tuned with it (BFLY_HUB_MIN_WORK), the hub task
# histogram, compute-sanitizer on the dense kernels, ncu --set full of the dense kernels.
mkdir -p gpurun_out
BOPT="--steps 5 --warmup 3 --no-cpu-baseline --no-samples --no-config3 --no-config5 --no-e2e --no-pairs"
bash tools/gpu/ab_envs.sh r18 "base:-" "mw2k:BFLY_HUB_MIN_WORK=2048" "mw4k:BFLY_HUB_MIN_WORK=4096" "mw16k:BFLY_HUB_MIN_WORK=16384" "mw32k:BFLY_HUB_MIN_WORK=32768" "mw64k:BFLY_HUB_MIN_WORK=65536"
BFLY_HUB_STATS=1 python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-samples --no-config3 --no-config5 --no-e2e --no-pairs 2>&1 >/dev/null | grep "^\[hub\]" | sort -u > gpurun_out/r18_hubstats.txt
for tool in memcheck racecheck; do
  timeout 900 compute-sanitizer --tool $tool --error-exitcode 9 python -m pytest -x -q -p no:cacheprovider "tests/test_gpu_exact.py::test_dense_top_hub_widths[8]" tests/test_gpu_exact.py::test_dense_top_hubs_on_bicliques > gpurun_out/r18_san_$tool.log 2>&1
  echo "sanitizer $tool rc=$?"; tail -4 gpurun_out/r18_san_$tool.log
done
export BFLY_AGG_CONCURRENT=0
timeout 900 ncu --set full --import-source on --clock-control none --kernel-name-base demangled \
  -k regex:"k_dense|k_hub_mask|k_hub_plan" -c 4 -f -o gpurun_out/r18_dense \
  python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-samples --no-config3 --no-config5 --no-e2e --no-pairs > gpurun_out/r18_ncu.log 2>&1
echo "ncu rc=$?"
ncu -i gpurun_out/r18_dense.ncu-rep --page raw --csv > gpurun_out/r18_dense_raw.csv 2>/dev/null
ncu -i gpurun_out/r18_dense.ncu-rep --page source --csv --print-kernel-base demangled > gpurun_out/r18_dense_source.csv 2>/dev/null
ls -la gpurun_out/r18_dense*
