# Profile the per-sample path, the radix sort kernels and the pair pass; the config goldens.
mkdir -p gpurun_out
date
timeout 900 python tools/profile_samples.py 12 > gpurun_out/r4_samples.jsonl 2> gpurun_out/r4_samples.err; echo "samples rc=$?"
date
timeout 600 ncu --set full --import-source on --clock-control none --kernel-name-base demangled -k regex:"k_sweep" -c 3 -f -o gpurun_out/r4_radix \
  python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-samples --no-config3 --no-config5 --no-e2e > gpurun_out/r4_ncu_radix.log 2>&1; echo "ncu radix rc=$?"
date
timeout 900 python tools/profile_pairs.py 3 > gpurun_out/r4_pairs.jsonl 2> gpurun_out/r4_pairs.err; echo "pairs rc=$?"
date
timeout 1500 python -m pytest -q -p no:cacheprovider tests/test_gpu_configs.py -k "not sample_paths" > gpurun_out/r4_configs.log 2>&1; echo "configs rc=$?"; tail -3 gpurun_out/r4_configs.log
date
