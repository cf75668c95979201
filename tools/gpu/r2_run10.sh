# Round-2 validation + measurement: the whole -m gpu suite, smoke(), the default bench line, the
# ncu launch list of a short bench and the DRAM traffic of the counting kernels.
mkdir -p gpurun_out
date
timeout 2700 python -m pytest tests -m gpu -q -p no:cacheprovider --durations=15 > gpurun_out/r10_gputest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r10_gputest.log
tail -4 gpurun_out/r10_gputest.log; date
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r10_smoke.log 2>&1; echo "smoke rc=$?"
timeout 1500 python bench.py > gpurun_out/r10_bench.json 2> gpurun_out/r10_bench.err; echo "bench rc=$?"
date
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/r10_launches.csv \
  python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-samples --no-config3 --no-config5 --no-e2e --no-pairs > gpurun_out/r10_ncu_bench.log 2>&1; echo "ncu launches rc=$?"
BFLY_AGG_CONCURRENT=0 timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none \
  --kernel-name-base demangled -k regex:"HubSrc|ExactSrc" -c 14 -f -o gpurun_out/r10_traffic \
  python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-samples --no-config3 --no-config5 --no-e2e --no-pairs > gpurun_out/r10_ncu_traffic.log 2>&1; echo "ncu traffic rc=$?"
python tools/ncu_traffic.py gpurun_out/r10_traffic.ncu-rep > gpurun_out/r10_ncu_traffic.json; rm -f gpurun_out/r10_traffic.ncu-rep
du -sh gpurun_out; date
