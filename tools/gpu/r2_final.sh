# Round-2 validation + measurement of the final tree: the whole -m gpu suite, smoke(), the default
# bench line, the ncu launch list of a short bench, the DRAM traffic of the counting kernels and
# one ncu --set full capture of the counting kernels (serialised buckets).
TAG=${TAG:-r2f}
mkdir -p gpurun_out
date
timeout 2700 python -m pytest tests -m gpu -q -p no:cacheprovider --durations=15 > gpurun_out/${TAG}_gputest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${TAG}_gputest.log
tail -4 gpurun_out/${TAG}_gputest.log; date
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1; echo "smoke rc=$?"
timeout 1500 python bench.py > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err; echo "bench rc=$?"
timeout 600 python bench.py --impl reference > gpurun_out/${TAG}_bench_ref.json 2> gpurun_out/${TAG}_bench_ref.err; echo "bench ref rc=$?"
date
BOPT="--no-cpu-baseline --no-samples --no-config3 --no-config5 --no-e2e --no-pairs"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/${TAG}_launches.csv \
  python bench.py --steps 2 --warmup 1 $BOPT > gpurun_out/${TAG}_ncu_bench.log 2>&1; echo "ncu launches rc=$?"
BFLY_AGG_CONCURRENT=0 timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none \
  --kernel-name-base demangled -k regex:"HubSrc|ExactSrc|k_dense_small|k_dense_big" -c 16 -f -o gpurun_out/${TAG}_traffic \
  python bench.py --steps 1 --warmup 0 $BOPT > gpurun_out/${TAG}_ncu_traffic.log 2>&1; echo "ncu traffic rc=$?"
python tools/ncu_traffic.py gpurun_out/${TAG}_traffic.ncu-rep > gpurun_out/${TAG}_ncu_traffic_light.json; rm -f gpurun_out/${TAG}_traffic.ncu-rep
BFLY_AGG_CONCURRENT=0 timeout 1200 ncu --set full --import-source on --clock-control none --kernel-name-base demangled \
  -k regex:"HubSrc|ExactSrc|k_dense_small|k_dense_big|k_hub_mask" -c 17 -f -o gpurun_out/${TAG}_count_full \
  python bench.py --steps 1 --warmup 0 $BOPT > gpurun_out/${TAG}_ncu_full.log 2>&1; echo "ncu full rc=$?"
ncu -i gpurun_out/${TAG}_count_full.ncu-rep --page raw --csv > gpurun_out/${TAG}_count_full.raw.csv 2>/dev/null
python tools/ncu_traffic.py gpurun_out/${TAG}_count_full.raw.csv > gpurun_out/${TAG}_ncu_traffic.json  # (the --set full capture)
ncu -i gpurun_out/${TAG}_count_full.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/${TAG}_count_full.src.csv 2>/dev/null
gzip -f gpurun_out/${TAG}_count_full.src.csv
rm -f gpurun_out/${TAG}_count_full.ncu-rep
du -sh gpurun_out; date
