# GPU-box run: the -m gpu suite, the default bench line, and the ncu launch list of a short
# bench (profiles are summarised under profiles/ afterwards).
mkdir -p gpurun_out
date; nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 2700 python -m pytest tests -m gpu -q -p no:cacheprovider --durations=40 > gpurun_out/r2_gputest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r2_gputest.log
date; tail -3 gpurun_out/r2_gputest.log
timeout 1500 python bench.py > gpurun_out/r2_bench.json 2> gpurun_out/r2_bench.err; echo "bench rc=$?"
date
