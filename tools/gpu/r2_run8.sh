# validation of the drained heavy parts + chunked wedge/edge jobs; sample / pair profiles; bench
mkdir -p gpurun_out
date
timeout 2400 python -m pytest -q -p no:cacheprovider tests -m gpu --durations=20 -k "not refsuite" > gpurun_out/r8_tests.log 2>&1
echo "tests rc=$?"; tail -25 gpurun_out/r8_tests.log; date
timeout 600 python tools/profile_samples.py 12 > gpurun_out/r8_samples.jsonl 2> gpurun_out/r8_samples.err; echo "samples rc=$?"
timeout 900 python tools/profile_pairs.py 4 > gpurun_out/r8_pairs.jsonl 2> gpurun_out/r8_pairs.err; echo "pairs rc=$?"
date
timeout 1500 python bench.py > gpurun_out/r8_bench.json 2> gpurun_out/r8_bench.err; echo "bench rc=$?"
date
