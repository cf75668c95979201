# Packed (one-word) CTA tables for the start path's medium / medium-wide buckets
mkdir -p gpurun_out
timeout 1500 python -m pytest -x -q -p no:cacheprovider tests/test_gpu_exact.py tests/test_gpu_local.py tests/test_gpu_configs.py tests/test_gpu_estimators.py -k "not config5" > gpurun_out/r24_tests.log 2>&1
echo "tests rc=$?"; tail -3 gpurun_out/r24_tests.log
bash tools/gpu/ab_envs.sh r24 "packed:-" "unpacked:BFLY_PACKED_MED=0" "packed_w512:BFLY_EXACT_WIDE_BLOCK=512" "packed_ser:BFLY_AGG_CONCURRENT=0" "unpacked_ser:BFLY_PACKED_MED=0 BFLY_AGG_CONCURRENT=0" "packed_w512_ser:BFLY_EXACT_WIDE_BLOCK=512 BFLY_AGG_CONCURRENT=0"
