BFLY_TRACE=1 python tools/debug_e2e.py 2> gpurun_out/trace.txt | tail -12
tail -80 gpurun_out/trace.txt
