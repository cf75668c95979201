# ncu --set full of the LOCAL kernels on config 3 (source-level), exported on the box
mkdir -p gpurun_out
NCU="ncu --set full --import-source on --clock-control none --kernel-name-base demangled -f"
timeout 900 $NCU -k regex:"k_(small|medium)<.*HubSrc, .bool.1" -c 4 -o gpurun_out/r33_local python tools/ncu_secondary.py local > gpurun_out/r33_local.log 2>&1
echo "rc=$?"
ncu -i gpurun_out/r33_local.ncu-rep --page raw --csv > gpurun_out/r33_local.raw.csv 2>/dev/null
ncu -i gpurun_out/r33_local.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/r33_local.src.csv 2>/dev/null
gzip -f gpurun_out/r33_local.src.csv
rm -f gpurun_out/r33_local.ncu-rep
ls -la gpurun_out/r33_local*
