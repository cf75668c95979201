# ncu --set full captures of the secondary paths (one driver per capture, kernel filters):
# the LOCAL pass on config 3, the per-sample kernels on config 2, sparsify on config 5.
mkdir -p gpurun_out
NCU="ncu --set full --import-source on --clock-control none --kernel-name-base demangled -f"
timeout 900 $NCU -k regex:"k_(tiny|small|medium|split|heavy_el|heavy)<" -c 14 -o gpurun_out/r2_local \
  python tools/ncu_secondary.py local > gpurun_out/r2_ncu_local.log 2>&1; echo "local rc=$?"
timeout 900 $NCU -k regex:"VertexSrc|k_edge_job_run|k_wedge_samples" -c 14 -o gpurun_out/r2_samples \
  python tools/ncu_secondary.py samples > gpurun_out/r2_ncu_samples.log 2>&1; echo "samples rc=$?"
timeout 900 $NCU -k regex:"k_keep_bits|k_colours|k_emit|k_degree2|k_mark_live|k_fill_left|k_scatter_right|k_bm_|k_row_of" -c 24 -o gpurun_out/r2_spar \
  python tools/ncu_secondary.py spar > gpurun_out/r2_ncu_spar.log 2>&1; echo "spar rc=$?"
