# ncu --set full captures of the secondary paths (one driver per capture, kernel filters):
# the LOCAL pass on config 3, the per-sample kernels on config 2, sparsify on config 5.
# Reports are exported to CSV on the box (raw metrics + source lines) and deleted, so the
# results fit the copy-back limit.
mkdir -p gpurun_out
NCU="ncu --set full --import-source on --clock-control none --kernel-name-base demangled -f"
cap() {  # name regex count mode
  timeout 900 $NCU -k regex:"$2" -c $3 -o gpurun_out/$1 python tools/ncu_secondary.py $4 > gpurun_out/$1.log 2>&1
  echo "$1 rc=$?"
  ncu -i gpurun_out/$1.ncu-rep --page raw --csv > gpurun_out/$1.raw.csv 2>/dev/null
  ncu -i gpurun_out/$1.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/$1.src.csv 2>/dev/null
  gzip -f gpurun_out/$1.src.csv
  rm -f gpurun_out/$1.ncu-rep
}
cap r2_local "k_(tiny|small|medium|split|heavy_el|heavy)<" 14 local
cap r2_samples "VertexSrc|k_edge_job_run|k_wedge_samples" 14 samples
cap r2_spar "k_keep_bits|k_colours|k_emit|k_degree2|k_mark_live|k_fill_left|k_scatter_right|k_bm_|k_row_of" 24 spar
