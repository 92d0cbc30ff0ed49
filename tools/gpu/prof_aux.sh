# ncu --set full of the non-headline kernels (one launch each), summarised on the box
# usage: bash tools/gpu/prof_aux.sh "name regex mode" ...  e.g.
#   "r02_ncu_knn_grid grid_query knn" "r02_ncu_dcache build_dcache dcache"
#   "r02_ncu_tiny_m10 loglik_tiny m10" "r02_ncu_dmma_m20 ^loglik_kernel m20"
#   "r02_ncu_ws_m30 loglik_ws_kernel m30" "r02_ncu_maxmin maxmin_cluster maxmin"
mkdir -p gpurun_out
prof() {  # name kernel-regex mode
  name=$1; kre=$2; mode=$3
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$kre -c 1 -o /tmp/$name python tools/prof_aux.py $mode > gpurun_out/$name.log 2>&1
  echo "$name rc=$?"
  python tools/ncu_summary.py /tmp/$name.ncu-rep 1 gpurun_out/$name.json > /dev/null 2>&1; echo "summary rc=$?"
  ncu -i /tmp/$name.ncu-rep --page raw --csv > gpurun_out/$name.raw.csv 2>/dev/null
}
for job in "$@"; do prof $job; done
ls -la gpurun_out | tail -30
