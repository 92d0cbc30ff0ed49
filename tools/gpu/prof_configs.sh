# ncu --set full of each BASELINE config's dominant kernel at full size (one launch
# after the warm-up), summarised on the box (reports are too big to bring back),
# plus the launch list of the default bench (c2)
mkdir -p gpurun_out
prof() {  # name kernel-regex blocks bench-args...
  name=$1; kre=$2; blocks=$3; shift 3
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$kre -s 3 -c 1 -o /tmp/$name python bench.py "$@" --steps 1 --warmup 3 --e2e-steps 1 --no-cpu-baseline > gpurun_out/$name.log 2>&1
  echo "$name rc=$?"
  python tools/ncu_summary.py /tmp/$name.ncu-rep $blocks gpurun_out/$name.json > /dev/null 2>&1; echo "summary rc=$?"
  ncu -i /tmp/$name.ncu-rep --page source --csv --print-source sass > /tmp/$name.src.csv 2>/dev/null
  gzip -c /tmp/$name.src.csv > gpurun_out/$name.src.csv.gz
}
prof r02_ncu_c2_final loglik_ws3 999940
prof r02_ncu_c4_final loglik_big 3999880 --n 4000000 --m 120
prof r02_ncu_c5_final loglik_ws3 1999940 --n 2000000 --locations clustered --ordering maxmin --nu 0.8
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02_launches_c2.csv python bench.py --steps 2 --warmup 3 --e2e-steps 1 --no-cpu-baseline > gpurun_out/r02_launches_run.log 2>&1; echo "launches rc=$?"
ls -la gpurun_out
