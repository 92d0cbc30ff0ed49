# ncu full capture of the fused kernel (one launch) at reduced n for turnaround
N=${1:-200000}
timeout 600 ncu --set full --clock-control none --import-source on -k regex:loglik_kernel -s 1 -c 1 -o gpurun_out/prof_fused python bench.py --n $N --steps 1 --warmup 1 --e2e-steps 1 --no-cpu-baseline > gpurun_out/prof_fused.log 2>&1
tail -3 gpurun_out/prof_fused.log
