#!/bin/bash
mkdir -p gpurun_out
for v in 11 12; do
timeout 600 ncu --set full --import-source on --clock-control none -k regex:loglik_big -s 3 -c 1 -o gpurun_out/prof_c5_v$v -f \
  python bench.py --n 200000 --m 60 --nu 0.8 --steps 1 --warmup 3 --e2e-steps 1 --no-cpu-baseline --variant $v > gpurun_out/prof_c5_v$v.log 2>&1
echo "v$v rc=$?"
done
