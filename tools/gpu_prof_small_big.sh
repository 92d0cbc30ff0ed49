#!/bin/bash
mkdir -p gpurun_out
timeout 600 ncu --set full --import-source on --clock-control none -k regex:loglik_big -s 3 -c 1 -o gpurun_out/prof_big_m120 -f \
  python bench.py --n 250000 --m 120 --steps 1 --warmup 3 --e2e-steps 1 --no-cpu-baseline > gpurun_out/prof_big_m120.log 2>&1
echo "big rc=$?"
timeout 600 ncu --set full --import-source on --clock-control none -k regex:loglik_tiny -s 3 -c 1 -o gpurun_out/prof_tiny_m10 -f \
  python bench.py --n 250000 --m 10 --steps 1 --warmup 3 --e2e-steps 1 --no-cpu-baseline > gpurun_out/prof_tiny_m10.log 2>&1
echo "tiny rc=$?"
