set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 600 python bench.py --steps 10 --warmup 3 2>&1 | tail -5 | tee gpurun_out/bench1.log
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --n 1000000 --steps 2 --warmup 1 --e2e-steps 1 --no-cpu-baseline > gpurun_out/launches_run.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:loglik_dmma -s 1 -c 1 -o gpurun_out/prof_dmma python bench.py --n 1000000 --steps 1 --warmup 1 --e2e-steps 1 --no-cpu-baseline > gpurun_out/prof_run.log 2>&1
ls -la gpurun_out
