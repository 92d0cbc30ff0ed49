# ncu captures of the production kernels + launch list of the default bench
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:loglik_ws3 -s 1 -c 1 -o gpurun_out/prof_ws3 python bench.py --steps 1 --warmup 1 --e2e-steps 1 --no-cpu-baseline > gpurun_out/prof_ws3.log 2>&1; echo "ncu ws3 rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:loglik_big -s 1 -c 1 -o gpurun_out/prof_big120 python bench.py --n 250000 --m 120 --steps 1 --warmup 1 --e2e-steps 1 --no-cpu-baseline > gpurun_out/prof_big.log 2>&1; echo "ncu big rc=$?"
timeout 400 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 1 --e2e-steps 1 --no-cpu-baseline > gpurun_out/launches_run.log 2>&1; echo "launches rc=$?"
