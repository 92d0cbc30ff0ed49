# ncu --set full of each BASELINE config's dominant kernel at full size (one launch
# after the warm-up), plus the launch list of the default bench (c2)
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:loglik_ws3 -s 4 -c 1 -o gpurun_out/r02_ncu_c2 python bench.py --steps 2 --warmup 3 --e2e-steps 1 --no-cpu-baseline > gpurun_out/r02_ncu_c2.log 2>&1; echo "c2 rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:loglik_big -s 4 -c 1 -o gpurun_out/r02_ncu_c4 python bench.py --n 4000000 --m 120 --steps 1 --warmup 3 --e2e-steps 1 --no-cpu-baseline > gpurun_out/r02_ncu_c4.log 2>&1; echo "c4 rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:loglik_ws3 -s 4 -c 1 -o gpurun_out/r02_ncu_c5 python bench.py --n 2000000 --locations clustered --ordering maxmin --nu 0.8 --steps 1 --warmup 3 --e2e-steps 1 --no-cpu-baseline > gpurun_out/r02_ncu_c5.log 2>&1; echo "c5 rc=$?"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02_launches_c2.csv python bench.py --steps 2 --warmup 3 --e2e-steps 1 --no-cpu-baseline > gpurun_out/r02_launches_run.log 2>&1; echo "launches rc=$?"
