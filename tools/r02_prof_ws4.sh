mkdir -p gpurun_out
V=${V:-14}
timeout 900 ncu --set full --clock-control none --import-source on -k regex:loglik_ws -s 1 -c 1 -o gpurun_out/prof_ws$V python bench.py --n 250000 --steps 1 --warmup 1 --e2e-steps 1 --no-cpu-baseline --variant $V > gpurun_out/prof_ws$V.log 2>&1; echo "ncu rc=$?"
