mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_cli.py -q -p no:cacheprovider > gpurun_out/pytest_cli.log 2>&1; echo "cli rc=$?"; tail -3 gpurun_out/pytest_cli.log
timeout 900 python tools/mle_runs.py c5 --out gpurun_out/r02_mle_c5_ktab.jsonl > gpurun_out/mle_c5.log 2>&1; echo "mle c5 rc=$?"; tail -c 600 gpurun_out/mle_c5.log
for cfg in "--n 4000000 --m 120" "--n 2000000 --locations clustered --ordering maxmin --nu 0.8"; do
  timeout 900 python bench.py $cfg --steps 10 --warmup 3 --e2e-steps 3 >> gpurun_out/r02_bench_configs.jsonl 2>gpurun_out/bench_cfg.err; echo "cfg rc=$?"
done
bash tools/gpu/sweep.sh 10 20 30 45 60 90 120 150 200 300 400 > gpurun_out/sweep.txt 2>&1; cat gpurun_out/sweep.txt
cat gpurun_out/sweep_m*.log | grep '^{' > gpurun_out/r02_sweep_c3_n250k.jsonl
