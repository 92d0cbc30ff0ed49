mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py -q -x -k "golden or free_nu or bessel or cov" -p no:cacheprovider > gpurun_out/pytest_gen.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gen.log
timeout 900 python -m pytest tests/test_gpu_scale.py -q -x -k "c5 or simulate" -p no:cacheprovider > gpurun_out/pytest_scale5.log 2>&1; echo "pytest scale rc=$?"; tail -2 gpurun_out/pytest_scale5.log
timeout 600 python bench.py --n 2000000 --locations clustered --ordering maxmin --nu 0.8 --steps 10 --warmup 3 --e2e-steps 3 > gpurun_out/bench_c5.log 2>&1; echo "c5 rc=$?"; tail -1 gpurun_out/bench_c5.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['kernel_variant'], d['parity'])"
