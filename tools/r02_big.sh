mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "golden and (11 or 12)" -p no:cacheprovider > gpurun_out/pytest_big.log 2>&1; echo "pytest big rc=$?"; tail -2 gpurun_out/pytest_big.log
timeout 900 python -m pytest tests/test_gpu_scale.py -q -x -k "c4 or c5" -p no:cacheprovider > gpurun_out/pytest_scale45.log 2>&1; echo "pytest scale rc=$?"; tail -2 gpurun_out/pytest_scale45.log
timeout 600 python bench.py --n 4000000 --m 120 --steps 5 --warmup 3 --e2e-steps 2 > gpurun_out/bench_c4.log 2>&1; echo "c4 rc=$?"; tail -1 gpurun_out/bench_c4.log | cut -c1-400
timeout 600 python bench.py --n 2000000 --locations clustered --ordering maxmin --nu 0.8 --steps 5 --warmup 3 --e2e-steps 2 > gpurun_out/bench_c5.log 2>&1; echo "c5 rc=$?"; tail -1 gpurun_out/bench_c5.log | cut -c1-400
