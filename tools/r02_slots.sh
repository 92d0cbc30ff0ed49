mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "golden and (11 or 12)" -p no:cacheprovider > gpurun_out/pytest_slots.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_slots.log
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "acceptance_c1 or seeded or krige" -p no:cacheprovider > gpurun_out/pytest_slots2.log 2>&1; echo "pytest2 rc=$?"; tail -2 gpurun_out/pytest_slots2.log
timeout 900 python -m pytest tests/test_gpu_scale.py -q -x -k "c4" -p no:cacheprovider 2>&1 | tail -1
bash tools/gpu_sweep.sh 90 120 150 200 300
timeout 600 python bench.py --n 4000000 --m 120 --steps 5 --warmup 3 --e2e-steps 1 --no-cpu-baseline > gpurun_out/bench_slots_c4.log 2>&1; tail -1 gpurun_out/bench_slots_c4.log | cut -c1-100
