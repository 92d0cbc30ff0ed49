# large-m kernel check: parity (CTA-per-block variants, c4 prefix), c4 bench, c3 m=90/120/200 quick sweep
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "golden and (11 or 12)" -p no:cacheprovider > gpurun_out/pytest_big.log 2>&1; echo "pytest big rc=$?"; tail -2 gpurun_out/pytest_big.log
timeout 900 python -m pytest tests/test_gpu_scale.py -q -x -k "c4" -p no:cacheprovider > gpurun_out/pytest_scale4.log 2>&1; echo "pytest scale rc=$?"; tail -2 gpurun_out/pytest_scale4.log
timeout 600 python bench.py --n 4000000 --m 120 --steps 5 --warmup 3 --e2e-steps 2 --no-cpu-baseline > gpurun_out/bench_c4.log 2>&1; echo "c4 rc=$?"; tail -1 gpurun_out/bench_c4.log | cut -c1-300
for m in 90 150 200; do timeout 300 python bench.py --n 250000 --m $m --steps 5 --warmup 3 --e2e-steps 1 --no-cpu-baseline 2>/dev/null | tail -1 | cut -c1-120; done
