mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_scale.py -q -x --timeout 1100 -p no:cacheprovider > gpurun_out/pytest_scale.log 2>&1; echo "pytest rc=$?"; tail -15 gpurun_out/pytest_scale.log
timeout 600 python bench.py --steps 20 --warmup 3 > gpurun_out/bench.log 2>&1; echo "bench rc=$?"; tail -3 gpurun_out/bench.log
