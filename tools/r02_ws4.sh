mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "golden and (14 or 16)" -p no:cacheprovider > gpurun_out/pytest_ws4.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_ws4.log
for v in ${VARIANTS:-16 14}; do timeout 300 python bench.py --steps 20 --warmup 3 --variant $v --no-cpu-baseline --e2e-steps 2 ${BENCH_ARGS} > gpurun_out/bench_v$v.log 2>&1; echo "v=$v rc=$?"; tail -1 gpurun_out/bench_v$v.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['roofline']['frac'], d['total'])"; done
