# parity tests + bench A/B over kernel variants
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x --timeout 800 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -15 gpurun_out/pytest_gpu.log
for v in 3 2 1; do
  timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 1 --variant $v > gpurun_out/bench_v$v.log 2>&1
  echo "variant $v rc=$?"; tail -1 gpurun_out/bench_v$v.log | python -c "import sys,json; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'], d['roofline']['kernel_ms'], d['kernel_variant'], d['total'])" 2>&1 | tail -2
done
