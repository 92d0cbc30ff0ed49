# quick GPU check: parity tests + one bench line
timeout 600 python -m pytest tests -m gpu -q -x --timeout 500 2>&1 | tail -4
timeout 600 python bench.py --steps 20 --warmup 3 --no-cpu-baseline 2>&1 | tail -2 | tee gpurun_out/bench_quick.log
