mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "golden or seeded or distance_cache" -p no:cacheprovider > gpurun_out/pytest_ws.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_ws.log
for m in 30 45 54; do for v in 4 8; do timeout 300 python bench.py --n 250000 --m $m --steps 5 --warmup 3 --e2e-steps 1 --no-cpu-baseline --variant $v > gpurun_out/mid_$m_$v.log 2>&1; echo "m=$m v=$v $(tail -1 gpurun_out/mid_$m_$v.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["value"],1), d["total"])')"; done; done
