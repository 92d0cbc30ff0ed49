#!/bin/bash
# small-m regime: every kernel variant at n = 250k
for m in ${MS:-10 20 30}; do for v in ${VS:-0 1 2 3 4 7 8 11 12}; do
  timeout 300 python bench.py --n 250000 --m $m --steps 10 --warmup 3 --e2e-steps 1 --no-cpu-baseline --variant $v 2>&1 | tail -1 | python -c "
import json,sys
try:
    d=json.loads(sys.stdin.read()); print($m, $v, round(d['value'],1), d['kernel_variant'], round(d['roofline']['kernel_ms'],3))
except Exception as e: print($m, $v, 'fail')"
done; done
