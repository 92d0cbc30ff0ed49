#!/bin/bash
# general-nu (config 5) kernel variants at n = 200k and 2M
for n in 200000 2000000; do for v in 11 12; do
  timeout 600 python bench.py --n $n --m 60 --nu 0.8 --locations clustered --ordering maxmin --steps 3 --warmup 3 --e2e-steps 1 --no-cpu-baseline --variant $v 2>&1 | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print($n, $v, round(d['value'],3), d['kernel_variant'], d['clocks']['sm_mhz'])"
done; done
timeout 300 python -m pytest tests/test_gpu_parity.py -q -x -k "golden and (nu08 or nu23 or general)" 2>&1 | tail -2
