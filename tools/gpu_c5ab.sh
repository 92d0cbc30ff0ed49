for args in "--locations uniform --ordering random --variant 12" "--locations uniform --ordering random --variant 11" "--locations clustered --ordering maxmin --variant 12" "--locations clustered --ordering maxmin --variant 11"; do
  timeout 600 python bench.py --n 2000000 --m 60 --nu 0.8 --steps 3 --warmup 3 --e2e-steps 1 --no-cpu-baseline $args 2>&1 | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$args', round(d['value'],3), d['kernel_variant'], d['clocks'])"
done
