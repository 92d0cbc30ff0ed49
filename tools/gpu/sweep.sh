# BASELINE config 3: conditioning-size sweep at n = 250,000 (one bench line per m)
mkdir -p gpurun_out
for m in ${@:-10 20 30 45 60 90 120 150 200 300 400}; do
  timeout 600 python bench.py --n 250000 --m $m --steps 3 --warmup 3 --e2e-steps 1 --no-cpu-baseline > gpurun_out/sweep_m$m.log 2>&1
  echo "m=$m rc=$?"; tail -1 gpurun_out/sweep_m$m.log | python -c "import sys,json; d=json.loads(sys.stdin.read()); print(d['config']['m'], round(d['value'],2), round(d['ms_per_step'],2), d['kernel_variant'], round(d['roofline']['frac'],4), d['plan_s'])" 2>&1 | tail -1
done
