# A/B over VGP_TUNE values: one bench line each (no cpu baseline)
for t in "$@"; do
  echo "TUNE=$t"
  VGP_TUNE=$t timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --e2e-steps 1 2>&1 | tail -1 | \
    python -c "import sys,json; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'], d['roofline']['kernel_ms'])"
done
