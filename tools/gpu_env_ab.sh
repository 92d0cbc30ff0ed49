# A/B over environment settings: bash tools/gpu_env_ab.sh "VGP_DCACHE=0" "VGP_DCACHE=1"
for envs in "$@"; do
  echo "ENV: $envs"
  env $envs timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --e2e-steps 2 2>&1 | tail -1 | \
    python -c "import sys,json; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'], d['roofline']['kernel_ms'], d['kernel_variant'], 'e2e', d['e2e']['value'])"
done
