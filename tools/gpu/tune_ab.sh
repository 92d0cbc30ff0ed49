# A/B of VGP_TUNE experiment selectors on one box: bash tools/gpu/tune_ab.sh "<tunes>" <bench args>
# (tune 0 = default kernels; prints value, e2e and the evaluation total)
tunes="$1"; shift
mkdir -p gpurun_out
for r in 1 2; do for t in $tunes; do
  VGP_TUNE=$t timeout 600 python bench.py "$@" --steps 10 --warmup 3 --e2e-steps 1 --no-cpu-baseline 2>/dev/null | tail -1 | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); print('tune=$t', round(d['value'],2), round(d['e2e']['value'],2), repr(d['total']), d.get('kernel_variant'))"
done; done
