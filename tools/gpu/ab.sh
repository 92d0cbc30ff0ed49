# A/B of two builds of the native library on one box: bash tools/gpu/ab.sh <bench args>
# (abtest/libA.so, abtest/libB.so; B is left installed)
cfg="$*"
for r in 1 2; do for v in A B; do
  cp abtest/lib$v.so paper_2403_07412_b200/libvecchia_b200.so
  echo "$v $(timeout 600 python bench.py $cfg --steps 10 --warmup 3 --e2e-steps 1 --no-cpu-baseline 2>/dev/null | tail -1 | cut -c1-110)"
done; done
cp abtest/libB.so paper_2403_07412_b200/libvecchia_b200.so
