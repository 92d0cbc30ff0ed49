# ncu --set full of one config's dominant kernel (summary + gzipped source page)
# usage: bash tools/gpu/prof_one.sh NAME KERNEL_REGEX BLOCKS bench-args...
mkdir -p gpurun_out
name=$1; kre=$2; blocks=$3; shift 3
timeout 900 ncu --set full --clock-control none --import-source on -k regex:$kre -s 3 -c 1 -o /tmp/$name python bench.py "$@" --steps 1 --warmup 3 --e2e-steps 1 --no-cpu-baseline > gpurun_out/$name.log 2>&1
echo "$name rc=$?"
python tools/ncu_summary.py /tmp/$name.ncu-rep $blocks gpurun_out/$name.json > /dev/null 2>&1; echo "summary rc=$?"
ncu -i /tmp/$name.ncu-rep --page source --csv --print-source sass > /tmp/$name.src.csv 2>/dev/null
gzip -c /tmp/$name.src.csv > gpurun_out/$name.src.csv.gz
