# ncu full capture of the grouped kernel
mkdir -p gpurun_out
V=${1:-3}
TAG=${2:-ll}
timeout 900 ncu --set full --clock-control none --import-source on -k regex:loglik_ -s 1 -c 1 -o gpurun_out/prof_$TAG python bench.py --steps 1 --warmup 1 --e2e-steps 1 --no-cpu-baseline --variant $V > gpurun_out/prof_$TAG.log 2>&1; echo "ncu rc=$?"
tail -2 gpurun_out/prof_$TAG.log
