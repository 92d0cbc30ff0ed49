# Round-2 first pass: smoke, default bench, DMMA pipe accounting check
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv | tee gpurun_out/nvsmi.txt
nproc; lscpu | grep -E "Model name|^CPU\(s\)|Thread|Socket" | tee gpurun_out/lscpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -2 gpurun_out/smoke.log
timeout 600 python bench.py --steps 20 --warmup 3 > gpurun_out/bench.log 2>&1; echo "bench rc=$?"; tail -1 gpurun_out/bench.log
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/fp64_peak tools/fp64_peak.cu && \
timeout 300 ncu --metrics gpu__time_duration.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_tensor.avg.pct_of_peak_sustained_active,smsp__inst_executed_op_dmma.sum,sm__pipe_fp64_cycles_active.sum,sm__cycles_elapsed.avg --clock-control none -c 6 --csv --log-file gpurun_out/fp64_pipe.csv /tmp/fp64_peak > gpurun_out/fp64_peak.log 2>&1; echo "fp64 ncu rc=$?"
timeout 300 ncu --query-metrics > gpurun_out/ncu_metrics.txt 2>&1
ls gpurun_out
