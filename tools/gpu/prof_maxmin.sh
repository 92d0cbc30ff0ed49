mkdir -p gpurun_out
timeout 1500 ncu --section SpeedOfLight --section Occupancy --section SchedulerStats --section WarpStateStats --section MemoryWorkloadAnalysis --clock-control none -k regex:maxmin_cluster -c 1 -o /tmp/mm python tools/prof_aux.py maxmin > gpurun_out/r02_ncu_maxmin.log 2>&1; echo rc=$?
ncu -i /tmp/mm.ncu-rep --page raw --csv > gpurun_out/r02_ncu_maxmin.raw.csv 2>/dev/null
ncu -i /tmp/mm.ncu-rep --page details --csv > gpurun_out/r02_ncu_maxmin.details.csv 2>/dev/null
