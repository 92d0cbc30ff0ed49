#!/bin/bash
mkdir -p gpurun_out
MM_UNIFORM=1 timeout 900 ncu --set full --import-source on --clock-control none -k regex:maxmin_cluster --launch-skip 1 -c 1 \
  -o gpurun_out/prof_maxmin -f python tools/maxmin_time.py 100000 > gpurun_out/prof_maxmin.log 2>&1
tail -5 gpurun_out/prof_maxmin.log
