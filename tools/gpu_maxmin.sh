#!/bin/bash
# maxmin ordering: parity tests + timing on the B200
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k maxmin 2>&1 | tail -15
timeout 900 python tools/maxmin_time.py 250000 1000000 2000000 2>&1 | tee gpurun_out/maxmin.jsonl
