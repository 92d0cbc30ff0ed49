#!/bin/bash
# maxmin ordering: memcheck on a small case, parity tests, timing on the B200
mkdir -p gpurun_out
timeout 300 compute-sanitizer --tool memcheck --print-limit 5 python -c "
import sys; sys.path.insert(0, '.')
import numpy as np, paper_2403_07412_b200 as vg
for n in (1, 2, 700, 3000, 70000):
    vg.geo.maxmin_ordering(np.random.default_rng(n).random((n, 2)))
print('memcheck run done')" 2>&1 | tail -4
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k maxmin 2>&1 | tail -15
timeout 900 python tools/maxmin_time.py ${MM_SIZES:-250000 1000000 2000000} 2>&1 | tee gpurun_out/maxmin.jsonl
