#!/bin/bash
# K1 iteration loop: decode parity tests + grouped timings.
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_grouped.py tests/test_gpu_domain.py tests/test_gpu_sharded.py -x -q 2>&1 | tail -15 > gpurun_out/k1_tests.txt
for M in 1 4 8 16; do timeout 200 python tools/prof_group.py --M $M 2>&1 | tail -1; done > gpurun_out/k1_times.txt
timeout 200 python tools/prof_group.py --Ms 1,2,4,8 2>&1 | tail -1 >> gpurun_out/k1_times.txt
cat gpurun_out/k1_tests.txt gpurun_out/k1_times.txt
