#!/bin/bash
# K1 timing (graph replay) at several M + ncu full captures of the grouped GEMV.
mkdir -p gpurun_out
for M in 1 4 8 16; do timeout 200 python tools/prof_group.py --M $M 2>&1 | tail -1; done > gpurun_out/k1_times.txt
timeout 200 python tools/prof_group.py --Ms 1,2,4,8 2>&1 | tail -1 >> gpurun_out/k1_times.txt
timeout 300 ncu --set full --clock-control none --import-source on -k regex:gemv_kernel -s 2 -c 1 -o gpurun_out/k1_m1 -f python tools/prof_group.py --M 1 --eager --launches 3 > gpurun_out/ncu_m1.log 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:gemv_kernel -s 2 -c 1 -o gpurun_out/k1_m16 -f python tools/prof_group.py --M 16 --eager --launches 3 > gpurun_out/ncu_m16.log 2>&1
cat gpurun_out/k1_times.txt
