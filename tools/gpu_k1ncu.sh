#!/bin/bash
# ncu full captures of the grouped decode GEMV (M=1 layer, and the bench's M<=8 launch).
mkdir -p gpurun_out
timeout 300 ncu --set full --clock-control none --import-source on -k regex:gemv_kernel -s 2 -c 1 -o gpurun_out/k1_m1 -f python tools/prof_group.py --M 1 --eager --launches 3 > gpurun_out/ncu_m1.log 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:gemv_kernel -s 2 -c 1 -o gpurun_out/k1_mle8 -f python tools/prof_group.py --Ms 1,2,4,8 --eager --launches 3 > gpurun_out/ncu_mle8.log 2>&1
ls -la gpurun_out/*.ncu-rep
