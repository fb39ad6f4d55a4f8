#!/bin/bash
# ncu evidence for profiles/: full captures of the two hot kernels + the bench launch list.
mkdir -p gpurun_out
timeout 300 ncu --set full --clock-control none --import-source on -k regex:gemm_kernel -s 1 -c 1 -o gpurun_out/prof_gemm_gate -f python tools/prof_gemm.py --proj gate_proj --M 2048 --eager --launches 2 > gpurun_out/ncu1.log 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:gemv_kernel -s 2 -c 1 -o gpurun_out/prof_gemv_group_m1 -f python tools/prof_group.py --M 1 --eager --launches 3 > gpurun_out/ncu2.log 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:gemv_kernel -s 2 -c 1 -o gpurun_out/prof_gemv_group_m16 -f python tools/prof_group.py --M 16 --eager --launches 3 > gpurun_out/ncu3.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 1 --no-graph --no-cpu-baseline --soak-ms 0 > gpurun_out/b_ncu.log 2>&1
ls -la gpurun_out/*.ncu-rep
