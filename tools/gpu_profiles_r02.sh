#!/bin/bash
# Round-2 ncu evidence: full captures of the decode GEMV (bench's M<=8 and M=16
# launches) and of the prefill GEMM (8B gate, 70B down at M=2048), plus the
# bench launch list.  Summaries -> profiles/r02_*.json (tools/ncu_summary.py).
mkdir -p gpurun_out
timeout 300 ncu --set full --clock-control none --import-source on -k regex:gemv_kernel -s 2 -c 1 -o gpurun_out/r02_gemv_mle8 -f python tools/prof_group.py --Ms 1,2,4,8 --eager --launches 3 > gpurun_out/n1.log 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:gemv_kernel -s 2 -c 1 -o gpurun_out/r02_gemv_m16 -f python tools/prof_group.py --M 16 --eager --launches 3 > gpurun_out/n2.log 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:gemm_kernel -s 1 -c 1 -o gpurun_out/r02_gemm_gate8b -f python tools/prof_gemm.py --proj gate_proj --M 2048 --eager --launches 2 > gpurun_out/n3.log 2>&1
timeout 400 ncu --set full --clock-control none --import-source on -k regex:gemm_kernel -s 1 -c 1 -o gpurun_out/r02_gemm_down70b -f python tools/prof_gemm.py --model 70b --proj down_proj --bits 2.5 --M 2048 --eager --launches 2 > gpurun_out/n4.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 400 --csv --log-file gpurun_out/r02_launches.csv python bench.py --steps 2 --warmup 3 --no-graph --no-cpu-baseline --no-extras --no-prefill --soak-ms 0 > gpurun_out/n5.log 2>&1
ls -la gpurun_out/*.ncu-rep gpurun_out/r02_launches.csv
