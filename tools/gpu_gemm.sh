#!/bin/bash
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_gemm.py -x -q 2>&1 | tail -15 > gpurun_out/pytest_gemm.txt
{
for proj in q_proj k_proj gate_proj down_proj; do timeout 120 python tools/prof_gemm.py --proj $proj --M 2048; done
timeout 120 python tools/prof_gemm.py --proj q_proj --M 256
} > gpurun_out/gemm_timing.txt 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:gemm_kernel -s 1 -c 1 -o gpurun_out/prof_gemm -f python tools/prof_gemm.py --proj gate_proj --M 2048 --eager --launches 2 > gpurun_out/ncu_gemm.log 2>&1
