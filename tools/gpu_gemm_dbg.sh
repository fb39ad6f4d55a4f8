#!/bin/bash
mkdir -p gpurun_out
{
for c in 1 2 4; do for d in 0 16 23; do echo "CLUSTER=$c DEBUG=$d"; for proj in k_proj gate_proj; do SFMP_GEMM_CLUSTER=$c SFMP_GEMM_DEBUG=$d timeout 120 python tools/prof_gemm.py --proj $proj --M 2048; done; done; done
echo "xprep only"; SFMP_GEMM_DEBUG=8 timeout 120 python tools/prof_gemm.py --proj gate_proj --M 2048
} > gpurun_out/gemm_dbg.txt 2>&1
