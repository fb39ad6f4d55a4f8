#!/bin/bash
mkdir -p gpurun_out
{
timeout 300 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -2
for sp in 0 4 8 16; do echo "SPLIT=$sp"; for M in 1 16; do for proj in q_proj k_proj gate_proj down_proj; do SFMP_GEMV_SPLIT=$sp timeout 60 python tools/prof_gemv.py --proj $proj --M $M --launches 24 --copies 12; done; done; done
timeout 60 python tools/prof_gemv.py --model 70b --proj down_proj --M 1 --bits 2.5 --launches 12 --copies 4
timeout 60 python tools/timeline_warm.py q_proj 1
timeout 60 python tools/timeline_warm.py gate_proj 1
} > gpurun_out/gemv_dbg.txt 2>&1
