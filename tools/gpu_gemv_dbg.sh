#!/bin/bash
mkdir -p gpurun_out
{
for sp in 0 4 8 16 32; do echo "SPLIT=$sp"; for proj in q_proj k_proj gate_proj down_proj; do SFMP_GEMV_SPLIT=$sp timeout 60 python tools/prof_gemv.py --proj $proj --M 1 --launches 24 --copies 12; done; done
for proj in q_proj gate_proj; do timeout 60 python tools/prof_gemv.py --proj $proj --M 16 --launches 24 --copies 12; done
timeout 60 python tools/timeline_warm.py q_proj 1
timeout 60 python tools/timeline_warm.py gate_proj 1
} > gpurun_out/gemv_dbg.txt 2>&1
