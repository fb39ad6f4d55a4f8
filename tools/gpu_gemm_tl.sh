#!/bin/bash
mkdir -p gpurun_out
{
timeout 120 python tools/gemm_timeline.py gate_proj 2048 | grep -A1 "interval\|afull -> mma commit\|deq wfull -> deq math"
timeout 120 python tools/gemm_timeline.py k_proj 2048 | grep -A1 "interval\|afull -> mma commit\|deq wfull -> deq math"
} > gpurun_out/gemm_tl.txt 2>&1
