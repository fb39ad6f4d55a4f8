#!/bin/bash
mkdir -p gpurun_out
nvidia-smi --query-gpu=clocks.sm,power.draw,clocks_event_reasons.active --format=csv,noheader -lms 50 > gpurun_out/clk_gemm.csv &
SMI=$!
sleep 1
timeout 120 python tools/prof_gemm.py --proj gate_proj --M 2048 --launches 200 > gpurun_out/gemm_clk.txt 2>&1
kill $SMI
