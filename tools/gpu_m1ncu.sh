#!/bin/bash
# ncu full capture of the single-linear decode GEMV on 8192x28672 at M=1 (2.0 and 4.0 bits)
mkdir -p gpurun_out
for b in 2.0 4.0; do
  python tools/prof_gemv.py --model 70b --proj down_proj --bits $b --M 1 2>&1 | tail -1
  timeout 300 ncu --set full --clock-control none --import-source on -k regex:gemv_kernel -s 2 -c 1 -o gpurun_out/k1_m1_b$b -f python tools/prof_gemv.py --model 70b --proj down_proj --bits $b --M 1 --eager --launches 3 > gpurun_out/ncu_m1_b$b.log 2>&1
done
ls gpurun_out/*.ncu-rep
