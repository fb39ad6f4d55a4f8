#!/bin/bash
# prefill GEMM points (8B q/k/down, 70B q) for each experiment build in variants/
for v in default $(ls paper_2602_01027_b200/variants/ 2>/dev/null | sed 's/lib_//;s/.so//'); do
  if [ $v = default ]; then export SFMP_LIB=; else export SFMP_LIB=$PWD/paper_2602_01027_b200/variants/lib_$v.so; fi
  for pr in q_proj k_proj down_proj; do echo "$v $(timeout 120 python tools/prof_gemm.py --proj $pr --M 2048 2>&1 | tail -1)"; done
  echo "$v $(timeout 200 python tools/prof_gemm.py --model 70b --proj q_proj --bits 2.5 --M 2048 2>&1 | tail -1)"
done
