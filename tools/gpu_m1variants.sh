#!/bin/bash
# single-linear M=1 decode on 8192x28672 at 2.0 / 4.0 bits + the 8B step, for each build in variants/
for v in default $(ls paper_2602_01027_b200/variants/ 2>/dev/null | sed 's/lib_//;s/.so//'); do
  if [ $v = default ]; then export SFMP_LIB=; else export SFMP_LIB=$PWD/paper_2602_01027_b200/variants/lib_$v.so; fi
  for b in 2.0 4.0; do echo "$v $(timeout 120 python tools/prof_gemv.py --model 70b --proj down_proj --bits $b --M 1 --copies 3 2>&1 | tail -1)"; done
  echo "$v $(timeout 120 python tools/prof_group.py --Ms 1,2,4,8,16 2>&1 | tail -1)"
done
