#!/bin/bash
# prefill GEMM points for the default build and each prefill experiment build
# given on the command line (paper_2602_01027_b200/variants/lib_<name>.so, make gvariant)
for v in default "$@"; do
  if [ $v = default ]; then export SFMP_LIB=; else export SFMP_LIB=$PWD/paper_2602_01027_b200/variants/lib_$v.so; fi
  timeout 300 python tools/sweep.py --bits 3.0 --Ms 32,64,128,256,2048 --out gpurun_out/sweep_$v.json 2>&1 | grep '"M"' | python -c "
import sys,json
for l in sys.stdin: d=json.loads(l); print('$v', 'M=%d'%d['M'], d['us'], 'us frac', d['frac'])"
  for pr in q_proj k_proj down_proj; do echo "$v 8b $pr $(timeout 120 python tools/prof_gemm.py --proj $pr --M 2048 2>&1 | tail -1)"; done
done
