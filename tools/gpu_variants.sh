#!/bin/bash
# Time the grouped decode GEMV for each experiment build in variants/ (and the default library).
for v in default $(ls paper_2602_01027_b200/variants/ 2>/dev/null | sed 's/lib_//;s/.so//'); do
  if [ $v = default ]; then export SFMP_LIB=; else export SFMP_LIB=$PWD/paper_2602_01027_b200/variants/lib_$v.so; fi
  for M in ${VARIANT_MS:-1 8 16}; do echo "$v M=$M $(timeout 120 python tools/prof_group.py --M $M 2>&1 | tail -1)"; done
  echo "$v Ms=1,2,4,8 $(timeout 120 python tools/prof_group.py --Ms 1,2,4,8 2>&1 | tail -1)"
done
