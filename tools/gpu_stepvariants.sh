#!/bin/bash
# the one-launch decode step (8B layer; default M=1..16) for each experiment build in variants/
MS=${MS:-1,2,4,8,16}
for v in default $(ls paper_2602_01027_b200/variants/ 2>/dev/null | sed 's/lib_//;s/.so//'); do
  if [ $v = default ]; then export SFMP_LIB=; else export SFMP_LIB=$PWD/paper_2602_01027_b200/variants/lib_$v.so; fi
  echo "$v $(timeout 120 python tools/prof_group.py --Ms $MS 2>&1 | tail -1)"
done
