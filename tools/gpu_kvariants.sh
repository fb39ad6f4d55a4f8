#!/bin/bash
# prefill points for each experiment build in variants/ (and the default library)
PTS="1024,4096,3.25,2048 4096,4096,3.25,2048 14336,4096,3.25,2048 4096,14336,3.25,2048 8192,28672,2.5,2048 8192,28672,2.5,64 8192,28672,2.5,256"
for v in default $(ls paper_2602_01027_b200/variants/ 2>/dev/null | sed 's/lib_//;s/.so//'); do
  if [ $v = default ]; then export SFMP_LIB=; else export SFMP_LIB=$PWD/paper_2602_01027_b200/variants/lib_$v.so; fi
  timeout 300 python tools/prefill_points.py $PTS 2>&1 | sed "s/^/$v /" | grep -v Warn
done
