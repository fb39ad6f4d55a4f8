#!/bin/bash
# ncu full capture of the bench step's single grouped GEMV launch (35 problems, M=1..16) + the bench line.
mkdir -p gpurun_out
timeout 300 ncu --set full --clock-control none --import-source on -k regex:gemv_kernel -s 2 -c 1 -o gpurun_out/r02_gemv_step -f python tools/prof_group.py --Ms 1,2,4,8,16 --eager --launches 3 > gpurun_out/n6.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 400 --csv --log-file gpurun_out/r02_launches.csv python bench.py --steps 2 --warmup 3 --no-graph --no-cpu-baseline --no-extras --no-prefill --soak-ms 0 > gpurun_out/n5.log 2>&1
timeout 900 python bench.py > gpurun_out/bench_full.txt 2> gpurun_out/bench_full.err
tail -2 gpurun_out/bench_full.err
