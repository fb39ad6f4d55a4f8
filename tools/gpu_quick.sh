#!/bin/bash
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_grouped.py tests/test_gpu_parity.py -x -q 2>&1 | tail -5 > gpurun_out/pytest_q.txt
timeout 900 python bench.py --no-prefill --no-cpu-baseline > gpurun_out/bench_q.json 2> gpurun_out/bench_q.err
