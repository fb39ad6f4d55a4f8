#!/bin/bash
for M in 1 16; do timeout 120 python tools/prof_group.py --M $M 2>&1 | tail -1; done
timeout 120 python tools/prof_group.py --Ms 1,2,4,8 2>&1 | tail -1
timeout 200 python bench.py --steps 20 --warmup 3 --no-prefill --no-cpu-baseline --soak-ms 200 > gpurun_out/b.txt 2>gpurun_out/b.err; python - <<'PY'
import json
d=json.loads(open('gpurun_out/b.txt').read().strip().splitlines()[-1])
print("step",d["value"],"e2e",d["e2e"]["value"], json.dumps(d["roofline"]["per_launch"]))
for k in ("config0","mode_none","n_b_256","dropin_gemv_host"): print(k, d["extras"][k])
print("70b", d["extras"]["llama70b"]["decode_step"])
s=d["extras"]["sweep_8192x28672"]; print({k:(v["us"],v["frac"]) for k,v in s.items()})
PY
timeout 600 python -m pytest tests/test_gpu_domain.py tests/test_gpu_grouped.py tests/test_gpu_sharded.py tests/test_gpu_sharded_group.py tests/test_gpu_parity.py -x -q 2>&1 | tail -2
