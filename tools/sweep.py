"""configs[4]: average bit-width 2.0-4.0 x batch M 1-4096 on the 8192 x 28672
linear (Llama-3.1-70B down_proj shape); per point: device time per call (CUDA
graph of back-to-back calls over rotating weight copies, CUDA events), the
roofline time t* = max(bytes / HBM, flops / TC) from MEASURED_PEAKS.json and
the achieved fraction t* / t.  Writes one JSON (default profiles/r01_sweep_8192x28672.json)."""
import argparse
import json
import os
import sys
import time

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import paper_2602_01027_b200 as sfmp  # noqa: E402
from oracle.oracle import Port  # noqa: E402
from synth import activations, model_bytes  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--rows", type=int, default=8192)
ap.add_argument("--cols", type=int, default=28672)
ap.add_argument("--bits", default="2.0,2.5,3.0,3.5,4.0")
ap.add_argument("--Ms", default="1,2,4,8,16,32,64,128,256,512,1024,2048,4096")
ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "r01_sweep_8192x28672.json"))
args = ap.parse_args()
peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
HBM, TC = float(peaks["hbm_gbs"]), float(peaks["bf16_tflops"])
P = Port()
res = {"shape": [args.rows, args.cols], "peaks": {"hbm_gbs": HBM, "bf16_tflops": TC}, "points": []}
for b in [float(v) for v in args.bits.split(",")]:
    t0 = time.time()
    data = model_bytes(P, args.rows, args.cols, b)
    copies = 2 if b >= 3.0 else 3
    models = [sfmp.DeviceModel(data) for _ in range(copies)]
    info = models[0].info
    for M in [int(v) for v in args.Ms.split(",")]:
        x = torch.from_numpy(activations(P, M, args.cols, seed=M)).cuda().to(torch.bfloat16)
        y = torch.empty(M, args.rows, device="cuda")
        ws = models[0].workspace(M)
        for m in models:
            m.gemm(x, out=y, workspace=ws)
        torch.cuda.synchronize()
        reps = 8 if M <= 256 else 3
        s = torch.cuda.Stream()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            for i in range(reps):
                models[i % copies].gemm(x, out=y, workspace=ws)
        g.replay()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        e0.record()
        for _ in range(3):
            g.replay()
        e1.record()
        torch.cuda.synchronize()
        us = e0.elapsed_time(e1) * 1e3 / (3 * reps)
        byts = info["payload_bytes"] + 4 * args.cols + 4 * args.rows + 2 * M * args.cols + 4 * M * args.rows
        flops = 2.0 * M * args.rows * args.cols
        t_hbm, t_tc = byts / HBM / 1e3, flops / TC / 1e6
        tstar = max(t_hbm, t_tc)
        pt = {"avg_code_bits": b, "M": M, "path": "gemv" if M <= 16 else "gemm", "us": round(us, 2),
              "GBps": round(byts / us / 1e3, 1), "TFLOPs": round(flops / us / 1e6, 1),
              "bound": "hbm" if t_hbm >= t_tc else "tensor", "t_star_us": round(tstar, 2),
              "frac": round(tstar / us, 4)}
        res["points"].append(pt)
        print(json.dumps(pt), flush=True)
        del g
    del models
    torch.cuda.empty_cache()
    print(f"bits {b}: {time.time() - t0:.0f}s", flush=True)
json.dump(res, open(args.out, "w"), indent=1)
