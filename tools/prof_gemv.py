"""Profiling driver: a few GEMV launches on one Llama-3.1-8B shape (for ncu), plus a
back-to-back event timing of N launches over rotating weight copies."""
import argparse
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import paper_2602_01027_b200 as sfmp  # noqa: E402
from oracle.oracle import Port  # noqa: E402
from synth import LLAMA_8B, activations, model_bytes  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--proj", default="gate_proj")
ap.add_argument("--M", type=int, default=1)
ap.add_argument("--bits", type=float, default=3.25)
ap.add_argument("--launches", type=int, default=4)
ap.add_argument("--copies", type=int, default=1)
ap.add_argument("--path", type=int, default=sfmp.PATH_GEMV)
args = ap.parse_args()
P = Port()
rows, cols = LLAMA_8B[args.proj]
data = model_bytes(P, rows, cols, args.bits)
dms = [sfmp.DeviceModel(data) for _ in range(args.copies)]
x = torch.from_numpy(activations(P, args.M, cols)).cuda().to(torch.bfloat16)
y = torch.empty(args.M, rows, device="cuda")
for dm in dms:
    dm.gemm(x, out=y, path=args.path)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
e0.record()
for i in range(args.launches):
    dms[i % len(dms)].gemm(x, out=y, path=args.path)
e1.record()
torch.cuda.synchronize()
t = e0.elapsed_time(e1) * 1e3 / args.launches
pay = dms[0].info["payload_bytes"]
byts = pay + 4 * cols + 4 * rows + 2 * args.M * cols + 4 * args.M * rows
print(f"{args.proj} M={args.M} bits={args.bits}: {t:.2f} us/launch (incl. host gaps), "
      f"{byts / t / 1e3:.1f} GB/s", flush=True)
