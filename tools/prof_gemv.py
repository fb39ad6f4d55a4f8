"""Profiling driver: GEMV launches on one Llama-3.1-8B shape.

Default: a CUDA graph of --launches back-to-back calls over --copies rotating
weight copies, timed with CUDA events (device time per call, no host gaps).
--eager: plain launches (for ncu)."""
import argparse
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import paper_2602_01027_b200 as sfmp  # noqa: E402
from oracle.oracle import Port  # noqa: E402
from synth import LLAMA_8B, LLAMA_70B, activations, model_bytes  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--proj", default="gate_proj")
ap.add_argument("--model", default="8b")
ap.add_argument("--M", type=int, default=1)
ap.add_argument("--bits", type=float, default=3.25)
ap.add_argument("--m_b", type=int, default=512)
ap.add_argument("--launches", type=int, default=4)
ap.add_argument("--copies", type=int, default=1)
ap.add_argument("--path", type=int, default=sfmp.PATH_GEMV)
ap.add_argument("--eager", action="store_true")
args = ap.parse_args()
P = Port()
rows, cols = (LLAMA_8B if args.model == "8b" else LLAMA_70B)[args.proj]
data = model_bytes(P, rows, cols, args.bits, m_b=args.m_b)
dms = [sfmp.DeviceModel(data) for _ in range(args.copies)]
x = torch.from_numpy(activations(P, args.M, cols)).cuda().to(torch.bfloat16)
y = torch.empty(args.M, rows, device="cuda")
ws = dms[0].workspace(args.M, args.path)
for dm in dms:
    dm.gemm(x, out=y, path=args.path, workspace=ws)
torch.cuda.synchronize()


def run():
    for i in range(args.launches):
        dms[i % len(dms)].gemm(x, out=y, path=args.path, workspace=ws)


if args.eager:
    run()
    torch.cuda.synchronize()
    sys.exit(0)
s = torch.cuda.Stream()
g = torch.cuda.CUDAGraph()
with torch.cuda.graph(g, stream=s):
    run()
g.replay()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
reps = 5
e0.record()
for _ in range(reps):
    g.replay()
e1.record()
torch.cuda.synchronize()
t = e0.elapsed_time(e1) * 1e3 / (args.launches * reps)
pay = dms[0].info["payload_bytes"]
byts = pay + 4 * cols + 4 * rows + 2 * args.M * cols + 4 * args.M * rows
print(f"{args.model} {args.proj} M={args.M} bits={args.bits}: {t:.2f} us/call (graph), "
      f"{byts / t / 1e3:.1f} GB/s = {byts / t / 1e3 / 6550.7 * 100:.1f}% of 6550.7", flush=True)
