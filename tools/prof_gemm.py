"""Prefill GEMM timing: CUDA graph of back-to-back calls, CUDA events, TFLOP/s."""
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
ap.add_argument("--proj", default="q_proj")
ap.add_argument("--model", default="8b")
ap.add_argument("--M", type=int, default=2048)
ap.add_argument("--bits", type=float, default=3.25)
ap.add_argument("--launches", type=int, default=8)
ap.add_argument("--eager", action="store_true")
ap.add_argument("--m_b", type=int, default=0, help="row block (0: synth default; the bench uses 128 for k/v)")
args = ap.parse_args()
P = Port()
rows, cols = (LLAMA_8B if args.model == "8b" else LLAMA_70B)[args.proj]
data = model_bytes(P, rows, cols, args.bits, **({'m_b': args.m_b} if args.m_b else {}))
dm = sfmp.DeviceModel(data)
x = torch.from_numpy(activations(P, args.M, cols)).cuda().to(torch.bfloat16)
y = torch.empty(args.M, rows, device="cuda")
ws = dm.workspace(args.M, sfmp.PATH_GEMM)
dm.gemm(x, out=y, path=sfmp.PATH_GEMM, workspace=ws)
torch.cuda.synchronize()
if args.eager:
    for _ in range(args.launches):
        dm.gemm(x, out=y, path=sfmp.PATH_GEMM, workspace=ws)
    torch.cuda.synchronize()
    sys.exit(0)
s = torch.cuda.Stream()
g = torch.cuda.CUDAGraph()
with torch.cuda.graph(g, stream=s):
    for _ in range(args.launches):
        dm.gemm(x, out=y, path=sfmp.PATH_GEMM, workspace=ws)
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
fl = 2.0 * args.M * rows * cols
print(f"{args.model} {args.proj} {rows}x{cols} M={args.M} bits={args.bits}: {t:.1f} us/call, "
      f"{fl / t / 1e6:.1f} TFLOP/s = {fl / t / 1e6 / 1678.6 * 100:.1f}% of 1678.6", flush=True)
