"""Grouped decode (the bench step for one M): the 7 Llama-3.1-8B linears in one launch.
--eager: plain launches for ncu; else graph + events timing.
SFMP_LIB=<variant .so> times an experiment build (tools/gpu_variants.sh)."""
import argparse
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import paper_2602_01027_b200 as sfmp  # noqa: E402
from oracle.oracle import Port  # noqa: E402
from synth import LLAMA_8B, activations, model_bytes  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--M", type=int, default=1)
ap.add_argument("--copies", type=int, default=4)
ap.add_argument("--launches", type=int, default=8)
ap.add_argument("--eager", action="store_true")
ap.add_argument("--order", default="", help="comma list of projections (default: LLAMA_8B order)")
ap.add_argument("--Ms", default="", help="comma list: one grouped call over these token counts "
                "(each on its own weight copy), as bench.py's step does for M<=8")
args = ap.parse_args()
P = Port()
projs = args.order.split(",") if args.order else list(LLAMA_8B)
datas = {p: model_bytes(P, *LLAMA_8B[p], 3.25, m_b=128 if p in ("k_proj", "v_proj") else 512,
                        seed={"up_proj": 4, "v_proj": 1}.get(p, 0)) for p in projs}
Ms = [int(v) for v in args.Ms.split(",")] if args.Ms else [args.M]
copies = max(args.copies, len(Ms))
models_c = [[sfmp.DeviceModel(datas[p]) for p in projs] for _ in range(copies)]
# problem list of one call: (copy, projection index, M)
keys = [(k % copies, j, M) for k, M in enumerate(Ms) for j in range(len(projs))]
xs = [torch.from_numpy(activations(P, M, LLAMA_8B[projs[j]][1])).cuda().to(torch.bfloat16) for c, j, M in keys]
ys = [torch.empty(M, LLAMA_8B[projs[j]][0], device="cuda") for c, j, M in keys]
ws = [torch.zeros_like(models_c[0][j].workspace(16, sfmp.PATH_GEMV)) for c, j, M in keys]
models = models_c  # (timeline code below uses models[0])
args.M = max(Ms)


def run():
    for i in range(args.launches):
        sfmp.gemm_grouped([models_c[(c + i) % copies][j] for c, j, M in keys], xs, outs=ys, workspaces=ws)


run()
torch.cuda.synchronize()
if args.eager:
    sys.exit(0)
s = torch.cuda.Stream()
g = torch.cuda.CUDAGraph()
with torch.cuda.graph(g, stream=s):
    run()
g.replay()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
e0.record()
for _ in range(5):
    g.replay()
e1.record()
torch.cuda.synchronize()
t = e0.elapsed_time(e1) * 1e3 / (5 * args.launches)
byts = sum(models_c[0][j].info["payload_bytes"] + 4 * models_c[0][j].cols + 4 * models_c[0][j].rows +
           2 * M * models_c[0][j].cols + 4 * M * models_c[0][j].rows for c, j, M in keys)
print(f"algorithmic bytes per call: {byts}")
print(f"grouped 8B layer M={args.Ms or args.M}: {t:.2f} us/launch, {byts / t / 1e3:.1f} GB/s = "
      f"{byts / t / 1e3 / 6514.2 * 100:.1f}% of 6514.2", flush=True)
