"""Time K2 (prefill GEMM) points: graph replay over 2 weight copies, CUDA events.
usage: prefill_points.py rows,cols,bits,M [...]"""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import paper_2602_01027_b200 as sfmp  # noqa: E402
from oracle.oracle import Port  # noqa: E402
from synth import model_bytes, prebuild  # noqa: E402



def main():
    P = Port()
    pts = [tuple(float(v) if i == 2 else int(v) for i, v in enumerate(a.split(","))) for a in sys.argv[1:]]
    prebuild([(r, c, b, {}) for r, c, b, M in pts])
    for r, c, b, M in pts:
        data = model_bytes(P, r, c, b)
        ms = [sfmp.DeviceModel(data) for _ in range(2)]
        x = torch.from_numpy(P.gen_activation(M, c, 9)).cuda().to(torch.bfloat16)
        y = torch.empty(M, r, device="cuda")
        ws = ms[0].workspace(M, sfmp.PATH_AUTO)
        s = torch.cuda.Stream()
        with torch.cuda.stream(s):
            for m in ms:
                m.gemm(x, out=y, workspace=ws, stream=s)
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            for m in ms:
                m.gemm(x, out=y, workspace=ws, stream=s)
        g.replay()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        reps = 5
        with torch.cuda.stream(s):
            e0.record(s)
            for _ in range(reps):
                g.replay()
            e1.record(s)
        torch.cuda.synchronize()
        us = e0.elapsed_time(e1) * 1e3 / (reps * 2)
        tf = 2.0 * M * r * c / us / 1e6
        print(f"{r}x{c} b{b} M={M}: {us:.1f} us  {tf:.0f} TFLOP/s  {tf / 1648:.3f} of peak", flush=True)


if __name__ == "__main__":
    main()
