"""Quick diagnostic: time the decode GEMV on Llama-3.1-8B shapes (CUDA events, L2 rotated)."""
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import paper_2602_01027_b200 as sfmp  # noqa: E402
from oracle.oracle import Port  # noqa: E402
from synth import LLAMA_8B, activations, errors, model_bytes  # noqa: E402

P = Port()
flush = torch.empty(512 * 1024 * 1024, dtype=torch.uint8, device="cuda")
for proj, (rows, cols) in LLAMA_8B.items():
    if proj in ("v_proj", "up_proj"):
        continue
    data = model_bytes(P, rows, cols, 3.25)
    dm = sfmp.DeviceModel(data)
    pay = dm.info["payload_bytes"]
    for M in (1, 8, 16):
        x = torch.from_numpy(activations(P, M, cols)).cuda().to(torch.bfloat16)
        y = dm.gemm(x, path=sfmp.PATH_GEMV)
        torch.cuda.synchronize()
        ts = []
        for it in range(12):
            flush.zero_()
            e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
            e0.record()
            dm.gemm(x, out=y, path=sfmp.PATH_GEMV)
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1) * 1e3)
        t = float(np.median(ts[2:]))
        byts = pay + 4 * cols + 4 * rows + 2 * M * cols + 4 * M * rows
        print(f"{proj:10s} {rows}x{cols} M={M:2d}: {t:8.2f} us  {byts / t / 1e3:8.1f} GB/s  "
              f"({byts / t / 1e3 / 6550.7 * 100:5.1f}% of 6550.7)", flush=True)
    ref = P.matmul(activations(P, 16, cols), P.load(data).dequantize(), threads=8)
    print("   err", errors(y.cpu().numpy(), ref))
