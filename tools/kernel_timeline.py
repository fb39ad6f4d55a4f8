"""Per-kernel device timestamps of GEMM calls replayed in a CUDA graph (SFMP_GEMV_DEBUG=5)."""
import ctypes as C
import os
import sys

import numpy as np
import torch

os.environ["SFMP_GEMV_DEBUG"] = "5"
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import paper_2602_01027_b200 as sfmp  # noqa: E402
from oracle.oracle import Port  # noqa: E402
from synth import LLAMA_8B, activations, model_bytes  # noqa: E402

proj = sys.argv[1] if len(sys.argv) > 1 else "q_proj"
M = int(sys.argv[2]) if len(sys.argv) > 2 else 1
P = Port()
rows, cols = LLAMA_8B[proj]
dms = [sfmp.DeviceModel(model_bytes(P, rows, cols, 3.25)) for _ in range(4)]
x = torch.from_numpy(activations(P, M, cols)).cuda().to(torch.bfloat16)
y = torch.empty(M, rows, device="cuda")
ws = dms[0].workspace(M, sfmp.PATH_GEMV)
for d in dms:
    d.gemm(x, out=y, path=sfmp.PATH_GEMV, workspace=ws)
torch.cuda.synchronize()
buf = np.zeros(512 * 128, np.uint64)
for k in range(3):
    dms[k % 4].gemm(x, out=y, path=sfmp.PATH_GEMV, workspace=ws)
    torch.cuda.synchronize()
sfmp.lib().sfmp_debug_gemv_timeline(buf.ctypes.data_as(C.POINTER(C.c_ulonglong)), buf.size)
t = buf.reshape(512, 128).astype(np.int64)
k = t[511, 100:106]
gemv_start = t[:511, 0][t[:511, 0] > 0].min()
gemv_end = max(t[:511, 1].max(), k[3])
print(f"{proj} M={M} (eager call): xprep start 0, xprep end {(k[1]-k[0])/1e3:.2f}, gemv first CTA start "
      f"{(gemv_start-k[0])/1e3:.2f}, gemv end {(gemv_end-k[0])/1e3:.2f}, reduce start {(k[4]-k[0])/1e3:.2f}, "
      f"reduce after wait {(k[5]-k[0])/1e3:.2f} us")
