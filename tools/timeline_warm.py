"""Warm timeline: replay a CUDA graph of calls (SFMP_GEMV_DEBUG=5) and dump the
stamps of the last call (weights rotated over copies, x/col_perm L2-warm)."""
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
dms = [sfmp.DeviceModel(model_bytes(P, rows, cols, 3.25)) for _ in range(8)]
x = torch.from_numpy(activations(P, M, cols)).cuda().to(torch.bfloat16)
y = torch.empty(M, rows, device="cuda")
ws = dms[0].workspace(M, sfmp.PATH_GEMV)
for d in dms:
    d.gemm(x, out=y, path=sfmp.PATH_GEMV, workspace=ws)
torch.cuda.synchronize()
st = torch.cuda.Stream()
g = torch.cuda.CUDAGraph()
with torch.cuda.graph(g, stream=st):
    for i in range(16):
        dms[i % 8].gemm(x, out=y, path=sfmp.PATH_GEMV, workspace=ws)
g.replay()
torch.cuda.synchronize()
g.replay()
torch.cuda.synchronize()
buf = np.zeros(512 * 128, np.uint64)
sfmp.lib().sfmp_debug_gemv_timeline(buf.ctypes.data_as(C.POINTER(C.c_ulonglong)), buf.size)
t = buf.reshape(512, 128).astype(np.int64)
valid = t[:511, 0] > 0
t0 = t[:511][valid, 0].min()
nunits = np.array([sum(1 for j in range(40) if 2 + 3 * j < 128 and t[c, 2 + 3 * j] >= t0) for c in range(511)])
sel = valid & (nunits > 0)
def pct(a):
    a = a[:511][sel]
    return " ".join(f"{np.percentile((a - t0) / 1e3, q):6.2f}" for q in (0, 10, 50, 90, 100))
last_done = np.array([t[c, 4 + 3 * (n - 1)] if n > 0 else 0 for c, n in enumerate(nunits)])
print(f"{proj} M={M} warm: percentiles (0/10/50/90/100) us")
print("  start      ", pct(t[:, 0]))
print("  first issue", pct(t[:, 2]))
print("  first full ", pct(t[:, 3]))
print("  last done  ", pct(np.concatenate([last_done, [0]])))
print("  end        ", pct(t[:, 1]))
