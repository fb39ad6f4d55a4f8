"""Dump the per-CTA unit timeline of one GEMV launch (SFMP_GEMV_DEBUG=5)."""
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

proj = sys.argv[1] if len(sys.argv) > 1 else "gate_proj"
M = int(sys.argv[2]) if len(sys.argv) > 2 else 1
P = Port()
rows, cols = LLAMA_8B[proj]
dm = sfmp.DeviceModel(model_bytes(P, rows, cols, 3.25))
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
x = torch.from_numpy(activations(P, M, cols)).cuda().to(torch.bfloat16)
y = torch.empty(M, rows, device="cuda")
for _ in range(3):
    dm.gemm(x, out=y, path=sfmp.PATH_GEMV)
flush.zero_()
torch.cuda.synchronize()
dm.gemm(x, out=y, path=sfmp.PATH_GEMV)
torch.cuda.synchronize()
buf = np.zeros(512 * 128, np.uint64)
sfmp.lib().sfmp_debug_gemv_timeline(buf.ctypes.data_as(C.POINTER(C.c_ulonglong)), buf.size)
t = buf.reshape(512, 128).astype(np.int64)
valid = t[:, 0] > 0
t0 = t[valid, 0].min()
print(f"{proj} M={M}: CTAs {valid.sum()}, kernel span {(t[valid,1].max()-t0)/1e3:.2f} us; "
      f"start spread {(t[valid,0].max()-t0)/1e3:.2f} us")
for c in list(range(0, 6)) + [100, 200, 300]:
    if not valid[c]:
        continue
    r = t[c]
    n = 0
    while 2 + 3 * n < 128 and r[2 + 3 * n] > 0:
        n += 1
    iss = (r[2:2 + 3 * n:3] - t0) / 1e3
    full = (r[3:3 + 3 * n:3] - t0) / 1e3
    done = (r[4:4 + 3 * n:3] - t0) / 1e3
    print(f"cta {c:3d}: start {(r[0]-t0)/1e3:6.2f} end {(r[1]-t0)/1e3:6.2f}  units {n}")
    print("   issue", np.round(iss, 2).tolist())
    print("   full ", np.round(full, 2).tolist())
    print("   done ", np.round(done, 2).tolist())
# distribution over all recorded CTAs
nunits = np.array([sum(1 for j in range(40) if 2 + 3 * j < 128 and t[c, 2 + 3 * j] > 0) for c in range(512)])
sel = valid & (nunits > 0)
def pct(a):
    a = a[sel]
    return " ".join(f"{np.percentile((a - t0) / 1e3, q):6.2f}" for q in (0, 10, 50, 90, 100))
first_issue = t[:, 2]
first_full = t[:, 3]
last_done = np.array([t[c, 4 + 3 * (n - 1)] if n > 0 else 0 for c, n in enumerate(nunits)])
print("percentiles (0/10/50/90/100) us")
print("  start      ", pct(t[:, 0]))
print("  first issue", pct(first_issue))
print("  first full ", pct(first_full))
print("  last done  ", pct(last_done))
print("  end        ", pct(t[:, 1]))
print("  units/CTA  ", np.bincount(nunits[sel]).tolist())
