"""GEMM per-unit timeline of CTA 0 (SFMP_GEMM_DEBUG=32): intervals between pipeline events (ns)."""
import ctypes as C
import os
import sys

import numpy as np
import torch

os.environ["SFMP_GEMM_DEBUG"] = str(32 | int(os.environ.get("EXTRA_DBG", "0")))
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import paper_2602_01027_b200 as sfmp  # noqa: E402
from oracle.oracle import Port  # noqa: E402
from synth import LLAMA_8B, activations, model_bytes  # noqa: E402

proj = sys.argv[1] if len(sys.argv) > 1 else "k_proj"
import time as _time
M = int(sys.argv[2]) if len(sys.argv) > 2 else 2048
P = Port()
rows, cols = LLAMA_8B[proj]
dm = sfmp.DeviceModel(model_bytes(P, rows, cols, 3.25))
x = torch.from_numpy(activations(P, M, cols)).cuda().to(torch.bfloat16)
y = dm.gemm(x, path=sfmp.PATH_GEMM)
torch.cuda.synchronize()
y = dm.gemm(x, path=sfmp.PATH_GEMM)
torch.cuda.synchronize()
_ph = np.zeros(512 * 16, np.uint64)
sfmp.lib().sfmp_debug_gemm_phases(_ph.ctypes.data_as(C.POINTER(C.c_ulonglong)), C.c_size_t(_ph.size))  # clears
if os.environ.get("FLUSH"):
    _fl = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
    _fl.zero_()
    torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
e0.record()
y = dm.gemm(x, path=sfmp.PATH_GEMM)
e1.record()
torch.cuda.synchronize()
print(f"call time (events, incl. pre-pass): {e0.elapsed_time(e1) * 1e3:.1f} us")
buf = np.zeros(2 * 8 * 256, np.uint64)
sfmp.lib().sfmp_debug_gemm_timeline(buf.ctypes.data_as(C.POINTER(C.c_ulonglong)), C.c_size_t(buf.size))
t = buf.reshape(2, 8, 256).astype(np.int64)[0]
n = int((t[4] > 0).sum())
t0 = t[0, 0]
names = ["deq wfull", "deq math", "deq aempty", "deq afull", "mma afull", "mma xfull", "mma commit"]
print(f"{proj} M={M}: {n} units on CTA 0; times rel. to first wfull (us)")
ph = np.zeros(512 * 16, np.uint64)
sfmp.lib().sfmp_debug_gemm_phases(ph.ctypes.data_as(C.POINTER(C.c_ulonglong)), C.c_size_t(ph.size))
ph = ph.astype(np.int64).reshape(512, 16)
print("CTA 0 phases (us rel. to first wfull): entry %.2f setup %.2f firstW %.2f pdl_wait %.2f firstX %.2f exit %.2f"
      % tuple((ph[0, i] - t0) / 1e3 for i in range(6)))
live = ph[:, 0] > 0
e0_ = ph[live, 0].min()
for i, nm in enumerate(["entry", "setup", "firstW", "pdl_wait", "firstX", "exit", "W end", "X end", "MMA end",
                        "epi end", "deq end"]):
    v = (ph[live, i] - e0_) / 1e3
    print("  all %d CTAs %-8s (us rel. to first entry) p0 %.2f p50 %.2f p90 %.2f p100 %.2f" %
          (live.sum(), nm, *np.percentile(v, [0, 50, 90, 100])))
for k in list(range(0, min(n, 4))) + list(range(28, min(n, 38))) + list(range(max(6, n - 3), n)):
    print(f"unit {k:3d}: " + " ".join(f"{nm}={(t[i, k] - t0) / 1e3:7.2f}" for i, nm in enumerate(names)))
d = np.diff(t[4, :n]) / 1e3
print(f"mma afull-to-afull interval us: median {np.median(d):.3f} p90 {np.percentile(d, 90):.3f}")
for i, nm in enumerate(names[1:4], 1):
    print(f"  {names[i-1]} -> {nm}: median {np.median((t[i, :n] - t[i-1, :n])) / 1e3:.3f} us")
print(f"  deq afull -> mma afull: median {np.median(t[4, :n] - t[3, :n]) / 1e3:.3f} us")
print(f"  mma commit(k) -> deq aempty(k+2): median {np.median(t[2, 2:n] - t[6, :n-2]) / 1e3:.3f} us")
print(f"  mma afull -> mma commit: median {np.median(t[6, :n] - t[4, :n]) / 1e3:.3f} us")
ef = t[7][:128]; er = t[7][128:]
n_t = int((ef > 0).sum())
print("epilogue accfull:", (ef[:n_t] - t0) / 1e3)
print("epilogue acc released after (us):", (er[:n_t] - ef[:n_t]) / 1e3)
# per position-in-tile intervals (KC units per tile assumed 32)
iv = np.diff(t[4, :n]) / 1e3
pos = np.arange(1, n) % 32
for kpos in range(32):
    sel = iv[pos == kpos]
    if len(sel):
        print(f"  kc={kpos:2d}: afull interval median {np.median(sel):.3f} us; wfull-lead {np.median((t[4, 1:n][pos == kpos] - t[0, 1:n][pos == kpos]) / 1e3):.2f} us")
