"""Time grouped decode launches of the Llama-3.1-8B layer (7 linears @3.25 b).

One grouped call per --groups entry (e.g. "1,2,4,8" = 28 problems in one
launch, "16" = 7 problems); weights rotate over --copies device copies (> L2).
CUDA graph replay, CUDA events; prints per-launch us and the fraction of the
measured HBM peak (algorithmic bytes).  --eager: a few plain
launches for ncu.
"""
import argparse
import json
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
ap.add_argument("--groups", default="1,2,4,8;16")
ap.add_argument("--dtype", default="bfloat16")
ap.add_argument("--copies", type=int, default=4)
ap.add_argument("--reps", type=int, default=20)
ap.add_argument("--model", default="8b")
ap.add_argument("--bits", type=float, default=3.25)
ap.add_argument("--eager", action="store_true")
ap.add_argument("--json", default="")
ap.add_argument("--timeline", action="store_true", help="per-CTA timeline (needs a -DSFMP_GEMV_TIMELINE=1 build)")
args = ap.parse_args()
P = Port()
SH = LLAMA_8B if args.model == "8b" else LLAMA_70B
projs = list(SH)
datas = {p: model_bytes(P, *SH[p], args.bits, m_b=128 if p in ("k_proj", "v_proj") else 512) for p in projs}
copies = [[sfmp.DeviceModel(datas[p]) for p in projs] for _ in range(args.copies)]
peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"] if os.path.exists(
    os.path.join(ROOT, "MEASURED_PEAKS.json")) else 6514.2
dt = getattr(torch, args.dtype)
out = {}
for grp in args.groups.split(";"):
    Ms = [int(v) for v in grp.split(",")]
    keys = [(j, M) for M in Ms for j in range(len(projs))]
    xs = [torch.from_numpy(activations(P, M, SH[projs[j]][1], seed=M)).cuda().to(dt) for j, M in keys]
    ys = [torch.empty(M, SH[projs[j]][0], device="cuda") for j, M in keys]
    ws = [[torch.zeros_like(copies[0][j].workspace(16, sfmp.PATH_GEMV)) for j, M in keys] for _ in range(2)]

    def run(n):
        for i in range(n):
            c = copies[i % len(copies)]
            sfmp.gemm_grouped([c[j] for j, M in keys], xs, outs=ys, workspaces=ws[i % 2])

    run(4)
    torch.cuda.synchronize()
    if args.eager:
        continue
    s = torch.cuda.Stream()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        run(2 * len(copies))
    g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(args.reps):
        g.replay()
    e1.record()
    torch.cuda.synchronize()
    t = e0.elapsed_time(e1) * 1e3 / (args.reps * 2 * len(copies))
    m0 = copies[0]
    esz = torch.tensor([], dtype=dt).element_size()
    byts = sum(m0[j].info["payload_bytes"] + 4 * m0[j].cols + 4 * m0[j].rows + esz * M * m0[j].cols +
               4 * M * m0[j].rows for j, M in keys)
    frac = byts / t / 1e3 / peak
    print(f"{args.model} layer M={grp} {args.dtype}: {t:.2f} us/launch  {byts / 1e6:.1f} MB  "
          f"{byts / t / 1e3:.0f} GB/s = {frac * 100:.1f}% of {peak}", flush=True)
    out[grp] = {"us": t, "bytes": byts, "frac": frac}
    if args.timeline:
        import ctypes as C
        import numpy as np
        run(1)
        torch.cuda.synchronize()
        buf = np.zeros(4096 * 4 + 16, np.uint64)
        sfmp.lib().sfmp_debug_gemv_timeline(buf.ctypes.data_as(C.POINTER(C.c_ulonglong)), C.c_size_t(buf.size))
        run(1)  # the kernel-level stamps were reset by the first read: one clean launch
        torch.cuda.synchronize()
        sfmp.lib().sfmp_debug_gemv_timeline(buf.ctypes.data_as(C.POINTER(C.c_ulonglong)), C.c_size_t(buf.size))
        kk = buf[4096 * 4:].astype(np.int64)
        tl = buf[:4096 * 4].reshape(4096, 4).astype(np.int64)
        tl = tl[tl[:, 0] > 0]
        t0 = tl[:, 0].min()
        st, en, sm, it = (tl[:, 0] - t0) / 1e3, (tl[:, 1] - t0) / 1e3, tl[:, 2], tl[:, 3]
        sm_end = np.array([en[sm == k].max() for k in np.unique(sm)])
        sm_busy = np.array([(en[sm == k] - st[sm == k]).sum() for k in np.unique(sm)])
        pct = lambda a: " ".join(f"{np.percentile(a, q):6.2f}" for q in (0, 10, 50, 90, 100))
        print(f"  CTAs {len(tl)}  start p0/10/50/90/100 {pct(st)}")
        print(f"  CTA end            {pct(en)}")
        print(f"  SM  end            {pct(sm_end)}")
        print(f"  items/CTA          {pct(it)}")
        print(f"  SM busy CTA-us     {pct(sm_busy)}")
        z = kk[0]
        print("  kernels (us from xprep start): xprep %.2f..%.2f  gemv %.2f..%.2f  fixup %.2f..%.2f" %
              tuple((kk[i] - z) / 1e3 if kk[i] > 0 and kk[i] < 2**62 else -1 for i in range(6)))
if args.json:
    json.dump(out, open(args.json, "w"), indent=1)
