"""Grouped decode (the bench step for one M): the 7 Llama-3.1-8B linears in one launch.
--eager: plain launches for ncu; else graph + events timing.
SFMP_GEMV_DEBUG=5 prints the per-CTA timeline; its per-unit stamps need a build with
`make -C paper_2602_01027_b200 EXTRA=-DSFMP_GEMV_TIMELINE=1`."""
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

if os.environ.get("SFMP_GEMV_DEBUG") == "5":
    import ctypes as C
    import numpy as np
    g.replay()
    torch.cuda.synchronize()
    buf = np.zeros(512 * 128, np.uint64)
    sfmp.lib().sfmp_debug_gemv_timeline(buf.ctypes.data_as(C.POINTER(C.c_ulonglong)), C.c_size_t(buf.size))
    t = buf.reshape(512, 128).astype(np.int64)
    valid = t[:511, 0] > 0
    t0 = t[:511][valid, 0].min()
    nun = np.array([sum(1 for j in range(40) if 2 + 3 * j < 128 and t[c, 2 + 3 * j] >= t0) for c in range(511)])
    sel = valid & (nun > 0)

    def pct(a):
        a = a[:511][sel]
        return " ".join(f"{np.percentile((a - t0) / 1e3, q):6.2f}" for q in (0, 10, 50, 90, 100))
    last = np.array([t[c, 4 + 3 * (n - 1)] if n > 0 else 0 for c, n in enumerate(nun)])
    print("timeline (us) percentiles 0/10/50/90/100 over CTAs 0..510")
    print("  start      ", pct(t[:, 0]))
    print("  first issue", pct(t[:, 2]))
    print("  first full ", pct(t[:, 3]))
    print("  last done  ", pct(np.concatenate([last, [0]])))
    print("  end        ", pct(t[:, 1]))
    print("  units/CTA  ", np.percentile(nun[sel], [0, 50, 100]))
    print("  xprep first CTA start / last CTA end (us, rel. to first GEMV CTA start): %.2f / %.2f" %
          ((t[511, 100] - t0) / 1e3, (t[511, 101] - t0) / 1e3))
    print("  GEMV grid %d, last CTA end (all CTAs) %.2f us; launch period %.2f us; prev GEMV end -> xprep start %.2f us" %
          (t[511, 103], (t[511, 102] - t0) / 1e3, e0.elapsed_time(e1) * 1e3 / (5 * args.launches),
           (t[511, 100] - t[511, 104]) / 1e3))
    ce = (t[:511, 127] - t0) / 1e3
    order = np.argsort(-np.where(sel, ce, -1))[:8]
    print("  latest compute ends (cta: end, last unit done, last seam barrier, flag, fixup end):")
    for c in order:
        n = nun[c]
        print("    %4d: %6.2f %6.2f %6.2f %6.2f %6.2f" % (c, ce[c], (t[c, 4 + 3 * (n - 1)] - t0) / 1e3,
              (t[c, 124] - t0) / 1e3, (t[c, 125] - t0) / 1e3, (t[c, 126] - t0) / 1e3 if t[c, 126] > t0 else -1))
    sm = t[:511, 123]
    ends = {}
    for c in np.where(sel)[0]:
        ends.setdefault(int(sm[c]), []).append(ce[c])
    sm_last = np.array([max(v) for v in ends.values()])
    if os.environ.get("SM_DUMP"):
        np.save(os.environ["SM_DUMP"], np.array([[k, max(v), min(v), len(v)] for k, v in sorted(ends.items())]))
    sm_first = np.array([min(v) for v in ends.values()])
    print("  per-SM (%d SMs) latest compute end p0/p10/p50/p90/p100: %s" % (len(ends), " ".join("%.2f" % np.percentile(sm_last, q) for q in (0, 10, 50, 90, 100))))
    print("  per-SM earliest CTA end p0/p50/p100: %s" % " ".join("%.2f" % np.percentile(sm_first, q) for q in (0, 50, 100)))
    hb = t[:511, 122]
    busy = (last[:511] - t[:511, 3]) / 1e3
    ok = sel & (nun > 0)
    if hb[ok].any():  # (needs a build that counts ceil-bit units in slot 122)
      A = np.stack([nun[ok], hb[ok], np.ones(ok.sum())], 1)
      coef, *_ = np.linalg.lstsq(A, busy[ok], rcond=None)
      pred = A @ coef
      print("  busy(us) ~ %.3f*units + %.3f*ceil_units + %.2f; R2 %.3f; ceil units/CTA p0/p50/p100 %s" %
          (coef[0], coef[1], coef[2], 1 - ((busy[ok] - pred) ** 2).sum() / ((busy[ok] - busy[ok].mean()) ** 2).sum(),
           np.percentile(hb[ok], [0, 50, 100])))
    rank = np.arange(511) // 148
    for rk in range(4):
        m = sel & (rank == rk)
        if m.any():
            print("  CTA rank %d (blockIdx//148): last done mean %.2f p90 %.2f; first full mean %.2f" %
                  (rk, ((last[:511] - t0)[m] / 1e3).mean(), np.percentile((last[:511] - t0)[m] / 1e3, 90),
                   ((t[:511, 3] - t0)[m] / 1e3).mean()))
    # per-unit processing interval (compute warp 0) median over CTAs
    iv = []
    for c in np.where(sel)[0]:
        n = nun[c]
        d = [t[c, 4 + 3 * (j + 1)] - t[c, 4 + 3 * j] for j in range(min(n, 40) - 1) if 4 + 3 * (j + 1) < 128]
        iv += d
    print("  unit interval us: median %.3f p90 %.3f" % (np.median(iv) / 1e3, np.percentile(iv, 90) / 1e3))
    fw = [t[c, 3 + 3 * j] - t[c, 4 + 3 * (j - 1)] for c in np.where(sel)[0] for j in range(1, min(nun[c], 40)) if 4 + 3 * j < 128]
    print("  wait-for-full after prev unit us: median %.3f p90 %.3f" % (np.median(fw) / 1e3, np.percentile(fw, 90) / 1e3))
