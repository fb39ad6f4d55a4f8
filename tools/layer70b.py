"""configs[3] at one GPU: the seven Llama-3.1-70B linears at avg 2.5 code bits
(k/v at m_b=128 so they shard 8 ways), decode M in {1,2,4,8,16} as grouped
launches and prefill M=2048 per linear; CUDA graphs, CUDA events, weights
rotated over 2 copies.  Writes profiles/r01_llama70b_layer.json."""
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import paper_2602_01027_b200 as sfmp  # noqa: E402
from oracle.oracle import Port  # noqa: E402
from synth import LLAMA_70B, activations, errors, model_bytes  # noqa: E402

P = Port()
peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
HBM, TC = float(peaks["hbm_gbs"]), float(peaks["bf16_tflops"])
projs = list(LLAMA_70B)
datas = {p: model_bytes(P, *LLAMA_70B[p], 2.5, m_b=128 if p in ("k_proj", "v_proj") else 512,
                        seed={"up_proj": 4, "v_proj": 1}.get(p, 0)) for p in projs}
COPIES = 2
models = [[sfmp.DeviceModel(datas[p]) for p in projs] for _ in range(COPIES)]
out = {"config": "Llama-3.1-70B linears, avg 2.5 code bits, rowcol reorder, 1 GPU", "decode": {}, "prefill": {}}


def timed(fn, reps):
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        fn(0)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        for i in range(reps):
            fn(i)
    g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(3):
        g.replay()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) * 1e3 / (3 * reps)


for M in (1, 2, 4, 8, 16):
    xs = [torch.from_numpy(activations(P, M, LLAMA_70B[p][1], seed=M)).cuda().to(torch.bfloat16) for p in projs]
    ys = [torch.empty(M, LLAMA_70B[p][0], device="cuda") for p in projs]
    ws = [m.workspace(16, sfmp.PATH_GEMV) for m in models[0]]
    us = timed(lambda i: sfmp.gemm_grouped(models[i % COPIES], xs, outs=ys, workspaces=ws), 4)
    byts = sum(m.info["payload_bytes"] + 4 * m.cols + 4 * m.rows + 2 * M * m.cols + 4 * M * m.rows for m in models[0])
    out["decode"][M] = {"us_per_layer": round(us, 2), "GBps": round(byts / us / 1e3, 1),
                        "frac_hbm": round(byts / us / 1e3 / HBM, 4)}
    print("decode", M, out["decode"][M], flush=True)
    if M == 16:  # parity spot check, q_proj
        ref = P.matmul(xs[0].float().cpu().numpy(), P.load(datas["q_proj"]).dequantize(), threads=8)
        out["decode"]["parity_max_rel_q_M16"] = round(errors(ys[0].cpu().numpy(), ref)[0], 8)
M = 2048
tot_us, tot_fl = 0.0, 0.0
for pi, p in enumerate(projs):
    rows, cols = LLAMA_70B[p]
    x = torch.from_numpy(activations(P, M, cols, seed=7)).cuda().to(torch.bfloat16)
    y = torch.empty(M, rows, device="cuda")
    ws = models[0][pi].workspace(M, sfmp.PATH_GEMM)
    us = timed(lambda i: models[i % COPIES][pi].gemm(x, out=y, path=sfmp.PATH_GEMM, workspace=ws), 2)
    fl = 2.0 * M * rows * cols
    tot_us += us
    tot_fl += fl
    out["prefill"][p] = {"us": round(us, 1), "tflops": round(fl / us / 1e6, 1), "frac_bf16": round(fl / us / 1e6 / TC, 4)}
    print("prefill", p, out["prefill"][p], flush=True)
out["prefill"]["layer"] = {"us": round(tot_us, 1), "frac_bf16": round(tot_fl / tot_us / 1e6 / TC, 4)}
json.dump(out, open(os.path.join(ROOT, "gpurun_out", "r01_llama70b_layer.json"), "w"), indent=1)
print(json.dumps(out["prefill"]["layer"]))
