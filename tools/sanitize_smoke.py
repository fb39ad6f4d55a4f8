"""Small calls of every kernel family, for compute-sanitizer (memcheck / racecheck /
synccheck): device ingest (model creation), grouped decode with mixed token counts
(one launch), f32 decode, fused RMSNorm (decode and prefill), the prefill GEMM (whole
tiles, K splits), both pre-passes, dequant/unpack/gemv_block, the LUT comparison
kernel, and the sharded path (packed local GEMMs + grouped un-permute)."""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import paper_2602_01027_b200 as sfmp  # noqa: E402
from oracle.oracle import Port  # noqa: E402
from synth import activations, model_bytes  # noqa: E402

P = Port()
shapes = [(1024, 512, 512), (512, 1024, 128), (768, 512, 256)]
datas = [model_bytes(P, r, c, 3.25, m_b=mb, seed=i) for i, (r, c, mb) in enumerate(shapes)]
models = [sfmp.DeviceModel(d) for d in datas]
Ms = [1, 5, 8, 12, 16, 3]
sel = [models[i % len(models)] for i in range(len(Ms))]
xs = [torch.from_numpy(activations(P, M, m.cols, seed=i)).cuda().to(torch.bfloat16) for i, (M, m) in enumerate(zip(Ms, sel))]
ws = [torch.zeros(m.workspace_bytes(16), dtype=torch.uint8, device="cuda") for m in sel]
sfmp.gemm_grouped(sel, xs, workspaces=ws)
sfmp.gemm_grouped(sel, [x.float() for x in xs], workspaces=ws)  # f32 x (hi/lo split)
g = torch.ones(512, device="cuda")
sfmp.gemm_grouped(sel, xs, workspaces=ws, norms=[(g if m.cols == 512 else None, 1e-5) for m in sel])
for m in models:
    x = torch.from_numpy(activations(P, 300, m.cols, seed=7)).cuda()
    m.gemm(x.to(torch.bfloat16), path=sfmp.PATH_GEMM)
    m.gemm(x, path=sfmp.PATH_GEMM)  # f32 x
    m.gemm(x[:40].to(torch.bfloat16), path=sfmp.PATH_GEMM)  # stream-K
    m.dequantize()
    m.gemm(x[:64].to(torch.bfloat16), norm=(None, 1e-5))  # fused norm, prefill
    m.gemv_block(0, x[0])
lut = sfmp.DeviceModel(datas[0], flags=sfmp.MODEL_LUT_LAYOUT)
lut.gemm(torch.from_numpy(activations(P, 2, lut.cols, seed=9)).cuda(), path=sfmp.PATH_LUT)
sh = [sfmp.DeviceModel(datas[0], shard=g, num_shards=2) for g in range(2)]
Ms2 = [1, 3]
bufs = []
for s_ in sh:
    b = torch.zeros(sfmp.sharded_gather_bytes([s_, s_], Ms2) // 4, device="cuda")
    xx = [torch.from_numpy(activations(P, M, s_.cols, seed=M)).cuda().to(torch.bfloat16) for M in Ms2]
    w2 = [torch.zeros(s_.workspace_bytes(16), dtype=torch.uint8, device="cuda") for _ in Ms2]
    sfmp.gemm_sharded_local([s_, s_], xx, b, w2)
    bufs.append(b)
tot = sfmp.packed_offsets([sh[0], sh[0]], Ms2)[-1]
for b in bufs:
    b[tot:].copy_(torch.cat([bb[:tot] for bb in bufs]))
    sfmp.sharded_unpermute([sh[0], sh[0]], Ms2, b, [torch.empty(M, 1024, device="cuda") for M in Ms2])
x = torch.from_numpy(activations(P, 3, sh[0].cols, seed=3)).cuda().to(torch.bfloat16)
sh[0].unpermute_gathered(torch.stack([s.gemm(x) for s in sh]), 3)
torch.cuda.synchronize()
print("sanitize smoke done")
