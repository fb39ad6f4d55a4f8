"""Small calls of every kernel family, for compute-sanitizer (memcheck / racecheck /
synccheck): grouped decode with mixed token counts, the prefill GEMM (whole tiles,
stream-K), both pre-passes, dequant/unpack parity kernels and the shard un-permute."""
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
for m in models:
    x = torch.from_numpy(activations(P, 300, m.cols, seed=7)).cuda()
    m.gemm(x.to(torch.bfloat16), path=sfmp.PATH_GEMM)
    m.gemm(x, path=sfmp.PATH_GEMM)  # f32 x
    m.gemm(x[:40].to(torch.bfloat16), path=sfmp.PATH_GEMM)  # stream-K
    m.dequantize()
sh = [sfmp.DeviceModel(datas[0], shard=g, num_shards=2) for g in range(2)]
x = torch.from_numpy(activations(P, 3, sh[0].cols, seed=3)).cuda().to(torch.bfloat16)
sh[0].unpermute_gathered(torch.stack([s.gemm(x) for s in sh]), 3)
torch.cuda.synchronize()
print("sanitize smoke done")
