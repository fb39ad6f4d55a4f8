"""Grouped decode (sfmp_gemm_grouped): independent linears, each with its own
x and reorder indices, in one pre-pass + one GEMV launch."""
import numpy as np
import pytest

from synth import activations, errors, model_bytes

pytestmark = pytest.mark.gpu

SHAPES = [(1024, 512, 512), (2048, 1024, 128), (512, 1024, 512), (1536, 768, 512), (1024, 1024, 128)]


@pytest.mark.parametrize("M", [1, 5, 16])
def test_grouped_matches_oracle(gpu, port, M):
    import torch
    datas = [model_bytes(port, r, c, 3.25, m_b=mb, seed=i) for i, (r, c, mb) in enumerate(SHAPES)]
    models = [gpu.DeviceModel(d) for d in datas]
    xs_np = [activations(port, M, c, seed=10 + i) for i, (r, c, mb) in enumerate(SHAPES)]
    xs = [torch.from_numpy(x).cuda().to(torch.bfloat16) for x in xs_np]
    ys = gpu.gemm_grouped(models, xs)
    ys2 = gpu.gemm_grouped(models, xs)
    for i, (d, x, y, y2) in enumerate(zip(datas, xs_np, ys, ys2)):
        assert torch.equal(y, y2)  # deterministic
        ref = port.matmul(x, port.load(d).dequantize(), threads=8)
        e_max, e_l2 = errors(y.cpu().numpy(), ref)
        assert e_max <= 1e-3, (i, e_max, e_l2)


def test_grouped_mixed_geometry_and_prefill(gpu, port):
    """Different floor bits / n_b split the group into runs; M > 16 goes per model."""
    import torch
    datas = [model_bytes(port, 1024, 512, 3.25), model_bytes(port, 1024, 512, 2.5),
             model_bytes(port, 1024, 512, 3.0, n_b=256, m_b=512), model_bytes(port, 512, 256, 3.25, n_b=64, m_b=128)]
    models = [gpu.DeviceModel(d) for d in datas]
    for M in (3, 40):
        xs_np = [activations(port, M, m.cols, seed=M + i) for i, m in enumerate(models)]
        ys = gpu.gemm_grouped(models, [torch.from_numpy(x).cuda() for x in xs_np])
        for d, x, y in zip(datas, xs_np, ys):
            ref = port.matmul(x, port.load(d).dequantize(), threads=8)
            assert errors(y.cpu().numpy(), ref)[0] <= 1e-3


def test_grouped_per_problem_token_counts(gpu, port):
    """sfmp_gemm_grouped_v: problems with different M in one call -- M <= 8 ones
    share a launch, 9..16 another, M > 16 and M = 0 go their own way; a shared
    workspace splits the launch instead of aliasing its records."""
    import torch
    datas = [model_bytes(port, r, c, 3.25, m_b=mb, seed=i) for i, (r, c, mb) in enumerate(SHAPES)]
    models = [gpu.DeviceModel(d) for d in datas]
    Ms = [1, 3, 8, 5, 2, 12, 16, 9, 40, 0]
    picks = [i % len(models) for i in range(len(Ms))]
    xs_np = [activations(port, max(M, 1), models[k].cols, seed=30 + i)[:M] for i, (M, k) in enumerate(zip(Ms, picks))]
    xs = [torch.from_numpy(np.ascontiguousarray(x)).cuda().to(torch.bfloat16).reshape(M, models[k].cols)
          for x, M, k in zip(xs_np, Ms, picks)]
    sel = [models[k] for k in picks]
    # every problem its own zeroed workspace, except problems 0 and 3 (both
    # M <= 8) which share one: the M <= 8 run must split there
    ws = [torch.zeros(m.workspace_bytes(max(M, 1)), dtype=torch.uint8, device="cuda") for m, M in zip(sel, Ms)]
    ws[0] = ws[3] = torch.zeros(max(sel[0].workspace_bytes(16), sel[3].workspace_bytes(16)), dtype=torch.uint8,
                                device="cuda")
    ys = gpu.gemm_grouped(sel, xs, workspaces=ws)
    for i, (M, k) in enumerate(zip(Ms, picks)):
        assert ys[i].shape == (M, models[k].out_rows)
        if M == 0:
            continue
        ref = port.matmul(xs[i].float().cpu().numpy(), port.load(datas[k]).dequantize(), threads=8)
        assert errors(ys[i].cpu().numpy(), ref)[0] <= 1e-3, (i, M)
        # bit-identical with the single-problem call (canonical segment order)
        y1 = sel[i].gemm(xs[i])
        assert torch.equal(ys[i], y1), (i, M)


def test_whole_k_items_bit_identical(gpu, port):
    """The 8B decode step (7 linears x M in {1, 2, 4, 8, 16}) in one call is
    large enough for whole-K work items: the K = 4096 linears sum their
    segments in registers (their partial region stays untouched), down_proj
    keeps per-segment items and the fix-up.  Either way the bits equal the
    single-linear calls, which use per-segment items only."""
    import torch
    from synth import LLAMA_8B
    names = list(LLAMA_8B)
    models = {p: gpu.DeviceModel(model_bytes(port, *LLAMA_8B[p], 3.25, m_b=128 if p in ("k_proj", "v_proj") else 512))
              for p in names}
    keys = [(p, M) for M in (1, 2, 4, 8, 16) for p in names]
    xs = [torch.from_numpy(activations(port, M, LLAMA_8B[p][1], seed=M)).cuda().to(torch.bfloat16) for p, M in keys]
    ws = [torch.zeros(models[p].workspace_bytes(16), dtype=torch.uint8, device="cuda") for p, M in keys]
    ys = gpu.gemm_grouped([models[p] for p, M in keys], xs, workspaces=ws)
    torch.cuda.synchronize()
    for (p, M), x, y, w in zip(keys, xs, ys, ws):
        rows, cols = LLAMA_8B[p]
        part = (rows // 128) * (cols // 1024) * 16 * 128 * 4  # [tiles][segments][16 tokens][128 rows] f32
        touched = bool(w[-(part + 128):-128].any())
        assert touched == (p == "down_proj"), (p, M)
        assert torch.equal(y, models[p].gemm(x)), (p, M)
