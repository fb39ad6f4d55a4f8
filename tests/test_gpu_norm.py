"""RMSNorm fused into the activation pre-pass ("fused
activation producer"): y = RMSNorm(h; gamma, eps) . W^T with the norm applied
while the pre-pass stages each token row (sfmp_gemm_norm /
sfmp_gemm_grouped_v_norm).  Oracle: the f32 norm on the host, then
matmul_reference(x, dequantize_model(model)); bar 1e-3."""
import numpy as np
import pytest

from synth import activations, errors, model_bytes

pytestmark = pytest.mark.gpu
TOL = 1e-3


def host_norm(h, gamma, eps):
    h = h.astype(np.float64)
    inv = 1.0 / np.sqrt((h * h).mean(axis=1, keepdims=True) + eps)
    return (h * inv * (1.0 if gamma is None else gamma.astype(np.float64))).astype(np.float32)


@pytest.mark.parametrize("M", [1, 7, 16, 40, 300])
@pytest.mark.parametrize("gdt", ["float32", "bfloat16", None])
def test_fused_rmsnorm_single(gpu, port, M, gdt):
    import torch
    data = model_bytes(port, 2048, 4096, 3.25)
    dm = gpu.DeviceModel(data)
    h = (activations(port, M, 4096, seed=M) * 37.0).astype(np.float32)
    rng = np.random.default_rng(M)
    gamma = None if gdt is None else (1.0 + 0.2 * rng.standard_normal(4096)).astype(np.float32)
    hb = torch.from_numpy(h).cuda().to(torch.bfloat16)
    gt = None if gamma is None else torch.from_numpy(gamma).cuda().to(getattr(torch, gdt))
    y = dm.gemm(hb, norm=(gt, 1e-5)).cpu().numpy()
    g_eff = None if gt is None else gt.float().cpu().numpy()
    ref = port.matmul(host_norm(hb.float().cpu().numpy(), g_eff, 1e-5), port.load(data).dequantize(), threads=8)
    assert errors(y, ref)[0] <= TOL


def test_fused_rmsnorm_grouped(gpu, port):
    """Three linears (own gammas and token counts, decode and prefill) in one
    call, plus a plain problem (norm disabled) in the same launch."""
    import torch
    shapes = [(1024, 4096, 3.25), (2048, 4096, 2.5), (512, 4096, 3.5)]
    blobs = [model_bytes(port, r, c, b) for r, c, b in shapes]
    ms = [gpu.DeviceModel(b) for b in blobs]
    Ms = [1, 8, 40]
    hs = [torch.from_numpy(activations(port, M, 4096, seed=20 + M) * 5.0).cuda().to(torch.bfloat16) for M in Ms]
    rng = np.random.default_rng(3)
    gs = [torch.from_numpy((1.0 + 0.1 * rng.standard_normal(4096)).astype(np.float32)).cuda() for _ in Ms]
    ws = [torch.zeros(max(m.workspace_bytes(16 if M <= 16 else M), 128), dtype=torch.uint8, device="cuda")
          for m, M in zip(ms, Ms)]
    ys = gpu.gemm_grouped(ms, hs, workspaces=ws, norms=[(g, 1e-6) for g in gs])
    for b, h, g, y in zip(blobs, hs, gs, ys):
        ref = port.matmul(host_norm(h.float().cpu().numpy(), g.cpu().numpy(), 1e-6), port.load(b).dequantize(),
                          threads=8)
        assert errors(y.cpu().numpy(), ref)[0] <= TOL
    mixed = gpu.gemm_grouped(ms[:2], hs[:2], workspaces=ws[:2], norms=[(gs[0], 1e-6), None])
    assert torch.equal(mixed[0], ys[0])
    assert torch.equal(mixed[1], ms[1].gemm(hs[1], workspace=ws[1]))


def test_fused_rmsnorm_errors(gpu, port):
    import torch
    data = model_bytes(port, 1024, 1024, 3.25)
    dm = gpu.DeviceModel(data)
    h = torch.zeros(2, 1024, device="cuda", dtype=torch.bfloat16)
    with pytest.raises(gpu.ConfigError):
        dm.gemm(h, norm=(None, 1e-5), path=gpu.PATH_GENERIC)
    with pytest.raises(gpu.SfmpError):
        dm.gemm(h, norm=(None, -1.0))
