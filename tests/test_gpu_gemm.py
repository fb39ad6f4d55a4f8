"""K2 (tcgen05 prefill GEMM) parity through the C ABI against the CPU oracle.

Bar (BASELINE.json north_star): max|d|/max|y_ref| <= 1e-3 against the
reference's fp32-accumulate matmul_reference(x, dequantize_model(model))
(SPEC.md:540).  Weights are rounded once to f16 on the tensor-core path
(SURVEY §7 hard part 1), so the tolerance is the north-star's 1e-3, not the
GEMV's ~1e-5.
"""
import numpy as np
import pytest

from conftest import golden_cases, load_golden
from synth import LLAMA_8B, activations, errors, model_bytes

pytestmark = pytest.mark.gpu
TOL = 1e-3


@pytest.mark.parametrize("name", golden_cases())
def test_golden_gemm_path(gpu, index, name):
    import torch
    meta, g = index[name], load_golden(name)
    dm = gpu.DeviceModel(bytes(g["model"]))
    if meta["n_b"] % 128:
        with pytest.raises(gpu.UnsupportedError):
            dm.gemm(torch.from_numpy(g["x"]).cuda(), path=gpu.PATH_GEMM)
        return
    for dtype in (torch.float32, torch.bfloat16, torch.float16):
        x = torch.from_numpy(g["x"]).cuda().to(dtype)
        y = dm.gemm(x, path=gpu.PATH_GEMM).cpu().numpy()
        e_max, e_l2 = errors(y, g["y_ref"])
        assert e_max <= TOL, (name, dtype, e_max, e_l2)


@pytest.mark.parametrize("M", [17, 64, 100, 128, 129, 300])
def test_gemm_token_counts(gpu, port, M):
    """Ragged token tiles (N = 128 or round-up-16 of M), padding tokens masked."""
    import torch
    data = model_bytes(port, 1024, 1024, 3.5)
    dm = gpu.DeviceModel(data)
    x = activations(port, M, 1024, seed=M)
    ref = port.matmul(x, port.load(data).dequantize(), threads=8)
    y = dm.gemm(torch.from_numpy(x).cuda().to(torch.bfloat16), path=gpu.PATH_GEMM).cpu().numpy()
    e_max, e_l2 = errors(y, ref)
    assert e_max <= TOL, (M, e_max, e_l2)
    assert y.shape == (M, 1024)


@pytest.mark.parametrize("bits", [1.5, 2.0, 2.5, 3.0, 3.25, 4.0, 5.5, 7.75])
def test_gemm_bit_mixes(gpu, port, bits):
    """Every floor/ceil pair incl. the >4-bit exact-code unpack path."""
    import torch
    data = model_bytes(port, 1024, 512, bits)
    dm = gpu.DeviceModel(data)
    x = activations(port, 200, 512, seed=3)
    ref = port.matmul(x, port.load(data).dequantize(), threads=8)
    y = dm.gemm(torch.from_numpy(x).cuda(), path=gpu.PATH_GEMM).cpu().numpy()
    assert errors(y, ref)[0] <= TOL, bits


@pytest.mark.parametrize("mode", [0, 1, 2, 3])
@pytest.mark.parametrize("m_b,n_b", [(512, 128), (128, 256), (64, 128), (256, 256)])
def test_gemm_modes_and_blocks(gpu, port, mode, m_b, n_b):
    import torch
    data = model_bytes(port, 1024, 768 if n_b == 128 else 1024, 3.25, mode=mode, m_b=m_b, n_b=n_b)
    dm = gpu.DeviceModel(data)
    cols = dm.cols
    x = activations(port, 150, cols, seed=5)
    ref = port.matmul(x, port.load(data).dequantize(), threads=8)
    y = dm.gemm(torch.from_numpy(x).cuda().to(torch.bfloat16), path=gpu.PATH_GEMM).cpu().numpy()
    assert errors(y, ref)[0] <= TOL, (mode, m_b, n_b)


def test_gemm_deterministic_linear_zero(gpu, port):
    import torch
    data = model_bytes(port, 2048, 1024, 3.25)
    dm = gpu.DeviceModel(data)
    x = torch.from_numpy(activations(port, 256, 1024, seed=9)).cuda().to(torch.bfloat16)
    a = dm.gemm(x, path=gpu.PATH_GEMM)
    b = dm.gemm(x, path=gpu.PATH_GEMM)
    assert torch.equal(a, b)
    z = dm.gemm(torch.zeros_like(x), path=gpu.PATH_GEMM)
    assert torch.count_nonzero(z) == 0
    y2 = dm.gemm(2 * x, path=gpu.PATH_GEMM)  # power-of-two scaling is exact in f16
    assert torch.equal(y2, 2 * a)


@pytest.mark.parametrize("proj", ["q_proj", "k_proj", "gate_proj", "down_proj"])
def test_llama8b_prefill_parity(gpu, port, proj):
    """configs[2]: Llama-3.1-8B linears at avg 3.25 bits, prefill M=2048
    (q/down: whole tiles; k: stream-K; gate: whole-tile rounds + stream-K over
    the last partial wave); checked on a seeded sample of token rows."""
    import torch
    rows, cols = LLAMA_8B[proj]
    M = 2048
    data = model_bytes(port, rows, cols, 3.25)
    dm = gpu.DeviceModel(data)
    x = activations(port, M, cols, seed=11)
    y = dm.gemm(torch.from_numpy(x).cuda().to(torch.bfloat16)).cpu().numpy()  # AUTO -> GEMM
    rng = np.random.default_rng(0)
    sample = np.unique(np.concatenate([[0, M - 1], rng.choice(M, 30, replace=False)]))
    ref = port.matmul(np.ascontiguousarray(x[sample]), port.load(data).dequantize(), threads=8)
    e_max, e_l2 = errors(y[sample], ref)
    assert e_max <= TOL, (proj, e_max, e_l2)


def test_gemm_misaligned_x_routes_to_gemv(gpu, port):
    """AUTO with a non-16-byte-aligned x takes the decode path (same result);
    forcing the tensor-core path on it is an argument error, not a fault."""
    import torch
    data = model_bytes(port, 1024, 512, 3.5)
    dm = gpu.DeviceModel(data)
    buf = torch.from_numpy(activations(port, 40, 512 + 1, seed=2)).cuda()
    x = buf.reshape(-1)[1:1 + 40 * 512].view(40, 512)  # 4-byte offset: misaligned for 16 B loads
    assert x.data_ptr() % 16 != 0
    ref = port.matmul(x.cpu().numpy(), port.load(data).dequantize(), threads=8)
    y = dm.gemm(x).cpu().numpy()
    assert errors(y, ref)[0] <= TOL
    with pytest.raises(gpu.SfmpError):
        dm.gemm(x, path=gpu.PATH_GEMM)


@pytest.mark.parametrize("dtype,cols", [("bfloat16", 14336), ("float32", 14336), ("float16", 14336)])
def test_gemm_prepass_variants(gpu, port, dtype, cols):
    """Both prefill pre-passes: the persistent row-streaming one (bf16 rows of
    a 14336-column linear) and the one-token-per-CTA one (f32 rows whose two
    staging buffers exceed its shared-memory budget; rows of >= 65536 columns)."""
    import torch
    rows, M = 512, 300
    data = model_bytes(port, rows, cols, 3.0)
    dm = gpu.DeviceModel(data)
    xt = torch.from_numpy(activations(port, M, cols, seed=21)).cuda().to(getattr(torch, dtype))
    y = dm.gemm(xt, path=gpu.PATH_GEMM).cpu().numpy()
    ref = port.matmul(xt.float().cpu().numpy(), port.load(data).dequantize(), threads=8)
    assert errors(y, ref)[0] <= TOL
