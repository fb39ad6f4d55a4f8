"""GPU parity of the CUDA path (through the C ABI) against the CPU oracle.

Bars (BASELINE.json north_star): unpack/dequant bit-exact; GEMM outputs within
max|d|/max|y_ref| <= 1e-3 of the reference's fp32-accumulate result
matmul_reference(x, dequantize_model(model)).
"""
import hashlib

import numpy as np
import pytest

from conftest import golden_cases, load_golden
from synth import LLAMA_8B, activations, errors, model_bytes

pytestmark = pytest.mark.gpu
TOL = 1e-3


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def paths_for(sfmp, dm, M):
    out = [sfmp.PATH_GENERIC, sfmp.PATH_AUTO]
    info = dm.info
    if info["m_b"] % 128 == 0 and info["n_b"] % 128 == 0:
        out.append(sfmp.PATH_GEMV)
    return out


@pytest.mark.parametrize("name", golden_cases())
def test_golden_unpack_dequant_bit_exact(gpu, index, name):
    import torch
    meta, g = index[name], load_golden(name)
    dm = gpu.DeviceModel(bytes(g["model"]))
    codes = dm.unpack_codes().cpu().numpy()
    assert sha(codes) == meta["codes_sha256"]
    w = dm.dequantize().cpu().numpy()
    assert sha(w) == meta["w_sha256"]
    torch.cuda.synchronize()


@pytest.mark.parametrize("name", golden_cases())
@pytest.mark.parametrize("dtype", ["float32", "bfloat16", "float16"])
def test_golden_gemm_parity(gpu, index, name, dtype):
    import torch
    meta, g = index[name], load_golden(name)
    dm = gpu.DeviceModel(bytes(g["model"]))
    x = torch.from_numpy(g["x"]).cuda().to(getattr(torch, dtype))
    for path in paths_for(gpu, dm, meta["M"]):
        y = dm.gemm(x, path=path).cpu().numpy()
        e_max, e_l2 = errors(y, g["y_ref"])
        assert e_max <= TOL, (name, path, e_max, e_l2)
        e_lut, _ = errors(y, g["y_lut"])
        assert e_lut <= TOL


def test_gemv_deterministic_and_linear(gpu, port):
    import torch
    data = model_bytes(port, 4096, 4096, 3.5)
    dm = gpu.DeviceModel(data)
    x = torch.from_numpy(activations(port, 16, 4096)).cuda()
    for M in (1, 5, 16):
        a = dm.gemm(x[:M], path=gpu.PATH_GEMV)
        b = dm.gemm(x[:M], path=gpu.PATH_GEMV)
        assert torch.equal(a, b)
    z = dm.gemm(torch.zeros_like(x[:3]), path=gpu.PATH_GEMV)
    assert torch.count_nonzero(z) == 0
    y1 = dm.gemm(x[:4], path=gpu.PATH_GEMV)
    y2 = dm.gemm(2 * x[:4], path=gpu.PATH_GEMV)
    assert torch.allclose(y2, 2 * y1, rtol=1e-5, atol=1e-5)


def test_shape_errors(gpu, port):
    import torch
    dm = gpu.DeviceModel(model_bytes(port, 1024, 512, 3.0))
    with pytest.raises(gpu.ShapeError):
        dm.gemm(torch.zeros(2, 511, device="cuda"))
    y = dm.gemm(torch.zeros(0, 512, device="cuda"))
    assert y.shape == (0, 1024)


@pytest.mark.parametrize("proj", list(LLAMA_8B))
@pytest.mark.parametrize("M", [1, 3, 8, 16])
def test_llama8b_decode_parity(gpu, port, proj, M):
    """configs[1]: Llama-3.1-8B linears at avg 3.25 bits, decode M=1..16."""
    import torch
    rows, cols = LLAMA_8B[proj]
    data = model_bytes(port, rows, cols, 3.25)
    dm = gpu.DeviceModel(data)
    x = activations(port, M, cols, seed=M)
    y = dm.gemm(torch.from_numpy(x).cuda().to(torch.bfloat16)).cpu().numpy()
    pm = port.load(data)
    w = pm.dequantize()
    ref = port.matmul(x, w, threads=8)
    e_max, e_l2 = errors(y, ref)
    assert e_max <= TOL, (proj, M, e_max, e_l2)
    # The GPU dequant of the same model is bit-exact with the oracle's.
    if proj in ("q_proj", "k_proj"):
        wg = dm.dequantize().cpu().numpy()
        assert np.array_equal(wg.view(np.uint32), w.view(np.uint32))


@pytest.mark.parametrize("bits", [2.0, 2.5, 3.0, 4.0])
def test_bit_sweep_parity(gpu, port, bits):
    """configs[4] shape family at reduced K: every bit-width mix of the sweep."""
    import torch
    data = model_bytes(port, 2048, 4096, bits)
    dm = gpu.DeviceModel(data)
    x = activations(port, 9, 4096, seed=7)
    ref = port.matmul(x, port.load(data).dequantize(), threads=8)
    for path in (gpu.PATH_GEMV, gpu.PATH_GENERIC):
        y = dm.gemm(torch.from_numpy(x).cuda(), path=path).cpu().numpy()
        assert errors(y, ref)[0] <= TOL


@pytest.mark.parametrize("dtype", ["float32", "bfloat16"])
def test_gemv_wide_rows(gpu, port, dtype):
    """Decode pre-pass on a 53248-column linear: the bf16 row (104 KB) is
    staged in shared memory, the f32 row (208 KB) exceeds the staging limit
    and takes the gather pre-pass; both within the parity bar."""
    import torch
    data = model_bytes(port, 512, 53248, 3.0)
    dm = gpu.DeviceModel(data)
    x = activations(port, 5, 53248, seed=11)
    xt = torch.from_numpy(x).cuda().to(getattr(torch, dtype))
    ref = port.matmul(xt.float().cpu().numpy(), port.load(data).dequantize(), threads=8)
    y = dm.gemm(xt, path=gpu.PATH_GEMV).cpu().numpy()
    assert errors(y, ref)[0] <= TOL


def test_gemv_misaligned_rows_f16(gpu, port):
    """x rows at a 2-byte offset: the staged pre-pass copies them element-wise."""
    import torch
    data = model_bytes(port, 1024, 1024, 3.5)
    dm = gpu.DeviceModel(data)
    buf = torch.from_numpy(activations(port, 7, 1025, seed=5)).cuda().to(torch.float16)
    x = buf.reshape(-1)[1:1 + 7 * 1024].view(7, 1024)
    assert x.data_ptr() % 16 != 0
    ref = port.matmul(x.float().cpu().numpy(), port.load(data).dequantize(), threads=8)
    y = dm.gemm(x, path=gpu.PATH_GEMV).cpu().numpy()
    assert errors(y, ref)[0] <= TOL
