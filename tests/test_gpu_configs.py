"""Parity of the CUDA path against the CPU oracle at BASELINE.json's own
config shapes (configs[0], [3], [4]) -- not reduced stand-ins.

Oracle: matmul_reference(x, dequantize_model(model)) (matrix.cpp:5-17,
layout.cpp:316-332) restated in oracle/sfmp_oracle.c, and for
configs[0] also the reference's own LUT gemv (lutgemm.cpp:95-135) from
oracle/_ref when it was built.  Bar: max|d|/max|y_ref| <= 1e-3.  At large M
the oracle checks a seeded sample of token rows incl. the first and last
(SURVEY §8d), the GPU computes all of them.
"""
import numpy as np
import pytest

from synth import LLAMA_70B, activations, errors, f32_activations, model_bytes, prebuild

pytestmark = pytest.mark.gpu
TOL = 1e-3


def sample_rows(M, k=16, seed=0):
    if M <= k:
        return np.arange(M)
    rng = np.random.default_rng(seed)
    mid = rng.choice(np.arange(1, M - 1), size=k - 2, replace=False)
    return np.sort(np.concatenate([[0, M - 1], mid]))


def check(gpu, port, dm, w_ref, x_np, dtype, path=None, label=""):
    import torch
    xt = torch.from_numpy(x_np).cuda().to(getattr(torch, dtype))
    y = dm.gemm(xt, path=path if path is not None else gpu.PATH_AUTO)
    rows = sample_rows(x_np.shape[0])
    ysel = y[torch.from_numpy(rows).cuda()].cpu().numpy()
    ref = port.matmul(np.ascontiguousarray(xt.float().cpu().numpy()[rows]), w_ref, threads=8)
    e_max, e_l2 = errors(ysel, ref)
    assert np.isfinite(ysel).all(), label
    assert e_max <= TOL, (label, e_max, e_l2)
    return e_max


@pytest.mark.parametrize("dtype", ["bfloat16", "float32"])
def test_config0_4096sq_3p5bit_m1(gpu, port, dtype):
    """configs[0]: single 4096x4096 linear, avg 3.5 bits, rowcol reorder, M=1,
    against matmul_reference AND the reference's own LUT gemv."""
    import torch
    data = model_bytes(port, 4096, 4096, 3.5, mode=3)
    dm = gpu.DeviceModel(data)
    pm = port.load(data)
    w = pm.dequantize()
    for x in (activations(port, 1, 4096, seed=0), f32_activations(1, 4096, seed=1)):
        if dtype == "bfloat16":  # the values the kernel actually sees
            x = torch.from_numpy(x).to(torch.bfloat16).float().numpy()
        y = dm.gemm(torch.from_numpy(x).cuda().to(getattr(torch, dtype))).cpu().numpy()
        ref = port.matmul(x, w, threads=8)
        assert errors(y, ref)[0] <= TOL
        y_lut, _ = pm.gemv_lut(x[0])  # the LUT algorithm of lutgemm.cpp:95 (C port)
        assert errors(y, y_lut[None])[0] <= TOL
    from oracle.oracle import Reference, reference_available
    if reference_available():
        rm = Reference().load(data)
        y_gemv, _ = rm.gemv(x[0])  # the unmodified reference's sfmp::gemv
        assert errors(y, y_gemv[None])[0] <= TOL


_70B = [(r, c, 2.5, {"m_b": 128 if p in ("k_proj", "v_proj") else 512}) for p, (r, c) in LLAMA_70B.items()]


@pytest.fixture(scope="module")
def models_70b(port):
    prebuild(_70B)
    return {p: model_bytes(port, r, c, 2.5, m_b=128 if p in ("k_proj", "v_proj") else 512)
            for p, (r, c) in LLAMA_70B.items()}


@pytest.mark.parametrize("proj", list(LLAMA_70B))
def test_llama70b_linears_decode_and_prefill(gpu, port, models_70b, proj):
    """configs[3] at 1 GPU: every Llama-3.1-70B linear @2.5 bits, decode
    M in {1, 16} and prefill M = 2048 (16 sampled token rows)."""
    rows, cols = LLAMA_70B[proj]
    data = models_70b[proj]
    dm = gpu.DeviceModel(data)
    w = port.load(data).dequantize()
    for M in (1, 16, 2048):
        check(gpu, port, dm, w, activations(port, M, cols, seed=M), "bfloat16", label=(proj, M))
    check(gpu, port, dm, w, f32_activations(16, cols, seed=3), "float32", label=(proj, "f32"))


_SWEEP = [(8192, 28672, b, {}) for b in (2.0, 3.0, 4.0)]


@pytest.fixture(scope="module")
def models_sweep(port):
    prebuild(_SWEEP)
    return {b: model_bytes(port, 8192, 28672, b) for b in (2.0, 3.0, 4.0)}


@pytest.mark.parametrize("bits", [2.0, 3.0, 4.0])
def test_sweep_8192x28672(gpu, port, models_sweep, bits):
    """configs[4] points: 8192x28672 at 2.0/3.0/4.0 bits x M in {1, 16, 64, 4096}."""
    data = models_sweep[bits]
    dm = gpu.DeviceModel(data)
    w = port.load(data).dequantize()
    for M in (1, 16, 64, 4096):
        check(gpu, port, dm, w, activations(port, M, 28672, seed=M), "bfloat16", label=(bits, M))
