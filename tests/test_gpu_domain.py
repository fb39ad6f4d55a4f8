"""The f32 activation domain and determinism across decompositions (GPU).

* f32 activations with a full 24-bit mantissa (not bf16-representable), from
  1e-3 to 1e30 in magnitude, with an outlier column: the decode GEMV splits x
  into two f16 terms after a per-token power-of-two scaling, so it stays
  within K1_F32_TOL of the f32 oracle matmul_reference(x, dequantize_model)
  (SPEC.md:540); the prefill GEMM rounds the scaled x to f16 once and stays
  within the 1e-3 bar.  No finite input produces inf.
* inf / NaN in x propagate: the non-finite pattern of y equals the oracle's.
* Determinism: a linear's bits do not depend on grouping,
  token count (decode), shard count or repeated calls -- torch.equal.
"""
import numpy as np
import pytest

from synth import activations, errors, f32_activations, model_bytes

pytestmark = pytest.mark.gpu
K1_F32_TOL = 1e-4   # decode GEMV with f32 x (hi/lo split): max|d|/max|y_ref|
TOL = 1e-3          # north_star bar


@pytest.fixture(scope="module")
def mid(port):
    data = model_bytes(port, 2048, 4096, 3.25)
    return data, port.load(data).dequantize()


@pytest.mark.parametrize("scale", [1e-3, 1.0, 1e4, 1e6, 1e30])
@pytest.mark.parametrize("M", [1, 5, 16])
def test_f32_full_mantissa_decode(gpu, port, mid, scale, M):
    import torch
    data, w = mid
    dm = gpu.DeviceModel(data)
    x = f32_activations(M, 4096, seed=M, scale=scale)
    ref = port.matmul(x, w, threads=8)
    assert np.isfinite(ref).all()
    y = dm.gemm(torch.from_numpy(x).cuda(), path=gpu.PATH_GEMV).cpu().numpy()
    assert np.isfinite(y).all(), "finite input must give finite output"
    e_max, e_l2 = errors(y, ref)
    assert e_max <= K1_F32_TOL, (scale, M, e_max, e_l2)


@pytest.mark.parametrize("scale", [1e-3, 1.0, 1e6, 1e30])
@pytest.mark.parametrize("M", [40, 300])
def test_f32_full_mantissa_prefill(gpu, port, mid, scale, M):
    import torch
    data, w = mid
    dm = gpu.DeviceModel(data)
    x = f32_activations(M, 4096, seed=M, scale=scale)
    rows = np.unique(np.r_[0, M - 1, np.arange(1, M, max(1, M // 16))])
    ref = port.matmul(x[rows], w, threads=8)
    y = dm.gemm(torch.from_numpy(x).cuda(), path=gpu.PATH_GEMM).cpu().numpy()[rows]
    assert np.isfinite(y).all()
    e_max, e_l2 = errors(y, ref)
    assert e_max <= TOL, (scale, M, e_max, e_l2)


@pytest.mark.parametrize("path", ["gemv", "gemm"])
def test_bf16_beyond_f16_range(gpu, port, mid, path):
    """bf16 values far above 65504: scaled per token, exact, finite."""
    import torch
    data, w = mid
    dm = gpu.DeviceModel(data)
    M = 3 if path == "gemv" else 64
    xb = torch.from_numpy(activations(port, M, 4096, seed=9) * 1e20).to(torch.bfloat16)
    x = xb.float().numpy()
    ref = port.matmul(x[:3], w, threads=8)
    y = dm.gemm(xb.cuda(), path=gpu.PATH_GEMV if path == "gemv" else gpu.PATH_GEMM).cpu().numpy()[:3]
    assert np.isfinite(y).all()
    assert errors(y, ref)[0] <= (K1_F32_TOL if path == "gemv" else TOL)


@pytest.mark.parametrize("path", ["gemv", "gemm"])
def test_nonfinite_propagation(gpu, port, mid, path):
    import torch
    data, w = mid
    dm = gpu.DeviceModel(data)
    M = 4 if path == "gemv" else 48
    x = f32_activations(M, 4096, seed=3)
    x[1, 17] = np.inf
    x[2, 4000] = np.nan
    x[3, 5] = -np.inf
    ref = port.matmul(x[:4], w, threads=8)
    y = dm.gemm(torch.from_numpy(x).cuda(), path=gpu.PATH_GEMV if path == "gemv" else gpu.PATH_GEMM).cpu().numpy()[:4]
    assert np.array_equal(np.isfinite(y), np.isfinite(ref))
    assert np.isfinite(y[0]).all()
    assert errors(y[0], ref[0])[0] <= TOL


def test_zero_rows(gpu, port, mid):
    import torch
    data, _ = mid
    dm = gpu.DeviceModel(data)
    for path, M in ((gpu.PATH_GEMV, 3), (gpu.PATH_GEMM, 33)):
        y = dm.gemm(torch.zeros(M, 4096, device="cuda"), path=path)
        assert torch.count_nonzero(y) == 0


# ---- determinism across decompositions -------------------------------------------

SHAPES = [(1024, 512, 512), (2048, 1024, 128), (512, 1024, 512), (1536, 768, 512), (4096, 4096, 512)]


@pytest.mark.parametrize("dtype", ["bfloat16", "float32"])
def test_decode_bits_independent_of_grouping_and_M(gpu, port, dtype):
    """K1: single call == grouped call == any token subset, bit for bit."""
    import torch
    dt = getattr(torch, dtype)
    datas = [model_bytes(port, r, c, 3.25, m_b=mb, seed=i) for i, (r, c, mb) in enumerate(SHAPES)]
    models = [gpu.DeviceModel(d) for d in datas]
    xs = [torch.from_numpy(f32_activations(16, c, seed=i)).cuda().to(dt) for i, (r, c, mb) in enumerate(SHAPES)]
    single = [m.gemm(x, path=gpu.PATH_GEMV) for m, x in zip(models, xs)]
    grouped = gpu.gemm_grouped(models, xs)
    for a, b in zip(single, grouped):
        assert torch.equal(a, b)
    # mixed token counts in one grouped call; each token's row is the same bits
    Ms = [1, 3, 8, 12, 5]
    sub = gpu.gemm_grouped(models, [x[:M] for x, M in zip(xs, Ms)])
    for a, b, M in zip(single, sub, Ms):
        assert torch.equal(a[:M], b)
    for m, x, a in zip(models, xs, single):  # one token at a time
        for t in (0, 7, 15):
            assert torch.equal(m.gemm(x[t:t + 1], path=gpu.PATH_GEMV), a[t:t + 1])


@pytest.mark.parametrize("G", [2, 4, 8])
@pytest.mark.parametrize("M,path", [(1, 1), (16, 1), (160, 2)])
def test_sharded_bits_equal_unsharded(gpu, port, G, M, path):
    """Snake-sharded outputs, gathered and un-permuted, equal the unsharded
    result bit for bit (K1 segment order and K2 split count depend on the
    unsharded matrix only)."""
    import torch
    data = model_bytes(port, 8192, 1024, 2.5, m_b=512)
    x = torch.from_numpy(activations(port, M, 1024, seed=G)).cuda().to(torch.bfloat16)
    full = gpu.DeviceModel(data)
    y_full = full.gemm(x, path=path)
    shards = [gpu.DeviceModel(data, shard=g, num_shards=G) for g in range(G)]
    gathered = torch.stack([s.gemm(x, path=path) for s in shards])
    y = shards[0].unpermute_gathered(gathered, M)
    assert torch.equal(y, y_full)


def test_repeated_calls_and_streams(gpu, port, mid):
    import torch
    data, _ = mid
    dm = gpu.DeviceModel(data)
    x = torch.from_numpy(f32_activations(16, 4096, seed=1)).cuda()
    base = {M: dm.gemm(x[:M]) for M in (1, 16)}
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    ws1, ws2 = torch.zeros_like(dm.workspace(16)), torch.zeros_like(dm.workspace(16))
    torch.cuda.synchronize()
    for _ in range(3):
        with torch.cuda.stream(s1):
            a = dm.gemm(x, workspace=ws1, stream=s1)
        with torch.cuda.stream(s2):
            b = dm.gemm(x[:1], workspace=ws2, stream=s2)
        torch.cuda.synchronize()
        assert torch.equal(a, base[16])
        assert torch.equal(b, base[1])
