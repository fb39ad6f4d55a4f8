"""N-sharded path on one B200 ("virtual shards"): the G shard
device models run one after another on cuda:0, their outputs are stacked as
an all-gather would deliver them and un-permuted by the device kernel.  The
result must equal the unsharded GPU result bit for bit (same kernels, same
per-row accumulation order) and the oracle within the parity bar."""
import numpy as np
import pytest

from synth import LLAMA_70B, activations, errors, model_bytes

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("G", [2, 4, 8])
@pytest.mark.parametrize("M,path", [(1, 1), (16, 1), (160, 2)])
def test_virtual_shards_match_unsharded(gpu, port, G, M, path):
    import torch
    data = model_bytes(port, 8192, 1024, 2.5, m_b=512)
    x = torch.from_numpy(activations(port, M, 1024, seed=G)).cuda().to(torch.bfloat16)
    full = gpu.DeviceModel(data)
    y_full = full.gemm(x, path=path)
    shards = [gpu.DeviceModel(data, shard=g, num_shards=G) for g in range(G)]
    SR = shards[0].out_rows
    gathered = torch.stack([s.gemm(x, path=path) for s in shards])  # [G, M, SR]
    assert gathered.shape == (G, M, SR)
    y = shards[0].unpermute_gathered(gathered, M)
    # same per-row accumulation order (segments / K splits fixed by the
    # unsharded matrix): bit for bit
    assert torch.equal(y, y_full)
    ref = port.matmul(x.float().cpu().numpy()[:4], port.load(data).dequantize(), threads=8)
    assert errors(y.cpu().numpy()[:4], ref)[0] <= 1e-3


def test_llama70b_down_proj_shards_8way(gpu, port):
    """configs[3] shape: 70B down_proj (8192 x 28672) at avg 2.5 bits, 8 shards."""
    import torch
    rows, cols = LLAMA_70B["down_proj"]
    data = model_bytes(port, rows, cols, 2.5)
    x = torch.from_numpy(activations(port, 2, cols, seed=3)).cuda().to(torch.bfloat16)
    shards = [gpu.DeviceModel(data, shard=g, num_shards=8) for g in range(8)]
    y = shards[0].unpermute_gathered(torch.stack([s.gemm(x) for s in shards]), 2).cpu().numpy()
    ref = port.matmul(x.float().cpu().numpy(), port.load(data).dequantize(), threads=8)
    e_max, e_l2 = errors(y, ref)
    assert e_max <= 1e-3, (e_max, e_l2)
