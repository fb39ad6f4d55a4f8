"""Sharded calls with ONE collective (sfmp_gemm_sharded_local / sfmp_sharded_unpermute /
sfmp_gemm_sharded), call statistics (sfmp_stats, the GemvStats counterpart of
lutgemm.hpp:47-52) and gemv_block (lutgemm.cpp:87-93) on the GPU.

Sharded results must be bit-identical to the unsharded call: every output
row is computed by exactly one shard in the same canonical order, the merge
is a pure scatter.
"""
import os
import socket
import subprocess
import sys

import numpy as np
import pytest

from synth import activations, errors, model_bytes

pytestmark = pytest.mark.gpu

SHAPES = [(1024, 1024, 3.25, 128), (2048, 1024, 2.5, 512), (512, 2048, 3.5, 128)]


def _blobs(port):
    return [model_bytes(port, r, c, b, m_b=mb) for r, c, b, mb in SHAPES]


def _unsharded(gpu, blobs, xs):
    import torch
    ms = [gpu.DeviceModel(b) for b in blobs]
    outs = []
    for m, x in zip(ms, xs):
        outs.append(m.gemm(x))
    torch.cuda.synchronize()
    return outs


@pytest.mark.parametrize("G", [2, 4])
def test_virtual_shards_packed_one_collective(gpu, port, G):
    """G virtual ranks on one GPU: each runs ONE grouped shard GEMM into its
    packed send block; the all-gather is emulated by concatenating the send
    blocks; ONE un-permute launch per rank gives the unsharded bits."""
    import torch
    blobs = _blobs(port)
    Ms = [1, 5, 40]  # two decode problems and one prefill problem in one call
    xs = [torch.from_numpy(activations(port, M, c, seed=M)).cuda().to(torch.bfloat16)
          for M, (r, c, b, mb) in zip(Ms, SHAPES)]
    ref = _unsharded(gpu, blobs, xs)
    ranks = []
    for g in range(G):
        models = [gpu.DeviceModel(b, shard=g, num_shards=G) for b in blobs]
        nbytes = gpu.sharded_gather_bytes(models, Ms)
        buf = torch.zeros(nbytes // 4, dtype=torch.float32, device="cuda")
        ws = [torch.zeros(max(m.workspace_bytes(16 if M <= 16 else M), 128), dtype=torch.uint8, device="cuda")
              for m, M in zip(models, Ms)]
        gpu.gemm_sharded_local(models, xs, buf, ws)
        ranks.append((models, buf))
    total = gpu.packed_offsets(ranks[0][0], Ms)[-1]
    send = torch.cat([buf[:total] for _, buf in ranks])
    for models, buf in ranks:
        buf[total:].copy_(send)  # the all-gather
        outs = [torch.full((M, r), float("nan"), device="cuda") for M, (r, c, b, mb) in zip(Ms, SHAPES)]
        gpu.sharded_unpermute(models, Ms, buf, outs)
        torch.cuda.synchronize()
        for o, y in zip(outs, ref):
            assert torch.equal(o, y)


def test_nccl_world1_and_graph_capture(gpu, port):
    """The C-ABI NCCL path (sfmp_gemm_sharded, library-created communicator)
    at world size 1, eagerly and replayed from a CUDA graph."""
    import torch
    blobs = _blobs(port)
    Ms = [1, 16, 3]
    xs = [torch.from_numpy(activations(port, M, c, seed=10 + M)).cuda().to(torch.bfloat16)
          for M, (r, c, b, mb) in zip(Ms, SHAPES)]
    ref = _unsharded(gpu, blobs, xs)
    comm = gpu.NcclComm(1, 0, 0, gpu.NcclComm.unique_id())
    try:
        from paper_2602_01027_b200.sharded import ShardedLayer
        layer = ShardedLayer(blobs, 0, 1, 0, comm=comm)
        outs = layer(xs)
        torch.cuda.synchronize()
        for o, y in zip(outs, ref):
            assert torch.equal(o, y)
        s = torch.cuda.Stream()
        outs2 = [torch.zeros_like(o) for o in outs]
        with torch.cuda.stream(s):
            layer(xs, outs=outs2, stream=s)  # warm (allocates nothing new)
        torch.cuda.synchronize()
        for o in outs2:
            o.zero_()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            layer(xs, outs=outs2, stream=s)
        g.replay()
        torch.cuda.synchronize()
        for o, y in zip(outs2, ref):
            assert torch.equal(o, y)
    finally:
        comm.close()


def test_sharded_errors(gpu, port):
    import torch
    blobs = _blobs(port)
    plain = gpu.DeviceModel(blobs[0])
    with pytest.raises(gpu.ConfigError):
        gpu.sharded_gather_bytes([plain], [1])
    a = gpu.DeviceModel(blobs[0], shard=0, num_shards=2)
    b = gpu.DeviceModel(blobs[1], shard=1, num_shards=2)
    with pytest.raises(gpu.ConfigError):
        gpu.sharded_gather_bytes([a, b], [1, 1])
    comm = gpu.NcclComm(1, 0, 0, gpu.NcclComm.unique_id())
    try:  # communicator of size 1 for a 2-way partition
        x = torch.zeros(1, 1024, device="cuda", dtype=torch.bfloat16)
        buf = torch.zeros(gpu.sharded_gather_bytes([a], [1]) // 4, device="cuda")
        ws = [torch.zeros(a.workspace_bytes(16), dtype=torch.uint8, device="cuda")]
        with pytest.raises(gpu.ConfigError):
            gpu.gemm_sharded([a], [x], [torch.empty(1, 1024, device="cuda")], ws, buf, comm)
    finally:
        comm.close()


def test_call_stats(gpu, port):
    """sfmp_stats: device time from events, algorithmic bytes, path and launches."""
    import torch
    data = model_bytes(port, 1024, 1024, 3.25)
    dm = gpu.DeviceModel(data)
    x = torch.from_numpy(activations(port, 4, 1024)).cuda().to(torch.bfloat16)
    y, st = dm.gemm_stats(x)
    info = dm.info
    assert st["device_us"] > 0 and st["wall_us"] >= st["device_us"] * 0.5
    assert st["path"] == gpu.PATH_GEMV and st["launches"] >= 2
    assert st["bytes"] == info["payload_bytes"] + 4 * 1024 + 4 * 1024 + 2 * 4 * 1024 + 4 * 4 * 1024
    assert st["flops"] == 2.0 * 4 * 1024 * 1024
    assert torch.equal(y, dm.gemm(x))
    xh = activations(port, 2, 1024, seed=3)
    yh, sh = dm.gemm_host(xh, stats=True)
    assert sh["h2d_us"] > 0 and sh["d2h_us"] > 0 and sh["device_us"] > 0
    assert np.array_equal(yh, dm.gemm(torch.from_numpy(xh).cuda()).cpu().numpy())
    n0 = gpu.launch_count()
    dm.gemm(x)
    assert gpu.launch_count() - n0 == st["launches"]


def test_gemv_block(gpu, port):
    """gemv_block vs the oracle's dequantized block times the reordered x."""
    import torch
    data = model_bytes(port, 1024, 2048, 3.25, m_b=256)
    dm = gpu.DeviceModel(data)
    pm = port.load(data)
    w = pm.dequantize().astype(np.float64)
    x = activations(port, 1, 2048, seed=5)[0].astype(np.float64)
    xr = x[pm.col_perm]
    BC = 2048 // 128
    for k in (0, 1, BC + 3, 4 * BC - 1):
        br, bc = divmod(k, BC)
        rows = pm.row_perm[br * 256:(br + 1) * 256]
        cols = pm.col_perm[bc * 128:(bc + 1) * 128]
        ref = w[np.ix_(rows, cols)] @ x[cols]
        got = dm.gemv_block(k, torch.from_numpy(xr).cuda()).cpu().numpy()
        assert errors(got[None], ref[None])[0] <= 1e-5
    with pytest.raises(gpu.ShapeError):
        dm.gemv_block(4 * BC, torch.from_numpy(xr).cuda())


_WORKER = r"""
import os, sys, torch, torch.distributed as dist
sys.path.insert(0, os.environ["SFMP_ROOT"]); sys.path.insert(0, os.path.join(os.environ["SFMP_ROOT"], "tests"))
import paper_2602_01027_b200 as sfmp
from paper_2602_01027_b200.sharded import ShardedLayer
from oracle.oracle import Port
from synth import activations, model_bytes
rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
dist.init_process_group("gloo")
port = Port()
shapes = [(1024, 1024, 3.25, 128), (2048, 1024, 2.5, 512), (512, 2048, 3.5, 128)]
blobs = [model_bytes(port, r, c, b, m_b=mb) for r, c, b, mb in shapes]
Ms = [2, 16, 33]
xs = [torch.from_numpy(activations(port, M, c, seed=M)).cuda().to(torch.bfloat16) for M, (r, c, b, mb) in zip(Ms, shapes)]
layer = ShardedLayer(blobs, rank, world, 0)
outs = layer(xs)
torch.cuda.synchronize()
ref = [sfmp.DeviceModel(b).gemm(x) for b, x in zip(blobs, xs)]
ok = all(torch.equal(o, y) for o, y in zip(outs, ref))
dist.destroy_process_group()
sys.exit(0 if ok else 1)
"""


def test_two_processes_gloo_real_shard_kernels(gpu, port, tmp_path):
    """world_size 2 over gloo, both ranks on cuda:0: the real shard kernels,
    packed send block, host all-gather and un-permute kernel, bit-exact."""
    _blobs(port)  # build the fixtures once (cached for the workers)
    script = tmp_path / "worker.py"
    script.write_text(_WORKER)
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port_no = s.getsockname()[1]
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    procs = []
    for r in range(2):
        env = dict(os.environ, RANK=str(r), WORLD_SIZE="2", MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port_no),
                   SFMP_ROOT=root)
        procs.append(subprocess.Popen([sys.executable, str(script)], env=env))
    codes = [p.wait(timeout=300) for p in procs]
    assert codes == [0, 0]


def test_decode_only_model_memory(gpu, port):
    """SFMP_MODEL_DECODE_ONLY: one resident weight layout (<= 1.1x the SFMPPKD1
    payload); decode bits equal the default model's; M > 16 runs the decode
    GEMV in 16-token chunks within the parity bar; the GEMM path is refused."""
    import torch
    data = model_bytes(port, 4096, 4096, 3.25)
    full = gpu.DeviceModel(data)
    lean = gpu.DeviceModel(data, flags=gpu.MODEL_DECODE_ONLY)
    assert lean.info["device_bytes"] <= 1.1 * lean.info["payload_bytes"], lean.info
    assert full.info["device_bytes"] > 1.8 * full.info["payload_bytes"]
    x = torch.from_numpy(activations(port, 5, 4096, seed=4)).cuda().to(torch.bfloat16)
    assert torch.equal(lean.gemm(x), full.gemm(x, path=gpu.PATH_GEMV))
    x40 = activations(port, 40, 4096, seed=6)
    y = lean.gemm(torch.from_numpy(x40).cuda()).cpu().numpy()
    ref = port.matmul(x40, port.load(data).dequantize(), threads=8)
    assert errors(y, ref)[0] <= 1e-3
    with pytest.raises(gpu.UnsupportedError):
        lean.gemm(torch.from_numpy(x40).cuda(), path=gpu.PATH_GEMM)
