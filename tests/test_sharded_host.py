"""Multi-rank host logic of the N-sharded path on CPU (gloo, world_size 2):
snake partition -> per-shard SFMPPKD1 -> per-rank GEMV (oracle stands in
for the GPU kernel) -> all-gather -> un-permute == the unsharded oracle,
bit for bit (every output element is produced by exactly one rank)."""
import os
import socket

import numpy as np
import pytest

from synth import activations, model_bytes


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, data, x, ref, result_q):
    import torch.distributed as dist
    from oracle.oracle import Port
    from paper_2602_01027_b200.sharded import ShardPlan, gather_assemble_cpu
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        plan = ShardPlan(data, world)
        P = Port()
        local = P.load(plan.shard_bytes(rank))
        y_local = P.matmul(x, local.dequantize(), threads=1)
        assert y_local.shape[1] == plan.local_rows(rank)
        y = gather_assemble_cpu(y_local, plan)
        result_q.put((rank, bool(np.array_equal(y.view(np.uint32), ref.view(np.uint32))),
                      float(np.abs(y - ref).max())))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("mode", [3, 1, 0])
def test_gloo_two_rank_sharded_gemv_matches_oracle(port, mode):
    import torch.multiprocessing as mp
    data = model_bytes(port, 2048, 512, 2.5, mode=mode)
    x = activations(port, 3, 512, seed=1)
    ref = port.matmul(x, port.load(data).dequantize(), threads=1)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    p0 = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, p0, data, x, ref, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert [r[0] for r in res] == [0, 1]
    assert all(r[1] for r in res), res


@pytest.mark.parametrize("G", [2, 4, 8])
def test_snake_partition_balances_high_bit_rows(port, G):
    """salience-sorted rows put high-bit blocks first; the snake
    partition keeps per-shard code bits within a few % of each other."""
    from paper_2602_01027_b200.sharded import ShardPlan
    data = model_bytes(port, 8192, 1024, 2.5, m_b=512)
    plan = ShardPlan(data, G)
    bits = plan.shard_code_bits()
    assert bits.max() / bits.min() < 1.05, bits
    # every original row appears exactly once across the shards
    gm = plan.gather_map
    rows = gm[gm != 0xFFFFFFFF]
    assert np.array_equal(np.sort(rows), np.arange(8192))


def test_single_process_assembly_all_shard_counts(port):
    """Assembly over G = 1..8 shards in one process (no collective)."""
    from oracle.oracle import Port  # noqa: F401
    import paper_2602_01027_b200 as sfmp
    data = model_bytes(port, 4096, 256, 3.0, m_b=512)
    x = activations(port, 2, 256, seed=2)
    ref = port.matmul(x, port.load(data).dequantize(), threads=1)
    for G in range(1, 9):
        gmap, SR = sfmp.shard_plan(data, G)
        gathered = np.zeros((G, 2, SR), np.float32)
        for g in range(G):
            loc = port.load(sfmp.shard_extract(data, g, G))
            y = port.matmul(x, loc.dequantize(), threads=1)
            gathered[g, :, :y.shape[1]] = y
        y = sfmp.assemble_gathered(gathered, gmap, 4096)
        assert np.array_equal(y.view(np.uint32), ref.view(np.uint32)), G


def test_shard_errors(port):
    import paper_2602_01027_b200 as sfmp
    data = model_bytes(port, 1024, 256, 3.0, m_b=512)
    with pytest.raises(sfmp.ConfigError):
        sfmp.shard_extract(data, 2, 2)
    with pytest.raises(sfmp.ShapeError):  # 2 block rows cannot split 4 ways
        sfmp.shard_plan(data, 4)
