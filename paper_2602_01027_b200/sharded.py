"""N-sharded mixed-precision linear over torch.distributed.

The output rows of one SFMP matrix are split by the snake (boustrophedon)
block-row partition (``sfmp_shard_plan``): rank g holds the block rows
``g, 2G-1-g, 2G+g, ...`` so the salience-sorted high-bit block rows spread
evenly.  Each rank runs the GEMM on its shard (device model built from the
shard's SFMPPKD1 spans only), the shard outputs ``[M, SR]`` (SR = padded rows
per shard, shard-local reordered order) are all-gathered into
``[G, M, SR]`` and un-permuted to the original row order ``[M, rows]``.

There is no reference counterpart (the reference is single-threaded,
SPEC.md:553 only permits row-range parallelism with a deterministic merge);
the merge here is deterministic because every output element comes from
exactly one rank.

On GPUs the collective is NCCL ``all_gather_into_tensor`` over NVLink and the
un-permutation is the ``sfmp_unpermute_gathered`` kernel; the same host logic
runs on CPU with the gloo backend (tests/test_sharded_host.py), where the
per-rank GEMM result is supplied by the caller.
"""
from __future__ import annotations

import numpy as np

from . import (DeviceModel, PATH_AUTO, assemble_gathered, parse_header, shard_extract,
               shard_plan)


class ShardPlan:
    """Host-side description of one matrix split over ``world`` ranks."""

    def __init__(self, data: bytes, world: int):
        self.data = data
        self.world = world
        self.info = parse_header(data)
        self.rows = int(self.info["rows"])
        self.gather_map, self.shard_rows = shard_plan(data, world)

    def shard_bytes(self, rank: int) -> bytes:
        return shard_extract(self.data, rank, self.world)

    def local_rows(self, rank: int) -> int:
        return int(np.count_nonzero(self.gather_map[rank] != 0xFFFFFFFF))

    def shard_code_bits(self) -> np.ndarray:
        """Sum of code bits held by each shard (load balance of the partition)."""
        return np.array([parse_header(self.shard_bytes(g))["avg_code_bits"] *
                         parse_header(self.shard_bytes(g))["block_count"]
                         for g in range(self.world)])


def gather_assemble_cpu(y_local: np.ndarray, plan: ShardPlan, group=None) -> np.ndarray:
    """All-gather this rank's [M, local_rows] result (gloo) and un-permute."""
    import torch
    import torch.distributed as dist
    M = y_local.shape[0]
    padded = np.zeros((M, plan.shard_rows), np.float32)
    padded[:, :y_local.shape[1]] = y_local
    t = torch.from_numpy(padded)
    outs = [torch.empty_like(t) for _ in range(plan.world)]
    dist.all_gather(outs, t, group=group)
    gathered = torch.stack(outs).numpy()
    return assemble_gathered(gathered, plan.gather_map, plan.rows)


class ShardedLinear:
    """One rank's view of an N-sharded matrix on its GPU (NCCL all-gather)."""

    def __init__(self, data: bytes, rank: int, world: int, device: int, group=None):
        self.plan = ShardPlan(data, world)
        self.rank, self.world, self.group = rank, world, group
        self.model = DeviceModel(data, device=device, shard=rank, num_shards=world)
        self.device = device

    def __call__(self, x, out=None, path: int = PATH_AUTO, workspace=None, y_local=None, gathered=None):
        import torch
        import torch.distributed as dist
        M = x.shape[0]
        y_local = self.model.gemm(x, out=y_local, path=path, workspace=workspace)
        if gathered is None:
            gathered = torch.empty(self.world, M, self.model.out_rows, device=x.device)
        dist.all_gather_into_tensor(gathered, y_local, group=self.group)
        return self.model.unpermute_gathered(gathered, M, out=out)
