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

A decoder layer has several linears and a decode step several token counts:
``ShardedLayer`` runs ALL of them with one grouped shard GEMM into one packed
send buffer, ONE all-gather and ONE un-permute launch (``sfmp_gemm_sharded``
with the library's NCCL communicator, or the same three steps over any
torch.distributed group -- gloo included -- for tests).  ``ShardedLinear``
is the one-matrix form.  The host logic also runs on CPU with gloo
(tests/test_sharded_host.py), where the per-rank GEMM result is supplied by
the caller.
"""
from __future__ import annotations

import numpy as np

from . import (PATH_AUTO, PATH_GEMV, DeviceModel, NcclComm, assemble_gathered, gemm_sharded,
               gemm_sharded_local, parse_header, shard_extract, shard_plan, sharded_gather_bytes,
               sharded_unpermute)


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


class ShardedLayer:
    """This rank's shards of several linears (e.g. q,k,v,o,gate,up,down), all
    computed with ONE collective per call.

    comm: a ``NcclComm`` (the library's own all-gather inside
    ``sfmp_gemm_sharded``, CUDA-graph capturable); otherwise ``group`` (any
    torch.distributed group; gloo groups gather through host memory)."""

    def __init__(self, blobs, rank: int, world: int, device: int, comm: NcclComm | None = None, group=None):
        self.rank, self.world, self.device = rank, world, device
        self.comm, self.group = comm, group
        self.models = [DeviceModel(b, device=device, shard=rank, num_shards=world) for b in blobs]
        self.rows = [m.info["global_rows"] for m in self.models]
        self._ws = {}
        self._buf = {}

    def workspaces(self, Ms):
        import torch
        out = []
        for i, (m, M) in enumerate(zip(self.models, Ms)):
            key = (i, M if M > 16 else 16)
            if key not in self._ws:
                n = m.workspace_bytes(key[1], PATH_GEMV if M <= 16 else PATH_AUTO)
                self._ws[key] = torch.zeros(max(n, 128), dtype=torch.uint8, device=f"cuda:{self.device}")
            out.append(self._ws[key])
        return out

    def gather_buffer(self, Ms):
        import torch
        key = tuple(Ms)
        if key not in self._buf:
            n = sharded_gather_bytes(self.models, Ms)
            self._buf[key] = torch.zeros(max(n // 4, 1), dtype=torch.float32, device=f"cuda:{self.device}")
        return self._buf[key]

    def __call__(self, xs, outs=None, stream=None):
        import torch
        Ms = [x.shape[0] for x in xs]
        if outs is None:
            outs = [torch.empty(M, r, dtype=torch.float32, device=x.device) for M, r, x in zip(Ms, self.rows, xs)]
        ws = self.workspaces(Ms)
        buf = self.gather_buffer(Ms)
        if self.comm is not None:
            return gemm_sharded(self.models, xs, outs, ws, buf, self.comm, stream=stream)
        import torch.distributed as dist
        total = sum(M * m.out_rows for m, M in zip(self.models, Ms))
        gemm_sharded_local(self.models, xs, buf, ws, stream=stream)
        send, recv = buf[:total], buf[total:total * (1 + self.world)]
        if dist.get_backend(self.group) == "gloo":
            host = send.cpu()
            parts = [torch.empty_like(host) for _ in range(self.world)]
            dist.all_gather(parts, host, group=self.group)
            recv.copy_(torch.cat(parts))
        else:
            dist.all_gather_into_tensor(recv, send, group=self.group)
        return sharded_unpermute(self.models, Ms, buf, outs, stream=stream)
