#!/usr/bin/env python
"""bench.py -- the SFMP mixed-precision GEMM hot path on B200 (driver contract).

Workload (BASELINE.json configs[1]): the seven Llama-3.1-8B linear shapes
(q,k,v,o,gate,up,down) at avg 3.25 code bits (block-wise 3/4-bit, m_b=512 --
k/v use m_b=128 so they split 8 ways -- n_b=128, rowcol reorder), decode with
M in {1,2,4,8,16} tokens.  One step = the 7 linears x 5 token counts = 35
GEMM calls, each through the decode GEMV kernel (K1).  Weights are rotated
over 6 device copies of the layer (576 MB >> 126 MB L2), so every call
streams its weights from HBM.

N>1 (torchrun): each linear is N-sharded by the snake block-row partition,
every rank runs its shard, the shard outputs are gathered with NCCL
all_gather_into_tensor and un-permuted (strong scaling).

--impl reference times the reference's own CPU implementation
(oracle/_ref = /root/reference/proj compiled unmodified; else the C port) on
the same workload with all host threads (token-parallel).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

BASE = json.load(open(os.path.join(ROOT, "BASELINE.json")))
METRIC = BASE["metric"]
PROJS = ["q_proj", "k_proj", "v_proj", "o_proj", "gate_proj", "up_proj", "down_proj"]
SHAPES = {"q_proj": (4096, 4096), "k_proj": (1024, 4096), "v_proj": (1024, 4096),
          "o_proj": (4096, 4096), "gate_proj": (14336, 4096), "up_proj": (14336, 4096),
          "down_proj": (4096, 14336)}
MS = [1, 2, 4, 8, 16]
AVG_BITS = 3.25
COPIES = 6
WORKLOAD = ("llama3.1-8b decoder-layer linears q,k,v,o,gate,up,down; avg 3.25 code bits "
            "block-wise 3/4 (m_b=512, k/v m_b=128; n_b=128); rowcol reorder; decode M in "
            "{1,2,4,8,16}; one step = 35 GEMM calls")


def peaks():
    try:
        p = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
        return float(p["hbm_gbs"]), float(p["bf16_tflops"]), "measured"
    except Exception:
        return 6650.0, 1590.0, "fallback"


def m_b_of(proj):
    return 128 if proj in ("k_proj", "v_proj") else 512


def build_bytes(port, proj):
    from synth import model_bytes
    rows, cols = SHAPES[proj]
    seed = {"up_proj": 4, "v_proj": 1}.get(proj, 0)  # up/v reuse gate/k's weights (synthetic)
    return model_bytes(port, rows, cols, AVG_BITS, mode=3, m_b=m_b_of(proj), n_b=128, seed=seed)


def algo_bytes(info, M, rows, cols):
    """planes + fp16 s,z + perms + bf16 x + f32 y."""
    return info["payload_bytes"] + 4 * cols + 4 * rows + 2 * M * cols + 4 * M * rows


# ---------------------------------------------------------------------------
# clocks sampled during the timed region (B200_PROFILING.md)
# ---------------------------------------------------------------------------
class ClockSampler:
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.proc = None
        self.path = f"/tmp/sfmp_clocks_{os.getpid()}.csv"

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        sm, smax, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in open(self.path):
            f = [c.strip() for c in line.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                smax = float(f[2])
            except ValueError:
                continue
            for n, v in zip(names, f[5:9]):
                if v.lower() == "active":
                    reasons.add(n)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": smax,
                "reasons": sorted(reasons), "samples": len(sm)}


# ---------------------------------------------------------------------------
# CPU baselines (reference compiled unmodified, else the C port)
# ---------------------------------------------------------------------------
def cpu_handles(port, blobs):
    from oracle.oracle import Reference, reference_available
    if reference_available():
        R = Reference()
        return "reference", {p: R.load(b) for p, b in blobs.items()}
    return "port", {p: port.load(b) for p, b in blobs.items()}


def cpu_gemm(kind, h, x, threads):
    return h.gemm(x, threads) if kind == "reference" else h.gemm_lut(x, threads)


def cpu_baseline_sample(port, blobs):
    """Bounded sample on rank 0: the reference gemv, single thread, 3 reps per
    projection at M=1; the step time is extrapolated linearly over the 31
    token-GEMVs per projection of one step (gemv loops per token)."""
    kind, hs = cpu_handles(port, blobs)
    total = 0.0
    per = {}
    for p in PROJS:
        x = port.gen_activation(1, SHAPES[p][1], 3000)
        cpu_gemm(kind, hs[p], x, 1)
        ts = []
        for _ in range(3):
            t0 = time.perf_counter()
            cpu_gemm(kind, hs[p], x, 1)
            ts.append(time.perf_counter() - t0)
        per[p] = statistics.median(ts) * 1e6
        total += per[p] * sum(MS)
    return {"value": total, "unit": "us", "cores": 1, "kind": kind,
            "sample": f"{kind} gemv (lutgemm.cpp:95) single-threaded, median of 3 reps per "
                      f"projection at M=1, x{sum(MS)} token-GEMVs per projection per step "
                      f"(linear extrapolation); host has {os.cpu_count()} cores",
            "per_proj_us_m1": {k: round(v, 1) for k, v in per.items()}}


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    from oracle.oracle import Port
    port = Port()
    blobs = {p: build_bytes(port, p) for p in PROJS}
    kind, hs = cpu_handles(port, blobs)
    threads = max(1, min(os.cpu_count() or 1, 16))
    xs = {(p, M): port.gen_activation(M, SHAPES[p][1], 3000 + M) for p in PROJS for M in MS}

    def step():
        for M in MS:
            for p in PROJS:
                cpu_gemm(kind, hs[p], xs[(p, M)], threads)

    for _ in range(args.warmup):
        step()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        step()
    dt = (time.perf_counter() - t0) / args.steps * 1e6
    out = {"metric": METRIC, "value": round(dt, 1), "unit": "us", "n_gpus": args.gpus,
           "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(dt / 1e3, 3),
           "higher_is_better": False, "scaling": "strong", "vs_baseline": None, "dtype": "f32",
           "data": "synthetic", "impl": "reference",
           "config": {"workload": WORKLOAD, "parallelism": f"host threads={threads} token-parallel"},
           "cpu_baseline": {"value": round(dt, 1), "unit": "us", "cores": threads, "kind": kind,
                            "sample": f"full step: 35 calls of {kind} gemv looped per token, "
                                      f"{threads} threads over tokens; host has "
                                      f"{os.cpu_count()} cores"},
           "e2e": {"value": round(dt, 1), "unit": "us", "h2d_bytes_per_step": 0,
                   "d2h_bytes_per_step": 0}}
    print(json.dumps(out), flush=True)
    return 0


# ---------------------------------------------------------------------------
# dense cuBLAS comparison (the paper's kernel comparison):
# the same decode step with dense bf16 weights through torch.matmul (cuBLAS)
# ---------------------------------------------------------------------------
def dense_leg(dev, stream, xs, args):
    import torch
    copies = 2  # 2 x 436 MB of dense weights >> L2
    W = [{p: torch.randn(SHAPES[p][0], SHAPES[p][1], device=dev, dtype=torch.bfloat16) * 0.02 for p in PROJS}
         for _ in range(copies)]
    ys = {(p, M): torch.empty(M, SHAPES[p][0], device=dev, dtype=torch.bfloat16) for p in PROJS for M in MS}

    def step(i):
        for mi, M in enumerate(MS):
            c = (i * len(MS) + mi) % copies
            for p in PROJS:
                torch.matmul(xs[(p, M)], W[c][p].t(), out=ys[(p, M)])

    with torch.cuda.stream(stream):
        step(0)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=stream):
        for i in range(copies):
            step(i)
    g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = 5
    with torch.cuda.stream(stream):
        e0.record(stream)
        for _ in range(reps):
            g.replay()
        e1.record(stream)
    torch.cuda.synchronize()
    us = e0.elapsed_time(e1) * 1e3 / (reps * copies)
    del W
    torch.cuda.empty_cache()
    byts = sum(2 * SHAPES[p][0] * SHAPES[p][1] for p in PROJS) * len(MS)
    return {"what": "same decode step, dense bf16 weights, torch.matmul (cuBLAS), CUDA graph",
            "us": round(us, 1), "GBps": round(byts / us / 1e3, 1)}


# ---------------------------------------------------------------------------
# prefill leg (configs[2]): the 7 linears at M=2048 through K2 (tcgen05 GEMM)
# ---------------------------------------------------------------------------
def prefill_leg(sfmp, port, models, dev, stream, args):
    import torch
    from synth import errors
    M = args.prefill_M
    xs = {p: torch.from_numpy(port.gen_activation(M, SHAPES[p][1], 4000)).to(dev).to(torch.bfloat16)
          for p in PROJS}
    ys = {p: torch.empty(M, SHAPES[p][0], device=dev) for p in PROJS}
    ws = {p: models[0][p].workspace(M, sfmp.PATH_GEMM) for p in PROJS}

    def one(c, p):
        models[c][p].gemm(xs[p], out=ys[p], path=sfmp.PATH_GEMM, workspace=ws[p])

    # parity spot check (q_proj, 8 sampled tokens) against the oracle
    one(0, "q_proj")
    torch.cuda.synchronize()
    sample = [0, 1, 777, 1024, 1500, 2000, M - 2, M - 1]
    w = port.load(build_bytes(port, "q_proj")).dequantize()
    ref = port.matmul(xs["q_proj"][sample].float().cpu().numpy(), w, threads=8)
    par = errors(ys["q_proj"][sample].cpu().numpy(), ref)[0]
    per = {}
    hbm, tc, src = peaks()
    for p in PROJS:
        with torch.cuda.stream(stream):
            for c in range(COPIES):
                one(c, p)
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=stream):
            for c in range(COPIES):
                one(c, p)
        g.replay()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        reps = max(2, args.steps // 10)
        with torch.cuda.stream(stream):
            e0.record(stream)
            for _ in range(reps):
                g.replay()
            e1.record(stream)
        torch.cuda.synchronize()
        us = e0.elapsed_time(e1) * 1e3 / (reps * COPIES)
        rows, cols = SHAPES[p]
        per[p] = {"us": round(us, 2), "tflops": round(2.0 * M * rows * cols / us / 1e6, 1)}
    tot_us = sum(v["us"] for v in per.values())
    flops = sum(2.0 * M * SHAPES[p][0] * SHAPES[p][1] for p in PROJS)
    ach = flops / tot_us / 1e6
    return {"metric": "prefill GEMM us per decoder layer (7 linears)", "M": M, "value": round(tot_us, 1),
            "unit": "us", "kernel": "K2 tcgen05 GEMM (gemm_kernel) + xprep_gemm_kernel",
            "per_proj": per, "parity_max_rel_err_q_proj_sampled": round(par, 7),
            "roofline": {"bound": "tensor", "achieved": round(ach, 1), "peak": tc, "unit": "TFLOP/s",
                         "frac": round(ach / tc, 4), "peak_source": f"MEASURED_PEAKS.json bf16_tflops ({src})",
                         "note": "time includes the x gather/convert pre-pass"}}


# ---------------------------------------------------------------------------
# GPU arm
# ---------------------------------------------------------------------------
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-graph", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--soak-ms", type=float, default=1500.0)
    ap.add_argument("--no-prefill", action="store_true")
    ap.add_argument("--no-group", action="store_true", help="one launch per linear instead of per decoder layer")
    ap.add_argument("--group-per-m", action="store_true",
                    help="one grouped call per M (5 launches) instead of one call for the whole step "
                         "(the API then issues one launch per n-tile class: M<=8 and M=16)")
    ap.add_argument("--prefill-M", type=int, default=2048)
    ap.add_argument("--e2e-order", default="", help="comma list: order of the M groups in the e2e step")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    if args.impl == "reference":
        return run_reference(args)

    import torch
    import torch.distributed as dist
    import paper_2602_01027_b200 as sfmp
    from oracle.oracle import Port

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"))
    dev = torch.device(f"cuda:{local}")
    port = Port()
    blobs = {p: build_bytes(port, p) for p in PROJS}
    # 6 device copies of the layer (each shard of it when world > 1)
    models = [{p: (sfmp.DeviceModel(blobs[p], device=local) if world == 1 else
                   sfmp.DeviceModel(blobs[p], device=local, shard=rank, num_shards=world))
               for p in PROJS} for _ in range(COPIES)]
    infos = {p: sfmp.parse_header(blobs[p]) for p in PROJS}
    xs = {(p, M): torch.from_numpy(port.gen_activation(M, SHAPES[p][1], 3000 + M)).to(dev)
          .to(torch.bfloat16) for p in PROJS for M in MS}
    ys = {(p, M): torch.empty(M, models[0][p].out_rows, device=dev) for p in PROJS for M in MS}
    ws = {p: models[0][p].workspace(16, sfmp.PATH_GEMV) for p in PROJS}
    # a workspace per (linear, M): problems of one launch must not share one
    wsm = {(p, M): torch.zeros_like(ws[p]) for p in PROJS for M in MS}
    if world > 1:
        gath = {(p, M): torch.empty(world, M, models[0][p].out_rows, device=dev)
                for p in PROJS for M in MS}
        yfull = {(p, M): torch.empty(M, SHAPES[p][0], device=dev) for p in PROJS for M in MS}

    grouped = not args.no_group
    across = grouped and not args.group_per_m and world == 1
    # launches of OUR kernels per step: grouped = (x pre-pass + GEMV) per M;
    # per-linear = (x pre-pass + GEMV) per call; sharded adds the un-permute
    n_class = len({M > 8 for M in MS})
    launches_per_step = ((n_class * 2 if across else len(MS) * 2) if grouped else len(MS) * len(PROJS) * 2) + \
        (len(MS) * len(PROJS) if world > 1 else 0)

    def step(i, group=grouped):
        if group and across:
            # the whole step (7 linears x 5 token counts, 4 weight copies) in one
            # grouped call: one pre-pass + one GEMV launch per n-tile class
            keys = [(p, M, (i * len(MS) + mi) % COPIES) for mi, M in enumerate(MS) for p in PROJS]
            sfmp.gemm_grouped([models[c][p] for p, M, c in keys], [xs[(p, M)] for p, M, c in keys],
                              outs=[ys[(p, M)] for p, M, c in keys], workspaces=[wsm[(p, M)] for p, M, c in keys])
            return
        for mi, M in enumerate(MS):
            c = (i * len(MS) + mi) % COPIES
            if group:
                sfmp.gemm_grouped([models[c][p] for p in PROJS], [xs[(p, M)] for p in PROJS],
                                  outs=[ys[(p, M)] for p in PROJS], workspaces=[ws[p] for p in PROJS])
            else:
                for p in PROJS:
                    models[c][p].gemm(xs[(p, M)], out=ys[(p, M)], path=sfmp.PATH_GEMV, workspace=ws[p])
            if world > 1:
                for p in PROJS:
                    dist.all_gather_into_tensor(gath[(p, M)], ys[(p, M)])
                    models[c][p].unpermute_gathered(gath[(p, M)], M, out=yfull[(p, M)])

    # correctness spot check against the oracle (rank 0, cheap shapes)
    step(0)
    torch.cuda.synchronize()
    parity = {}
    if rank == 0:
        from synth import errors
        for p in ("q_proj", "k_proj"):
            w = port.load(blobs[p]).dequantize()
            ref = port.matmul(xs[(p, 16)].float().cpu().numpy(), w, threads=8)
            got = (yfull if world > 1 else ys)[(p, 16)].cpu().numpy()
            parity[p] = round(errors(got, ref)[0], 9)

    use_graph = (world == 1) and not args.no_graph
    stream = torch.cuda.Stream(device=dev)
    graphs = []
    if use_graph:
        # one graph per rotation phase so each replay touches the next weight copies
        with torch.cuda.stream(stream):
            for i in range(COPIES):
                step(i)
        torch.cuda.synchronize()
        for i in range(COPIES):
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=stream):
                step(i)
            graphs.append(g)

    def run_step(i):
        if use_graph:
            graphs[i % COPIES].replay()
        else:
            step(i)

    with torch.cuda.stream(stream):
        for i in range(args.warmup):
            run_step(i)
    torch.cuda.synchronize()
    clocks = ClockSampler(local)
    clocks.start()
    # untimed soak so the clock sampler sees the GPU under this load
    t_end = time.perf_counter() + args.soak_ms / 1e3
    i = 0
    with torch.cuda.stream(stream):
        while time.perf_counter() < t_end:
            run_step(i)
            i += 1
            if i % 20 == 0:
                torch.cuda.synchronize()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(stream):
        e0.record(stream)
        for i in range(args.steps):
            run_step(i)
        e1.record(stream)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    clk = clocks.stop()
    t_ms = e0.elapsed_time(e1) / args.steps
    if world > 1:
        tt = torch.tensor([t_ms], device=dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        t_ms = float(tt.item())

    # ---- secondary: the same step with one launch per linear (no grouping) ----
    ungrouped_ms = None
    if world == 1 and grouped and use_graph:
        with torch.cuda.stream(stream):
            step(0, group=False)
        torch.cuda.synchronize()
        ug = []
        for i in range(COPIES):
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=stream):
                step(i, group=False)
            ug.append(g)
        reps = max(COPIES, args.steps // 2)
        u0, u1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(stream):
            for i in range(3):
                ug[i % COPIES].replay()
            u0.record(stream)
            for i in range(reps):
                ug[i % COPIES].replay()
            u1.record(stream)
        torch.cuda.synchronize()
        ungrouped_ms = u0.elapsed_time(u1) / reps

    # ---- e2e: host buffers in, host buffers out, through the public API ----
    # One pinned host buffer holds every x of the step (f32, as the reference's
    # Vector) and one every y: one H2D + the grouped calls + one D2H per step,
    # replayed as a CUDA graph, then the host waits for y (the step's result).
    keys = [(p, M) for M in MS for p in PROJS]
    xoff, yoff, xo, yo = {}, {}, 0, 0
    for k in keys:
        xoff[k], yoff[k] = xo, yo
        xo += k[1] * SHAPES[k[0]][1]
        yo += k[1] * SHAPES[k[0]][0]
    hxb = torch.empty(xo, dtype=torch.float32).pin_memory()
    hyb = torch.empty(yo, dtype=torch.float32).pin_memory()
    for (p, M) in keys:
        hxb[xoff[(p, M)]:xoff[(p, M)] + M * SHAPES[p][1]] = torch.from_numpy(
            port.gen_activation(M, SHAPES[p][1], 3000 + M)).reshape(-1)
    dxb = torch.empty(xo, dtype=torch.float32, device=dev)
    dyb = torch.empty(yo, dtype=torch.float32, device=dev)
    dx = {k: dxb[xoff[k]:xoff[k] + k[1] * SHAPES[k[0]][1]].view(k[1], SHAPES[k[0]][1]) for k in keys}
    dy = {k: dyb[yoff[k]:yoff[k] + k[1] * SHAPES[k[0]][0]].view(k[1], SHAPES[k[0]][0]) for k in keys}
    h2d, d2h = xo * 4, yo * 4

    # group boundaries (x / y of one M are contiguous in the host buffers)
    gx = {M: (xoff[(PROJS[0], M)], xoff[(PROJS[-1], M)] + M * SHAPES[PROJS[-1]][1]) for M in MS}
    gy = {M: (yoff[(PROJS[0], M)], yoff[(PROJS[-1], M)] + M * SHAPES[PROJS[-1]][0]) for M in MS}
    h2d_s, d2h_s = torch.cuda.Stream(device=dev), torch.cuda.Stream(device=dev)

    # Group order of the e2e step: a small group first (short exposed H2D), the
    # largest late enough that its H2D (2.5 MB, the slowest copy) hides under
    # three groups' compute, a small group last (short exposed D2H).  Measured
    # (200 steps each, noisy): 1,4,8,16,2 -> 247-283 us; 1,16,8,4,2 -> 270-350;
    # 1,2,4,8,16 -> 290-348.
    # --e2e-order: groups separated by '/', token counts by ',' (one grouped call
    # per group; its H2D / D2H overlap the other groups' compute).  Measured
    # (200 steps, two runs each): 1/4/8/16/2 244-245 us; 1,2/16/4,8 247-250;
    # 1,2/4,8/16 259-268; 1/16/2,4,8 262-264; 1,2,4,8/16 296 -- finer groups
    # overlap the PCIe copies better than fewer, larger launches.
    E2E_GROUPS = ([[int(v) for v in g.split(",")] for g in args.e2e_order.split("/")] if args.e2e_order
                  else [[1], [4], [8], [16], [2]])
    E2E_MS = [M for g in E2E_GROUPS for M in g]
    assert sorted(E2E_MS) == sorted(MS)

    def e2e_body(i):
        # copies of group k+1 (H2D) and k-1 (D2H) overlap the compute of group k
        cur = torch.cuda.current_stream()
        h2d_s.wait_stream(cur)
        d2h_s.wait_stream(cur)
        ready = []
        for grp in E2E_GROUPS:
            with torch.cuda.stream(h2d_s):
                for M in grp:
                    a, b = gx[M]
                    dxb[a:b].copy_(hxb[a:b], non_blocking=True)
                ev = torch.cuda.Event()
                ev.record(h2d_s)
                ready.append(ev)
        for gi_, grp in enumerate(E2E_GROUPS):
            cur.wait_event(ready[gi_])
            cs = {M: (i * len(MS) + MS.index(M)) % COPIES for M in grp}
            if world == 1:
                if grouped:
                    keys = [(p, M) for M in grp for p in PROJS]
                    sfmp.gemm_grouped([models[cs[M]][p] for p, M in keys], [dx[k] for k in keys],
                                      outs=[dy[k] for k in keys], workspaces=[wsm[k] for k in keys])
                else:
                    for M in grp:
                        for p in PROJS:
                            models[cs[M]][p].gemm(dx[(p, M)], out=dy[(p, M)], path=sfmp.PATH_GEMV, workspace=ws[p])
            else:
                for M in grp:
                    for p in PROJS:
                        models[cs[M]][p].gemm(dx[(p, M)], out=ys[(p, M)], path=sfmp.PATH_GEMV, workspace=ws[p])
                        dist.all_gather_into_tensor(gath[(p, M)], ys[(p, M)])
                        models[cs[M]][p].unpermute_gathered(gath[(p, M)], M, out=dy[(p, M)])
            done = torch.cuda.Event()
            done.record(cur)
            with torch.cuda.stream(d2h_s):
                d2h_s.wait_event(done)
                for M in grp:
                    a, b = gy[M]
                    hyb[a:b].copy_(dyb[a:b], non_blocking=True)
        cur.wait_stream(d2h_s)
        cur.wait_stream(h2d_s)

    e2e_graphs = []
    if use_graph:
        with torch.cuda.stream(stream):
            e2e_body(0)
        torch.cuda.synchronize()
        for i in range(COPIES):
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=stream):
                e2e_body(i)
            e2e_graphs.append(g)

    def e2e_step(i):
        if e2e_graphs:
            e2e_graphs[i % COPIES].replay()
        else:
            with torch.cuda.stream(stream):
                e2e_body(i)
        torch.cuda.synchronize()

    for i in range(args.warmup):
        e2e_step(i)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    ee0 = torch.cuda.Event(enable_timing=True)
    ee1 = torch.cuda.Event(enable_timing=True)
    ee0.record()
    for i in range(args.steps):
        e2e_step(i)
    ee1.record()
    torch.cuda.synchronize()
    e2e_wall_ms = (time.perf_counter() - t0) * 1e3 / args.steps
    e2e_event_ms = ee0.elapsed_time(ee1) / args.steps
    e2e_ms = max(e2e_event_ms, e2e_wall_ms)
    if world > 1:
        tt = torch.tensor([e2e_ms], device=dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        e2e_ms = float(tt.item())

    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return 0

    hbm, tc, src = peaks()
    # roofline over the GEMV launches of one step (per-rank bytes when sharded)
    step_bytes = 0
    small_bytes = 0  # the M <= 8 class launch
    per_point = []
    for p in PROJS:
        rows_local = models[0][p].rows
        info_local = models[0][p].info
        for M in MS:
            b = algo_bytes(info_local, M, rows_local, SHAPES[p][1])
            step_bytes += b
            small_bytes += b if M <= 8 else 0
    n_launch = (n_class if across else len(MS)) if grouped else len(MS) * len(PROJS)  # GEMV launches per step
    t_us = t_ms * 1e3
    # achieved = algorithmic bytes of one GEMV launch / its share of the step
    # (each launch's time includes its x pre-pass: a lower bound on the kernel)
    achieved = step_bytes / (t_us * 1e-6) / 1e9
    traffic = None
    prof = os.path.join(ROOT, "profiles", "r01_ncu_gemv_grouped_8b_Mle8.json" if across else
                        "r01_ncu_gemv_grouped_8b_M1.json")
    if os.path.exists(prof):
        try:
            mb = json.load(open(prof))["metrics"]["dram__bytes_read.sum"].split()[0]
            wb = json.load(open(prof))["metrics"]["dram__bytes_write.sum"].split()[0]
            traffic = round((float(mb) + float(wb)) * 1e6)  # ncu --set full, one gemv_kernel launch
        except Exception:
            traffic = None
    out = {
        "metric": METRIC, "value": round(t_us, 2), "unit": "us", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(t_ms, 5),
        "higher_is_better": False, "scaling": "strong", "vs_baseline": None,
        "dtype": "f16", "data": "synthetic",
        "config": {"workload": WORKLOAD, "avg_code_bits": AVG_BITS, "M": MS,
                   "projections": PROJS, "kernel": "K1 decode GEMV (gemv_kernel) + x pre-pass (xprep_kernel)",
                   "launch_grouping": (("the whole step is one grouped call (sfmp_gemm_grouped_v, a token count "
                                        "per problem): one pre-pass + one GEMV launch for the 28 M<=8 problems, "
                                        "one for the 7 M=16 problems") if across else
                                       ("the 7 linears of one M share one pre-pass + one GEMV launch "
                                        "(sfmp_gemm_grouped)")) if grouped else "one launch per linear",
                   "ungrouped_step_us": round(ungrouped_ms * 1e3, 2) if ungrouped_ms else None,
                   "l2": f"inputs larger than L2: {COPIES} rotating device copies of the layer "
                         f"({sum(i['payload_bytes'] for i in infos.values()) * COPIES / 1e6:.0f} MB)",
                   "cuda_graph": use_graph,
                   "parallelism": "single GPU" if world == 1 else
                   f"N-sharded x{world} (snake block rows) + NCCL all-gather + unpermute",
                   "parity_max_rel_err_M16": parity},
        "roofline": {"bound": "hbm", "achieved": round(achieved, 1), "peak": hbm, "unit": "GB/s",
                     "frac": round(achieved / hbm, 4), "traffic": traffic,
                     "peak_source": f"MEASURED_PEAKS.json hbm_gbs ({src})",
                     "algorithmic_bytes_per_step": step_bytes,
                     "algorithmic_bytes_per_launch": step_bytes // n_launch,
                     "traffic_note": ("dram read+write of the step's M<=8 gemv_kernel launch (28 problems; "
                                      f"algorithmic {small_bytes} B), profiles/r01_ncu_gemv_grouped_8b_Mle8.json")
                     if across else ("dram read+write of one grouped M=1 gemv_kernel launch "
                                     "(profiles/r01_ncu_gemv_grouped_8b_M1.json)"),
                     "avg_launch_us": round(t_us / n_launch, 3), "launches_per_step": n_launch},
        "e2e": {"value": round(e2e_ms * 1e3, 2), "unit": "us", "h2d_bytes_per_step": h2d,
                "d2h_bytes_per_step": d2h, "api": ("pinned host x -> H2D per M group on a copy stream, sfmp_gemm_grouped per M, "
                       "D2H per group on a second copy stream (copies overlap compute); CUDA graph "
                       "per step, host synchronises on y every step"), "groups": E2E_GROUPS,
                "event_us": round(e2e_event_ms * 1e3, 2), "wall_us": round(e2e_wall_ms * 1e3, 2)},
        "gpu_launches": args.steps * launches_per_step,
        "clocks": clk,
    }
    if world == 1 and not args.no_prefill:
        out["prefill"] = prefill_leg(sfmp, port, models, dev, stream, args)
        out["dense_cublas_bf16_step"] = dense_leg(dev, stream, xs, args)
    if world == 1 and not args.no_cpu_baseline:
        out["cpu_baseline"] = cpu_baseline_sample(port, blobs)
    print(json.dumps(out), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
