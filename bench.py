#!/usr/bin/env python
"""bench.py -- the SFMP mixed-precision GEMM hot path on B200 (driver contract).

Workload (BASELINE.json configs[1]): the seven Llama-3.1-8B linear shapes
(q,k,v,o,gate,up,down) at avg 3.25 code bits (block-wise 3/4-bit, m_b=512 --
k/v use m_b=128 so they split 8 ways -- n_b=128, rowcol reorder), decode with
M in {1,2,4,8,16} tokens.  One step = the 7 linears x 5 token counts = 35
GEMM calls, each through the decode GEMV kernel (K1).  Weights are rotated
over 6 device copies of the layer (576 MB >> 126 MB L2), so every call
streams its weights from HBM.

N>1 (torchrun): each linear is N-sharded by the snake block-row partition;
the whole step is ONE sfmp_gemm_sharded call: every rank runs its shards of
all 35 problems into one packed buffer, ONE NCCL all-gather (the library's
own communicator) moves them, ONE kernel un-permutes (strong scaling).

Sub-results ("extras"): configs[0] (4096x4096 @3.5 bits, M=1) with the
reference's CPU gemv beside it and the drop-in host-buffer call; the reorder
overhead (mode none) and an n_b=256 point; configs[3] (Llama-3.1-70B linears
@2.5 bits, decode step and prefill M=2048; sharded with kernel and collective
time split when N>1); configs[4] (8192x28672 at 2/3/4 bits x M).

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
    # the 7 linears as independent problems on 7 streams (fork / join inside one
    # graph): the small ones (k/v: 64 tiles) fill the SMs the large ones leave idle
    side = [torch.cuda.Stream(device=dev) for _ in PROJS]

    def layer(c):
        cur = torch.cuda.current_stream()
        for s_ in side:
            s_.wait_stream(cur)
        for s_, p in zip(side, sorted(PROJS, key=lambda q: -SHAPES[q][0] * SHAPES[q][1])):
            with torch.cuda.stream(s_):
                models[c][p].gemm(xs[p], out=ys[p], path=sfmp.PATH_GEMM, workspace=ws[p], stream=s_)
        for s_ in side:
            cur.wait_stream(s_)
    with torch.cuda.stream(stream):
        layer(0)
    torch.cuda.synchronize()
    gl = torch.cuda.CUDAGraph()
    with torch.cuda.graph(gl, stream=stream):
        for c in range(COPIES):
            layer(c)
    gl.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = max(2, args.steps // 10)
    with torch.cuda.stream(stream):
        e0.record(stream)
        for _ in range(reps):
            gl.replay()
        e1.record(stream)
    torch.cuda.synchronize()
    conc_us = e0.elapsed_time(e1) * 1e3 / (reps * COPIES)
    return {"metric": "prefill GEMM us per decoder layer (7 linears)", "M": M, "value": round(tot_us, 1),
            "concurrent_streams_us": round(conc_us, 1),
            "concurrent_streams_frac": round(flops / conc_us / 1e6 / tc, 4),
            "unit": "us", "kernel": "K2 tcgen05 GEMM (gemm_kernel) + xprep_gemm_kernel",
            "per_proj": per, "parity_max_rel_err_q_proj_sampled": round(par, 7),
            "roofline": {"bound": "tensor", "achieved": round(ach, 1), "peak": tc, "unit": "TFLOP/s",
                         "frac": round(ach / tc, 4), "peak_source": f"MEASURED_PEAKS.json bf16_tflops ({src})",
                         "note": "time includes the x gather/convert pre-pass"}}


# ---------------------------------------------------------------------------
# GPU helpers
# ---------------------------------------------------------------------------
def graph_us(body, stream, reps, per=1):
    """Capture body() in a CUDA graph, replay it `reps` times between CUDA
    events on `stream`; microseconds per body() / per."""
    import torch
    with torch.cuda.stream(stream):
        body()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=stream):
        body()
    g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(stream):
        e0.record(stream)
        for _ in range(reps):
            g.replay()
        e1.record(stream)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) * 1e3 / (reps * per)


def roof(bytes_, flops, us, hbm, tc):
    """t* = max(B/BW, FLOP/TC); fraction = t*/t."""
    t_h, t_t = bytes_ / (hbm * 1e3), flops / (tc * 1e6)
    return {"us": round(us, 2), "GBps": round(bytes_ / us / 1e3, 1), "TFLOPs": round(flops / us / 1e6, 1),
            "bound": "hbm" if t_h >= t_t else "tensor", "frac": round(max(t_h, t_t) / us, 4)}


def ws_for(sfmp, m, M):
    import torch
    n = m.workspace_bytes(16 if M <= 16 else M, sfmp.PATH_GEMV if M <= 16 else sfmp.PATH_AUTO)
    return torch.zeros(max(n, 128), dtype=torch.uint8, device=f"cuda:{m.device}")


# ---------------------------------------------------------------------------
# sub-results (BASELINE.json configs[0], [3], [4]; SURVEY §8(d) extra points)
# ---------------------------------------------------------------------------
def single_linear_points(sfmp, port, dev, stream, hbm, tc, args):
    """configs[0] (4096x4096, 3.5 bits, rowcol, M=1) with the reference CPU gemv
    beside it, the drop-in host-buffer call, the reorder overhead (mode none,
    PAPER.md:487) and an n_b=256 point."""
    import torch
    from synth import model_bytes
    out = {}
    copies = 32  # 32 x 7.9 MB >> L2
    x1 = torch.from_numpy(port.gen_activation(1, 4096, 3001)).to(dev).to(torch.bfloat16)
    for key, kw in (("config0", dict(mode=3)), ("mode_none", dict(mode=0)), ("n_b_256", dict(mode=3, n_b=256))):
        data = model_bytes(port, 4096, 4096, 3.5, **kw)
        ms = [sfmp.DeviceModel(data, device=dev.index) for _ in range(copies)]
        ws = ws_for(sfmp, ms[0], 16)
        y = torch.empty(1, 4096, device=dev)
        us = graph_us(lambda: [m.gemm(x1, out=y, workspace=ws, stream=stream) for m in ms], stream, 20, copies)
        b = algo_bytes(ms[0].info, 1, 4096, 4096)
        out[key] = {"what": f"4096x4096 @3.5 bits {kw}, M=1, bf16 x", **roof(b, 2.0 * 4096 * 4096, us, hbm, tc)}
        if key == "n_b_256":
            xp = torch.from_numpy(port.gen_activation(2048, 4096, 3002)).to(dev).to(torch.bfloat16)
            yp = torch.empty(2048, 4096, device=dev)
            wsp = ws_for(sfmp, ms[0], 2048)
            usp = graph_us(lambda: [m.gemm(xp, out=yp, workspace=wsp, stream=stream) for m in ms[:4]], stream, 5, 4)
            out[key]["prefill_M2048"] = roof(algo_bytes(ms[0].info, 2048, 4096, 4096), 2.0 * 2048 * 4096 * 4096,
                                             usp, hbm, tc)
        if key == "config0":
            # the drop-in call a reference user makes: host f32 in/out (sfmp_gemm_host,
            # = sfmp::cuda::gemv in include/sfmp/cuda.hpp), synchronous per call
            xh = port.gen_activation(1, 4096, 3001)
            walls, devs = [], []
            for i in range(60):
                _, st = ms[i % copies].gemm_host(xh, stats=True)
                if i >= 10:
                    walls.append(st["wall_us"])
                    devs.append(st["device_us"])
            out["dropin_gemv_host"] = {
                "what": "configs[0] through sfmp_gemm_host (host f32 x -> host y, H2D + kernels + D2H + sync per "
                        "call), the call behind sfmp::cuda::gemv", "wall_us_median": round(statistics.median(walls), 2),
                "device_us_median": round(statistics.median(devs), 2)}
            try:
                kind, hs = cpu_handles(port, {"c0": data})
                if kind == "reference":
                    r = hs["c0"].bench_gemv(xh[0], 5)
                    out["config0"]["cpu_reference_gemv_us"] = round(r["median_us"], 1)
                    out["config0"]["cpu_kind"] = "reference bench_gemv (lutgemm.cpp:137), 1 thread"
            except Exception as e:  # the CPU leg is informative only
                out["config0"]["cpu_reference_error"] = str(e)[:100]
        del ms
    out["reorder_overhead_pct"] = round(100.0 * (out["config0"]["us"] / out["mode_none"]["us"] - 1.0), 2)
    # the paper's kernel comparison: ours vs the
    # paper-faithful LUT GEMV on the GPU (K6) vs dense bf16 cuBLAS, M=1
    cmp = {}
    for name, (r, c, b) in (("4096x4096_b3.5", (4096, 4096, 3.5)), ("8192x28672_b3.0", (8192, 28672, 3.0))):
        data = model_bytes(port, r, c, b)
        ncp = max(2, int(400e6 // (r * c * b / 8)) + 1)
        ms = [sfmp.DeviceModel(data, device=dev.index, flags=sfmp.MODEL_LUT_LAYOUT) for _ in range(min(ncp, 8))]
        x32 = torch.from_numpy(port.gen_activation(1, c, 3100)).to(dev)
        xb = x32.to(torch.bfloat16)
        y = torch.empty(1, r, device=dev)
        ws = ws_for(sfmp, ms[0], 16)
        ours = graph_us(lambda: [m.gemm(xb, out=y, workspace=ws, stream=stream) for m in ms], stream, 10, len(ms))
        lut = graph_us(lambda: [m.gemm(x32, out=y, path=sfmp.PATH_LUT, stream=stream) for m in ms], stream, 3,
                       len(ms))
        Wd = [torch.randn(r, c, device=dev, dtype=torch.bfloat16) for _ in range(max(2, int(400e6 // (2 * r * c)) + 1))]
        yd = torch.empty(1, r, device=dev, dtype=torch.bfloat16)
        dense = graph_us(lambda: [torch.matmul(xb, w.t(), out=yd) for w in Wd], stream, 10, len(Wd))
        byts = algo_bytes(ms[0].info, 1, r, c)
        cmp[name] = {"ours_us": round(ours, 2), "lut_gpu_us": round(lut, 2), "dense_bf16_cublas_us": round(dense, 2),
                     "ours_frac_hbm": round(byts / ours / 1e3 / hbm, 4)}
        del ms, Wd
        torch.cuda.empty_cache()
    out["kernel_comparison_M1"] = cmp
    torch.cuda.empty_cache()
    return out


def sweep_points(sfmp, port, dev, stream, hbm, tc, args):
    """configs[4]: 8192x28672 at 2.0/3.0/4.0 bits x M, roofline fraction per point."""
    import torch
    from synth import model_bytes, prebuild
    bits_l, Ms = (2.0, 3.0, 4.0), (1, 16, 64, 256, 2048)
    prebuild([(8192, 28672, b, {}) for b in bits_l])
    xs = {M: torch.from_numpy(port.gen_activation(M, 28672, 5000 + M)).to(dev).to(torch.bfloat16) for M in Ms}
    out = {}
    for b in bits_l:
        data = model_bytes(port, 8192, 28672, b)
        ms = [sfmp.DeviceModel(data, device=dev.index) for _ in range(2)]
        for M in Ms:
            y = torch.empty(M, 8192, device=dev)
            ws = ws_for(sfmp, ms[0], M)
            us = graph_us(lambda: [m.gemm(xs[M], out=y, workspace=ws, stream=stream) for m in ms], stream,
                          10 if M <= 64 else 3, 2)
            out[f"b{b}_M{M}"] = roof(algo_bytes(ms[0].info, M, 8192, 28672), 2.0 * M * 8192 * 28672, us, hbm, tc)
        del ms
        torch.cuda.empty_cache()
    return out


def llama70b_points(sfmp, port, dev, stream, hbm, tc, world, rank, comm, args, sharded=None):
    """configs[3]: the seven Llama-3.1-70B linears @2.5 bits (k/v m_b=128 so they
    split 8 ways), decode step M in {1,2,4,8,16} as one call, prefill M=2048;
    N>1: snake-sharded, ONE NCCL all-gather per call -- kernel and collective
    time reported separately."""
    import torch
    from synth import LLAMA_70B, model_bytes, prebuild
    sharded = sharded if sharded is None else sharded
    specs = [(r, c, 2.5, {"m_b": 128 if p in ("k_proj", "v_proj") else 512}) for p, (r, c) in LLAMA_70B.items()]
    prebuild(specs)
    blobs = {p: model_bytes(port, r, c, 2.5, m_b=128 if p in ("k_proj", "v_proj") else 512)
             for p, (r, c) in LLAMA_70B.items()}
    copies = 2
    mk = (lambda b: sfmp.DeviceModel(b, device=dev.index)) if not sharded else \
        (lambda b: sfmp.DeviceModel(b, device=dev.index, shard=rank, num_shards=world))
    models = [{p: mk(blobs[p]) for p in PROJS} for _ in range(copies)]
    out = {"workload": "llama3.1-70b decoder-layer linears @2.5 code bits (3/2 mix), rowcol; decode M in "
                       "{1,2,4,8,16} (35 problems, one call) and prefill M=2048 (7 problems)",
           "parallelism": "single GPU" if not sharded else f"N-sharded x{world}, one NCCL all-gather per call"}
    xs = {(p, M): torch.from_numpy(port.gen_activation(M, LLAMA_70B[p][1], 6000 + M)).to(dev).to(torch.bfloat16)
          for p in PROJS for M in MS}
    keys = [(p, M) for M in MS for p in PROJS]
    ys = {k: torch.empty(k[1], LLAMA_70B[k[0]][0], device=dev) for k in keys}
    wsm = {k: ws_for(sfmp, models[0][k[0]], k[1]) for k in keys}

    def run(i, kk, local_only=False, bufs=None):
        ms = [models[(i + j) % copies][p] for j, (p, M) in enumerate(kk)]
        if not sharded:
            sfmp.gemm_grouped(ms, [xs[k] for k in kk], outs=[ys[k] for k in kk], workspaces=[wsm[k] for k in kk],
                              stream=stream)
        elif local_only:
            sfmp.gemm_sharded_local(ms, [xs[k] for k in kk], bufs, [wsm[k] for k in kk], stream=stream)
        else:
            sfmp.gemm_sharded(ms, [xs[k] for k in kk], [ys[k] for k in kk], [wsm[k] for k in kk], bufs, comm,
                              stream=stream)

    buf = None
    if sharded:
        buf = torch.zeros(sfmp.sharded_gather_bytes([models[0][p] for p, M in keys], [M for p, M in keys]) // 4,
                          device=dev)
    us = graph_us(lambda: [run(i, keys, bufs=buf) for i in range(copies)], stream, 10, copies)
    byts = sum(algo_bytes(models[0][p].info, M, models[0][p].rows, LLAMA_70B[p][1]) for p, M in keys)
    out["decode_step"] = {"M": MS, **roof(byts, sum(2.0 * M * models[0][p].rows * LLAMA_70B[p][1] for p, M in keys),
                                          us, hbm, tc)}
    if sharded:
        kus = graph_us(lambda: [run(i, keys, local_only=True, bufs=buf) for i in range(copies)], stream, 10, copies)
        out["decode_step"].update({"kernel_us": round(kus, 2), "collective_and_unpermute_us": round(us - kus, 2),
                                   "bytes_gathered_per_rank": buf.numel() * 4 // (1 + world) * world})
    # prefill
    Mp = 2048
    xp = {p: torch.from_numpy(port.gen_activation(Mp, LLAMA_70B[p][1], 7000)).to(dev).to(torch.bfloat16) for p in PROJS}
    yp = {p: torch.empty(Mp, LLAMA_70B[p][0], device=dev) for p in PROJS}
    wsp = {p: ws_for(sfmp, models[0][p], Mp) for p in PROJS}
    if not sharded:
        per = {}
        for p in PROJS:
            t = graph_us(lambda: [models[c][p].gemm(xp[p], out=yp[p], workspace=wsp[p], stream=stream)
                                  for c in range(copies)], stream, 3, copies)
            r, c_ = LLAMA_70B[p]
            per[p] = roof(algo_bytes(models[0][p].info, Mp, r, c_), 2.0 * Mp * r * c_, t, hbm, tc)
        tot = sum(v["us"] for v in per.values())
        fl = sum(2.0 * Mp * r * c for r, c in LLAMA_70B.values())
        out["prefill"] = {"M": Mp, "us": round(tot, 1), "TFLOPs": round(fl / tot / 1e6, 1),
                          "frac": round(fl / tot / 1e6 / tc, 4), "per_proj": per}
    else:
        pk = [(p, Mp) for p in PROJS]
        pbuf = torch.zeros(sfmp.sharded_gather_bytes([models[0][p] for p in PROJS], [Mp] * 7) // 4, device=dev)

        def prun(local_only):
            ms = [models[0][p] for p in PROJS]
            if local_only:
                sfmp.gemm_sharded_local(ms, [xp[p] for p in PROJS], pbuf, [wsp[p] for p in PROJS], stream=stream)
            else:
                sfmp.gemm_sharded(ms, [xp[p] for p in PROJS], [yp[p] for p in PROJS], [wsp[p] for p in PROJS], pbuf,
                                  comm, stream=stream)
        t = graph_us(lambda: prun(False), stream, 3)
        tk = graph_us(lambda: prun(True), stream, 3)
        fl = sum(2.0 * Mp * models[0][p].rows * LLAMA_70B[p][1] for p in PROJS)
        out["prefill"] = {"M": Mp, "us": round(t, 1), "kernel_us": round(tk, 1),
                          "collective_and_unpermute_us": round(t - tk, 1),
                          "per_rank_TFLOPs": round(fl / tk / 1e6, 1), "frac_kernel": round(fl / tk / 1e6 / tc, 4),
                          "problems": len(pk)}
    del models
    torch.cuda.empty_cache()
    return out


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
    ap.add_argument("--no-extras", action="store_true", help="skip configs[0]/[3]/[4] sub-results")
    ap.add_argument("--no-group", action="store_true", help="one launch per linear instead of per decoder layer")
    ap.add_argument("--prefill-M", type=int, default=2048)
    ap.add_argument("--e2e-order", default="", help="groups of token counts for the e2e step, e.g. '1/4/8/16/2'")
    ap.add_argument("--force-sharded", action="store_true",
                    help="run the sharded path (shard models, sfmp_gemm_sharded, library NCCL communicator) even "
                         "at N=1 (1-way shards): exercises the multi-GPU code path on one GPU")
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
    dev = torch.device(f"cuda:{local}")
    comm = None
    sharded = world > 1 or args.force_sharded
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
        # the library's own NCCL communicator (sfmp_gemm_sharded): id over torch.distributed
        uid = [sfmp.NcclComm.unique_id() if rank == 0 else None]
        dist.broadcast_object_list(uid, src=0)
        comm = sfmp.NcclComm(world, rank, local, uid[0])
    elif sharded:
        comm = sfmp.NcclComm(1, 0, local, sfmp.NcclComm.unique_id())
    port = Port()
    blobs = {p: build_bytes(port, p) for p in PROJS}
    # COPIES device copies of the layer (this rank's shard of it when world > 1)
    models = [{p: (sfmp.DeviceModel(blobs[p], device=local) if not sharded else
                   sfmp.DeviceModel(blobs[p], device=local, shard=rank, num_shards=world))
               for p in PROJS} for _ in range(COPIES)]
    infos = {p: sfmp.parse_header(blobs[p]) for p in PROJS}
    xs = {(p, M): torch.from_numpy(port.gen_activation(M, SHAPES[p][1], 3000 + M)).to(dev)
          .to(torch.bfloat16) for p in PROJS for M in MS}
    ys = {(p, M): torch.empty(M, SHAPES[p][0], device=dev) for p in PROJS for M in MS}
    # a workspace per (linear, M): problems of one launch must not share one
    wsm = {(p, M): ws_for(sfmp, models[0][p], 16) for p in PROJS for M in MS}
    keys_all = [(p, M) for M in MS for p in PROJS]
    gbuf = None
    if sharded:
        gbuf = torch.zeros(sfmp.sharded_gather_bytes([models[0][p] for p, M in keys_all],
                                                     [M for p, M in keys_all]) // 4, device=dev)
    grouped = not args.no_group

    def call(i, kk, local_only=False):
        """One API call over the problems kk = [(proj, M)], weight copy rotating with i."""
        ms = [models[(i * len(MS) + MS.index(M)) % COPIES][p] for p, M in kk]
        if not sharded:
            if grouped:
                sfmp.gemm_grouped(ms, [xs[k] for k in kk], outs=[ys[k] for k in kk], workspaces=[wsm[k] for k in kk])
            else:
                for m, k in zip(ms, kk):
                    m.gemm(xs[k], out=ys[k], path=sfmp.PATH_GEMV, workspace=wsm[k])
        elif local_only:
            sfmp.gemm_sharded_local(ms, [xs[k] for k in kk], gbuf, [wsm[k] for k in kk])
        else:
            sfmp.gemm_sharded(ms, [xs[k] for k in kk], [ys[k] for k in kk], [wsm[k] for k in kk], gbuf, comm)

    def step(i):
        # the whole step (7 linears x 5 token counts) in ONE call: one pre-pass + one
        # GEMV launch per n-tile class (M <= 8: 28 problems, M = 16: 7); N>1 adds ONE
        # all-gather of every problem's shard rows and ONE un-permute launch
        call(i, keys_all)

    # correctness spot check against the oracle (rank 0, cheap shapes)
    n0 = sfmp.launch_count()
    step(0)
    launches_per_step = sfmp.launch_count() - n0
    torch.cuda.synchronize()
    parity = {}
    if rank == 0:
        from synth import errors
        for p in ("q_proj", "k_proj"):
            w = port.load(blobs[p]).dequantize()
            ref = port.matmul(xs[(p, 16)].float().cpu().numpy(), w, threads=8)
            parity[p] = round(errors(ys[(p, 16)].cpu().numpy(), ref)[0], 9)

    use_graph = not args.no_graph
    stream = torch.cuda.Stream(device=dev)
    graphs, block = [], None
    if use_graph:
        # one graph per rotation phase so each replay touches the next weight copies,
        # and one graph of COPIES consecutive steps (a serving loop runs steps back to
        # back; a graph boundary per step adds launch latency between steps)
        with torch.cuda.stream(stream):
            for i in range(COPIES):
                step(i)
        torch.cuda.synchronize()
        for i in range(COPIES):
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=stream):
                step(i)
            graphs.append(g)
        block = torch.cuda.CUDAGraph()
        with torch.cuda.graph(block, stream=stream):
            for i in range(COPIES):
                step(i)

    def run_step(i):
        if use_graph:
            graphs[i % COPIES].replay()
        else:
            step(i)

    def run_steps(n):
        """Exactly n steps (phases 0, 1, ...): whole COPIES-step blocks, then single steps."""
        i = 0
        if use_graph:
            while n - i >= COPIES:
                block.replay()
                i += COPIES
        while i < n:
            run_step(i)
            i += 1

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
        run_steps(args.steps)
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

    hbm, tc, src = peaks()
    # ---- per-launch roofline: each n-tile class alone (its pre-pass + GEMV + fix-up),
    # graph replay over the rotating copies, CUDA events on the launching stream ----
    per_launch = {}
    if not sharded and grouped:
        for name, kk in (("M<=8", [k for k in keys_all if k[1] <= 8]), ("M=16", [k for k in keys_all if k[1] > 8])):
            with torch.cuda.stream(stream):
                us = graph_us(lambda: [call(i, kk) for i in range(COPIES)], stream, max(3, args.steps // 5), COPIES)
            b = sum(algo_bytes(models[0][p].info, M, models[0][p].rows, SHAPES[p][1]) for p, M in kk)
            per_launch[name] = {"problems": len(kk), "bytes": b, **roof(b, sum(2.0 * M * SHAPES[p][0] * SHAPES[p][1]
                                                                               for p, M in kk), us, hbm, tc)}
    # ---- §8(f)1: RMSNorm fused into the activation pre-pass vs a separate norm ----
    fused_norm = None
    if not sharded and grouped and not args.no_extras:
        import torch.nn.functional as F
        normed = ("q_proj", "k_proj", "v_proj", "gate_proj", "up_proj")  # o/down take other inputs
        gam = {p: (0.9 + 0.2 * torch.rand(SHAPES[p][1], device=dev)).to(torch.bfloat16) for p in PROJS}
        norms = [(gam[p], 1e-5) if p in normed else None for p, M in keys_all]

        def fused(i):
            ms = [models[(i * len(MS) + MS.index(M)) % COPIES][p] for p, M in keys_all]
            sfmp.gemm_grouped(ms, [xs[k] for k in keys_all], outs=[ys[k] for k in keys_all],
                              workspaces=[wsm[k] for k in keys_all], norms=norms)

        xn = {}

        def unfused(i):
            # the separate norm kernels a model would run first: one per shared input
            for M in MS:
                for p in ("q_proj", "gate_proj"):
                    xn[(p, M)] = F.rms_norm(xs[(p, M)], (SHAPES[p][1],), gam[p], 1e-5)
            ms = [models[(i * len(MS) + MS.index(M)) % COPIES][p] for p, M in keys_all]
            src = [xn[("q_proj" if p in ("q_proj", "k_proj", "v_proj") else "gate_proj", M)] if p in normed
                   else xs[(p, M)] for p, M in keys_all]
            sfmp.gemm_grouped(ms, src, outs=[ys[k] for k in keys_all], workspaces=[wsm[k] for k in keys_all])
        with torch.cuda.stream(stream):
            fu = graph_us(lambda: [fused(i) for i in range(COPIES)], stream, max(3, args.steps // 5), COPIES)
            un = graph_us(lambda: [unfused(i) for i in range(COPIES)], stream, max(3, args.steps // 5), COPIES)
        fused_norm = {"what": "8B decode step with the pre-attention / pre-MLP RMSNorm: fused into the activation "
                              "pre-pass (sfmp_gemm_grouped_v_norm) vs torch rms_norm kernels + the grouped call",
                      "fused_us": round(fu, 2), "separate_us": round(un, 2)}

    kernel_us = None
    if sharded:
        with torch.cuda.stream(stream):
            kernel_us = graph_us(lambda: [call(i, keys_all, local_only=True) for i in range(COPIES)], stream,
                                 max(3, args.steps // 5), COPIES)

    # ---- e2e: host buffers in, host buffers out, through the public API ----
    # One pinned host buffer holds every x of the step (f32, as the reference's
    # Vector) and one every y; per group of token counts: H2D on a copy stream,
    # the API call, D2H on a second copy stream (copies overlap the other
    # groups' compute); CUDA graph per step; the host waits for y every step.
    keys = keys_all
    xoff, yoff, xo, yo = {}, {}, 0, 0
    for k in keys:
        xoff[k], yoff[k] = xo, yo
        xo += k[1] * SHAPES[k[0]][1]
        yo += k[1] * SHAPES[k[0]][0]
    # x travels as bf16 (the activations of this workload are bf16 values; the
    # API takes bf16 directly), y comes back as the API's f32
    hxb = torch.empty(xo, dtype=torch.bfloat16).pin_memory()
    hyb = torch.empty(yo, dtype=torch.float32).pin_memory()
    for (p, M) in keys:
        hxb[xoff[(p, M)]:xoff[(p, M)] + M * SHAPES[p][1]] = torch.from_numpy(
            port.gen_activation(M, SHAPES[p][1], 3000 + M)).reshape(-1)
    dxb = torch.empty(xo, dtype=torch.bfloat16, device=dev)
    dyb = torch.empty(yo, dtype=torch.float32, device=dev)
    dx = {k: dxb[xoff[k]:xoff[k] + k[1] * SHAPES[k[0]][1]].view(k[1], SHAPES[k[0]][1]) for k in keys}
    dy = {k: dyb[yoff[k]:yoff[k] + k[1] * SHAPES[k[0]][0]].view(k[1], SHAPES[k[0]][0]) for k in keys}
    h2d, d2h = xo * 2, yo * 4

    # a group element is "M" (all seven linears at M) or "M:i-j" (PROJS[i..j] at M,
    # contiguous in the x and y buffers)
    def elem(tok):
        M, _, rng = tok.partition(":")
        M = int(M)
        a, _, b = rng.partition("-")
        i, j = (int(a), int(b or a)) if rng else (0, len(PROJS) - 1)
        return M, PROJS[i:j + 1]

    def span(off, M, ps, dim):
        return off[(ps[0], M)], off[(ps[-1], M)] + M * SHAPES[ps[-1]][dim]
    h2d_s, d2h_s = torch.cuda.Stream(device=dev), torch.cuda.Stream(device=dev)
    # group order: a small group first (short exposed H2D), then the largest so its
    # 2.75 MB D2H hides under the later groups' compute, M=4 and 8 in one call (one
    # launch's fixed costs fewer), the smallest last (short exposed D2H); measured
    # (tools/gpu_e2e_orders.sh, profiles/r02_e2e_orders.txt): 2/16/4,8/1 221-223 us,
    # 2/16/8/4/1 235-250 us, 1/4/8/16/2 259 us, one group 334 us
    E2E_ORDER = args.e2e_order or "2/16/4,8/1"
    E2E_GROUPS = [[elem(v) for v in g.split(",")] for g in E2E_ORDER.split("/")]
    assert sorted((p, M) for g in E2E_GROUPS for M, ps in g for p in ps) == sorted(keys_all)
    ebufs = {}
    if sharded:
        for gi_, grp in enumerate(E2E_GROUPS):
            kk = [(p, M) for M, ps in grp for p in ps]
            ebufs[gi_] = torch.zeros(sfmp.sharded_gather_bytes([models[0][p] for p, M in kk], [M for p, M in kk]) // 4,
                                     device=dev)

    def e2e_body(i):
        cur = torch.cuda.current_stream()
        h2d_s.wait_stream(cur)
        d2h_s.wait_stream(cur)
        ready = []
        for grp in E2E_GROUPS:
            with torch.cuda.stream(h2d_s):
                for M, ps in grp:
                    a, b = span(xoff, M, ps, 1)
                    dxb[a:b].copy_(hxb[a:b], non_blocking=True)
                ev = torch.cuda.Event()
                ev.record(h2d_s)
                ready.append(ev)
        for gi_, grp in enumerate(E2E_GROUPS):
            cur.wait_event(ready[gi_])
            kk = [(p, M) for M, ps in grp for p in ps]
            ms = [models[(i * len(MS) + MS.index(M)) % COPIES][p] for p, M in kk]
            if not sharded:
                sfmp.gemm_grouped(ms, [dx[k] for k in kk], outs=[dy[k] for k in kk], workspaces=[wsm[k] for k in kk])
            else:
                sfmp.gemm_sharded(ms, [dx[k] for k in kk], [dy[k] for k in kk], [wsm[k] for k in kk], ebufs[gi_], comm)
            done = torch.cuda.Event()
            done.record(cur)
            with torch.cuda.stream(d2h_s):
                d2h_s.wait_event(done)
                for M, ps in grp:
                    a, b = span(yoff, M, ps, 0)
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

    # ---- sub-results (every rank takes part in the sharded 70B one) ----
    extras = {}
    if not args.no_extras:
        with torch.cuda.stream(stream):
            extras["llama70b"] = llama70b_points(sfmp, port, dev, stream, hbm, tc, world, rank, comm, args, sharded)
            if not sharded:
                extras.update(single_linear_points(sfmp, port, dev, stream, hbm, tc, args))
                extras["sweep_8192x28672"] = sweep_points(sfmp, port, dev, stream, hbm, tc, args)

    if rank != 0:
        if comm is not None:
            comm.close()
        if world > 1:
            dist.destroy_process_group()
        return 0

    # roofline over the step (per-rank bytes when sharded)
    step_bytes = sum(algo_bytes(models[0][p].info, M, models[0][p].rows, SHAPES[p][1]) for p, M in keys_all)
    t_us = t_ms * 1e3
    step_ach = step_bytes / (t_us * 1e-6) / 1e9
    traffic, traffic_src = None, None
    for prof in ("r02_ncu_gemv_step_8b.json", "r02_ncu_gemv_grouped_8b_Mle8.json"):
        path = os.path.join(ROOT, "profiles", prof)
        if os.path.exists(path):
            try:
                mt = json.load(open(path))["metrics"]
                traffic = round((float(mt["dram__bytes_read.sum"].split()[0]) +
                                 float(mt["dram__bytes_write.sum"].split()[0])) * 1e6)
                traffic_src = prof
                break
            except Exception:
                traffic = None
    roofline = {"bound": "hbm", "achieved": round(step_ach, 1), "peak": hbm, "unit": "GB/s",
                "frac": round(step_ach / hbm, 4), "traffic": traffic,
                "kernel": (f"the step's single grouped launch (35 problems: x pre-pass + gemv_kernel + fix-up, "
                           f"{launches_per_step} kernels), {round(t_us, 2)} us for {step_bytes} algorithmic bytes")
                if not sharded else "whole step (per-rank bytes / step time)",
                "traffic_note": f"ncu dram read+write of that gemv_kernel launch, profiles/{traffic_src}" if traffic
                else None,
                "algorithmic_bytes_per_step": step_bytes, "peak_source": f"MEASURED_PEAKS.json hbm_gbs ({src})"}
    if per_launch:
        roofline["split_by_token_class"] = per_launch  # the same problems as two launches, for reference
    if kernel_us:
        roofline.update({"kernel_us": round(kernel_us, 2), "collective_and_unpermute_us": round(t_us - kernel_us, 2),
                         "kernel_frac": round(step_bytes / (kernel_us * 1e-6) / 1e9 / hbm, 4)})
    out = {
        "metric": METRIC, "value": round(t_us, 2), "unit": "us", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(t_ms, 5),
        "higher_is_better": False, "scaling": "strong", "vs_baseline": None,
        "dtype": "f16", "data": "synthetic",
        "config": {"workload": WORKLOAD, "avg_code_bits": AVG_BITS, "M": MS, "projections": PROJS,
                   "kernel": "K1 decode GEMV (gemv_kernel) + x pre-pass (xprep_gather_kernel) + fix-up (gemv_fixup_kernel, split linears only)",
                   "launch_grouping": ("the whole step is one call (sfmp_gemm_grouped_v): ONE pre-pass + ONE GEMV "
                                       "launch (token counts 1..16 mixed, each linear at its own n-tile count) + "
                                       "ONE fix-up for all 35 problems" if grouped else "one launch per linear") +
                                      ("; sfmp_gemm_sharded: + ONE NCCL all-gather of all 35 problems' shard rows "
                                       "and ONE un-permute launch" if sharded else ""),
                   "l2": f"inputs larger than L2: {COPIES} rotating device copies of the layer "
                         f"({sum(i['payload_bytes'] for i in infos.values()) * COPIES / 1e6:.0f} MB)",
                   "cuda_graph": (f"{COPIES} consecutive steps per graph replay (+ single-step graphs for the "
                                  f"remainder of --steps)") if use_graph else False,
                   "parallelism": "single GPU" if not sharded else
                   f"N-sharded x{world} (snake block rows), one NCCL all-gather per step (library communicator)",
                   "parity_max_rel_err_M16": parity},
        "roofline": roofline,
        "e2e": {"value": round(e2e_ms * 1e3, 2), "unit": "us", "h2d_bytes_per_step": h2d,
                "d2h_bytes_per_step": d2h,
                "api": ("pinned host bf16 x -> H2D per M group on a copy stream, one sfmp_gemm_grouped_v "
                        + ("" if not sharded else "/ sfmp_gemm_sharded ") +
                        "call per group, D2H per group on a second copy stream (copies overlap compute); CUDA "
                        "graph per step, host synchronises on y every step"), "groups": E2E_ORDER,
                "event_us": round(e2e_event_ms * 1e3, 2), "wall_us": round(e2e_wall_ms * 1e3, 2)},
        "gpu_launches": args.steps * launches_per_step,
        "gpu_launches_note": f"{launches_per_step} kernels per step, counted by sfmp_launch_count() "
                             f"when the step was enqueued",
        "clocks": clk,
    }
    if fused_norm:
        extras["fused_rmsnorm"] = fused_norm
    if extras:
        out["extras"] = extras
    if not sharded and not args.no_prefill:
        out["prefill"] = prefill_leg(sfmp, port, models, dev, stream, args)
        out["dense_cublas_bf16_step"] = dense_leg(dev, stream, xs, args)
    if world == 1 and not args.no_cpu_baseline:
        out["cpu_baseline"] = cpu_baseline_sample(port, blobs)
    print(json.dumps(out), flush=True)
    if comm is not None:
        comm.close()
    if world > 1:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
