"""Summarise ncu reports into profiles/*.json (key SOL metrics, instruction mix,
stall reasons, dram bytes) and the bench launch list into per-kernel shares."""
import collections
import csv
import io
import json
import subprocess
import sys


def page(rep, name, extra=()):
    out = subprocess.run(["ncu", "-i", rep, "--page", name, "--csv", *extra], capture_output=True, text=True).stdout
    return list(csv.reader(io.StringIO(out)))


def summarise(rep):
    d = {}
    for r in page(rep, "details"):
        if len(r) > 14 and r[0] != "ID":
            d[f"{r[11]} | {r[12]}"] = f"{r[14]} {r[13]}".strip()
    keep = ["Duration", "DRAM Throughput", "Memory Throughput", "Compute (SM) Throughput", "Executed Ipc Active",
            "Issue Slots Busy", "Achieved Occupancy", "Registers Per Thread", "Grid Size", "Block Size",
            "Dynamic Shared Memory Per Block", "L2 Hit Rate", "SM Frequency", "Eligible Warps Per Scheduler"]
    sol = {k.split(" | ")[1]: v for k, v in d.items() if k.split(" | ")[1] in keep}
    raw = page(rep, "raw")
    h, v = raw[0], raw[2]
    rd = dict(zip(h, v))
    pick = {}
    for k in ("dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__time_duration.sum",
              "sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
              "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
              "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
              "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
              "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
              "sm__pipe_shared_cycles_active.avg.pct_of_peak_sustained_active",
              "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
              "l1tex__data_pipe_tc_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
              "smsp__inst_executed.sum", "sm__throughput.avg.pct_of_peak_sustained_elapsed"):
        if k in rd:
            pick[k] = rd[k] + (" " + raw[1][h.index(k)] if len(raw) > 1 else "")
    src = page(rep, "source", ["--print-source=sass"])
    sh, data = src[1], src[2:]
    ei = sh.index("Instructions Executed")
    names = [n for n in sh if n.startswith("stall_") and "Not Issued" not in n]
    ops, stalls, tot = collections.Counter(), collections.Counter(), 0
    for r in data:
        try:
            n = int(r[ei])
        except ValueError:
            continue
        tot += n
        t = r[1].split()
        op = (t[1] if t[0].startswith("@") else t[0]).split(".")[0]
        ops[op] += n
        for nm in names:
            try:
                stalls[nm] += int(r[sh.index(nm)])
            except ValueError:
                pass
    return {"report": rep.split("/")[-1], "speed_of_light": sol, "metrics": pick, "warp_instructions": tot,
            "instruction_mix_pct": {k: round(100.0 * c / tot, 1) for k, c in ops.most_common(14)},
            "stall_samples": dict(stalls.most_common(10))}


def launches(path):
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    h = rows[0]
    ki, mi, vi = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value")
    per = collections.defaultdict(lambda: collections.defaultdict(list))
    for r in rows[1:]:
        k = r[ki].split("(")[0].replace("void ", "")
        per[k][r[mi]].append(float(r[vi].replace(",", "")))
    tot = sum(sum(m["gpu__time_duration.sum"]) for m in per.values())
    out = {}
    for k, m in per.items():
        t = m["gpu__time_duration.sum"]
        out[k] = {"launches": len(t), "mean_ns": round(sum(t) / len(t), 1), "share_of_time": round(sum(t) / tot, 4)}
        for key in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
            if key in m:
                out[k]["mean_" + key] = round(sum(m[key]) / len(m[key]), 1)
    return out


if __name__ == "__main__":
    kind, src, dst = sys.argv[1:4]
    res = summarise(src) if kind == "rep" else launches(src)
    json.dump(res, open(dst, "w"), indent=1)
    print(json.dumps(res, indent=1)[:3000])
