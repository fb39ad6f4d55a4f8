"""Model upload time (sfmp_model_create): host bookkeeping + device ingest.
usage: load_time.py rows,cols,bits[,m_b] ...   (SFMP_LIB selects a build)"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))


def main():
    import torch
    import paper_2602_01027_b200 as sfmp
    from oracle.oracle import Port
    from synth import model_bytes, prebuild
    P = Port()
    pts = [a.split(",") for a in sys.argv[1:]]
    specs = [(int(p[0]), int(p[1]), float(p[2]), {"m_b": int(p[3])} if len(p) > 3 else {}) for p in pts]
    prebuild(specs)
    torch.zeros(1, device="cuda")
    for r, c, b, kw in specs:
        data = model_bytes(P, r, c, b, **kw)
        sfmp.DeviceModel(data)  # warm
        ts = []
        for _ in range(3):
            t0 = time.perf_counter()
            m = sfmp.DeviceModel(data)
            torch.cuda.synchronize()
            ts.append(time.perf_counter() - t0)
            del m
        print(f"{r}x{c} b{b}: {len(data) / 1e6:.1f} MB, create {min(ts) * 1e3:.1f} ms", flush=True)


if __name__ == "__main__":
    main()
