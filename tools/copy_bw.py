import torch
for mb in (0.25, 1, 2.5, 5):
    n = int(mb * 2**20 / 4)
    h = torch.empty(n).pin_memory(); d = torch.empty(n, device="cuda")
    for name, f in (("H2D", lambda: d.copy_(h, non_blocking=True)), ("D2H", lambda: h.copy_(d, non_blocking=True))):
        f(); torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        e0.record()
        for _ in range(20): f()
        e1.record(); torch.cuda.synchronize()
        us = e0.elapsed_time(e1) * 1e3 / 20
        print(f"{name} {mb} MB: {us:.1f} us, {n*4/us/1e3:.1f} GB/s")
