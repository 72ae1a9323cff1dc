"""Raw pinned-host <-> device copy rates (the e2e leg's ceiling)."""
import json

import torch

dev = torch.device("cuda:0")
res = {}
for mb in (33, 201):
    n = mb * (1 << 20) // 4
    h = torch.empty(n, dtype=torch.float32).pin_memory()
    d = torch.empty(n, dtype=torch.float32, device=dev)
    for name, fn in (("h2d", lambda: d.copy_(h, non_blocking=True)), ("d2h", lambda: h.copy_(d, non_blocking=True))):
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(10):
            fn()
        b.record()
        torch.cuda.synchronize()
        res[f"{name}_{mb}MB_GBps"] = round(10 * n * 4 / (a.elapsed_time(b) * 1e-3) / 1e9, 1)
# both directions at once on two streams
n = 201 * (1 << 20) // 4
h1 = torch.empty(n, dtype=torch.float32).pin_memory()
h2 = torch.empty(n // 2, dtype=torch.float32).pin_memory()
d1 = torch.empty(n, dtype=torch.float32, device=dev)
d2 = torch.empty(n // 2, dtype=torch.float32, device=dev)
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
for _ in range(10):
    with torch.cuda.stream(s1):
        d1.copy_(h1, non_blocking=True)
    with torch.cuda.stream(s2):
        h2.copy_(d2, non_blocking=True)
torch.cuda.current_stream().wait_stream(s1)
torch.cuda.current_stream().wait_stream(s2)
b.record()
torch.cuda.synchronize()
res["duplex_201MB_h2d_plus_100MB_d2h_ms"] = round(a.elapsed_time(b) / 10, 3)
print(json.dumps(res))
