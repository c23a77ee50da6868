"""Kernel timeline of one modify call (torch.profiler / CUPTI: start, duration, stream per kernel,
relative to the call's first kernel).  usage: kernel_timeline.py n k [algo]"""
import os
import sys

import torch
from torch.profiler import ProfilerActivity, profile

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1011_1173_b200 as gcm  # noqa: E402

n, k = int(sys.argv[1]), int(sys.argv[2])
algo = sys.argv[3] if len(sys.argv) > 3 else "panel"
g = torch.Generator(device="cuda")
g.manual_seed(1)
L = torch.empty((n, n), dtype=torch.float64, device="cuda")
L.uniform_(-1 / n**0.5, 1 / n**0.5, generator=g)
L.diagonal().uniform_(1.0, 2.0, generator=g)
V = torch.rand((k, n), dtype=torch.float64, device="cuda", generator=g) / n**0.5
for i in range(4):
    gcm.modify(L, V.clone(), 1 if i % 2 == 0 else -1, algo=algo)
torch.cuda.synchronize()
Vc = V.clone()
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    gcm.modify(L, Vc, 1, algo=algo)
    torch.cuda.synchronize()
ev = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
ev.sort(key=lambda e: e.time_range.start)
t0 = ev[0].time_range.start
end = max(e.time_range.end for e in ev)
print(f"n={n} k={k} algo={algo}: {len(ev)} device events, span {end - t0:.1f} us")
rows = {}
for e in ev:
    nm = e.name.split("<")[0].split("(")[0][:40]
    r = rows.setdefault(nm, [0, 0.0, 1e18, 0.0])
    r[0] += 1
    r[1] += e.time_range.end - e.time_range.start
    r[2] = min(r[2], e.time_range.start - t0)
    r[3] = max(r[3], e.time_range.end - t0)
print(f"{'kernel':40s} {'n':>4s} {'sum us':>9s} {'first':>8s} {'last end':>8s}")
for nm, r in sorted(rows.items(), key=lambda x: x[1][2]):
    print(f"{nm:40s} {r[0]:4d} {r[1]:9.1f} {r[2]:8.1f} {r[3]:8.1f}")
if "-v" in sys.argv:
    for e in ev:
        print(f"{e.time_range.start - t0:9.1f} {e.time_range.end - e.time_range.start:8.1f} {e.name[:60]}")
