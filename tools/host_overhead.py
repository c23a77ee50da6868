"""Host time of one modify call (no sync) vs its device time (events); a GPU idling on the
host's launches shows as host >= device.  usage: host_overhead.py n k algo"""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1011_1173_b200 as gcm  # noqa: E402

n, k, algo = int(sys.argv[1]), int(sys.argv[2]), sys.argv[3]
g = torch.Generator(device="cuda")
g.manual_seed(1)
L = torch.empty((n, n), dtype=torch.float64, device="cuda")
L.uniform_(-1 / n**0.5, 1 / n**0.5, generator=g)
L.diagonal().uniform_(1.0, 2.0, generator=g)
V = torch.rand((k, n), dtype=torch.float64, device="cuda", generator=g) / n**0.5
hs, ds, hq = [], [], []
Vc = V.clone()  # one buffer for every call (as bench.py): the panel tail's graph is replayed
for i in range(10):
    Vc.copy_(V)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda._sleep(2_000_000)  # ~1 ms of queued GPU work: the call's launches all land behind it
    e0.record()
    t0 = time.perf_counter()
    gcm.modify(L, Vc, 1 if i % 2 == 0 else -1, algo=algo)
    t1 = time.perf_counter()
    e1.record()
    torch.cuda.synchronize()
    ds.append(e0.elapsed_time(e1))
    # same call without the sleep: the GPU waits on the host wherever it is faster
    Vc.copy_(V)
    torch.cuda.synchronize()
    e0.record()
    t2 = time.perf_counter()
    gcm.modify(L, Vc, 1 if i % 2 == 0 else -1, algo=algo)
    t3 = time.perf_counter()
    e1.record()
    torch.cuda.synchronize()
    hs.append((t1 - t0) * 1e3)
    hq.append(e0.elapsed_time(e1))
print(f"{n} {k} {algo}: host enqueue {sorted(hs)[2]:.4f} ms, device (launches pre-queued) {sorted(ds)[2]:.4f} ms, "
      f"device (host-paced) {sorted(hq)[2]:.4f} ms")
