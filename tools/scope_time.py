"""Per-scope device time (library profiling hook) of one algorithm at (n, k): usage scope_time.py n k algo"""
import os
import sys

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
for i in range(3):
    gcm.modify(L, V.clone(), 1 if i % 2 == 0 else -1, algo=algo)
torch.cuda.synchronize()
gcm.profile_read()
gcm.profile_enable(True)
reps = 4
for i in range(reps):
    gcm.modify(L, V.clone(), 1 if i % 2 == 0 else -1, algo=algo)
torch.cuda.synchronize()
gcm.profile_enable(False)
prof = gcm.profile_read()
print(n, k, algo, {name: round(ms / reps, 4) for name, (cnt, ms) in prof.items()})
