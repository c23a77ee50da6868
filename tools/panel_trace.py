"""Chain timeline of the panel path (GCM_PANEL_TRACE): n, k from argv; synthetic SPD-factor input."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1011_1173_b200 as gcm  # noqa: E402

n, k = int(sys.argv[1]), int(sys.argv[2])
g = torch.Generator(device="cuda")
g.manual_seed(1)
L = torch.empty((n, n), dtype=torch.float64, device="cuda")
L.uniform_(-1 / n**0.5, 1 / n**0.5, generator=g)
L.diagonal().uniform_(1.0, 2.0, generator=g)
V = torch.rand((k, n), dtype=torch.float64, device="cuda", generator=g) / n**0.5
for i in range(3):
    if i == 2:
        os.environ["GCM_PANEL_TRACE"] = "1"
    gcm.modify(L, V.clone(), 1 if i % 2 == 0 else -1, algo="panel")
    torch.cuda.synchronize()
