"""Phase times of pdiag_kernel's diagonal blocks (needs a -DGCM_TRACE build via GCM_LIB_PATH).
Marks: 0 start, 1 L/P loaded, 2 w and U^{-1}, 3 V states, 4 closed-form rows, 5 triangle.
usage: pdiag_phases.py n k"""
import ctypes
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1011_1173_b200 as gcm  # noqa: E402
from paper_1011_1173_b200 import _native  # noqa: E402

n, k = int(sys.argv[1]), int(sys.argv[2])
g = torch.Generator(device="cuda")
g.manual_seed(1)
L = torch.empty((n, n), dtype=torch.float64, device="cuda")
L.uniform_(-1 / n**0.5, 1 / n**0.5, generator=g)
L.diagonal().uniform_(1.0, 2.0, generator=g)
V = torch.rand((k, n), dtype=torch.float64, device="cuda", generator=g) / n**0.5
for i in range(3):
    gcm.modify(L, V.clone(), 1 if i % 2 == 0 else -1, algo="panel")
torch.cuda.synchronize()
buf = (ctypes.c_longlong * 2048)()
_native.lib().gcm_debug_dtrace_panel(buf, 2048)
tr = np.frombuffer(buf, dtype=np.int64).reshape(256, 8)[: (n + 63) // 64, :6].astype(np.float64)
d = np.diff(tr, axis=1)
names = ["L/P loaded", "w, U^-1", "V states", "closed rows", "triangle"]
print(f"pdiag phases over {tr.shape[0]} blocks (median / max ns): total {np.median(tr[:, 5] - tr[:, 0]):.0f} / {np.max(tr[:, 5] - tr[:, 0]):.0f}")
for i, nm in enumerate(names):
    print(f"  {nm:12s} {np.median(d[:, i]):8.0f} {np.max(d[:, i]):8.0f}")
