"""Solver step timeline of the persistent panel chain (needs a -DGCM_PC_TRACE build via GCM_LIB_PATH).
Per 64-row step b (globaltimer ns): 0 step top, 1 W/tiles landed, 2 hand-off values in registers,
3 q_b published.  usage: pchain_trace.py n k"""
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
NB = (n + 63) // 64
buf = (ctypes.c_longlong * (4096 * 4))()
_native.lib().gcm_debug_pc_trace(buf, 4096 * 4)
tr = np.frombuffer(buf, dtype=np.int64).reshape(4096, 4)[:NB].astype(np.float64)
step = np.diff(tr[:, 0])
print(f"{NB} steps, solver span {(tr[-1, 3] - tr[0, 0]) / 1e3:.1f} us, step median {np.median(step):.0f} ns")
for i, nm in [(1, "W/tiles landed"), (2, "hand-off in regs"), (3, "q published")]:
    d = tr[3:, i] - tr[3:, i - 1]
    print(f"  {nm:18s} +{np.median(d):7.0f} ns (p90 {np.percentile(d, 90):7.0f})")
hp = np.frombuffer(buf, dtype=np.int64).reshape(4096, 4)[3072:3072 + 1024].astype(np.float64)
nt = int(np.argmax(hp[:, 0] == 0)) or 1024
if nt > 4:
    hp = hp[:nt]
    per = np.diff(hp[:, 0])
    print(f"helper CTA 40: {nt} tiles, period median {np.median(per):.0f} ns")
    for i, nm in [(1, "P in smem"), (2, "tile landed"), (3, "MMA (warp 0)")]:
        d = hp[2:, i] - hp[2:, i - 1]
        print(f"  {nm:16s} +{np.median(d):7.0f} ns (p90 {np.percentile(d, 90):7.0f})")
    ep = hp[3:, 0] - hp[2:-1, 3]
    print(f"  epilogue + next top +{np.median(ep):7.0f} ns")
    # when did P_b become visible vs the solver's publish of step b (tile b of this helper)
    pub = tr[:, 3]
    lag = [hp[q, 1] - pub[q] for q in range(min(nt, NB)) if pub[q] > 0]
    print(f"  P in smem - solver publish (same b): median {np.median(lag):.0f} ns")
