"""Phase timing of the blocked diagonal kernel, block 0 (needs a -DGCM_SWEEP_TRACE build via GCM_LIB_PATH)."""
import ctypes
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1011_1173_b200 as gcm  # noqa: E402
from paper_1011_1173_b200 import _native  # noqa: E402
import synth  # noqa: E402

n, k = int(sys.argv[1]), int(sys.argv[2])
Lbuf, Vbuf, _ = synth.paper_instance(n, k, 1)
L = torch.from_numpy(Lbuf).cuda()
V = torch.from_numpy(Vbuf).cuda()
for _ in range(3):
    gcm.modify(L.clone(), V.clone(), 1, algo="blocked")
torch.cuda.synchronize()
buf = (ctypes.c_longlong * 2048)()
_native.lib().gcm_debug_sweep_trace(buf, 2048)
tr = np.frombuffer(buf, dtype=np.int64).astype(np.float64)
kb = 4 if k <= 4 else 8 if k <= 8 else 16 if k <= 16 else 32
ticks = 64 + kb - 1
t = tr[:4 * ticks].reshape(ticks, 4)
print(f"bdiag block 0: prologue {tr[1001] - tr[1000]:.0f} cycles, sweep {tr[1002] - tr[1001]:.0f} cycles ({ticks} ticks)")
per = np.diff(t[:, 0])
print(f"  tick period median {np.median(per):.0f}; coefficient warp done +{np.median(t[:, 1] - t[:, 0]):.0f}; "
      f"column apply done +{np.median(t[:, 3] - t[:, 0]):.0f}")
print(f"  loads -> +{tr[1003]-tr[1000]:.0f}; chol done +{tr[1004]-tr[1000]:.0f}; w done (thread 0) +{tr[1005]-tr[1000]:.0f}; "
      f"U^-1 + w synced +{tr[1006]-tr[1000]:.0f}; V states +{tr[1001]-tr[1000]:.0f}")
NB = (n + 63) // 64
st = tr[1536:1536 + NB]; en = tr[1024:1024 + NB]
d = [en[b] - st[b] for b in range(1, NB) if en[b] > 0 and st[b] > 0]
print(f"Gram CTA chol+inverse per block: median {np.median(d):.0f} cycles (max {np.max(d):.0f}); first G ready -> last U done "
      f"{en[NB-1] - st[1]:.0f} cycles")
