"""Print GPU-vs-oracle errors of the near-singular downdates (tests/test_gpu_edge.py instances)
beside rho^2 and the test tolerance, for every algorithm (R19 calibration)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]
import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle  # noqa: E402
import paper_1011_1173_b200 as gcm  # noqa: E402
from gcm_testutil import col_scaled_max, rel_fro, upper  # noqa: E402
from test_gpu_edge import near_singular, rho2  # noqa: E402

EPS = np.finfo(np.float64).eps
for algo in ("sweep", "blocked"):
    for n, k, m in [(200, 1, 77), (700, 4, 300), (700, 16, 640), (2000, 16, 1500)]:
        for delta in (1e-2, 1e-4, 1e-6, 1e-8):
            Lb, V = near_singular(n, k, m, delta, seed=n + m)
            r2 = rho2(Lb, V)
            Lo, Vo = Lb.copy(), V.copy()
            oracle.modify_a(Lo, Vo, -1)
            L = torch.from_numpy(Lb.copy()).cuda()
            Vg = torch.from_numpy(V.copy()).cuda()
            gcm.modify(L, Vg, -1, algo=algo)
            torch.cuda.synchronize()
            Lg = L.cpu().numpy()
            e = rel_fro(upper(Lg), upper(Lo))
            c = col_scaled_max(upper(Lg), upper(Lo))
            ev = rel_fro(Vg.cpu().numpy(), Vo)
            print(f"{algo:8s} n={n:5d} k={k:3d} m={m:5d} delta={delta:.0e} rho2={r2:.3e} relF={e:.3e} "
                  f"colmax={c:.3e} V_relF={ev:.3e} eps/rho2={EPS / r2:.3e} ratio={e / (EPS / r2):.3f}", flush=True)
