"""Phase clocks of the TMA batched kernel (build: tools/build_variant.sh bttrace -DGCM_BT_TRACE;
run with GCM_LIB_PATH pointing at it).  Prints per 64-row block: Ls load, in-block solve,
closed-form rows, triangle, L~ store, Apply, in SM cycles, for CTA 0 and CTA batch/2."""
import ctypes
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1011_1173_b200 as gcm  # noqa: E402
import synth  # noqa: E402

n, k, batch = 512, 8, int(sys.argv[1]) if len(sys.argv) > 1 else 4096
Ls, Vs, _ = synth.batched_instances(32, n, k, 1, seed=3)
reps = batch // 32
L = torch.from_numpy(np.tile(Ls, (reps, 1, 1))).cuda()
V0 = torch.from_numpy(np.tile(Vs, (reps, 1, 1))).cuda()
for i in range(3):
    V = V0.clone()
    gcm.modify_batched(L, V, 1 if i % 2 == 0 else -1)
torch.cuda.synchronize()
lib = gcm._native.lib()
buf = (ctypes.c_longlong * (2 * 16 * 8))()
lib.gcm_debug_bt_trace(buf, 2 * 16 * 8)
a = np.array(buf, dtype=np.int64).reshape(2, 16, 8)
names = ["load", "trsv", "closed", "tri", "store", "apply"]
for c in range(2):
    print(f"CTA {'0' if c == 0 else 'mid'}: cycles per phase (block rows)")
    tot = np.zeros(6)
    for b in range(8):
        r = a[c, b]
        d = [r[1] - r[0], r[2] - r[1], r[3] - r[2], r[4] - r[3], r[5] - r[4], (r[6] - r[5]) if b < 7 else 0]
        tot += d
        print(f"  b={b}: " + "  ".join(f"{nm}={x:7d}" for nm, x in zip(names, d)))
    print("  total: " + "  ".join(f"{nm}={int(x):7d}" for nm, x in zip(names, tot)), " sum", int(tot.sum()))

buf2 = (ctypes.c_longlong * (16 * 8))()
if lib.gcm_debug_dc_trace(buf2, 16 * 8) == 0:
    d = np.array(buf2, dtype=np.int64).reshape(16, 8)
    print("diag_closed sub-steps (CTA 0): A+prefix, B (per-row chol), C (row compute), mu scan, D")
    for b in range(8):
        r = d[b]
        print(f"  b={b}: " + "  ".join(str(int(r[i + 1] - r[i])) for i in range(5)))
