"""Hand-off timeline of the blocked TRSV (needs a -DGCM_TRACE build, loaded via GCM_LIB_PATH).

For every strip s (globaltimer ns, consistent across SMs to ~30 ns):
  0 chain 0 stores P_{s-kLookC-1}      4 helper: contraction done
  1 helper: hand-off tile's slot full  5 helper: hand-off values stored
  2 helper: thread 0 has its P values  6 chain 0 has the hand-off value (prep of block s)
  3 helper: all P values in smem       7 chain 0 starts the critical step of block s
usage: trace_chain.py n k"""
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
    gcm.modify(L, V.clone(), 1, algo="blocked")
torch.cuda.synchronize()
lib = _native.lib()
hb = (ctypes.c_longlong * (4096 * 8))()
lib.gcm_debug_htrace(hb, 4096 * 8)
hall = np.frombuffer(hb, dtype=np.int64).reshape(4096, 8).astype(np.float64)
h = hall[3000:]
reach = hall[3500:3500 + 600, 0]
NT = (n + 31) // 32
rows = [s for s in range(12, NT - 2) if np.all(h[s, :] > 0)]
d = h[rows] - h[rows, :1]
names = ["P stored", "helper slot full", "helper t0 has P", "helper all P", "helper GEMM done", "hand-off stored",
         "chain sees hand-off", "chain crit start"]
print(f"{len(rows)} strips; ns after chain 0 stored P_(s-5) (median / p10 / p90):")
for i in range(1, 8):
    print(f"  {names[i]:22s} {np.median(d[:, i]):8.0f} {np.percentile(d[:, i], 10):8.0f} {np.percentile(d[:, i], 90):8.0f}")
step = np.diff(h[12:NT - 2, 7])
print(f"chain step (crit start to crit start): median {np.median(step):.0f} ns")
print(f"  mean {step.mean():.0f} p90 {np.percentile(step, 90):.0f} max {step.max():.0f}; total chain span {h[NT-3,7]-h[12,7]:.0f} ns")
wait = np.array([h[s, 6] - reach[s] for s in rows])
print(f"chain waits for the hand-off (seen - reached poll): median {np.median(wait):.0f} p90 {np.percentile(wait,90):.0f} ns")
print(f"hand-off stored - chain reached poll: median {np.median([h[s,5]-reach[s] for s in rows]):.0f} ns (negative = stored before needed)")

# chain CTA 0 phase timing (clock64 of one SM; needs GCM_TRACE): per step tb
#  0 crit start  1 p stored  2 prep(tb+1) start  3 stage ready  4 partials done  5 hand-off read  6 prep done  7 loader issued
cb = (ctypes.c_longlong * (4096 * 8))()
lib.gcm_debug_trace(cb, 4096 * 8)
ct = np.frombuffer(cb, dtype=np.int64).reshape(4096, 8).astype(np.float64)[12:NT - 2]
print("chain CTA 0, cycles relative to crit start of the same step (median):")
for i, nm in [(1, "p stored"), (2, "prep start"), (3, "stage ready"), (4, "partials done"), (5, "hand-off read"),
              (6, "prep done")]:
    print(f"  {nm:16s} {np.median(ct[:, i] - ct[:, 0]):8.0f}")
print(f"  step (crit start to crit start) {np.median(np.diff(ct[:, 0])):.0f} cycles")

# fused diagonal sweeps (worker mode): per block b, globaltimer ns relative to chain 0's first P store
NB = (n + 63) // 64
w = hall[1000:1000 + NB]
t0 = h[12, 7]
ok = w[:, 2] > 0
if ok.any():
    print("worker sweeps (us after chain span start): ticket / U ready / L free / done, CTA")
    for b in list(range(0, NB, 8)) + [NB - 2, NB - 1]:
        r = w[b]
        print(f"  b={b:3d}  {(r[0]-t0)/1e3:8.1f} {(r[4]-t0)/1e3:8.1f} {(r[1]-t0)/1e3:8.1f} {(r[2]-t0)/1e3:8.1f}  cta {int(r[3])}")
    dur = w[ok, 2] - w[ok, 1]
    print(f"  sweep duration median {np.median(dur)/1e3:.1f} us, max {dur.max()/1e3:.1f}")

db = (ctypes.c_longlong * (256 * 8))()
if hasattr(lib, "gcm_debug_dtrace") and lib.gcm_debug_dtrace(db, 256 * 8) == 0:
    dt = np.frombuffer(db, dtype=np.int64).reshape(256, 8).astype(np.float64)[:NB]
    ok = dt[:, 5] > 0
    print("diagonal sweep phases (us, median over blocks): loads+P polled / w+U^-1 / V,q / closed rows / triangle")
    ph = [np.median(dt[ok, i + 1] - dt[ok, i]) / 1e3 for i in range(5)]
    print("  " + "  ".join(f"{x:.1f}" for x in ph))

# kernel timeline (TLINE): us after trsv entry, max over CTAs
tl = hall[2000]
if tl[0] > 0:
    names = ["trsv entry", "J1 done (last helper)", "chain start (CTA 0)", "chain end (last CTA)", "btma end (last CTA)"]
    sw = hall[1000:1000 + NB]
    print("kernel timeline (us after trsv entry):")
    for i, nm in enumerate(names):
        print(f"  {nm:24s} {(tl[i] - tl[0]) / 1e3:8.1f}")
    print(f"  last sweep done          {(sw[:, 2].max() - tl[0]) / 1e3:8.1f}")
jm = hall[2001]
if jm[0] > 0:
    print("J1 of helper 0, block 0 (us after trsv entry): start / Lb+X loads / X / tiles+segment / M,N / published")
    print("  " + " ".join(f"{(x - tl[0]) / 1e3:.1f}" for x in jm[:5]))
