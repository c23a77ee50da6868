"""Per-step phase timing of the blocked TRSV chain CTA (needs a -DGCM_TRACE build via GCM_LIB_PATH)."""
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
buf = (ctypes.c_longlong * (4096 * 8))()
lib.gcm_debug_trace(buf, 4096 * 8)
tr = np.frombuffer(buf, dtype=np.int64).reshape(4096, 8)
NT = (n + 31) // 32
t = tr[:NT].astype(np.float64)
step = np.diff(t[:, 0])
print(f"steps {NT}: chain step cycles median {np.median(step):.0f} mean {step.mean():.0f}")
pubt = tr[1024:1024 + NT, 0].astype(np.float64)
R = [t[tb - 1, 5] - pubt[tb - 5] for tb in range(10, NT - 2)]
print(f"chain-local hand-off round trip (publish P_tb -> sees r for strip tb+5), cycles: median {np.median(R):.0f} p10 {np.percentile(R,10):.0f} p90 {np.percentile(R,90):.0f}")
P2 = [pubt[tb] - t[tb, 1] for tb in range(10, NT - 2)]
print(f"  p_done -> publish: median {np.median(P2):.0f}")
names = ["crit.start", "crit.p_done", "prep.start", "prep.mbar_ok", "prep.partials", "prep.rflag_ok", "prep.done", "svc.issued"]
for s in range(1, 8):
    d = t[1:-2, s] - t[1:-2, 0]
    print(f"  {names[s]:22s} - crit.start: median {np.median(d):8.0f}  p10 {np.percentile(d,10):8.0f} p90 {np.percentile(d,90):8.0f}")

if hasattr(lib, "gcm_debug_htrace"):
    hb = (ctypes.c_longlong * (4096 * 8))()
    lib.gcm_debug_htrace(hb, 4096 * 8)
    h = np.frombuffer(hb, dtype=np.int64).reshape(4096, 8)[:NT].astype(np.float64)
    ok = (h[:, 0] > 0) & (h[:, 1] > 0) & (h[:, 2] > 0) & (h[:, 3] > 0)
    hh = h[ok]
    print(f"hand-off timeline (ns, globaltimer) over {ok.sum()} strips:")
    print(f"  chain publish P -> helper starts hand-off tile: median {np.median(hh[:,1]-hh[:,0]):.0f}")
    print(f"  helper tile start -> rflag published:           median {np.median(hh[:,2]-hh[:,1]):.0f}")
    print(f"  rflag published -> chain prep sees it:          median {np.median(hh[:,3]-hh[:,2]):.0f}")
    print(f"  chain publish P -> chain sees hand-off:         median {np.median(hh[:,3]-hh[:,0]):.0f}")
    hs = tr[3000:3060].astype(np.float64)
    base = hs[0, 3]
    print("helper 60 clock64 (kcycles rel): feeder[reach, got-empty, got-P, P-issued] compute[start, gemm, end]")
    for q in range(0, 60, 3):
        print(q, np.round((hs[q, [3, 4, 5, 6, 0, 1, 2]] - base) / 1000, 2))
print("helper 60 tiles 44..58 (kcycles rel. to tile 44 start): [full-wait done, pfast loaded (fast tiles), gemm done, end]")
b0 = tr[3000 + 44, 0]
for q in range(44, 59):
    r = tr[3000 + q]
    print(q, [round((r[i] - b0) / 1000, 2) if r[i] > 0 else None for i in (0, 7, 1, 2)])
print("helper 60 tiles: [full-wait done, before fast, pfast loaded, fma loop done, all done]")
for q in range(44, 59):
    r = tr[3000 + q]; r2 = tr[3500 + q]
    print(q, [round((x - b0) / 1000, 2) if x > 0 else None for x in (r[0], r2[1], r[7], r2[0], r[1])])
print("helper 60 tiles: [full-wait done, before fast, pfast loaded, fma loop done, sums done, r updated, all done]")
for q in range(44, 59):
    r = tr[3000 + q]; r2 = tr[3500 + q]
    print(q, [round((x - b0) / 1000, 2) if x > 0 else None for x in (r[0], r2[1], r[7], r2[0], r2[3], r2[2], r[1])])
w = tr[2048:2048 + NT].astype(np.float64)
print(f"hand-off not yet there at first poll: {int(w[10:NT-2,0].sum())} of {NT-12} steps; wait cycles median {np.median(w[10:NT-2,2]-w[10:NT-2,1]):.0f} p90 {np.percentile(w[10:NT-2,2]-w[10:NT-2,1],90):.0f}")
print("first-poll time - crit.start (median):", np.median(w[10:NT-2,1] - t[10-1:NT-2-1,0]))
