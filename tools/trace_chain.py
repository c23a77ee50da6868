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
    ok2 = ok & (h[:, 4] > 0) & (h[:, 5] > 0) & (h[:, 6] > 0)
    h2 = h[ok2]
    print(f"  publish -> feeder sees progress: {np.median(h2[:,6]-h2[:,0]):.0f}; feeder -> data landed (tile start): {np.median(h2[:,1]-h2[:,6]):.0f}")
    print(f"  tile start -> thread0 GEMM done: {np.median(h2[:,4]-h2[:,1]):.0f}; -> all compute done: {np.median(h2[:,5]-h2[:,1]):.0f}; -> rflag: {np.median(h2[:,2]-h2[:,1]):.0f}")
    ok3 = ok2 & (h[:, 7] > 0)
    h3 = h[ok3]
    print(f"  feeder reaches hand-off tile - publish: median {np.median(h3[:,7]-h3[:,0]):.0f} p10 {np.percentile(h3[:,7]-h3[:,0],10):.0f} p90 {np.percentile(h3[:,7]-h3[:,0],90):.0f}")
    print(f"  per-chain publish skew unknown; feeder poll time (seen - max(reach, publish)): {np.median(h3[:,6]-np.maximum(h3[:,7],h3[:,0])):.0f}")
    hc = np.frombuffer(hb, dtype=np.int64).reshape(4096, 8)[2048:2048 + NT].astype(np.float64)
    okc = np.all(hc > 0, axis=1)
    print("  per-chain publish time - chain0 (median over strips):", np.median(hc[okc] - hc[okc][:, :1], axis=0))
    rows = np.nonzero(ok3 & okc)[0]
    print("  feeder reach - last chain publish: median", np.median(h[rows, 7] - hc[rows].max(axis=1)))
    hs = np.frombuffer(hb, dtype=np.int64).reshape(4096, 8)[3000:3060].astype(np.float64)
    pub = np.frombuffer(hb, dtype=np.int64).reshape(4096, 8)[2048:2048+NT, 0].astype(np.float64)  # chain0 publish of tb = s-5 at row s
    base = hs[0, 3]
    print("helper 60, per tile seq (tb = seq): times rel. to feeder start (us): feeder[pre-empty, got-empty, got-P] compute[start, gemm, end]  P_tb published")
    for q in range(0, 60, 3):
        ptb = pub[q + 5] - base if q + 5 < NT and pub[q + 5] > 0 else float('nan')
        print(q, np.round((hs[q, [3, 4, 5, 0, 1, 2]] - base) / 1000, 2), round(ptb / 1000, 2))
    hs = tr[3000:3060].astype(np.float64)
    base = hs[0, 3]
    print("helper 60 clock64 (kcycles rel): feeder[reach, got-empty, got-P, P-issued] compute[start, gemm, end]")
    for q in range(0, 60, 3):
        print(q, np.round((hs[q, [3, 4, 5, 6, 0, 1, 2]] - base) / 1000, 2))
