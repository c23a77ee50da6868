"""Per-tile phase timing (clock64) of helper CTA h=100 of the blocked TRSV (needs a -DGCM_TRACE build).
slots: 0 loop top  1 slot full  2 P validated  3 GEMM sums done  4 tile done; 6 tb, 7 strip"""
import ctypes, os, sys
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1011_1173_b200 as gcm  # noqa: E402
from paper_1011_1173_b200 import _native  # noqa: E402
import synth  # noqa: E402
n, k = int(sys.argv[1]), int(sys.argv[2])
Lbuf, Vbuf, _ = synth.paper_instance(n, k, 1)
L = torch.from_numpy(Lbuf).cuda(); V = torch.from_numpy(Vbuf).cuda()
for _ in range(3):
    gcm.modify(L, V.clone(), 1, algo="blocked")
torch.cuda.synchronize()
hb = (ctypes.c_longlong * (4096 * 8))()
_native.lib().gcm_debug_htrace(hb, 4096 * 8)
h = np.frombuffer(hb, dtype=np.int64).reshape(4096, 8)[:2900].astype(np.float64)
nt = int(np.argmax(h[:, 0] == 0)) or 2900
h = h[:nt]
d = np.diff(h[:, 0])
print(f"helper 100: {nt} tiles; per-tile period median {np.median(d):.0f} cycles (mean {d.mean():.0f})")
for i, nm in [(1, "slot full"), (2, "P validated"), (3, "GEMM sums"), (4, "tile done")]:
    print(f"  {nm:12s} +{np.median(h[:, i] - h[:, 0]):6.0f}  (p90 {np.percentile(h[:, i] - h[:, 0], 90):6.0f})")
print("  last 8 tiles (tb, strip, full-wait, validate, gemm, rest):")
for r in h[-8:]:
    print(f"   {int(r[6]):4d} {int(r[7]):4d} {r[1]-r[0]:7.0f} {r[2]-r[1]:7.0f} {r[3]-r[2]:7.0f} {r[4]-r[3]:7.0f}")
