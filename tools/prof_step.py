"""Per-step time of one modify call plus the per-kernel-family breakdown
(library CUDA-event hooks).  usage: prof_step.py n k [algo] [steps]"""
import sys
import numpy as np
import torch
sys.path.insert(0, '.')
import paper_1011_1173_b200 as gcm, synth
n, k = int(sys.argv[1]), int(sys.argv[2])
algo = sys.argv[3] if len(sys.argv) > 3 else "auto"
steps = int(sys.argv[4]) if len(sys.argv) > 4 else 20
Lbuf, Vbuf, _ = synth.paper_instance(n, k, 1)
L0 = torch.from_numpy(Lbuf).cuda(); V0 = torch.from_numpy(Vbuf).cuda()
L = L0.clone(); V = V0.clone()
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
for _ in range(3):
    L.copy_(L0); V.copy_(V0); gcm.modify(L, V, 1, algo=algo)
torch.cuda.synchronize()
ts = []
gcm.profile_enable(True); gcm.profile_read()
for i in range(steps):
    L.copy_(L0); V.copy_(V0); flush.zero_()
    a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
    a.record(); gcm.modify(L, V, 1, algo=algo); b.record(); torch.cuda.synchronize()
    ts.append(a.elapsed_time(b))
prof = gcm.profile_read(); gcm.profile_enable(False)
fl = 6 * k * n * (n - 1) / 2
t = float(np.median(ts))
print(f"n={n} k={k} algo={algo}: median {t:.4f} ms ({fl / t / 1e9:.3f} TFLOP/s)  "
      + "  ".join(f"{nm}={ms / steps * 1e3:.1f}us" for nm, (c, ms) in prof.items()))
