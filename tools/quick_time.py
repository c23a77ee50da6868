import sys, time, torch, numpy as np
sys.path.insert(0, '.')
import paper_1011_1173_b200 as gcm, synth
n, k = int(sys.argv[1]), int(sys.argv[2])
algo = sys.argv[3] if len(sys.argv) > 3 else "auto"
Lbuf, Vbuf, _ = synth.paper_instance(n, k, 1)
L = torch.from_numpy(Lbuf).cuda(); V0 = torch.from_numpy(Vbuf).cuda(); V = V0.clone()
for _ in range(3):
    V.copy_(V0); gcm.modify(L, V, 1, algo=algo); V.copy_(V0); gcm.modify(L, V, -1, algo=algo)
torch.cuda.synchronize()
ts = []
for i in range(10):
    V.copy_(V0)
    a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
    a.record(); gcm.modify(L, V, 1 if i % 2 == 0 else -1, algo=algo); b.record(); torch.cuda.synchronize()
    ts.append(a.elapsed_time(b))
t = np.median(ts)
print(f"n={n} k={k} algo={algo}: median {t:.3f} ms  GFLOP/s {6*k*n*(n-1)/2/t/1e6:.1f}")
