"""One warm-up + one measured modify call (small driver for ncu captures)."""
import sys
import torch
sys.path.insert(0, '.')
import paper_1011_1173_b200 as gcm, synth
n, k = int(sys.argv[1]), int(sys.argv[2])
algo = sys.argv[3] if len(sys.argv) > 3 else "auto"
Lbuf, Vbuf, _ = synth.paper_instance(n, k, 1)
L = torch.from_numpy(Lbuf).cuda(); V0 = torch.from_numpy(Vbuf).cuda()
for _ in range(2):
    gcm.modify(L, V0.clone(), 1, algo=algo)
torch.cuda.synchronize()
print("ok")
