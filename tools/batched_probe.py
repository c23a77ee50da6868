import sys, torch
sys.path.insert(0, '.')
import paper_1011_1173_b200 as gcm, synth
n, k, batch = (int(x) for x in sys.argv[1:4])
Ls, Vs, _ = synth.batched_instances(batch, n, k, 1, seed=3)
L = torch.from_numpy(Ls).cuda(); V = torch.from_numpy(Vs).cuda()
gcm.modify_batched(L, V, 1)
torch.cuda.synchronize(); print("ok", n, k, batch)
