"""Small cases of every algorithm for compute-sanitizer (memcheck / synccheck / racecheck):
the panel sweep (n < 256), the blocked path (cooperative TRSV kernel with fused diagonal
sweeps + the programmatic-dependent TMA Apply; k = 40 = two passes), the blocked path with an
unaligned leading dimension (plain Apply after the TRSV kernel), and the batched kernel.
Each result is checked against the oracle, so a silent corruption also fails the run."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]
import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle  # noqa: E402
import paper_1011_1173_b200 as gcm  # noqa: E402
import synth  # noqa: E402
from gcm_testutil import rel_fro, upper  # noqa: E402


def single(n, k, sigma, algo, ldl=None):
    Lb, Vb, _ = synth.paper_instance(n, k, sigma, seed=5, ldl=ldl)
    Lo, Vo = Lb.copy(), Vb.copy()
    oracle.modify_a(Lo, Vo, sigma)
    L, V = torch.from_numpy(Lb).cuda(), torch.from_numpy(Vb).cuda()
    gcm.modify(L, V, sigma, algo=algo)
    torch.cuda.synchronize()
    e = rel_fro(upper(L.cpu().numpy()), upper(Lo))
    print(f"{algo} n={n} k={k} ldl={ldl or n} sigma={sigma}: rel-F {e:.2e}", flush=True)
    assert e < 1e-11


def batched(n, k, batch, sigma):
    Ls, Vs, _ = synth.batched_instances(batch, n, k, sigma, seed=9)
    Lo, Vo = Ls.copy(), Vs.copy()
    for f in range(batch):
        oracle.modify_a(Lo[f], Vo[f], sigma)
    L, V = torch.from_numpy(Ls).cuda(), torch.from_numpy(Vs).cuda()
    gcm.modify_batched(L, V, sigma)
    torch.cuda.synchronize()
    e = max(rel_fro(upper(L.cpu().numpy()[f]), upper(Lo[f])) for f in range(batch))
    print(f"batched {batch} x n={n} k={k} sigma={sigma}: rel-F {e:.2e}", flush=True)
    assert e < 1e-11


def f32(n, k, sigma):
    Lb, Vb, _ = synth.paper_instance(n, k, sigma, seed=6)
    L32, V32 = Lb.astype(np.float32), Vb.astype(np.float32)
    Lo, Vo = L32.copy(), V32.copy()
    oracle.modify_a_f32(Lo, Vo, sigma)
    L, V = torch.from_numpy(L32).cuda(), torch.from_numpy(V32).cuda()
    gcm.modify_f32(L, V, sigma)
    torch.cuda.synchronize()
    e = rel_fro(upper(L.cpu().numpy()).astype(np.float64), upper(Lo).astype(np.float64))
    print(f"f32 n={n} k={k} sigma={sigma}: rel-F {e:.2e}", flush=True)
    assert e < 1e-5


def virtual(n, k, nb, R, sigma):
    from paper_1011_1173_b200 import dist
    Lb, Vb, _ = synth.paper_instance(n, k, sigma, seed=7, ldl=n + 1)
    Lo, Vo = Lb.copy(), Vb.copy()
    oracle.modify_a(Lo, Vo, sigma)
    sh = dist.shard(torch.from_numpy(Lb).cuda(), torch.from_numpy(Vb).cuda(), nb, R)
    dist.modify_dist_virtual([s[0] for s in sh], [s[1] for s in sh], n, nb, sigma)
    torch.cuda.synchronize()
    Lg = np.zeros_like(Lb)
    for Ls, _, g in sh:
        Lg[g] = Ls.cpu().numpy()
    e = rel_fro(upper(Lg), upper(Lo))
    print(f"dist virtual R={R} n={n} k={k} nb={nb} sigma={sigma}: rel-F {e:.2e}", flush=True)
    assert e < 1e-11


if __name__ == "__main__":
    single(200, 5, 1, "sweep")
    single(330, 16, -1, "blocked")
    single(512, 40, 1, "blocked")
    single(300, 7, 1, "blocked", ldl=303)
    single(600, 16, -1, "panel")
    batched(512, 8, 4, 1)
    batched(300, 16, 3, -1)
    f32(200, 5, 1)
    virtual(700, 16, 256, 3, 1)
    print("sanitize cases ok")
