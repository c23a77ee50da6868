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


if __name__ == "__main__":
    single(200, 5, 1, "sweep")
    single(330, 16, -1, "blocked")
    single(512, 40, 1, "blocked")
    single(300, 7, 1, "blocked", ldl=303)
    batched(512, 8, 4, 1)
    print("sanitize cases ok")
