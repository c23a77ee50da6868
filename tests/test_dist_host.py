"""CPU tests of the column-sharded path's host logic (no GPU).

* the block-cyclic ownership functions exported by libgcm (gcm_dist_local_cols,
  gcm_dist_global_col) partition the columns correctly;
* a world_size-2 gloo run of the SAME schedule dist.cu executes (owner of the
  columns of each 64-row block computes its rotations, one broadcast per block from
  that owner, every rank applies them to its own columns to the right; V rows follow
  their columns), with the oracle as the per-rank arithmetic, reproduces the
  single-process oracle result.  This pins the ownership/broadcast choreography;
  the GPU kernels themselves are covered by the -m gpu tests.
"""
import os
import socket

import numpy as np
import pytest

from paper_1011_1173_b200 import dist as gdist

D = 64


@pytest.mark.parametrize("n,nb,world", [(1, 64, 1), (100, 64, 2), (300, 64, 3), (1000, 128, 4), (640, 192, 2)])
def test_block_cyclic_partition(n, nb, world):
    allcols = []
    total = 0
    for r in range(world):
        g = gdist.global_cols(n, nb, world, r)
        assert gdist.local_cols(n, nb, world, r) == len(g)
        assert np.all(np.diff(g) > 0)
        assert np.all(((g // nb) % world) == r)  # owner of column j is (j / nb) mod P
        total += len(g)
        allcols.extend(g.tolist())
    assert total == n
    assert sorted(allcols) == list(range(n))


def test_invalid_layout():
    with pytest.raises(ValueError):
        gdist.local_cols(10, 0, 2, 0)
    with pytest.raises(ValueError):
        gdist.local_cols(10, 64, 2, 2)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _rank_main(rank, world, port, n, k, nb, sigma, outdir):
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import torch
    import torch.distributed as dist

    import oracle
    import synth
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    Lbuf, Vbuf, _ = synth.paper_instance(n, k, sigma, seed=123)
    gcols = gdist.global_cols(n, nb, world, rank)
    Lloc = Lbuf[gcols].copy()       # local columns, all rows (row c of Lloc = column gcols[c])
    Vloc = Vbuf[:, gcols].copy()    # V entries of the local columns
    for b in range((n + D - 1) // D):
        r0 = b * D
        Db = min(D, n - r0)
        owner = (r0 // nb) % world
        cs = torch.zeros(2, Db, k, dtype=torch.float64)
        if owner == rank:
            lc = np.searchsorted(gcols, np.arange(r0, r0 + Db))
            assert np.array_equal(gcols[lc], np.arange(r0, r0 + Db))
            Lbb = np.zeros((Db, Db))
            Lbb[:, :] = Lloc[lc][:, r0:r0 + Db]  # rows of Lbb = block columns
            Vb = np.ascontiguousarray(Vloc[:, lc])
            c, s, _ = oracle.modify_a(Lbb, Vb, sigma)  # the diagonal chain of block b
            Lloc[lc, r0:r0 + Db] = Lbb
            Vloc[:, lc] = Vb
            cs[0] = torch.from_numpy(c)
            cs[1] = torch.from_numpy(s)
        dist.broadcast(cs, src=owner)  # the one exchange step per block
        c, s = cs[0].numpy(), cs[1].numpy()
        right = np.nonzero(gcols >= r0 + D)[0]
        for j in range(Db):  # Apply (PAPER.md 52-54) to the rank's columns right of the block
            for e in range(k):
                Lr = Lloc[right, r0 + j]
                Vr = Vloc[e, right]
                lnew = (Lr + sigma * s[j, e] * Vr) / c[j, e]
                Lloc[right, r0 + j] = lnew
                Vloc[e, right] = c[j, e] * Vr - s[j, e] * lnew
    np.save(os.path.join(outdir, f"L{rank}.npy"), Lloc)
    np.save(os.path.join(outdir, f"V{rank}.npy"), Vloc)
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("sigma", [1, -1])
def test_gloo_world2_schedule_matches_oracle(tmp_path, sigma):
    import torch.multiprocessing as mp

    import oracle
    import synth
    from gcm_testutil import rel_fro, upper
    n, k, nb, world = 300, 3, 64, 2
    port = _free_port()
    mp.spawn(_rank_main, args=(world, port, n, k, nb, sigma, str(tmp_path)), nprocs=world, join=True)
    Lbuf, Vbuf, _ = synth.paper_instance(n, k, sigma, seed=123)
    Lo, Vo = Lbuf.copy(), Vbuf.copy()
    oracle.modify_a(Lo, Vo, sigma)
    Lg = np.zeros_like(Lbuf)
    Vg = np.zeros_like(Vbuf)
    for r in range(world):
        g = gdist.global_cols(n, nb, world, r)
        Lg[g] = np.load(tmp_path / f"L{r}.npy")
        Vg[:, g] = np.load(tmp_path / f"V{r}.npy")
    assert rel_fro(upper(Lg), upper(Lo)) < 1e-13
    assert rel_fro(Vg, Vo) < 1e-12
