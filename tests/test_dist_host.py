"""CPU tests of the column-sharded path's host logic (no GPU).

* the block-cyclic ownership functions exported by libgcm (gcm_dist_local_cols,
  gcm_dist_global_col) partition the columns correctly;
* a world_size-2 (and 3) gloo job in which every rank asks the library for ITS share of
  gcm_modify_dist's work (gcm_dist_plan: the Apply tiles, the 64-row diagonal blocks it
  sweeps, the column blocks whose rows of P it solves) and the ranks all-gather them: the
  union must cover every tile (b < s), diagonal block and column block exactly once, every
  tile must lie in the rank's own columns, and the owner of column block g must be rank
  g mod R.  This pins the C++ planner the GPU path runs (panel.cu make_plan); the GPU
  kernels themselves are covered by tests/test_gpu_dist.py (virtual ranks on one GPU).
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
    with pytest.raises(ValueError):
        gdist.plan(100, 48, 2, 0, "tiles")  # nb must be a multiple of 64


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _rank_main(rank, world, port, cases, outdir):
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import torch.distributed as dist

    from paper_1011_1173_b200 import dist as gd
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    for ci, (n, nb) in enumerate(cases):
        mine = {w: gd.plan(n, nb, world, rank, w).tolist() for w in ("tiles", "diag", "solve")}
        mine["cols"] = gd.global_cols(n, nb, world, rank).tolist()
        everyone = [None] * world
        dist.all_gather_object(everyone, mine)
        if rank == 0:
            import json
            with open(os.path.join(outdir, f"case{ci}.json"), "w") as f:
                json.dump(everyone, f)
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_gloo_plan_covers_the_factor_once(tmp_path, world):
    import json

    import torch.multiprocessing as mp
    cases = [(300, 64), (1000, 256), (2113, 512), (777, 128)]
    mp.spawn(_rank_main, args=(world, _free_port(), cases, str(tmp_path)), nprocs=world, join=True)
    for ci, (n, nb) in enumerate(cases):
        everyone = json.load(open(tmp_path / f"case{ci}.json"))
        NB = (n + D - 1) // D
        NBc = (n + nb - 1) // nb
        tiles, diag, solve = [], [], []
        for r, w in enumerate(everyone):
            cols = set(w["cols"])
            for b, s in w["tiles"]:
                assert b < s and s * D in cols, (r, b, s)  # the rank's own columns, above the diagonal
                tiles.append((b, s))
            for b in w["diag"]:
                assert b * D in cols
                diag.append(b)
            for g in w["solve"]:
                assert g % world == r
                solve.append(g)
        assert sorted(tiles) == sorted((b, s) for s in range(NB) for b in range(s))
        assert sorted(diag) == list(range(NB))
        assert sorted(solve) == list(range(NBc))


@pytest.mark.parametrize("n,nb", [(3000, 512), (1000, 256), (700, 64)])
def test_one_rank_plan_sorted_by_row_block(n, nb):
    """One rank (the persistent chain's overlapped tail takes Apply items row block by row block):
    the plan's Apply items cover every tile (b, s), b < s, exactly once, and each of the two item
    lists (TMA groups, then single tiles) is ordered by row block b."""
    from paper_1011_1173_b200 import dist as gdist
    pairs = gdist.plan(n, nb, 1, 0, "tiles")
    NB = (n + 63) // 64
    assert sorted(map(tuple, pairs.tolist())) == sorted((b, s) for s in range(NB) for b in range(s))
    bs = pairs[:, 0]
    runs = 1 + int(np.sum(bs[1:] < bs[:-1]))
    assert runs <= 2
