"""Multi-GPU partition host logic, and the exchange pattern
exercised with world_size=2 on the gloo backend (CPU): each rank computes
the far field of its Morton range of level-3 subtrees with the oracle, an
all-reduce sums the partials, and the sum equals the reference's golden
far field."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from _support import golden, inputs, rel
from paper_2408_02274_b200.partition import level3_partition, subtree_work


@pytest.mark.parametrize("n_ranks", [2, 4, 8])
def test_partition_nearest_cuts_balanced_and_nonempty(n_ranks):
    """Cuts go to the nearer level-3 boundary: every rank owns subtrees and
    no rank is further from the mean than one level-3 subtree's work."""
    inp = inputs("c1")
    tree, hier, disc = inp["tree"], inp["hier"], inp["disc"]
    work = subtree_work(tree, hier)
    parts = level3_partition(tree, hier, n_ranks, disc.n_patches, disc.n_c)
    assert all(p.box3[1] > p.box3[0] for p in parts)
    mean = work.sum() / n_ranks
    assert max(abs(p.work - mean) for p in parts) <= work.max() + 1e-6 * mean


@pytest.mark.parametrize("n_ranks", [1, 2, 3, 8])
def test_partition_covers_everything_once(n_ranks):
    inp = inputs("c1")
    tree, hier, disc = inp["tree"], inp["hier"], inp["disc"]
    parts = level3_partition(tree, hier, n_ranks, disc.n_patches, disc.n_c)
    assert len(parts) == n_ranks
    for d in range(3, tree.depth + 1):
        cl = hier.level(d)
        for key, total in (("box", tree.level(d).n_boxes), ("seg", cl.n_segments),
                           ("pair", cl.cpt_idx.size)):
            rngs = [p.levels[d][key] for p in parts]
            assert rngs[0][0] == 0 and rngs[-1][1] == total
            assert all(rngs[i][1] == rngs[i + 1][0] for i in range(n_ranks - 1))
    t = [p.targets for p in parts]
    assert t[0][0] == 0 and t[-1][1] == disc.n_points
    assert all(x[0] % disc.n_c**2 == 0 for x in t)
    # children of an owned box are owned (no cross-rank parents)
    for p in parts:
        for d in range(4, tree.depth + 1):
            lo, hi = p.levels[d]["box"]
            plo, phi_ = p.levels[d - 1]["box"]
            par = tree.level(d).parent[lo:hi]
            assert par.size == 0 or (par.min() >= plo and par.max() < phi_)


def test_partition_balances_modelled_work():
    inp = inputs("c1")
    parts = level3_partition(inp["tree"], inp["hier"], 4, inp["disc"].n_patches,
                             inp["disc"].n_c)
    w = np.array([p.work for p in parts])
    assert abs(w.sum() - subtree_work(inp["tree"], inp["hier"]).sum()) < 1e-6 * w.sum()
    assert w.max() / w.mean() < 1.6        # 56 level-3 subtrees over 4 ranks


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _rank_main(rank, world, port, result_path):
    import oracle
    os.environ["OMP_NUM_THREADS"] = "2"
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}",
                            rank=rank, world_size=world)
    z, inp = golden("rand_ifgf"), inputs("rand_ifgf")
    parts = level3_partition(inp["tree"], inp["hier"], world, inp["disc"].n_patches,
                             inp["disc"].n_c)
    box_ranges = {d: parts[rank].levels[d]["box"] for d in parts[rank].levels}
    out, od = oracle.far_field(inp["tree"], inp["hier"], z["weights"], inp["kappas"],
                               inp["disc"].normals, 1e-6, box_ranges=box_ranges)
    t = torch.from_numpy(np.stack([out, od]))
    dist.all_reduce(t)                      # the cross-rank exchange (sum)
    if rank == 0:
        np.save(result_path, t.numpy())
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_far_field_exchange_gloo(tmp_path):
    res = tmp_path / "far.npy"
    mp.spawn(_rank_main, args=(2, _free_port(), str(res)), nprocs=2, join=True)
    got = np.load(res)
    z = golden("rand_ifgf")
    assert rel(got[0], z["far"]) < 1e-13
    assert rel(got[1], z["far_disp"]) < 1e-13
