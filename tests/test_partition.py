"""Multi-GPU partition host logic: windowed plans (a rank's
level-3 subtrees) equal the slices of the full plan, the rank-restricted
near-field tables equal the full tables' rows, the tree-only work estimate
balances like the exact model, and the exchange pattern runs with
world_size=2 on the gloo backend (CPU): each rank computes the far field of
its window with the oracle, the reduce-scatter / all-gather of
``RankExchange`` deliver the full far field, equal to the reference's
golden output."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from _support import golden, inputs, rel
from paper_2408_02274_b200 import nearfield, octree
from paper_2408_02274_b200.partition import (RankExchange, level3_partition, rank_targets,
                                             subtree_work, subtree_work_estimate)


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
    # targets: rank r owns rows r*chunk .. (r+1)*chunk (clipped), patch aligned
    chunk, t = rank_targets(disc.n_patches, disc.n_c, n_ranks)
    assert [p.targets for p in parts] == t and all(p.chunk == chunk for p in parts)
    assert t[0][0] == 0 and t[-1][1] == disc.n_points and chunk * n_ranks >= disc.n_points
    assert all(x[0] == r * chunk and x[0] % disc.n_c**2 == 0 for r, x in enumerate(t))
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


def test_tree_only_estimate_balances_like_exact_model():
    """Ranks partition before building anything (no cone hierarchy): the
    tree-only estimate tracks the exact per-subtree model and its cuts
    balance the exact work as well as the exact cuts do (within 5%)."""
    inp = inputs("c1")
    tree, hier, disc = inp["tree"], inp["hier"], inp["disc"]
    exact, est = subtree_work(tree, hier), subtree_work_estimate(tree)
    assert np.corrcoef(exact, est)[0, 1] > 0.95
    for n in (2, 3, 4, 8):
        pe = level3_partition(tree, None, n, disc.n_patches, disc.n_c)
        px = level3_partition(tree, hier, n, disc.n_patches, disc.n_c)
        imb = lambda parts: max(exact[p.box3[0]:p.box3[1]].sum() for p in parts) / (
            exact.sum() / n)
        assert imb(pe) <= 1.05 * imb(px)


@pytest.mark.parametrize("box3", [(0, 7), (7, 30), (30, 56), (0, 56), (20, 20)])
def test_window_plan_is_slice_of_full_plan(box3):
    """A rank's windowed cones / propagation / emission plans hold exactly
    the full plan's integers (and geometry) for its subtrees, re-based."""
    inp = inputs("c1")
    tree, hier = inp["tree"], inp["hier"]
    win = octree.tree_window(tree, *box3)
    view = octree.window_view(tree, win)
    hw = octree.build_cone_hierarchy(view)
    for d in range(3, tree.depth + 1):
        a, b = win.ranges[d]
        cl, cw = hier.level(d), hw.level(d)
        assert np.array_equal(cw.seg_ids, cl.seg_ids[cl.seg_off[a]:cl.seg_off[b]])
        assert np.array_equal(cw.seg_off, cl.seg_off[a:b + 1] - cl.seg_off[a])
        assert np.array_equal(cw.cpt_idx, cl.cpt_idx[cl.cpt_off[a]:cl.cpt_off[b]])
        if d >= 4:
            apf = octree.accumulation_plan(tree, hier, d)
            apw = octree.accumulation_plan(view, hw, d)
            pcl = hier.level(d - 1)
            r0, r1 = pcl.seg_off[win.ranges[d - 1][0]], pcl.seg_off[win.ranges[d - 1][1]]
            i0, i1 = apf.inst_off[r0], apf.inst_off[r1]
            assert np.array_equal(apw.inst_off, apf.inst_off[r0:r1 + 1] - i0)
            assert np.array_equal(apw.inst_child + a, apf.inst_child[i0:i1])
            crows = apf.crow[apf.inst_crow_off[i0]:apf.inst_crow_off[i1]]
            assert np.array_equal(apw.crow + cl.seg_off[a], crows)
            key = lambda ap, t: ap.type_gamma[t] * 8 + ap.type_octant[t]
            assert np.array_equal(key(apw, apw.inst_type), key(apf, apf.inst_type[i0:i1]))
            assert np.array_equal(apw.node_geom[apw.inst_type],
                                  apf.node_geom[apf.inst_type[i0:i1]])
        ef, ew = octree.emission_plan(tree, hier, d), octree.emission_plan(view, hw, d)
        p0, p1 = cl.cpt_off[a], cl.cpt_off[b]
        assert np.array_equal(ew.row + cl.seg_off[a], ef.row[p0:p1])
        assert np.array_equal(ew.geom, ef.geom[p0:p1])


@pytest.mark.parametrize("n_ranks", [2, 3])
def test_rank_near_field_tables_are_rows_of_full_tables(n_ranks):
    """classify_targets / correction_pairs restricted to a rank's targets
    equal the full tables' rows of those targets."""
    inp = inputs("c1")
    disc, tree, full = inp["disc"], inp["tree"], inp["smap"]
    cfull = nearfield.correction_pairs(disc, tree, full)
    _, ranges = rank_targets(disc.n_patches, disc.n_c, n_ranks)
    got_ell = []
    for t0, t1 in ranges:
        sm = nearfield.classify_targets(disc, target_range=(t0, t1))
        assert sm.target_lo == t0 and sm.n_targets == t1 - t0
        o0, o1 = full.offsets[t0], full.offsets[t1]
        assert np.array_equal(sm.offsets, full.offsets[t0:t1 + 1] - o0)
        assert np.array_equal(sm.patch_ids, full.patch_ids[o0:o1])
        assert np.array_equal(sm.closest_uv, full.closest_uv[o0:o1])
        cp = nearfield.correction_pairs(disc, tree, sm)
        sel = (cfull.ell_idx >= t0) & (cfull.ell_idx < t1)
        assert np.array_equal(cp.ell_idx, cfull.ell_idx[sel])
        assert np.array_equal(cp.src_idx, cfull.src_idx[sel])
        got_ell.append(cp.ell_idx)
    assert sum(e.size for e in got_ell) == cfull.nnz


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
    disc, tree = inp["disc"], inp["tree"]
    part = level3_partition(tree, None, world, disc.n_patches, disc.n_c)[rank]
    # this rank builds only its window's plan (tree-only partition)
    view = octree.window_view(tree, octree.tree_window(tree, *part.box3))
    hier = octree.build_cone_hierarchy(view)
    out, od = oracle.far_field(view, hier, z["weights"], inp["kappas"], disc.normals, 1e-6)
    # point-major exchange rows (the device layout): n_ranks*chunk x 8 values
    n, rows = disc.n_points, world * part.chunk
    full = np.zeros((rows, 2, out.shape[0] * out.shape[1]), dtype=complex)
    full[:n, 0] = out.reshape(-1, n).T
    full[:n, 1] = od.reshape(-1, n).T
    xfar = torch.from_numpy(full.reshape(-1).view(np.float64).copy())
    mine = torch.zeros(part.chunk * full.shape[1] * full.shape[2] * 2, dtype=torch.float64)
    ex = RankExchange()
    ex.reduce_scatter(xfar, mine)           # this rank's target rows, summed
    back = torch.zeros_like(xfar)
    ex.all_gather(back, mine)               # every rank's rows
    if rank == 0:
        np.save(result_path, back.numpy().view(complex).reshape(full.shape)[:n])
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_far_field_exchange_gloo(tmp_path):
    res = tmp_path / "far.npy"
    mp.spawn(_rank_main, args=(2, _free_port(), str(res)), nprocs=2, join=True)
    got = np.load(res)
    z = golden("rand_ifgf")
    n = got.shape[0]
    assert rel(got[:, 0].T.reshape(z["far"].shape), z["far"]) < 1e-13
    assert rel(got[:, 1].T.reshape(z["far_disp"].shape), z["far_disp"]) < 1e-13
    assert n == z["far"].shape[-1]
