"""Native (device) plan builder against the host numpy builder, which is
itself bit-exact with the reference plan digests (tests/test_plan.py): the
cone hierarchy built on the GPU (csrc/planbuild.cu) has identical integer
arrays at every golden configuration, including windows (multi-GPU ranks)."""

import numpy as np
import pytest

from _support import GOLDEN, golden_digests, framework_digests, inputs
from paper_2408_02274_b200 import octree

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("name", ["s1", "c1", "se1", "sl1", "c2n4", "c2n8"])
def test_device_cones_equal_host_cones(name):
    if not (GOLDEN / f"{name}.npz").exists():
        pytest.skip(f"{name} fixture not generated")
    inp = inputs(name)
    tree, host = inp["tree"], inp["hier"]
    dev = octree.build_cone_hierarchy(tree, device=True)
    for d in host.cone_levels:
        a, b = host.level(d), dev.level(d)
        assert np.array_equal(a.seg_off, b.seg_off), d
        assert np.array_equal(a.seg_ids, b.seg_ids), d
        assert np.array_equal(a.cpt_idx, b.cpt_idx) and np.array_equal(a.cpt_off, b.cpt_off)
    # and therefore the reference's digests (cone arrays; the propagation
    # types are compared in test_device_propagation_types_equal_host)
    dev.device_plan = False
    ref = golden_digests(name)
    mine = framework_digests(dict(inp, hier=dev))
    assert all(str(mine[k]) == str(ref[k]) for k in ref if k.startswith("C"))


def test_device_cones_in_windows():
    inp = inputs("c1")
    tree, host = inp["tree"], inp["hier"]
    for box3 in [(0, 9), (9, 40), (40, tree.level(3).n_boxes)]:
        win = octree.tree_window(tree, *box3)
        view = octree.window_view(tree, win)
        hv = octree.build_cone_hierarchy(view)
        hd = octree.build_cone_hierarchy(view, device=True)
        for d in hv.cone_levels:
            assert np.array_equal(hv.level(d).seg_ids, hd.level(d).seg_ids)
            assert np.array_equal(hv.level(d).seg_off, hd.level(d).seg_off)


@pytest.mark.parametrize("name", ["s1", "c1", "se1", "sl1", "c2n4"])
def test_device_propagation_types_equal_host(name):
    """Propagation types (sigma groups per parent node, child rows per
    instance) from the device builder equal the host builder's integers; the
    continuous node tables agree to a few ulp (CUDA vs numpy acos/atan2)."""
    if not (GOLDEN / f"{name}.npz").exists():
        pytest.skip(f"{name} fixture not generated")
    inp = inputs(name)
    tree, host = inp["tree"], inp["hier"]
    dev = octree.build_cone_hierarchy(tree, device=True)
    for d in range(4, tree.depth + 1):
        a = octree.accumulation_plan(tree, host, d)
        b = octree.accumulation_plan(tree, dev, d)
        assert b.pending_geometry is not None
        for f in ("type_gamma", "type_octant", "sig_off", "group_sigma", "gid", "inst_off",
                  "inst_type", "inst_child", "inst_crow_off", "crow"):
            assert np.array_equal(getattr(a, f), getattr(b, f)), (d, f)
        ga, ra = octree.node_tables(a)
        gb, rb = octree.node_tables(b)
        assert np.abs(ga - gb).max() < 1e-12 and np.abs(ra - rb).max() < 1e-12 * np.abs(ra).max()
