"""Drop-in host path on the REFERENCE's own plan objects (build container
only: skipped when /root/reference is absent, e.g. on the GPU hosts).

``from_reference`` feeds the reference's BoxTree / ConeHierarchy /
SingularityMap / moment table / CorrectionSet to the same device-plan
flattening the framework uses for its own objects; this checks that the
flattened arrays are identical either way."""

import sys
from pathlib import Path

import numpy as np
import pytest

from _support import inputs
from paper_2408_02274_b200 import octree
from paper_2408_02274_b200.operator import _near_desc

REF = Path("/root/reference/pkg/src")
pytestmark = pytest.mark.skipif(not REF.exists(), reason="reference not mounted")


@pytest.fixture(scope="module")
def ref_op():
    sys.path.insert(0, str(REF))
    import emscat.geometry as rg
    from emscat.operators import MaterialPair, build_muller_operator
    op = build_muller_operator(rg.make_sphere_surface(1, 10),
                               MaterialPair(1.0, 1.0, 2.25, 1.0, 2 * np.pi))
    op.apply(np.ones(op.n_unknowns, complex))    # fills the reference's caches
    return op


def test_accumulation_and_emission_plans_from_reference_objects(ref_op):
    mine = inputs("s1")
    disp_r = ref_op.tree.points + 1e-6 * ref_op.disc.normals[ref_op.tree.perm]
    disp_m = mine["tree"].points + 1e-6 * mine["disc"].normals[mine["tree"].perm]
    for d in range(4, ref_op.tree.depth + 1):
        a = octree.accumulation_plan(ref_op.tree, ref_op.hierarchy, d)
        b = octree.accumulation_plan(mine["tree"], mine["hier"], d)
        for f in ("sig_off", "group_bounds", "group_end", "group_sigma", "scatter",
                  "xs", "xt", "xp", "r_parent", "r_child", "inst_off", "inst_type",
                  "inst_child", "inst_crow_off", "crow"):
            assert np.array_equal(getattr(a, f), getattr(b, f)), (d, f)
        for x, y in zip(octree.row_tiles(a), octree.row_tiles(b)):
            assert np.array_equal(x, y)
    for d in range(3, ref_op.tree.depth + 1):
        a = octree.emission_plan(ref_op.tree, ref_op.hierarchy, d, disp_r)
        b = octree.emission_plan(mine["tree"], mine["hier"], d, disp_m)
        for f in ("row", "target", "geom", "geom_disp"):
            assert np.array_equal(getattr(a, f), getattr(b, f)), (d, f)


def test_near_field_descriptor_from_reference_objects(ref_op):
    mine = inputs("s1")
    cs = ref_op.moments.corrections
    ka, kb = [], []
    _near_desc(ref_op.disc, ref_op.tree, ref_op.smap, ref_op.moments,
               cs.ell_idx, cs.src_idx, ka)
    _near_desc(mine["disc"], mine["tree"], mine["smap"], mine["moments"],
               mine["corr"].ell_idx, mine["corr"].src_idx, kb)
    assert len(ka) == len(kb)
    for x, y in zip(ka, kb):
        assert np.array_equal(x, y)
