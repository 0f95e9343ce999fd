"""Device side of the multi-GPU partition on ONE GPU: P logical ranks run
one after another (each with its own plan and partition, no collective, no
waiting between kernels); their far-field partials and output rows are
summed on the host side exactly as the NCCL all-reduces would, and the
result equals the single-GPU apply and the reference's golden output."""

import ctypes

import numpy as np
import pytest
import torch

from _support import golden, inputs, plan_matches_golden, rel
from paper_2408_02274_b200 import _lib
from paper_2408_02274_b200.engine import device_stream
from paper_2408_02274_b200.operator import MullerOperator
from paper_2408_02274_b200.partition import DistributedMullerOperator, level3_partition

pytestmark = pytest.mark.gpu


class _NoComm:
    """Stand-in for torch.distributed in the single-GPU emulation."""

    def all_reduce(self, t, group=None):
        pass


def _rank_ops(name, n_ranks):
    inp = inputs(name)
    parts = level3_partition(inp["tree"], inp["hier"], n_ranks, inp["disc"].n_patches,
                             inp["disc"].n_c)
    ops = []
    for part in parts:
        op = MullerOperator(inp["disc"], inp["mats"], inp["smap"], inp["moments"],
                            (inp["corr"].ell_idx, inp["corr"].src_idx),
                            tree=inp["tree"], hierarchy=inp["hier"])
        dop = DistributedMullerOperator(op, part)
        dop.dist = _NoComm()
        ops.append(dop)
    return ops


@pytest.mark.parametrize("name,n_ranks", [("s1", 2), ("c1", 3)])
def test_partitioned_apply_equals_single_gpu(name, n_ranks):
    z = golden(name)
    y = torch.from_numpy(z["y"]).cuda()
    ops = _rank_ops(name, n_ranks)
    lib, st = _lib.load(), device_stream()
    for o in ops:       # phase 1 on every logical rank
        _lib.check(lib.ifgfb_muller_far_phase(o.op.plan.handle, y.data_ptr(), st), "far")
    far = sum(o.far.clone() for o in ops)            # == NCCL all-reduce
    far_d = sum(o.far_disp.clone() for o in ops)
    outs = []
    for o in ops:       # phase 2
        o.far.copy_(far)
        o.far_disp.copy_(far_d)
        out = torch.zeros_like(y)
        _lib.check(lib.ifgfb_muller_near_phase(o.op.plan.handle, y.data_ptr(),
                                               out.data_ptr(), st), "near")
        outs.append(out)
    got = sum(outs).cpu().numpy()                    # == NCCL all-reduce
    single = ops[0].op.__class__(ops[0].op.disc, ops[0].op.materials, ops[0].op.smap,
                                 ops[0].op.moments, ops[0].op.corrections,
                                 tree=ops[0].op.tree, hierarchy=ops[0].op.hierarchy)
    ref1 = single.apply(z["y"])
    assert rel(got, ref1) < 1e-10
    # each rank only holds coefficient rows of its own subtrees
    assert all(o.op.plan.device_bytes() < single.plan.device_bytes() for o in ops)
    if plan_matches_golden(name):
        assert rel(got, z["apply_y"]) < 1e-10


def test_one_rank_partition_is_identity():
    z = golden("s1")
    ops = _rank_ops("s1", 1)
    y = torch.from_numpy(z["y"]).cuda()
    got = ops[0].apply_device(y).cpu().numpy()
    assert np.array_equal(got, ops[0].op.apply(z["y"]))


@pytest.mark.parametrize("name,n_parts", [("s1", 3), ("c1", 4)])
def test_streaming_equals_single_pass(name, n_parts):
    """Single-GPU streaming (sequential level-3 subtree groups, smaller
    coefficient buffers) gives the single-pass result."""
    inp, z = inputs(name), golden(name)
    args = (inp["disc"], inp["mats"], inp["smap"], inp["moments"],
            (inp["corr"].ell_idx, inp["corr"].src_idx))
    full = MullerOperator(*args, tree=inp["tree"], hierarchy=inp["hier"], stream_parts=1)
    st = MullerOperator(*args, tree=inp["tree"], hierarchy=inp["hier"],
                        stream_parts=n_parts)
    a, b = full.apply(z["y"]), st.apply(z["y"])
    assert rel(b, a) < 1e-10
    assert st.plan.device_bytes() < full.plan.device_bytes()
    if plan_matches_golden(name):
        assert rel(b, z["apply_y"]) < 1e-10
