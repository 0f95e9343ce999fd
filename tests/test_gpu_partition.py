"""Device side of the multi-GPU matvec on ONE GPU.

* P logical ranks run one after another in one process, each with its own
  windowed plan (its level-3 subtrees) and target rows; the reduce-scatter
  and all-gather are emulated by summing / slicing the exchange buffers
  (no collective, nothing waits on another rank).  The result equals the
  single-GPU apply and the reference's golden output.
* Two processes (both on cuda:0) drive ``DistributedMullerOperator``
  end to end through ``RankExchange`` on the gloo backend (host copies; the
  NCCL path differs only in the collective calls)."""

import os
import socket

import numpy as np
import pytest
import torch

from _support import golden, inputs, plan_matches_golden, rel
from paper_2408_02274_b200.operator import MullerOperator
from paper_2408_02274_b200.partition import DistributedMullerOperator, level3_partition

pytestmark = pytest.mark.gpu


def _single_op(name):
    inp = inputs(name)
    return MullerOperator(inp["disc"], inp["mats"], inp["smap"], inp["moments"],
                          (inp["corr"].ell_idx, inp["corr"].src_idx),
                          tree=inp["tree"], hierarchy=inp["hier"])


def _rank_ops(name, n_ranks, exact_partition=False):
    inp = inputs(name)
    parts = level3_partition(inp["tree"], inp["hier"] if exact_partition else None,
                             n_ranks, inp["disc"].n_patches, inp["disc"].n_c)
    return [DistributedMullerOperator(inp["disc"], inp["mats"], part, tree=inp["tree"],
                                      exchange=False, device_moments=False)
            for part in parts]


def _emulated_apply(ops, y):
    """The exchange of a matvec, emulated on one GPU: sum of the partial
    far rows (reduce-scatter) and concatenation of the result rows
    (all-gather)."""
    for o in ops:
        o.far_phase(y)
    full = sum(o.xfar.clone() for o in ops)
    for o in ops:
        c = o.xfar_mine.numel()
        o.xfar_mine.copy_(full[o.part.rank * c:(o.part.rank + 1) * c])
        o.near_phase(y)
    gathered = torch.cat([o.xout_mine.clone() for o in ops])
    out = torch.empty_like(y)
    ops[0].xout.copy_(gathered)
    ops[0].unpack(out)
    return out


@pytest.mark.parametrize("name,n_ranks", [("s1", 2), ("c1", 3), ("c1", 8)])
def test_rank_plans_reproduce_single_gpu(name, n_ranks):
    z = golden(name)
    y = torch.from_numpy(z["y"]).cuda()
    ops = _rank_ops(name, n_ranks)
    got = _emulated_apply(ops, y).cpu().numpy()
    single = _single_op(name)
    assert rel(got, single.apply(z["y"])) < 1e-10
    # each rank holds its own subtrees' plan and its own near-field rows
    assert all(o.device_bytes() < single.plan.device_bytes() for o in ops)
    if plan_matches_golden(name):
        assert rel(got, z["apply_y"]) < 1e-10


def test_one_rank_is_bitwise_single_gpu():
    z = golden("s1")
    ops = _rank_ops("s1", 1)
    y = torch.from_numpy(z["y"]).cuda()
    got = _emulated_apply(ops, y).cpu().numpy()
    assert np.array_equal(got, _single_op("s1").apply(z["y"]))


def test_rank_plan_rejects_whole_plan_entry_points():
    """A rank plan holds partial sums: the single-GPU entry points refuse it
    instead of returning partial results."""
    z = golden("s1")
    op = _rank_ops("s1", 2)[0].op
    with pytest.raises(RuntimeError, match="rank"):
        op.apply(z["y"])
    with pytest.raises(RuntimeError, match="rank"):
        op.apply_device(torch.from_numpy(z["y"]).cuda())


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


def test_rank_plan_with_streaming():
    """A rank's window streamed in parts (cfg-5 ranks stream too)."""
    z = golden("c1")
    inp = inputs("c1")
    part = level3_partition(inp["tree"], None, 2, inp["disc"].n_patches, inp["disc"].n_c)
    ops = [DistributedMullerOperator(inp["disc"], inp["mats"], p, tree=inp["tree"],
                                     exchange=False, device_moments=False, stream_parts=3)
           for p in part]
    y = torch.from_numpy(z["y"]).cuda()
    assert rel(_emulated_apply(ops, y).cpu().numpy(), _single_op("c1").apply(z["y"])) < 1e-10


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _two_rank_main(rank, world, port, result_path):
    import torch.distributed as dist
    os.environ["OMP_NUM_THREADS"] = "2"
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}",
                            rank=rank, world_size=world)
    z, inp = golden("c1"), inputs("c1")
    part = level3_partition(inp["tree"], None, world, inp["disc"].n_patches,
                            inp["disc"].n_c)[rank]
    op = DistributedMullerOperator(inp["disc"], inp["mats"], part, device_moments=False)
    out = op.apply(z["y"])
    torch.cuda.synchronize()
    np.save(f"{result_path}.{rank}.npy", out)
    dist.barrier()
    dist.destroy_process_group()


def test_two_process_distributed_operator_gloo(tmp_path):
    import torch.multiprocessing as mp
    res = str(tmp_path / "out")
    mp.spawn(_two_rank_main, args=(2, _free_port(), res), nprocs=2, join=True)
    a, b = np.load(res + ".0.npy"), np.load(res + ".1.npy")
    assert np.array_equal(a, b)          # every rank holds the full result
    ref = _single_op("c1").apply(golden("c1")["y"])
    assert rel(a, ref) < 1e-10
    if plan_matches_golden("c1"):
        assert rel(a, golden("c1")["apply_y"]) < 1e-10
