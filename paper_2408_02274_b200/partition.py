"""Multi-GPU partition of the IFGF N-Muller matvec.

Upward pass (leaf spectra, propagation, emission): contiguous Morton ranges
of level-3 boxes per rank, balanced by modelled subtree work.  Levels <= 2
carry no cone segments (reference ifgf.py:433), so every parent a rank
needs is computed from its own children: no exchange until the far-field
outputs, which are summed over ranks (each (source box, target) pair is
emitted by exactly one rank).  Near field and assembly: contiguous patch
ranges (original point order), rows summed over ranks (each row written by
one rank, zeros elsewhere: the sum is exact).

Per matvec traffic per rank: one all-reduce of 2 x 16 x N complex (far
field and its displaced copy) and one of 4 N complex (the result).
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np

from . import _lib

__all__ = ["RankPart", "level3_partition", "DistributedMullerOperator"]

W_PROP = 75 * 75 * 16 * 4
W_COEF = 62_400
W_EMIT = 9_600
W_LEAF = 128 * 75


@dataclass
class RankPart:
    rank: int
    box3: tuple                 # owned level-3 box range [lo, hi)
    levels: dict                # d -> dict(box=(lo,hi), seg=(lo,hi), pair=(lo,hi))
    targets: tuple              # owned original-order target range [lo, hi)
    work: float                 # modelled FLOP of the owned upward pass


def _level3_ancestor(tree, d):
    codes3 = tree.level(3).codes
    return np.searchsorted(codes3, tree.level(d).codes >> np.uint64(3 * (d - 3)))


# Leaf pairs cost ~10x their 128 algorithmic FLOP relative to propagation
# instances in device time (B200, (4,10): 1.74 ms / 27.3 M pairs against
# 22.5 ms / 1.21 M instances; the sincos and the per-segment K3 + store are
# not in the FLOP count), so the balance weights a pair at 10 W_LEAF.
W_LEAF_TIME = 10 * W_LEAF


def subtree_work(tree, hier) -> np.ndarray:
    """Modelled cost (FLOP-equivalents, time-calibrated leaf weight) of the
    upward pass attributed to each level-3 box."""
    n3 = tree.level(3).n_boxes
    work = np.zeros(n3)
    D = tree.depth
    for d in range(3, D + 1):
        cl, lvl = hier.level(d), tree.level(d)
        anc = _level3_ancestor(tree, d)
        w = W_EMIT * np.diff(cl.cpt_off) + W_COEF * np.diff(cl.seg_off)
        if d == D:
            w = w + W_LEAF_TIME * np.diff(cl.seg_off) * lvl.pt_count
        if d >= 4:
            pcl = hier.level(d - 1)
            w = w + W_PROP * np.diff(pcl.seg_off)[lvl.parent]
        np.add.at(work, anc, w)
    return work


def level3_partition(tree, hier, n_ranks: int, n_patches: int,
                     n_c: int) -> list:
    """Balanced contiguous level-3 ranges and patch ranges for n_ranks."""
    if tree.depth < 3:
        raise ValueError("no cone levels: nothing to partition")
    work = subtree_work(tree, hier)
    cum = np.concatenate([[0.0], np.cumsum(work)])
    total = cum[-1]
    cuts = [0]
    for r in range(1, n_ranks):
        target = total * r / n_ranks
        i = int(np.searchsorted(cum, target))      # first boundary >= target
        if 0 < i <= work.size and target - cum[i - 1] < cum[i] - target:
            i -= 1                                  # the nearer boundary
        cuts.append(i)
    cuts.append(work.size)
    cuts = np.maximum.accumulate(np.minimum(cuts, work.size))
    n2 = n_c * n_c
    pcuts = [(n_patches * r) // n_ranks for r in range(n_ranks + 1)]
    parts = []
    for r in range(n_ranks):
        b3 = (int(cuts[r]), int(cuts[r + 1]))
        levels = {}
        for d in range(3, tree.depth + 1):
            anc = _level3_ancestor(tree, d)
            lo = int(np.searchsorted(anc, b3[0], side="left"))
            hi = int(np.searchsorted(anc, b3[1], side="left"))
            cl = hier.level(d)
            levels[d] = dict(box=(lo, hi),
                             seg=(int(cl.seg_off[lo]), int(cl.seg_off[hi])),
                             pair=(int(cl.cpt_off[lo]), int(cl.cpt_off[hi])))
        parts.append(RankPart(r, b3, levels, (pcuts[r] * n2, pcuts[r + 1] * n2),
                              float(work[b3[0]:b3[1]].sum())))
    return parts


class _CudaView:
    """Expose a raw device buffer to torch through __cuda_array_interface__."""

    def __init__(self, ptr: int, n_complex: int):
        self.__cuda_array_interface__ = {
            "shape": (n_complex,), "typestr": "<c16", "data": (ptr, False),
            "version": 3, "strides": None}


class DistributedMullerOperator:
    """One rank of the partitioned matvec: wraps this rank's MullerOperator
    (full plan on its GPU) and a torch.distributed process group (NCCL)."""

    def __init__(self, op, part: RankPart, group=None):
        import torch
        import torch.distributed as dist
        self.op, self.part, self.group = op, part, group
        self.dist = dist
        lib = _lib.load()
        depth = op.tree.depth
        lv = (_lib.LevelPart * max(0, depth - 2))()
        for i, d in enumerate(range(3, depth + 1)):
            L = part.levels[d]
            lv[i] = _lib.LevelPart(d, L["seg"][0], L["seg"][1], L["pair"][0],
                                   L["pair"][1])
        desc = _lib.PartitionDesc(depth - 2, lv, part.targets[0], part.targets[1])
        _lib.check(lib.ifgfb_plan_set_partition(op.plan.handle, desc),
                   "ifgfb_plan_set_partition")
        far, far_d = ctypes.c_void_p(), ctypes.c_void_p()
        n = ctypes.c_int64()
        _lib.check(lib.ifgfb_plan_far_buffers(op.plan.handle, far, far_d, n),
                   "ifgfb_plan_far_buffers")
        self.far = torch.as_tensor(_CudaView(far.value, n.value), device="cuda")
        self.far_disp = torch.as_tensor(_CudaView(far_d.value, n.value),
                                        device="cuda")

    @property
    def n_unknowns(self):
        return self.op.n_unknowns

    def apply_device(self, y, out=None):
        import torch
        from .engine import device_stream
        lib = _lib.load()
        y = y.contiguous()
        if out is None:
            out = torch.empty_like(y)
        st = device_stream()
        _lib.check(lib.ifgfb_muller_far_phase(self.op.plan.handle, y.data_ptr(), st),
                   "ifgfb_muller_far_phase")
        self.dist.all_reduce(self.far, group=self.group)
        self.dist.all_reduce(self.far_disp, group=self.group)
        out.zero_()
        _lib.check(lib.ifgfb_muller_near_phase(self.op.plan.handle, y.data_ptr(),
                                               out.data_ptr(), st),
                   "ifgfb_muller_near_phase")
        self.dist.all_reduce(out, group=self.group)
        return out

    def last_launches(self) -> int:
        return self.op.last_launches()
