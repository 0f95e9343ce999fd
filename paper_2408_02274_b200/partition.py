"""Multi-GPU matvec: one process per GPU, each owning a window of the
octree.

* **Far field (sources).**  Rank r owns a contiguous Morton range of level-3
  boxes and builds the plan of those subtrees only (``octree.window_view``:
  cones, propagation and emission of the window, the same integers as the
  full plan's slice).  Levels <= 2 carry no cones (reference ifgf.py:433),
  so every parent a rank needs is built from its own children: the upward
  pass needs no exchange.  Its emission covers every cousin target of its
  boxes, i.e. the rank's far field is the partial sum of its sources at all
  N targets.
* **Near field + assembly (targets).**  Rank r owns the original-order
  target rows [r*chunk, min((r+1)*chunk, N)), chunk = ceil(P/n)*n_c^2 (equal
  patch counts; the target-indexed near-field tables of reference
  quadrature.py:251-257 and :431-449 shard with them).
* **Exchange per matvec.**  One reduce-scatter (sum) of the partial far
  field, point-major 32 complex per target (8 channels x 2 kernels at x and
  at x + h n; 622 MB per rank at cfg 5), so each rank receives its target
  rows; one all-gather of the 4 result rows per target.  Source-owner
  emission moves ~700x fewer bytes than gathering coarse-level
  coefficients (SURVEY 8(e) (A) vs (B)).

The partition of level-3 boxes is balanced by a work model that needs only
the tree (every rank computes it identically before building anything).
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np

from . import _lib

__all__ = ["RankPart", "rank_targets", "level3_partition", "subtree_work",
           "subtree_work_estimate", "RankExchange", "DistributedMullerOperator"]

W_PROP = 75 * 75 * 16 * 4
W_COEF = 62_400
W_EMIT = 9_600
W_LEAF = 128 * 75
# Leaf pairs cost ~10x their 128 algorithmic FLOP relative to propagation
# instances in device time (B200, (4,10): 1.74 ms / 27.3 M pairs against
# 22.5 ms / 1.21 M instances; the sincos and the per-segment K3 + store are
# not in the FLOP count), so the balance weights a pair at 10 W_LEAF.
W_LEAF_TIME = 10 * W_LEAF


@dataclass
class RankPart:
    rank: int
    n_ranks: int
    box3: tuple                 # owned level-3 boxes [lo, hi): far-field sources
    targets: tuple              # owned original-order targets [lo, hi)
    chunk: int                  # exchange rows per rank (targets padded)
    work: float                 # modelled cost of the owned upward pass
    levels: dict | None = None  # d -> dict(box, seg, pair) (full hierarchy only)


def rank_targets(n_patches: int, n_c: int, n_ranks: int):
    """Equal patch counts per rank (the last one shorter): (chunk, ranges)."""
    n2 = n_c * n_c
    per = -(-n_patches // n_ranks)
    chunk = per * n2
    n = n_patches * n2
    return chunk, [(min(r * chunk, n), min((r + 1) * chunk, n)) for r in range(n_ranks)]


def _level3_ancestor(tree, d):
    from .octree import level3_ancestors
    return level3_ancestors(tree, d)


def subtree_work(tree, hier) -> np.ndarray:
    """Modelled cost (FLOP-equivalents, time-calibrated leaf weight) of the
    upward pass attributed to each level-3 box, from a full hierarchy."""
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


def subtree_work_estimate(tree, config=None) -> np.ndarray:
    """The same model without a cone hierarchy (each rank must partition
    before it builds its window): a box's relevant segments are estimated
    from its cousin points, capped by the level's segment count, and every
    child inherits its parent's estimate as propagation instances."""
    from .octree import IfgfConfig, cone_counts
    config = config or IfgfConfig()
    counts = cone_counts(tree, config)
    n3 = tree.level(3).n_boxes
    work = np.zeros(n3)
    D = tree.depth
    seg_est = {}
    for d in range(3, D + 1):
        lvl = tree.level(d)
        n_s, n_a = counts[d]
        full = n_s * n_a * 2 * n_a
        czo = lvl.cousin_off
        cz = lvl.cousin_idx
        cpt_cz = lvl.pt_count[cz]
        cpt = np.add.reduceat(cpt_cz, czo[:-1]) if cz.size else np.zeros(lvl.n_boxes)
        cpt = np.where(np.diff(czo) > 0, cpt, 0)
        est = np.minimum(full, cpt + (np.diff(czo) > 0) * 0.25 * full)
        if d > 3:
            est = np.maximum(est, np.minimum(full, seg_est[d - 1][lvl.parent]))
        seg_est[d] = est
        w = W_EMIT * cpt + W_COEF * est
        if d == D:
            w = w + W_LEAF_TIME * est * lvl.pt_count
        if d >= 4:
            w = w + W_PROP * seg_est[d - 1][lvl.parent]
        np.add.at(work, _level3_ancestor(tree, d), w)
    return work


def _cuts(work: np.ndarray, n_ranks: int) -> list:
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
    return list(np.maximum.accumulate(np.minimum(cuts, work.size)))


def level3_partition(tree, hier, n_ranks: int, n_patches: int, n_c: int,
                     work: np.ndarray | None = None) -> list:
    """Balanced contiguous level-3 ranges (sources) and equal patch ranges
    (targets) for n_ranks.  hier=None: tree-only work estimate (what the
    ranks use); with a full hierarchy the exact model and the per-level
    segment / pair ranges of each rank (single-GPU streaming)."""
    if tree.depth < 3:
        raise ValueError("no cone levels: nothing to partition")
    if work is None:
        work = subtree_work(tree, hier) if hier is not None else subtree_work_estimate(tree)
    cuts = _cuts(work, n_ranks)
    chunk, tranges = rank_targets(n_patches, n_c, n_ranks)
    parts = []
    for r in range(n_ranks):
        b3 = (int(cuts[r]), int(cuts[r + 1]))
        levels = None
        if hier is not None:
            levels = {}
            for d in range(3, tree.depth + 1):
                anc = _level3_ancestor(tree, d)
                lo = int(np.searchsorted(anc, b3[0], side="left"))
                hi = int(np.searchsorted(anc, b3[1], side="left"))
                cl = hier.level(d)
                levels[d] = dict(box=(lo, hi),
                                 seg=(int(cl.seg_off[lo]), int(cl.seg_off[hi])),
                                 pair=(int(cl.cpt_off[lo]), int(cl.cpt_off[hi])))
        parts.append(RankPart(r, n_ranks, b3, tranges[r], chunk,
                              float(work[b3[0]:b3[1]].sum()), levels))
    return parts


class _CudaView:
    """Expose a raw device buffer to torch through __cuda_array_interface__."""

    def __init__(self, ptr: int, n_double: int):
        self.__cuda_array_interface__ = {
            "shape": (n_double,), "typestr": "<f8", "data": (ptr, False),
            "version": 3, "strides": None}


class RankExchange:
    """The two collectives of a matvec over a torch.distributed group.
    NCCL: reduce_scatter_tensor / all_gather_into_tensor on the device
    buffers (NVLink).  gloo (CPU tests; several ranks sharing one GPU): the
    same reductions through host copies (gloo has no reduce-scatter, so an
    all-reduce is sliced: identical sums)."""

    def __init__(self, group=None):
        import torch.distributed as dist
        self.dist, self.group = dist, group
        self.rank = dist.get_rank(group)
        self.size = dist.get_world_size(group)
        self.nccl = dist.get_backend(group) == "nccl"

    def reduce_scatter(self, full, mine):
        if self.nccl:
            self.dist.reduce_scatter_tensor(mine, full, group=self.group)
            return
        t = full.cpu()
        self.dist.all_reduce(t, group=self.group)
        c = mine.numel()
        mine.copy_(t[self.rank * c:(self.rank + 1) * c])

    def all_gather(self, full, mine):
        if self.nccl:
            self.dist.all_gather_into_tensor(full, mine, group=self.group)
            return
        import torch
        parts = [torch.empty(mine.numel(), dtype=mine.dtype) for _ in range(self.size)]
        self.dist.all_gather(parts, mine.cpu(), group=self.group)
        full.copy_(torch.cat(parts))


class DistributedMullerOperator:
    """One rank's share of the N-Muller matvec (one process per GPU).

    Builds, on this rank only, the far-field plan of its window of level-3
    subtrees and the near-field plan of its target rows, then per apply:
    far phase (partial sums) -> reduce-scatter -> near phase (owned rows) ->
    all-gather -> unpack.  ``apply_device`` returns the full 4N result on
    every rank (GMRES runs replicated on top of it)."""

    def __init__(self, disc, materials, part: RankPart, tree=None, group=None,
                 exchange=None, quad_config=None, device_moments: bool = True,
                 config=None, stream_parts=None, geometry_on_device=None,
                 seam: str = "unwrap", moments=None, smap=None,
                 device_plan: bool = False):
        import torch
        from . import nearfield, octree
        from .operator import MullerOperator, OperatorConfig
        self.disc, self.materials, self.part = disc, materials, part
        kmax = max(abs(materials.kappa_e), abs(materials.kappa_i))
        self.tree = tree if tree is not None else octree.build_box_tree(disc.points, kmax)
        self.window = octree.tree_window(self.tree, *part.box3)
        self.view = octree.window_view(self.tree, self.window)
        self.hier = octree.build_cone_hierarchy(self.view, device=device_plan)
        qc = quad_config or nearfield.SingularQuadratureConfig()
        t0, t1 = part.targets
        if smap is None:
            smap = nearfield.classify_targets(disc, qc, target_range=(t0, t1))
        if moments is None:
            kw = dict(target_points=disc.points[t0:t1], target_normals=disc.normals[t0:t1])
            moments = (nearfield.compute_moments_device(disc, smap, qc, materials.kappas,
                                                        groups=False, **kw)
                       if device_moments else
                       nearfield.compute_moments(disc, smap, qc, materials.kappas, **kw))
        cp = nearfield.correction_pairs(disc, self.tree, smap)
        self.op = MullerOperator(disc, materials, smap, moments, (cp.ell_idx, cp.src_idx),
                                 config or OperatorConfig(), tree=self.view,
                                 hierarchy=self.hier, near_tree=self.tree,
                                 stream_parts=stream_parts,
                                 geometry_on_device=geometry_on_device, seam=seam)
        lib = _lib.load()
        desc = _lib.RankDesc(t0, t1, part.chunk, part.rank, part.n_ranks)
        _lib.check(lib.ifgfb_plan_set_rank(self.op.plan.handle, ctypes.byref(desc)),
                   "ifgfb_plan_set_rank")
        ptrs = [ctypes.c_void_p() for _ in range(4)]
        chunk = ctypes.c_int64()
        _lib.check(lib.ifgfb_plan_rank_buffers(self.op.plan.handle, *ptrs, chunk),
                   "ifgfb_plan_rank_buffers")
        rows = part.n_ranks * part.chunk
        sizes = (rows * 64, part.chunk * 64, part.chunk * 8, rows * 8)   # doubles
        self.xfar, self.xfar_mine, self.xout_mine, self.xout = (
            torch.as_tensor(_CudaView(p.value, n), device="cuda")
            for p, n in zip(ptrs, sizes))
        self.exchange = exchange if exchange is not None else RankExchange(group)

    @property
    def n_unknowns(self):
        return self.op.n_unknowns

    @property
    def plan(self):
        return self.op.plan

    def far_phase(self, y):
        from .engine import device_stream
        _lib.check(_lib.load().ifgfb_muller_far_phase(self.op.plan.handle, y.data_ptr(),
                                                      device_stream()),
                   "ifgfb_muller_far_phase")

    def near_phase(self, y):
        from .engine import device_stream
        _lib.check(_lib.load().ifgfb_muller_near_phase(self.op.plan.handle, y.data_ptr(),
                                                       None, device_stream()),
                   "ifgfb_muller_near_phase")

    def unpack(self, out):
        from .engine import device_stream
        _lib.check(_lib.load().ifgfb_rank_unpack(self.op.plan.handle, out.data_ptr(),
                                                 device_stream()), "ifgfb_rank_unpack")

    def apply_device(self, y, out=None):
        import torch
        y = y.contiguous()
        if y.numel() != self.n_unknowns:
            raise ValueError("unknown vector has wrong length")
        if out is None:
            out = torch.empty_like(y)
        self.far_phase(y)
        self.exchange.reduce_scatter(self.xfar, self.xfar_mine)
        self.near_phase(y)
        self.exchange.all_gather(self.xout, self.xout_mine)
        self.unpack(out)
        return out

    def apply(self, y) -> np.ndarray:
        import torch
        yd = torch.from_numpy(np.ascontiguousarray(np.asarray(y, dtype=complex))).cuda()
        return self.apply_device(yd).cpu().numpy()

    def last_launches(self) -> int:
        return self.op.last_launches()

    def device_bytes(self) -> int:
        return self.op.plan.device_bytes()
