"""IFGF plan: linear octree, cone-segment hierarchy, propagation types and
emission geometry (host, plan time; vectorised numpy).

Every integer the device consumes (Morton codes, neighbour/cousin lists,
relevant segment ids, accumulation sigma/rows, emission segment rows) is
produced here with the *same floating-point expressions* the reference uses,
so it is bit-identical to the reference plan on the same host (checked by
``tests/test_plan_vs_reference.py`` against golden digests):

* Morton codes                 -- reference ``ifgf.py:70-102``
* ``build_box_tree``           -- reference ``ifgf.py:176-277``
* ``cone_coords``              -- reference ``ifgf.py:305-317``
* ``ConeLevel``                -- reference ``ifgf.py:324-387``
* ``build_cone_hierarchy``     -- reference ``ifgf.py:417-482``
* ``accumulation_plan``        -- reference ``ifgf.py:676-749`` (_AccumType,
  _accum_types) regrouped per parent segment for owner-computes on device
* ``emission_plan``            -- reference ``ifgf.py:630-673`` geometry part
  (segment row, local coordinates, radii of x and x + h n)

Unlike the reference (Python loops over boxes and types), every stage here
is a handful of whole-level array operations.
"""

from __future__ import annotations

import json
from dataclasses import dataclass, field
from functools import cached_property

import numpy as np

from . import cheb

__all__ = ["ETA", "IfgfConfig", "BoxTree", "LevelBoxes", "ConeLevel",
           "ConeHierarchy", "morton_encode", "morton_decode",
           "build_box_tree", "build_cone_hierarchy", "cone_coords",
           "accumulation_plan", "emission_plan", "tree_stats", "TreeWindow",
           "tree_window", "window_view", "level3_ancestors", "level_tables"]

ETA = np.sqrt(3.0) / 3.0


@dataclass(frozen=True)
class IfgfConfig:
    """Interpolation orders and cone seeds (reference ``ifgf.py:49-63``)."""

    p_s: int = 3
    p_a: int = 5
    n_s_seed: int = 1
    n_a_seed: int = 2
    mode: str = "vec"

    def __post_init__(self):
        if self.p_s < 2 or self.p_a < 2:
            raise ValueError("interpolation orders must be >= 2")
        if self.mode not in ("vec", "seq"):
            raise ValueError("mode must be 'vec' or 'seq'")

    @property
    def n_nodes(self) -> int:
        return self.p_s * self.p_a * self.p_a


# ---------------------------------------------------------------------------
# Morton codes (x -> bit 2, y -> bit 1, z -> bit 0; 21 bits per axis)
# ---------------------------------------------------------------------------

_SPREAD = ((32, 0x1F00000000FFFF), (16, 0x1F0000FF0000FF),
           (8, 0x100F00F00F00F00F), (4, 0x10C30C30C30C30C3),
           (2, 0x1249249249249249))


def _spread3(x):
    x = np.asarray(x).astype(np.uint64) & np.uint64(0x1FFFFF)
    for sh, mask in _SPREAD:
        x = (x | (x << np.uint64(sh))) & np.uint64(mask)
    return x


def _gather3(x):
    x = np.asarray(x).astype(np.uint64) & np.uint64(0x1249249249249249)
    for sh, mask in ((2, 0x10C30C30C30C30C3), (4, 0x100F00F00F00F00F),
                     (8, 0x1F0000FF0000FF), (16, 0x1F00000000FFFF),
                     (32, 0x1FFFFF)):
        x = (x | (x >> np.uint64(sh))) & np.uint64(mask)
    return x


def morton_encode(coords) -> np.ndarray:
    c = np.asarray(coords, dtype=np.uint64)
    return ((_spread3(c[..., 0]) << np.uint64(2)) |
            (_spread3(c[..., 1]) << np.uint64(1)) | _spread3(c[..., 2]))


def morton_decode(codes) -> np.ndarray:
    codes = np.asarray(codes, dtype=np.uint64)
    return np.stack([_gather3(codes >> np.uint64(2)),
                     _gather3(codes >> np.uint64(1)),
                     _gather3(codes)], axis=-1).astype(np.int64)


# ---------------------------------------------------------------------------
# CSR helpers
# ---------------------------------------------------------------------------

def _expand_ranges(lo: np.ndarray, hi: np.ndarray):
    """Concatenate [lo_i, hi_i) ranges -> (values, owner index i)."""
    lo = np.asarray(lo, dtype=np.int64)
    cnt = np.asarray(hi, dtype=np.int64) - lo
    owner = np.repeat(np.arange(lo.size, dtype=np.int64), cnt)
    if owner.size == 0:
        return np.empty(0, np.int64), owner
    starts = np.cumsum(cnt) - cnt
    vals = np.arange(owner.size, dtype=np.int64) - starts[owner] + lo[owner]
    return vals, owner


def _offsets_from_owner(owner: np.ndarray, n: int) -> np.ndarray:
    off = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(np.bincount(owner, minlength=n), out=off[1:])
    return off


# ---------------------------------------------------------------------------
# box tree
# ---------------------------------------------------------------------------

@dataclass
class LevelBoxes:
    level: int
    side: float
    codes: np.ndarray
    coords: np.ndarray
    centers: np.ndarray
    pt_start: np.ndarray
    pt_count: np.ndarray
    parent: np.ndarray
    child_start: np.ndarray
    child_end: np.ndarray
    nbr_idx: np.ndarray
    nbr_off: np.ndarray
    cousin_idx: np.ndarray
    cousin_off: np.ndarray
    box_lo: int = 0               # window views: global id of local box 0
    full: "LevelBoxes | None" = None   # window views: the whole level

    @property
    def n_boxes(self) -> int:
        return self.codes.size

    def neighbors(self, b: int) -> np.ndarray:
        return self.nbr_idx[self.nbr_off[b]:self.nbr_off[b + 1]]

    def cousins(self, b: int) -> np.ndarray:
        return self.cousin_idx[self.cousin_off[b]:self.cousin_off[b + 1]]


@dataclass
class BoxTree:
    origin: np.ndarray
    root_side: float
    depth: int
    kappa_max: float
    perm: np.ndarray
    iperm: np.ndarray
    points: np.ndarray
    point_codes: np.ndarray
    levels: list = field(default_factory=list)

    def level(self, d: int) -> LevelBoxes:
        return self.levels[d - 1]

    def side(self, d: int) -> float:
        return self.root_side / 2 ** (d - 1)

    def point_level_codes(self, d: int) -> np.ndarray:
        return self.point_codes >> np.uint64(3 * (self.depth - d))

    def point_level_coords(self, d: int) -> np.ndarray:
        return morton_decode(self.point_level_codes(d))[self.iperm]

    def point_boxes(self, d: int) -> np.ndarray:
        return np.searchsorted(self.level(d).codes, self.point_level_codes(d))

    def box_points(self, d: int, b: int) -> np.ndarray:
        lvl = self.level(d)
        return np.arange(lvl.pt_start[b], lvl.pt_start[b] + lvl.pt_count[b])


_STENCIL = np.array(np.meshgrid(*[[-1, 0, 1]] * 3, indexing="ij")
                    ).reshape(3, -1).T


def build_box_tree(points, kappa_max: float, padding: float = 0.01) -> BoxTree:
    """Octree over the points; depth minimal with finest side <= lambda/4."""
    pts = np.atleast_2d(np.asarray(points, dtype=float))
    if pts.shape[0] == 0:
        raise ValueError("empty point set")
    kappa_max = float(abs(kappa_max))
    lo, hi = pts.min(axis=0), pts.max(axis=0)
    extent = max((hi - lo).max(), 1e-300)
    side = extent * (1.0 + padding)
    origin = 0.5 * (lo + hi) - side / 2.0
    quarter = 0.25 * (2 * np.pi / kappa_max) if kappa_max > 0 else np.inf
    depth = 1
    while side / 2 ** (depth - 1) > quarter:
        depth += 1
    h_fine = side / 2 ** (depth - 1)
    cells = np.clip(((pts - origin) / h_fine).astype(np.int64), 0,
                    2 ** (depth - 1) - 1)
    codes = morton_encode(cells)
    perm = np.argsort(codes, kind="stable")
    iperm = np.empty_like(perm)
    iperm[perm] = np.arange(perm.size)
    tree = BoxTree(origin, side, depth, kappa_max, perm, iperm, pts[perm],
                   codes[perm])
    for d in range(1, depth + 1):
        pc = tree.point_level_codes(d)
        bcodes, starts, counts = np.unique(pc, return_index=True,
                                           return_counts=True)
        coords = morton_decode(bcodes)
        h = tree.side(d)
        nb = bcodes.size
        cand = coords[:, None, :] + _STENCIL[None, :, :]
        valid = np.all((cand >= 0) & (cand < 2 ** (d - 1)), axis=-1)
        ccodes = morton_encode(np.clip(cand, 0, None))
        pos = np.minimum(np.searchsorted(bcodes, ccodes), nb - 1)
        hit = valid & (bcodes[pos] == ccodes)
        nbr_off = np.zeros(nb + 1, dtype=np.int64)
        nbr_off[1:] = np.cumsum(hit.sum(axis=1))
        if d == 1:
            parent = np.full(nb, -1, dtype=np.int64)
        else:
            up = tree.level(d - 1)
            shifted = bcodes >> np.uint64(3)
            parent = np.searchsorted(up.codes, shifted)
            up.child_start = np.searchsorted(shifted, up.codes, side="left")
            up.child_end = np.searchsorted(shifted, up.codes, side="right")
        tree.levels.append(LevelBoxes(
            level=d, side=h, codes=bcodes, coords=coords,
            centers=origin + (coords + 0.5) * h, pt_start=starts,
            pt_count=counts, parent=parent,
            child_start=np.zeros(nb, dtype=np.int64),
            child_end=np.zeros(nb, dtype=np.int64),
            nbr_idx=pos[hit], nbr_off=nbr_off,
            cousin_idx=np.empty(0, dtype=np.int64),
            cousin_off=np.zeros(nb + 1, dtype=np.int64)))
    # cousins: children of the parent's neighbours that are not neighbours
    # (sorted ascending per box)
    for d in range(2, depth + 1):
        lvl, up = tree.level(d), tree.level(d - 1)
        pn, owner = _expand_ranges(up.nbr_off[lvl.parent],
                                   up.nbr_off[lvl.parent + 1])
        pn = up.nbr_idx[pn]
        kids, k_own = _expand_ranges(up.child_start[pn], up.child_end[pn])
        box = owner[k_own]
        far = np.abs(lvl.coords[kids] - lvl.coords[box]).max(axis=1) >= 2
        kids, box = kids[far], box[far]
        order = np.lexsort((kids, box))
        lvl.cousin_idx = kids[order]
        lvl.cousin_off = _offsets_from_owner(box, lvl.n_boxes)
    return tree


# ---------------------------------------------------------------------------
# windows: Morton ranges of level-3 subtrees (multi-GPU ranks, streaming)
# ---------------------------------------------------------------------------

@dataclass
class TreeWindow:
    """Level-3 boxes [box3[0], box3[1]) and their subtrees: per level d >= 3
    the contiguous global box range ``ranges[d]`` (Morton order keeps every
    subtree contiguous)."""

    box3: tuple
    ranges: dict


def level3_ancestors(tree: BoxTree, d: int) -> np.ndarray:
    """Level-3 ancestor (index into level 3) of every box at level d."""
    return np.searchsorted(tree.level(3).codes,
                           tree.level(d).codes >> np.uint64(3 * (d - 3)))


def tree_window(tree: BoxTree, box3_lo: int, box3_hi: int) -> TreeWindow:
    if tree.depth < 3:
        raise ValueError("no cone levels: nothing to window")
    n3 = tree.level(3).n_boxes
    if not 0 <= box3_lo <= box3_hi <= n3:
        raise ValueError("level-3 box range out of bounds")
    ranges = {}
    for d in range(3, tree.depth + 1):
        anc = level3_ancestors(tree, d)
        ranges[d] = (int(np.searchsorted(anc, box3_lo, side="left")),
                     int(np.searchsorted(anc, box3_hi, side="left")))
    return TreeWindow((int(box3_lo), int(box3_hi)), ranges)


def _slice_csr(idx, off, lo, hi):
    return idx[off[lo]:off[hi]], off[lo:hi + 1] - off[lo]


def window_view(tree: BoxTree, win: TreeWindow) -> BoxTree:
    """The tree restricted to a window's subtrees: levels >= 3 sliced to
    their box ranges with LOCAL box ids (parent / child links re-based,
    ``box_lo`` and ``full`` kept); neighbour / cousin lists keep GLOBAL box
    ids; points, permutation and codes are shared.  Every plan builder
    (cones, propagation, emission, device upload) runs on a view unchanged
    and yields exactly the window's slice of the full plan."""
    view = BoxTree(tree.origin, tree.root_side, tree.depth, tree.kappa_max,
                   tree.perm, tree.iperm, tree.points, tree.point_codes)
    for d in range(1, tree.depth + 1):
        lvl = tree.level(d)
        if d < 3:
            view.levels.append(lvl)
            continue
        lo, hi = win.ranges[d]
        sl = slice(lo, hi)
        parent = lvl.parent[sl]
        if d > 3:
            parent = parent - win.ranges[d - 1][0]
        if d < tree.depth:
            clo = win.ranges[d + 1][0]
            cs, ce = lvl.child_start[sl] - clo, lvl.child_end[sl] - clo
        else:
            cs, ce = lvl.child_start[sl], lvl.child_end[sl]
        nbr_idx, nbr_off = _slice_csr(lvl.nbr_idx, lvl.nbr_off, lo, hi)
        cz_idx, cz_off = _slice_csr(lvl.cousin_idx, lvl.cousin_off, lo, hi)
        view.levels.append(LevelBoxes(
            level=d, side=lvl.side, codes=lvl.codes[sl], coords=lvl.coords[sl],
            centers=lvl.centers[sl], pt_start=lvl.pt_start[sl],
            pt_count=lvl.pt_count[sl], parent=parent, child_start=cs,
            child_end=ce, nbr_idx=nbr_idx, nbr_off=nbr_off,
            cousin_idx=cz_idx, cousin_off=cz_off, box_lo=lo, full=lvl))
    return view


# ---------------------------------------------------------------------------
# cone coordinates and levels
# ---------------------------------------------------------------------------

def _norm3(dx: np.ndarray) -> np.ndarray:
    return np.linalg.norm(dx, axis=-1)


def cone_coords(x, x_center, side):
    """(s, theta, phi, r) about a box centre; s = (sqrt(3)/2 side) / r."""
    dx = np.atleast_2d(np.asarray(x, float) - np.asarray(x_center, float))
    r = _norm3(dx)
    if np.any(r == 0.0):
        raise ValueError("point coincides with the box center")
    s = np.sqrt(3.0) / 2.0 * side / r
    theta = np.arccos(np.clip(dx[:, 2] / r, -1.0, 1.0))
    phi = np.mod(np.arctan2(dx[:, 1], dx[:, 0]), 2.0 * np.pi)
    return s, theta, phi, r


def _cell_nodes(p: int, count: int, width: float) -> np.ndarray:
    lo = np.arange(count) * width
    return lo[:, None] + (cheb.nodes(p)[None, :] + 1.0) * 0.5 * width


@dataclass
class ConeLevel:
    level: int
    n_s: int
    n_a: int
    delta_s: float
    delta_a: float
    h: float
    s_nodes: np.ndarray
    ang_nodes_t: np.ndarray
    ang_nodes_p: np.ndarray
    seg_ids: np.ndarray
    seg_off: np.ndarray
    cpt_idx: np.ndarray
    cpt_off: np.ndarray

    @property
    def n_segments(self) -> int:
        return self.seg_ids.size

    @property
    def id_stride(self) -> int:
        return id_stride(self)

    def segs_of(self, b: int) -> np.ndarray:
        return self.seg_ids[self.seg_off[b]:self.seg_off[b + 1]]

    def seg_index(self, s, theta, phi) -> np.ndarray:
        return seg_index(self, s, theta, phi)

    def seg_unpack(self, flat):
        return seg_unpack(self, flat)

    def local_coords(self, flat, s, theta, phi):
        return local_coords(self, flat, s, theta, phi)

    def segment_nodes_xyz(self, flat, center):
        return segment_nodes_xyz(self, flat, center)

    def box_keys(self) -> np.ndarray:
        return box_keys(self)


# Cone-level helpers as free functions over the level's attributes, so they
# apply unchanged to the reference's own ConeLevel objects (drop-in path).

def id_stride(cl) -> int:
    return cl.n_s * cl.n_a * 2 * cl.n_a + 1


def seg_index(cl, s, theta, phi) -> np.ndarray:
    """Flat segment id, upper edges clamped (reference ifgf.py:349-354)."""
    i_s = np.minimum((s / cl.delta_s).astype(np.int64), cl.n_s - 1)
    i_t = np.minimum((theta / cl.delta_a).astype(np.int64), cl.n_a - 1)
    i_p = np.minimum((phi / cl.delta_a).astype(np.int64), 2 * cl.n_a - 1)
    return (i_s * cl.n_a + i_t) * (2 * cl.n_a) + i_p


def seg_unpack(cl, flat):
    i_p = flat % (2 * cl.n_a)
    rest = flat // (2 * cl.n_a)
    return rest // cl.n_a, rest % cl.n_a, i_p


def local_coords(cl, flat, s, theta, phi):
    """[-1,1]^3 coordinates inside segment `flat` (ifgf.py:361-367)."""
    i_s, i_t, i_p = seg_unpack(cl, flat)
    return (2.0 * (s / cl.delta_s - i_s) - 1.0,
            2.0 * (theta / cl.delta_a - i_t) - 1.0,
            2.0 * (phi / cl.delta_a - i_p) - 1.0)


def segment_nodes_xyz(cl, flat, center):
    """Cartesian nodes (nseg, p_s*p_a*p_a, 3) = center + r * dir and node
    radii (ifgf.py:369-387); ``center`` is (3,) or per segment (nseg, 3)."""
    flat = np.asarray(flat, dtype=np.int64)
    i_s, i_t, i_p = seg_unpack(cl, flat)
    r = cl.h / cl.s_nodes[i_s]
    th = cl.ang_nodes_t[i_t]
    ph = cl.ang_nodes_p[i_p]
    st, ct = np.sin(th), np.cos(th)
    cp, sp = np.cos(ph), np.sin(ph)
    dirs = np.stack([st[:, :, None] * cp[:, None, :],
                     st[:, :, None] * sp[:, None, :],
                     np.broadcast_to(ct[:, :, None],
                                     (flat.size, th.shape[1], ph.shape[1]))],
                    axis=-1)
    c = np.asarray(center, dtype=float)
    if c.ndim == 2:
        c = c[:, None, None, None, :]
    xyz = c + r[:, :, None, None, None] * dirs[:, None]
    rr = np.broadcast_to(r[:, :, None, None],
                         xyz.shape[:-1]).reshape(flat.size, -1)
    return xyz.reshape(flat.size, -1, 3), rr


def box_keys(cl) -> np.ndarray:
    """Globally sorted (box, segment id) keys, one per segment row."""
    nb = cl.seg_off.size - 1
    return (np.repeat(np.arange(nb, dtype=np.int64), np.diff(cl.seg_off))
            * np.int64(id_stride(cl)) + cl.seg_ids)


@dataclass
class ConeHierarchy:
    config: IfgfConfig
    kappa_max: float
    cone_levels: dict
    _accum_cache: dict = field(default_factory=dict)

    def level(self, d: int) -> ConeLevel:
        return self.cone_levels[d]

    def spectra_bytes(self, n_channels: int) -> int:
        sizes = sorted((cl.n_segments for cl in self.cone_levels.values()),
                       reverse=True)
        return sum(sizes[:2]) * self.config.n_nodes * n_channels * 16


def cone_counts(tree: BoxTree, config: IfgfConfig) -> dict:
    """(n_s, n_a) per level; doubles going coarser wherever kappa*H_d > 1/2."""
    out = {}
    n_s, n_a = config.n_s_seed, config.n_a_seed
    for d in range(tree.depth, 2, -1):
        if tree.kappa_max * tree.side(d) > 0.5:
            n_s, n_a = 2 * n_s, 2 * n_a
        out[d] = (n_s, n_a)
    return out


def _cousin_points(tree: BoxTree, d: int):
    """CSR of the cousin points (tree order) of every box at level d
    (cousin ids are global box ids, also in a window view)."""
    lvl = tree.level(d)
    glob = lvl.full if lvl.full is not None else lvl
    cz, owner = _expand_ranges(lvl.cousin_off[:-1], lvl.cousin_off[1:])
    cz = lvl.cousin_idx[cz]
    pts, p_own = _expand_ranges(glob.pt_start[cz],
                                glob.pt_start[cz] + glob.pt_count[cz])
    box = owner[p_own]
    return pts, _offsets_from_owner(box, lvl.n_boxes), box


_POOL = None


def _pool():
    """Shared thread pool for plan construction (numpy releases the GIL)."""
    global _POOL
    if _POOL is None:
        import concurrent.futures
        import os
        _POOL = concurrent.futures.ThreadPoolExecutor(
            max_workers=max(1, min(32, os.cpu_count() or 1)))
    return _POOL


def _chunks(off: np.ndarray, budget: int):
    """Split box ranges so that each chunk holds <= budget items."""
    nb = off.size - 1
    b = 0
    while b < nb:
        e = int(np.searchsorted(off, off[b] + budget, side="right")) - 1
        e = max(e, b + 1)
        e = min(e, nb)
        yield b, e
        b = e


def level_tables(cl) -> np.ndarray:
    """Node tables of a cone level in the device layout: s_nodes | sin_t |
    cos_t | sin_p | cos_p, from numpy's own sin / cos of the node angles
    (the values segment_nodes_xyz uses)."""
    return np.ascontiguousarray(np.concatenate([
        np.ravel(cl.s_nodes), np.ravel(np.sin(cl.ang_nodes_t)),
        np.ravel(np.cos(cl.ang_nodes_t)), np.ravel(np.sin(cl.ang_nodes_p)),
        np.ravel(np.cos(cl.ang_nodes_p))]), dtype=np.float64)


def _device_relevant(tree, d, cl, pcl, cpts, cbox):
    """Relevant (box, segment) set of level d on the device
    (csrc/planbuild.cu), edge cases decided here with numpy's expressions:
    identical to the host pass below.  Returns (seg_ids, seg_off, n_edge)."""
    import ctypes
    from . import _lib
    lib = _lib.load()
    lvl = tree.level(d)
    nb = lvl.n_boxes
    desc = _lib.ConeLevelDesc(cl.n_s, cl.n_a, cl.delta_s, cl.delta_a,
                              float(np.sqrt(3.0) / 2.0 * lvl.side), nb, 1 << 20)
    h = ctypes.c_void_p()
    _lib.check(lib.ifgfb_cones_begin(ctypes.byref(desc), ctypes.byref(h)), "ifgfb_cones_begin")
    i32 = lambda a: np.ascontiguousarray(a, dtype=np.int32)
    p32 = lambda a: a.ctypes.data_as(ctypes.POINTER(ctypes.c_int32))
    try:
        centers = np.ascontiguousarray(lvl.centers, dtype=np.float64)
        if cpts.size:
            cb, cp_ = i32(cbox), i32(cpts)
            pts = np.ascontiguousarray(tree.points, dtype=np.float64)
            _lib.check(lib.ifgfb_cones_mark_points(h, cpts.size, p32(cb), p32(cp_),
                                                   pts.shape[0], _lib.dptr(pts),
                                                   _lib.dptr(centers)),
                       "ifgfb_cones_mark_points")
        if pcl is not None:
            up = tree.level(d - 1)
            cnt = pcl.seg_off[lvl.parent + 1] - pcl.seg_off[lvl.parent]
            inst_off = np.zeros(nb + 1, dtype=np.int64)
            np.cumsum(cnt, out=inst_off[1:])
            row0 = np.ascontiguousarray(pcl.seg_off[lvl.parent], dtype=np.int64)
            pbox, pseg = i32(lvl.parent), i32(pcl.seg_ids)
            pctr = np.ascontiguousarray(up.centers, dtype=np.float64)
            tabs = level_tables(pcl)
            pd = _lib.ConeParentDesc(nb, _lib.iptr(inst_off), _lib.iptr(row0), p32(pbox),
                                     pseg.size, p32(pseg), up.n_boxes, _lib.dptr(pctr),
                                     _lib.dptr(centers), pcl.n_s, pcl.n_a, pcl.h,
                                     _lib.dptr(tabs))
            _lib.check(lib.ifgfb_cones_mark_parents(h, ctypes.byref(pd)),
                       "ifgfb_cones_mark_parents")
        n = ctypes.c_int64()
        _lib.check(lib.ifgfb_cones_ambiguous(h, ctypes.byref(n), None, None),
                   "ifgfb_cones_ambiguous")
        n_edge = n.value
        if n_edge:
            box = np.empty(n_edge, dtype=np.int64)
            dx = np.empty((n_edge, 3))
            _lib.check(lib.ifgfb_cones_ambiguous(h, ctypes.byref(n), _lib.iptr(box),
                                                 _lib.dptr(dx)), "ifgfb_cones_ambiguous")
            s, th, ph, _ = cone_coords(dx, np.zeros(3), lvl.side)
            key = np.ascontiguousarray(seg_index(cl, s, th, ph), dtype=np.int64)
            _lib.check(lib.ifgfb_cones_set(h, n_edge, _lib.iptr(box), _lib.iptr(key)),
                       "ifgfb_cones_set")
        seg_off = np.zeros(nb + 1, dtype=np.int64)
        total = ctypes.c_int64()
        _lib.check(lib.ifgfb_cones_finish(h, _lib.iptr(seg_off), None, ctypes.byref(total)),
                   "ifgfb_cones_finish")
        seg_ids = np.empty(total.value, dtype=np.int64)
        _lib.check(lib.ifgfb_cones_ids(h, _lib.iptr(seg_off), _lib.iptr(seg_ids)),
                   "ifgfb_cones_ids")
    finally:
        lib.ifgfb_cones_free(h)
    return seg_ids, seg_off, n_edge


def build_cone_hierarchy(tree: BoxTree, config: IfgfConfig = IfgfConfig(),
                         device: bool = False) -> ConeHierarchy:
    """Relevant segments per box: those holding a cousin point or a node of a
    relevant parent segment (sorted per box).

    device=True runs the relevance pass on the GPU (csrc/planbuild.cu,
    ifgfb_cones_*): bit-identical result, the edge cases decided on the host
    with the same numpy expressions (hier.edge_cases counts them)."""
    counts = cone_counts(tree, config)
    hier = ConeHierarchy(config, tree.kappa_max, {})
    hier.device_plan = bool(device)   # propagation types on the device too
    nn = config.n_nodes
    for d in range(3, tree.depth + 1):
        n_s, n_a = counts[d]
        lvl = tree.level(d)
        cl = ConeLevel(
            level=d, n_s=n_s, n_a=n_a, delta_s=ETA / n_s,
            delta_a=np.pi / n_a, h=np.sqrt(3.0) / 2.0 * lvl.side,
            s_nodes=_cell_nodes(config.p_s, n_s, ETA / n_s),
            ang_nodes_t=_cell_nodes(config.p_a, n_a, np.pi / n_a),
            ang_nodes_p=_cell_nodes(config.p_a, 2 * n_a, np.pi / n_a),
            seg_ids=np.empty(0, dtype=np.int64),
            seg_off=np.zeros(lvl.n_boxes + 1, dtype=np.int64),
            cpt_idx=np.empty(0, dtype=np.int64),
            cpt_off=np.zeros(lvl.n_boxes + 1, dtype=np.int64))
        stride = np.int64(id_stride(cl))
        cpts, cpt_off, cbox = _cousin_points(tree, d)
        cl.cpt_idx, cl.cpt_off = cpts, cpt_off
        if device:
            cl.seg_ids, cl.seg_off, n_edge = _device_relevant(
                tree, d, cl, hier.cone_levels.get(d - 1), cpts, cbox)
            hier.__dict__.setdefault("edge_cases", {})[d] = n_edge
            hier.cone_levels[d] = cl
            continue
        keys = []
        if cpts.size:
            s, th, ph, _ = cone_coords(tree.points[cpts], lvl.centers[cbox],
                                       lvl.side)
            keys.append(cbox * stride + seg_index(cl, s, th, ph))
        pcl = hier.cone_levels.get(d - 1)
        if pcl is not None:
            up = tree.level(d - 1)
            # parent segment rows of every child box
            prow_off = pcl.seg_off[lvl.parent]
            prow_end = pcl.seg_off[lvl.parent + 1]
            inst_off = np.zeros(lvl.n_boxes + 1, dtype=np.int64)
            np.cumsum(prow_end - prow_off, out=inst_off[1:])
            pbox_of_row = np.repeat(np.arange(up.n_boxes),
                                    np.diff(pcl.seg_off))
            budget = max(1, 1_000_000 // nn)

            def chunk_keys(b0, b1):
                rows, own = _expand_ranges(prow_off[b0:b1], prow_end[b0:b1])
                if rows.size == 0:
                    return None
                xyz, _ = segment_nodes_xyz(
                    pcl, pcl.seg_ids[rows], up.centers[pbox_of_row[rows]])
                box = own + b0
                dx = xyz - lvl.centers[box][:, None, :]
                s, th, ph, _ = cone_coords(dx.reshape(-1, 3), np.zeros(3),
                                           lvl.side)
                k = np.repeat(box, nn) * stride + seg_index(cl, s, th, ph)
                return np.unique(k)

            # numpy ufuncs release the GIL: chunks run concurrently, each
            # element computed by the same expression (bit-identical)
            keys.extend(k for k in _pool().map(
                lambda r: chunk_keys(*r), list(_chunks(inst_off, budget)))
                if k is not None)
        if keys:
            uk = np.unique(np.concatenate(keys))
            box = uk // stride
            cl.seg_ids = uk - box * stride
            cl.seg_off = _offsets_from_owner(box, lvl.n_boxes)
        hier.cone_levels[d] = cl
    return hier


# ---------------------------------------------------------------------------
# propagation plan (child level d -> parent level d-1)
# ---------------------------------------------------------------------------

@dataclass
class AccumulationPlan:
    """Types (parent segment id, child octant) with shared child-frame
    geometry, and instances regrouped per parent segment row.

    Stored per type t, in PARENT node order (what the device consumes; about
    3.2 KB per type): ``gid[t, n]`` = sigma group (local to t) of parent node
    n, ``node_geom[t, n]`` = (xs, xt, xp) local coordinates in its child
    segment, ``node_r[t, n]`` = (r_parent, r_child); ``scatter[t, j]`` =
    parent node at sorted slot j (nodes sorted by child segment, as the
    reference's ``_AccumType``).  ``sig_off[t]:sig_off[t+1]`` index the
    type's groups in ``group_sigma`` (child segment id per group).  The
    reference-layout views (sorted order) ``xs``, ``xt``, ``xp``,
    ``r_parent``, ``r_child``, ``group_bounds``, ``group_end`` are computed
    on demand.

    Instances (one per (parent segment row, child box)) sorted by parent
    row then child box: ``inst_off`` (per parent row), ``inst_type``,
    ``inst_child``, ``inst_crow_off`` into ``crow`` (child segment row per
    sigma group of the type).
    """

    level: int
    n_types: int
    type_gamma: np.ndarray
    type_octant: np.ndarray
    sig_off: np.ndarray
    group_sigma: np.ndarray       # child segment id of each group
    gid: np.ndarray               # (n_types, 75) uint8, parent order
    scatter: np.ndarray           # (n_types, 75) uint8, sorted slot -> node
    node_geom: np.ndarray         # (n_types, 75, 3) f64, parent order
    node_r: np.ndarray            # (n_types, 75, 2) f64, parent order
    inst_off: np.ndarray
    inst_type: np.ndarray
    inst_child: np.ndarray
    inst_crow_off: np.ndarray
    crow: np.ndarray
    crow_misses: int = 0
    trimmed: bool = False         # per-type arrays released (trim_...)

    @property
    def n_instances(self) -> int:
        return self.inst_type.size

    def _sorted(self, arr):
        return np.take_along_axis(arr, self.scatter.astype(np.int64), axis=1)

    @cached_property
    def xs(self):
        return self._sorted(self.node_geom[..., 0])

    @cached_property
    def xt(self):
        return self._sorted(self.node_geom[..., 1])

    @cached_property
    def xp(self):
        return self._sorted(self.node_geom[..., 2])

    @cached_property
    def r_parent(self):
        return self._sorted(self.node_r[..., 0])

    @cached_property
    def r_child(self):
        return self._sorted(self.node_r[..., 1])

    @cached_property
    def group_end(self):
        """Per group (flat): one past its last sorted slot (local to the
        type; groups are contiguous in sorted order, local ids ascending)."""
        nn = self.gid.shape[1]
        flat = (self.sig_off[:-1, None] + self.gid).ravel()
        size = np.bincount(flat, minlength=self.group_sigma.size)
        owner = np.repeat(np.arange(self.n_types), np.diff(self.sig_off))
        return np.cumsum(size) - nn * owner

    @cached_property
    def group_bounds(self):
        """Per group (flat): its first sorted slot (local to the type)."""
        end = self.group_end
        nn = self.gid.shape[1]
        flat = (self.sig_off[:-1, None] + self.gid).ravel()
        return end - np.bincount(flat, minlength=self.group_sigma.size)


def _type_geometry(pcl: ConeLevel, cl: ConeLevel, gamma, octant, child_side):
    """Vectorised reference ``_AccumType.__init__`` (ifgf.py:686-702)."""
    n_t = gamma.size
    bits = np.stack([(octant >> 2) & 1, (octant >> 1) & 1, octant & 1],
                    axis=-1)
    offset = 0.5 * child_side * (bits * 2.0 - 1.0)
    xyz, rp = segment_nodes_xyz(pcl, gamma, -offset)
    nn = xyz.shape[1]
    s, th, ph, rc = cone_coords(xyz.reshape(-1, 3), np.zeros(3), child_side)
    flat = seg_index(cl, s, th, ph).reshape(n_t, nn)
    order = np.argsort(flat, axis=1, kind="stable")
    fs = np.take_along_axis(flat, order, axis=1)
    take = lambda a: np.take_along_axis(a.reshape(n_t, nn), order, axis=1)
    xs, xt, xp = local_coords(cl, fs, take(s), take(th), take(ph))
    return fs, order, xs, xt, xp, take(rp), take(rc)


def _device_types(pcl, cl, gamma, toct, child_side, geometry: bool,
                  chunk: int = 1 << 22):
    """Per type: sigma groups (gid, sigma ascending, count) and optionally
    the node geometry, from the device (csrc/planbuild.cu,
    ifgfb_accum_types); types with a node within a few ulp of a child
    segment edge are recomputed here by ``_type_geometry`` (the reference's
    expressions), so gid / sigma equal the host builder's bit for bit."""
    import ctypes
    from . import _lib
    lib = _lib.load()
    n_t, nn = gamma.size, 75
    gid = np.empty((n_t, nn), dtype=np.uint8)
    sigma = np.empty((n_t, nn), dtype=np.int32)
    nsig = np.empty(n_t, dtype=np.uint8)
    amb = np.empty(n_t, dtype=np.uint8)
    geom = np.empty((n_t, nn, 3)) if geometry else None
    node_r = np.empty((n_t, nn, 2)) if geometry else None
    tabs = level_tables(pcl)
    g32 = np.ascontiguousarray(gamma, dtype=np.int32)
    o8 = np.ascontiguousarray(toct, dtype=np.uint8)
    u8 = lambda a: a.ctypes.data_as(ctypes.POINTER(ctypes.c_uint8))
    for t0 in range(0, n_t, chunk):
        t1 = min(n_t, t0 + chunk)
        desc = _lib.AccumTypesDesc(
            t1 - t0, g32[t0:t1].ctypes.data_as(ctypes.POINTER(ctypes.c_int32)), u8(o8[t0:t1]),
            pcl.n_s, pcl.n_a, pcl.h, _lib.dptr(tabs), cl.n_s, cl.n_a, cl.delta_s, cl.delta_a,
            float(np.sqrt(3.0) / 2.0 * child_side), 0.5 * child_side)
        _lib.check(lib.ifgfb_accum_types(
            ctypes.byref(desc), u8(gid[t0:t1]),
            sigma[t0:t1].ctypes.data_as(ctypes.POINTER(ctypes.c_int32)), u8(nsig[t0:t1]),
            u8(amb[t0:t1]), _lib.dptr(geom[t0:t1]) if geometry else None,
            _lib.dptr(node_r[t0:t1]) if geometry else None), "ifgfb_accum_types")
    sel = np.nonzero(amb)[0]
    if sel.size:
        fs, order, xs, xt, xp, rp, rc = _type_geometry(pcl, cl, gamma[sel], toct[sel],
                                                       child_side)
        rows = np.arange(sel.size)[:, None]
        newgrp = np.ones(fs.shape, dtype=bool)
        newgrp[:, 1:] = fs[:, 1:] != fs[:, :-1]
        local = np.cumsum(newgrp, axis=1) - 1
        g = np.empty((sel.size, nn), dtype=np.uint8)
        g[rows, order] = local
        gid[sel] = g
        sig = np.full((sel.size, nn), -1, dtype=np.int32)
        for i in range(sel.size):
            u = fs[i][newgrp[i]]
            sig[i, :u.size] = u
        sigma[sel] = sig
        nsig[sel] = newgrp.sum(axis=1)
        if geometry:
            for k, v in enumerate((xs, xt, xp)):
                tmp = np.empty((sel.size, nn))
                tmp[rows, order] = v
                geom[sel, :, k] = tmp
            tmp = np.empty((sel.size, nn))
            tmp[rows, order] = rp
            node_r[sel, :, 0] = tmp
            tmp[rows, order] = rc
            node_r[sel, :, 1] = tmp
    return gid, sigma, nsig, geom, node_r, int(sel.size)


def accumulation_plan(tree: BoxTree, hier: ConeHierarchy, d: int,
                      geometry: bool = True, device: bool | None = None) -> AccumulationPlan:
    """Plan for folding level-d child interpolants into level d-1, cached
    on the hierarchy.  ``geometry=False`` accepts a cached plan whose
    per-type arrays were released by ``trim_accumulation_plans`` (instance
    counts and child rows only); otherwise a trimmed plan is rebuilt."""
    cache = hier.__dict__.setdefault("_b200_accum", {})
    if d in cache and (not geometry or not cache[d].trimmed):
        return cache[d]
    from .engine import _StageLog
    log = _StageLog(f"accum {d}")
    cl, pcl = hier.level(d), hier.level(d - 1)
    lvl = tree.level(d)
    nn = hier.config.p_s * hier.config.p_a ** 2
    octant = (lvl.codes & np.uint64(7)).astype(np.int64)
    prow, child = _parent_row_major_instances(lvl.parent, pcl.seg_off)
    key = pcl.seg_ids[prow] * 8 + octant[child]
    ukeys, inst_type = np.unique(key, return_inverse=True)
    del key
    inst_type = inst_type.astype(np.int64)
    gamma, toct = ukeys >> 3, ukeys & 7
    n_t = ukeys.size
    if device is None:
        device = bool(hier.__dict__.get("device_plan", False))
    if device:
        log(f"instances + types ({n_t} types)")
        gid, sigma, nsig, _, _, n_edge = _device_types(pcl, cl, gamma, toct, lvl.side, False)
        log(f"device type groups ({n_edge} edge types on the host)")
        sig_off = np.zeros(n_t + 1, dtype=np.int64)
        np.cumsum(nsig, out=sig_off[1:])
        g_sigma = sigma[sigma >= 0].astype(np.int64)
        del sigma
        return _finish_accumulation_plan(
            cache, d, cl, pcl, gamma, toct, sig_off, g_sigma, gid, None, None, None,
            prow, child, inst_type, log, pending=(pcl, cl, lvl.side))
    gid = np.empty((n_t, nn), dtype=np.uint8)
    scatter = np.empty((n_t, nn), dtype=np.uint8)
    node_geom = np.empty((n_t, nn, 3))
    node_r = np.empty((n_t, nn, 2))
    step = max(1, 250_000 // nn)
    blocks = list(range(0, n_t, step))
    sig_parts = [None] * len(blocks)

    def chunk(ib):
        t0 = blocks[ib]
        t1 = min(n_t, t0 + step)
        fs, order, xs, xt, xp, rp, rc = _type_geometry(
            pcl, cl, gamma[t0:t1], toct[t0:t1], lvl.side)
        rows = np.arange(t1 - t0)[:, None]
        newgrp = np.ones(fs.shape, dtype=bool)
        newgrp[:, 1:] = fs[:, 1:] != fs[:, :-1]
        local = np.cumsum(newgrp, axis=1) - 1           # group of sorted slot
        if local.size and local.max() >= nn:
            raise ValueError("more than 75 sigma groups in a type")
        gid[t0:t1][rows, order] = local
        scatter[t0:t1] = order
        for k, v in enumerate((xs, xt, xp)):
            node_geom[t0:t1, :, k][rows, order] = v
        node_r[t0:t1, :, 0][rows, order] = rp
        node_r[t0:t1, :, 1][rows, order] = rc
        sig_parts[ib] = (newgrp.sum(axis=1), fs[newgrp])

    log(f"instances + types ({n_t} types)")
    list(_pool().map(chunk, range(len(blocks))))   # disjoint row blocks
    log("type geometry")
    n_sig = np.concatenate([c for c, _ in sig_parts]) if blocks else np.zeros(0, np.int64)
    g_sigma = (np.concatenate([g for _, g in sig_parts]) if blocks
               else np.zeros(0, np.int64)).astype(np.int64)
    del sig_parts
    sig_off = np.zeros(n_t + 1, dtype=np.int64)
    np.cumsum(n_sig, out=sig_off[1:])
    return _finish_accumulation_plan(cache, d, cl, pcl, gamma, toct, sig_off, g_sigma, gid,
                                     scatter, node_geom, node_r, prow, child, inst_type, log)


def _parent_row_major_instances(parent: np.ndarray, pseg_off: np.ndarray):
    """(parent segment row, child box) of every propagation instance, sorted
    by parent row then child, built directly: the children of a parent box
    are consecutive boxes and its rows are consecutive, so each parent box
    contributes a rows x children block in row-major order (the same order
    np.lexsort((child, prow)) gives, without the sort)."""
    nb = parent.size
    if nb == 0:
        z = np.empty(0, np.int64)
        return z, z
    new = np.ones(nb, dtype=bool)
    new[1:] = parent[1:] != parent[:-1]
    first = np.nonzero(new)[0]                      # first child of each parent box
    kids = np.diff(np.append(first, nb))
    pb = parent[first]
    r0 = pseg_off[pb]
    rows = pseg_off[pb + 1] - r0
    local, own = _expand_ranges(np.zeros(pb.size, np.int64), rows * kids)
    k = kids[own]
    return r0[own] + local // k, first[own] + local % k


def _finish_accumulation_plan(cache, d, cl, pcl, gamma, toct, sig_off, g_sigma, gid,
                              scatter, node_geom, node_r, prow, child, inst_type, log,
                              pending=None):
    n_t = gamma.size
    # instances are already sorted by (parent row, child)
    nsig = np.diff(sig_off)[inst_type]
    crow_off = np.zeros(prow.size + 1, dtype=np.int64)
    np.cumsum(nsig, out=crow_off[1:])
    bkeys = box_keys(cl)
    stride = np.int64(id_stride(cl))
    crow = np.empty(int(crow_off[-1]), dtype=np.int64)
    misses = []

    def rows_of(rng):      # child segment row of every (instance, group)
        i0, i1 = rng
        gidx, g_own = _expand_ranges(sig_off[inst_type[i0:i1]], sig_off[inst_type[i0:i1] + 1])
        want = child[i0:i1][g_own] * stride + g_sigma[gidx]
        c = np.searchsorted(bkeys, want)
        misses.append(int(np.count_nonzero(bkeys[np.minimum(c, bkeys.size - 1)] != want)))
        crow[crow_off[i0]:crow_off[i1]] = c

    step = 1 << 20
    list(_pool().map(rows_of, [(i, min(prow.size, i + step))
                               for i in range(0, prow.size, step)]))
    misses = sum(misses)
    log("child rows")
    plan = AccumulationPlan(
        level=d, n_types=n_t, type_gamma=gamma, type_octant=toct,
        sig_off=sig_off, group_sigma=g_sigma, gid=gid, scatter=scatter,
        node_geom=node_geom, node_r=node_r,
        inst_off=_offsets_from_owner(prow, pcl.n_segments),
        inst_type=inst_type, inst_child=child, inst_crow_off=crow_off,
        crow=crow, crow_misses=misses)
    plan.pending_geometry = pending
    cache[d] = plan
    return plan


def trim_accumulation_plans(hier: ConeHierarchy) -> None:
    """Release the per-type arrays (gid, scatter, node_geom, node_r: about
    3.2 KB per type) of the cached plans once the device plan holds them;
    instance arrays stay for work counts and partitioning."""
    for ap in hier.__dict__.get("_b200_accum", {}).values():
        ap.gid = ap.scatter = ap.node_geom = ap.node_r = None
        ap.pending_geometry = None
        for k in ("xs", "xt", "xp", "r_parent", "r_child", "group_end", "group_bounds"):
            ap.__dict__.pop(k, None)
        ap.trimmed = True


WARP_PARTS = 5          # parent nodes owned per warp: fixed theta index b


def _local_group_ids(ap: AccumulationPlan, nn: int) -> np.ndarray:
    """gid[t, node] = sigma group (local to type t) of parent node `node`."""
    return ap.gid


def _warp_set_tiles(gid, t, orow, w, per):
    """Tiles of warp w for a block of instances: (tile id per element,
    tiles per instance, sorted groups, slots, position in run)."""
    nodes = orow[:, per * w:per * (w + 1)]                   # (ni, per)
    g = gid[t[:, None], nodes]                              # (ni, per) int16
    order = np.argsort(g, axis=1, kind="stable")
    gs = np.take_along_axis(g, order, axis=1)
    new = np.ones(gs.shape, dtype=bool)
    new[:, 1:] = gs[:, 1:] != gs[:, :-1]
    idx = np.broadcast_to(np.arange(per, dtype=np.int16), gs.shape)
    start = np.maximum.accumulate(np.where(new, idx, 0), axis=1)
    pos = idx - start                                       # position in run
    newt = new | (pos % 8 == 0)
    tid = np.cumsum(newt, axis=1, dtype=np.int32) - 1       # tile per element
    return tid, tid[:, -1] + 1, gs, order, pos


def row_order_cuts(ap: AccumulationPlan, cut_radius: int = 4, n_threads: int = 0,
                   wide: bool = False):
    """The first half of ``row_tiles``: per parent row the signature order
    and the warp cuts, without tile records (tile-free device plans form
    the tiles in the kernel from the nodes' sigma groups).  ``wide``: cuts
    for the wide-warp kernel (``ifgfb_row_cuts_wide``: ifgfb_wide_warps()
    sets of <= 32 nodes; env IFGFB_WIDE_CUT = radius, IFGFB_WIDE_TW /
    IFGFB_WIDE_BW = weights of the row's tile count / the largest per-warp
    count)."""
    from . import _lib
    lib = _lib.load()
    nn = 75
    gid = np.ascontiguousarray(_local_group_ids(ap, nn), dtype=np.uint8)
    n_rows = ap.inst_off.size - 1
    io = np.ascontiguousarray(ap.inst_off, dtype=np.int64)
    it = np.ascontiguousarray(ap.inst_type, dtype=np.int64)
    row_order = np.empty((n_rows, nn), dtype=np.uint8)
    row_cuts = np.empty((n_rows, WARP_PARTS + 1), dtype=np.uint8)
    if wide:
        import os
        _lib.check(lib.ifgfb_row_cuts_wide(
            n_rows, _lib.iptr(io), _lib.iptr(it), ap.n_types, _lib.u8ptr(gid),
            _lib.u8ptr(row_order), _lib.u8ptr(row_cuts), lib.ifgfb_wide_warps(),
            int(os.environ.get("IFGFB_WIDE_CUT", "6")), int(os.environ.get("IFGFB_WIDE_TW", "2")),
            int(os.environ.get("IFGFB_WIDE_BW", "1")), n_threads), "ifgfb_row_cuts_wide")
        return row_order, row_cuts
    _lib.check(lib.ifgfb_row_tiles_plan(
        n_rows, _lib.iptr(io), _lib.iptr(it), ap.n_types, _lib.u8ptr(gid),
        _lib.u8ptr(row_order), _lib.u8ptr(row_cuts), None, cut_radius, n_threads),
        "ifgfb_row_tiles_plan")
    return row_order, row_cuts


def row_tiles(ap: AccumulationPlan, cut_radius: int = 4, n_threads: int = 0):
    """Per parent row partition of its 75 nodes into 5 contiguous warp-owned
    sets and the MMA row tiles of every (instance, warp); native builder
    (csrc/tiles.cpp, ``ifgfb_row_tiles_plan`` / ``_fill``).

    Nodes are sorted by their child-segment signature over the row's
    instances; the 4 cuts of that order are chosen per row within +-cut_radius
    of 15k to minimise the largest per-warp tile count (cut_radius 0 gives
    ``row_tiles_equal_split``, bit for bit).

    Returns
      row_order (n_rows, 75) uint8  node at set position
      row_cuts  (n_rows, 6) uint8   warp w owns positions cuts[w]..cuts[w+1]-1
      tile_off  (n_instances*5+1,)  tiles of (instance, warp)
      tiles     (n_tiles, 16) uint8 [local group, rows, slot0..7, pad];
                                    slot = position within the warp's set
    """
    from . import _lib
    lib = _lib.load()
    nn = 75
    gid = _local_group_ids(ap, nn)
    if gid.size and (gid.min() < 0 or gid.max() >= nn):
        raise ValueError("sigma group id outside 0..74")
    gid = np.ascontiguousarray(gid, dtype=np.uint8)
    n_rows = ap.inst_off.size - 1
    io = np.ascontiguousarray(ap.inst_off, dtype=np.int64)
    it = np.ascontiguousarray(ap.inst_type, dtype=np.int64)
    row_order = np.empty((n_rows, nn), dtype=np.uint8)
    row_cuts = np.empty((n_rows, WARP_PARTS + 1), dtype=np.uint8)
    tile_off = np.zeros(ap.n_instances * WARP_PARTS + 1, dtype=np.int64)
    _lib.check(lib.ifgfb_row_tiles_plan(
        n_rows, _lib.iptr(io), _lib.iptr(it), ap.n_types, _lib.u8ptr(gid),
        _lib.u8ptr(row_order), _lib.u8ptr(row_cuts), _lib.iptr(tile_off),
        cut_radius, n_threads), "ifgfb_row_tiles_plan")
    tiles = np.empty((int(tile_off[-1]), 16), dtype=np.uint8)
    _lib.check(lib.ifgfb_row_tiles_fill(
        n_rows, _lib.iptr(io), _lib.iptr(it), ap.n_types, _lib.u8ptr(gid),
        _lib.u8ptr(row_order), _lib.u8ptr(row_cuts), _lib.iptr(tile_off),
        _lib.u8ptr(tiles), n_threads), "ifgfb_row_tiles_fill")
    return row_order, row_cuts, tile_off, tiles


def row_tiles_equal_split(ap: AccumulationPlan, p_s: int = 3, p_a: int = 5,
                          chunk: int = 1 << 17):
    """Numpy statement of ``row_tiles(ap, cut_radius=0)`` (equal sets of 15),
    kept to cross-check the native builder (tests/test_plan.py).

    Nodes are sorted by their child-segment signature over the row's
    instances (the sigma group of the node under each child), so nodes that
    share child segments under every child land in the same warp set and
    its row tiles fill up (11.1-12.7 tiles per instance against 12.2-13.9
    for a fixed theta-index split; lower bound 10.5-10.9).

    Returns
      row_order (n_rows, 75) uint8  node at set position (warp w owns
                                    positions 15w..15w+14)
      tile_off  (n_instances*5+1,)  tiles of (instance, warp)
      tiles     (n_tiles, 16) uint8 [local group, rows, slot0..7, pad];
                                    slot = position within the warp's set
    """
    nn = p_s * p_a * p_a
    per = nn // WARP_PARTS
    gid = _local_group_ids(ap, nn)
    n_rows = ap.inst_off.size - 1
    cnt = np.diff(ap.inst_off)
    if cnt.size and cnt.max() > 8:
        raise ValueError("more than 8 children per parent box")
    # signature key per (row, node): 4 bits per instance slot
    key = np.zeros((n_rows, nn), dtype=np.int64)
    for i in range(8):
        has = cnt > i
        rows = np.nonzero(has)[0]
        t = ap.inst_type[ap.inst_off[rows] + i]
        key[rows] |= gid[t].astype(np.int64) << (4 * (7 - i))
        key[~has] |= np.int64(0xF) << (4 * (7 - i))
    row_order = np.argsort(key, axis=1, kind="stable").astype(np.uint8)
    del key
    prow = np.repeat(np.arange(n_rows), cnt)
    ni_all = ap.n_instances
    blocks = [(i0, min(ni_all, i0 + chunk)) for i0 in range(0, ni_all, chunk)]
    counts = np.zeros((ni_all, WARP_PARTS), dtype=np.int64)

    def count(blk):                       # pass 1: tiles per (instance, warp)
        i0, i1 = blk
        t = ap.inst_type[i0:i1]
        orow = row_order[prow[i0:i1]]
        for w in range(WARP_PARTS):
            counts[i0:i1, w] = _warp_set_tiles(gid, t, orow, w, per)[1]

    list(_pool().map(count, blocks))
    tile_off = np.zeros(ni_all * WARP_PARTS + 1, dtype=np.int64)
    np.cumsum(counts.ravel(), out=tile_off[1:])
    tiles = np.full((int(tile_off[-1]), 16), 0xFF, dtype=np.uint8)

    def fill(blk):                        # pass 2: disjoint records per block
        i0, i1 = blk
        t = ap.inst_type[i0:i1]
        orow = row_order[prow[i0:i1]]
        for w in range(WARP_PARTS):
            tid, ntile, gs, order, pos = _warp_set_tiles(gid, t, orow, w, per)
            base = tile_off[np.arange(i0, i1) * WARP_PARTS + w]
            gidx = (base[:, None] + tid).ravel()
            tiles[gidx, 0] = gs.ravel().astype(np.uint8)
            tiles[gidx, 2 + (pos.ravel() % 8)] = order.ravel().astype(np.uint8)
            lo = int(gidx.min())
            rows_per = np.bincount(gidx - lo)
            nz = np.nonzero(rows_per)[0]
            tiles[lo + nz, 1] = rows_per[nz].astype(np.uint8)

    list(_pool().map(fill, blocks))
    cuts = np.tile(np.arange(0, nn + 1, per, dtype=np.uint8), (n_rows, 1))
    return row_order, cuts, tile_off, tiles


def node_tables(ap: AccumulationPlan, p_s: int = 3, p_a: int = 5):
    """Per type and PARENT node: local coordinates in its child segment
    (xs, xt, xp) and the radii (r_parent, r_child).  Plans built on the
    device compute them here, on demand (only levels whose tables are
    uploaded need them)."""
    pend = getattr(ap, "pending_geometry", None)
    if ap.node_geom is None and pend is not None:
        pcl, cl, side = pend
        _, _, _, ap.node_geom, ap.node_r, _ = _device_types(
            pcl, cl, ap.type_gamma, ap.type_octant, side, True)
    return ap.node_geom, ap.node_r


# ---------------------------------------------------------------------------
# emission plan (level d boxes -> their cousin points)
# ---------------------------------------------------------------------------

@dataclass
class EmissionPlan:
    """One entry per (box, cousin point) pair, box-major as ``cpt_idx``:
    segment row, target (tree order) and local coordinates / radius of the
    target and of its displaced copy (same segment, reference ifgf.py:651)."""

    level: int
    row: np.ndarray
    target: np.ndarray
    geom: np.ndarray              # (n_pairs, 4): xs, xt, xp, r
    geom_disp: np.ndarray | None  # (n_pairs, 4) or None
    row_misses: int = 0

    @property
    def n_pairs(self) -> int:
        return self.row.size


SEAM_MODES = ("unwrap", "reference")


def emission_plan(tree: BoxTree, hier: ConeHierarchy, d: int,
                  disp_points_t: np.ndarray | None = None,
                  seam: str = "unwrap") -> EmissionPlan:
    """seam: how the displaced point's phi is taken.  "unwrap" (default)
    keeps it on the undisplaced point's branch; "reference" takes it mod
    2 pi exactly as reference ifgf.py:647-651 (parity runs at seam-crossing
    configurations).  Rows whose displacement does not cross phi = 0 are
    bitwise identical under both.

    Pairs are processed in chunks of whole boxes on the plan thread pool
    (every element by the same expressions: bit-identical to one pass); a
    chunk's segment rows are looked up among its own boxes' keys only."""
    if seam not in SEAM_MODES:
        raise ValueError(f"seam must be one of {SEAM_MODES}")
    cl, lvl = hier.level(d), tree.level(d)
    tg = cl.cpt_idx
    n_pairs = tg.size
    if n_pairs == 0:
        z = np.empty((0, 4))
        return EmissionPlan(d, np.empty(0, np.int64), tg, z,
                            None if disp_points_t is None else z)
    keys = box_keys(cl)
    stride = np.int64(id_stride(cl))
    row = np.empty(n_pairs, dtype=np.int64)
    geom = np.empty((n_pairs, 4))
    gd = None if disp_points_t is None else np.empty((n_pairs, 4))
    miss = []

    def chunk(rng):
        b0, b1 = rng
        p0, p1 = int(cl.cpt_off[b0]), int(cl.cpt_off[b1])
        if p1 == p0:
            return
        box = np.repeat(np.arange(b0, b1, dtype=np.int64), np.diff(cl.cpt_off[b0:b1 + 1]))
        ctr = lvl.centers[box]
        t = tg[p0:p1]
        s, th, ph, r = cone_coords(tree.points[t] - ctr, np.zeros(3), lvl.side)
        flat = seg_index(cl, s, th, ph)
        want = box * stride + flat
        k0, k1 = int(cl.seg_off[b0]), int(cl.seg_off[b1])
        kk = keys[k0:k1]
        rr = np.searchsorted(kk, want).astype(np.int64)
        if kk.size:
            miss.append(int(np.count_nonzero(kk[np.minimum(rr, kk.size - 1)] != want)))
        else:
            miss.append(int(want.size))
        row[p0:p1] = rr + k0
        geom[p0:p1] = np.stack(local_coords(cl, flat, s, th, ph) + (r,), axis=1)
        if gd is not None:
            sd, td, pd, rd = cone_coords(disp_points_t[t] - ctr, np.zeros(3), lvl.side)
            # Deliberate deviation from the reference (ifgf.py:647-651): the
            # displaced point is evaluated with the undisplaced point's
            # segment polynomial, but its phi is taken mod 2 pi, so a
            # displacement across the phi = 0 seam lands ~2 n_a intervals
            # away and the angular polynomial is extrapolated there (D_far =
            # (S(x+hn) - S(x))/h then blows up by ~1e5 at those rows; GMRES
            # stagnates from sphere(12,10) on).  Keep the displaced phi on
            # the undisplaced point's branch.  Bitwise unchanged wherever
            # the seam is not crossed (every golden configuration).
            if seam == "unwrap":
                pd = np.where(pd - ph > np.pi, pd - 2.0 * np.pi,
                              np.where(ph - pd > np.pi, pd + 2.0 * np.pi, pd))
            gd[p0:p1] = np.stack(local_coords(cl, flat, sd, td, pd) + (rd,), axis=1)

    list(_pool().map(chunk, list(_chunks(cl.cpt_off, 1 << 18))))
    return EmissionPlan(d, row, tg, geom, gd, sum(miss))


def tree_stats(tree: BoxTree, hier: ConeHierarchy | None = None) -> str:
    """JSON per-level box/segment counts (reference ifgf.py:926-950)."""
    rows = []
    for d in range(1, tree.depth + 1):
        lvl = tree.level(d)
        row = {"level": d, "side": lvl.side,
               "relevant_boxes": int(lvl.n_boxes),
               "max_points_per_box": int(lvl.pt_count.max())}
        if hier is not None and d in hier.cone_levels:
            cl = hier.level(d)
            row["cone_counts"] = [cl.n_s, cl.n_a]
            row["relevant_segments"] = int(cl.n_segments)
        rows.append(row)
    payload = {"depth": tree.depth, "root_side": tree.root_side,
               "points": int(tree.points.shape[0]), "levels": rows}
    if hier is not None:
        payload["spectra_bytes_vec16"] = hier.spectra_bytes(16)
    return json.dumps(payload, indent=2)
