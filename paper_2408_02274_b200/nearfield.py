"""Near-field plan: singular/near patch classification, singular moments and
the local-correction pair lists (plan time, host).

These are one-time precomputations whose OUTPUT the per-matvec device kernel
(``csrc/nearfield.cu``) consumes; restated from the reference so the framework
runs standalone:

* ``SingularQuadratureConfig``      -- reference ``quadrature.py:46-65``
* ``classify_targets``              -- reference ``quadrature.py:97-156``
* ``graded_map`` / ``clustered_nodes`` -- reference ``quadrature.py:163-228``
* ``compute_moments``               -- reference ``quadrature.py:271-331``
* ``compute_moments_device``       -- the same moments from the sm_100a
  kernel ``csrc/moments.cu`` (C ABI ``ifgfb_singular_moments``)
* ``correction_pairs``              -- reference ``quadrature.py:490-525``
  (only the (target, source) index lists; the device recomputes the kernel
  values, so no CSR values are stored)
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from . import cheb
from .octree import _pool
from .surface import SurfaceDiscretization, closest_point_batch

__all__ = ["SingularQuadratureConfig", "SingularityMap", "MomentGroup",
           "SingularMomentTable", "classify_targets", "graded_map",
           "clustered_nodes", "compute_moments", "compute_moments_device",
           "correction_pairs"]


@dataclass(frozen=True)
class SingularQuadratureConfig:
    d: int = 4
    n_beta: int | None = None
    delta_factor: float = 1.0

    def __post_init__(self):
        if self.d < 2:
            raise ValueError("grading order must be >= 2")

    def resolve_n_beta(self, n_c: int) -> int:
        n = self.n_beta if self.n_beta is not None else max(4 * n_c, 48)
        if n < n_c:
            raise ValueError("refined node count must be >= n_c")
        return n + (n % 2)


@dataclass
class SingularityMap:
    """CSR per target: singular/near patch ids, closest (u, v), distance.
    A rank's map (classify_targets(..., target_range=(lo, hi))) covers the
    on-surface targets lo..hi-1 only: local target j is point lo + j."""

    n_targets: int
    n_patches: int
    delta: np.ndarray
    offsets: np.ndarray
    patch_ids: np.ndarray
    closest_uv: np.ndarray
    dists: np.ndarray
    target_lo: int = 0

    def singular_patches(self, ell: int) -> np.ndarray:
        return self.patch_ids[self.offsets[ell]:self.offsets[ell + 1]]

    def pairs_for_patch(self, p: int):
        sel = np.nonzero(self.patch_ids == p)[0]
        tg = (np.searchsorted(self.offsets, sel, side="right") - 1).astype(
            np.int64)
        return tg, self.closest_uv[sel, 0], self.closest_uv[sel, 1]


def classify_targets(disc: SurfaceDiscretization,
                     config: SingularQuadratureConfig | None = None,
                     targets=None, target_range=None) -> SingularityMap:
    """(target, patch) is singular when dist <= delta_factor * spacing_p.

    target_range=(lo, hi): the map of the surface points lo..hi-1 only (a
    rank's targets).  Each patch still runs its closest-point search on its
    FULL candidate batch (the golden-section loop runs until the whole batch
    converges, so a point's (u, v) depends on its batch), hence the rank's
    rows equal the full map's rows bit for bit; patches with no candidate in
    the range are skipped."""
    config = config or SingularQuadratureConfig()
    on_surface = targets is None
    t0, t1 = 0, None
    pts = disc.points if on_surface else np.atleast_2d(
        np.asarray(targets, dtype=float))
    if on_surface and target_range is not None:
        t0, t1 = (int(v) for v in target_range)
        if not 0 <= t0 <= t1 <= disc.n_points:
            raise ValueError("target range out of bounds")
    t1 = pts.shape[0] if t1 is None else t1
    n_t = t1 - t0
    delta = config.delta_factor * disc.max_spacing
    grid = cheb.nodes(disc.n_c)
    global _CLASSIFY_CTX
    _CLASSIFY_CTX = (disc, pts, delta, grid, on_surface, t0, t1, _point_index(pts))
    # per-patch work is independent (the golden-section loops are
    # Python-bound: processes when fork is available, else in-process); each
    # patch returns its hits as arrays, merged here and sorted per target by
    # patch id (a patch appears at most once per target)
    parts = [(p, h) for p, h in enumerate(_map_patches(_classify_patch, disc.n_patches))
             if h is not None and h[0].size]
    _CLASSIFY_CTX = None
    if parts:
        ell = np.concatenate([h[0] for _, h in parts]) - t0
        pid = np.concatenate([np.full(h[0].size, p, dtype=np.int64) for p, h in parts])
        uv = np.concatenate([h[1] for _, h in parts])
        dist = np.concatenate([h[2] for _, h in parts])
        order = np.lexsort((pid, ell))
        ell, pid, uv, dist = ell[order], pid[order], uv[order], dist[order]
    else:
        ell = pid = np.empty(0, np.int64)
        uv, dist = np.empty((0, 2)), np.empty(0)
    offsets = np.zeros(n_t + 1, dtype=np.int64)
    np.cumsum(np.bincount(ell, minlength=n_t), out=offsets[1:])
    return SingularityMap(n_t, disc.n_patches, delta, offsets, pid.astype(np.int32),
                          np.ascontiguousarray(uv, dtype=float).reshape(-1, 2),
                          np.ascontiguousarray(dist, dtype=float), t0)


_CLASSIFY_CTX = None


def _point_index(pts):
    """k-d tree over the targets for the per-patch candidate search (the
    exact candidate test below is the reference's expression)."""
    try:
        from scipy.spatial import cKDTree
    except ImportError:       # pragma: no cover - scipy is a dependency
        return None
    return cKDTree(pts)


def _map_patches(fn, n_patches):
    """Map fn over patch ids in forked worker processes (results in order)."""
    import multiprocessing as mp
    import os
    workers = min(os.cpu_count() or 1, 32, n_patches)
    if workers > 1 and n_patches >= 16:
        import warnings
        try:
            with warnings.catch_warnings():
                # children only run numpy on the inherited (read-only) plan
                # inputs; a stuck worker falls back to in-process below
                warnings.simplefilter("ignore", DeprecationWarning)
                ctx = mp.get_context("fork")
                with ctx.Pool(workers) as pool:
                    res = pool.map_async(
                        fn, range(n_patches),
                        chunksize=max(1, n_patches // (4 * workers)))
                    return res.get(timeout=600 + n_patches)
        except (OSError, ValueError, mp.TimeoutError):
            pass
    return [fn(p) for p in range(n_patches)]


def _classify_patch(p):
    """Singular/near pairs of patch p (runs in a worker process): arrays
    (targets, (u, v), distances), or None.  Targets outside [t0, t1) are
    searched (same batch as the full map) but not reported."""
    hits = _classify_patch_list(p)
    if not hits:
        return None
    ell = np.array([h[0] for h in hits], dtype=np.int64)
    uv = np.array([(h[1][1], h[1][2]) for h in hits], dtype=float).reshape(-1, 2)
    dist = np.array([h[1][3] for h in hits], dtype=float)
    return ell, uv, dist


def _classify_patch_list(p):
    disc, pts, delta, grid, on_surface, t0, t1, kd = _CLASSIFY_CTX
    patch = disc.patches[p]
    hits = []
    if kd is not None:
        reach = (patch.bound_radius + delta[p]) * (1.0 + 1e-9) + 1e-300
        cand = np.sort(np.asarray(kd.query_ball_point(patch.center, reach), dtype=np.int64))
        lower = np.linalg.norm(pts[cand] - patch.center, axis=1) - patch.bound_radius
        cand = cand[lower <= delta[p]]
    else:
        lower = np.linalg.norm(pts - patch.center, axis=1) - patch.bound_radius
        cand = np.nonzero(lower <= delta[p])[0]
    if cand.size == 0 or not np.any((cand >= t0) & (cand < t1)):
        return hits
    mine = lambda ell: t0 <= ell < t1
    own = np.zeros(cand.size, dtype=bool)
    if on_surface:
        own = disc.patch_of[cand] == p
        for ell in cand[own]:
            if mine(ell):
                _, i, j = disc.decode_index(int(ell))
                hits.append((int(ell), (p, grid[i], grid[j], 0.0)))
    rest = cand[~own]
    if rest.size == 0:
        return hits
    seed = disc.patch_points(p).reshape(disc.n_c, disc.n_c, 3)
    dmin = np.min(np.linalg.norm(
        pts[rest][:, None, :] - seed.reshape(-1, 3)[None, :, :], axis=-1),
        axis=1)
    rest = rest[dmin - disc.max_spacing[p] <= delta[p]]
    if rest.size == 0 or not np.any((rest >= t0) & (rest < t1)):
        return hits
    u, v, dist = closest_point_batch(patch, pts[rest], seed)
    for ell, uu, vv, dd in zip(rest, u, v, dist):
        if dd <= delta[p] and mine(ell):
            hits.append((int(ell), (p, uu, vv, dd)))
    return hits


# ---------------------------------------------------------------------------
# graded clustered quadrature
# ---------------------------------------------------------------------------

def _nu(tau, d):
    return ((1.0 / d - 0.5) * ((np.pi - tau) / np.pi) ** 3
            + (tau - np.pi) / (d * np.pi) + 0.5)


def _nu_prime(tau, d):
    return (3.0 * (0.5 - 1.0 / d) * (np.pi - tau) ** 2 / np.pi**3
            + 1.0 / (d * np.pi))


def graded_map(tau, d: int):
    """Polynomially graded map of [0, 2pi] onto itself (order-d flat ends)."""
    if d < 2:
        raise ValueError("grading order must be >= 2")
    tau = np.asarray(tau, dtype=float)
    if np.any(tau < -1e-12) or np.any(tau > 2 * np.pi + 1e-12):
        raise ValueError("argument outside [0, 2*pi]")
    tau = np.clip(tau, 0.0, 2 * np.pi)
    a = _nu(tau, d) ** d
    b = _nu(2 * np.pi - tau, d) ** d
    return 2 * np.pi * a / (a + b)


def _graded_map_prime(tau, d):
    tau = np.asarray(tau, dtype=float)
    n1, n2 = _nu(tau, d), _nu(2 * np.pi - tau, d)
    dn1 = _nu_prime(tau, d)
    dn2 = -_nu_prime(2 * np.pi - tau, d)
    a, b = n1**d, n2**d
    da = d * n1 ** (d - 1) * dn1
    db = d * n2 ** (d - 1) * dn2
    return 2 * np.pi * (da * b - a * db) / (a + b) ** 2


def clustered_nodes(alpha, base, d: int):
    """Base nodes on [-1,1] remapped to accumulate at alpha (+ derivative)."""
    t = np.asarray(base, dtype=float)
    alpha = np.asarray(alpha, dtype=float)
    scalar = alpha.ndim == 0
    a = np.atleast_1d(alpha)[:, None]
    tt = np.broadcast_to(t, (a.shape[0], t.size))
    sg = np.sign(tt)
    w_mid = graded_map(np.pi * np.abs(tt), d)
    xi = a + (sg - a) / np.pi * w_mid
    dxi = (1.0 - a * sg) * _graded_map_prime(np.pi * np.abs(tt), d)
    hi = (a >= 1.0 - 1e-12)[:, 0]
    if hi.any():
        arg = np.pi * np.abs(tt[hi] - 1.0) / 2.0
        xi[hi] = 1.0 - (2.0 / np.pi) * graded_map(arg, d)
        dxi[hi] = _graded_map_prime(arg, d)
    lo = (a <= -1.0 + 1e-12)[:, 0]
    if lo.any():
        arg = np.pi * np.abs(tt[lo] + 1.0) / 2.0
        xi[lo] = -1.0 + (2.0 / np.pi) * graded_map(arg, d)
        dxi[lo] = _graded_map_prime(arg, d)
    if scalar:
        return xi[0], dxi[0]
    return xi, dxi


def clustered_nodes_many(alpha, base, d: int):
    """``clustered_nodes`` for many alphas at once, bitwise equal to it: the
    graded map (np.power, the costly part) depends on the base node only, so
    it is evaluated once on one row of base nodes and broadcast; the
    alpha-dependent remainder is the same elementwise expressions."""
    t = np.asarray(base, dtype=float)[None, :]
    a = np.asarray(alpha, dtype=float).reshape(-1)[:, None]
    sg = np.sign(t)
    arg = np.pi * np.abs(t)
    w_mid, g_mid = graded_map(arg, d), _graded_map_prime(arg, d)
    xi = a + (sg - a) / np.pi * w_mid
    dxi = (1.0 - a * sg) * g_mid
    for mask, arg, sign in (((a >= 1.0 - 1e-12)[:, 0], np.pi * np.abs(t - 1.0) / 2.0, 1.0),
                            ((a <= -1.0 + 1e-12)[:, 0], np.pi * np.abs(t + 1.0) / 2.0, -1.0)):
        if mask.any():
            w = graded_map(arg, d)
            xi[mask] = (1.0 - (2.0 / np.pi) * w) if sign > 0 else (-1.0 + (2.0 / np.pi) * w)
            dxi[mask] = _graded_map_prime(arg, d)
    return xi, dxi


@dataclass
class MomentGroup:
    targets: np.ndarray          # (B,)
    beta_s: np.ndarray           # (2, B, n_c, n_c)
    beta_d: np.ndarray           # (2, B, n_c, n_c)


@dataclass
class SingularMomentTable:
    n_c: int
    kappas: tuple
    groups: dict = field(default_factory=dict)
    corrections: object = None


def compute_moments(disc: SurfaceDiscretization, smap: SingularityMap,
                    config: SingularQuadratureConfig, kappas,
                    target_points=None, target_normals=None):
    """Integrals of G * T_m(u) T_n(v) * J (and of dG/dn_x) per singular pair
    on the graded grid clustered at the pair's closest point."""
    kappas = tuple(kappas)
    n_c = disc.n_c
    nb = config.resolve_n_beta(n_c)
    base = cheb.nodes(nb)
    wb = cheb.fejer(nb)
    pts = disc.points if target_points is None else target_points
    nrms = disc.normals if target_normals is None else target_normals
    table = SingularMomentTable(n_c, kappas)

    def one_patch(p):
        patch = disc.patches[p]
        tg, u0, v0 = smap.pairs_for_patch(int(p))
        b = tg.size
        xu, dxu = clustered_nodes(u0, base, config.d)
        xv, dxv = clustered_nodes(v0, base, config.d)
        tu = cheb.basis(patch.n, xu.ravel()).reshape(b, nb, patch.n)
        tv = cheb.basis(patch.n, xv.ravel()).reshape(b, nb, patch.n)
        tvt = tv.transpose(0, 2, 1)

        def on_grid(cf):
            return np.stack([tu @ cf[c] @ tvt for c in range(3)])

        pos = on_grid(patch.coeffs)
        eu = on_grid(patch.coeffs_du)
        ev = on_grid(patch.coeffs_dv)
        jac = np.linalg.norm(np.cross(np.moveaxis(eu, 0, -1),
                                      np.moveaxis(ev, 0, -1)), axis=-1)
        dx = pts[tg].T[:, :, None, None] - pos
        r = np.sqrt((dx**2).sum(axis=0))
        ndx = np.einsum("cbij,bc->bij", dx, nrms[tg])
        pu = cheb.basis(n_c, xu.ravel()).reshape(b, nb, n_c)
        pv = cheb.basis(n_c, xv.ravel()).reshape(b, nb, n_c)
        put = (pu * (dxu * wb)[:, :, None]).transpose(0, 2, 1).copy()
        pvw = (pv * (dxv * wb)[:, :, None]).copy()
        bs = np.empty((2, b, n_c, n_c), dtype=complex)
        bd = np.empty((2, b, n_c, n_c), dtype=complex)
        for k, kappa in enumerate(kappas):
            phase = np.exp(1j * kappa * r) / (4.0 * np.pi * r)
            ks = phase * jac
            kd = ks * (ndx * (1j * kappa * r - 1.0) / r**2)
            bs[k] = (put.astype(complex) @ ks) @ pvw
            bd[k] = (put.astype(complex) @ kd) @ pvw
        return int(p), MomentGroup(tg, bs, bd)

    for p, grp in _pool().map(one_patch, np.unique(smap.patch_ids)):
        table.groups[p] = grp
    return table


def compute_moments_device(disc: SurfaceDiscretization, smap: SingularityMap,
                           config: SingularQuadratureConfig, kappas,
                           target_points=None, target_normals=None,
                           groups: bool = True, exact: bool = True):
    """``compute_moments`` on the GPU (csrc/moments.cu): same table, the
    pairs' moments computed by one CTA each.

    exact=True (default): the graded nodes come from the host
    (``clustered_nodes``, the reference's np.power expressions) and the
    device replays the reference's float64 operation order for the patch
    geometry (csrc/moments.cu ``dot_exact``), so beta_s and beta_d agree with
    the reference to rounding.  exact=False: graded map on the device; beta_d
    then carries the ~1e-7 conditioning of (x - y).n_x at the clustered nodes
    (tests/test_gpu_moments.py).

    groups=False skips the per-patch regrouping: the table then carries the
    blocks in the singularity map's CSR order (``csr_blocks``, n_mom x 4 x
    n_c^2, target-major with ascending patch ids -- the order the near-field
    plan consumes) and an empty ``groups``."""
    import ctypes

    from . import _lib
    kappas = tuple(kappas)
    if len(kappas) != 2:
        raise ValueError("compute_moments_device: two wavenumbers")
    n_c = disc.n_c
    nb = config.resolve_n_beta(n_c)
    pts = disc.points if target_points is None else target_points
    nrms = disc.normals if target_normals is None else target_normals
    n_pairs = smap.patch_ids.size
    tg = np.repeat(np.arange(smap.n_targets, dtype=np.int64),
                   np.diff(smap.offsets))
    npg = disc.patches[0].n
    if any(p.n != npg for p in disc.patches):
        raise ValueError("compute_moments_device: patches of mixed order")
    cf = np.ascontiguousarray(np.stack(
        [np.concatenate([p.coeffs, p.coeffs_du, p.coeffs_dv]) for p in disc.patches]),
        dtype=np.float64)
    txyz = np.ascontiguousarray(pts[tg], dtype=np.float64)
    tnrm = np.ascontiguousarray(nrms[tg], dtype=np.float64)
    pid = np.ascontiguousarray(smap.patch_ids, dtype=np.int32)
    uv = np.ascontiguousarray(smap.closest_uv, dtype=np.float64)
    base = np.ascontiguousarray(cheb.nodes(nb), dtype=np.float64)
    wb = np.ascontiguousarray(cheb.fejer(nb), dtype=np.float64)
    kap = np.array([complex(kappas[0]).real, complex(kappas[0]).imag,
                    complex(kappas[1]).real, complex(kappas[1]).imag])
    out = np.empty((n_pairs, 4, n_c, n_c), dtype=np.complex128)
    dp = lambda a: a.ctypes.data_as(ctypes.POINTER(ctypes.c_double))
    # OpenBLAS's N-tail columns (empirical, OpenBLAS 0.3.30 SkylakeX: the
    # 20 x 20 patch products reduce columns 16..19 in 8 interleaved lanes)
    tail = lambda n: n - n % 16 if (n > 16 and n % 16) else 0
    lib = _lib.load()
    step = n_pairs if not exact else 1 << 20
    for c0 in range(0, max(n_pairs, 1), max(step, 1)):
        c1 = min(n_pairs, c0 + step)
        if c1 <= c0:
            break
        nodes = None
        if exact:
            nodes = np.empty((c1 - c0, 4, nb))
            nodes[:, 0], nodes[:, 1] = clustered_nodes_many(uv[c0:c1, 0], base, config.d)
            nodes[:, 2], nodes[:, 3] = clustered_nodes_many(uv[c0:c1, 1], base, config.d)
        desc = _lib.MomentDesc(c1 - c0, dp(txyz[c0:c1]), dp(tnrm[c0:c1]),
                               pid[c0:c1].ctypes.data_as(ctypes.POINTER(ctypes.c_int32)),
                               dp(uv[c0:c1]), disc.n_patches, npg, dp(cf), n_c, nb,
                               int(config.d), dp(base), dp(wb), dp(kap),
                               dp(nodes) if exact else None,
                               tail(npg) if exact else 0, tail(nb) if exact else 0)
        _lib.check(lib.ifgfb_singular_moments(ctypes.byref(desc),
                                              dp(out[c0:c1].view(np.float64))),
                   "ifgfb_singular_moments")
    table = SingularMomentTable(n_c, kappas)
    if not groups:
        table.csr_blocks = out.reshape(n_pairs, 4, n_c * n_c)
        return table
    order = np.argsort(smap.patch_ids, kind="stable")
    bounds = np.searchsorted(smap.patch_ids[order], np.arange(disc.n_patches + 1))
    for p in range(disc.n_patches):
        sel = order[bounds[p]:bounds[p + 1]]
        if sel.size == 0:
            continue
        blk = out[sel]
        table.groups[p] = MomentGroup(tg[sel], np.ascontiguousarray(blk[:, 0:2].transpose(1, 0, 2, 3)),
                                      np.ascontiguousarray(blk[:, 2:4].transpose(1, 0, 2, 3)))
    return table


@dataclass
class CorrectionPairs:
    """(target, source) pairs the far field double counts (sources on a
    target's singular patch lying >= 2 finest boxes away)."""

    ell_idx: np.ndarray
    src_idx: np.ndarray

    @property
    def nnz(self) -> int:
        return self.ell_idx.size


def correction_pairs(disc: SurfaceDiscretization, tree,
                     smap: SingularityMap) -> CorrectionPairs:
    """Entries per patch in ascending patch order (reference
    quadrature.py:490-525); targets are global point ids (a rank's map
    yields its targets' entries in the same order)."""
    coords = tree.point_level_coords(tree.depth)
    n2 = disc.n_c**2
    # (patch, target) pairs in ascending patch order, targets ascending
    # within a patch; chunks of pairs on the plan thread pool, each pair
    # against the patch's n_c^2 sources (Chebyshev-box separation >= 2)
    order = np.argsort(smap.patch_ids, kind="stable")
    pid = smap.patch_ids[order].astype(np.int64)
    tg = (np.repeat(np.arange(smap.n_targets, dtype=np.int64),
                    np.diff(smap.offsets)) + smap.target_lo)[order]
    step = max(1, (1 << 22) // n2)
    chunks = [(i, min(pid.size, i + step)) for i in range(0, pid.size, step)]

    def one(rng):
        i0, i1 = rng
        src = pid[i0:i1, None] * n2 + np.arange(n2)[None, :]
        sep = np.abs(coords[src] - coords[tg[i0:i1]][:, None, :]).max(-1)
        ti, si = np.nonzero(sep >= 2)
        return tg[i0:i1][ti], src[ti, si]

    res = list(_pool().map(one, chunks))
    ell = np.concatenate([r[0] for r in res]) if res else np.empty(0, dtype=np.int64)
    src = np.concatenate([r[1] for r in res]) if res else np.empty(0, dtype=np.int64)
    return CorrectionPairs(ell.astype(np.int64), src.astype(np.int64))
