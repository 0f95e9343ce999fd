"""N-Muller operator on the B200: host mirror of the reference operator API
whose ``apply``/``potentials`` run entirely on device through libifgfb200.

Mirrors reference ``operators.py``:
* ``MaterialPair``          -- operators.py:58-101
* ``DensityBlock``          -- operators.py:104-128
* ``OperatorConfig``        -- operators.py:131-141
* ``MullerOperator``        -- operators.py:207-412 (decode/encode/rhs on host;
  ``apply`` / ``potentials`` / ``apply_device`` on device)
* ``build_muller_operator`` -- operators.py:415-441
* ``from_reference``        -- wraps an existing reference ``MullerOperator``
  (the drop-in path: plan objects are read, never rebuilt)

There is no CPU fallback: without the CUDA library these raise.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib, cheb
from .engine import FarFieldPlan, _StageLog, device_stream
from .nearfield import (SingularQuadratureConfig, classify_targets,
                        compute_moments, compute_moments_device,
                        correction_pairs)
from .octree import IfgfConfig, build_box_tree, build_cone_hierarchy

__all__ = ["MaterialPair", "DensityBlock", "OperatorConfig", "MullerOperator",
           "build_muller_operator", "from_reference", "surface_divergence",
           "J_X", "J_Y", "J_Z", "M_X", "M_Y", "M_Z", "DIV_J", "DIV_M"]

J_X, J_Y, J_Z, M_X, M_Y, M_Z, DIV_J, DIV_M = range(8)


@dataclass(frozen=True)
class MaterialPair:
    eps_e: complex
    mu_e: complex
    eps_i: complex
    mu_i: complex
    omega: float

    def __post_init__(self):
        if not self.omega > 0:
            raise ValueError("angular frequency must be positive")

    @property
    def kappa_e(self):
        return self.omega * np.sqrt(self.eps_e * self.mu_e)

    @property
    def kappa_i(self):
        return self.omega * np.sqrt(self.eps_i * self.mu_i)

    @property
    def kappas(self):
        return (self.kappa_e, self.kappa_i)

    @classmethod
    def from_wavenumbers(cls, kappa_e, kappa_i, eps_e=1.0, mu_e=1.0,
                         mu_i=1.0):
        omega = float(np.real(kappa_e / np.sqrt(eps_e * mu_e)))
        eps_i = (kappa_i / omega) ** 2 / mu_i
        pair = cls(eps_e, mu_e, eps_i, mu_i, omega)
        if abs(pair.kappa_i - kappa_i) > 1e-12 * abs(kappa_i):
            raise ValueError("inconsistent wavenumber inputs")
        return pair

    def check_consistency(self, kappa_e=None, kappa_i=None):
        for given, own in ((kappa_e, self.kappa_e), (kappa_i, self.kappa_i)):
            if given is not None and abs(given - own) > 1e-12 * abs(own):
                raise ValueError("wavenumbers inconsistent with eps/mu/omega")


@dataclass(frozen=True)
class OperatorConfig:
    fd_step: float = 1e-6
    mode: str = "vec"

    def __post_init__(self):
        if not self.fd_step > 0:
            raise ValueError("finite-difference step must be positive")


def _metric(disc):
    e = np.einsum("ij,ij->i", disc.e_u, disc.e_u)
    f = np.einsum("ij,ij->i", disc.e_u, disc.e_v)
    g = np.einsum("ij,ij->i", disc.e_v, disc.e_v)
    return e, f, g, e * g - f * f


def surface_divergence(disc, density, tol: float = 1e-8) -> np.ndarray:
    """Host surface divergence (plan-time / API helper; the device computes
    the same quantity inside ``apply``).  Reference operators.py:170-189."""
    density = np.asarray(density)
    normal_part = np.abs(np.einsum("ij,ij->i", density, disc.normals))
    scale = np.linalg.norm(density, axis=1).max() + 1e-300
    if normal_part.max() > tol * max(scale, 1.0):
        raise ValueError("density is not tangential")
    e, f, g, det = _metric(disc)
    cu = np.einsum("ij,ij->i", density, disc.e_u)
    cv = np.einsum("ij,ij->i", density, disc.e_v)
    fu = (g * cu - f * cv) / det
    fv = (e * cv - f * cu) / det
    jac = disc.jacobians
    n_c = disc.n_c
    dmat = cheb.diff_matrix(n_c)
    gu = (jac * fu).reshape(disc.n_patches, n_c, n_c)
    gv = (jac * fv).reshape(disc.n_patches, n_c, n_c)
    du = np.matmul(dmat[None], gu).reshape(-1)
    dv = np.matmul(gv, dmat.T[None]).reshape(-1)
    return (du + dv) / jac


@dataclass
class DensityBlock:
    values: np.ndarray          # (8, N) complex

    @property
    def j(self):
        return self.values[J_X:J_Z + 1].T

    @property
    def m(self):
        return self.values[M_X:M_Z + 1].T

    @classmethod
    def from_currents(cls, disc, j, m) -> "DensityBlock":
        vals = np.empty((8, disc.n_points), dtype=complex)
        vals[J_X:J_Z + 1] = np.asarray(j, dtype=complex).T
        vals[M_X:M_Z + 1] = np.asarray(m, dtype=complex).T
        vals[DIV_J] = surface_divergence(disc, j)
        vals[DIV_M] = surface_divergence(disc, m)
        return cls(vals)


def _c(a, dt):
    return np.ascontiguousarray(a, dtype=dt)


def _complex2(z) -> np.ndarray:
    z = complex(z)
    return np.array([z.real, z.imag])


def _near_desc(disc, tree, smap, moments, corr_ell, corr_src, keep):
    """Per-target singular moment pairs and the signed direct list.  A
    rank's map (smap.target_lo, smap.n_targets) yields entries for its
    targets only; the per-target offsets stay full length (N + 1) with
    empty ranges elsewhere, so the device indexes targets globally."""
    n, n_c = disc.n_points, disc.n_c
    n2 = n_c * n_c
    t0 = int(getattr(smap, "target_lo", 0))
    t1 = t0 + int(smap.n_targets)
    # ---- moments, per (target, patch) sorted by target then patch
    tg, pt, blocks = [], [], []
    csr = getattr(moments, "csr_blocks", None)
    if csr is not None:   # device moments, already in the map's CSR order
        pt = _c(smap.patch_ids, np.int64)
        blocks = np.ascontiguousarray(csr)
        tg = np.repeat(np.arange(t0, t1, dtype=np.int64), np.diff(smap.offsets))
    for p in sorted(moments.groups) if csr is None else ():
        grp = moments.groups[p]
        tg.append(np.asarray(grp.targets, dtype=np.int64) + t0)
        pt.append(np.full(grp.targets.size, p, dtype=np.int64))
        blk = np.stack([grp.beta_s[0], grp.beta_s[1], grp.beta_d[0],
                        grp.beta_d[1]], axis=1).reshape(-1, 4, n2)
        blocks.append(blk)
    if csr is None:
        tg = np.concatenate(tg) if tg else np.empty(0, np.int64)
        pt = np.concatenate(pt) if pt else np.empty(0, np.int64)
        blocks = (np.concatenate(blocks) if blocks
                  else np.empty((0, 4, n2), complex))
        order = np.lexsort((pt, tg))
        tg, pt, blocks = tg[order], pt[order], np.ascontiguousarray(blocks[order])
    mom_off = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(np.bincount(tg, minlength=n), out=mom_off[1:])
    # ---- + neighbour-box sources not on the target's singular patches
    d = tree.depth
    lvl = tree.level(d)
    tgt = np.arange(t0, t1, dtype=np.int64)
    box_of = np.searchsorted(lvl.codes, tree.point_codes[tree.iperm[tgt]])
    nb_lo = lvl.nbr_off[box_of]
    nb_hi = lvl.nbr_off[box_of + 1]
    cnt = nb_hi - nb_lo
    own = np.repeat(tgt, cnt)
    starts = np.cumsum(cnt) - cnt
    nb = lvl.nbr_idx[np.arange(own.size) - np.repeat(starts - nb_lo, cnt)]
    pc = lvl.pt_count[nb]
    own2 = np.repeat(own, pc)
    st2 = np.cumsum(pc) - pc
    src_t = np.arange(own2.size) - np.repeat(st2, pc) + np.repeat(
        lvl.pt_start[nb], pc)
    src = tree.perm[src_t]
    P = disc.n_patches
    sing_key = (np.repeat(tgt, np.diff(smap.offsets)) * P +
                smap.patch_ids.astype(np.int64))
    pair_key = own2 * P + disc.patch_of[src].astype(np.int64)
    keep_mask = ~np.isin(pair_key, sing_key)
    pos_t, pos_s = own2[keep_mask], src[keep_mask]
    # ---- - corrections
    neg_t = np.asarray(corr_ell, dtype=np.int64)
    if neg_t.size and (neg_t.min() < t0 or neg_t.max() >= t1):
        raise ValueError("correction targets outside the map's target range")
    neg_s = -np.asarray(corr_src, dtype=np.int64) - 1
    all_t = np.concatenate([pos_t, neg_t])
    all_s = np.concatenate([pos_s, neg_s])
    order = np.lexsort((np.arange(all_t.size), all_t))
    dir_src = np.ascontiguousarray(all_s[order])
    dir_off = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(np.bincount(all_t, minlength=n), out=dir_off[1:])
    arrs = [mom_off, _c(pt, np.int64), blocks, dir_off, dir_src]
    keep.extend(arrs)
    desc = _lib.NearDesc(tg.size, _lib.iptr(mom_off), _lib.iptr(arrs[1]),
                         _lib.dptr(blocks), dir_src.size, _lib.iptr(dir_off),
                         _lib.iptr(dir_src))
    return desc, {"moment_pairs": int(tg.size), "neighbor_entries":
                  int(pos_t.size), "correction_entries": int(neg_t.size),
                  "targets": (t0, t1)}


def _surface_desc(disc, materials, fd_step, keep):
    arrs = dict(
        pts=_c(disc.points, np.float64), nrm=_c(disc.normals, np.float64),
        w=_c(disc.weights, np.float64), jac=_c(disc.jacobians, np.float64),
        eu=_c(disc.e_u, np.float64), ev=_c(disc.e_v, np.float64),
        t1=_c(disc.tangent1, np.float64), t2=_c(disc.tangent2, np.float64),
        dm=_c(cheb.diff_matrix(disc.n_c), np.float64),
        cm=_c(cheb.to_coeff_matrix(disc.n_c), np.float64),
        ee=_complex2(materials.eps_e), me=_complex2(materials.mu_e),
        ei=_complex2(materials.eps_i), mi=_complex2(materials.mu_i),
        kap=np.concatenate([_complex2(materials.kappa_e),
                            _complex2(materials.kappa_i)]))
    keep.extend(arrs.values())
    D = _lib.dptr
    return _lib.SurfaceDesc(
        disc.n_patches, disc.n_c, D(arrs["pts"]), D(arrs["nrm"]),
        D(arrs["w"]), D(arrs["jac"]), D(arrs["eu"]), D(arrs["ev"]),
        D(arrs["t1"]), D(arrs["t2"]), D(arrs["dm"]), D(arrs["cm"]),
        D(arrs["ee"]), D(arrs["me"]), D(arrs["ei"]), D(arrs["mi"]),
        float(materials.omega), D(arrs["kap"]), float(fd_step))


class MullerOperator:
    """Matrix-free N-Muller system on device; y = [m1, m2, j1, j2] blocks in
    the per-point tangent frame (reference operators.py:207-211)."""

    def __init__(self, disc, materials, smap, moments, corrections,
                 config: OperatorConfig = OperatorConfig(), tree=None,
                 hierarchy=None, stream_parts=None,
                 geometry_on_device: str | None = None, seam: str = "unwrap",
                 near_tree=None):
        """seam: "unwrap" (default) or "reference" phi branch of the
        displaced emission points (octree.emission_plan, DESIGN 2).
        near_tree: the whole tree for the near-field neighbour lists when
        ``tree`` is a window view (multi-GPU ranks); default ``tree``."""
        self.disc = disc
        self.materials = materials
        self.smap = smap
        self.moments = moments
        self.corrections = corrections
        self.config = config
        self.tree = tree
        self.hierarchy = hierarchy
        self.accelerated = True
        self.corrections_enabled = True
        keep = []
        log = _StageLog("operator")
        corr_ell, corr_src = corrections
        surf = _surface_desc(disc, materials, config.fd_step, keep)
        near, self.near_stats = _near_desc(disc, tree if near_tree is None else near_tree,
                                           smap, moments, corr_ell, corr_src, keep)
        log("near-field description")
        self.plan = FarFieldPlan(tree, hierarchy, disc.normals,
                                 config.fd_step, surface=surf, near=near,
                                 kappas=materials.kappas,
                                 geometry_on_device=geometry_on_device, seam=seam)
        # memory: stream the upward pass over groups of level-3 subtrees when
        # two full coefficient levels do not fit (None = automatic)
        if stream_parts is None:
            self.plan.auto_stream()
        elif stream_parts > 1:
            self.plan.set_streaming(stream_parts)
        log("device plan")
        del keep
        self._dev = torch.device("cuda")

    @property
    def n_unknowns(self) -> int:
        return 4 * self.disc.n_points

    # ---- host-side encoding helpers (reference operators.py:230-245)
    def decode(self, y):
        n = self.disc.n_points
        y = np.asarray(y, dtype=complex)
        if y.size != 4 * n:
            raise ValueError("unknown vector has wrong length")
        t1, t2 = self.disc.tangent1, self.disc.tangent2
        m = y[0:n, None] * t1 + y[n:2 * n, None] * t2
        j = y[2 * n:3 * n, None] * t1 + y[3 * n:, None] * t2
        return m, j

    def encode(self, m, j):
        t1, t2 = self.disc.tangent1, self.disc.tangent2
        return np.concatenate([
            np.einsum("ij,ij->i", m, t1), np.einsum("ij,ij->i", m, t2),
            np.einsum("ij,ij->i", j, t1), np.einsum("ij,ij->i", j, t2)])

    def rhs(self, incident):
        e_inc, h_inc = incident.fields(self.disc.points)
        nrm = self.disc.normals
        return self.encode(np.cross(nrm, e_inc) / self.materials.omega,
                           np.cross(nrm, h_inc) / self.materials.omega)

    # ---- device paths
    def _check(self):
        if not self.accelerated:
            raise NotImplementedError(
                "the dense O(N^2) path is not part of the B200 build")
        if not self.corrections_enabled:
            raise NotImplementedError("corrections toggle not supported")

    def apply_device(self, y: torch.Tensor, out: torch.Tensor | None = None):
        """A y for a device complex128 tensor of length 4N (no host copies)."""
        self._check()
        if y.numel() != self.n_unknowns:
            raise ValueError("unknown vector has wrong length")
        y = y.contiguous()
        if out is None:
            out = torch.empty_like(y)
        _lib.check(_lib.load().ifgfb_muller_apply(
            self.plan.handle, y.data_ptr(), out.data_ptr(), device_stream()),
            "ifgfb_muller_apply")
        return out

    def apply(self, y) -> np.ndarray:
        """Host numpy in / out (reference operators.py:399-403)."""
        self._check()
        y = np.ascontiguousarray(np.asarray(y, dtype=complex).ravel())
        if y.size != self.n_unknowns:
            raise ValueError("unknown vector has wrong length")
        out = np.empty_like(y)
        _lib.check(_lib.load().ifgfb_muller_apply_host(
            self.plan.handle, y.ctypes.data_as(ctypes.c_void_p),
            out.ctypes.data_as(ctypes.c_void_p), device_stream()),
            "ifgfb_muller_apply_host")
        return out

    def potentials(self, dens: DensityBlock):
        """(S (8,2,N), D (6,2,N)) of packed densities (operators.py:321)."""
        self._check()
        n = self.disc.n_points
        phi = torch.from_numpy(np.ascontiguousarray(
            dens.values, dtype=np.complex128)).to(self._dev)
        s = torch.empty((8, 2, n), dtype=torch.complex128, device=self._dev)
        d = torch.empty((6, 2, n), dtype=torch.complex128, device=self._dev)
        _lib.check(_lib.load().ifgfb_potentials(
            self.plan.handle, phi.data_ptr(), s.data_ptr(), d.data_ptr(),
            device_stream()), "ifgfb_potentials")
        return s.cpu().numpy(), d.cpu().numpy()

    def last_launches(self) -> int:
        return self.plan.last_launches()


def build_muller_operator(disc, materials, quad_config=None, ifgf_config=None,
                          op_config=None, accelerated: bool = True, smap=None,
                          moments=None, device_moments: bool = False) -> MullerOperator:
    """Plan (classification, moments, octree, cones, corrections) on the
    host, then the device plan (reference operators.py:415-441).
    device_moments: singular moments from the GPU kernel (csrc/moments.cu)
    instead of the host restatement -- much faster plan for large surfaces;
    beta_d then differs from the reference's at its ~1e-7 conditioning, so
    parity runs keep the host moments (tests/test_gpu_moments.py)."""
    if not accelerated:
        raise NotImplementedError(
            "the dense O(N^2) path is not part of the B200 build")
    quad_config = quad_config or SingularQuadratureConfig()
    op_config = op_config or OperatorConfig()
    if smap is None:
        smap = classify_targets(disc, quad_config)
    if moments is None and device_moments:
        moments = compute_moments_device(disc, smap, quad_config, materials.kappas,
                                         groups=False)
    elif moments is None:
        moments = compute_moments(disc, smap, quad_config, materials.kappas)
    kmax = max(abs(materials.kappa_e), abs(materials.kappa_i))
    tree = build_box_tree(disc.points, kmax)
    hier = build_cone_hierarchy(tree, ifgf_config or IfgfConfig())
    cp = correction_pairs(disc, tree, smap)
    return MullerOperator(disc, materials, smap, moments,
                          (cp.ell_idx, cp.src_idx), op_config, tree, hier)


def from_reference(ref_op) -> MullerOperator:
    """Device operator from a reference ``emscat`` MullerOperator: its
    SurfaceDiscretization, SingularityMap, moment table, correction lists,
    BoxTree and ConeHierarchy are read as they are (drop-in path)."""
    cs = ref_op.moments.corrections
    return MullerOperator(ref_op.disc, ref_op.materials, ref_op.smap,
                          ref_op.moments, (cs.ell_idx, cs.src_idx),
                          ref_op.config, ref_op.tree, ref_op.hierarchy)
