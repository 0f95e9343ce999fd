"""CPU ORACLE (test infrastructure only -- never imported by the product).

Plain numpy restatement of the reference N-Muller forward map, used as the
checker for the CUDA path and as the timed CPU baseline in bench.py.  Each
function cites the reference file:line it restates (paths relative to the
reference's pkg/src/emscat/).

Plan inputs (BoxTree, ConeHierarchy with the reference's attribute layout,
SingularityMap, moment table, correction (target, source) lists) are
consumed as given; everything computed per matvec is restated here.
"""

from __future__ import annotations

import time
from dataclasses import dataclass, field

import numpy as np

# ---------------------------------------------------------------------------
# Chebyshev helpers (chebyshev.py:60-138)
# ---------------------------------------------------------------------------


def _cheb_vals(n, x):
    x = np.atleast_1d(np.asarray(x, dtype=float))
    t = np.empty((x.size, n))
    t[:, 0] = 1.0
    if n > 1:
        t[:, 1] = x
    for i in range(2, n):
        t[:, i] = 2.0 * x * t[:, i - 1] - t[:, i - 2]
    return t


def _grid(n):
    return np.cos((np.arange(n) + 0.5) * np.pi / n)


def _fwd(n):
    m = (2.0 / n) * _cheb_vals(n, _grid(n)).T
    m[0] *= 0.5
    return m


def _dmat(n):
    """Spectral differentiation on the n-point open grid."""
    der = np.zeros((n, n))
    for col in range(n):
        a = np.zeros(n)
        a[col] = 1.0
        b = np.zeros(n)
        for k in range(n - 1, 0, -1):
            b[k - 1] = (b[k + 1] if k + 1 < n else 0.0) + 2.0 * k * a[k]
        b[0] *= 0.5
        der[:, col] = b
    return _cheb_vals(n, _grid(n)) @ der @ _fwd(n)


# ---------------------------------------------------------------------------
# cone geometry (ifgf.py:305-387)
# ---------------------------------------------------------------------------


def _cone(dx, side):
    r = np.linalg.norm(dx, axis=-1)
    s = np.sqrt(3.0) / 2.0 * side / r
    th = np.arccos(np.clip(dx[:, 2] / r, -1.0, 1.0))
    ph = np.mod(np.arctan2(dx[:, 1], dx[:, 0]), 2.0 * np.pi)
    return s, th, ph, r


def _flat(cl, s, th, ph):
    i_s = np.minimum((s / cl.delta_s).astype(np.int64), cl.n_s - 1)
    i_t = np.minimum((th / cl.delta_a).astype(np.int64), cl.n_a - 1)
    i_p = np.minimum((ph / cl.delta_a).astype(np.int64), 2 * cl.n_a - 1)
    return (i_s * cl.n_a + i_t) * (2 * cl.n_a) + i_p


def _unflat(cl, f):
    two = 2 * cl.n_a
    return (f // two) // cl.n_a, (f // two) % cl.n_a, f % two


def _local(cl, f, s, th, ph):
    i_s, i_t, i_p = _unflat(cl, f)
    return (2.0 * (s / cl.delta_s - i_s) - 1.0,
            2.0 * (th / cl.delta_a - i_t) - 1.0,
            2.0 * (ph / cl.delta_a - i_p) - 1.0)


def _nodes(cl, f, center):
    """(nseg, nodes, 3) interpolation nodes about `center` and radii."""
    i_s, i_t, i_p = _unflat(cl, f)
    r = cl.h / cl.s_nodes[i_s]
    th, ph = cl.ang_nodes_t[i_t], cl.ang_nodes_p[i_p]
    st, ct, cp, sp = np.sin(th), np.cos(th), np.cos(ph), np.sin(ph)
    d = np.stack([st[:, :, None] * cp[:, None, :], st[:, :, None] * sp[:, None, :],
                  np.broadcast_to(ct[:, :, None], (f.size, th.shape[1], ph.shape[1]))],
                 axis=-1)
    xyz = center + r[:, :, None, None, None] * d[:, None]
    rr = np.broadcast_to(r[:, :, None, None], xyz.shape[:-1]).reshape(f.size, -1)
    return xyz.reshape(f.size, -1, 3), rr


def _basis(ps, pa, xs, xt, xp):
    b = (_cheb_vals(ps, xs)[:, :, None, None] * _cheb_vals(pa, xt)[:, None, :, None]
         * _cheb_vals(pa, xp)[:, None, None, :])
    return b.reshape(xs.shape[0], -1)


def _row_keys(cl):
    stride = np.int64(cl.n_s * cl.n_a * 2 * cl.n_a + 1)
    nb = cl.seg_off.size - 1
    return stride, np.repeat(np.arange(nb, dtype=np.int64), np.diff(cl.seg_off)) * stride + cl.seg_ids


def _coeffs(vals, ps, pa):
    """Node values (nseg, ps*pa*pa, C) -> tensor Chebyshev coefficients
    (ifgf.py:502-522): one real matrix per axis applied to the interleaved
    real view of the complex data."""
    n, _, c = vals.shape

    def axis(mat, arr, left, m, right):
        a = np.ascontiguousarray(arr).reshape(left, m, right).view(np.float64)
        return np.matmul(mat[None], a).view(complex)

    v = axis(_fwd(ps), vals, n, ps, pa * pa * c)
    v = axis(_fwd(pa), v, n * ps, pa, pa * c)
    v = axis(_fwd(pa), v, n * ps * pa, pa, c)
    return v.reshape(n, ps * pa * pa, c)


# ---------------------------------------------------------------------------
# far field (ifgf.py:788-923)
# ---------------------------------------------------------------------------


def far_field(tree, hier, weights, kappas, normals=None, step=1e-6,
              box_stride: int = 1, box_ranges: dict | None = None):
    """out[c, k, ell] = sum over sources outside ell's finest neighbour boxes
    of G_k(x_ell, y) w[c, y] (and the same at x_ell + step * n_ell).

    box_stride > 1 processes only boxes b % box_stride == 0 (leaf spectra,
    emission, propagation): a bounded, scalable CPU-baseline sample whose
    output is NOT the full result.

    box_ranges {level d: (lo, hi)} restricts the upward pass to those boxes
    per level (one rank of the multi-GPU partition): the result is that
    rank's partial sum; summing the partials of a partition gives the full
    far field.
    """
    cfg = hier.config
    ps, pa = cfg.p_s, cfg.p_a
    nn = ps * pa * pa
    kap = np.asarray(tuple(kappas))
    nk = kap.size
    w_t = np.atleast_2d(weights)[:, tree.perm]
    nch = w_t.shape[0]
    n = tree.points.shape[0]
    out = np.zeros((n, nch, nk), dtype=complex)
    outd = np.zeros_like(out) if normals is not None else None
    if tree.depth < 3:
        out = out.transpose(1, 2, 0)
        return out, (None if outd is None else outd.transpose(1, 2, 0))
    disp = None
    if normals is not None:
        disp = tree.points + step * np.asarray(normals)[tree.perm]
    D = tree.depth
    # segment-row window per level: only the rows of the processed boxes are
    # materialised (whole level without box_ranges)
    win = {}
    for d in range(3, D + 1):
        lo, hi = ((0, tree.level(d).n_boxes) if box_ranges is None
                  else box_ranges[d])
        win[d] = (int(hier.level(d).seg_off[lo]), int(hier.level(d).seg_off[hi]))
    # --- leaf values (ifgf.py:535-554)
    cl, lvl = hier.level(D), tree.level(D)
    base = win[D][0]
    vals = np.zeros((win[D][1] - base, nn, nch, nk), dtype=complex)
    for b in _boxes(box_ranges, D, lvl.n_boxes, box_stride):
        g0, g1 = cl.seg_off[b], cl.seg_off[b + 1]
        r0, r1 = g0 - base, g1 - base
        if r1 == r0:
            continue
        xyz, rt = _nodes(cl, cl.seg_ids[g0:g1], lvl.centers[b])
        x = xyz.reshape(-1, 3)
        src = np.arange(lvl.pt_start[b], lvl.pt_start[b] + lvl.pt_count[b])
        dist = np.linalg.norm(x[:, None, :] - tree.points[src][None], axis=-1)
        rt = rt.reshape(-1, 1)
        for k in range(nk):
            g = rt / dist * np.exp(1j * kap[k] * (dist - rt))
            vals[r0:r1, :, :, k] = (g @ w_t[:, src].T).reshape(r1 - r0, nn, nch)
    for d in range(D, 2, -1):
        cl, lvl = hier.level(d), tree.level(d)
        coef = _coeffs(vals.reshape(vals.shape[0], nn, -1), ps, pa)
        _emit(tree, hier, d, coef, kap, nch, out, outd, disp, box_stride,
              box_ranges, win[d][0])
        if d > 3:
            vals = _propagate(tree, hier, d, coef, kap, nch, box_stride,
                              box_ranges, win[d][0], win[d - 1])
    out = out.transpose(1, 2, 0)[:, :, tree.iperm]
    if outd is not None:
        outd = outd.transpose(1, 2, 0)[:, :, tree.iperm]
    return out, outd


def _boxes(box_ranges, d, n_boxes, stride):
    lo, hi = (0, n_boxes) if box_ranges is None else box_ranges[d]
    return range(lo, hi, stride) if stride > 1 else range(lo, hi)


def _emit(tree, hier, d, coef, kap, nch, out, outd, disp, box_stride,
          box_ranges=None, row_base=0):
    """Cousin-point evaluation of level-d interpolants (ifgf.py:630-673)."""
    cfg = hier.config
    cl, lvl = hier.level(d), tree.level(d)
    nk = kap.size
    stride, keys = _row_keys(cl)
    boxes = np.array(list(_boxes(box_ranges, d, lvl.n_boxes, box_stride)),
                     dtype=np.int64)
    cnt = cl.cpt_off[boxes + 1] - cl.cpt_off[boxes]
    box = np.repeat(boxes, cnt)
    if box.size == 0:
        return
    sel = np.concatenate([np.arange(cl.cpt_off[b], cl.cpt_off[b + 1]) for b in boxes])
    tg = cl.cpt_idx[sel]
    ctr = lvl.centers[box]
    s, th, ph, r = _cone(tree.points[tg] - ctr, lvl.side)
    f = _flat(cl, s, th, ph)
    rows = np.searchsorted(keys, box * stride + f) - row_base
    pts = [(s, th, ph, r, out)]
    if outd is not None:
        pts.append(_cone(disp[tg] - ctr, lvl.side) + (outd,))
    chunk = 4096
    for (ss, tt, pp, rr, dst) in pts:
        xs, xt, xp = _local(cl, f, ss, tt, pp)
        fac = np.exp(1j * np.multiply.outer(rr, kap)) / (4.0 * np.pi * rr)[:, None]
        for a in range(0, tg.size, chunk):
            z = slice(a, min(tg.size, a + chunk))
            bas = _basis(cfg.p_s, cfg.p_a, xs[z], xt[z], xp[z])
            # real basis against the interleaved real view of the complex
            # coefficients (the reference's dgemm trick, ifgf.py:594-611)
            cv = coef[rows[z]].view(np.float64)
            v = np.matmul(bas[:, None, :], cv)[:, 0].view(complex).reshape(-1, nch, nk)
            v *= fac[z][:, None, :]
            np.add.at(dst, tg[z], v)


def _propagate(tree, hier, d, coef, kap, nch, box_stride, box_ranges=None,
               row_base=0, parent_win=None):
    """Fold level-d interpolants into the level-(d-1) node values
    (ifgf.py:676-785): per (parent segment id, child octant) type, the
    parent nodes in child coordinates, their child segments and the
    re-centering ratio."""
    cfg = hier.config
    ps, pa = cfg.p_s, cfg.p_a
    nn = ps * pa * pa
    nk = kap.size
    cl, lvl = hier.level(d), tree.level(d)
    pcl = hier.level(d - 1)
    stride, keys = _row_keys(cl)
    plo, phi = parent_win if parent_win is not None else (0, pcl.n_segments)
    pvals = np.zeros((phi - plo, nn, nch, nk), dtype=complex)
    flat_c = coef.reshape(coef.shape[0], nn, -1)
    octant = (lvl.codes & np.uint64(7)).astype(np.int64)
    inst = {}
    for b in _boxes(box_ranges, d, lvl.n_boxes, box_stride):
        pb = lvl.parent[b]
        for p in range(pcl.seg_off[pb], pcl.seg_off[pb + 1]):
            inst.setdefault((int(pcl.seg_ids[p]), int(octant[b])), []).append((p, b))
    half = 0.5 * lvl.side
    for (gam, octv), lst in inst.items():
        sgn = np.array([(octv >> 2) & 1, (octv >> 1) & 1, octv & 1]) * 2.0 - 1.0
        xyz, rp = _nodes(pcl, np.array([gam]), -(half * sgn))
        s, th, ph, rc = _cone(xyz[0], lvl.side)
        f = _flat(cl, s, th, ph)
        xs, xt, xp = _local(cl, f, s, th, ph)
        bas = _basis(ps, pa, xs, xt, xp)
        ratio = (rp[0] / rc)[:, None] * np.exp(1j * np.multiply.outer(rc - rp[0], kap))
        prow = np.array([q[0] for q in lst])
        kids = np.array([q[1] for q in lst])
        for sig in np.unique(f):
            nodes = np.nonzero(f == sig)[0]
            rows = np.searchsorted(keys, kids * stride + sig) - row_base
            blk = flat_c[rows].view(np.float64)                  # (inst, nn, 2C)
            v = np.matmul(bas[nodes], blk).view(complex).reshape(len(lst), nodes.size, nch, nk)
            v *= ratio[nodes][None, :, None, :]
            pvals[prow[:, None] - plo, nodes[None, :]] += v
    return pvals


# ---------------------------------------------------------------------------
# operator (operators.py:121-412, quadrature.py:343-487)
# ---------------------------------------------------------------------------


@dataclass
class OperatorData:
    """Plan inputs of one N-Muller operator."""

    disc: object
    materials: object
    smap: object
    moments: object
    corr_ell: np.ndarray
    corr_src: np.ndarray
    tree: object
    hier: object
    fd_step: float = 1e-6
    _nbr: list = field(default_factory=list)


def _metric(disc):
    e = np.einsum("ij,ij->i", disc.e_u, disc.e_u)
    f = np.einsum("ij,ij->i", disc.e_u, disc.e_v)
    g = np.einsum("ij,ij->i", disc.e_v, disc.e_v)
    return e, f, g, e * g - f * f


def _uv_derivs(disc, fields):
    nc = disc.n_c
    dm = _dmat(nc)
    lead = fields.shape[:-1]
    gr = fields.reshape(-1, disc.n_patches, nc, nc)
    du = np.matmul(dm[None, None], gr)
    dv = np.matmul(gr, dm.T[None, None])
    return du.reshape(lead + (-1,)), dv.reshape(lead + (-1,))


def _divergence(disc, vec):
    e, f, g, det = _metric(disc)
    cu = np.einsum("ij,ij->i", vec, disc.e_u)
    cv = np.einsum("ij,ij->i", vec, disc.e_v)
    jac = disc.jacobians
    du, _ = _uv_derivs(disc, (jac * (g * cu - f * cv) / det)[None])
    _, dv = _uv_derivs(disc, (jac * (e * cv - f * cu) / det)[None])
    return (du[0] + dv[0]) / jac


def _grads(disc, fields):
    e, f, g, det = _metric(disc)
    du, dv = _uv_derivs(disc, fields)
    a = (g * du - f * dv) / det
    b = (e * dv - f * du) / det
    return a[..., None] * disc.e_u + b[..., None] * disc.e_v


def _neighbor_sums(op, phi, kap, stride=1):
    disc, tree, smap = op.disc, op.tree, op.smap
    lvl = tree.level(tree.depth)
    n = disc.n_points
    s_out = np.zeros((8, 2, n), dtype=complex)
    d_out = np.zeros((6, 2, n), dtype=complex)
    phiw = (phi * disc.weights).T
    pt = disc.points[tree.perm]
    nt = disc.normals[tree.perm]
    ptch = disc.patch_of
    for b in range(0, lvl.n_boxes, stride):
        tt = np.arange(lvl.pt_start[b], lvl.pt_start[b] + lvl.pt_count[b])
        st = np.concatenate([np.arange(lvl.pt_start[q], lvl.pt_start[q] + lvl.pt_count[q])
                             for q in lvl.neighbors(b)])
        to, so = tree.perm[tt], tree.perm[st]
        dx = pt[tt][:, None, :] - pt[st][None, :, :]
        r = np.sqrt((dx**2).sum(-1))
        r[r == 0.0] = 1.0
        inv = 1.0 / (4.0 * np.pi * r)
        for row, ell in enumerate(to):
            inv[row, np.isin(ptch[so], smap.singular_patches(int(ell)))] = 0.0
        ndx = np.einsum("tsc,tc->ts", dx, nt[tt])
        w = phiw[so]
        for k in range(2):
            g = np.exp(1j * kap[k] * r) * inv
            s_out[:, k, to] = (g @ w).T
            q = g * (ndx * (1j * kap[k] * r - 1.0) / r**2)
            d_out[:, k, to] = (q @ w[:, :6]).T
    return s_out, d_out


def _corrections(op, phi, kap, stride=1):
    disc = op.disc
    ell, src = op.corr_ell[::stride], op.corr_src[::stride]
    dx = disc.points[ell] - disc.points[src]
    r = np.linalg.norm(dx, axis=1)
    ndx = np.einsum("ec,ec->e", dx, disc.normals[ell])
    jw = disc.weights[src]
    n = disc.n_points
    cs = np.zeros((2, 8, n), dtype=complex)
    cd = np.zeros((2, 6, n), dtype=complex)
    for k in range(2):
        g = np.exp(1j * kap[k] * r) / (4.0 * np.pi * r)
        for c in range(8):
            np.add.at(cs[k, c], ell, g * jw * phi[c, src])
            if c < 6:
                np.add.at(cd[k, c], ell, g * ndx * (1j * kap[k] * r - 1.0) / r**2 * jw * phi[c, src])
    return cs, cd


def potentials(op: OperatorData, phi, stride: int = 1, box_ranges=None,
               far_stride: int | None = None):
    """(S (8,2,N), D (6,2,N)) (operators.py:321-350).  Bounded samples:
    stride > 1 takes every stride-th near-field box / moment / correction,
    box_ranges restricts the far field to a box window, far_stride samples
    every far_stride-th box inside it (default: 1 with a window, else
    stride)."""
    disc = op.disc
    kap = op.materials.kappas
    nc = disc.n_c
    T = _fwd(nc)
    grids = phi.reshape(8, disc.n_patches, nc, nc)
    coeffs = np.matmul(np.matmul(T[None, None], grids), T.T[None, None])
    n = disc.n_points
    s_near = np.zeros((8, 2, n), dtype=complex)
    d_near = np.zeros((8, 2, n), dtype=complex)
    for p, grp in list(op.moments.groups.items())[::stride]:
        s_near[:, :, grp.targets] += np.einsum("kbmn,cmn->ckb", grp.beta_s, coeffs[:, p])
        d_near[:, :, grp.targets] += np.einsum("kbmn,cmn->ckb", grp.beta_d, coeffs[:, p])
    csr = getattr(op.moments, "csr_blocks", None)
    if csr is not None:   # moments in the singularity map's CSR order
        smap = op.smap
        tg = np.repeat(np.arange(smap.n_targets), np.diff(smap.offsets)) + getattr(
            smap, "target_lo", 0)
        for q in range(0, tg.size, stride):
            blk = csr[q].reshape(4, nc, nc)
            cf = coeffs[:, int(smap.patch_ids[q])]
            s_near[:, :, tg[q]] += np.einsum("kmn,cmn->ck", blk[0:2], cf)
            d_near[:, :, tg[q]] += np.einsum("kmn,cmn->ck", blk[2:4], cf)
    if far_stride is None:
        far_stride = 1 if box_ranges is not None else stride
    s_if, s_disp = far_field(op.tree, op.hier, phi * disc.weights, kap,
                             disc.normals, op.fd_step, box_stride=far_stride,
                             box_ranges=box_ranges)
    s_nb, d_nb = _neighbor_sums(op, phi, kap, stride)
    s_far = s_if + s_nb
    d_far = (s_disp[:6] - s_if[:6]) / op.fd_step + d_nb
    cs, cd = _corrections(op, phi, kap, stride)
    for k in range(2):
        s_far[:, k] -= cs[k]
        d_far[:, k] -= cd[k]
    return s_near + s_far, d_near[:6] + d_far


def muller_apply(op: OperatorData, y, stride: int = 1, box_ranges=None,
                 far_stride: int | None = None):
    """y (4N) -> A y (operators.py:399-403 with apply_block :354-397).

    stride > 1 runs a bounded CPU-baseline sample (every stride-th box /
    patch group / correction entry); its output is NOT the full result."""
    disc, mats = op.disc, op.materials
    n = disc.n_points
    y = np.asarray(y, dtype=complex)
    t1, t2 = disc.tangent1, disc.tangent2
    m = y[:n, None] * t1 + y[n:2 * n, None] * t2
    j = y[2 * n:3 * n, None] * t1 + y[3 * n:, None] * t2
    phi = np.empty((8, n), dtype=complex)
    phi[0:3], phi[3:6] = j.T, m.T
    phi[6], phi[7] = _divergence(disc, j), _divergence(disc, m)
    S, D = potentials(op, phi, stride, box_ranges, far_stride)
    G = _grads(disc, S)
    nrm = disc.normals
    kap = mats.kappas

    def nxcurl(k, c0):
        w = D[c0:c0 + 3, k].T
        wt = w - nrm * np.einsum("ij,ij->i", nrm, w)[:, None]
        return sum(nrm[:, q, None] * G[c0 + q, k] for q in range(3)) - wt

    def rt(c0, cdiv):
        acc = np.zeros((n, 3), dtype=complex)
        for k, sg in ((0, 1.0), (1, -1.0)):
            acc = acc + sg * (kap[k] ** 2 * np.cross(nrm, S[c0:c0 + 3, k].T)
                              + np.cross(nrm, G[cdiv, k]))
        return -1j / mats.omega * acc

    row_m = (0.5 * (mats.mu_e + mats.mu_i) * m
             + (mats.mu_e * nxcurl(0, 3) - mats.mu_i * nxcurl(1, 3)) - rt(0, 6))
    row_j = (rt(3, 7) + 0.5 * (mats.eps_e + mats.eps_i) * j
             + (mats.eps_e * nxcurl(0, 0) - mats.eps_i * nxcurl(1, 0)))
    dot = lambda a, b: np.einsum("ij,ij->i", a, b)
    return np.concatenate([dot(row_m, t1), dot(row_m, t2), dot(row_j, t1), dot(row_j, t2)])


# ---------------------------------------------------------------------------
# GMRES (solver.py:30-93)
# ---------------------------------------------------------------------------


def gmres(apply_op, b, tol=1e-4, max_iter=1000):
    """Non-restarted GMRES, modified Gram-Schmidt, complex Givens rotations;
    returns (x, iterations, residual history, converged, wall seconds)."""
    if tol <= 0:
        raise ValueError("tolerance must be positive")
    t0 = time.time()
    b = np.asarray(b, dtype=complex)
    beta = np.linalg.norm(b)
    if beta == 0.0:
        return np.zeros_like(b), 0, [0.0], True, time.time() - t0
    m = min(max_iter, b.size)
    V = np.zeros((m + 1, b.size), dtype=complex)
    V[0] = b / beta
    H = np.zeros((m + 1, m), dtype=complex)
    c = np.zeros(m, dtype=complex)
    s = np.zeros(m, dtype=complex)
    g = np.zeros(m + 1, dtype=complex)
    g[0] = beta
    hist, ok, k = [], False, 0
    for k in range(m):
        w = np.array(apply_op(V[k]), dtype=complex)
        for i in range(k + 1):
            H[i, k] = np.vdot(V[i], w)
            w -= H[i, k] * V[i]
        H[k + 1, k] = np.linalg.norm(w)
        if H[k + 1, k] != 0.0:
            V[k + 1] = w / H[k + 1, k]
        for i in range(k):
            t = c[i] * H[i, k] + s[i] * H[i + 1, k]
            H[i + 1, k] = -np.conj(s[i]) * H[i, k] + np.conj(c[i]) * H[i + 1, k]
            H[i, k] = t
        den = np.sqrt(np.abs(H[k, k]) ** 2 + np.abs(H[k + 1, k]) ** 2)
        if den == 0.0:
            hist.append(hist[-1] if hist else 1.0)
            break
        c[k] = np.conj(H[k, k]) / den
        s[k] = np.conj(H[k + 1, k]) / den
        H[k, k] = den
        H[k + 1, k] = 0.0
        g[k + 1] = -np.conj(s[k]) * g[k]
        g[k] = c[k] * g[k]
        hist.append(abs(g[k + 1]) / beta)
        if hist[-1] <= tol:
            ok = True
            k += 1
            break
    else:
        k = m
    y = np.linalg.solve(H[:k, :k], g[:k]) if k else np.zeros(0, complex)
    x = V[:k].T @ y if k else np.zeros_like(b)
    return x, k, hist, ok, time.time() - t0
