"""Device singular moments (csrc/moments.cu, ifgfb_singular_moments) against
the host restatement of reference quadrature.py:271-331 (compute_moments).

Exact mode (default) reproduces the reference to rounding.  Without it (graded
map on the device) beta_s agrees to 1e-12 and beta_d does NOT reproduce
the reference bit for bit and cannot agree to rounding: the graded grid
clusters nodes within ~1e-8 of the target, where dx = x - y(u, v) and
(x - y).n_x / r^2 lose all but a few digits, so the float64 value of beta_d
carries ~1e-7 relative noise (measured against an extended-precision
evaluation of the same float64 inputs) whose exact bits depend on the
evaluation order.  The tests therefore hold the device to (i) the same
accuracy as the reference's own arithmetic against the extended-precision
value, and (ii) apply(y) within 5e-9 of the reference golden (host moments,
bit-identical to the reference, give 2.9e-11; tests/test_gpu_apply.py).
Device moments are the plan-time accelerator for configurations the
reference cannot run; parity runs use the host moments."""

import numpy as np
import pytest

from _support import golden, inputs, rel
from paper_2408_02274_b200 import cheb, nearfield
from paper_2408_02274_b200.operator import MullerOperator

pytestmark = pytest.mark.gpu


def _dev(name, kappas=None, exact=True):
    inp = inputs(name)
    return nearfield.compute_moments_device(
        inp["disc"], inp["smap"], nearfield.SingularQuadratureConfig(),
        kappas or inp["kappas"], exact=exact)


def _beta_d_extended(disc, smap, p, kappa, n_pairs=12):
    """beta_d of the first pairs of patch p evaluated in long double from the
    same float64 inputs (nodes, coefficients, targets): the accuracy yardstick."""
    cfg = nearfield.SingularQuadratureConfig()
    tg, u0, v0 = smap.pairs_for_patch(p)
    tg, u0, v0 = tg[:n_pairs], u0[:n_pairs], v0[:n_pairs]
    patch, n_c = disc.patches[p], disc.n_c
    nb = cfg.resolve_n_beta(n_c)
    base, wb = cheb.nodes(nb), cheb.fejer(nb)
    ld = np.longdouble
    xu, dxu = nearfield.clustered_nodes(u0, base, cfg.d)
    xv, dxv = nearfield.clustered_nodes(v0, base, cfg.d)
    b = tg.size
    tu = cheb.basis(patch.n, xu.ravel()).reshape(b, nb, patch.n).astype(ld)
    tv = cheb.basis(patch.n, xv.ravel()).reshape(b, nb, patch.n).astype(ld)
    grid = lambda cf: np.stack([tu @ cf[c].astype(ld) @ tv.transpose(0, 2, 1)
                                for c in range(3)])
    pos, eu, ev = grid(patch.coeffs), grid(patch.coeffs_du), grid(patch.coeffs_dv)
    crs = np.cross(np.moveaxis(eu, 0, -1), np.moveaxis(ev, 0, -1))
    jac = np.sqrt((crs**2).sum(-1))
    dx = disc.points[tg].astype(ld).T[:, :, None, None] - pos
    r = np.sqrt((dx**2).sum(axis=0))
    ndx = np.einsum("cbij,bc->bij", dx, disc.normals[tg].astype(ld))
    pu = cheb.basis(n_c, xu.ravel()).reshape(b, nb, n_c).astype(ld)
    pv = cheb.basis(n_c, xv.ravel()).reshape(b, nb, n_c).astype(ld)
    put = (pu * (dxu * wb)[:, :, None].astype(ld)).transpose(0, 2, 1)
    pvw = pv * (dxv * wb)[:, :, None].astype(ld)
    kr = ld(float(np.real(kappa)))
    amp = jac / (4 * ld(np.pi) * r)
    fac = ndx / r**2
    re_ks, im_ks = np.cos(kr * r) * amp, np.sin(kr * r) * amp
    # kd = ks * fac * (i kappa r - 1)
    re = (-re_ks - im_ks * kr * r) * fac
    im = (re_ks * kr * r - im_ks) * fac
    out = (np.einsum("bmi,bij,bjn->bmn", put, re, pvw).astype(np.float64)
           + 1j * np.einsum("bmi,bij,bjn->bmn", put, im, pvw).astype(np.float64))
    return out


@pytest.mark.parametrize("name", ["s1", "c1", "se1", "sl1"])
def test_exact_device_moments_match_reference_order(name):
    """Exact mode (host graded nodes, reference operation order for the
    patch geometry): beta_s and beta_d both agree with the reference's
    float64 values to rounding -- the ~1e-7 conditioning noise of beta_d is
    reproduced, not averaged away."""
    inp = inputs(name)
    dev, host = _dev(name), inp["moments"]
    ws = wd = 0.0
    for p, g in host.groups.items():
        d = dev.groups[p]
        np.testing.assert_array_equal(d.targets, g.targets)
        ws = max(ws, rel(d.beta_s, g.beta_s))
        wd = max(wd, rel(d.beta_d, g.beta_d))
    print(f"{name}: beta_s {ws:.2e} beta_d {wd:.2e}")
    assert ws < 1e-14, ws      # measured 3.6e-16
    assert wd < 1e-14, wd      # measured 3.8e-16 .. 4.2e-16


@pytest.mark.parametrize("name", ["s1", "c1"])
def test_device_moments_vs_host(name):
    inp = inputs(name)
    dev, host = _dev(name, exact=False), inp["moments"]
    assert sorted(dev.groups) == sorted(host.groups)
    ws, wd = 0.0, 0.0
    for p, g in host.groups.items():
        d = dev.groups[p]
        np.testing.assert_array_equal(d.targets, g.targets)
        ws = max(ws, rel(d.beta_s, g.beta_s))
        wd = max(wd, rel(d.beta_d, g.beta_d))
    assert ws < 1e-12, ws
    assert wd < 1e-7, wd


@pytest.mark.parametrize("name", ["s1", "c1"])
def test_device_beta_d_as_accurate_as_reference(name):
    inp = inputs(name)
    dev, host = _dev(name, exact=False), inp["moments"]
    for p in sorted(host.groups)[:3]:
        ext = _beta_d_extended(inp["disc"], inp["smap"], p, inp["kappas"][0])
        k = ext.shape[0]
        e_host = rel(host.groups[p].beta_d[0, :k], ext)
        e_dev = rel(dev.groups[p].beta_d[0, :k], ext)
        assert e_dev < max(3.0 * e_host, 1e-12), (p, e_dev, e_host)


def test_device_moments_lossy_kappa():
    """Complex wavenumbers (lossy interior) follow the same formulas."""
    inp = inputs("s1")
    kap = (inp["kappas"][0], complex(inp["kappas"][1]) + 0.7j)
    cfg = nearfield.SingularQuadratureConfig()
    dev = nearfield.compute_moments_device(inp["disc"], inp["smap"], cfg, kap)
    host = nearfield.compute_moments(inp["disc"], inp["smap"], cfg, kap)
    for p, g in host.groups.items():
        assert rel(dev.groups[p].beta_s, g.beta_s) < 1e-14
        assert rel(dev.groups[p].beta_d, g.beta_d) < 1e-14


@pytest.mark.parametrize("name", ["c1", "c2n4"])
def test_apply_with_device_moments_vs_reference_golden(name):
    """The plan path the bench uses above 100k points (device moments,
    exact mode) at the north-star apply tolerance."""
    inp = inputs(name)
    z = golden(name)
    op = MullerOperator(inp["disc"], inp["mats"], inp["smap"], _dev(name),
                        (inp["corr"].ell_idx, inp["corr"].src_idx), tree=inp["tree"],
                        hierarchy=inp["hier"])
    e = rel(op.apply(z["y"]), z["apply_y"])
    print(f"{name}: apply with device moments {e:.2e}")
    assert e < 1e-10, e      # measured 2.9e-11 (c1), 1.9e-11 (c2n4)


def test_apply_with_inexact_device_moments():
    inp = inputs("c1")
    z = golden("c1")
    op = MullerOperator(inp["disc"], inp["mats"], inp["smap"], _dev("c1", exact=False),
                        (inp["corr"].ell_idx, inp["corr"].src_idx), tree=inp["tree"],
                        hierarchy=inp["hier"])
    assert rel(op.apply(z["y"]), z["apply_y"]) < 5e-9


def test_csr_moment_table_same_apply():
    """groups=False (CSR blocks straight into the near-field plan) gives the
    same operator as the per-patch table."""
    inp = inputs("s1")
    z = golden("s1")
    cfg = nearfield.SingularQuadratureConfig()
    ops = []
    for grouped in (True, False):
        mom = nearfield.compute_moments_device(inp["disc"], inp["smap"], cfg,
                                               inp["kappas"], groups=grouped)
        ops.append(MullerOperator(inp["disc"], inp["mats"], inp["smap"], mom,
                                  (inp["corr"].ell_idx, inp["corr"].src_idx),
                                  tree=inp["tree"], hierarchy=inp["hier"]))
    np.testing.assert_array_equal(ops[0].apply(z["y"]), ops[1].apply(z["y"]))
