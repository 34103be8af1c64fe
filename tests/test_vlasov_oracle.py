"""Pins of the Vlasov-Poisson driver oracle (oracle/vlasov.py, NEXT-2; readings V1-V6)
against what the mathematics fixes: closed forms, brute-force quadrature, invariants, and the
linear Landau damping rate from the dispersion relation (scipy's Faddeeva function).  None of
them compares the oracle with a retyped copy of itself."""
import math

import numpy as np
import pytest
from scipy.special import wofz

import oracle
import sldg_inputs
from oracle import vlasov as vp


def _tensor(dims, k, tables):
    """Coefficients of sum_t prod_d T_t[d][i_d, m_d] (cells dim-0 fastest, slots m_0 fastest)."""
    return sldg_inputs.assemble_separable(tables, dims, k)


# ------------------------------------------------------------------------------- density (V2)
def test_density_constant():
    dims, k, lo, hi = [8, 6], 3, [0.0, -6.0], [4 * np.pi, 6.0]
    c = np.zeros((48, 9))
    c[:, 0] = 0.7
    rho = vp.density(c, dims, k, 1, lo, hi)
    assert rho.shape == (8, 3)
    assert np.allclose(rho[:, 0], 0.7 * 12.0, rtol=1e-15, atol=0)  # rho_0 = 2 V kappa
    assert np.all(rho[:, 1:] == 0.0)


@pytest.mark.parametrize("dx", [1, 2])
def test_density_separable(dx):
    """f = g(x) m(v): rho = (int m dv) * projection of g."""
    k = 3
    nx, nv = [10, 6][:dx], [12, 8][:dx]
    dims = nx + nv
    lo = [0.0] * dx + [-5.0] * dx
    hi = [2 * np.pi] * dx + [5.0] * dx
    gs = [lambda x, a=a: 1.0 + 0.3 * np.sin((a + 1) * x) for a in range(dx)]
    ms = [lambda v: np.exp(-v * v / 2), lambda v: (1 + v * v) * np.exp(-v * v / 3)][:dx]
    tab = [sldg_inputs.project_1d(gs[a], nx[a], lo[a], hi[a], k, 12) for a in range(dx)]
    tab += [sldg_inputs.project_1d(ms[a], nv[a], lo[dx + a], hi[dx + a], k, 12) for a in range(dx)]
    c = _tensor(dims, k, [tab])
    rho = vp.density(c, dims, k, dx, lo, hi)
    # int m dv of the projected m = sum_i h_v c_{i,0}
    mint = [np.sum(tab[dx + a][:, 0]) * (hi[dx + a] - lo[dx + a]) / nv[a] for a in range(dx)]
    want = np.einsum("im,jn->jinm", tab[0], tab[1]).reshape(nx[0] * nx[1], k * k) if dx == 2 else tab[0]
    assert np.allclose(rho, np.prod(mint) * want, rtol=0, atol=1e-13 * np.max(np.abs(want)))


def test_density_bruteforce_quadrature():
    """Reconstruct f at Gauss nodes (numpy Legendre series), integrate over v with a Gauss rule,
    project onto the x Legendre basis with another Gauss rule: a path independent of V2's
    'keep m_v = 0' shortcut."""
    dims, k, lo, hi = [3, 4], 3, [0.0, -2.0], [3.0, 2.0]
    c = sldg_inputs.random_coeffs(dims, k, 5)
    rho = vp.density(c, dims, k, 1, lo, hi)
    xg, wg = np.polynomial.legendre.leggauss(8)
    hv = 1.0
    for ix in range(3):
        for m in range(k):
            acc = 0.0
            for iv in range(4):
                cell = ix + 3 * iv
                C = c[cell].reshape(k, k)  # [m_v, m_x]
                for a, (xa, wa) in enumerate(zip(xg, wg)):   # x node
                    for b, (vb, wb) in enumerate(zip(xg, wg)):  # v node
                        f = np.polynomial.legendre.legval2d(xa, vb, C.T)
                        # projection coefficient: (2m+1)/2 int P_m(xi) ... dxi, v integral h_v/2 dvi
                        acc += wa * wb * f * np.polynomial.legendre.legval(xa, np.eye(k)[m]) * (2 * m + 1) / 2 * hv / 2
            assert abs(acc - rho[ix, m]) <= 1e-13, (ix, m)


# ------------------------------------------------------------------------------- Poisson (V3, V4)
def test_poisson_1d_uniform_is_zero():
    rho = np.zeros((16, 3))
    rho[:, 0] = 2.5
    e = vp.poisson_1d(rho, 16, 4 * np.pi)
    assert np.max(np.abs(e)) <= 1e-15


@pytest.mark.parametrize("k", [2, 3, 4])
def test_poisson_1d_cosine_convergence(k):
    """rho = 1 + eps cos(kappa x) -> E = (eps/kappa) sin(kappa x); error O(h^(k+1))."""
    eps, kap, L = 0.3, 0.5, 4 * np.pi
    errs = []
    for n in [8, 16, 32]:
        rho = sldg_inputs.project_1d(lambda x: 1 + eps * np.cos(kap * x), n, 0.0, L, k, 12)
        e = vp.poisson_1d(rho, n, L)
        xi = np.linspace(-1, 1, 7)
        h = L / n
        x = (np.arange(n)[:, None] + 0.5) * h + xi[None, :] * h / 2
        got = vp.eval_legendre_cells(e, xi)
        errs.append(np.max(np.abs(got - eps / kap * np.sin(kap * x))))
    rates = np.log2(np.array(errs[:-1]) / np.array(errs[1:]))
    assert np.all(rates >= k + 0.5), (errs, rates)


def test_poisson_1d_invariants():
    """Continuity at interfaces, zero mean, d_x E = rho - rho_bar pointwise, gauge invariance."""
    rng = np.random.default_rng(3)
    n, k, L = 12, 4, 3.0
    h = L / n
    rho = rng.standard_normal((n, k))
    e = vp.poisson_1d(rho, n, L)
    right = vp.eval_legendre_cells(e, 1.0)
    left = vp.eval_legendre_cells(e, -1.0)
    assert np.max(np.abs(right - np.roll(left, -1))) <= 1e-13  # periodic continuity
    assert abs(np.sum(e[:, 0]) * h) <= 1e-13                     # zero mean
    rb = rho[:, 0].mean()
    for i in range(n):
        dE = np.polynomial.legendre.legder(e[i]) * 2 / h         # d/dx = (2/h) d/dxi
        g = rho[i].copy()
        g[0] -= rb
        assert np.allclose(np.pad(dE, (0, k - dE.size)), g, atol=1e-12)
    e2 = vp.poisson_1d(rho + np.eye(k)[0] * 5.0, n, L)           # rho + const: same E
    assert np.max(np.abs(e2 - e)) <= 1e-13


def test_poisson_2d_modes_closed_form():
    """Cell means of cos(kappa.x) are cos(kappa.x_c) * prod_c sinc(kappa_c h_c / 2); the spectral
    solve gives E = (kappa/|kappa|^2) * eps * that factor * sin(kappa.x_c)."""
    n1, n2, l1, l2 = 16, 12, 4 * np.pi, 2 * np.pi
    h1, h2 = l1 / n1, l2 / n2
    x1 = (np.arange(n1) + 0.5) * h1
    x2 = (np.arange(n2) + 0.5) * h2
    X1, X2 = np.meshgrid(x1, x2, indexing="xy")  # [i2, i1]
    for (a1, a2) in [(1, 0), (0, 1), (2, 1), (3, -2)]:
        k1, k2 = 2 * np.pi * a1 / l1, 2 * np.pi * a2 / l2
        sinc = lambda z: 1.0 if z == 0 else math.sin(z) / z  # noqa: E731
        fac = sinc(k1 * h1 / 2) * sinc(k2 * h2 / 2)
        eps = 0.05
        rho = 1.0 + eps * fac * np.cos(k1 * X1 + k2 * X2)
        e1, e2 = vp.poisson_2d(rho.reshape(-1), n1, n2, l1, l2)
        kk = k1 * k1 + k2 * k2
        s = eps * fac * np.sin(k1 * X1 + k2 * X2)
        assert np.max(np.abs(e1 - k1 / kk * s.reshape(-1))) <= 1e-15
        assert np.max(np.abs(e2 - k2 / kk * s.reshape(-1))) <= 1e-15


def test_poisson_3d_modes_closed_form():
    """The dx = 3 solve (numpy fftn) on single Fourier modes: E = (kappa/|kappa|^2) eps fac
    sin(kappa.x_c) with the product of the three cell-mean sinc factors; and the 2D wrapper
    agrees with the N-D routine."""
    ns, ls = [8, 6, 10], [4 * np.pi, 2 * np.pi, 3.0]
    hs = [ls[c] / ns[c] for c in range(3)]
    xc = [(np.arange(ns[c]) + 0.5) * hs[c] for c in range(3)]
    X = np.meshgrid(*xc[::-1], indexing="ij")  # [i3, i2, i1]
    X3, X2, X1 = X
    sinc = lambda z: 1.0 if z == 0 else np.sin(z) / z  # noqa: E731
    for a in [(1, 0, 0), (0, 2, 1), (3, -1, 2), (0, 0, 1)]:
        kv = [2 * np.pi * a[c] / ls[c] for c in range(3)]
        fac = np.prod([sinc(kv[c] * hs[c] / 2) for c in range(3)])
        ph = kv[0] * X1 + kv[1] * X2 + kv[2] * X3
        rho = 1.0 + 0.03 * fac * np.cos(ph)
        es = vp.poisson_nd(rho.reshape(-1), ns, ls)
        kk = sum(q * q for q in kv)
        for c in range(3):
            want = (kv[c] / kk * 0.03 * fac * np.sin(ph)).reshape(-1)
            assert np.max(np.abs(es[c] - want)) <= 1e-15
    r2 = np.random.default_rng(1).standard_normal(12 * 10)
    e1, e2 = vp.poisson_2d(r2, 12, 10, 3.0, 2.0)
    f1, f2 = vp.poisson_nd(r2, [12, 10], [3.0, 2.0])
    assert np.max(np.abs(e1 - f1)) <= 1e-15 and np.max(np.abs(e2 - f2)) <= 1e-15


def test_poisson_2d_reduces_to_1d():
    """A density constant along x2 gives E2 = 0 and, for a pure Fourier mode, E1 equal to the 1D
    spectral answer -- consistency between the two solvers at cell centres up to the DG/spectral
    difference of the 1D polynomial solve (checked through the cosine closed form)."""
    n1, n2, l1, l2 = 32, 4, 4 * np.pi, 1.0
    rho = np.tile(1 + 0.01 * np.cos(0.5 * (np.arange(n1) + 0.5) * l1 / n1), n2)
    e1, e2 = vp.poisson_2d(rho, n1, n2, l1, l2)
    assert np.max(np.abs(e2)) <= 1e-16
    assert np.max(np.abs(e1[:n1] - 0.02 * np.sin(0.5 * (np.arange(n1) + 0.5) * l1 / n1))) <= 1e-15


# ------------------------------------------------------------------------------- energy
def test_energy_1d_exact():
    """E = sin(2 pi x) on [0,1] -> 1/2 int E^2 = 0.25, within the projection error."""
    n, k = 64, 4
    e = sldg_inputs.project_1d(lambda x: np.sin(2 * np.pi * x), n, 0.0, 1.0, k, 12)
    w = vp.energy_1d(e, 1.0 / n)
    assert abs(w - 0.25) <= 1e-9
    assert vp.energy_1d(np.zeros((4, 3)), 0.1) == 0.0


# ------------------------------------------------------------------------------- Strang step (V5, V6)
def _landau_ic(dims, k, dx, eps=0.01, kappa=0.5):
    kinds = ["x"] * dx + ["v"] * dx
    lo = [0.0] * dx + [-6.0] * dx
    hi = [2 * np.pi / kappa] * dx + [6.0] * dx
    terms = sldg_inputs.landau_terms(dims, k, kinds, lo, hi, eps=eps, kappa=kappa)
    return sldg_inputs.assemble_separable(terms, dims, k), lo, hi


def test_strang_mass_conservation():
    dims, k = [16, 32], 3
    c, lo, hi = _landau_ic(dims, k, 1, eps=0.05)
    vol = (hi[0] - lo[0]) / 16 * (hi[1] - lo[1]) / 32
    c = oracle.round_layout(c, 9, 1)
    m0 = oracle.mass(c, 9, vol)
    for _ in range(50):
        c, _, _ = vp.strang_step(c, dims, k, 1, lo, hi, 0.1, n_double=1)
    assert abs(oracle.mass(c, 9, vol) - m0) / m0 <= 1e-13


def test_strang_homogeneous_state_is_stationary():
    """f = g(v), homogeneous in x: rho is uniform so E = 0, the x-translations of an x-constant
    function are exact and the v-sweeps shift by nu = 0 (copies): the Strang step leaves f
    unchanged up to rounding (equilibrium of the Vlasov-Poisson system)."""
    for dx, dims in [(1, [8, 16]), (2, [4, 6, 8, 10]), (3, [3, 4, 2, 4, 5, 4])]:
        k = 2
        lo = [0.0] * dx + [-4.0] * dx
        hi = [1.0] * dx + [4.0] * dx
        tabs = []
        for d in range(2 * dx):
            if d < dx:
                t = np.zeros((dims[d], k))
                t[:, 0] = 1.0
            else:
                t = sldg_inputs.project_1d(lambda v: np.exp(-v * v), dims[d], lo[d], hi[d], k, 12)
            tabs.append(t)
        c = sldg_inputs.assemble_separable([tabs], dims, k)
        es, w = vp.field(c, dims, k, dx, lo, hi)
        assert max(np.max(np.abs(e)) for e in es) <= 1e-15 and w <= 1e-30
        c1, _, _ = vp.strang_step(c, dims, k, dx, lo, hi, 0.05, n_double=k ** (2 * dx))
        assert np.max(np.abs(c1 - c)) <= 1e-14 * np.max(np.abs(c))


def _landau_gamma(kappa):
    """Root of 1 + (1 + zeta Z(zeta)) / kappa^2 = 0, zeta = omega / (sqrt(2) kappa),
    Z(zeta) = i sqrt(pi) w(zeta) (Faddeeva): the linear Landau damping rate Im(omega)."""
    def eps(w):
        z = w / (math.sqrt(2) * kappa)
        Z = 1j * math.sqrt(math.pi) * wofz(z)
        return 1 + (1 + z * Z) / kappa ** 2
    w = 1.4 - 0.15j
    for _ in range(50):
        d = (eps(w + 1e-7) - eps(w - 1e-7)) / 2e-7
        w = w - eps(w) / d
    return w


def test_landau_rate_reference_value():
    w = _landau_gamma(0.5)
    assert abs(w.real - 1.4156) < 1e-3 and abs(w.imag + 0.1533) < 1e-3  # textbook values


def landau_rate(energies, dt):
    """Fit log(W) through its local maxima: W ~ exp(2 gamma t)."""
    w = np.asarray(energies)
    t = dt * np.arange(1, len(w) + 1)
    pk = [i for i in range(1, len(w) - 1) if w[i] > w[i - 1] and w[i] >= w[i + 1]]
    pk = [i for i in pk if 1.0 < t[i] < 18.0]
    slope = np.polyfit(t[pk], np.log(w[pk]), 1)[0]
    return slope / 2, len(pk)


def test_strang_landau_damping_rate():
    """1+1D weak Landau damping (eps = 0.01, kappa = 0.5): the electric energy decays at the
    rate 2 gamma of the dispersion relation (within 2%: the cell-centre velocity reading V5
    and the grid resolution are the error sources)."""
    dims, k, dt = [32, 128], 3, 0.1
    c, lo, hi = _landau_ic(dims, k, 1)
    c = oracle.round_layout(c, 9, 1)
    ws = []
    for _ in range(190):
        c, _, w = vp.strang_step(c, dims, k, 1, lo, hi, dt, n_double=1)
        ws.append(w)
    gamma, npk = landau_rate(ws, dt)
    want = _landau_gamma(0.5).imag
    assert npk >= 4
    assert abs(gamma - want) <= 0.02 * abs(want), (gamma, want)  # measured: -0.1545 vs -0.1534
