"""CPU ORACLE for the Vlasov-Poisson driver around the SLDG sweep (NEXT-2 of SURVEY 8(f)) --
TEST INFRASTRUCTURE.

Same import rule as the rest of ``oracle/``: only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s reference legs may use it; it never imports the product package.  Plain numpy in
fp64, each step in the order the sources state it.  The sweeps themselves are ``oracle.advect``.

The paper states the model and the splitting only:
  * P:136-139 (SS II): d_t f + v d_x f + E(x) d_v f = 0 (1+1 dims; "up to 6 dimensions");
  * Cheng-Knorr time splitting reduces it to a sequence of 1D advections;
  * the CFL number of a 1D line "can depend ... on the electric field".
It does not state the field solver.  The rest follows SPEC.md's vlasov_driver,
with the readings V1-V6 of DESIGN.md section 6c:
  V1 grid: D = 2 dx (dx = 1, 2, 3), dims [x_1..x_dx, v_1..v_dx]; x_c is advected with v_c, v_c with E_c.
  V2 density: rho_{i_x, m_x} = (prod_c h_vc) * sum_{i_v} c_{(i_x, i_v), (m_x, 0)}
     (v-integration keeps only the m_v = 0 coefficient, whose Legendre integral is h_v).
  V3 Poisson, dx = 1: d_x E = rho - rho_bar, periodic, zero mean; the cell-wise
     exact antiderivative of the DG density plus cumulative interface constants, then the
     domain mean subtracted.  E is a degree-k polynomial per cell.
  V4 Poisson, dx = 2, 3 (not in SPEC; reading): -Lap(phi) = rho - rho_bar, E = -grad(phi), solved
     spectrally on the cell means (trigonometric interpolant; Nyquist modes of the derivative
     set to zero); E sampled at cell centres.
  V5 CFL fields (R7, cell-centre reading): x_c sweeps nu = v_c(centre of v_c cell) * tau / h_xc,
     v_c sweeps nu = E_c(centre of the x cell) * tau / h_vc.
  V6 Strang step: x-sweeps dt/2, density, Poisson, v-sweeps dt, x-sweeps dt/2.
Electric energy: 1/2 int |E|^2 dx -- exact Legendre orthogonality for dx = 1,
cell-centre rule for dx = 2.
"""
from __future__ import annotations

import numpy as np

from . import advect as _advect


def _split_dims(dims, dx):
    dims = [int(n) for n in dims]
    assert len(dims) == 2 * dx and dx in (1, 2, 3)
    return dims[:dx], dims[dx:]


def density(c: np.ndarray, dims, k: int, dx: int, lo, hi) -> np.ndarray:
    """V2: rho[i_x, m_x] = (prod_c h_vc) sum_{i_v} c[(i_x, i_v), (m_x, 0)].

    c: [cells, k^D] with cell = sum_d i_d S_d (dim 0 fastest) and slot q = sum_d m_d k^d.
    Returns [N_x, k^dx] with i_x = sum_{c<dx} i_xc S_c, m_x = sum_c m_xc k^c."""
    nx, nv = _split_dims(dims, dx)
    Nx, Nv, Kx = int(np.prod(nx)), int(np.prod(nv)), k ** dx
    hv = np.prod([(hi[dx + j] - lo[dx + j]) / nv[j] for j in range(dx)])
    # cells ordered x fastest then v: cell = i_x + Nx * i_v; slots with m_v = 0 are q < k^dx
    cv = np.asarray(c, dtype=np.float64).reshape(Nv, Nx, k ** len(dims))[:, :, :Kx]
    return hv * cv.sum(axis=0)


def poisson_1d(rho: np.ndarray, n: int, length: float) -> np.ndarray:
    """V3: Legendre coefficients e[i, 0..k] of E on each cell, d_x E = rho - rho_bar,
    E continuous and periodic, mean(E) = 0.  rho: [n, k] Legendre coefficients per cell."""
    rho = np.asarray(rho, dtype=np.float64)
    k = rho.shape[1]
    h = length / n
    rho_bar = rho[:, 0].mean()  # mean density: cell means are the P_0 coefficients
    g = rho.copy()
    g[:, 0] -= rho_bar
    # antiderivative F_i(xi) = (h/2) int_{-1}^{xi} g_i(s) ds, Legendre coefficients f[i, 0..k]:
    #   int_{-1}^{xi} P_0 = P_1 + P_0;  int_{-1}^{xi} P_m = (P_{m+1} - P_{m-1}) / (2m+1), m >= 1
    f = np.zeros((n, k + 1))
    f[:, 0] += g[:, 0]
    f[:, 1] += g[:, 0]
    for m in range(1, k):
        f[:, m + 1] += g[:, m] / (2 * m + 1)
        f[:, m - 1] -= g[:, m] / (2 * m + 1)
    f *= h / 2
    # left-edge values: E_i(-1) = C_0 + sum_{j<i} F_j(1), F_j(1) = h g_j0
    jumps = h * g[:, 0]
    left = np.concatenate([[0.0], np.cumsum(jumps)[:-1]])
    # gauge: domain mean of E = mean_i (left_i + f_i0) = 0
    c0 = -np.mean(left + f[:, 0])
    e = f.copy()
    e[:, 0] += c0 + left
    return e


def eval_legendre_cells(e: np.ndarray, xi) -> np.ndarray:
    """Value of sum_m e[i, m] P_m(xi) for every cell i (numpy's Legendre series)."""
    return np.stack([np.polynomial.legendre.legval(xi, e[i]) for i in range(e.shape[0])])


def field_centres_1d(e: np.ndarray) -> np.ndarray:
    """E at the cell centres (xi = 0)."""
    return eval_legendre_cells(e, 0.0)


def poisson_nd(rho_mean: np.ndarray, ns, ls):
    """V4 for dx = len(ns) >= 2: E = -grad(phi), -Lap(phi) = rho - mean, spectral on the cell
    means rho_mean[i_1 + n_1 i_2 + ...] (numpy.fft.fftn); returns [E_1, .., E_dx] at the cell
    centres, same indexing; Nyquist modes of each derivative set to zero."""
    ns = [int(n) for n in ns]
    dx = len(ns)
    r = np.asarray(rho_mean, dtype=np.float64).reshape(ns[::-1])  # axes [i_dx, ..., i_1]
    rh = np.fft.fftn(r)
    ks = [2 * np.pi * np.fft.fftfreq(ns[c], d=ls[c] / ns[c]) for c in range(dx)]
    grids = np.meshgrid(*ks[::-1], indexing="ij")  # grids[a] varies along axis a = dim dx-1-a
    kk = sum(gq ** 2 for gq in grids)
    phi = np.zeros_like(rh)
    nz = kk > 0
    phi[nz] = rh[nz] / kk[nz]
    out = []
    for c in range(dx):
        dsym = 1j * grids[dx - 1 - c].copy()
        if ns[c] % 2 == 0:
            idx = [slice(None)] * dx
            idx[dx - 1 - c] = ns[c] // 2
            dsym[tuple(idx)] = 0
        out.append(np.real(np.fft.ifftn(-dsym * phi)).reshape(-1))
    return out


def poisson_2d(rho_mean: np.ndarray, n1: int, n2: int, l1: float, l2: float):
    """V4: E = -grad(phi), -Lap(phi) = rho - mean, spectral on the cell means rho_mean[i1 + n1 i2];
    returns (E1, E2) at the cell centres, same indexing."""
    r = np.asarray(rho_mean, dtype=np.float64).reshape(n2, n1)  # [i2, i1]
    rh = np.fft.fft2(r)  # axes (i2, i1)
    k1 = 2 * np.pi * np.fft.fftfreq(n1, d=l1 / n1)
    k2 = 2 * np.pi * np.fft.fftfreq(n2, d=l2 / n2)
    K2, K1 = np.meshgrid(k2, k1, indexing="ij")
    kk = K1 ** 2 + K2 ** 2
    phi = np.zeros_like(rh)
    nz = kk > 0
    phi[nz] = rh[nz] / kk[nz]
    # derivative symbols, Nyquist modes zeroed (the interpolant's odd derivative is ambiguous there)
    d1 = 1j * K1
    d2 = 1j * K2
    if n1 % 2 == 0:
        d1[:, n1 // 2] = 0
    if n2 % 2 == 0:
        d2[n2 // 2, :] = 0
    e1 = np.real(np.fft.ifft2(-d1 * phi)).reshape(-1)
    e2 = np.real(np.fft.ifft2(-d2 * phi)).reshape(-1)
    return e1, e2


def energy_1d(e: np.ndarray, h: float) -> float:
    """1/2 int E^2 dx = 1/2 sum_i (h/2) sum_m e_im^2 * 2/(2m+1) (Legendre orthogonality)."""
    m = np.arange(e.shape[1])
    return 0.5 * float(np.sum(h * e ** 2 / (2 * m + 1)))


def energy_2d(e1: np.ndarray, e2: np.ndarray, h1: float, h2: float) -> float:
    """1/2 int |E|^2 dx by the cell-centre rule."""
    return 0.5 * h1 * h2 * float(np.sum(e1 ** 2 + e2 ** 2))


def field(c: np.ndarray, dims, k: int, dx: int, lo, hi):
    """density -> Poisson -> E at the x-cell centres, one array per component, and the
    electric energy."""
    nx, _ = _split_dims(dims, dx)
    rho = density(c, dims, k, dx, lo, hi)
    if dx == 1:
        e = poisson_1d(rho, nx[0], hi[0] - lo[0])
        return [field_centres_1d(e)], energy_1d(e, (hi[0] - lo[0]) / nx[0])
    if dx == 2:
        e1, e2 = poisson_2d(rho[:, 0], nx[0], nx[1], hi[0] - lo[0], hi[1] - lo[1])
        return [e1, e2], energy_2d(e1, e2, (hi[0] - lo[0]) / nx[0], (hi[1] - lo[1]) / nx[1])
    es = poisson_nd(rho[:, 0], nx, [hi[c] - lo[c] for c in range(dx)])
    hprod = np.prod([(hi[c] - lo[c]) / nx[c] for c in range(dx)])
    return es, 0.5 * hprod * float(sum(np.sum(e ** 2) for e in es))


def x_field(dims, dx: int, lo, hi, c: int, tau: float) -> np.ndarray:
    """V5: nu of the x_c sweep per v_c cell: v_centre * tau / h_xc (mask: bit dx + c)."""
    nv = int(dims[dx + c])
    hv = (hi[dx + c] - lo[dx + c]) / nv
    hx = (hi[c] - lo[c]) / dims[c]
    v = lo[dx + c] + (np.arange(nv) + 0.5) * hv
    return v * tau / hx


def _x_sweep(c, dims, k, dx, lo, hi, a, tau, n_double, nodal):
    if not nodal:  # V5: cell-centre velocity
        return _advect(c, dims, k, a, field=x_field(dims, dx, lo, hi, a, tau), field_mask=1 << (dx + a),
                       n_double=n_double)
    # V7 (NEXT-3): one CFL number per Gauss node of every v_a cell
    from . import vnodes
    nv = int(dims[dx + a])
    nu = vnodes.nodal_velocity_field(nv, lo[dx + a], hi[dx + a], k, tau / ((hi[a] - lo[a]) / dims[a]))
    return vnodes.advect_vnodes(c, dims, k, a, dx + a, nu, n_double=n_double)


def strang_step(c: np.ndarray, dims, k: int, dx: int, lo, hi, dt: float, n_double: int, nodal: bool = False):
    """V6: one Strang step; returns (new coefficients, [E_c at centres], energy)
    with the field of the mid-step density.  nodal=True: x-sweeps by the Gauss-node velocity
    treatment (V7) instead of the cell-centre reading (V5)."""
    dims = [int(n) for n in dims]
    for a in range(dx):  # x half-steps
        c = _x_sweep(c, dims, k, dx, lo, hi, a, dt / 2, n_double, nodal)
    es, w = field(c, dims, k, dx, lo, hi)
    xmask = (1 << dx) - 1
    for a in range(dx):  # v full steps, nu = E_a(x centre) dt / h_va
        hv = (hi[dx + a] - lo[dx + a]) / dims[dx + a]
        c = _advect(c, dims, k, dx + a, field=es[a] * dt / hv, field_mask=xmask, n_double=n_double)
    for a in range(dx):
        c = _x_sweep(c, dims, k, dx, lo, hi, a, dt / 2, n_double, nodal)
    return c, es, w
