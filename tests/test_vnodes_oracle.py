"""Pins of the Gauss-node velocity oracle (oracle/vnodes.py, NEXT-3; V7)."""
import numpy as np
import pytest

import oracle
import sldg_inputs
from oracle import vnodes


def _project2d(f, nx, nv, lox, hix, lov, hiv, k, q=10):
    """Exact-to-quadrature L2 projection of f(x, v) on a [nx, nv] grid (cells dim 0 fastest,
    slot m_x + k m_v) with a q x q Gauss rule per cell."""
    xg, wg = np.polynomial.legendre.leggauss(q)
    P = np.polynomial.legendre.legvander(xg, k - 1)  # [q, m]
    hx, hv = (hix - lox) / nx, (hiv - lov) / nv
    c = np.zeros((nv, nx, k, k))  # [j, i, m_v, m_x]
    for j in range(nv):
        vv = lov + (j + 0.5) * hv + xg * hv / 2
        for i in range(nx):
            xx = lox + (i + 0.5) * hx + xg * hx / 2
            F = f(xx[:, None], vv[None, :])  # [qx, qv]
            c[j, i] = np.einsum("a,b,ab,am,bn->nm", wg, wg, F, P, P)
    s = (2 * np.arange(k) + 1) / 2
    c *= s[None, None, :, None] * s[None, None, None, :]
    return c.reshape(nx * nv, k * k)


@pytest.mark.parametrize("dims,k,dim,vdim", [([8, 6], 3, 0, 1), ([5, 4, 6], 2, 1, 2), ([6, 3, 4, 5], 2, 0, 2)])
def test_equal_node_shifts_reduce_to_the_plain_sweep(dims, k, dim, vdim):
    """nu equal at all nodes of a v-cell: modal -> nodal -> modal is the identity, so the result
    is the plain sweep with that per-v-cell field."""
    c = sldg_inputs.random_coeffs(dims, k, 3)
    K = k ** len(dims)
    nu_cell = np.linspace(-2.7, 3.9, dims[vdim])
    got = vnodes.advect_vnodes(c, dims, k, dim, vdim, np.repeat(nu_cell, k), n_double=K)
    want = oracle.advect(c, dims, k, dim, field=nu_cell, field_mask=1 << vdim, n_double=K)
    assert np.max(np.abs(got - want)) <= 1e-13 * np.max(np.abs(want))


def test_mass_conserved():
    dims, k = [10, 8], 3
    c = sldg_inputs.random_coeffs(dims, k, 4)
    nu = vnodes.nodal_velocity_field(8, -4.0, 4.0, k, 0.7)
    got = vnodes.advect_vnodes(c, dims, k, 0, 1, nu, n_double=9)
    assert abs(np.sum(got[:, 0]) - np.sum(c[:, 0])) <= 1e-14 * np.sum(np.abs(c[:, 0]))


def test_free_streaming_accuracy_in_v():
    """d_t f + v d_x f = 0 for one step of length t: the exact solution f0(x - v t, v), projected.
    The nodal treatment resolves the v-dependence of the shift inside a v-cell (error falls at
    order >= k in h_v), the cell-centre reading R7 does not (first order)."""
    k, nx, t = 3, 48, 0.3
    lox, hix, lov, hiv = 0.0, 1.0, -2.0, 2.0
    f0 = lambda x, v: np.sin(2 * np.pi * x) * np.exp(-v * v)  # noqa: E731
    fe = lambda x, v: f0(x - v * t, v)  # noqa: E731
    err_node, err_cent = [], []
    for nv in [4, 8, 16]:
        dims = [nx, nv]
        c0 = _project2d(f0, nx, nv, lox, hix, lov, hiv, k)
        ce = _project2d(fe, nx, nv, lox, hix, lov, hiv, k)
        scale = t / ((hix - lox) / nx)
        node = vnodes.advect_vnodes(c0, dims, k, 0, 1, vnodes.nodal_velocity_field(nv, lov, hiv, k, scale), 9)
        vc = lov + (np.arange(nv) + 0.5) * (hiv - lov) / nv
        cent = oracle.advect(c0, dims, k, 0, field=vc * scale, field_mask=2, n_double=9)
        h = ((hix - lox) / nx) * ((hiv - lov) / nv)
        norm = lambda d: np.sqrt(h * np.sum(d.reshape(-1, k, k) ** 2 /  # noqa: E731
                                            np.outer(2 * np.arange(k) + 1, 2 * np.arange(k) + 1)))
        err_node.append(norm(node - ce))
        err_cent.append(norm(cent - ce))
    rate_node = np.log2(err_node[1] / err_node[2])
    rate_cent = np.log2(err_cent[1] / err_cent[2])
    assert err_node[2] < 0.05 * err_cent[2], (err_node, err_cent)
    assert rate_node >= k - 0.5, (err_node, rate_node)
    assert rate_cent < 2.0, (err_cent, rate_cent)
