"""CPU ORACLE for the Gauss-node velocity treatment of x-sweeps (NEXT-3 of SURVEY 8(f)) --
TEST INFRASTRUCTURE.  Same import rule as the rest of ``oracle/``.

An x-sweep whose speed varies with v inside a v-cell (d_t f + v d_x f = 0) is not a
constant-coefficient 1D advection per cell.  SPEC's reading ("v-advection with
x-dependent speed: ... transform the x-dependence from modal to nodal at the o Gauss nodes,
advect each nodal line ... with constant speed, transform back") applied to the v-dependence of
an x-sweep (P:221-227 for the nodal Lagrange basis at Gauss-Legendre nodes; V7):

  1. modal -> nodal in the v dim e:   u_n = sum_m c_m P_m(xi_n)          (xi_n: k Gauss nodes)
  2. each nodal line (fixed v-cell j, node n, all other indices) is a 1D DG function along the
     x dim d in the modal x basis; translate-and-project it with its own CFL number nu_{j,n}
     (oracle.advect on that line, the paper's update P:259-272);
  3. nodal -> modal:                  c'_m = (2m+1)/2 sum_n w_n P_m(xi_n) u'_n
     (Gauss quadrature of the L2 projection, exact for the degree k-1 nodal interpolant).
All arithmetic in fp64; the result is rounded to the precision layout once at the end.
"""
from __future__ import annotations

import numpy as np

from . import advect as _advect
from . import round_layout as _round


def _nodes(k: int):
    x, w = np.polynomial.legendre.leggauss(k)
    V = np.polynomial.legendre.legvander(x, k - 1)  # V[n, m] = P_m(xi_n)
    Vinv = (w[:, None] * V).T * ((2 * np.arange(k) + 1) / 2)[:, None]  # [m, n]
    return x, w, V, Vinv


def advect_vnodes(c: np.ndarray, dims, k: int, dim: int, vdim: int, nodal_nu: np.ndarray,
                  n_double: int) -> np.ndarray:
    """One x-sweep along `dim` with one CFL number per Gauss node of every v-cell of `vdim`:
    nodal_nu[j * k + n] (node n ascending in xi).  c: [cells, k^D] (dim 0 fastest; slot
    q = sum_d m_d k^d).  Steps 1-3 above; returns the rounded coefficients."""
    dims = [int(n) for n in dims]
    D = len(dims)
    K = k ** D
    assert dim != vdim
    _, _, V, Vinv = _nodes(k)
    # [i_{D-1}, ..., i_0, m_{D-1}, ..., m_0]
    A = np.asarray(c, dtype=np.float64).reshape(dims[::-1] + [k] * D)
    ax_i = D - 1 - vdim          # array axis of the cell index along vdim
    ax_m = 2 * D - 1 - vdim      # array axis of the slot index along vdim
    nv = dims[vdim]
    out = np.empty_like(A)
    sub_dims = [dims[e] for e in range(D) if e != vdim]
    sub_dim = dim if dim < vdim else dim - 1
    for j in range(nv):
        Aj = np.take(A, j, axis=ax_i)  # drop the vdim cell axis: m axis shifts by one
        mj = ax_m - 1
        nodal = np.tensordot(Aj, V, axes=([mj], [1]))  # [..., n] (node axis last)
        res = np.empty_like(nodal)
        for n in range(k):
            u = nodal[..., n]  # [i (D-1 dims reversed), m (D-1 dims reversed)]
            u2 = u.reshape(-1, k ** (D - 1))
            v2 = _advect(u2, sub_dims, k, sub_dim, shift=float(nodal_nu[j * k + n]),
                         n_double=k ** (D - 1))
            res[..., n] = v2.reshape(u.shape)
        back = np.tensordot(res, Vinv, axes=([res.ndim - 1], [1]))  # [..., m_e] (m_e axis last)
        back = np.moveaxis(back, -1, mj)
        idx = [slice(None)] * A.ndim
        idx[ax_i] = j
        out[tuple(idx)] = back
    return _round(out.reshape(-1, K), K, n_double)


def nodal_velocity_field(nv: int, lo: float, hi: float, k: int, scale: float) -> np.ndarray:
    """nu at the Gauss nodes of every v-cell: (v_j + xi_n h_v / 2) * scale, v_j the centre."""
    xi, _, _, _ = _nodes(k)
    h = (hi - lo) / nv
    vc = lo + (np.arange(nv) + 0.5) * h
    return ((vc[:, None] + xi[None, :] * h / 2) * scale).reshape(-1)
