"""Seeded synthetic inputs shared by the oracle side and the CUDA side.

This module holds NO arithmetic of the SLDG method (no shift decomposition, no A/B weights,
no sweep).  It only produces inputs:

* ``random_coeffs`` -- the counter-based parity generator of SURVEY 8(d):
    u = (splitmix64(seed * 2**40 + g * K + q) >> 11) * 2**-53,  r = 2u - 1,
    c_0 = 1 + r/2,  c_m = r / n0**|m|_1  (m != 0),
  with g the global linear cell index, q the linear coefficient index, n0 the number of
  cells along dim 0.  Keeps the decay c_j ~ h^j of P:245-247 (SS II-A) while stressing
  cancellation.  The CUDA library implements the same counter-based generator
  independently (sldg_fill_random); both are bit-exact by construction (integer hash, exact
  scaling by a power-of-two-or-integer divisor, IEEE division).
* ``landau_terms`` -- separable 1D tables of the Landau-type initial value
    f0 = (1 + eps * sum_{x dims} cos(kappa x_d)) * prod_{v dims} exp(-v^2/2)/sqrt(2 pi),
  projected per cell with numpy's Gauss-Legendre routine (library primitive, independent
  of both the oracle's and the kernel's quadrature).  A sum of tensor products of 1D
  tables is the exact L2 projection of a sum of separable functions.
* ``vlasov_fields`` -- per-line CFL fields of the 4D/2D Vlasov-type workloads (SURVEY 8(d),
  C11): x-sweeps nu = v_c * dt / h_x (field over the matching v dim), v-sweeps
  nu = E(x_c) * dt / h_v with E_d(x) = (eps/kappa) sin(kappa x_d) (field over the x dims).
"""
from __future__ import annotations

import math

import numpy as np

GOLDEN = np.uint64(0x9E3779B97F4A7C15)
M1 = np.uint64(0xBF58476D1CE4E5B9)
M2 = np.uint64(0x94D049BB133111EB)


def splitmix64(z: np.ndarray) -> np.ndarray:
    """The standard splitmix64 output function applied to state z (uint64, wrapping)."""
    z = np.asarray(z, dtype=np.uint64)
    with np.errstate(over="ignore"):
        z = z + GOLDEN
        z = (z ^ (z >> np.uint64(30))) * M1
        z = (z ^ (z >> np.uint64(27))) * M2
        z = z ^ (z >> np.uint64(31))
    return z


def coef_degree(k: int, D: int) -> np.ndarray:
    """|m|_1 for every linear coefficient index q = sum_d m_d k^d."""
    q = np.arange(k ** D)
    deg = np.zeros_like(q)
    for d in range(D):
        deg += (q // (k ** d)) % k
    return deg


def random_coeffs(dims, k: int, seed: int, first_cell: int = 0, n_cells: int | None = None,
                  cells: np.ndarray | None = None) -> np.ndarray:
    """fp64 coefficients [n_cells, k**D] for global cells first_cell.. (or an explicit list)."""
    dims = [int(x) for x in dims]
    D = len(dims)
    K = k ** D
    total = int(np.prod(dims))
    if cells is None:
        if n_cells is None:
            n_cells = total - first_cell
        cells = np.arange(first_cell, first_cell + n_cells, dtype=np.uint64)
    else:
        cells = np.asarray(cells, dtype=np.uint64)
    q = np.arange(K, dtype=np.uint64)
    with np.errstate(over="ignore"):
        z = np.uint64(seed) * np.uint64(1 << 40) + cells[:, None] * np.uint64(K) + q[None, :]
    u = (splitmix64(z) >> np.uint64(11)).astype(np.float64) * (2.0 ** -53)
    r = 2.0 * u - 1.0
    deg = coef_degree(k, D)
    # n0 ** |m| as an exact double (integer product, exact while < 2**53)
    scale = np.array([float(dims[0] ** int(m)) for m in deg])
    out = r / scale[None, :]
    out[:, 0] = 1.0 + 0.5 * r[:, 0]
    return out


# ---------------------------------------------------------------------------------------
# Landau-type initial value, as separable 1D projections.
# ---------------------------------------------------------------------------------------
def project_1d(f, n: int, lo: float, hi: float, k: int, quad_n: int = 10) -> np.ndarray:
    """[n, k] per-cell Legendre coefficients of f (numpy Gauss rule; input generation only)."""
    xq, wq = np.polynomial.legendre.leggauss(max(quad_n, k))
    V = np.polynomial.legendre.legvander(xq, k - 1)  # [quad, j]
    h = (hi - lo) / n
    centers = lo + (np.arange(n) + 0.5) * h
    vals = f(centers[:, None] + 0.5 * h * xq[None, :])
    c = (vals * wq[None, :]) @ V
    return c * ((2.0 * np.arange(k) + 1.0) / 2.0)[None, :]


def landau_terms(dims, k: int, kinds, lo, hi, eps: float = 0.01, kappa: float = 0.5):
    """List of separable terms; each term is a list (one per dim) of [n_d, k] tables.

    kinds[d] in {'x', 'v'}.  f0 = (1 + eps sum_x cos(kappa x)) prod_v g(v).
    """
    D = len(dims)
    g = lambda v: np.exp(-0.5 * v * v) / math.sqrt(2.0 * math.pi)  # noqa: E731
    one = lambda x: np.ones_like(x)  # noqa: E731
    cosk = lambda x: eps * np.cos(kappa * x)  # noqa: E731
    base = []
    for d in range(D):
        f = g if kinds[d] == "v" else one
        base.append(project_1d(f, dims[d], lo[d], hi[d], k))
    terms = [base]
    for d in range(D):
        if kinds[d] == "x":
            t = list(base)
            t[d] = project_1d(cosk, dims[d], lo[d], hi[d], k)
            terms.append(t)
    return terms


def assemble_separable(terms, dims, k: int) -> np.ndarray:
    """Host assembly c[cell, q] = sum_t prod_d T_t,d[i_d, m_d] (small grids only)."""
    D = len(dims)
    total = None
    for t in terms:
        prod = t[0]  # [n0, k]
        for d in range(1, D):
            # prod has index layout [cells so far][q so far]; outer product with dim d
            # new cell = a + cells_prev * b, new q = q_prev + K_prev * m
            prod = np.einsum("aq,bm->bamq", prod, t[d]).reshape(
                prod.shape[0] * t[d].shape[0], prod.shape[1] * k)
        total = prod if total is None else total + prod
    return total


def vlasov_fields(dims, kinds, lo, hi, dt: float = 0.1, eps: float = 0.01, kappa: float = 0.5):
    """Per-sweep (dim, field, field_mask) for a dimension-split step over every dim.

    x dim d is paired with the v dim at the same position in the list of v dims; its field is
    nu = v_c dt / h_x over that v dim.  A v dim's field is nu = E(x_c) dt / h_v over ALL x
    dims (mask of x dims), with E_j(x) = (eps/kappa) sin(kappa x_j), x_j the x dim paired
    with this v dim.
    """
    D = len(dims)
    xd = [d for d in range(D) if kinds[d] == "x"]
    vd = [d for d in range(D) if kinds[d] == "v"]
    h = [(hi[d] - lo[d]) / dims[d] for d in range(D)]
    ctr = [lo[d] + (np.arange(dims[d]) + 0.5) * h[d] for d in range(D)]
    sweeps = []
    for a, d in enumerate(xd):
        v = vd[a]
        sweeps.append((d, ctr[v] * dt / h[d], 1 << v))
    for a, d in enumerate(vd):
        xj = xd[a]
        mask = 0
        for e in xd:
            mask |= 1 << e
        # field over all x dims (ascending, lower dims fastest); depends on x_j only
        grids = np.meshgrid(*[ctr[e] for e in xd], indexing="ij")
        E = (eps / kappa) * np.sin(kappa * grids[xd.index(xj)])
        # flatten with the lowest masked dim fastest
        field = np.transpose(E, axes=list(range(len(xd)))[::-1]).reshape(-1)
        sweeps.append((d, field * dt / h[d], mask))
    return sweeps
