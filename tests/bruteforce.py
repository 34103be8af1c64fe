"""Independent brute-force route for pinning the oracle (tests only).

Reconstruct the piecewise Legendre function, translate it exactly, and re-project it onto
each target cell by Eq. (2) (SS II-A) with a high-order numpy Gauss rule on each
piece where the translated function is smooth.  Uses numpy's leggauss/legval (library
primitives) -- none of the oracle's quadrature, Legendre recurrence or A/B matrices.
Cell units: cell i covers [i, i+1); local coordinate xi = 2 (x - i) - 1.
"""
import math

import numpy as np
from numpy.polynomial import legendre as npleg

_XQ, _WQ = npleg.leggauss(24)


def _eval_line(c, y):
    """u(y) for the periodic piecewise polynomial with coefficients c[N, k] (cell units)."""
    N = c.shape[0]
    fl = np.floor(y)
    cell = (fl.astype(np.int64) % N)
    xi = 2.0 * (y - fl) - 1.0
    V = npleg.legvander(xi, c.shape[1] - 1)  # [pts, j]
    return np.sum(V * c[cell], axis=1)


def reproject_line(c, nu):
    """Exact translate-by-nu (cells) then L2 re-projection of a 1D periodic line c[N, k]."""
    c = np.asarray(c, dtype=np.float64)
    N, k = c.shape
    out = np.zeros_like(c)
    for i in range(N):
        # target cell [i, i+1) pulls from y = x - nu; split where y crosses an integer
        a, b = i - nu, i + 1 - nu
        cuts = [a] + [float(m) for m in range(math.floor(a) + 1, math.ceil(b))] + [b]
        for lo, hi in zip(cuts[:-1], cuts[1:]):
            if hi <= lo:
                continue
            y = 0.5 * (hi + lo) + 0.5 * (hi - lo) * _XQ
            x = y + nu  # position inside the target cell
            xi_t = 2.0 * (x - i) - 1.0
            u = _eval_line(c, y)
            P = npleg.legvander(xi_t, k - 1)
            # (2j+1)/2 * int_{-1}^{1} u P_j dxi, dxi = 2 dx = 2 dy
            out[i] += (2.0 * np.arange(k) + 1.0) / 2.0 * ((u * _WQ)[:, None] * P).sum(0) * (hi - lo)
    return out
