"""CPU ORACLE for the mixed-precision SLDG step (arXiv:1603.07008) -- TEST INFRASTRUCTURE.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs may import this package.  The product package
(``paper_1603_07008_b200``) never imports it, and it never imports the product package.

The arithmetic lives in ``sldg_oracle.c`` (plain C loops, fp64, ``-O2 -fno-fast-math
-ffp-contract=off``), loaded here with ctypes.  This file adds only marshalling plus the
paper's Eq. (2) projection and the L2 norm used by the convergence pins, each written from
the paper:

* ``project_1d``  -- Eq. (2): c_j = (2j+1)/2 * (2/h) * int u(x) P_j(2x/h) dx  (SS II-A),
  by a Gauss-Legendre rule of ``quad_n`` nodes (over-integration).
* ``l2_norm_diff`` -- discrete L2 norm of the difference of two DG functions,
  sqrt(sum_i h sum_j dc_ij^2 / (2j+1)) by Legendre orthogonality.

Citation keys: P:NNN = PAPER.md line, S:NNN = SPEC.md line, SURVEY Cn = SURVEY.md 8(c) reading n.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "sldg_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")
CFLAGS = ["-O2", "-fno-fast-math", "-ffp-contract=off", "-fPIC", "-shared", "-std=c11"]


def build(force: bool = False) -> str:
    """Compile the oracle shared library with gcc (host only; no CUDA)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        subprocess.check_call(["gcc", *CFLAGS, "-o", _LIB, _SRC, "-lm"])
    return _LIB


_lib = None


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_LIB)
        dp = ctypes.POINTER(ctypes.c_double)
        i64p = ctypes.POINTER(ctypes.c_int64)
        L.or_legendre_all.argtypes = [ctypes.c_int, ctypes.c_double, dp]
        L.or_legendre_all.restype = None
        L.or_gauss_legendre.argtypes = [ctypes.c_int, dp, dp]
        L.or_shift_decompose.argtypes = [ctypes.c_double, i64p, dp]
        L.or_shift_matrices.argtypes = [ctypes.c_double, ctypes.c_int, dp, dp]
        L.or_round_layout.argtypes = [ctypes.c_int64, ctypes.c_int64, ctypes.c_int64, dp]
        L.or_advect.argtypes = [ctypes.c_int, i64p, ctypes.c_int, ctypes.c_int64, dp, dp,
                                ctypes.c_int, ctypes.c_double, dp, ctypes.c_uint32]
        L.or_mass.argtypes = [ctypes.c_int64, ctypes.c_int64, ctypes.c_double, dp]
        L.or_mass.restype = ctypes.c_double
        _lib = L
    return _lib


def _dp(a: np.ndarray):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_double))


class OracleError(ValueError):
    pass


def legendre_all(p: int, x: float) -> np.ndarray:
    out = np.zeros(p + 1)
    lib().or_legendre_all(p, float(x), _dp(out))
    return out


def gauss_legendre(n: int):
    x = np.zeros(n)
    w = np.zeros(n)
    if lib().or_gauss_legendre(n, _dp(x), _dp(w)) != 0:
        raise OracleError(f"invalid node count {n}")
    return x, w


def shift_decompose(nu: float):
    i = ctypes.c_int64()
    a = ctypes.c_double()
    if lib().or_shift_decompose(float(nu), ctypes.byref(i), ctypes.byref(a)) != 0:
        raise OracleError(f"invalid shift {nu}")
    return int(i.value), float(a.value)


def shift_matrices(alpha: float, k: int):
    A = np.zeros((k, k))
    B = np.zeros((k, k))
    if lib().or_shift_matrices(float(alpha), int(k), _dp(A), _dp(B)) != 0:
        raise OracleError(f"invalid alpha {alpha} / k {k}")
    return A, B


def n_double_of(precision: str, K: int) -> int:
    """'mixed' keeps only q = 0 in fp64; 'fp64' keeps all K slots."""
    return {"mixed": 1, "fp64": K, "fp32": 0}[precision]


def round_layout(c: np.ndarray, K: int, n_double: int) -> np.ndarray:
    """Return a copy of host coefficients c[cell, q] rounded through the precision layout."""
    out = np.ascontiguousarray(c, dtype=np.float64).copy()
    lib().or_round_layout(out.size // K, K, n_double, _dp(out))
    return out


def advect(c: np.ndarray, dims, k: int, dim: int, shift: float = 0.0, field=None,
           field_mask: int = 0, n_double: int | None = None) -> np.ndarray:
    """One SLDG sweep (see sldg_oracle.c or_advect).  c has shape [cells, k**D]."""
    dims = [int(x) for x in dims]
    D = len(dims)
    K = k ** D
    if n_double is None:
        n_double = K
    src = np.ascontiguousarray(c, dtype=np.float64).reshape(-1)
    assert src.size == int(np.prod(dims)) * K
    dst = np.empty_like(src)
    n = (ctypes.c_int64 * D)(*dims)
    fptr = None
    if field is not None:
        field = np.ascontiguousarray(field, dtype=np.float64)
        fptr = _dp(field)
    rc = lib().or_advect(D, n, int(k), int(n_double), _dp(src), _dp(dst), int(dim),
                         float(shift), fptr, ctypes.c_uint32(field_mask))
    if rc != 0:
        raise OracleError(f"or_advect failed rc={rc}")
    return dst.reshape(-1, K)


def mass(c: np.ndarray, K: int, cell_volume: float) -> float:
    src = np.ascontiguousarray(c, dtype=np.float64).reshape(-1)
    return float(lib().or_mass(src.size // K, K, float(cell_volume), _dp(src)))


def project_1d(f, n: int, lo: float, hi: float, k: int, quad_n: int | None = None) -> np.ndarray:
    """Eq. (2): c_ij = (2j+1)/2 * sum_q w_q f(x_i + h xi_q / 2) P_j(xi_q)."""
    quad_n = quad_n or max(k, 8)
    xq, wq = gauss_legendre(quad_n)
    h = (hi - lo) / n
    P = np.array([legendre_all(k - 1, x) for x in xq])  # [quad, j]
    centers = lo + (np.arange(n) + 0.5) * h
    vals = f(centers[:, None] + 0.5 * h * xq[None, :])  # [cell, quad]
    c = (vals * wq[None, :]) @ P  # [cell, j]
    return c * ((2.0 * np.arange(k) + 1.0) / 2.0)[None, :]


def l2_norm_diff(a: np.ndarray, b: np.ndarray, h: float, k: int) -> float:
    """sqrt(sum_i h sum_j (a_ij - b_ij)^2 / (2j+1)) for 1D grids."""
    d = (np.asarray(a) - np.asarray(b)).reshape(-1, k)
    return float(np.sqrt(h * np.sum(d * d / (2.0 * np.arange(k) + 1.0)[None, :])))
