"""Pins of the CPU oracle against what the paper and mathematics fix (runs without a GPU).

Each test names the pin it implements and the passage it follows.
None of these compare the oracle with itself: the references are printed values
(tests/golden/), exact rational closed forms (tests/exact_poly.py), an independent
brute-force re-projection (tests/bruteforce.py), library routines for special cases, or
invariants that a dropped term / wrong sign / transposed operand would break.
"""
import json
import math
import os

import numpy as np
import pytest

import oracle
from tests import bruteforce
from tests.exact_poly import exact_AB
import sldg_inputs

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _gold(name):
    with open(os.path.join(GOLD, name)) as f:
        return json.load(f)


# ----------------------------------------------------------------------------- Legendre
def test_legendre_spec_examples():
    """S:48-50 worked examples."""
    for p, x, vals in _gold("spec_examples.json")["legendre"]["cases"]:
        assert np.array_equal(oracle.legendre_all(p, x), np.array(vals))


def test_legendre_against_explicit_polynomials():
    """P_j from textbook closed forms ('the jth Legendre polynomial')."""
    rng = np.random.default_rng(1603)
    for x in rng.uniform(-1, 1, 50):
        P = oracle.legendre_all(6, x)
        exact = [1, x, (3 * x**2 - 1) / 2, (5 * x**3 - 3 * x) / 2, (35 * x**4 - 30 * x**2 + 3) / 8,
                 (63 * x**5 - 70 * x**3 + 15 * x) / 8, (231 * x**6 - 315 * x**4 + 105 * x**2 - 5) / 16]
        np.testing.assert_allclose(P, exact, rtol=0, atol=1e-14)


# ----------------------------------------------------------------------------- Gauss
def test_gauss_spec_examples():
    """n=1 midpoint, n=2 nodes +-1/sqrt3 weights 1, n=5 integrates x^8 to 2/9."""
    g = _gold("spec_examples.json")["gauss"]
    x, w = oracle.gauss_legendre(1)
    assert np.array_equal(x, g["n1"]["nodes"]) and np.array_equal(w, g["n1"]["weights"])
    x, w = oracle.gauss_legendre(2)
    np.testing.assert_allclose(np.abs(x), g["n2_nodes_abs"], rtol=0, atol=1e-16)
    np.testing.assert_allclose(w, [1.0, 1.0], rtol=0, atol=4.5e-16)
    x, w = oracle.gauss_legendre(5)
    assert abs(np.sum(w * x**8) - 2.0 / 9.0) < 1e-15


@pytest.mark.parametrize("n", list(range(1, 17)))
def test_gauss_exactness_and_library(n):
    """Special case that reduces to a library routine (numpy.leggauss) + exactness for x^m,
    m <= 2n-1."""
    x, w = oracle.gauss_legendre(n)
    xr, wr = np.polynomial.legendre.leggauss(n)
    np.testing.assert_allclose(x, xr, rtol=0, atol=2e-15)
    np.testing.assert_allclose(w, wr, rtol=0, atol=2e-15)
    for m in range(2 * n):
        exact = 0.0 if m % 2 else 2.0 / (m + 1)
        assert abs(np.sum(w * x**m) - exact) < 1e-14


# ----------------------------------------------------------------------------- shift decomposition
def test_shift_decompose_spec_examples():
    """P8: S:213-215."""
    for nu, i, a in _gold("spec_examples.json")["shift_decompose"]["cases"]:
        assert oracle.shift_decompose(nu) == (i, a)


def test_shift_decompose_floor_and_edge():
    """floor (not truncation) for nu<0; fl(alpha)==1 becomes (i*+1, 0)."""
    assert oracle.shift_decompose(-2.75) == (-3, 0.25)
    assert oracle.shift_decompose(-1e-20) == (0, 0.0)
    assert oracle.shift_decompose(-0.0) == (0, 0.0)
    with pytest.raises(oracle.OracleError):
        oracle.shift_decompose(float("nan"))
    with pytest.raises(oracle.OracleError):
        oracle.shift_decompose(float("inf"))


# ----------------------------------------------------------------------------- A, B
@pytest.mark.parametrize("k", [1, 2, 3, 4, 5, 6, 7, 8])
def test_matrices_exact_rational(k):
    """P1/P5: A(alpha), B(alpha) against exact rational integration of S:219's integrals."""
    for alpha in [0.37, 0.5, 0.02130859375, 0.999, 1e-3, 0.75, 0.123456789]:
        A, B = oracle.shift_matrices(alpha, k)
        Ae, Be = exact_AB(alpha, k)
        Ae = np.array([[float(v) for v in r] for r in Ae])
        Be = np.array([[float(v) for v in r] for r in Be])
        np.testing.assert_allclose(A, Ae, rtol=0, atol=4e-15 * k)
        np.testing.assert_allclose(B, Be, rtol=0, atol=4e-15 * k)


def test_matrices_closed_form_k1_k2():
    """P1 (S:223, S:472 upwind) and Appendix-A k=2 closed form."""
    for a in np.linspace(0.01, 0.99, 37):
        A, B = oracle.shift_matrices(a, 1)
        assert abs(A[0, 0] - a) < 1e-15 and abs(B[0, 0] - (1 - a)) < 1e-15
        A, B = oracle.shift_matrices(a, 2)
        Ac = [[a, a - a * a], [3 * a * a - 3 * a, -2 * a**3 + 6 * a * a - 3 * a]]
        Bc = [[1 - a, a * a - a], [3 * a - 3 * a * a, 2 * a**3 - 3 * a + 1]]
        np.testing.assert_allclose(A, Ac, rtol=0, atol=2e-15)
        np.testing.assert_allclose(B, Bc, rtol=0, atol=2e-15)


def test_mass_row_exact_in_floating_point():
    """DESIGN.md R3 (Table II): the rounded mass row sums to delta_0l
    exactly, so mass drift is not coherent.  Randomized over alpha and k."""
    rng = np.random.default_rng(99)
    for k in range(1, 9):
        for a in np.concatenate([rng.uniform(0, 1, 300), [0.37, 0.5, 1 - 2**-53, 2**-60]]):
            A, B = oracle.shift_matrices(a, k)
            assert A[0, 0] + B[0, 0] == 1.0
            assert abs(A[0, 0] - a) <= 2**-54
            for l in range(1, k):
                assert A[0, l] + B[0, l] == 0.0


def test_matrices_alpha_zero_exact():
    """P2 / SURVEY C10: alpha = 0 gives exactly A = 0, B = I."""
    for k in range(1, 9):
        A, B = oracle.shift_matrices(0.0, k)
        assert np.array_equal(A, np.zeros((k, k))) and np.array_equal(B, np.eye(k))


@pytest.mark.parametrize("k", [2, 3, 4, 5, 6, 7])
def test_matrices_invariants(k):
    """P3 mass row / constant column, P4 reflection A(a) = D B(1-a) D, P6 |.|<=1."""
    rng = np.random.default_rng(k)
    Dm = np.diag([(-1.0) ** j for j in range(k)])
    for a in rng.uniform(0, 1, 200):
        A, B = oracle.shift_matrices(a, k)
        e0 = np.eye(k)[0]
        np.testing.assert_allclose(A[0] + B[0], e0, atol=1e-14)
        np.testing.assert_allclose(A[:, 0] + B[:, 0], e0, atol=1e-14)
        A2, B2 = oracle.shift_matrices(1.0 - a, k)
        np.testing.assert_allclose(A, Dm @ B2 @ Dm, atol=1e-13)
        assert np.max(np.abs(A)) <= 1 + 1e-12 and np.max(np.abs(B)) <= 1 + 1e-12


# ----------------------------------------------------------------------------- single sweep
def test_upwind_worked_example():
    """P7: S:233 -- k=1, N=2, values [1,0], nu=0.5 -> [0.5, 0.5]."""
    g = _gold("spec_examples.json")["upwind_k1"]["advect"]
    out = oracle.advect(np.array(g["in"])[:, None], [2], 1, 0, shift=g["nu"])
    assert np.array_equal(out[:, 0], np.array(g["out"]))


@pytest.mark.parametrize("seed", range(50))
def test_advect_vs_bruteforce_reprojection(seed):
    """P9: matrix update vs reconstruct -> translate -> re-project, N<=32, 1e-13."""
    rng = np.random.default_rng(seed)
    N = int(rng.integers(1, 33))
    k = int(rng.integers(1, 7))
    nu = float(rng.uniform(-40, 40))
    c = rng.standard_normal((N, k)) / (1.0 + np.arange(k))[None, :]
    got = oracle.advect(c, [N], k, 0, shift=nu)
    ref = bruteforce.reproject_line(c, nu)
    assert np.max(np.abs(got - ref)) <= 1e-13 * max(1.0, np.max(np.abs(ref)))


def test_integer_shift_bit_exact_rotation():
    """P2: integer nu is a bit-exact permutation, incl. -0.0 and subnormals."""
    rng = np.random.default_rng(7)
    c = rng.standard_normal((13, 4))
    c[3, 1] = -0.0
    c[5, 2] = 5e-324
    for nu in [0.0, 1.0, -1.0, 5.0, -27.0, 13.0, 1e6]:
        out = oracle.advect(c, [13], 4, 0, shift=nu)
        ref = np.roll(c, int(nu) % 13, axis=0)
        assert out.tobytes() == ref.tobytes()


def test_polynomial_exactness():
    """P10: polynomials of degree < k are translated exactly (P:204-209 'exact translation' +
    L2 projection reproduces polynomials) on every cell whose sources don't wrap."""
    for k in [2, 3, 4, 6]:
        N, L = 40, 1.0
        h = L / N
        q = lambda x: 0.3 - 1.7 * x + 2.1 * x**2 - 0.9 * x**3 + 0.4 * x**5  # noqa: E731
        deg = min(k - 1, 5)
        coef = np.array([0.3, -1.7, 2.1, -0.9, 0.0, 0.4])[: deg + 1]
        poly = lambda x: np.polyval(coef[::-1], x)  # noqa: E731
        del q
        c = oracle.project_1d(poly, N, 0.0, L, k, quad_n=12)
        nu = 3.37
        out = oracle.advect(c, [N], k, 0, shift=nu)
        ref = oracle.project_1d(lambda x: poly(x - nu * h), N, 0.0, L, k, quad_n=12)
        ok = slice(5, N)  # sources (i - 4, i - 3) stay in [0, N): no periodic jump
        assert np.max(np.abs(out[ok] - ref[ok])) < 1e-13


@pytest.mark.parametrize("k", [2, 3, 4, 5, 6])
def test_convergence_order(k):
    """P11: order k on smooth data (P:207-209 'approximation of order o').
    Fixed CFL nu = 0.8 (alpha = 0.8 at every N), one full period, N = 20..160."""
    errs = []
    Ns = [20, 40, 80, 160] if k <= 4 else [20, 40, 80]
    f = lambda x: np.sin(2 * np.pi * x)  # noqa: E731
    for N in Ns:
        nu = 0.8
        steps = N * 5 // 4  # steps * nu == N exactly: one period
        c0 = oracle.project_1d(f, N, 0.0, 1.0, k, quad_n=12)
        c = c0
        for _ in range(steps):
            c = oracle.advect(c, [N], k, 0, shift=nu)
        errs.append(oracle.l2_norm_diff(c, c0, 1.0 / N, k))
    orders = [math.log2(errs[i] / errs[i + 1]) for i in range(len(errs) - 1)]
    assert min(orders) >= k - 0.3, (errs, orders)


# ----------------------------------------------------------------------------- precision / mass
def _smooth_ic(N, k):
    return oracle.project_1d(lambda x: 1.0 + 0.5 * np.sin(2 * np.pi * x), N, 0.0, 1.0, k, quad_n=12)


def _osc_ic(N, k):
    rng = np.random.default_rng(5)
    ph = rng.uniform(0, 2 * np.pi, 8)
    f = lambda x: 1.0 + sum(np.sin(2 * np.pi * m * x + ph[m - 1]) / m for m in range(1, 9)) / 4  # noqa
    return oracle.project_1d(f, N, 0.0, 1.0, k, quad_n=16)


@pytest.mark.parametrize("k", [2, 4])
@pytest.mark.parametrize("ic", ["smooth", "oscillatory"])
def test_table_II_mechanism(k, ic):
    """P12/P13 (Table II): 1e4 steps at N=256, nu=2.25 (S:427 defaults).
    mixed (c0 fp64): mass drift <= 1e-12 (paper 4.4e-15..1.6e-14) and L2 distance to the fp64
    run within two orders of magnitude of the paper's 1e-10..6e-8; pure fp32 (d=0) loses mass
    conservation (paper 2.4e-6..1.3e-5)."""
    N, steps, nu = 256, 10000, 2.25
    c0 = _smooth_ic(N, k) if ic == "smooth" else _osc_ic(N, k)
    h = 1.0 / N
    runs = {}
    for nd in [k, 1, 0]:
        c = oracle.round_layout(c0, k, nd)
        m0 = oracle.mass(c, k, h)
        for _ in range(steps):
            c = oracle.advect(c, [N], k, 0, shift=nu, n_double=nd)
        runs[nd] = (c, abs(oracle.mass(c, k, h) - m0) / abs(m0))
    assert runs[k][1] <= 1e-13   # paper prints 4.4e-15 .. 1.6e-14 for every d >= 1 row
    assert runs[1][1] <= 1e-13
    l2 = oracle.l2_norm_diff(runs[1][0], runs[k][0], h, k)
    assert 1e-13 < l2 < 1e-6, l2
    assert runs[0][1] >= 1e-9, runs[0][1]
    assert oracle.l2_norm_diff(runs[0][0], runs[k][0], h, k) > 10 * l2


def test_mass_compensated_sum():
    """mass = volume * sum c0, accurate like math.fsum."""
    rng = np.random.default_rng(11)
    c = rng.standard_normal((100000, 3)) * 1e3
    c[::2, 0] += 1e12
    c[1::2, 0] -= 1e12
    ref = math.fsum(c[:, 0]) * 0.25
    assert abs(oracle.mass(c, 3, 0.25) - ref) <= 1e-15 * abs(ref) + 1e-9


# ----------------------------------------------------------------------------- L2 norm
def test_l2_norm_spec_constant_vs_zeros():
    """S:94 worked example: a = constant 1 on [0,1], b = zeros -> 1.0 within 1e-13, any N."""
    for N, k in [(1, 1), (7, 3), (64, 4), (33, 6)]:
        a = np.zeros((N, k))
        a[:, 0] = 1.0
        assert abs(oracle.l2_norm_diff(a, np.zeros((N, k)), 1.0 / N, k) - 1.0) <= 1e-13
        assert oracle.l2_norm_diff(a, a, 1.0 / N, k) == 0.0  # S:93 a = b -> 0


def test_l2_norm_closed_forms_x_and_x2():
    """Exact per-cell Legendre coefficients of x and x^2 on [0,1] (x = x_c + (h/2) xi,
    xi^2 = P_0/3 + 2 P_2/3): ||x||_2 = 1/sqrt(3), ||x^2||_2 = 1/sqrt(5).  Exercises every
    factor of S:90's formula: a dropped h, a dropped or wrong 1/(2j+1) changes the value."""
    for N in (1, 2, 3, 10):
        h = 1.0 / N
        xc = (np.arange(N) + 0.5) * h
        lin = np.zeros((N, 3))
        lin[:, 0], lin[:, 1] = xc, h / 2
        sq = np.zeros((N, 3))
        sq[:, 0], sq[:, 1], sq[:, 2] = xc * xc + h * h / 12, xc * h, h * h / 6
        z = np.zeros((N, 3))
        assert abs(oracle.l2_norm_diff(lin, z, h, 3) - 1 / math.sqrt(3)) <= 1e-14
        assert abs(oracle.l2_norm_diff(sq, z, h, 3) - 1 / math.sqrt(5)) <= 1e-14


def test_l2_norm_node_formula_library():
    """the node-based formula sqrt(sum_i (h/2) sum_q w_q (u_a - u_b)(x_iq)^2) with the
    DG functions evaluated by numpy's Legendre series (library routines legval / leggauss)
    agrees with the coefficient formula within 1e-12 on random grids."""
    rng = np.random.default_rng(94)
    for k in range(1, 8):
        N = int(rng.integers(1, 40))
        h = 2.5 / N
        a, b = rng.standard_normal((N, k)), rng.standard_normal((N, k))
        xq, wq = np.polynomial.legendre.leggauss(k + 1)
        s = 0.0
        for i in range(N):
            du = np.polynomial.legendre.legval(xq, a[i] - b[i])
            s += 0.5 * h * float(np.sum(wq * du * du))
        assert abs(oracle.l2_norm_diff(a, b, h, k) - math.sqrt(s)) <= 1e-12 * max(1.0, math.sqrt(s))


# ----------------------------------------------------------------------------- multi-D
def _tensor(F, G, nF, kF):
    """c[cell, q] for cell = i0 + n0 * rest, q = m0 + k * qrest, from F[i0,m0] x G[rest,qrest]."""
    return np.einsum("aq,bm->bamq", F, G).reshape(F.shape[0] * G.shape[0], kF * G.shape[1])


@pytest.mark.parametrize("k", [2, 3])
def test_separable_multid_dim0(k):
    """P18: f(x1) g(rest) swept along dim 0 equals (1D sweep of f) x g."""
    rng = np.random.default_rng(3)
    dims = [7, 5, 4, 3]
    F = rng.standard_normal((7, k))
    G = rng.standard_normal((5 * 4 * 3, k ** 3))
    c = _tensor(F, G, 7, k)
    out = oracle.advect(c, dims, k, 0, shift=-2.62)
    ref = _tensor(bruteforce.reproject_line(F, -2.62), G, 7, k)
    assert np.max(np.abs(out - ref)) < 1e-13 * np.max(np.abs(ref))


@pytest.mark.parametrize("dim", [1, 2, 3])
def test_multid_lines_vs_bruteforce_with_field(dim):
    """Per-line CFL fields in 4D: every line along `dim` and every
    coupled group equals the brute-force 1D re-projection with that line's nu.  Pins the
    field indexing (lowest masked dim fastest), the coupled-group indexing (m_dim varies,
    other m spectators) and the strides."""
    rng = np.random.default_rng(dim)
    dims, k = [4, 3, 5, 4], 2
    D, K = 4, k ** 4
    c = rng.standard_normal((int(np.prod(dims)), K))
    other = [d for d in range(D) if d != dim]
    mask = (1 << other[0]) | (1 << other[-1])
    fd = [d for d in range(D) if mask >> d & 1]
    field = rng.uniform(-7, 7, dims[fd[0]] * dims[fd[1]])
    field[0] = 2.0  # an integer entry: copy path
    out = oracle.advect(c, dims, k, dim, field=field, field_mask=mask)
    S = [1, dims[0], dims[0] * dims[1], dims[0] * dims[1] * dims[2]]
    cr = c.reshape(dims[3], dims[2], dims[1], dims[0], *([k] * 4))  # [i3,i2,i1,i0,m3,m2,m1,m0]
    orr = out.reshape(cr.shape)
    import itertools
    for idx in itertools.product(*[range(dims[d]) for d in other]):
        full = dict(zip(other, idx))
        nu = field[full[fd[0]] + dims[fd[0]] * full[fd[1]]]
        for mq in itertools.product(range(k), repeat=3):
            mfull = dict(zip(other, mq))
            sl_c, sl_m = [], []
            for d in [3, 2, 1, 0]:
                sl_c.append(slice(None) if d == dim else full[d])
            for d in [3, 2, 1, 0]:
                sl_m.append(slice(None) if d == dim else mfull[d])
            line = cr[tuple(sl_c + sl_m)]  # [n_dim, k]
            ref = bruteforce.reproject_line(line, nu)
            got = orr[tuple(sl_c + sl_m)]
            assert np.max(np.abs(got - ref)) < 1e-12
    del S


def test_constant_field_equals_constant_shift():
    """all nus equal -> identical to the constant sweep (bit-exact)."""
    rng = np.random.default_rng(9)
    dims, k = [6, 5, 4], 3
    c = rng.standard_normal((120, 27))
    a = oracle.advect(c, dims, k, 1, shift=0.731)
    b = oracle.advect(c, dims, k, 1, field=np.full(24, 0.731), field_mask=0b101)
    assert a.tobytes() == b.tobytes()


def test_multid_mixed_mass_drift_4d():
    """P18 drift: mixed 4D split steps with per-line fields keep mass at fp64 level."""
    dims, k = [8, 8, 8, 8], 2
    kinds = ["x", "x", "v", "v"]
    lo, hi = [0, 0, -6, -6], [4 * np.pi, 4 * np.pi, 6, 6]
    terms = sldg_inputs.landau_terms(dims, k, kinds, lo, hi, eps=0.5)
    c = oracle.round_layout(sldg_inputs.assemble_separable(terms, dims, k), k ** 4, 1)
    vol = np.prod([(hi[d] - lo[d]) / dims[d] for d in range(4)])
    m0 = oracle.mass(c, k ** 4, vol)
    sweeps = sldg_inputs.vlasov_fields(dims, kinds, lo, hi, eps=0.5)
    for _ in range(20):
        for d, field, mask in sweeps:
            c = oracle.advect(c, dims, k, d, field=field, field_mask=mask, n_double=1)
    assert abs(oracle.mass(c, k ** 4, vol) - m0) / abs(m0) < 1e-13


def test_invalid_arguments():
    c = np.zeros((4, 2))
    with pytest.raises(oracle.OracleError):
        oracle.advect(c, [4], 2, 0, shift=float("nan"))
    with pytest.raises(oracle.OracleError):
        oracle.advect(np.zeros((12, 4)), [4, 3], 2, 0, field=np.zeros(4), field_mask=0b1)
