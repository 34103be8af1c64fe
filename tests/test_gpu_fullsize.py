"""GPU parity at the benchmarked sizes (SURVEY 8(d) "Parity at C5 scale").

Every configuration bench.py reports is checked here at its own size, in the launch
configuration the bench times (one GPU, ping-pong arrays, the same plan and kernels):

* C3 4096^2, k = 2..6, mixed and fp64, dims 0 and 1: the order-sweep shift (nu = 2.37, P:268
  decomposition i* = 2, alpha = 0.37) and the Vlasov per-line fields of the bench;
* C4 64^4, k = 2, mixed and fp64, all four sweeps of the split step (eps = 0.01 and 0.5);
* C5 128^4, k = 3, mixed, all four sweeps, 64 lines per sweep including the first and the last
  tile of every sweep, eps = 0.01 and 0.5;
* 32^4, k = 3 (C5's kernels and tiling on a grid the oracle sweeps whole): full-grid
  element-wise parity, random and smooth (Landau) data, mixed and fp64;
* the separable-product check at 128^4 with constant shifts: a
  tensor-product input stays the product of the 1D oracle results.

The update under test is P:259-272 (SS II-A).  Lines are recomputed by the oracle alone: the
update is line-local, so an output line needs only its own source line.
Tolerances as in test_gpu_parity.assert_parity (DESIGN R8).
"""

import numpy as np
import pytest

import oracle
import sldg_inputs
from tests.test_gpu_parity import assert_parity, n_double

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")

X4 = ["x", "x", "v", "v"]
LO4, HI4 = [0.0, 0.0, -6.0, -6.0], [4 * np.pi, 4 * np.pi, 6.0, 6.0]
X2 = ["x", "v"]
LO2, HI2 = [0.0, -6.0], [4 * np.pi, 6.0]


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    torch.cuda.set_device(0)
    yield


def _Grid(*a, **kw):
    from paper_1603_07008_b200 import Grid
    return Grid(*a, **kw)


def _strides(dims):
    return np.cumprod([1] + list(dims[:-1])).astype(np.int64)


def _field_value(field, mask, perp, dims):
    if field is None:
        return 0.0
    fi, st = 0, 1
    for e in range(len(dims)):
        if mask >> e & 1:
            fi += perp[e] * st
            st *= dims[e]
    return float(field[fi])


def _windows(dims, dim, rng, n_lines, width=8):
    """Line windows along `dim`: the first tile (every perpendicular index 0), the last tile
    (every perpendicular index at its maximum) and random ones.  A window is (perp, w): w
    consecutive i0 values starting at perp[0] (dim > 0; lines along a strided dim), or one line
    (dim == 0)."""
    D = len(dims)
    w = 1 if dim == 0 else min(width, dims[0])
    first = {e: 0 for e in range(D) if e != dim}
    last = {e: dims[e] - 1 for e in range(D) if e != dim}
    if dim > 0:
        last[0] = dims[0] - w
    out = [(first, w), (last, w)]
    while sum(x[1] for x in out) < n_lines:
        p = {e: int(rng.integers(0, dims[e])) for e in range(D) if e != dim}
        if dim > 0:
            p[0] = int(rng.integers(0, dims[0] - w + 1))
        out.append((p, w))
    return out


def _gather_window(g, dims, dim, perp, w):
    """Device coefficients of the w lines of a window, [w, n_dim, K] (and their cell indices)."""
    S = _strides(dims)
    base = int(sum(perp[e] * S[e] for e in perp))
    n = dims[dim]
    if dim == 0:
        cells = base + np.arange(n)
        return g.get_coeffs(base, n)[None], cells[None]
    rows = [g.get_coeffs(base + int(x * S[dim]), w) for x in range(n)]  # [n][w, K]
    got = np.stack(rows, axis=1)
    cells = base + np.arange(w)[:, None] + np.arange(n)[None, :] * S[dim]
    return got, cells


def check_lines(g, dims, k, precision, dim, field, mask, windows, src_of, shift=0.0, tag=""):
    """Compare every line of `windows` after a sweep along dim with the oracle's sweep of the
    line alone.  src_of(cells) -> the stored (layout-rounded) source coefficients."""
    D, K = len(dims), k ** len(dims)
    nd = n_double(precision, K)
    ldims = [1] * D
    ldims[dim] = dims[dim]
    nlines = 0
    for perp, w in windows:
        got, cells = _gather_window(g, dims, dim, perp, w)
        for j in range(got.shape[0]):
            p = dict(perp)
            if dim > 0:
                p[0] = perp[0] + j
            nu = shift if field is None else _field_value(field, mask, p, dims)
            src = src_of(cells[j])
            ref = oracle.advect(src, ldims, k, dim, shift=nu, n_double=nd)
            assert_parity(got[j], ref, K, precision, f"{tag} dim={dim} perp={p} nu={nu:.4f}", src, dim, k)
            nlines += 1
    return nlines


def _random_src(dims, k, precision, seed):
    K = k ** len(dims)
    return lambda cells: oracle.round_layout(
        sldg_inputs.random_coeffs(dims, k, seed, cells=cells), K, n_double(precision, K))


# ------------------------------------------------------------------------------------- C3
@pytest.mark.parametrize("precision", ["mixed", "fp64"])
@pytest.mark.parametrize("k", [2, 3, 4, 5, 6])
def test_c3_4096sq_all_orders(k, precision):
    """BASELINE configs[2] at size: every k of the order sweep, both storages, both sweep dims,
    the order-sweep shift (nu = 2.37) and the bench's Vlasov fields (eps = 0.5: per-lane
    spans up to 2 cells on the strided sweep)."""
    dims = [4096, 4096]
    g = _Grid(dims, k, lo=LO2, hi=HI2, precision=precision)
    rng = np.random.default_rng(100 + k)
    src_of = _random_src(dims, k, precision, 7008)
    fields = {d: (f, m) for d, f, m in sldg_inputs.vlasov_fields(dims, X2, LO2, HI2, eps=0.5)}
    n = 0
    for dim in [0, 1]:
        g.fill_random(7008)
        g.advect(dim, shift=2.37)
        n += check_lines(g, dims, k, precision, dim, None, 0, _windows(dims, dim, rng, 12), src_of,
                         shift=2.37, tag=f"C3 k={k} {precision} nu=2.37")
        f, m = fields[dim]
        g.fill_random(7008)
        g.advect(dim, field=f, field_mask=m)
        n += check_lines(g, dims, k, precision, dim, f, m, _windows(dims, dim, rng, 12), src_of,
                         tag=f"C3 k={k} {precision} vlasov")
    g.destroy()
    assert n >= 48


# ------------------------------------------------------------------------------------- C4
@pytest.mark.parametrize("eps", [0.01, 0.5])
@pytest.mark.parametrize("precision", ["mixed", "fp64"])
def test_c4_64e4_all_sweeps(precision, eps):
    """BASELINE configs[3] at size (64^4, k = 2): each sweep of the split step with the bench's
    fields, 64 lines per sweep including the first and last tile."""
    dims, k = [64, 64, 64, 64], 2
    g = _Grid(dims, k, lo=LO4, hi=HI4, precision=precision)
    rng = np.random.default_rng(4)
    src_of = _random_src(dims, k, precision, 1603)
    for d, f, m in sldg_inputs.vlasov_fields(dims, X4, LO4, HI4, eps=eps):
        g.fill_random(1603)
        g.advect(d, field=f, field_mask=m)
        n = check_lines(g, dims, k, precision, d, f, m, _windows(dims, d, rng, 64), src_of,
                        tag=f"C4 {precision} eps={eps}")
        assert n >= 64
    g.destroy()


# ------------------------------------------------------------------------------------- C5
@pytest.mark.parametrize("eps", [0.01, 0.5])
def test_c5_128e4_64_lines_per_sweep(eps):
    """BASELINE configs[4] at size (128^4, k = 3, mixed; the bench's own grid): each sweep of
    the split step, 64 lines per sweep including the first and the last tile."""
    dims, k = [128, 128, 128, 128], 3
    g = _Grid(dims, k, lo=LO4, hi=HI4, precision="mixed")
    rng = np.random.default_rng(55)
    src_of = _random_src(dims, k, "mixed", 1603)
    for d, f, m in sldg_inputs.vlasov_fields(dims, X4, LO4, HI4, eps=eps):
        g.fill_random(1603)
        g.advect(d, field=f, field_mask=m)
        n = check_lines(g, dims, k, "mixed", d, f, m, _windows(dims, d, rng, 64), src_of,
                        tag=f"C5 eps={eps}")
        assert n >= 64
    g.destroy()


# ------------------------------------------------------------------------------------- 32^4
def _full_grid_sequence(dims, k, precision, kinds, lo, hi, eps, c0, tag):
    """The four sweeps of a split step on the whole grid, each compared element-wise with the
    oracle's sweep of the same stored state (the state is re-synchronised after each sweep, so
    every comparison is one sweep from identical inputs)."""
    K = k ** len(dims)
    nd = n_double(precision, K)
    g = _Grid(dims, k, lo=lo, hi=hi, precision=precision)
    cur = oracle.round_layout(c0, K, nd)  # the stored (layout-rounded) state, host side
    g.set_coeffs(cur)
    for d, f, m in sldg_inputs.vlasov_fields(dims, kinds, lo, hi, eps=eps):
        g.advect(d, field=f, field_mask=m)
        ref = oracle.advect(cur, dims, k, d, field=f, field_mask=m, n_double=nd)
        got = g.get_coeffs()
        assert_parity(got, ref, K, precision, f"{tag} sweep {d}", cur, d, k)
        cur = oracle.round_layout(ref, K, nd)
        g.set_coeffs(cur)
    g.destroy()


@pytest.mark.parametrize("eps", [0.01, 0.5])
@pytest.mark.parametrize("precision", ["mixed", "fp64"])
def test_32e4_k3_full_grid_random(precision, eps):
    """a reduced 4D grid (32^4, k = 3) through the same kernels
    (TMA d = 0 and strided paths, k = 3 instances), every element compared."""
    dims, k = [32, 32, 32, 32], 3
    c0 = sldg_inputs.random_coeffs(dims, k, 1603)
    _full_grid_sequence(dims, k, precision, X4, LO4, HI4, eps, c0, f"32^4 random {precision}")


@pytest.mark.parametrize("precision", ["mixed", "fp64"])
def test_32e4_k3_full_grid_smooth_landau(precision):
    """smooth data (the bench's Landau IC, c_j ~ h^j formed by cancellation of O(1)
    terms) at k = 3 in 4D, every element compared -- where fp32 arithmetic would fail the bar."""
    dims, k = [32, 32, 32, 32], 3
    c0 = sldg_inputs.assemble_separable(sldg_inputs.landau_terms(dims, k, X4, LO4, HI4, eps=0.5), dims, k)
    assert np.all(np.isfinite(c0)) and np.min(c0[:, 0]) > 0
    _full_grid_sequence(dims, k, precision, X4, LO4, HI4, 0.5, c0, f"32^4 landau {precision}")


# ------------------------------------------------------------------------------------- P18
def _dyadic_factors(n, k, rng):
    """[n, k] 1D factors r * 2^-(5 + 7m), r a 5-bit integer (m = 0: 16..31).  Four of them
    multiply to at most 20 significant bits, so the tensor product is exact in fp32 storage."""
    r = rng.integers(-31, 32, size=(n, k)).astype(np.float64)
    r[:, 0] = rng.integers(16, 32, size=n)
    return r * 2.0 ** -(5 + 7 * np.arange(k))[None, :]


def test_c5_separable_product_constant_shifts():
    """on the 128^4, k = 3 grid a tensor-product input
    c(i, m) = prod_d a_d(i_d, m_d), swept along d with a constant shift, must equal
    oracle_1D(a_d) x prod_{e != d} a_e on every cell -- checked on sampled cells of every
    sweep, with the plane maxima known exactly from the factors."""
    dims, k = [128, 128, 128, 128], 3
    D, K = 4, 81
    rng = np.random.default_rng(18)
    fac = [_dyadic_factors(dims[d], k, rng) for d in range(D)]
    shifts = [2.37, -1.61, 0.43, -3.77]
    g = _Grid(dims, k, precision="mixed")
    S = _strides(dims)
    m_idx = np.array([[(q // k ** d) % k for d in range(D)] for q in range(K)])  # [K, D]
    for d in range(D):
        g.fill_separable([[f for f in fac]])
        g.advect(d, shift=shifts[d])
        a1 = oracle.advect(fac[d], [dims[d]], k, 0, shift=shifts[d], n_double=k)  # fp64 1D line
        cur = list(fac)
        cur[d] = a1
        # exact plane maxima of the swept tensor product: product of the per-dim column maxima
        pmax = np.ones(K)
        for e in range(D):
            pmax *= np.max(np.abs(cur[e]), axis=0)[m_idx[:, e]]
        idx = rng.integers(0, dims, size=(4096, D))
        idx[0] = 0
        idx[1] = np.array(dims) - 1
        cells = idx @ S
        order = np.argsort(cells)
        got = np.concatenate([g.get_coeffs(int(c), 1) for c in cells[order]])
        idx = idx[order]
        exp = np.ones((len(cells), K))
        for e in range(D):
            exp *= cur[e][idx[:, e]][:, m_idx[:, e]]
        for q in range(K):
            dq = np.max(np.abs(got[:, q] - exp[:, q]))
            tol = 1e-13 * pmax[q] if q == 0 else 8.0 * float(np.spacing(np.float32(pmax[q])))
            assert dq <= tol, f"sweep {d} slot {q}: |d|={dq:.3e} > {tol:.3e}"
    g.destroy()
