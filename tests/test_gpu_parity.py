"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle on identical seeded
inputs.  Tolerances (BASELINE.json north_star): fp64 mass slot |d| <= 1e-13 *
max|c0| per array; fp32 slots |d| <= 8 ulp_fp32(max|plane|) per plane; fp64 variant 1e-13 *
max|plane| per plane; integer shifts bit-exact; mass 1e-13 relative.
"""

import numpy as np
import pytest

import oracle
import sldg_inputs

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    torch.cuda.set_device(0)
    yield


def _Grid(*a, **kw):
    from paper_1603_07008_b200 import Grid
    return Grid(*a, **kw)


def assert_parity(got, ref, K, precision, tag="", src=None, dim=None, k=None):
    """Element-wise parity (reading R8).  fp64 slots: |d| <= 1e-13 * scale with
    scale = max(max|ref plane|, max|source planes it is computed from|) -- an fp64 result of
    a contraction is only accurate relative to its inputs (smooth data: c_j ~ h^j is formed by
    cancellation of O(1) terms).  fp32 slots: 8 ulp_fp32 of max|ref plane| (per plane, stricter
    than the north_star's per-array bar), plus the same fp64 contraction bound 1e-13 * max|source
    planes| when the sources are given: a plane formed by cancellation (e.g. the x1-sweep of the
    x2-slope of data constant along x1: (A_j0 + B_j0) c = O(1e-16) c) holds fp64 rounding noise,
    which the two sides round to fp32 differently."""
    got = np.asarray(got).reshape(-1, K)
    ref = np.asarray(ref).reshape(-1, K)
    if src is not None:
        src = np.asarray(src).reshape(-1, K)
    for q in range(K):
        m = np.max(np.abs(ref[:, q]))
        d = np.max(np.abs(got[:, q] - ref[:, q]))
        sscale = 0.0
        if src is not None:
            kd = k ** dim
            q0 = q - ((q // kd) % k) * kd
            sscale = max(np.max(np.abs(src[:, q0 + l * kd])) for l in range(k))
        if precision == "fp64" or q == 0:
            tol = 1e-13 * max(m, sscale)
        else:
            tol = 8.0 * float(np.spacing(np.float32(m))) + 1e-13 * sscale
        assert d <= tol, f"{tag} slot {q}: |d|={d:.3e} > tol={tol:.3e} (max {m:.3e})"


def n_double(precision, K):
    return 1 if precision == "mixed" else K


def oracle_input(c, K, precision):
    return oracle.round_layout(c, K, n_double(precision, K))


# ------------------------------------------------------------------------------ single sweeps
CASES = [
    # dims, k
    ([64], 4),
    ([100], 3),
    ([1000], 1),
    ([5], 6),
    ([256, 64], 2),
    ([100, 37], 4),
    ([31, 33], 5),
    ([48, 40], 6),
    ([33, 7, 10], 3),
    ([16, 6, 5, 9], 2),
    ([8, 4, 6, 5], 3),
    ([40, 3, 1, 7], 2),
    ([12, 5, 4, 3, 2], 2),
    # inner sweeps with < 256 cells below d: tiles of HC = 256 / M_lo hi values (dim 1 here)
    ([64, 16, 8, 6], 2),
    ([32, 8, 16, 4], 3),
]


@pytest.mark.parametrize("precision", ["mixed", "fp64"])
@pytest.mark.parametrize("dims,k", CASES)
def test_single_sweeps_all_dims(dims, k, precision):
    """Every dim, constant shifts of both signs and |nu| > n, and per-line fields over the
    other dims (including per-lane fields on strided sweeps)."""
    D, K = len(dims), k ** len(dims)
    rng = np.random.default_rng(abs(hash((tuple(dims), k))) % 2**32)
    c = sldg_inputs.random_coeffs(dims, k, 1603)
    ref_in = oracle_input(c, K, precision)
    g = _Grid(dims, k, precision=precision)
    for dim in range(D):
        others = [e for e in range(D) if e != dim]
        variants = [("const", 2.37, None, 0), ("neg", -0.63 - dims[dim], None, 0)]
        if others:
            mask = 0
            for e in others[: 2]:
                mask |= 1 << e
            nf = int(np.prod([dims[e] for e in range(D) if mask >> e & 1]))
            field = rng.uniform(-2.5 * dims[dim], 2.5 * dims[dim], nf)
            field[:: 7] = np.round(field[:: 7])  # some integer (copy) lines
            variants.append(("field", 0.0, field, mask))
            if 0 in others:
                mask0 = 1  # per-lane field over dim 0 only
                f0 = rng.uniform(-1.6, 1.6, dims[0])
                variants.append(("lane", 0.0, f0, mask0))
        for name, shift, field, mask in variants:
            g.set_coeffs(c)
            g.advect(dim, shift=shift, field=field, field_mask=mask)
            got = g.get_coeffs()
            ref = oracle.advect(ref_in, dims, k, dim, shift=shift, field=field, field_mask=mask,
                                n_double=n_double(precision, K))
            assert_parity(got, ref, K, precision, f"dims={dims} k={k} dim={dim} {name}", ref_in, dim, k)
    g.destroy()


@pytest.mark.parametrize("precision", ["mixed", "fp64"])
def test_integer_shifts_bit_exact(precision):
    """Integer nu is an exact permutation, incl. -0.0 and tiny-negative nu."""
    dims, k = [40, 12, 6], 3
    K = k ** 3
    c = sldg_inputs.random_coeffs(dims, k, 7008)
    c[5, 3] = -0.0
    c[7, 0] = -0.0
    ref_in = oracle_input(c, K, precision)
    g = _Grid(dims, k, precision=precision)
    for dim, nu in [(0, 3.0), (0, -41.0), (1, 5.0), (2, -1.0), (2, 0.0), (1, -1e-20)]:
        g.set_coeffs(c)
        g.advect(dim, shift=nu)
        got = g.get_coeffs()
        ref = oracle.advect(ref_in, dims, k, dim, shift=nu, n_double=n_double(precision, K))
        assert got.tobytes() == ref.tobytes(), (dim, nu)
    g.destroy()


def test_c1_config_100_steps():
    """BASELINE configs[0]: 1D, 64 cells, k=4, nu=0.37, 100 steps, IC 1 + sin(2 pi x)/2."""
    N, k, nu = 64, 4, 0.37
    c0 = sldg_inputs.project_1d(lambda x: 1.0 + 0.5 * np.sin(2 * np.pi * x), N, 0.0, 1.0, k, 12)
    for precision in ["mixed", "fp64"]:
        nd = n_double(precision, k)
        g = _Grid([N], k, precision=precision)
        g.set_coeffs(c0)
        ref = oracle.round_layout(c0, k, nd)
        g.advect(0, shift=nu)
        ref1 = oracle.advect(ref, [N], k, 0, shift=nu, n_double=nd)
        assert_parity(g.get_coeffs(), ref1, k, precision, "C1 step 1", ref, 0, k)
        ref = ref1
        for _ in range(99):
            g.advect(0, shift=nu)
            ref = oracle.advect(ref, [N], k, 0, shift=nu, n_double=nd)
        got = g.get_coeffs()
        # multi-step: L2 distance and mass drift, not per-ulp
        assert oracle.l2_norm_diff(got, ref, 1.0 / N, k) < (1e-12 if precision == "fp64" else 1e-7)
        m0 = oracle.mass(oracle.round_layout(c0, k, nd), k, 1.0 / N)
        assert abs(g.mass() - m0) / m0 < 1e-14
        exact = sldg_inputs.project_1d(lambda x: 1.0 + 0.5 * np.sin(2 * np.pi * (x - nu * 100 / N)),
                                       N, 0.0, 1.0, k, 12)
        err = oracle.l2_norm_diff(got, exact, 1.0 / N, k)
        assert err < 1e-8, err  # SURVEY P17 magnitude ~3e-9
        g.destroy()


def test_mass_and_drift_1000_steps():
    """Mass conserved to fp64 accuracy: mixed 2D Landau, 500 split steps
    (1000 sweeps) with per-line fields: relative drift <= 1e-12 (north_star)."""
    dims, k = [64, 64], 4
    kinds, lo, hi = ["x", "v"], [0.0, -6.0], [4 * np.pi, 6.0]
    terms = sldg_inputs.landau_terms(dims, k, kinds, lo, hi, eps=0.5)
    c = sldg_inputs.assemble_separable(terms, dims, k)
    g = _Grid(dims, k, lo=lo, hi=hi, precision="mixed")
    g.set_coeffs(c)
    vol = (hi[0] - lo[0]) / 64 * (hi[1] - lo[1]) / 64
    ref = oracle.round_layout(c, k * k, 1)
    m0 = oracle.mass(ref, k * k, vol)
    assert abs(g.mass() - m0) <= 1e-13 * abs(m0)
    sweeps = sldg_inputs.vlasov_fields(dims, kinds, lo, hi, eps=0.5)
    for _ in range(500):
        for d, f, mask in sweeps:
            g.advect(d, field=f, field_mask=mask)
    assert abs(g.mass() - m0) / abs(m0) <= 1e-12


def test_mass_matches_oracle():
    for dims, k, prec in [([1000], 3, "mixed"), ([50, 30, 7], 2, "fp64"), ([17, 9, 5, 4], 2, "mixed")]:
        K = k ** len(dims)
        c = sldg_inputs.random_coeffs(dims, k, 3)
        g = _Grid(dims, k, lo=[-1.0] * len(dims), hi=[2.0] * len(dims), precision=prec)
        g.set_coeffs(c)
        vol = np.prod([3.0 / n for n in dims])
        ref = oracle.mass(oracle.round_layout(c, K, n_double(prec, K)), K, vol)
        assert abs(g.mass() - ref) <= 1e-13 * abs(ref)
        g.destroy()


# ------------------------------------------------------------------------------ set / get / fill
def test_set_get_roundtrip_and_validation():
    from paper_1603_07008_b200 import SldgError
    dims, k = [20, 6], 2
    K = 4
    c = sldg_inputs.random_coeffs(dims, k, 1)
    c[3, 1] = 0.1
    c[4, 2] = 2.0 ** -150  # rounds to 0 or the smallest subnormal (RNE)
    g = _Grid(dims, k, precision="mixed")
    g.set_coeffs(c)
    got = g.get_coeffs()
    assert got[:, 0].tobytes() == c[:, 0].tobytes()  # fp64 slot bit-exact
    assert got[:, 1:].tobytes() == c[:, 1:].astype(np.float32).astype(np.float64).tobytes()
    # partial ranges
    part = g.get_coeffs(37, 50)
    assert part.tobytes() == got[37:87].tobytes()
    g.set_coeffs(np.zeros((5, K)), first_cell=100)
    assert np.all(g.get_coeffs(100, 5) == 0)
    before = g.get_coeffs()
    bad = c.copy()
    bad[10, 0] = np.nan
    with pytest.raises(SldgError):
        g.set_coeffs(bad)
    bad = c.copy()
    bad[11, 3] = 1e39
    with pytest.raises(SldgError):
        g.set_coeffs(bad)
    with pytest.raises(SldgError):
        g.set_coeffs(c[:10], first_cell=115)
    with pytest.raises(SldgError):
        g.advect(0, shift=float("inf"))
    with pytest.raises(SldgError):
        g.advect(0, field=np.zeros(20), field_mask=0b01)
    with pytest.raises(SldgError):
        g.advect(1, field=np.array([0.5, np.nan] * 10), field_mask=0b01)
    with pytest.raises(SldgError):
        g.advect(2, shift=0.5)
    assert g.get_coeffs().tobytes() == before.tobytes()  # EINVAL changed nothing
    g.destroy()


@pytest.mark.parametrize("precision", ["mixed", "fp64"])
def test_fill_random_bit_exact(precision):
    dims, k = [37, 11, 6], 3
    K = 27
    g = _Grid(dims, k, precision=precision)
    g.fill_random(1603)
    ref = oracle_input(sldg_inputs.random_coeffs(dims, k, 1603), K, precision)
    assert g.get_coeffs().tobytes() == ref.tobytes()
    g.destroy()


def test_fill_separable():
    dims, k = [16, 12], 4
    kinds, lo, hi = ["x", "v"], [0.0, -6.0], [4 * np.pi, 6.0]
    terms = sldg_inputs.landau_terms(dims, k, kinds, lo, hi)
    g = _Grid(dims, k, lo=lo, hi=hi, precision="fp64")
    g.fill_separable(terms)
    ref = sldg_inputs.assemble_separable(terms, dims, k)
    np.testing.assert_allclose(g.get_coeffs(), ref, rtol=0, atol=1e-15)
    g.destroy()


def test_device_field_and_sticky_error():
    from paper_1603_07008_b200 import SldgError
    dims, k = [64, 32], 3
    K = 9
    c = sldg_inputs.random_coeffs(dims, k, 5)
    g = _Grid(dims, k, precision="mixed")
    g.set_coeffs(c)
    field = np.linspace(-5.5, 7.25, 32)
    tf = torch.tensor(field, dtype=torch.float64, device="cuda")
    torch.cuda.synchronize()
    g.advect_device(0, tf.data_ptr(), 0b10)
    ref = oracle.advect(oracle_input(c, K, "mixed"), dims, k, 0, field=field, field_mask=0b10, n_double=1)
    assert_parity(g.get_coeffs(), ref, K, "mixed", "device field", oracle_input(c, K, "mixed"), 0, k)
    bad = tf.clone()
    bad[3] = float("nan")
    torch.cuda.synchronize()
    before = g.get_coeffs()
    g.advect_device(0, bad.data_ptr(), 0b10)
    with pytest.raises(SldgError):
        g.sync()
    after = g.get_coeffs()  # flag was reset by the failing sync
    v = after.reshape(32, 64, K)
    b = before.reshape(32, 64, K)
    assert v[3].tobytes() == b[3].tobytes()  # the invalid line was left unchanged
    g.destroy()


# ------------------------------------------------------------------------------ properties
def test_convergence_order_fp64():
    """P11 on the GPU path: order k on smooth data, fixed CFL 0.8, one period."""
    for k in [2, 3, 4]:
        errs = []
        for N in [40, 80, 160]:
            c0 = sldg_inputs.project_1d(lambda x: np.sin(2 * np.pi * x), N, 0.0, 1.0, k, 12)
            g = _Grid([N], k, precision="fp64")
            g.set_coeffs(c0)
            for _ in range(N * 5 // 4):
                g.advect(0, shift=0.8)
            errs.append(oracle.l2_norm_diff(g.get_coeffs(), c0, 1.0 / N, k))
            g.destroy()
        orders = np.log2(np.array(errs[:-1]) / np.array(errs[1:]))
        assert orders.min() >= k - 0.3, (k, errs)


# ------------------------------------------------------------------------------ full sizes
def _line_cells(dims, dim, perp):
    """Global cell indices of the line along `dim` with perpendicular indices perp (dict)."""
    S = np.cumprod([1] + list(dims[:-1]))
    base = sum(perp[e] * S[e] for e in perp)
    return base + np.arange(dims[dim]) * S[dim]


def _sampled_line_parity(g, dims, k, precision, dim, field, mask, seed, n_lines, rng):
    D, K = len(dims), k ** len(dims)
    nd = n_double(precision, K)
    fd = [e for e in range(D) if mask >> e & 1]
    for _ in range(n_lines):
        perp = {e: int(rng.integers(0, dims[e])) for e in range(D) if e != dim}
        cells = _line_cells(dims, dim, perp)
        src = oracle.round_layout(sldg_inputs.random_coeffs(dims, k, seed, cells=cells), K, nd)
        fi, st = 0, 1
        for e in fd:
            fi += perp[e] * st
            st *= dims[e]
        nu = float(field[fi]) if field is not None else 0.0
        ldims = [1] * D
        ldims[dim] = dims[dim]
        ref = oracle.advect(src, ldims, k, dim, shift=nu, n_double=nd)
        got = np.concatenate([g.get_coeffs(int(c), 1) for c in cells]) if dim > 0 else \
            g.get_coeffs(int(cells[0]), dims[0])
        assert_parity(got, ref, K, precision, f"line dim={dim} perp={perp}", src, dim, k)


@pytest.mark.parametrize("precision", ["mixed", "fp64"])
def test_c2_full_grid(precision):
    """BASELINE configs[1]: 2D 1024^2, k=4, v-dependent x-shift + E(x)-dependent v-shift,
    full-grid element-wise parity."""
    dims, k = [1024, 1024], 4
    K = 16
    kinds, lo, hi = ["x", "v"], [0.0, -6.0], [4 * np.pi, 6.0]
    c = sldg_inputs.random_coeffs(dims, k, 1603)
    g = _Grid(dims, k, lo=lo, hi=hi, precision=precision)
    g.set_coeffs(c)
    ref = oracle_input(c, K, precision)
    for d, f, mask in sldg_inputs.vlasov_fields(dims, kinds, lo, hi, eps=0.5):
        g.advect(d, field=f, field_mask=mask)
        prev = ref
        ref = oracle.advect(ref, dims, k, d, field=f, field_mask=mask, n_double=n_double(precision, K))
        assert_parity(g.get_coeffs(), ref, K, precision, f"C2 sweep {d}", prev, d, k)
        g.set_coeffs(oracle_input(ref, K, precision))  # re-sync state: one-sweep parity each time
    g.destroy()


@pytest.mark.parametrize("k", [2, 6])
def test_c3_order_sweep_sampled(k):
    """BASELINE configs[2]: 2D 4096^2, nu = 2.37 along dim 0 and dim 1, mixed; sampled lines."""
    dims = [4096, 4096]
    g = _Grid(dims, k, precision="mixed")
    rng = np.random.default_rng(k)
    for dim in [0, 1]:
        g.fill_random(7008)
        g.advect(dim, shift=2.37)
        _sampled_line_parity(g, dims, k, "mixed", dim, np.array([2.37]), 0, 7008, 6, rng)
    g.destroy()


def test_c5_full_size_sampled_lines():
    """BASELINE configs[4]: 4D 128^4, k=3, mixed, in the bench's launch configuration (one
    GPU, ping-pong): every sweep of the split step on the random parity input, sampled lines
    recomputed by the oracle (the update is line-local)."""
    dims, k = [128, 128, 128, 128], 3
    kinds = ["x", "x", "v", "v"]
    lo, hi = [0, 0, -6, -6], [4 * np.pi, 4 * np.pi, 6, 6]
    g = _Grid(dims, k, lo=lo, hi=hi, precision="mixed")
    rng = np.random.default_rng(5)
    for d, f, mask in sldg_inputs.vlasov_fields(dims, kinds, lo, hi, eps=0.5):
        g.fill_random(1603)
        g.advect(d, field=f, field_mask=mask)
        _sampled_line_parity(g, dims, k, "mixed", d, f, mask, 1603, 3, rng)
    g.destroy()


# ------------------------------------------------------------------------------ halo path (1 GPU)
@pytest.mark.parametrize("nccl_self", [False, True])
@pytest.mark.parametrize("precision", ["mixed", "fp64"])
@pytest.mark.parametrize("dims,k", [([64, 24], 3), ([32, 6, 20], 2), ([128, 4, 3, 18], 3), ([16, 8, 8, 9], 4)])
def test_forced_halo_path_matches_oracle(dims, k, precision, nccl_self):
    """The multi-GPU halo addressing (pad layers, halo exchange plan, interior/boundary launch
    split) run on one GPU: SLDG_DIST_FORCE_HALO makes the rank its own ring neighbour.  Every
    dim is swept (pad > 0 changes every kernel's addressing); the layer-dim sweeps use shifts
    up to the halo width and a per-lane field."""
    D, K = len(dims), k ** len(dims)
    c = sldg_inputs.random_coeffs(dims, k, 4242)
    ref_in = oracle_input(c, K, precision)
    # nccl_self: the wrap-around halo layers go through ncclSend/ncclRecv on a one-rank
    # communicator (the multi-GPU message code path)
    g = _Grid(dims, k, precision=precision, force_halo=True, max_halo=3, nccl_self=nccl_self)
    rng = np.random.default_rng(len(dims))
    cases = [(d, 1.37, None, 0) for d in range(D)]
    cases += [(D - 1, -2.25, None, 0), (D - 1, 2.0, None, 0), (D - 1, 0.0, rng.uniform(-2.9, 1.9, dims[0]), 1)]
    for d, shift, field, mask in cases:
        g.set_coeffs(c)
        g.advect(d, shift=shift, field=field, field_mask=mask)
        ref = oracle.advect(ref_in, dims, k, d, shift=shift, field=field, field_mask=mask,
                            n_double=n_double(precision, K))
        assert_parity(g.get_coeffs(), ref, K, precision, f"halo dims={dims} dim={d} nu={shift}", ref_in, d, k)
    # a halo of 5 layers > max_halo = 3 takes the transpose path
    assert g.transpose_count() == 0
    g.set_coeffs(c)
    g.advect(D - 1, shift=4.5)
    assert g.transpose_count() == 1
    ref = oracle.advect(ref_in, dims, k, D - 1, shift=4.5, n_double=n_double(precision, K))
    assert_parity(g.get_coeffs(), ref, K, precision, f"auto-transpose dims={dims}", ref_in, D - 1, k)
    g.destroy()


@pytest.mark.parametrize("nccl_self", [False, True])
@pytest.mark.parametrize("precision", ["mixed", "fp64"])
@pytest.mark.parametrize("dims,k", [([64, 24], 3), ([32, 6, 20], 2), ([8, 5, 3, 11], 3), ([12, 4, 7], 4)])
def test_forced_transpose_path_matches_oracle(dims, k, precision, nccl_self):
    """The transpose path (pack per slab, all-to-all, whole-line local sweep with the field
    restricted to the slab, inverse exchange, unpack) on one GPU (SLDG_DIST_FORCE_TRANSPOSE):
    sweeps along the layer dim with small and large constant shifts and per-line fields over
    the slab dim and another dim; sweeps along the other dims stay on the local path."""
    D, K = len(dims), k ** len(dims)
    c = sldg_inputs.random_coeffs(dims, k, 99)
    ref_in = oracle_input(c, K, precision)
    g = _Grid(dims, k, precision=precision, force_transpose=True, max_halo=1, nccl_self=nccl_self)
    rng = np.random.default_rng(D * 10 + k)
    nf = dims[0] * dims[D - 2] if D > 2 else dims[0]
    fmask = (1 | (1 << (D - 2))) if D > 2 else 1
    cases = [(D - 1, 1.37, None, 0), (D - 1, -7.75 - dims[-1], None, 0), (D - 1, 3.0, None, 0),
             (D - 1, 0.0, rng.uniform(-2.5 * dims[-1], 2.5 * dims[-1], nf), fmask), (0, 2.6, None, 0)]
    n_tr = 0
    for d, shift, field, mask in cases:
        g.set_coeffs(c)
        g.advect(d, shift=shift, field=field, field_mask=mask)
        n_tr += (d == D - 1)
        assert g.transpose_count() == n_tr
        ref = oracle.advect(ref_in, dims, k, d, shift=shift, field=field, field_mask=mask,
                            n_double=n_double(precision, K))
        got = g.get_coeffs()
        if shift == 3.0:
            assert got.tobytes() == ref.tobytes()  # integer shift: exact rotation through the transpose
        assert_parity(got, ref, K, precision, f"transpose dims={dims} dim={d} nu={shift}", ref_in, d, k)
    g.destroy()


# ------------------------------------------------------------------------------ bounded sharded sweeps
@pytest.mark.parametrize("nccl_self", [False, True])
@pytest.mark.parametrize("precision", ["mixed", "fp64"])
@pytest.mark.parametrize("dims,k", [([64, 24], 3), ([32, 6, 20], 2), ([16, 8, 8, 9], 4)])
def test_bounded_sharded_sweep_matches_oracle_and_captures(dims, k, precision, nccl_self):
    """sldg_advect_device_bounded along the sharded (layer) dim: the halo is sized from the
    caller's bound (lines read layers i - i* - 1 and i - i*), with no host read of
    the field; the result matches the oracle, and the same sweep captured in a CUDA graph on the
    sharded grid (halo exchange included) replays bit-identically."""
    D, K = len(dims), k ** len(dims)
    c = sldg_inputs.random_coeffs(dims, k, 515)
    ref_in = oracle_input(c, K, precision)
    rng = np.random.default_rng(D + k)
    f = rng.uniform(-1.9, 1.4, dims[0])  # per-lane field over dim 0: i* in [-2, 1] -> halo (2, 2)
    df = torch.tensor(f, dtype=torch.float64, device="cuda")
    g = _Grid(dims, k, precision=precision, force_halo=True, max_halo=2, nccl_self=nccl_self)
    ref = oracle.advect(ref_in, dims, k, D - 1, field=f, field_mask=1, n_double=n_double(precision, K))
    g.set_coeffs(c)
    g.advect_device_bounded(D - 1, df.data_ptr(), 1, -1.9, 1.4)
    got = g.get_coeffs()
    assert g.transpose_count() == 0
    assert_parity(got, ref, K, precision, f"bounded dims={dims}", ref_in, D - 1, k)
    # graph capture of two bounded layer-dim sweeps (an even number keeps the ping-pong buffer)
    g.set_coeffs(c)
    g.graph_begin()
    g.advect_device_bounded(D - 1, df.data_ptr(), 1, -1.9, 1.4)
    g.advect_device_bounded(D - 1, df.data_ptr(), 1, -1.9, 1.4)
    gr = g.graph_end()
    gr.launch()
    graph_out = g.get_coeffs()
    g.set_coeffs(c)
    g.advect_device_bounded(D - 1, df.data_ptr(), 1, -1.9, 1.4)
    g.advect_device_bounded(D - 1, df.data_ptr(), 1, -1.9, 1.4)
    assert graph_out.tobytes() == g.get_coeffs().tobytes()
    gr.destroy()
    g.destroy()


def test_bound_violation_and_unbounded_capture_are_errors():
    """An entry outside the caller's bound leaves its lines unchanged and raises the sticky
    EINVAL at the next blocking call; an unbounded device-field sweep along the sharded dim
    cannot be captured (its halo would be sized on the host)."""
    from paper_1603_07008_b200 import SldgError
    dims, k = [32, 6, 20], 2
    K = k ** 3
    c = sldg_inputs.random_coeffs(dims, k, 7)
    g = _Grid(dims, k, precision="mixed", force_halo=True, max_halo=2)
    f = np.full(dims[0], 0.5)
    f[5] = 3.7  # outside [-1, 1]
    df = torch.tensor(f, dtype=torch.float64, device="cuda")
    g.set_coeffs(c)
    before = g.get_coeffs()
    g.advect_device_bounded(2, df.data_ptr(), 1, -1.0, 1.0)
    with pytest.raises(SldgError):
        g.mass()
    after = g.get_coeffs().reshape(dims[2], dims[1], dims[0], K)
    b4 = before.reshape(dims[2], dims[1], dims[0], K)
    assert after[:, :, 5].tobytes() == b4[:, :, 5].tobytes()  # the violating lines are unchanged
    ref = oracle.advect(oracle_input(c, K, "mixed"), dims, k, 2, field=np.where(f > 1, 0.0, f), field_mask=1,
                        n_double=1).reshape(dims[2], dims[1], dims[0], K)
    assert_parity(np.delete(after, 5, axis=2).reshape(-1, K), np.delete(ref, 5, axis=2).reshape(-1, K), K, "mixed")
    with pytest.raises(SldgError):
        g.advect_device_bounded(2, df.data_ptr(), 1, 1.0, -1.0)  # nu_min > nu_max
    g.graph_begin()
    with pytest.raises(SldgError):
        g.advect_device(2, df.data_ptr(), 1)
    gr = g.graph_end()
    gr.destroy()
    g.destroy()


def test_timeline_records_halo_and_interior():
    """Profile-mode timeline of a sharded sweep (NCCL self-exchange on one GPU): one halo
    exchange interval on the comm stream and the interior + boundary sweep launches; the
    interior launch is enqueued before the boundary ones and the boundary ones start after the
    exchange ends (they wait on its event)."""
    dims, k = [128, 64, 16], 3
    g = _Grid(dims, k, precision="mixed", force_halo=True, max_halo=2, nccl_self=True)
    g.fill_random(3)
    df = torch.tensor(np.full(dims[0] * dims[1], 0.3), dtype=torch.float64, device="cuda")
    g.profile(True)
    g.timeline(reset=True)
    g.advect_device_bounded(2, df.data_ptr(), 3, 0.3, 0.3)
    tl = g.timeline()
    g.profile(False)
    kinds = [t[0] for t in tl]
    assert kinds.count(-1) == 1 and kinds.count(2) >= 2, tl
    halo = next(t for t in tl if t[0] == -1)
    sweeps = [t for t in tl if t[0] == 2]
    assert all(t[2] >= t[1] for t in tl)
    assert sweeps[-1][1] >= halo[2] - 1e-3  # boundary layers after the exchange
    g.destroy()


# ------------------------------------------------------------------------------ CUDA graphs
def test_graph_replay_matches_eager():
    """A captured split step (device CFL fields, a constant shift, a Gauss-node sweep) replayed
    from a CUDA graph gives bit-identical results to the same calls made eagerly."""
    from paper_1603_07008_b200 import Grid, SldgError
    from oracle import vnodes
    dims, k = [64, 32, 16, 12], 2
    kinds = ["x", "x", "v", "v"]
    lo, hi = [0, 0, -6, -6], [4 * np.pi, 4 * np.pi, 6, 6]
    sweeps = sldg_inputs.vlasov_fields(dims, kinds, lo, hi, eps=0.3)
    dev = [torch.tensor(f, dtype=torch.float64, device="cuda") for _, f, _ in sweeps]
    nodal = torch.tensor(vnodes.nodal_velocity_field(16, -6.0, 6.0, k, 0.8), dtype=torch.float64, device="cuda")

    def step(g):
        for (d, _, m), t in zip(sweeps, dev):
            g.advect_device(d, t.data_ptr(), m)
        g.advect(1, shift=0.37)
        g.advect_vnodes_device(0, 2, nodal.data_ptr())  # 6 sweeps: the buffer parity is restored

    ga, gb = Grid(dims, k, lo=lo, hi=hi), Grid(dims, k, lo=lo, hi=hi)
    for g in (ga, gb):
        g.fill_random(3)
        step(g)  # warm-up: weight buffers and tensor maps exist before the capture
    gb.graph_begin()
    with pytest.raises(SldgError):  # host fields cannot be captured
        gb.advect(0, field=np.ones(16), field_mask=4)
    step(gb)
    graph = gb.graph_end()
    for _ in range(3):
        step(ga)
        graph.launch()
    assert ga.get_coeffs().tobytes() == gb.get_coeffs().tobytes()
    assert ga.mass() == gb.mass()
    graph.destroy()
    # an odd number of sweeps flips the buffer: the second launch is refused
    gb.graph_begin()
    gb.advect(1, shift=0.37)
    odd = gb.graph_end()
    odd.launch()
    with pytest.raises(SldgError):
        odd.launch()
    odd.destroy()
    ga.destroy()
    gb.destroy()
    # sharded (forced-halo) grids capture too; an unbounded device field along the layer dim is
    # refused inside the capture (test_bound_violation_and_unbounded_capture_are_errors)
    gh = Grid([16, 8], 2, force_halo=True, max_halo=2)
    gh.graph_begin()
    gh.advect(1, shift=0.5)
    gh.advect(1, shift=0.5)
    gh.graph_end().destroy()
    gh.destroy()


# ------------------------------------------------------------------------------ randomized shapes
def _random_case(rng):
    D = int(rng.integers(1, 5))
    k = int(rng.integers(1, 5))
    dims = []
    for _ in range(D):
        n = int(rng.choice([1, 2, 3, 4, 5, 7, 8, 12, 16, 20, 24, 32, 36, 64, 68, 96, 128, 132, 256]))
        dims.append(n)
    while np.prod(dims) * k ** D > 2_000_000:
        i = int(np.argmax(dims))
        dims[i] = max(1, dims[i] // 2)
    prec = ["mixed", "fp64"][int(rng.integers(0, 2))]
    return dims, k, prec


@pytest.mark.parametrize("seed", list(range(48)))
def test_randomized_shapes_match_oracle(seed):
    """Random grids (1-4D, extents including 1, odd sizes, multiples of 4 for the TMA paths,
    partial tiles), random k, storage, sweep dim, constant or per-line / per-lane shift fields
    with spans up to several cells: every sweep kernel and plan branch against the oracle."""
    rng = np.random.default_rng(1000 + seed)
    dims, k, precision = _random_case(rng)
    D, K = len(dims), k ** len(dims)
    c = sldg_inputs.random_coeffs(dims, k, seed)
    ref_in = oracle_input(c, K, precision)
    g = _Grid(dims, k, precision=precision)
    for _ in range(3):
        dim = int(rng.integers(0, D))
        others = [e for e in range(D) if e != dim]
        if others and rng.random() < 0.6:
            mask = 0
            for e in others:
                if rng.random() < 0.6:
                    mask |= 1 << e
            if mask == 0:
                mask = 1 << others[0]
            nf = int(np.prod([dims[e] for e in range(D) if mask >> e & 1]))
            field = rng.uniform(-3.5, 3.5, nf) * (1 + dims[dim] * (rng.random() < 0.3))
            ints = rng.random(nf) < 0.1  # some integer shifts: exact-copy lines
            field[ints] = np.round(field[ints])
            shift = 0.0
        else:
            mask, field = 0, None
            shift = float(rng.uniform(-2.5, 2.5) * (1 + dims[dim]))
        g.set_coeffs(c)
        g.advect(dim, shift=shift, field=field, field_mask=mask)
        ref = oracle.advect(ref_in, dims, k, dim, shift=shift, field=field, field_mask=mask,
                            n_double=n_double(precision, K))
        assert_parity(g.get_coeffs(), ref, K, precision, f"seed={seed} dims={dims} k={k} dim={dim} "
                      f"kernel={g.sweep_kernel(dim)}", ref_in, dim, k)
    g.destroy()


@pytest.mark.parametrize("seed", list(range(32)))
def test_randomized_sharded_paths_match_oracle(seed):
    """Random 2-5D grids on the single-GPU stand-ins of the multi-GPU paths: forced halo layers
    (random max_halo), forced transposes, NCCL self-transfers; sweeps along the layer dim with
    shifts that fit the halo, exceed it (automatic transpose), or are per-line fields over the
    slab dim; plus a sweep along another dim."""
    rng = np.random.default_rng(5000 + seed)
    D = int(rng.integers(2, 6))
    k = int(rng.integers(1, 5))
    dims = [int(rng.choice([1, 2, 3, 4, 5, 8, 12, 16, 32, 64])) for _ in range(D)]
    dims[-1] = int(rng.integers(2, 20))
    while np.prod(dims) * k ** D > 1_000_000:
        i = int(np.argmax(dims[:-1]))
        dims[i] = max(1, dims[i] // 2)
    precision = ["mixed", "fp64"][int(rng.integers(0, 2))]
    mode = int(rng.integers(0, 3))
    kw = dict(max_halo=int(rng.integers(1, 4)), nccl_self=bool(rng.random() < 0.4))
    if mode == 0:
        kw["force_halo"] = True
    elif mode == 1:
        kw["force_transpose"] = True
    else:
        kw["force_halo"] = True
        kw["force_transpose"] = True
    K = k ** D
    c = sldg_inputs.random_coeffs(dims, k, seed)
    ref_in = oracle_input(c, K, precision)
    g = _Grid(dims, k, precision=precision, **kw)
    n = dims[-1]
    cases = [(D - 1, float(rng.uniform(-1.5, 1.5)), None, 0),
             (D - 1, float(rng.uniform(-3 * n, 3 * n)), None, 0)]
    mask = (1 << (D - 2)) | (1 if rng.random() < 0.5 else 0)
    nf = int(np.prod([dims[e] for e in range(D) if mask >> e & 1]))
    cases.append((D - 1, 0.0, rng.uniform(-2.2 * n, 2.2 * n, nf), mask))
    cases.append((int(rng.integers(0, D - 1)), float(rng.uniform(-5, 5)), None, 0))
    for dim, shift, field, fm in cases:
        g.set_coeffs(c)
        g.advect(dim, shift=shift, field=field, field_mask=fm)
        ref = oracle.advect(ref_in, dims, k, dim, shift=shift, field=field, field_mask=fm,
                            n_double=n_double(precision, K))
        assert_parity(g.get_coeffs(), ref, K, precision,
                      f"seed={seed} dims={dims} k={k} dim={dim} nu={shift} kw={kw}", ref_in, dim, k)
    g.destroy()


@pytest.mark.parametrize("seed", list(range(16)))
def test_randomized_medium_grids_match_oracle(seed):
    """Random 2-4D grids of up to ~8M DoF (TMA plan branches: W selection and the W = 64 rule,
    1- and 2-CTA instances, partial d = 0 tiles, R lines per tile, sub-chunk splits) -- every dim
    swept once against the oracle."""
    rng = np.random.default_rng(9000 + seed)
    D = int(rng.integers(2, 5))
    k = int(rng.integers(1, 5))
    dims = [int(rng.choice([4, 8, 12, 16, 20, 24, 28, 32, 36, 40, 48, 60, 64, 100, 128, 132, 192, 256, 260,
                            512, 1024, 1028, 2048]))
            for _ in range(D)]
    while np.prod(dims) * k ** D > 8_000_000:
        i = int(np.argmax(dims))
        dims[i] = max(4, (dims[i] // 2) // 4 * 4)
    precision = ["mixed", "fp64"][int(rng.integers(0, 2))]
    K = k ** D
    c = sldg_inputs.random_coeffs(dims, k, seed)
    ref_in = oracle_input(c, K, precision)
    g = _Grid(dims, k, precision=precision)
    for dim in range(D):
        others = [e for e in range(D) if e != dim]
        mask = 0
        for e in others:
            if rng.random() < 0.5:
                mask |= 1 << e
        if mask:
            nf = int(np.prod([dims[e] for e in range(D) if mask >> e & 1]))
            field, shift = rng.uniform(-4.5, 4.5, nf), 0.0
        else:
            field, shift = None, float(rng.uniform(-40, 40))
        g.set_coeffs(c)
        g.advect(dim, shift=shift, field=field, field_mask=mask)
        ref = oracle.advect(ref_in, dims, k, dim, shift=shift, field=field, field_mask=mask,
                            n_double=n_double(precision, K))
        assert_parity(g.get_coeffs(), ref, K, precision,
                      f"seed={seed} dims={dims} k={k} dim={dim} kernel={g.sweep_kernel(dim)}", ref_in, dim, k)
    g.destroy()


@pytest.mark.parametrize("precision", ["mixed", "fp64"])
@pytest.mark.parametrize("dims,k", [([64, 20], 5), ([48, 6, 5], 6), ([16, 4, 3], 7), ([12, 4, 3], 8),
                                    ([4096, 6], 5), ([20, 6, 4, 3], 5), ([1024, 9], 6)])
def test_high_order_d0_tma_matches_oracle(dims, k, precision):
    """k = 5..8 on d = 0: the TMA kernel reading the line weights from the record in shared memory
    (a copy in every stage of the tile); constant shifts, per-line fields (one record per tile
    and one per line) and copy lines.  A 4096-cell fp64 k = 5 line does not fit two whole-line
    stages: the windowed kernel (sweep_d0_win) runs it."""
    D, K = len(dims), k ** len(dims)
    rng = np.random.default_rng(77 + k)
    c = sldg_inputs.random_coeffs(dims, k, 5150 + k)
    ref_in = oracle_input(c, K, precision)
    g = _Grid(dims, k, precision=precision)
    want = "sweep_d0_win" if (dims[0] == 4096 and precision == "fp64") else "sweep_d0_tma"
    assert g.sweep_kernel(0) == want, g.sweep_kernel(0)
    cases = [(3.37, None, 0), (-0.41 - dims[0], None, 0)]
    if D >= 2:
        mask = (1 << (D - 1)) | (2 if D >= 3 else 0)
        nf = int(np.prod([dims[e] for e in range(D) if mask >> e & 1]))
        field = rng.uniform(-2.5 * dims[0], 2.5 * dims[0], nf)
        field[::5] = np.round(field[::5])
        cases.append((0.0, field, mask))
    for shift, field, mask in cases:
        g.set_coeffs(c)
        g.advect(0, shift=shift, field=field, field_mask=mask)
        ref = oracle.advect(ref_in, dims, k, 0, shift=shift, field=field, field_mask=mask,
                            n_double=n_double(precision, K))
        assert_parity(g.get_coeffs(), ref, K, precision, f"dims={dims} k={k} nu={shift} mask={mask}", ref_in, 0, k)
    g.destroy()


@pytest.mark.parametrize("precision", ["mixed", "fp64"])
@pytest.mark.parametrize("dims,k", [([64, 20], 5), ([32, 12, 6], 6), ([128, 9], 5), ([64, 8, 4, 3], 5),
                                    ([256, 40], 6)])
def test_high_order_strided_tma_matches_oracle(dims, k, precision):
    """k = 5, 6 on strided sweeps: the TMA kernel with two threads per column, each owning half of
    the output slots and their rows of A, B; constant shifts of both signs, per-lane fields over
    dim 0 (spans of several cells) and copy lines."""
    D, K = len(dims), k ** len(dims)
    rng = np.random.default_rng(91 + k + D)
    c = sldg_inputs.random_coeffs(dims, k, 6150 + k)
    ref_in = oracle_input(c, K, precision)
    g = _Grid(dims, k, precision=precision)
    for dim in range(1, D):
        assert g.sweep_kernel(dim) == "sweep_strided_tma", (dim, g.sweep_kernel(dim))
        f0 = rng.uniform(-3.2, 3.2, dims[0])
        f0[::6] = np.round(f0[::6])
        cases = [(2.37, None, 0), (-0.63 - dims[dim], None, 0), (0.0, f0, 1)]
        for shift, field, mask in cases:
            g.set_coeffs(c)
            g.advect(dim, shift=shift, field=field, field_mask=mask)
            ref = oracle.advect(ref_in, dims, k, dim, shift=shift, field=field, field_mask=mask,
                                n_double=n_double(precision, K))
            assert_parity(g.get_coeffs(), ref, K, precision, f"dims={dims} k={k} dim={dim} nu={shift} mask={mask}",
                          ref_in, dim, k)
    g.destroy()


@pytest.mark.parametrize("precision", ["mixed", "fp64"])
def test_host_field_not_retained(precision):
    """sldg_advect copies a host shift field before it returns (the library never
    retains host pointers): overwriting a PINNED host buffer right after the call -- before the
    GPU has run the sweep -- must not change the result; several calls back to back cycle the
    staging ring."""
    import torch
    dims, k = [256, 96], 3
    K = k ** 2
    c = sldg_inputs.random_coeffs(dims, k, 4242)
    ref_in = oracle_input(c, K, precision)
    rng = np.random.default_rng(17)
    fields = [rng.uniform(-5.0, 5.0, dims[0]) for _ in range(7)]
    g = _Grid(dims, k, precision=precision)
    g.set_coeffs(c)
    buf = torch.empty(dims[0], dtype=torch.float64, pin_memory=True)
    hv = buf.numpy()
    for f in fields:  # v-sweeps with per-lane fields, host buffer clobbered after every call
        hv[:] = f
        g.advect(1, field=hv, field_mask=1)
        hv[:] = 1e6  # a bogus shift: would fail parity (and wrap) if the DMA read it later
    got = g.get_coeffs()
    ref = ref_in
    for f in fields:
        ref = oracle.round_layout(oracle.advect(ref, dims, k, 1, field=f, field_mask=1, n_double=n_double(precision, K)),
                                  K, n_double(precision, K))
    assert_parity(got, ref, K, precision, "host field clobbered after sldg_advect", ref_in, 1, k)
    g.destroy()


@pytest.mark.parametrize("dims,k,precision", [([4096, 3], 4, "fp64"), ([4100, 2], 4, "fp64"), ([4100, 3], 3, "mixed"), ([4096, 2, 2], 6, "fp64"),
                                              ([2048, 3], 8, "fp64"), ([4096, 2], 6, "mixed"), ([4096, 2], 7, "mixed"), ([4096, 2], 8, "mixed"),
                                              ([8192, 2], 4, "fp64")])
def test_windowed_d0_matches_oracle(dims, k, precision):
    """d = 0 lines too long for two whole-line stages (sweep_d0_win): tiles are windows of cw
    targets whose cw + 1 sources start at (a - i* - 1) mod n0, loaded as one or two
    (periodic wrap) bulk copies per plane.  Shifts that put the window across the wrap at every
    offset mod 4, negative and multi-line shifts, integer shifts (copy lines) and per-line
    fields; a ragged last window (n0 = 4100)."""
    D, K = len(dims), k ** len(dims)
    rng = np.random.default_rng(31 * k + D)
    c = sldg_inputs.random_coeffs(dims, k, 7100 + k)
    ref_in = oracle_input(c, K, precision)
    g = _Grid(dims, k, precision=precision)
    assert g.sweep_kernel(0) == "sweep_d0_win", g.sweep_kernel(0)
    n0 = dims[0]
    cases = [(0.37, None, 0), (1.5, None, 0), (2.61, None, 0), (3.99, None, 0), (-0.41, None, 0),
             (-n0 / 2 - 0.3, None, 0), (2.5 * n0 + 0.77, None, 0), (5.0, None, 0), (-3.0, None, 0)]
    mask = (1 << (D - 1)) | (2 if D >= 3 else 0)
    nf = int(np.prod([dims[e] for e in range(D) if mask >> e & 1]))
    field = rng.uniform(-2.5 * n0, 2.5 * n0, nf)
    field[::3] = np.round(field[::3])
    cases.append((0.0, field, mask))
    for shift, field, mask in cases:
        g.set_coeffs(c)
        g.advect(0, shift=shift, field=field, field_mask=mask)
        got = g.get_coeffs()
        ref = oracle.advect(ref_in, dims, k, 0, shift=shift, field=field, field_mask=mask,
                            n_double=n_double(precision, K))
        if field is None and shift == round(shift):
            assert got.tobytes() == ref.tobytes()  # integer shift: an exact rotation
        assert_parity(got, ref, K, precision, f"dims={dims} k={k} nu={shift} mask={mask}", ref_in, 0, k)
    g.destroy()


@pytest.mark.parametrize("precision", ["fp64", "mixed"])
def test_windowed_d0_per_line_fields_and_halo_layout(precision):
    """sweep_d0_win on a 3D grid: per-line fields over dims 1 and 2 (the producer derives each
    line's field entry from its line and layer index), and the same sweeps on a grid with the
    halo layout (pad layers shift every layer's address) -- both against the oracle."""
    dims, k = ([4096, 3, 4], 4) if precision == "fp64" else ([4096, 2, 3], 7)
    D, K = len(dims), k ** len(dims)
    c = sldg_inputs.random_coeffs(dims, k, 2718)
    ref_in = oracle_input(c, K, precision)
    rng = np.random.default_rng(5)
    for kw in [{}, {"force_halo": True, "max_halo": 2}]:
        g = _Grid(dims, k, precision=precision, **kw)
        assert g.sweep_kernel(0) == "sweep_d0_win", g.sweep_kernel(0)
        for mask in [2, 4, 6]:
            nf = int(np.prod([dims[e] for e in range(D) if mask >> e & 1]))
            field = rng.uniform(-1.5 * dims[0], 1.5 * dims[0], nf)
            g.set_coeffs(c)
            g.advect(0, field=field, field_mask=mask)
            ref = oracle.advect(ref_in, dims, k, 0, field=field, field_mask=mask, n_double=n_double(precision, K))
            assert_parity(g.get_coeffs(), ref, K, precision, f"win dims={dims} mask={mask} {kw}", ref_in, 0, k)
        g.destroy()
