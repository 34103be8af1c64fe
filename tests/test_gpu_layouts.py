"""GPU parity of the general precision layouts (the paper's "# double" d, P:391-456 SS III-A) on
1D lines (the paper's own workload, Tables II-VI): slots q < d in fp64, the rest fp32.  Both 1D
kernels are covered: the TMA line kernel (N % 4 == 0, N >= 1024) and the simple kernel."""
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


def _parity(got, ref, k, nd, src):
    for q in range(k):
        m = np.max(np.abs(ref[:, q]))
        d = np.max(np.abs(got[:, q] - ref[:, q]))
        if q < nd:  # fp64 slot: relative to the planes it is computed from (R8)
            tol = 1e-13 * max(m, np.max(np.abs(src)))
        else:
            tol = 8.0 * float(np.spacing(np.float32(m)))
        assert d <= tol, (q, d, tol)


@pytest.mark.parametrize("N", [64, 100, 4096, 5000, 5001, 1 << 16])
@pytest.mark.parametrize("k", [1, 2, 3, 4])
def test_line_all_layouts(N, k):
    c = sldg_inputs.random_coeffs([N], k, 1603)
    for nd in range(0, k + 1):
        g = _Grid([N], k, precision=nd)
        if N >= 1024 and N % 4 == 0:
            assert g.sweep_kernel(0) == "line_tma_kernel"
        else:
            assert g.sweep_kernel(0) == "line_simple_kernel"
        src = oracle.round_layout(c, k, nd)
        for nu in [0.37, -2.61 - N, 1234.5, 3.0]:
            g.set_coeffs(c)
            g.advect(0, shift=nu)
            got = g.get_coeffs()
            ref = oracle.advect(src, [N], k, 0, shift=nu, n_double=nd)
            if nu == 3.0:
                assert got.tobytes() == ref.tobytes()  # integer shift: exact rotation
            else:
                _parity(got, ref, k, nd, src)
        assert g.memory_bytes() == N * (8 * nd + 4 * (k - nd))  # S:163-169 generalised
        g.destroy()


@pytest.mark.parametrize("k", [2, 4])
def test_table_II_mechanism_on_gpu(k):
    """P:396-431 (Table II): 1e4 steps, N = 256, nu = 2.25, smooth IC.  d >= 1 conserves mass
    to fp64 accuracy (paper 4.4e-15 .. 1.6e-14); d = 0 (pure fp32) does not (paper 2.6e-6,
    1.3e-5); the mixed-vs-fp64 L2 distance is ~1e-10 (paper 8.98e-10 / 3.55e-10)."""
    N, steps, nu = 256, 10000, 2.25
    c0 = sldg_inputs.project_1d(lambda x: 1.0 + 0.5 * np.sin(2 * np.pi * x), N, 0.0, 1.0, k, 12)
    out = {}
    for nd in [k, 1, 0]:
        g = _Grid([N], k, precision=nd)
        g.set_coeffs(c0)
        m0 = g.mass()
        for _ in range(steps):
            g.advect(0, shift=nu)
        out[nd] = (g.get_coeffs(), abs(g.mass() - m0) / m0)
        g.destroy()
    assert out[k][1] <= 1e-13 and out[1][1] <= 1e-13
    assert out[0][1] >= 1e-9
    l2 = oracle.l2_norm_diff(out[1][0], out[k][0], 1.0 / N, k)
    assert 1e-13 < l2 < 1e-6
    assert oracle.l2_norm_diff(out[0][0], out[k][0], 1.0 / N, k) > 10 * l2


def test_weight_reuse_sequence():
    """The library skips the weight build when a constant-shift sweep repeats the previous one's
    (shift, extent).  A mixed sequence of repeated / changed shifts, dims, extents and fields must
    still match the oracle step by step."""
    from paper_1603_07008_b200 import Grid
    k = 3
    c = sldg_inputs.random_coeffs([16, 16, 12], k, 7)
    g = Grid([16, 16, 12], k)
    g.set_coeffs(c)
    ref = oracle.round_layout(c, k, 1)
    f2 = np.linspace(-3.3, 2.7, 16 * 16)
    seq = [(0, 0.3, None, 0), (0, 0.3, None, 0), (1, 0.3, None, 0), (2, 0.3, None, 0), (2, 0.3, None, 0),
           (2, 0.0, None, 0), (2, 0.0, None, 0), (0, 0.0, None, 0), (2, 0.0, f2, 0b011), (2, 0.0, None, 0),
           (1, -1.75, None, 0), (0, -1.75, None, 0), (0, -1.75, None, 0)]
    for dim, nu, fld, mask in seq:
        if fld is None:
            g.advect(dim, shift=nu)
            ref = oracle.advect(ref, [16, 16, 12], k, dim, shift=nu, n_double=1)
        else:
            g.advect(dim, field=fld, field_mask=mask)
            ref = oracle.advect(ref, [16, 16, 12], k, dim, field=fld, field_mask=mask, n_double=1)
        got = g.get_coeffs()
        K = k ** 3
        d0 = np.max(np.abs(got[:, 0] - ref[:, 0]))
        assert d0 <= 1e-13 * np.max(np.abs(ref[:, 0])), (dim, nu)
        for q in range(1, K):
            m = np.max(np.abs(ref[:, q]))
            assert np.max(np.abs(got[:, q] - ref[:, q])) <= 8.0 * float(np.spacing(np.float32(m))), (dim, nu, q)
        ref = got.copy()  # continue from the GPU state so that only this step's error is measured
    g.destroy()


def test_general_layout_rejected_in_multid():
    from paper_1603_07008_b200 import SldgError
    with pytest.raises(SldgError):
        _Grid([8, 8], 2, precision=2)  # only d = 1 or d = k^D in multi-D
    g = _Grid([8, 8], 2, precision=1)  # == mixed
    assert g.memory_bytes() == 64 * (8 + 4 * 3)
    g.destroy()
    g = _Grid([8, 8], 2, precision=4)  # == fp64
    assert g.memory_bytes() == 64 * 8 * 4
    g.destroy()


@pytest.mark.parametrize("seed", list(range(16)))
def test_randomized_lines_all_layouts(seed):
    """Random 1D lines (N from 1 to 70000, with and without N % 4 == 0), random k and number of
    fp64 slots, random shifts: the line kernels against the oracle."""
    rng = np.random.default_rng(300 + seed)
    N = int(rng.choice([1, 2, 3, 5, 17, 63, 1024, 1028, 1030, 4099, 8192, 65536, 69996]))
    k = int(rng.integers(1, 5))
    nd = int(rng.integers(0, k + 1))
    c = sldg_inputs.random_coeffs([N], k, seed)
    src = oracle.round_layout(c, k, nd)
    g = _Grid([N], k, precision=nd)
    for nu in [float(rng.uniform(-3 * N, 3 * N)), float(rng.uniform(-1, 1)), float(rng.integers(-N, N))]:
        g.set_coeffs(c)
        g.advect(0, shift=nu)
        got = g.get_coeffs()
        ref = oracle.advect(src, [N], k, 0, shift=nu, n_double=nd)
        if nu == round(nu):
            assert got.tobytes() == ref.tobytes()
        else:
            _parity(got, ref, k, nd, src)
    g.destroy()
