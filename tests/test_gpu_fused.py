"""The fused dim-0 + dim-1 sweep pair (sldg_advect_pair, NEXT-4 multi-sweep fusion)
against the two sweeps it replaces (bit for bit) and against the oracle's two sweeps (P:144-149
splitting of the P:259-272 update; tolerances of DESIGN R8 with the intermediate as the source)."""

import numpy as np
import pytest

import oracle
import sldg_inputs
from tests.test_gpu_parity import assert_parity, n_double

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


def _fused_used(g):
    return any(kind == -2 for kind, _, _ in g.timeline(reset=True))


CASES = [
    # dims, k, (shift0, mask0 over dims >= 2), (shift1, mask1)
    ([64, 12, 5], 2, (1.37, 0b100), (-2.6, 0b100)),
    ([128, 16, 3, 4], 3, (2.25, 0b100), (-0.41, 0b1000)),
    ([32, 40, 6], 3, (-5.5, 0), (33.75, 0b100)),
    ([256, 9, 4], 1, (0.7, 0b100), (1.3, 0)),
    ([128, 8, 2, 3], 2, (3.0, 0b1100), (-1.0, 0b1100)),   # integer parts of both: copy paths
    ([64, 64, 3, 2], 3, (0.37, 0b100), (0.0, 0b1000)),
]


def _fields(dims, rng, spec, integer_every=0):
    shift, mask = spec
    if mask == 0:
        return shift, None
    n = int(np.prod([dims[e] for e in range(len(dims)) if mask >> e & 1]))
    f = rng.uniform(-3.5, 3.5, n) + shift
    if integer_every:
        f[::integer_every] = np.round(f[::integer_every])
    return 0.0, f


@pytest.mark.parametrize("precision", ["mixed", "fp64"])
@pytest.mark.parametrize("case", range(len(CASES)))
def test_pair_is_two_sweeps_bit_for_bit_and_matches_oracle(case, precision):
    dims, k, sp0, sp1 = CASES[case]
    D, K = len(dims), k ** len(dims)
    rng = np.random.default_rng(case)
    sh0, f0 = _fields(dims, rng, sp0, integer_every=5)
    sh1, f1 = _fields(dims, rng, sp1, integer_every=3)
    m0, m1 = (sp0[1] if f0 is not None else 0), (sp1[1] if f1 is not None else 0)
    c = sldg_inputs.random_coeffs(dims, k, 77 + case)
    g = _Grid(dims, k, precision=precision)
    g.set_coeffs(c)
    g.profile(True)
    g.timeline(reset=True)
    g.advect_pair(sh0, f0, m0, sh1, f1, m1)
    fused = g.get_coeffs()
    assert _fused_used(g), "the pair did not take the fused kernel"
    g.profile(False)
    g.set_coeffs(c)
    g.advect(0, shift=sh0, field=f0, field_mask=m0)
    g.advect(1, shift=sh1, field=f1, field_mask=m1)
    two = g.get_coeffs()
    g.destroy()
    assert fused.tobytes() == two.tobytes()
    nd = n_double(precision, K)
    src = oracle.round_layout(c, K, nd)
    mid = oracle.advect(src, dims, k, 0, shift=sh0, field=f0, field_mask=m0, n_double=nd)
    ref = oracle.advect(mid, dims, k, 1, shift=sh1, field=f1, field_mask=m1, n_double=nd)
    assert_parity(fused, ref, K, precision, f"pair dims={dims} k={k}", mid, 1, k)


def test_pair_unfusable_falls_back_to_two_sweeps():
    """A dim-0 field that varies along dim 1 (the 2D x-sweep) is not fusable: same result."""
    dims, k = [64, 16, 4], 2
    rng = np.random.default_rng(3)
    f0 = rng.uniform(-2, 2, dims[1])
    c = sldg_inputs.random_coeffs(dims, k, 5)
    g = _Grid(dims, k)
    g.set_coeffs(c)
    g.profile(True)
    g.timeline(reset=True)
    g.advect_pair(0.0, f0, 0b10, 0.7, None, 0)
    assert not _fused_used(g)
    g.profile(False)
    a = g.get_coeffs()
    g.set_coeffs(c)
    g.advect(0, field=f0, field_mask=0b10)
    g.advect(1, shift=0.7)
    assert a.tobytes() == g.get_coeffs().tobytes()
    g.destroy()


@pytest.mark.parametrize("eps", [0.01, 0.5])
def test_pair_c5_full_size_sampled(eps):
    """C5 (128^4, k = 3, mixed) with the bench's x1 / x2 CFL fields: the fused pair and the two
    sweeps agree bit for bit on sampled cells (first and last cells, random ones)."""
    dims, k = [128, 128, 128, 128], 3
    kinds = ["x", "x", "v", "v"]
    lo, hi = [0.0, 0.0, -6.0, -6.0], [4 * np.pi, 4 * np.pi, 6.0, 6.0]
    sweeps = sldg_inputs.vlasov_fields(dims, kinds, lo, hi, eps=eps)
    (d0, f0, m0), (d1, f1, m1) = sweeps[0], sweeps[1]
    assert (d0, d1) == (0, 1)
    rng = np.random.default_rng(11)
    cells = np.concatenate([[0, int(np.prod(dims)) - 1], rng.integers(0, int(np.prod(dims)), 600)])
    g = _Grid(dims, k, lo=lo, hi=hi)
    g.fill_random(1603)
    g.profile(True)
    g.timeline(reset=True)
    g.advect_pair(0.0, f0, m0, 0.0, f1, m1)
    assert _fused_used(g)
    g.profile(False)
    a = np.concatenate([g.get_coeffs(int(x), 1) for x in cells])
    g.fill_random(1603)
    g.advect(0, field=f0, field_mask=m0)
    g.advect(1, field=f1, field_mask=m1)
    b = np.concatenate([g.get_coeffs(int(x), 1) for x in cells])
    g.destroy()
    assert a.tobytes() == b.tobytes()


def test_pair_device_fields_and_graph_capture():
    """sldg_advect_pair_device (fields in HBM) equals the host-field pair, and a captured step
    of two pairs replays bit-identically."""
    dims, k = [128, 16, 6, 5], 3
    rng = np.random.default_rng(9)
    f0 = rng.uniform(-2.5, 2.5, dims[2])
    f1 = rng.uniform(-1.5, 3.5, dims[3])
    d0 = torch.tensor(f0, dtype=torch.float64, device="cuda")
    d1 = torch.tensor(f1, dtype=torch.float64, device="cuda")
    c = sldg_inputs.random_coeffs(dims, k, 21)
    g = _Grid(dims, k)
    g.set_coeffs(c)
    g.advect_pair(0.0, f0, 0b100, 0.0, f1, 0b1000)
    host = g.get_coeffs()
    g.set_coeffs(c)
    g.advect_pair_device(d0.data_ptr(), 0b100, d1.data_ptr(), 0b1000)
    assert g.get_coeffs().tobytes() == host.tobytes()
    g.set_coeffs(c)
    g.graph_begin()
    g.advect_pair_device(d0.data_ptr(), 0b100, d1.data_ptr(), 0b1000)
    g.advect_pair_device(d0.data_ptr(), 0b100, d1.data_ptr(), 0b1000)
    gr = g.graph_end()
    gr.launch()
    replay = g.get_coeffs()
    g.set_coeffs(c)
    g.advect_pair_device(d0.data_ptr(), 0b100, d1.data_ptr(), 0b1000)
    g.advect_pair_device(d0.data_ptr(), 0b100, d1.data_ptr(), 0b1000)
    assert g.get_coeffs().tobytes() == replay.tobytes()
    gr.destroy()
    g.destroy()
