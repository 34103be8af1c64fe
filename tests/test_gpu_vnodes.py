"""GPU parity of the Gauss-node velocity sweep (sldg_advect_vnodes, NEXT-3) against
oracle/vnodes.py, and the free-streaming accuracy the nodal treatment buys."""
import numpy as np
import pytest

import oracle
import sldg_inputs
from oracle import vnodes

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    torch.cuda.set_device(0)
    yield


def _parity(got, ref, K, precision, src, tag):
    for q in range(K):
        m = np.max(np.abs(ref[:, q]))
        d = np.max(np.abs(got[:, q] - ref[:, q]))
        if precision == "fp64" or q == 0:
            tol = 1e-13 * max(m, np.max(np.abs(src)))
        else:
            tol = 8.0 * float(np.spacing(np.float32(m)))
        assert d <= tol, f"{tag} slot {q}: {d:.3e} > {tol:.3e}"


CASES = [
    ([16, 12], 3, 0, 1),          # d = 0 (contiguous), v = layer dim
    ([12, 10], 2, 1, 0),          # sweep along the layer dim, v = dim 0
    ([8, 6, 10], 3, 0, 2),
    ([6, 9, 8], 4, 1, 2),         # strided inner sweep
    ([8, 5, 6, 7], 2, 0, 2),      # 4D: x1 with v1
    ([5, 8, 4, 6], 3, 1, 3),      # 4D: x2 with v2 (the layer dim)
]


@pytest.mark.parametrize("precision", ["mixed", "fp64"])
@pytest.mark.parametrize("dims,k,dim,vdim", CASES)
def test_vnodes_parity(dims, k, dim, vdim, precision):
    from paper_1603_07008_b200 import Grid
    D, K = len(dims), k ** len(dims)
    nd = 1 if precision == "mixed" else K
    c = sldg_inputs.random_coeffs(dims, k, 21)
    src = oracle.round_layout(c, K, nd)
    g = Grid(dims, k, precision=precision)
    nv = dims[vdim]
    # wide velocity range (shifts of several cells of both signs) and a cell width in nu large
    # enough that the nodes of some v-cells straddle an integer (three source offsets)
    for scale in [0.37, 1.1]:
        nodal = vnodes.nodal_velocity_field(nv, -3.0, 3.0, k, scale * dims[dim] / 4)
        g.set_coeffs(c)
        g.advect_vnodes(dim, vdim, nodal)
        ref = vnodes.advect_vnodes(src, dims, k, dim, vdim, nodal, n_double=nd)
        _parity(g.get_coeffs(), ref, K, precision, src, f"dims={dims} dim={dim} vdim={vdim} scale={scale}")
    g.destroy()


# shapes where every CTA's 512 cells share their v-cell: the CPT = 2 kernel (vnode_sweep_multi)
MULTI_CASES = [
    ([64, 8, 16], 3, 0, 2),       # x1 (d = 0) with v = the layer dim
    ([32, 16, 8, 4], 3, 1, 2),    # x2 with v1 (S_e = 512)
    ([512, 6], 3, 0, 1),          # 2D C3-shaped
    ([64, 16, 4, 5], 2, 0, 2),    # 4D k = 2
    ([128, 4, 8], 1, 0, 2),       # k = 1
]


@pytest.mark.parametrize("precision", ["mixed", "fp64"])
@pytest.mark.parametrize("dims,k,dim,vdim", MULTI_CASES)
def test_vnodes_multi_cell_kernel(dims, k, dim, vdim, precision, monkeypatch):
    """Two cells per thread (vnode_sweep_multi): the same operation order per output as the
    one-cell kernel, so bit-identical to it (SLDG_VN_MULTI=0), and within the parity bar of the
    oracle; shifts of several cells of both signs with 2- and 3-offset v-cells."""
    from paper_1603_07008_b200 import Grid
    D, K = len(dims), k ** len(dims)
    nd = 1 if precision == "mixed" else K
    c = sldg_inputs.random_coeffs(dims, k, 33)
    src = oracle.round_layout(c, K, nd)
    g = Grid(dims, k, precision=precision)
    nv = dims[vdim]
    # a v-cell spans 0.4 and 2.0 cells of shift (2- and 3-offset cells, within kVnMaxOfs)
    for width in [0.4, 2.0]:
        nodal = vnodes.nodal_velocity_field(nv, -3.0, 3.0, k, width * nv / 6.0)
        outs = []
        for multi in ["1", "0"]:
            monkeypatch.setenv("SLDG_VN_MULTI", multi)
            g.set_coeffs(c)
            g.advect_vnodes(dim, vdim, nodal)
            outs.append(g.get_coeffs())
        assert outs[0].tobytes() == outs[1].tobytes(), f"multi-cell kernel differs: dims={dims} width={width}"
        ref = vnodes.advect_vnodes(src, dims, k, dim, vdim, nodal, n_double=nd)
        _parity(outs[0], ref, K, precision, src, f"multi dims={dims} dim={dim} vdim={vdim} width={width}")
    g.destroy()


def test_vnodes_mass_and_bad_field():
    from paper_1603_07008_b200 import Grid, SldgError
    dims, k = [32, 16], 3
    g = Grid(dims, k, lo=[0, -4], hi=[1, 4])
    g.fill_random(5)
    m0 = g.mass()
    for _ in range(50):
        g.advect_vnodes(0, 1, vnodes.nodal_velocity_field(16, -4.0, 4.0, k, 3.1))
    assert abs(g.mass() - m0) <= 1e-13 * abs(m0)
    bad = vnodes.nodal_velocity_field(16, -4.0, 4.0, k, 1.0)
    bad[7] = np.nan
    with pytest.raises(SldgError):
        g.advect_vnodes(0, 1, bad)
    with pytest.raises(SldgError):
        g.advect_vnodes(1, 1, bad)
    d = torch.tensor(bad, dtype=torch.float64, device="cuda")
    g.advect_vnodes_device(0, 1, d.data_ptr())
    with pytest.raises(SldgError):
        g.mass()  # sticky device error from the non-finite node
    g.destroy()


def test_vnodes_free_streaming_beats_cell_centre():
    """The GPU path reproduces the oracle's accuracy gain (tests/test_vnodes_oracle.py): one step
    of free streaming on a 2D grid against the projected exact solution."""
    from paper_1603_07008_b200 import Grid
    from tests import test_vnodes_oracle as T
    k, nx, nv, t = 3, 48, 16, 0.3
    lox, hix, lov, hiv = 0.0, 1.0, -2.0, 2.0
    f0 = lambda x, v: np.sin(2 * np.pi * x) * np.exp(-v * v)  # noqa: E731
    c0 = T._project2d(f0, nx, nv, lox, hix, lov, hiv, k)
    ce = T._project2d(lambda x, v: f0(x - v * t, v), nx, nv, lox, hix, lov, hiv, k)
    g = Grid([nx, nv], k, lo=[lox, lov], hi=[hix, hiv], precision="fp64")
    scale = t / ((hix - lox) / nx)
    g.set_coeffs(c0)
    g.advect_vnodes(0, 1, vnodes.nodal_velocity_field(nv, lov, hiv, k, scale))
    err_node = np.max(np.abs(g.get_coeffs() - ce))
    vc = lov + (np.arange(nv) + 0.5) * (hiv - lov) / nv
    g.set_coeffs(c0)
    g.advect(0, field=vc * scale, field_mask=2)
    err_cent = np.max(np.abs(g.get_coeffs() - ce))
    assert err_node < 1e-3 * err_cent * 10 and err_node < 2e-4, (err_node, err_cent)
    g.destroy()


@pytest.mark.parametrize("seed", list(range(12)))
def test_randomized_vnodes(seed):
    """Random grids, k, (dim, vdim) pairs and node-velocity fields against the oracle."""
    from paper_1603_07008_b200 import Grid
    rng = np.random.default_rng(700 + seed)
    D = int(rng.integers(2, 5))
    k = int(rng.integers(1, 5))
    dims = [int(rng.choice([1, 2, 3, 4, 6, 8, 12, 16, 33, 64])) for _ in range(D)]
    while np.prod(dims) * k ** D > 400_000:
        i = int(np.argmax(dims))
        dims[i] = max(1, dims[i] // 2)
    dim, vdim = [int(x) for x in rng.choice(D, 2, replace=False)]
    precision = ["mixed", "fp64"][int(rng.integers(0, 2))]
    K = k ** D
    nd = 1 if (precision == "mixed" and K > 1) else K
    c = sldg_inputs.random_coeffs(dims, k, seed)
    src = oracle.round_layout(c, K, nd)
    g = Grid(dims, k, precision=precision)
    nv = dims[vdim]
    # node shifts within one v-cell span at most ~2.5 cells (the kernel takes up to 6 offsets)
    scale = min(float(rng.uniform(0.1, 1.2)) * dims[dim] / 4, 2.5 / (4.0 / nv))
    nodal = vnodes.nodal_velocity_field(nv, -2.0, 2.0, k, scale)
    g.set_coeffs(c)
    g.advect_vnodes(dim, vdim, nodal)
    ref = vnodes.advect_vnodes(src, dims, k, dim, vdim, nodal, n_double=nd)
    _parity(g.get_coeffs(), ref, K, "fp64" if nd == K else "mixed", src, f"seed={seed} dims={dims} k={k}")
    g.destroy()
