"""Peer-mapped halo layers (SLDG_DIST_PEER_HALO) on one GPU: with world = 1 the
rank is its own ring neighbour, so the pad layers are virtual-memory mappings of the grid's own
opposite edge layers, and a sweep along the sharded dim is ONE launch whose boundary tiles read
them in place.  Checked against the copy-based forced-halo path (the same kernels on the same
layer-range arithmetic: bit-identical) and against the oracle on sampled lines (lines
read layers i - i* - 1 and i - i*, periodic)."""

import numpy as np
import pytest


pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")

from tests.test_gpu_parity import _Grid, _sampled_line_parity  # noqa: E402


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    torch.cuda.set_device(0)
    yield


# (dims, k, precision, pad): layouts sldg_peer_halo_check accepts at the 2 MiB granularity;
# the first has no middle chunk (layers == 2 pad)
CASES = [
    ([32, 32, 32, 32], 2, "mixed", 16),
    ([32, 32, 32, 32], 3, "mixed", 8),
    ([32, 32, 32, 32], 2, "fp64", 2),
    ([256, 256, 16], 3, "mixed", 4),
]


@pytest.mark.parametrize("dims,k,precision,pad", CASES)
def test_peer_halo_matches_copy_halo_and_oracle(dims, k, precision, pad):
    D = len(dims)
    gp = _Grid(dims, k, precision=precision, force_halo=True, peer_halo=True, max_halo=pad)
    gc = _Grid(dims, k, precision=precision, force_halo=True, max_halo=pad)
    rng = np.random.default_rng(D * 100 + k)
    f = rng.uniform(-pad + 0.05, pad - 0.05, dims[0])  # i* in [-pad, pad - 1]: left, right <= pad
    cases = [(D - 1, 1.37, None, 0), (D - 1, -1.6, None, 0), (D - 1, float(pad) - 0.5, None, 0),
             (D - 1, -float(pad), None, 0), (D - 1, 0.0, f, 1), (0, 0.7, None, 0)]
    for i, (d, shift, field, mask) in enumerate(cases):
        seed = 900 + i
        for g in (gp, gc):
            g.fill_random(seed)
            g.advect(d, shift=shift, field=field, field_mask=mask)
        a, b = gp.get_coeffs(), gc.get_coeffs()
        assert a.tobytes() == b.tobytes(), f"dim {d} nu {shift}: peer-mapped halo differs from the copy halo"
        fld = field if field is not None else np.array([shift])
        _sampled_line_parity(gp, dims, k, precision, d, fld, mask, seed, 3, rng)
    assert gp.transpose_count() == 0
    # a sequence alternating the ping-pong buffers: dim 0, sharded, dim 1, sharded
    for g in (gp, gc):
        g.fill_random(77)
        for d, s in [(0, 0.3), (D - 1, 1.2), (1, -0.45), (D - 1, -1.3)]:
            g.advect(d, shift=s)
    assert gp.get_coeffs().tobytes() == gc.get_coeffs().tobytes()
    # a halo wider than the pads takes the transpose path (its own exchange)
    gp.fill_random(5)
    gp.advect(D - 1, shift=pad + 1.5)
    assert gp.transpose_count() == 1
    gp.destroy()
    gc.destroy()


def test_peer_halo_sweep_is_one_launch_and_captures():
    """The sharded sweep runs as a single sweep launch (no exchange, no boundary/interior
    split, no halo interval on the timeline), and a bounded device-field sequence captured in a
    CUDA graph replays bit-identically."""
    dims, k, pad = [32, 32, 32, 32], 3, 8
    gp = _Grid(dims, k, precision="mixed", force_halo=True, peer_halo=True, max_halo=pad)
    gp.fill_random(1)
    df = torch.tensor(np.linspace(-1.9, 1.8, dims[0] * dims[1]), dtype=torch.float64, device="cuda")
    gp.profile(True)
    gp.timeline(reset=True)
    gp.advect_device_bounded(3, df.data_ptr(), 3, -1.9, 1.8)
    tl = gp.timeline()
    gp.profile(False)
    kinds = [t[0] for t in tl]
    assert kinds == [3], tl  # one sweep launch along the sharded dim, no halo exchange interval
    gp.fill_random(2)
    gp.graph_begin()
    gp.advect_device_bounded(3, df.data_ptr(), 3, -1.9, 1.8)
    gp.advect(0, shift=0.25)
    gp.advect_device_bounded(3, df.data_ptr(), 3, -1.9, 1.8)
    gp.advect(1, shift=-0.5)
    gr = gp.graph_end()
    gr.launch()
    out = gp.get_coeffs()
    gp.fill_random(2)
    gp.advect_device_bounded(3, df.data_ptr(), 3, -1.9, 1.8)
    gp.advect(0, shift=0.25)
    gp.advect_device_bounded(3, df.data_ptr(), 3, -1.9, 1.8)
    gp.advect(1, shift=-0.5)
    assert out.tobytes() == gp.get_coeffs().tobytes()
    gr.destroy()
    gp.destroy()


def test_peer_halo_rejects_unaligned_layouts():
    """Creation fails with ENOTSUP (no silent fallback) when the pad or layer chunks are not
    multiples of the allocation granularity, or a rank holds fewer than 2 pad layers."""
    from paper_1603_07008_b200 import SldgError
    for dims, k, pad in [([32, 32, 32, 32], 2, 8), ([32, 32, 16], 2, 2), ([128, 128, 128, 6], 3, 4)]:
        with pytest.raises(SldgError, match="ENOTSUP"):
            _Grid(dims, k, precision="mixed", force_halo=True, peer_halo=True, max_halo=pad)


def test_peer_halo_mass_conserved():
    """Mass is conserved through peer-halo sweeps with halos up to the full pad width (fp64
    slot)."""
    dims, k, pad = [32, 32, 32, 32], 3, 8
    gp = _Grid(dims, k, precision="mixed", force_halo=True, peer_halo=True, max_halo=pad)
    gp.fill_random(11)
    m0 = gp.mass()
    for s in [1.25, -0.75, 7.5, -8.0]:
        gp.advect(3, shift=s)
    m1 = gp.mass()
    assert abs(m1 - m0) <= 1e-13 * max(1.0, abs(m0))
    gp.destroy()


def test_peer_halo_descriptor_path_in_one_process():
    """SLDG_DIST_PEER_VIA_FD: the edge chunks go through the multi-process route (export as POSIX
    file descriptors, passed over a unix socket (SCM_RIGHTS), import, map) with the rank as its own neighbour; the sweeps
    are bit-identical to the directly mapped pads."""
    dims, k, pad = [32, 32, 32, 32], 3, 8
    ga = _Grid(dims, k, precision="mixed", force_halo=True, peer_halo=True, max_halo=pad)
    gb = _Grid(dims, k, precision="mixed", force_halo=True, peer_halo=True, peer_via_fd=True, max_halo=pad)
    for g in (ga, gb):
        g.fill_random(21)
        for d, s in [(3, 1.7), (0, 0.4), (3, -7.2), (2, 0.9), (3, 6.6)]:
            g.advect(d, shift=s)
    assert ga.get_coeffs().tobytes() == gb.get_coeffs().tobytes()
    ga.destroy()
    gb.destroy()
