"""The seeded input generators (sldg_inputs) -- no method arithmetic, CPU only."""
import numpy as np

import sldg_inputs


def test_splitmix64_reference_values():
    """Standard splitmix64 sequence from state 0 (first outputs of the public reference
    generator: 0xE220A8397B1DCDAF, 0x6E789E6AA1B965F4, 0x06C45D188009454F)."""
    z = np.array([0, 0x9E3779B97F4A7C15, 2 * 0x9E3779B97F4A7C15 % 2**64], dtype=np.uint64)
    out = sldg_inputs.splitmix64(z)
    assert [int(v) for v in out] == [0xE220A8397B1DCDAF, 0x6E789E6AA1B965F4, 0x06C45D188009454F]


def test_random_coeffs_ranges_and_keying():
    dims, k = [8, 4, 3], 2
    c = sldg_inputs.random_coeffs(dims, k, 1603)
    assert c.shape == (96, 8)
    assert np.all((c[:, 0] >= 0.5) & (c[:, 0] < 1.5))
    deg = sldg_inputs.coef_degree(k, 3)
    for q in range(1, 8):
        assert np.max(np.abs(c[:, q])) <= 8.0 ** -deg[q]
    # keyed by global cell index: any sub-range reproduces the same values
    sub = sldg_inputs.random_coeffs(dims, k, 1603, first_cell=37, n_cells=20)
    assert sub.tobytes() == c[37:57].tobytes()
    sel = sldg_inputs.random_coeffs(dims, k, 1603, cells=np.array([5, 90, 3]))
    assert sel.tobytes() == c[[5, 90, 3]].tobytes()
    assert not np.array_equal(c, sldg_inputs.random_coeffs(dims, k, 7008))


def test_separable_assembly_matches_direct_projection():
    """Sum of tensor products of 1D projections == direct 2D tensor Gauss projection."""
    dims, k = [5, 4], 3
    kinds, lo, hi = ["x", "v"], [0.0, -6.0], [4 * np.pi, 6.0]
    terms = sldg_inputs.landau_terms(dims, k, kinds, lo, hi, eps=0.3)
    c = sldg_inputs.assemble_separable(terms, dims, k)
    xq, wq = np.polynomial.legendre.leggauss(12)
    V = np.polynomial.legendre.legvander(xq, k - 1)
    hx, hv = (hi[0] - lo[0]) / 5, (hi[1] - lo[1]) / 4
    f = lambda x, v: (1 + 0.3 * np.cos(0.5 * x)) * np.exp(-v * v / 2) / np.sqrt(2 * np.pi)  # noqa
    norm = (2 * np.arange(k) + 1) / 2
    for i1 in range(4):
        for i0 in range(5):
            X = lo[0] + (i0 + 0.5) * hx + 0.5 * hx * xq
            Y = lo[1] + (i1 + 0.5) * hv + 0.5 * hv * xq
            F = f(X[:, None], Y[None, :])
            cc = np.einsum("ab,a,b,am,bn->nm", F, wq, wq, V, V) * norm[None, :] * norm[:, None]
            np.testing.assert_allclose(c[i0 + 5 * i1].reshape(k, k), cc, atol=1e-14)


def test_vlasov_fields_shapes():
    dims = [8, 6, 5, 4]
    kinds = ["x", "x", "v", "v"]
    sw = sldg_inputs.vlasov_fields(dims, kinds, [0, 0, -6, -6], [4 * np.pi, 4 * np.pi, 6, 6])
    assert [s[0] for s in sw] == [0, 1, 2, 3]
    assert [s[2] for s in sw] == [0b0100, 0b1000, 0b0011, 0b0011]
    assert sw[0][1].shape == (5,) and sw[2][1].shape == (48,)
    # v1 field depends only on x1 (dim 0, fastest), v2 field only on x2 (dim 1)
    f2 = sw[2][1].reshape(6, 8)
    assert np.all(f2 == f2[0:1, :])
    f3 = sw[3][1].reshape(6, 8)
    assert np.all(f3 == f3[:, 0:1])
