"""Multi-GPU parity (two processes, one GPU each; skipped on one-GPU boxes): the sharded sweep
with the NCCL halo exchange and with peer-mapped halo layers (SLDG_DIST_PEER_HALO: the pads map
the neighbour's edge layers over NVLink) against the oracle (P:259-272 periodic two-cell update;
P:214-219 the halo), and the two halo paths bit-identical to each other."""
import multiprocessing as mp
import os

import numpy as np
import pytest

import oracle
import sldg_inputs

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")

WORLD = 2


def _need_gpus():
    if not torch.cuda.is_available() or torch.cuda.device_count() < WORLD:
        pytest.skip(f"needs {WORLD} GPUs")


def _rank_main(rank, uid, dims, k, precision, pad, peer, cases, seed, q):
    try:
        torch.cuda.set_device(rank)
        from paper_1603_07008_b200 import Grid
        g = Grid(dims, k, precision=precision, rank=rank, world=WORLD, unique_id=uid, max_halo=pad,
                 peer_halo=peer)
        L = int(np.prod(dims[:-1]))
        c = sldg_inputs.random_coeffs(dims, k, seed, first_cell=g.first_layer * L, n_cells=g.n_layers * L)
        outs = []
        for d, shift in cases:
            g.set_coeffs(c)  # this rank's layers (local cell 0 = global cell first_layer * L)
            g.advect(d, shift=shift)
            outs.append(g.get_coeffs())
        m = g.mass()
        g.destroy()
        q.put((rank, outs, m, None))
    except Exception as e:  # reported to the parent
        q.put((rank, None, None, repr(e)))


def _run(dims, k, precision, pad, peer, cases, seed):
    from paper_1603_07008_b200 import sldg
    uid = sldg.nccl_unique_id()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    ps = [ctx.Process(target=_rank_main, args=(r, uid, dims, k, precision, pad, peer, cases, seed, q))
          for r in range(WORLD)]
    for p in ps:
        p.start()
    res = {}
    for _ in range(WORLD):
        r, outs, m, err = q.get(timeout=600)
        assert err is None, f"rank {r}: {err}"
        res[r] = (outs, m)
    for p in ps:
        p.join(timeout=60)
    # global arrays in layer order (rank 0 holds the first layers)
    return [np.concatenate([res[r][0][i] for r in range(WORLD)]) for i in range(len(cases))], res[0][1]


@pytest.mark.parametrize("peer", [False, True])
def test_two_gpu_sharded_sweeps_match_oracle(peer):
    _need_gpus()
    dims, k, precision, pad = [32, 32, 32, 32], 2, "fp64", 2
    K = k ** 4
    cases = [(3, 1.37), (3, -1.6), (3, 0.5), (0, 2.25), (2, -0.7)]
    outs, _ = _run(dims, k, precision, pad, peer, cases, 4242)
    src = oracle.round_layout(sldg_inputs.random_coeffs(dims, k, 4242), K, K)
    for (d, shift), got in zip(cases, outs):
        ref = oracle.advect(src, dims, k, d, shift=shift, n_double=K)
        scale = np.max(np.abs(src))
        assert np.max(np.abs(got - ref)) <= 1e-13 * scale, (d, shift)


def test_two_gpu_peer_halo_bit_identical_to_nccl_halo():
    _need_gpus()
    dims, k, precision, pad = [32, 32, 32, 32], 3, "mixed", 8
    cases = [(3, 1.37), (3, -7.6), (3, 7.5), (1, 0.4)]
    a, ma = _run(dims, k, precision, pad, False, cases, 99)
    b, mb = _run(dims, k, precision, pad, True, cases, 99)
    for (d, shift), x, y in zip(cases, a, b):
        assert x.tobytes() == y.tobytes(), (d, shift)
    assert ma == mb
