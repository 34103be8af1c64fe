"""Multi-process (gloo, CPU) tests of the sharded-grid layer's host logic.

The halo exchange of a sweep along the sharded dim is planned by `sldg_halo_plan` (the exact
plan `sldg_advect` executes with grouped NCCL send/recv on GPUs).  Here every rank runs that
plan with gloo point-to-point on CPU tensors holding its block of layers, and checks that each
halo slot received the right global layer (periodic wrap, several owners, self copies).  A
second test runs a sharded SLDG sweep on CPU: the received halos plus the local layers must be
all the source layers the rank's targets read (two adjacent source cells), and the
rank's output, computed by the oracle on exactly those layers, equals the global oracle.
"""
import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")
import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _split(n, world, r):
    base, extra = divmod(n, world)
    return r * base + min(r, extra), base + (1 if r < extra else 0)


def _exchange(plan, buf, rank):
    reqs = []
    for kind, peer, slot, src in plan:
        if kind == 2:
            buf[slot] = buf[src]
        elif kind == 0:
            reqs.append((slot, dist.irecv(buf[slot], src=peer)))
        else:
            reqs.append((None, dist.isend(buf[slot].clone(), dst=peer)))
    for _, r in reqs:
        r.wait()


def _worker(rank, world, port, n, pad, cases, q):
    import sys
    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_1603_07008_b200 import sldg
    try:
        first, layers = _split(n, world, rank)
        for left, right in cases:
            width = 3
            buf = torch.full((layers + 2 * pad, width), float("nan"), dtype=torch.float64)
            for l in range(layers):
                buf[pad + l] = first + l
            plan = sldg.halo_plan(n, world, rank, pad, left, right)
            _exchange(plan, buf, rank)
            for j in range(left):
                assert torch.all(buf[pad - left + j] == (first - left + j) % n), (rank, left, right, j)
            for j in range(right):
                assert torch.all(buf[pad + layers + j] == (first + layers + j) % n), (rank, left, right, j)
            assert torch.all(buf[pad:pad + layers, 0] == torch.arange(first, first + layers))
            dist.barrier()
        q.put((rank, "ok"))
    except Exception as e:  # pragma: no cover - reported to the parent
        q.put((rank, repr(e)))
    finally:
        dist.destroy_process_group()


def _run(world, n, pad, cases):
    import __graft_entry__
    __graft_entry__.build()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, n, pad, cases, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
    assert all(r[1] == "ok" for r in res), res


def test_halo_plan_world2():
    _run(2, 16, 3, [(1, 1), (1, 0), (0, 2), (3, 3), (2, 1)])


def test_halo_plan_world3_uneven_and_multi_owner():
    # 7 layers over 3 ranks (3, 2, 2): halos of 3 span two owners and wrap onto self
    _run(3, 7, 4, [(1, 1), (3, 2), (4, 4), (0, 3)])


def test_halo_plan_world4_c5_shape():
    # the C5 v2 sweep on 4 GPUs: 128 layers, eps=0.01 -> (1, 1); eps=0.5 -> (2, 2)
    _run(4, 128, 2, [(1, 1), (2, 2)])


def _sweep_worker(rank, world, port, q):
    import sys
    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import oracle
    import sldg_inputs
    from paper_1603_07008_b200 import sldg
    try:
        dims, k = [6, 10], 2
        K = 4
        n = dims[1]
        c = oracle.round_layout(sldg_inputs.random_coeffs(dims, k, 1603), K, 1)
        field = np.linspace(-2.7, 1.4, dims[0])  # per-lane shifts along the sharded dim
        istar = np.floor(field).astype(int)
        left, right = sldg.halo_widths(int(istar.min()), int(istar.max()))
        pad = max(left, right)
        first, layers = _split(n, world, rank)
        lay = c.reshape(n, dims[0] * K)  # layer-major view of the global grid
        buf = torch.full((layers + 2 * pad, dims[0] * K), float("nan"), dtype=torch.float64)
        buf[pad:pad + layers] = torch.from_numpy(lay[first:first + layers])
        _exchange(sldg.halo_plan(n, world, rank, pad, left, right), buf, rank)
        ext = buf.numpy()
        # every target layer t reads layers t - i* - 1 and t - i*: all must be present
        full = oracle.advect(c, dims, k, 1, field=field, field_mask=0b01, n_double=1).reshape(n, -1)
        for t in range(first, first + layers):
            for i0 in range(dims[0]):
                for src in (t - istar[i0] - 1, t - istar[i0]):
                    loc = src - first + pad
                    assert 0 <= loc < layers + 2 * pad
                    assert np.array_equal(ext[loc, i0 * K:(i0 + 1) * K], lay[src % n, i0 * K:(i0 + 1) * K])
        # the rank's output from its extended block alone: oracle per line on exactly those rows
        for i0 in range(dims[0]):
            rows = ext[:, i0 * K:(i0 + 1) * K]
            for t in range(first, first + layers):
                a_row = rows[t - istar[i0] - 1 - first + pad]
                b_row = rows[t - istar[i0] - first + pad]
                line = np.stack([a_row, b_row])  # a 2-cell line: target 1 reads (0, 1) at i* = 0
                out = oracle.advect(line, [1, 2], k, 1, shift=field[i0] - istar[i0], n_double=1)[1]
                assert np.max(np.abs(out - full[t, i0 * K:(i0 + 1) * K])) <= 1e-15
        q.put((rank, "ok"))
    except Exception as e:  # pragma: no cover
        import traceback
        q.put((rank, traceback.format_exc()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_sweep_from_halos_matches_global_oracle(world):
    import __graft_entry__
    __graft_entry__.build()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_sweep_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
    assert all(r[1] == "ok" for r in res), res


# ------------------------------------------------------------------------------ transpose path
def _transpose_worker(rank, world, port, cases, q):
    """The transpose path of a sweep along the sharded dim, run with gloo on CPU
    exactly as `sldg_transpose_plan` lays it out: rank r sends p its layers restricted to p's
    slab of dim D-2, receives whole lines for its own slab, sweeps them (oracle, periodic), and
    the inverse exchange returns them.  The result must equal the global oracle sweep."""
    import sys
    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import oracle
    import sldg_inputs
    from paper_1603_07008_b200 import sldg
    try:
        for dims, k, shift, use_field in cases:
            n0, ns, no = dims
            K = k ** 3
            c = oracle.round_layout(sldg_inputs.random_coeffs(dims, k, 7008), K, 1)
            glob = c.reshape(no, ns, n0, K)
            field = np.linspace(-3.3 * no, 2.1 * no, n0 * ns) if use_field else None
            mask = 0b011 if use_field else 0
            want = oracle.advect(c, dims, k, 2, shift=shift, field=field, field_mask=mask,
                                 n_double=1).reshape(no, ns, n0, K)
            plan = sldg.transpose_plan(no, ns, world, rank)
            f_r, c_r = plan[rank][0], plan[rank][1]
            a_r, s_r = plan[rank][6], plan[rank][7]
            mine = torch.from_numpy(glob[f_r:f_r + c_r].copy())
            T = torch.full((no, s_r, n0, K), float("nan"), dtype=torch.float64)
            reqs = []
            for p in range(world):
                sf, sc, af, ac, rf, rc, _, _ = plan[p]
                blk = mine[:, af:af + ac].contiguous()
                if p == rank:
                    T[rf:rf + rc] = blk
                    continue
                reqs.append(dist.isend(blk, dst=p))
                buf = torch.empty((rc, s_r, n0, K), dtype=torch.float64)
                reqs.append((rf, rc, buf, dist.irecv(buf, src=p)))
            for r_ in reqs:
                if isinstance(r_, tuple):
                    rf, rc, buf, h = r_
                    h.wait()
                    T[rf:rf + rc] = buf
                else:
                    r_.wait()
            assert not torch.isnan(T).any()
            # local sweep of whole lines on the slab; the field restricted to the slab (dim 1 offset a_r)
            tf = None
            if use_field:
                tf = field.reshape(ns, n0)[a_r:a_r + s_r].reshape(-1)
            if s_r > 0:  # a rank can own no slab when n_slab < world
                Tout = oracle.advect(T.numpy().reshape(-1, K), [n0, s_r, no], k, 2, shift=shift, field=tf,
                                     field_mask=mask, n_double=1).reshape(no, s_r, n0, K)
                Tout = torch.from_numpy(Tout)
            else:
                Tout = T
            out = torch.full_like(mine, float("nan"))
            reqs = []
            for p in range(world):
                sf, sc, af, ac, rf, rc, _, _ = plan[p]
                if p == rank:
                    out[:, af:af + ac] = Tout[rf:rf + rc]
                    continue
                reqs.append(dist.isend(Tout[rf:rf + rc].contiguous(), dst=p))
                buf = torch.empty((c_r, ac, n0, K), dtype=torch.float64)
                reqs.append((af, ac, buf, dist.irecv(buf, src=p)))
            for r_ in reqs:
                if isinstance(r_, tuple):
                    af, ac, buf, h = r_
                    h.wait()
                    out[:, af:af + ac] = buf
                else:
                    r_.wait()
            assert np.array_equal(out.numpy(), want[f_r:f_r + c_r]), (rank, dims, shift)
            dist.barrier()
        q.put((rank, "ok"))
    except Exception:  # pragma: no cover
        import traceback
        q.put((rank, traceback.format_exc()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_transpose_path_matches_global_oracle(world):
    import __graft_entry__
    __graft_entry__.build()
    # (dims [n0, n_slab, n_outer], k, constant shift, per-line field over dims 0 and 1)
    cases = [([4, 5, 7], 2, 5.3, False), ([3, 6, 8], 2, -9.75, True), ([2, 2, 9], 1, 0.5, False)]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_transpose_worker, args=(r, world, port, cases, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=180) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
    assert all(r[1] == "ok" for r in res), res
