#!/usr/bin/env python
"""Small invocations of every sweep kernel variant, for compute-sanitizer.

  compute-sanitizer --tool {memcheck,racecheck,synccheck,initcheck} python tools/sanitize_cases.py

Each case builds a small grid, runs the sweeps that select one kernel variant (printed from
sldg_sweep_kernel) and checks the result against the CPU oracle, so a sanitizer run is also a
parity run.  Shapes are chosen to hit: the d = 0 TMA kernel with 1 and 2 CTAs per SM and with
shared-memory weights (k >= 5); the strided TMA kernel in its PSPAN and long-tile instances,
1 and 2 CTAs per SM, the split consumer (k = 5, 6), per-lane spans and the direct-load fallback
for spans wider than a stage; the forced halo path (device copies and NCCL self-exchange); the
transpose path; the 1D line kernel; the Gauss-node sweep.
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402
import sldg_inputs  # noqa: E402
from paper_1603_07008_b200 import Grid  # noqa: E402


def check(g, c_in, dims, k, prec, dim, shift=0.0, field=None, mask=0, tag=""):
    K = k ** len(dims)
    nd = 1 if prec == "mixed" else K
    src = oracle.round_layout(c_in, K, nd)
    g.set_coeffs(c_in)
    g.advect(dim, shift=shift, field=field, field_mask=mask)
    got = g.get_coeffs()
    ref = oracle.advect(src, dims, k, dim, shift=shift, field=field, field_mask=mask, n_double=nd)
    scale = max(1.0, float(np.max(np.abs(src))))
    err = float(np.max(np.abs(got - ref)))
    ok = err <= 1e-5 * scale
    print(f"{'ok ' if ok else 'BAD'} {tag:34s} dims={dims} k={k} {prec:5s} dim={dim} kernel={g.sweep_kernel(dim):22s} "
          f"max|d|={err:.2e}", flush=True)
    return ok


def main():
    import torch
    torch.cuda.set_device(0)
    rng = np.random.default_rng(0)
    ok = True
    cases = [
        # dims, k, prec, {grid kwargs}, tag
        ([256, 64], 2, "mixed", {}, "d0 2-CTA / strided"),
        ([128, 48], 3, "mixed", {}, "d0 1-CTA / strided PSPAN"),
        ([128, 48], 3, "fp64", {}, "fp64 d0 / strided"),
        ([64, 4, 4, 256], 3, "mixed", {}, "strided long tiles (non-PSPAN)"),
        ([64, 40], 5, "mixed", {}, "k=5 smem weights / split"),
        ([48, 36], 6, "mixed", {}, "k=6 smem weights / split"),
        ([32, 6, 20], 2, "mixed", {"force_halo": True, "max_halo": 2}, "forced halo (device copies)"),
        ([32, 6, 20], 2, "fp64", {"force_halo": True, "max_halo": 2, "nccl_self": True}, "forced halo (NCCL self)"),
        ([12, 4, 7], 3, "mixed", {"force_transpose": True, "max_halo": 1}, "transpose path"),
        ([4096], 4, "mixed", {}, "1D line kernel"),
    ]
    for dims, k, prec, kw, tag in cases:
        g = Grid(dims, k, precision=prec, **kw)
        c = sldg_inputs.random_coeffs(dims, k, 11)
        D = len(dims)
        for d in range(D):
            ok &= check(g, c, dims, k, prec, d, shift=1.37, tag=tag)
            if D > 1 and d > 0:  # per-lane field over dim 0 (strided spans)
                f = rng.uniform(-1.6, 1.6, dims[0])
                ok &= check(g, c, dims, k, prec, d, field=f, mask=1, tag=tag + " per-lane")
        g.destroy()
    # spans wider than a stage: the strided direct-load fallback
    dims, k = [64, 128], 2
    g = Grid(dims, k, precision="mixed")
    f = rng.uniform(-60.0, 60.0, dims[0])
    ok &= check(g, sldg_inputs.random_coeffs(dims, k, 12), dims, k, "mixed", 1, field=f, mask=1,
                tag="strided wide-span fallback")
    g.destroy()
    # Gauss-node x sweep (NEXT-3)
    from oracle import vnodes
    dims, k = [32, 16], 3
    g = Grid(dims, k, lo=[0, -6], hi=[4 * np.pi, 6], precision="mixed")
    c = sldg_inputs.random_coeffs(dims, k, 13)
    nu = vnodes.nodal_velocity_field(dims[1], -6.0, 6.0, k, 0.8)
    g.set_coeffs(c)
    g.advect_vnodes(0, 1, nu)
    got = g.get_coeffs()
    ref = vnodes.advect_vnodes(oracle.round_layout(c, k * k, 1), dims, k, 0, 1, nu, n_double=1)
    err = float(np.max(np.abs(got - ref)))
    print(f"{'ok ' if err < 1e-5 else 'BAD'} gauss-node sweep max|d|={err:.2e}", flush=True)
    ok &= err < 1e-5
    g.destroy()
    print("ALL OK" if ok else "FAILURES")
    return 0 if ok else 1


if __name__ == "__main__":
    sys.exit(main())
