#!/usr/bin/env python
"""1D periodic advection, 64 cells, k = 4, nu = 0.37, 100 steps -- the
correctness / oracle-seconds config, reported as wall time (it is latency-bound: 256 DoF).

GPU: 100 sldg_advect calls (eager), and the same 100 steps captured once in a CUDA graph and
replayed (bit-identical to the eager run, checked here).  Parity of the 100 steps with the
oracle is tests/test_gpu_parity.py::test_c1_config_100_steps (tools/ do not run the oracle).

    python tools/c1_walltime.py [--out profiles/round1/c1_walltime.md]
"""
import argparse
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import sldg_inputs  # noqa: E402
from paper_1603_07008_b200 import Grid  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "round1", "c1_walltime.md"))
    a = ap.parse_args()
    torch.cuda.set_device(0)
    N, k, nu, steps = 64, 4, 0.37, 100
    c0 = sldg_inputs.project_1d(lambda x: 1 + 0.5 * np.sin(2 * np.pi * x), N, 0.0, 1.0, k, 12)
    rows = []
    for prec in ["mixed", "fp64"]:
        g = Grid([N], k, precision=prec)
        g.set_coeffs(c0)
        g.advect(0, shift=nu)
        g.set_coeffs(c0)
        g.sync()
        t0 = time.perf_counter()
        for _ in range(steps):
            g.advect(0, shift=nu)
        g.sync()
        eager = time.perf_counter() - t0
        got = g.get_coeffs()
        # graph: the 100 steps captured once (even count: the buffer parity is restored)
        g.set_coeffs(c0)
        g.graph_begin()
        for _ in range(steps):
            g.advect(0, shift=nu)
        gr = g.graph_end()
        t0 = time.perf_counter()
        gr.launch()
        g.sync()
        graph = time.perf_counter() - t0
        got_g = g.get_coeffs()
        gr.destroy()
        g.destroy()
        assert got.tobytes() == got_g.tobytes()
        rows.append((prec, eager, graph))
    lines = ["# SURVEY 8(d) C1 on one B200: 1D, 64 cells, k = 4, nu = 0.37, 100 steps", "",
             "Wall time of the 100 steps (host clock, synchronised); the graph replay is bit-identical to "
             "the eager run; parity with the oracle: tests/test_gpu_parity.py::test_c1_config_100_steps.", "",
             "| storage | GPU eager (100 sldg_advect calls) | GPU, one CUDA graph of the 100 steps |",
             "|---|---|---|"]
    for prec, e, gph in rows:
        lines.append(f"| {prec} | {e * 1e3:.2f} ms ({e / steps * 1e6:.1f} us/step) | {gph * 1e3:.3f} ms "
                     f"({gph / steps * 1e6:.2f} us/step) |")
    os.makedirs(os.path.dirname(a.out), exist_ok=True)
    open(a.out, "w").write("\n".join(lines) + "\n")
    print("\n".join(lines))


if __name__ == "__main__":
    main()
