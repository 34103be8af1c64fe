#!/usr/bin/env python
"""Tables III-VI of arXiv:1603.07008 re-measured on one B200 (NEXT-1 of SURVEY 8(f)).

The paper's performance tables time the 1D SLDG sweep for order o in {2, 4} and "# double"
d in {o, ..., 0} and report the achieved bandwidth (one load + one store of every stored
coefficient per step at its storage width), the speedup against the all-fp64 run
(d = o) and the memory reduction 8o / (8d + 4(o - d)).  Problem size, step count and nu are not
stated in the paper; here N = 2^24 cells (the SPEC default), nu = 2.25,
warm-up 5 and 20 timed steps, median of 5 repetitions, CUDA events on the grid's stream.

    python tools/paper_tables.py [--cells 16777216] [--out profiles/round1/paper_tables_b200.md]
"""
import argparse
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_1603_07008_b200 import Grid  # noqa: E402

PAPER = json.load(open(os.path.join(ROOT, "tests", "golden", "paper_tables.json")))


def run(N, o, d, steps, reps, nu):
    g = Grid([N], o, precision=d)
    g.fill_random(1603)
    stream = torch.cuda.ExternalStream(g.stream())
    for _ in range(5):
        g.advect(0, shift=nu)
    g.sync()
    times = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(stream):
            e0.record(stream)
        for _ in range(steps):
            g.advect(0, shift=nu)
        with torch.cuda.stream(stream):
            e1.record(stream)
        g.sync()
        times.append(e0.elapsed_time(e1) / steps)
    ms = statistics.median(times)
    # sweep kernel alone (events the library records around each sweep launch)
    g.profile(True)
    g.kernel_time(0, reset=True)
    for _ in range(steps):
        g.advect(0, shift=nu)
    g.sync()
    kms, kn, _ = g.kernel_time(0)
    g.profile(False)
    kern = g.sweep_kernel(0)
    g.destroy()
    bytes_step = 2 * N * (8 * d + 4 * (o - d))
    return ms, bytes_step / (ms * 1e-3) / 1e9, kern, kms / kn, bytes_step / (kms / kn * 1e-3) / 1e9


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--cells", type=int, default=1 << 24)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--nu", type=float, default=2.25)
    ap.add_argument("--orders", default="2,4")
    ap.add_argument("--doubles", default=None, help="comma list of d (default: o..0)")
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "round1", "paper_tables_b200.md"))
    args = ap.parse_args()
    torch.cuda.set_device(0)
    N = args.cells
    rows = []
    for o in [int(x) for x in args.orders.split(",")]:
        base = None
        ds = range(o, -1, -1) if args.doubles is None else [int(x) for x in args.doubles.split(",")]
        for d in ds:
            ms, gbs, kern, kms, kgbs = run(N, o, d, args.steps, args.reps, args.nu)
            if base is None:
                base = ms
            rows.append({"o": o, "d": d, "ms": ms, "gbs": gbs, "gdofs": N * o / (ms * 1e-3) / 1e9,
                         "kernel_ms": kms, "kernel_gbs": kgbs, "speedup": base / ms, "memorydown": 8.0 * o / (8 * d + 4 * (o - d)), "kernel": kern})
    paper = {}
    for key in ["table_III_cpu", "table_VI_k80_cell", "table_V_k80_smem"]:
        for r in PAPER[key]["rows"]:
            paper.setdefault((r[0], r[1]), {})[key] = r
    lines = ["# Tables III-VI of arXiv:1603.07008 re-measured on one B200", "",
             f"1D SLDG sweep, N = {N} cells, nu = {args.nu}, median of {args.reps} x {args.steps} steps "
             "(CUDA events).  Bandwidth = one load + one store of every stored coefficient per step "
             "(the paper's definition, pinned by its speedup identity, SURVEY 4).  Paper columns: "
             "Table III (2x Xeon E5-2630 v3) and Table VI (0.5x K80, thread per cell; Table V for o=2).",
             "",
             "Step = one `sldg_advect` call (weight build + sweep launch, host enqueue included); the "
             "kernel column is the sweep kernel alone (CUDA events around its launch).",
             "",
             "| o | # double d | B200 GB/s (step) | B200 GB/s (kernel) | B200 GDoF/s | B200 speedup vs d=o | memorydown | CPU GB/s (speedup) | K80 GB/s (speedup) | kernel |",
             "|---|---|---|---|---|---|---|---|---|---|"]
    for r in rows:
        p = paper.get((r["o"], r["d"]), {})
        cpu = p.get("table_III_cpu")
        k80 = p.get("table_VI_k80_cell") or p.get("table_V_k80_smem")
        fmt = lambda t: "--" if t is None else f"{t[2]} ({t[3] if t[3] is not None else '--'})"  # noqa: E731
        lines.append(f"| {r['o']} | {r['d']} | {r['gbs']:.0f} | {r['kernel_gbs']:.0f} | {r['gdofs']:.1f} | {r['speedup']:.2f} | "
                     f"{r['memorydown']:.2f} | {fmt(cpu)} | {fmt(k80)} | {r['kernel']} |")
    os.makedirs(os.path.dirname(args.out), exist_ok=True)
    open(args.out, "w").write("\n".join(lines) + "\n")
    print("\n".join(lines))
    print(json.dumps(rows))


if __name__ == "__main__":
    main()
