#!/usr/bin/env python
"""SURVEY 8(d) C3 as specified: 2D 4096^2, constant nu = 2.37 (alpha = 0.37, i* = 2: a misaligned
window), k = 2..6, one sweep along dim 0 (contiguous) and one along dim 1 (strided), mixed and
fp64 storage -- 20 points.  Device time of the sweep kernels (CUDA events the library records
around each launch), algorithmic bytes = one load + one store of every stored coefficient.

    python tools/order_sweep.py [--n 4096] [--reps 10] [--out profiles/round1/order_sweep_c3.md]
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_1603_07008_b200 import Grid  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=4096)
    ap.add_argument("--reps", type=int, default=10)
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "round1", "order_sweep_c3.md"))
    a = ap.parse_args()
    torch.cuda.set_device(0)
    peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))).get("hbm_gbs", 6529.7)
    rows = []
    for k in range(2, 7):
        res = {}
        for prec in ["mixed", "fp64"]:
            g = Grid([a.n, a.n], k, precision=prec)
            g.fill_random(1603)
            for dim in (0, 1):
                for _ in range(3):
                    g.advect(dim, shift=2.37)
                g.sync()
                g.profile(True)
                g.kernel_time(reset=True)
                for _ in range(a.reps):
                    g.advect(dim, shift=2.37)
                g.sync()
                ms, n, b = g.kernel_time(dim)
                g.profile(False)
                gbs = b / (ms * 1e-3) / 1e9
                res[(prec, dim)] = (ms / n, gbs, g.sweep_kernel(dim))
            g.destroy()
            torch.cuda.synchronize()
        for dim in (0, 1):
            mm, mg, mk = res[("mixed", dim)]
            fm, fg, fk = res[("fp64", dim)]
            dofs = a.n * a.n * k * k
            rows.append({"k": k, "dim": dim, "mixed_ms": mm, "mixed_gbs": mg, "mixed_gdofs": dofs / (mm * 1e-3) / 1e9,
                         "fp64_ms": fm, "fp64_gbs": fg, "speedup": fm / mm,
                         "bytes_ratio": (8 * k * k) / (8 + 4 * (k * k - 1)), "kernel_mixed": mk, "kernel_fp64": fk})
    lines = ["# SURVEY 8(d) C3 order sweep on one B200", "",
             f"2D {a.n}^2, constant nu = 2.37, k = 2..6, one sweep per dim, device time per sweep kernel "
             f"(median-free mean of {a.reps}); roofline = measured copy bandwidth {peak:.0f} GB/s.", "",
             "| k | dim | mixed ms | mixed GB/s (% roofline) | mixed GDoF/s | fp64 ms | fp64 GB/s | mixed / fp64 speedup | byte ratio | kernels (mixed / fp64) |",
             "|---|---|---|---|---|---|---|---|---|---|"]
    for r in rows:
        lines.append(f"| {r['k']} | {r['dim']} | {r['mixed_ms']:.3f} | {r['mixed_gbs']:.0f} ({100 * r['mixed_gbs'] / peak:.0f}%) | "
                     f"{r['mixed_gdofs']:.0f} | {r['fp64_ms']:.3f} | {r['fp64_gbs']:.0f} | {r['speedup']:.2f} | "
                     f"{r['bytes_ratio']:.2f} | {r['kernel_mixed']} / {r['kernel_fp64']} |")
    os.makedirs(os.path.dirname(a.out), exist_ok=True)
    open(a.out, "w").write("\n".join(lines) + "\n")
    print("\n".join(lines))


if __name__ == "__main__":
    main()
