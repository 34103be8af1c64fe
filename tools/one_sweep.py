#!/usr/bin/env python
"""Three sweeps of one dim of a 2D grid (for ncu captures): one_sweep.py K PREC DIM [N]."""
import sys
import os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1603_07008_b200 import Grid
k, prec, dim = int(sys.argv[1]), sys.argv[2], int(sys.argv[3])
n = int(sys.argv[4]) if len(sys.argv) > 4 else 4096
g = Grid([n, n], k, precision=prec)
g.fill_random(1)
for _ in range(3):
    g.advect(dim, shift=2.37)
g.sync()
print("ok", g.sweep_kernel(dim))
