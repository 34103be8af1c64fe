"""One Gauss-node x sweep on a C3- or C5-slab-shaped grid (profiling helper)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_1603_07008_b200 import Grid

cfg = sys.argv[1] if len(sys.argv) > 1 else "c3"
dims, k, vdim = {"c3": ([4096, 4096], 4, 1), "c5s": ([128, 128, 128, 16], 3, 2)}[cfg]
g = Grid(dims, k)
g.fill_random(1)
xg = np.polynomial.legendre.leggauss(k)[0]
nv = dims[vdim]
hv = 12.0 / nv
vc = -6.0 + (np.arange(nv) + 0.5) * hv
nodal = ((vc[:, None] + xg[None, :] * hv / 2) * 0.05 / (4 * np.pi / dims[0])).reshape(-1)
d = torch.tensor(nodal, dtype=torch.float64, device="cuda")
import time
for _ in range(5):
    g.advect_vnodes_device(0, vdim, d.data_ptr())
g.sync()
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 0
if reps:
    t0 = time.perf_counter()
    for _ in range(reps):
        g.advect_vnodes_device(0, vdim, d.data_ptr())
    g.sync()
    print(f"{cfg} k={k}: {(time.perf_counter() - t0) / reps * 1e3:.3f} ms per nodal sweep (wall clock, incl. weights kernel)")
print("ok")
