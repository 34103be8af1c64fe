"""Host cost per sldg_advect call (tiny grid, so device time is negligible): constant shift,
host field (pinned), device field; and sldg_mass."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_1603_07008_b200 import Grid

for dims, k in [([64, 64], 4), ([1024, 1024], 4)]:
    g = Grid(dims, k, precision="mixed")
    g.fill_random(1)
    f = torch.empty(dims[0], dtype=torch.float64, pin_memory=True)
    f.numpy()[:] = np.linspace(-0.4, 0.4, dims[0])
    df = f.cuda()
    for name, fn in [("const", lambda: g.advect(1, shift=0.37)),
                     ("host field", lambda: g.advect(1, field=f.numpy(), field_mask=1)),
                     ("device field", lambda: g.advect_device(1, df.data_ptr(), 1)),
                     ("mass", lambda: g.mass())]:
        for _ in range(20):
            fn()
        g.sync()
        n = 200
        t0 = time.perf_counter()
        for _ in range(n):
            fn()
        t1 = time.perf_counter()
        g.sync()
        t2 = time.perf_counter()
        print(f"{dims} {name}: host {1e6 * (t1 - t0) / n:.1f} us/call, with drain {1e6 * (t2 - t0) / n:.1f} us/call")
    g.destroy()
