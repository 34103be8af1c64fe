"""Where does a small grid's split step spend its time?  Per-dim: device time of N sweeps
(CUDA events on the grid stream) vs the library's per-kernel events; eager and graph-replayed."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import sldg_inputs
from paper_1603_07008_b200 import Grid

cfg = sys.argv[1] if len(sys.argv) > 1 else "c2"
dims, kinds, k = {"c2": ([1024, 1024], ["x", "v"], 4), "c3": ([4096, 4096], ["x", "v"], 4)}[cfg]
lo = [0.0 if t == "x" else -6.0 for t in kinds]
hi = [4 * np.pi if t == "x" else 6.0 for t in kinds]
g = Grid(dims, k, lo=lo, hi=hi)
g.fill_separable(sldg_inputs.landau_terms(dims, k, kinds, lo, hi))
sw = sldg_inputs.vlasov_fields(dims, kinds, lo, hi)
dev = [torch.tensor(f, dtype=torch.float64, device="cuda") for _, f, _ in sw]
st = torch.cuda.ExternalStream(g.stream())
N = 50
def timed(fn, n=N):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(st):
        e0.record(st)
    for _ in range(n):
        fn()
    with torch.cuda.stream(st):
        e1.record(st)
    g.sync()
    return e0.elapsed_time(e1) / n
for (d, _, m), t in zip(sw, dev):
    for _ in range(3):
        g.advect_device(d, t.data_ptr(), m)
    g.sync()
    ms = timed(lambda: g.advect_device(d, t.data_ptr(), m))
    g.profile(True); g.kernel_time(reset=True)
    for _ in range(N):
        g.advect_device(d, t.data_ptr(), m)
    g.sync(); kms, kn, kb = g.kernel_time(d); g.profile(False)
    print(f"dim {d}: per call {ms*1e3:.1f} us, kernel {kms/kn*1e3:.1f} us ({kb/kn/(kms/kn*1e-3)/1e9:.0f} GB/s), kernel={g.sweep_kernel(d)}")
    # a graph of two sweeps along d
    g.graph_begin(); g.advect_device(d, t.data_ptr(), m); g.advect_device(d, t.data_ptr(), m); gr = g.graph_end()
    gr.launch(); g.sync()
    ms2 = timed(gr.launch) / 2
    print(f"   graph: per sweep {ms2*1e3:.1f} us")
    gr.destroy()
# whole step
def step():
    for (d, _, m), t in zip(sw, dev):
        g.advect_device(d, t.data_ptr(), m)
print("step eager", timed(step) * 1e3, "us")
g.graph_begin(); step(); gr = g.graph_end(); gr.launch(); g.sync()
print("step graph", timed(gr.launch) * 1e3, "us")
