"""Device copy bandwidth vs size (L2 flushed before each copy): what a sweep of this size can reach."""
import torch
torch.cuda.set_device(0)
for mb in [36, 71, 142, 284, 1140]:
    n = mb * 1024 * 1024 // 4
    a = torch.randn(n, device='cuda'); b = torch.empty_like(a)
    flush = torch.empty(512 * 1024 * 1024 // 4, device='cuda')
    ts = []
    for i in range(12):
        flush.zero_()
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record(); b.copy_(a); e1.record(); torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    ts.sort(); t = ts[len(ts)//2]
    print(f"{mb} MB copy: {t*1e3:.1f} us, {2*mb*1.048576e6/(t*1e-3)/1e9:.0f} GB/s")
