"""GPU box: read-only streaming rate of torch reductions at the matvec's sizes (context for the
dense matvec's fraction of the copy peak)."""
import torch
for mb in (537, 2215, 8000):
    a = torch.empty(mb * 1024 * 1024 // 8, dtype=torch.float64, device="cuda").uniform_()
    for _ in range(3):
        a.sum()
    ev = []
    for _ in range(20):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); a.sum(); e1.record(); torch.cuda.synchronize(); ev.append(e0.elapsed_time(e1))
    ev.sort()
    ms = ev[len(ev) // 2]
    print("torch.sum over %d MB: %.4f ms = %.0f GB/s" % (mb, ms, a.numel() * 8 / ms / 1e6), flush=True)
    del a
