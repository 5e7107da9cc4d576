"""GPU box: device->host copy rate into pinned memory with 1, 2, 4 concurrent streams (copy engines)."""
import time
import torch
nbytes = 536_870_912
src = torch.empty(nbytes // 8, dtype=torch.float64, device="cuda").fill_(1.0)
dst = torch.empty(nbytes // 8, dtype=torch.float64, pin_memory=True)
for ns in (1, 2, 4, 8):
    streams = [torch.cuda.Stream() for _ in range(ns)]
    chunks = torch.chunk(torch.arange(src.numel()), ns)
    for rep in range(3):
        torch.cuda.synchronize(); t0 = time.perf_counter()
        per = src.numel() // ns
        for k, st in enumerate(streams):
            with torch.cuda.stream(st):
                a = k * per; b = src.numel() if k == ns - 1 else (k + 1) * per
                dst[a:b].copy_(src[a:b], non_blocking=True)
        torch.cuda.synchronize(); dt = time.perf_counter() - t0
    print("streams %d: %.2f ms = %.1f GB/s" % (ns, dt * 1e3, nbytes / dt / 1e9), flush=True)
