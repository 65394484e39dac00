"""Raw device->pinned-host copy bandwidth (the e2e ceiling), dev tool."""
import time, torch
for gb in (1, 4):
    n = gb * 2 ** 27
    d = torch.empty(n, dtype=torch.int64, device="cuda")
    h = torch.empty(n, dtype=torch.int64, pin_memory=True)
    h.copy_(d, non_blocking=True); torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(5):
        h.copy_(d, non_blocking=True)
    torch.cuda.synchronize()
    dt = (time.perf_counter() - t) / 5
    print(f"D2H {gb} GiB: {8 * n / dt / 1e9:.1f} GB/s", flush=True)
    t = time.perf_counter()
    for _ in range(5):
        d.copy_(h, non_blocking=True)
    torch.cuda.synchronize()
    dt = (time.perf_counter() - t) / 5
    print(f"H2D {gb} GiB: {8 * n / dt / 1e9:.1f} GB/s", flush=True)
