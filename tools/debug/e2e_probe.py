"""Where the e2e time goes: raw chunked D2H into one big pinned buffer vs
rs_sample_shard_host at several sizes (dev tool)."""
import os, sys, time, torch
sys.path.insert(0, os.getcwd())
import paper_1610_05141_b200 as rs

n = 2 ** 32
h = torch.empty(n, dtype=torch.uint64, pin_memory=True)
d = torch.empty(2 ** 27, dtype=torch.uint64, device="cuda")
for rep in range(2):
    torch.cuda.synchronize(); t = time.perf_counter()
    for i in range(n // 2 ** 27):
        h[i * 2 ** 27:(i + 1) * 2 ** 27].copy_(d, non_blocking=True)
    torch.cuda.synchronize(); dt = time.perf_counter() - t
    print(f"raw chunked D2H 32 GiB: {8 * n / dt / 1e9:.1f} GB/s", flush=True)
for N, m in [(2 ** 48, 2 ** 28), (2 ** 48, 2 ** 30), (2 ** 48, 2 ** 32)]:
    for rep in range(2):
        t = time.perf_counter()
        rs.sample_shard_host(rs.MODE_WOR, N, m, 1, 1, 0, h[:m])
        dt = time.perf_counter() - t
        print(f"shard_host n=2^{m.bit_length()-1}: {dt*1e3:.1f} ms  {8 * m / dt / 1e9:.1f} GB/s", flush=True)
