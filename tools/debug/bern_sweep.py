"""Bernoulli throughput vs rho at ~2^31 expected outputs (dev tool)."""
import sys, os, torch
sys.path.insert(0, os.getcwd())
import paper_1610_05141_b200 as rs

target = 2 ** 31
for rho in [0.5, 0.1, 0.01, 2 ** -10, 1e-4, 2 ** -16, 1e-6, 1e-8]:
    N = min(int(target / rho), 2 ** 62)
    cap = rs.bernoulli_capacity(N, rho)
    out = torch.empty(cap, dtype=torch.uint64, device="cuda")
    cnt = torch.zeros(1, dtype=torch.uint64, device="cuda")
    ws = torch.empty(rs.workspace_bytes(rs.MODE_BERNOULLI, N, 0, rho, 1), dtype=torch.uint8, device="cuda")
    for _ in range(2):
        rs.bernoulli_ws(N, rho, 1, 1, 0, out, cap, cnt, ws)
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    torch.cuda.synchronize(); e0.record()
    for _ in range(5):
        rs.bernoulli_ws(N, rho, 1, 1, 0, out, cap, cnt, ws)
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 5
    c = int(cnt.item())
    D = rs.plan(rs.MODE_BERNOULLI, N, 0, rho)[0]
    print(f"rho={rho:<10.3g} N=2^{N.bit_length()-1:<3} chunkr=2^{(N >> D).bit_length()-1:<3} count={c:.3e} "
          f"{ms:8.2f} ms  {c / ms / 1e6:8.3g} G/s  {8 * c / ms / 1e6:7.0f} GB/s", flush=True)
    del out, ws
