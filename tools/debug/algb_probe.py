"""Where Algorithm B's step time goes (dev tool): wall time per call, device
time per kernel class, with and without a caller workspace."""
import os, sys, time, torch
sys.path.insert(0, os.getcwd())
import paper_1610_05141_b200 as rs

N, n = 2 ** 48, 2 ** 32
out = torch.empty(n, dtype=torch.uint64, device="cuda")
ws = torch.empty(rs.algb_workspace_bytes(N, n), dtype=torch.uint8, device="cuda")
for rep in range(6):
    rs.timing_enable(True); rs.timing_read(reset=True)
    torch.cuda.synchronize(); t = time.perf_counter()
    _, att = rs.sample_wor_algb(N, n, 1, out=out, ws=ws, return_attempts=True)
    torch.cuda.synchronize(); dt = time.perf_counter() - t
    kt = rs.timing_read(reset=True); rs.timing_enable(False)
    print(f"rep {rep}: wall {dt*1e3:.1f} ms  attempts {att}  " + "  ".join(f"{k} {v[0]:.2f}" for k, v in kt.items()), flush=True)
