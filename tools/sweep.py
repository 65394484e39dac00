"""The paper-shaped sweep: rs_sample_wor at
N = 2^50 for n = 2^10 .. 2^32 (powers of 4), device time per call by CUDA
events over repeated calls (reps ~ 2^30 / n, capped), output resident in
HBM.  Prints one line per n: time per call, ns per sample, samples/s; then
the same calls captured in a CUDA graph (device time without the host's
per-call launch cost: Python marshalling + 4-5 launches)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1610_05141_b200 as rs  # noqa: E402

N = 2 ** 50
print(f"# rs_sample_wor, N = 2^50, one B200, CUDA events ({torch.cuda.get_device_name()})")
print(f"# {'n':>8} {'reps':>6} {'us/call':>10} {'ns/sample':>10} {'samples/s':>10}  D  {'graph us/call':>13} {'graph samples/s':>15}")
for e in ([int(x) for x in sys.argv[1:]] or range(10, 33, 2)):
    n = 2 ** e
    out = torch.empty(n, dtype=torch.uint64, device="cuda")
    ws = torch.empty(rs.workspace_bytes(rs.MODE_WOR, N, n), dtype=torch.uint8, device="cuda")
    reps = max(3, min(2000, 2 ** 30 // n))
    for _ in range(3):
        rs.sample_wor_ws(N, n, 1, 1, 0, out, ws)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    for r in range(reps):
        rs.sample_wor_ws(N, n, r, 1, 0, out, ws)
    e1.record()
    torch.cuda.synchronize()
    us = e0.elapsed_time(e1) * 1e3 / reps
    D = rs.plan(rs.MODE_WOR, N, n)[0]
    # graph: G calls (seeds 0..G-1) captured once, replayed
    G = min(reps, 100)
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            for r in range(G):
                rs.sample_wor_ws(N, n, r, 1, 0, out, ws)
    torch.cuda.current_stream().wait_stream(s)
    g.replay()
    torch.cuda.synchronize()
    R = max(1, reps // G)
    e0.record()
    for _ in range(R):
        g.replay()
    e1.record()
    torch.cuda.synchronize()
    gus = e0.elapsed_time(e1) * 1e3 / (R * G)
    del g
    print(f"  2^{e:<6} {reps:>6} {us:>10.1f} {us * 1e3 / n:>10.3f} {n / us * 1e6:>10.3g}  {D}  {gus:>13.1f} {n / gus * 1e6:>15.3g}",
          flush=True)
    del out, ws
    torch.cuda.empty_cache()
