"""Dev check of the wide-range warp leaf kernels: parity with the oracle on
wide shapes (r > 2^32), then the paper-shaped sweep's wide points."""
import sys, time
import numpy as np
import torch
sys.path.insert(0, '.')
import oracle as O
import paper_1610_05141_b200 as rs

cases = [(2**50, 2**12, 1), (2**45, 2**20, 3), (2**62 + 11, 5000, 1), (2**63 - 1, 77777, 2),
         (2**50, 2**22, 5), (2**44 + 12345, 2**18, 7), (2**40, 2**8, 1), (2**36 + 1, 16, 1)]
for N, n, s in cases:
    for mode in ("wor", "wr"):
        got = (rs.sample_wr if mode == "wr" else rs.sample_wor)(N, n, s).cpu().numpy()
        exp = (O.sample_wr if mode == "wr" else O.sample_wor)(N, n, s)
        ok = got.shape == exp.shape and np.array_equal(got, exp)
        print(mode, N, n, s, "OK" if ok else f"MISMATCH {np.flatnonzero(got != exp)[:5]}", flush=True)
print("device errors", rs.device_errors(clear=True))
N = 2**50
for e in (24, 26, 28):
    n = 2**e
    out = torch.empty(n, dtype=torch.uint64, device="cuda")
    ws = torch.empty(rs.workspace_bytes(rs.MODE_WOR, N, n), dtype=torch.uint8, device="cuda")
    for _ in range(3): rs.sample_wor_ws(N, n, 1, 1, 0, out, ws)
    torch.cuda.synchronize()
    rs.timing_enable(True); rs.timing_read(reset=True)
    reps = 5
    for r in range(reps): rs.sample_wor_ws(N, n, r, 1, 0, out, ws)
    torch.cuda.synchronize()
    kt = rs.timing_read(reset=True); rs.timing_enable(False)
    d = rs.digest(out); do = O.digest_range(N, n, reps - 1) if e <= 26 else None
    print(f"n=2^{e}: leaf {kt['leaf'][0]/reps:.3f} ms split {kt['split'][0]/reps:.3f} ms  "
          f"{n/((kt['leaf'][0]+kt['split'][0])/reps*1e-3)/1e9:.1f} G/s  digest==oracle {d == do if do else 'skip'}", flush=True)
print("device errors", rs.device_errors(clear=True))
