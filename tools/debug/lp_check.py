"""Dev check of the ordered linear-probing leaf kernels: parity with the oracle
on a few shapes, then leaf-kernel time vs the counting-sort warp kernel
(RS_OPT_LEAF_PATH = 2) at the headline / cfg1 / WR shapes."""
import sys, time
import numpy as np
import torch
sys.path.insert(0, '.')
import oracle as O
import paper_1610_05141_b200 as rs

cases = [(2**30, 2**20, 1), (2**40, 2**22, 3), (10**9 + 7, 100003, 1), (2**33 + 12345, 300001, 2),
         (2**21, 2**20, 1), (2**24 + 3, 2**16 + 1, 5), (2**20, 2**14, 7), (3**30, 2**18 + 17, 1)]
for N, n, s in cases:
    for mode in ("wor", "wr"):
        got = (rs.sample_wr if mode == "wr" else rs.sample_wor)(N, n, s).cpu().numpy()
        exp = (O.sample_wr if mode == "wr" else O.sample_wor)(N, n, s)
        ok = np.array_equal(got, exp)
        print(mode, N, n, s, "OK" if ok else f"MISMATCH at {np.flatnonzero(got != exp)[:5]}", flush=True)
print("device errors", rs.device_errors(clear=True))

def leaf_ms(mode, N, n, path, reps=5):
    rs.set_option(rs.OPT_LEAF_PATH, path)
    m = rs.MODE_WR if mode == "wr" else rs.MODE_WOR
    out = torch.empty(n, dtype=torch.uint64, device="cuda")
    ws = torch.empty(rs.workspace_bytes(m, N, n), dtype=torch.uint8, device="cuda")
    f = rs.sample_wr_ws if mode == "wr" else rs.sample_wor_ws
    for _ in range(2):
        f(N, n, 1, 1, 0, out, ws)
    torch.cuda.synchronize()
    rs.timing_enable(True); rs.timing_read(reset=True)
    for _ in range(reps):
        f(N, n, 1, 1, 0, out, ws)
    torch.cuda.synchronize()
    kt = rs.timing_read(reset=True); rs.timing_enable(False)
    d = rs.digest(out)
    rs.set_option(rs.OPT_LEAF_PATH, 0)
    return kt["leaf"][0] / reps, kt["split"][0] / reps, d

for mode, N, n in [("wor", 2**48, 2**32), ("wor", 2**40, 2**30), ("wr", 2**36, 2**32), ("wor", 2**48, 2**30)]:
    a = leaf_ms(mode, N, n, 0)
    b = leaf_ms(mode, N, n, 2)
    print(f"{mode} N={N} n={n}: LP leaf {a[0]:.3f} ms  old leaf {b[0]:.3f} ms  split {a[1]:.3f} ms  digest equal {a[2] == b[2]}", flush=True)
print("device errors", rs.device_errors(clear=True))
