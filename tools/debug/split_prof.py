"""Per-level split cycles (librs built with -DRS_SPLIT_PROF, via RS_LIB) for a
few small-n calls."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import paper_1610_05141_b200 as rs  # noqa: E402

N = 2 ** 50
for e in [int(x) for x in (sys.argv[1:] or ["10", "16"])]:
    n = 2 ** e
    out = torch.empty(n, dtype=torch.uint64, device="cuda")
    ws = torch.empty(rs.workspace_bytes(rs.MODE_WOR, N, n), dtype=torch.uint8, device="cuda")
    for r in range(4):
        print(f"# n=2^{e} seed {r}", flush=True)
        rs.sample_wor_ws(N, n, r, 1, 0, out, ws)
        torch.cuda.synchronize()
