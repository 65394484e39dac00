"""A few rs_sample_wor calls at small n (for an ncu launch list of the small-n path)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import paper_1610_05141_b200 as rs  # noqa: E402

N = 2 ** 50
for e in (10, 14, 18):
    n = 2 ** e
    out = torch.empty(n, dtype=torch.uint64, device="cuda")
    ws = torch.empty(rs.workspace_bytes(rs.MODE_WOR, N, n), dtype=torch.uint8, device="cuda")
    for r in range(5):
        rs.sample_wor_ws(N, n, r, 1, 0, out, ws)
    torch.cuda.synchronize()
print("ok")
