"""A few rs_sample_wor calls at N = 2^50 for the sweep's middle sizes (for an
ncu launch list): n = 2^22, 2^24, 2^26, 2^28."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import paper_1610_05141_b200 as rs  # noqa: E402

N = 2 ** 50
for e in [int(x) for x in (sys.argv[1:] or ["22", "24", "26", "28"])]:
    n = 2 ** e
    out = torch.empty(n, dtype=torch.uint64, device="cuda")
    ws = torch.empty(rs.workspace_bytes(rs.MODE_WOR, N, n), dtype=torch.uint8, device="cuda")
    for r in range(3):
        rs.sample_wor_ws(N, n, r, 1, 0, out, ws)
    torch.cuda.synchronize()
    del out, ws
print("ok")
