import sys; sys.path.insert(0, '.')
import torch, paper_1610_05141_b200 as rs
N, n = int(eval(sys.argv[1])), int(eval(sys.argv[2]))
out = torch.empty(n, dtype=torch.uint64, device="cuda")
ws = torch.empty(rs.workspace_bytes(rs.MODE_WOR, N, n), dtype=torch.uint8, device="cuda")
for r in range(3): rs.sample_wor_ws(N, n, r, 1, 0, out, ws)
torch.cuda.synchronize(); print("ok")
