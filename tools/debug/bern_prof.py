import sys; sys.path.insert(0, '.')
import torch, paper_1610_05141_b200 as rs
N, rho = 2**38, 0.01
cap = rs.bernoulli_capacity(N, rho)
out = torch.empty(cap, dtype=torch.uint64, device="cuda")
cnt = torch.zeros(1, dtype=torch.uint64, device="cuda")
ws = torch.empty(rs.workspace_bytes(rs.MODE_BERNOULLI, N, 0, rho, 1), dtype=torch.uint8, device="cuda")
for _ in range(2): rs.bernoulli_ws(N, rho, 1, 1, 0, out, cap, cnt, ws)
torch.cuda.synchronize(); print("ok", int(cnt.item()))
