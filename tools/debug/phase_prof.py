"""Dev: per-phase cycle split of the warp leaf kernel (needs an RS_EXP_CLOCK build in RS_LIB)."""
import ctypes as C
import sys
import torch
import paper_1610_05141_b200 as rs
N, n = int(sys.argv[1]), int(sys.argv[2])
L = rs.lib()
buf = (C.c_ulonglong * 8)()
out = torch.empty(n, dtype=torch.uint64, device="cuda")
for i in range(3):
    rs.sample_wor(N, n, 1, out=out)
torch.cuda.synchronize()
L.rs_debug_prof(buf, 1)
rs.sample_wor(N, n, 1, out=out)
torch.cuda.synchronize()
L.rs_debug_prof(buf, 1)
names = ["count-loop", "scan", "scatter", "finish:clear+load+sort", "finish:dedup", "finish total"]
tot = sum(buf[i] for i in (0, 1, 2, 5))
for i, nm in enumerate(names):
    print(f"{nm:26s} {buf[i]:16d} {buf[i] / tot * 100:6.1f}%")
leaves = n / 1024
print("cycles per leaf per warp:", tot / leaves)
