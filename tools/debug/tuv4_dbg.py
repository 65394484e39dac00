# locate leaves whose device output differs from the oracle at cfg1 (debug aid)
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np, torch
import oracle as O
import paper_1610_05141_b200 as rs
N, n, seed = 2 ** 40, 2 ** 30, 1
out = rs.sample_wor(N, n, seed); torch.cuda.synchronize()
a = out.cpu().numpy()
bad = np.flatnonzero(np.diff(a.astype(np.int64)) <= 0)
print("bad pairs", len(bad), bad[:10])
D = O.plan(N, n, O.MODE_WOR)[0]
seen = set()
for b in bad[:6]:
    for idx in (b, b + 1):
        L = int((int(a[idx]) - 1) >> (40 - D))
        if L in seen or L >= (1 << D): continue
        seen.add(L)
        vals, off = O.leaf(N, n, seed, L, O.MODE_WOR)
        got = a[off: off + len(vals)]
        d = np.flatnonzero(got != vals)
        print("leaf", L, "off", off, "k", len(vals), "h", off & 3, "ndiff", len(d), "at", d[:8])
        for j in d[:4]:
            print("   j", j, "got", got[j], "exp", vals[j], "exp nbrs", vals[max(0, j-2): j+3], "got nbrs", got[max(0, j-2): j+3])
