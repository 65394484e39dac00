import sys
import numpy as np
import oracle as O
import paper_1610_05141_b200 as rs
V, m = int(sys.argv[1]), int(sys.argv[2])
got = rs.gnm(V, m, 13).cpu().numpy()
exp = O.gnm(V, m, 13)
bad = np.nonzero(got != exp)[0]
print("bad", len(bad), bad[:20])
raw = O.sample_wor(V * (V - 1) // 2, m, 13)
for i in bad[:8]:
    g, e = int(got[i]), int(exp[i])
    print(i, raw[i], "got", g >> 32, g & 0xffffffff, "exp", e >> 32, e & 0xffffffff)
