"""Dev tool: first mismatching leaves between the CUDA path and the oracle."""
import sys
import numpy as np
import oracle as O
import paper_1610_05141_b200 as rs

N, n, seed = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
got = rs.sample_wor(N, n, seed).cpu().numpy()
exp = O.sample_wor(N, n, seed)
print("equal:", np.array_equal(got, exp), "errors", rs.device_errors(clear=True))

print("plan", O.plan(N, n))
D = O.plan(N, n)[0]
L = 1 << D
bad = np.nonzero(got != exp)[0]
print("mismatches", len(bad), "first", bad[:10])
# leaf boundaries from the oracle's values
lo = np.array([O.node(N, D, i)[0] for i in range(L)], dtype=np.uint64)
leaf_of = np.searchsorted(lo, exp - 1, side="right") - 1
bl = np.unique(leaf_of[bad])
print("bad leaves", len(bl), bl[:10])
for i in bl[:3]:
    idx = np.nonzero(leaf_of == i)[0]
    e = exp[idx] - 1 - lo[i]
    g = got[idx] - 1 - lo[i]
    k = len(idx)
    print(f"leaf {i} k={k} r={O.node(N, D, i)[1]}")
    d = np.nonzero(e != g)[0]
    print("  diff pos", d[:20], "n", len(d))
    print("  exp", e[d[:8]], "\n  got", g[d[:8]])
    print("  got sorted?", bool(np.all(np.diff(g.astype(np.int64)) > 0)), "set equal?", set(e.tolist()) == set(g.tolist()))
    ge = set(g.tolist()); ee = set(e.tolist())
    print("  missing", sorted(ee - ge)[:10], "extra", sorted(ge - ee)[:10])
