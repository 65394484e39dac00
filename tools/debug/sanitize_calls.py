"""Small calls of every path for compute-sanitizer (memcheck / racecheck):
warp leaves (32-bit, power-of-two and Lemire, top-up), fused small trees,
wide leaves, bitmap / complement leaves, the CTA spill kernel, WR, Bernoulli,
shards.  Sizes kept small: the tools slow kernels down 10-100x."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import paper_1610_05141_b200 as rs  # noqa: E402

cases = [(2 ** 30, 2 ** 20), (10 ** 9 + 7, 100003), (2 ** 50, 2 ** 12), (2 ** 22, 3 * 2 ** 20), (2 ** 20, 2 ** 14),
         (2 ** 40, 2 ** 22), (1000, 999), (2 ** 45, 2 ** 18)]
for N, n in cases:
    rs.sample_wor(N, n, 1)
    rs.sample_wr(N, n, 1)
rs.set_option(rs.OPT_LEAF_PATH, 1)
rs.sample_wor(2 ** 30, 2 ** 18, 2)
rs.set_option(rs.OPT_LEAF_PATH, 0)
rs.set_option(rs.OPT_FUSED, 0)
rs.sample_wor(2 ** 30, 2 ** 20, 3)
rs.set_option(rs.OPT_FUSED, 1)
rs.bernoulli(2 ** 24, 0.01, 4)
rs.bernoulli(2 ** 32, 1e-4, 5)
rs.sample_wor_shard(2 ** 34, 2 ** 22, 6, 4, 1)
torch.cuda.synchronize()
print("sanitize calls ok", rs.device_errors(clear=True))
