"""Whole-output parity at BASELINE's full sizes; -m gpu.

north_star asks for bit-exact agreement with the oracle "on every config and
seed".  Outputs of 8-32 GiB cannot be compared element by element on the host,
so both sides reduce the WHOLE output to the order-sensitive, shard-composable
digest sum_i mix64(i ^ mix64(v_i)) ("GPU vs oracle" row): the
device digest (rs.digest, a librs kernel over the device output) against the
oracle's streaming digest of every leaf (O.digest_range: the oracle's own tree,
leaves and complement, threaded over leaves; O.bern_digest: every Bernoulli
chunk, threaded over chunks).  A single wrong value anywhere changes the
digest (mix64 is a bijection; a collision needs ~2^64 tries).

Shards (Algorithm P; p-independence P:513-520): the per-rank
digests at their global offsets must sum to the p = 1 digest, for p = 2, 4, 8
at n = 2^33 of N = 2^48 (BASELINE configs[2]'s identity check at the largest
p = 1 size that fits one 180 GB B200), and the p = 1 digest equals the
oracle's.
"""
from __future__ import annotations

import pytest
import torch

import oracle as O
import paper_1610_05141_b200 as rs
from paper_1610_05141_b200 import workloads as W

pytestmark = pytest.mark.gpu

MASK = 2 ** 64 - 1


def _free(*ts):
    for t in ts:
        del t
    torch.cuda.synchronize()
    torch.cuda.empty_cache()


def _wor_digest(N, n, seed, mode):
    out = rs.sample_wr(N, n, seed) if mode == O.MODE_WR else rs.sample_wor(N, n, seed)
    torch.cuda.synchronize()
    assert out.numel() == n
    assert rs.validate(out, N, strict=(mode == O.MODE_WOR)) == 0
    d = rs.digest(out)
    assert rs.device_errors(clear=True) == 0
    del out
    torch.cuda.empty_cache()
    return d


@pytest.mark.parametrize("cfg,seed", [("HEADLINE", 1), ("HEADLINE", 2 ** 64 - 1)] +
                         [("CFG1", s) for s in W.PARITY_SEEDS])
def test_fullsize_wor_digest(cfg, seed):
    c = getattr(W, cfg)
    N, n = c["N"], c["n"]
    assert _wor_digest(N, n, seed, O.MODE_WOR) == O.digest_range(N, n, seed, O.MODE_WOR)


@pytest.mark.parametrize("seed", W.PARITY_SEEDS)
def test_fullsize_complement_digest(seed):
    c = W.CFG3A
    N, n = c["N"], c["n"]
    assert _wor_digest(N, n, seed, O.MODE_WOR) == O.digest_range(N, n, seed, O.MODE_WOR)


@pytest.mark.parametrize("seed", [1, 2 ** 64 - 1])
def test_fullsize_wr_digest(seed):
    c = W.CFG4
    N, n = c["N"], c["n"]
    assert _wor_digest(N, n, seed, O.MODE_WR) == O.digest_range(N, n, seed, O.MODE_WR)


@pytest.mark.parametrize("cfg,seed", [("CFG3B", s) for s in W.PARITY_SEEDS] +
                         [("CFG3B_ROOF", 1), ("CFG3B_ROOF", 2 ** 64 - 1)])
def test_fullsize_bernoulli_digest(cfg, seed):
    c = getattr(W, cfg)
    N, rho = c["N"], c["rho"]
    out = rs.bernoulli(N, rho, seed)
    torch.cuda.synchronize()
    d_gpu, cnt = rs.digest(out), out.numel()
    assert rs.validate(out, N, strict=True) == 0
    del out
    torch.cuda.empty_cache()
    d_or, cnt_or = O.bern_digest(N, rho, seed)
    assert cnt == cnt_or
    assert d_gpu == d_or


def test_shards_p248_digest_n2_33():
    N, n, seed = 2 ** 48, 2 ** 33, 1
    d1 = _wor_digest(N, n, seed, O.MODE_WOR)
    for world in (2, 4, 8):
        tot = 0
        for rank in range(world):
            cnt, off = rs.shard_info(N, n, seed, world, rank)
            part = rs.sample_wor_shard(N, n, seed, world, rank)
            assert part.numel() == cnt
            tot = (tot + rs.digest(part, base_index=off)) & MASK
            del part
            torch.cuda.empty_cache()
        assert tot == d1, world
    assert d1 == O.digest_range(N, n, seed, O.MODE_WOR)
