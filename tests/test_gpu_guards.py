"""Out-of-bounds writes: guard regions around the output and the workspace;
-m gpu.

compute-sanitizer is closed on the GPU pool, so memory safety of the global
stores is checked from the outside: every call writes into a view of a
larger buffer whose guard regions (and, for the workspace variants, the
workspace's own guards) hold a pattern that must survive the call; the view
starts at every offset mod 4 (the warp kernels' 32-byte store grid starts h
= 0..3 elements before the first value), and the output is then compared
with the oracle (every position written, none twice).  Paths: 32-bit warp
leaves (power-of-two / Lemire / top-up / complement bitmap), fused small
trees, wide (u64-range) leaves, the CTA kernels, WR, shards, Bernoulli.
"""
from __future__ import annotations

import numpy as np
import pytest
import torch

import oracle as O
import paper_1610_05141_b200 as rs

pytestmark = pytest.mark.gpu

G = 4096                                   # guard elements on each side
PAT = -0x5A5A5A5A5A5A5A5B                  # 0xA5A5A5A5A5A5A5A5 as int64


def _guarded(n, shift):
    buf = torch.full((G + shift + n + G,), PAT, dtype=torch.int64, device="cuda")
    return buf, buf[G + shift:G + shift + n].view(torch.uint64)


def _guards_intact(buf, shift, n):
    b = buf.cpu().numpy()
    lo, hi = b[:G + shift], b[G + shift + n:]
    return bool((lo == PAT).all() and (hi == PAT).all())


CASES = [(2 ** 30, 2 ** 20), (10 ** 9 + 7, 100003), (2 ** 20, 2 ** 14), (2 ** 24 + 3, 2 ** 16 + 1),
         (2 ** 22, 3 * 2 ** 20), (10 ** 6, 999_000), (2 ** 50, 2 ** 12), (2 ** 45, 2 ** 20), (2 ** 40, 2 ** 22),
         (12345, 6173), (2 ** 15, 2 ** 14), (100, 51)]


@pytest.mark.parametrize("N,n", CASES)
@pytest.mark.parametrize("mode", [0, 1])
def test_output_guards(N, n, mode):
    f = rs.sample_wr if mode else rs.sample_wor
    exp = (O.sample_wr if mode else O.sample_wor)(N, n, 11)
    for shift in range(4):
        buf, out = _guarded(n, shift)
        got = f(N, n, 11, out=out)
        torch.cuda.synchronize()
        assert _guards_intact(buf, shift, n), (N, n, mode, shift)
        assert np.array_equal(got.cpu().numpy(), exp), (N, n, mode, shift)
    assert rs.device_errors(clear=True) == 0


@pytest.mark.parametrize("leaf_path,fused", [(1, 1), (0, 0), (3, 1)])
def test_output_guards_other_paths(leaf_path, fused):
    rs.set_option(rs.OPT_LEAF_PATH, leaf_path)
    rs.set_option(rs.OPT_FUSED, fused)
    try:
        for N, n in [(2 ** 30, 2 ** 20), (2 ** 21, 2 ** 20), (2 ** 48, 2 ** 24)]:
            exp = O.sample_wor(N, n, 12)
            for shift in (1, 3):
                buf, out = _guarded(n, shift)
                got = rs.sample_wor(N, n, 12, out=out)
                torch.cuda.synchronize()
                assert _guards_intact(buf, shift, n), (leaf_path, fused, N, n, shift)
                assert np.array_equal(got.cpu().numpy(), exp)
    finally:
        rs.set_option(rs.OPT_LEAF_PATH, 0)
        rs.set_option(rs.OPT_FUSED, 1)
    assert rs.device_errors(clear=True) == 0


@pytest.mark.parametrize("N,n,world,rank", [(2 ** 34, 2 ** 22, 4, 1), (2 ** 50, 2 ** 20, 8, 7), (2 ** 30, 2 ** 20, 2, 0)])
def test_workspace_and_shard_guards(N, n, world, rank):
    cnt, _ = rs.shard_info(N, n, 13, world, rank)
    wsb = rs.workspace_bytes(rs.MODE_WOR, N, n, world=world)
    wbuf = torch.full((G * 8 + wsb + G * 8,), 0xA5, dtype=torch.uint8, device="cuda")
    ws = wbuf[G * 8:G * 8 + wsb]
    buf, out = _guarded(cnt, 2)
    got = rs.sample_wor_ws(N, n, 13, world, rank, out, ws)
    torch.cuda.synchronize()
    assert _guards_intact(buf, 2, cnt)
    w = wbuf.cpu().numpy()
    assert (w[:G * 8] == 0xA5).all() and (w[G * 8 + wsb:] == 0xA5).all()
    ref = rs.sample_wor_shard(N, n, 13, world, rank)
    assert torch.equal(got, ref)
    assert rs.device_errors(clear=True) == 0


@pytest.mark.parametrize("N,rho", [(2 ** 24, 0.01), (2 ** 32, 1e-4), (10 ** 6 + 17, 0.3), (2 ** 40 + 3, 1e-9)])
def test_bernoulli_guards(N, rho):
    cap = rs.bernoulli_capacity(N, rho)
    buf, out = _guarded(cap, 1)
    o, cnt = rs.bernoulli(N, rho, 14, out=out, return_count=True)
    torch.cuda.synchronize()
    c = int(cnt.item())
    assert c <= cap
    assert _guards_intact(buf, 1, cap)
    exp = O.bernoulli(N, rho, 14)
    assert np.array_equal(o[:c].cpu().numpy(), exp)
    # positions between the count and the capacity are not written either
    b = buf.cpu().numpy()
    assert (b[G + 1 + c:G + 1 + cap] == PAT).all()
    assert rs.device_errors(clear=True) == 0
