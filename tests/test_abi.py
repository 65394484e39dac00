"""C-ABI checks that need no GPU (-m "not gpu").

* librs.so loads and exports every symbol include/rs.h declares.
* The host-side planning and Algorithm P replay of librs (rs_plan,
  rs_shard_info -- compiled from csrc/rs_math.cuh by nvcc's host compiler)
  agree bit-exactly with the independent oracle.
* Without a CUDA device every compute call fails loudly (no CPU fallback).
"""
from __future__ import annotations

import ctypes
import os
import re

import pytest

import oracle as O
import paper_1610_05141_b200 as rs

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    src = open(os.path.join(ROOT, "include", "rs.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(rs_[a-z0-9_]+)\s*\(", src)))


def test_header_symbols_exported():
    names = _declared()
    assert len(names) >= 20
    L = rs.lib()
    for n in names:
        assert hasattr(L, n), n
    # the binding mirrors the header exactly
    assert set(names) == set(rs.SIGNATURES)


def test_version_and_status_strings():
    assert b"CANON v1" in rs.lib().rs_version()
    assert rs.lib().rs_status_string(1) == b"invalid argument"


@pytest.mark.parametrize("N,n", [(2 ** 30, 2 ** 20), (2 ** 40, 2 ** 30), (2 ** 48, 2 ** 32),
                                 (2 ** 32, 3 * 2 ** 30), (100, 50), (100, 51), (5, 0), (1, 1)])
def test_plan_matches_oracle(N, n):
    assert rs.plan(rs.MODE_WOR, N, n) == O.plan(N, n, O.MODE_WOR)
    assert rs.plan(rs.MODE_WR, N, n)[0] == O.plan(N, n, O.MODE_WR)[0]


@pytest.mark.parametrize("N,rho", [(2 ** 32, 0.01), (2 ** 38, 0.01), (1000, 0.5), (10, 1e-9)])
def test_bernoulli_depth_matches_oracle(N, rho):
    assert rs.plan(rs.MODE_BERNOULLI, N, 0, rho)[0] == O.bern_depth(N, rho)


SHARD_CASES = [(2 ** 48, 2 ** 32, 1), (2 ** 48, 2 ** 33, 7), (2 ** 40, 2 ** 30, 0xDEADBEEF),
               (2 ** 36, 2 ** 32, 3), (2 ** 32, 3 * 2 ** 30, 5), (10 ** 12 + 39, 123456789, 11),
               (1000, 999, 2), (7, 3, 2 ** 64 - 1)]


@pytest.mark.parametrize("N,n,seed", SHARD_CASES)
@pytest.mark.parametrize("mode", [rs.MODE_WOR, rs.MODE_WR])
def test_shard_replay_bit_exact_with_oracle(N, n, seed, mode):
    """Algorithm P path replay (<= 3 deviates per rank) on librs's
    host side equals the oracle's for every rank of p = 2, 4, 8."""
    for world in (1, 2, 4, 8):
        tot = 0
        for rank in range(world):
            got = rs.shard_info(N, n, seed, world, rank, mode)
            assert got == O.shard_info(N, n, seed, world, rank, mode), (world, rank)
            assert got[1] == tot
            tot += got[0]
        assert tot == n


def test_argument_errors():
    with pytest.raises(rs.RSError):
        rs.shard_info(10, 11, 0, 1, 0)          # n > N
    with pytest.raises(rs.RSError):
        rs.shard_info(2 ** 63, 1, 0, 1, 0)      # N >= 2^63
    with pytest.raises(rs.RSError):
        rs.shard_info(100, 5, 0, 3, 0)          # world not a power of two
    with pytest.raises(rs.RSError):
        rs.plan(rs.MODE_BERNOULLI, 100, 0, 1.5)
    with pytest.raises(rs.RSError):
        rs.plan(rs.MODE_BERNOULLI, 100, 0, float("nan"))


def test_capacity_formula():
    assert rs.bernoulli_capacity(2 ** 32, 0.01) >= 2 ** 32 * 0.01 + 10 * (2 ** 32 * 0.01 * 0.99) ** 0.5
    assert rs.bernoulli_capacity(100, 1.0) == 100
    assert rs.bernoulli_capacity(100, 0.0) == 0


def test_no_cpu_fallback():
    import torch
    if torch.cuda.is_available():
        pytest.skip("has a GPU")
    with pytest.raises(rs.RSError):
        rs.sample_wor(100, 10, 1)
    # the raw C call reports RS_ECUDA rather than computing anything
    st = rs.lib().rs_sample_wor(100, 10, 1, ctypes.c_void_p(0), ctypes.c_void_p(0))
    assert st == 2


def test_set_option_host_only():
    rs.set_option(rs.OPT_LEAF_PATH, 1)
    rs.set_option(rs.OPT_LEAF_PATH, 0)
    rs.set_option(rs.OPT_TOPUP_MAX, 0)
    rs.set_option(rs.OPT_TOPUP_MAX, 32)
    rs.set_option(rs.OPT_FUSED, 0)
    rs.set_option(rs.OPT_FUSED, 1)
    rs.set_option(rs.OPT_WARP_CAP, 900)
    rs.set_option(rs.OPT_WARP_CAP, 0)
    with pytest.raises(rs.RSError):
        rs.set_option(rs.OPT_WARP_CAP, 5000)
    with pytest.raises(rs.RSError):
        rs.set_option(rs.OPT_TOPUP_MAX, 33)
    with pytest.raises(rs.RSError):
        rs.set_option(99, 0)
    with pytest.raises(rs.RSError):
        rs.set_option(rs.OPT_LEAF_PATH, 7)


def test_leaf_range_nodes_partition():
    for D in (3, 5, 8):
        for lo in range(0, 1 << D, 3):
            for hi in range(lo, (1 << D) + 1, 5):
                nodes = rs.leaf_range_nodes(D, lo, hi)
                cur = lo
                for d, i in nodes:
                    assert 0 <= d <= D and 0 <= i < (1 << d)
                    assert i << (D - d) == cur          # aligned and contiguous
                    cur += 1 << (D - d)
                assert cur == hi


@pytest.mark.parametrize("N,n,mode", [(2 ** 30, 2 ** 20, 0), (2 ** 48, 2 ** 32, 0), (2 ** 36, 2 ** 32, 1),
                                      (2 ** 32, 3 * 2 ** 30, 0), (10 ** 9 + 7, 100003, 0)])
def test_node_info_matches_oracle_replay(N, n, mode):
    """rs_node_info (librs host replay) vs the oracle's independent replay
    (rso_path) for nodes at every depth down to the leaves."""
    D, comp, m = O.plan(N, n, mode)
    wr = mode == 1
    for d in sorted(set([0, 1, 3, min(D, 7), D])):
        for i in sorted(set([0, (1 << d) - 1, (1 << d) // 3])):
            cnt, off = rs.node_info(mode, N, n, 1, d, i)
            c, o = O.path(N, m, 1, d, i, wr)
            if comp:
                lo, R, _ = O.node(N, d, i)
                c, o = R - c, lo - o
            assert (cnt, off) == (c, o), (d, i)
    with pytest.raises(rs.RSError):
        rs.node_info(mode, N, n, 1, D + 1, 0)
    with pytest.raises(rs.RSError):
        rs.node_info(mode, N, n, 1, 2, 4)


@pytest.mark.parametrize("L,n", [([17, 3, 40, 0, 25, 9, 11, 30, 14, 22, 8, 31, 19], 50),
                                 ([2 ** 40, 5, 3 * 2 ** 33, 2 ** 20], 2 ** 30), ([7], 3),
                                 ([1, 2, 3, 4, 5, 6, 7, 8], 36), ([0, 0, 5], 2)])
def test_uneven_counts_match_oracle(L, n):
    for seed in (1, 2 ** 64 - 1, 12345):
        assert rs.uneven_counts(L, n, seed) == [int(v) for v in O.uneven_counts(L, n, seed)]
    for i in range(len(L)):
        assert rs.uneven_seed(seed, i) == O.uneven_seed(seed, i)
    with pytest.raises(rs.RSError):
        rs.uneven_counts(L, sum(L) + 1, 1)
