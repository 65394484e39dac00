"""GPU parity: the CUDA path (through the C ABI) vs the oracle, element by
element on the same (N, n, seed); -m gpu.

Bar: integer output, so bit-exact everywhere.  Small
and medium cases compare every element; full BASELINE sizes compare sampled
leaves the oracle replays one by one (Algorithm P path replay) plus
properties that hold at any size (count, strictly increasing, in range).
"""
from __future__ import annotations

import numpy as np
import pytest
import torch

import oracle as O
import paper_1610_05141_b200 as rs
from paper_1610_05141_b200 import workloads as W

pytestmark = pytest.mark.gpu

SEEDS = [0, 1, 0xDEADBEEF, 2 ** 64 - 1]


def _np(t):
    return t.cpu().numpy()


def _no_device_errors():
    assert rs.device_errors(clear=True) == 0


# ---- without replacement ---------------------------------------------------

@pytest.mark.parametrize("seed", SEEDS)
def test_cfg0_full_compare(seed):
    N, n = W.CFG0["N"], W.CFG0["n"]
    got = _np(rs.sample_wor(N, n, seed))
    exp = O.sample_wor(N, n, seed)
    assert np.array_equal(got, exp)
    _no_device_errors()


WOR_CASES = [
    # tiny / degenerate
    (1, 0), (1, 1), (2, 1), (7, 3), (8, 4), (9, 5), (10, 10), (100, 0), (100, 50), (100, 51),
    (1000, 999), (12345, 6172), (12345, 6173),
    # several tiles and ragged tails, non-power-of-two N (Lemire rejections)
    (10 ** 9 + 7, 100003), (3 ** 30, 2 ** 18 + 17), (2 ** 33 + 12345, 300001),
    # dense leaves: many rounds of first-k-distinct (n = N/2 not complemented)
    (2 ** 21, 2 ** 20), (2 ** 15, 2 ** 14), (3 * 2 ** 14 + 1, 3 * 2 ** 13),
    # top-up regime (leaf ranges 2^16..2^18: several new values per leaf, some leaves > 4)
    (2 ** 20, 2 ** 14), (2 ** 21 + 99, 2 ** 14 + 5), (2 ** 24 + 3, 2 ** 16 + 1),
    # complement (2n > N), incl. the cfg3a shape at reduced N
    (2 ** 22, 3 * 2 ** 20), (2 ** 20 + 3, 2 ** 20), (10 ** 6, 999_000),
    # leaf ranges above 2^32 (64-bit keys)
    (2 ** 50, 2 ** 12), (2 ** 45, 2 ** 20), (2 ** 62 + 11, 5000), (2 ** 63 - 1, 77777),
    # complement with huge leaves (tiled emission)
    (2 ** 24, 2 ** 24 - 3),
]


@pytest.mark.parametrize("N,n", WOR_CASES)
def test_wor_full_compare(N, n):
    for seed in (1, 0xDEADBEEF):
        got = _np(rs.sample_wor(N, n, seed))
        exp = O.sample_wor(N, n, seed)
        assert got.shape == exp.shape
        assert np.array_equal(got, exp), (N, n, seed, np.flatnonzero(got != exp)[:5])
    _no_device_errors()


# the CTA-per-leaf kernels (the spill path of the warp kernels) on every leaf
CTA_CASES = [(2 ** 30, 2 ** 20), (12345, 6172), (2 ** 22, 3 * 2 ** 20), (2 ** 24, 2 ** 24 - 3),
             (10 ** 9 + 7, 100003), (2 ** 21, 2 ** 20)]


@pytest.mark.parametrize("N,n", CTA_CASES)
def test_wor_cta_path(N, n):
    rs.set_option(rs.OPT_LEAF_PATH, 1)
    try:
        got = _np(rs.sample_wor(N, n, 7))
        gwr = _np(rs.sample_wr(N, n, 7))
    finally:
        rs.set_option(rs.OPT_LEAF_PATH, 0)
    assert np.array_equal(got, O.sample_wor(N, n, 7))
    assert np.array_equal(gwr, O.sample_wr(N, n, 7))
    _no_device_errors()


# the ordered linear-probing warp kernels (RS_OPT_LEAF_PATH = 3; a measured
# alternative to the counting-sort warp kernels)
LP_CASES = [(2 ** 30, 2 ** 20), (2 ** 40, 2 ** 22), (10 ** 9 + 7, 100003), (2 ** 21, 2 ** 20),
            (2 ** 24 + 3, 2 ** 16 + 1), (3 ** 30, 2 ** 18 + 17), (2 ** 48, 2 ** 24)]


@pytest.mark.parametrize("N,n", LP_CASES)
def test_lp_path(N, n):
    rs.set_option(rs.OPT_LEAF_PATH, 3)
    try:
        got = _np(rs.sample_wor(N, n, 5))
        gwr = _np(rs.sample_wr(N, n, 5))
    finally:
        rs.set_option(rs.OPT_LEAF_PATH, 0)
    assert np.array_equal(got, O.sample_wor(N, n, 5))
    assert np.array_equal(gwr, O.sample_wr(N, n, 5))
    _no_device_errors()


# split + leaves in one launch (RS_OPT_FUSED, default on for shard trees of
# <= 2^11 leaves on the warp-leaf paths; rs_fused.cuh) against the separate
# split / leaf launches and the oracle: 32-bit power-of-two and Lemire leaves,
# wide (> 2^32) leaves, depth < 4 (fewer leaves than one CTA's warps), the
# largest fused depth (11) and the first unfused one (12), shards (s > 0)
FUSED_CASES = [(2 ** 30, 2 ** 20), (2 ** 50, 2 ** 10), (2 ** 50, 2 ** 20), (10 ** 12 + 7, 123457),
               (2 ** 40, 2 ** 21), (2 ** 40, 2 ** 22), (2 ** 45, 3000), (2 ** 20, 2 ** 14)]


@pytest.mark.parametrize("N,n", FUSED_CASES)
def test_fused_vs_separate(N, n):
    for mode, f, orc in ((0, rs.sample_wor, O.sample_wor), (1, rs.sample_wr, O.sample_wr)):
        fused = _np(f(N, n, 3))
        shard = _np(rs.sample_wor_shard(N, n, 3, 4, 1) if mode == 0 else rs.sample_wr_shard(N, n, 3, 4, 1))
        rs.set_option(rs.OPT_FUSED, 0)
        try:
            sep = _np(f(N, n, 3))
            sep_shard = _np(rs.sample_wor_shard(N, n, 3, 4, 1) if mode == 0 else rs.sample_wr_shard(N, n, 3, 4, 1))
        finally:
            rs.set_option(rs.OPT_FUSED, 1)
        assert np.array_equal(fused, sep), (N, n, mode)
        assert np.array_equal(shard, sep_shard), (N, n, mode)
        assert np.array_equal(fused, orc(N, n, 3)), (N, n, mode)
    _no_device_errors()


# the warp kernels' spill pass (normally ~1 leaf in 10^4: a leaf of > 1149
# draws or a pathological bucket): RS_OPT_WARP_CAP hands most leaves to it --
# the fused kernels' last CTA, or the separate CTA launch -- 32-bit and wide
SPILL_CASES = [(2 ** 30, 2 ** 20), (2 ** 40, 2 ** 24), (2 ** 50, 2 ** 12), (2 ** 50, 2 ** 24), (10 ** 12 + 7, 123457)]


@pytest.mark.parametrize("N,n", SPILL_CASES)
def test_warp_spill_path(N, n):
    rs.set_option(rs.OPT_WARP_CAP, 1000)
    try:
        got = _np(rs.sample_wor(N, n, 8))
        gwr = _np(rs.sample_wr(N, n, 8))
        gsh = _np(rs.sample_wor_shard(N, n, 8, 4, 2))
    finally:
        rs.set_option(rs.OPT_WARP_CAP, 0)
    assert np.array_equal(got, O.sample_wor(N, n, 8))
    assert np.array_equal(gwr, O.sample_wr(N, n, 8))
    assert np.array_equal(gsh, _np(rs.sample_wor_shard(N, n, 8, 4, 2)))
    _no_device_errors()


# power-of-two WOR, leaf ranges >= 2^24, shard depth > 14: the warp kernel
# without the duplicate path lists its leaves with an equal neighbour and the
# top-up kernel completes them from the list (rs_leaf_warp.cuh SD / LS)
@pytest.mark.parametrize("N,n", [(2 ** 40, 2 ** 25), (2 ** 41, 2 ** 25 + 12345)])
def test_duplicate_list_path(N, n):
    got = _np(rs.sample_wor(N, n, 9))
    assert np.array_equal(got, O.sample_wor(N, n, 9))
    rs.set_option(rs.OPT_FUSED, 0)
    try:
        sh = _np(rs.sample_wor_shard(N, n, 9, 2, 1))
    finally:
        rs.set_option(rs.OPT_FUSED, 1)
    c, off = rs.shard_info(N, n, 9, 2, 1)
    assert np.array_equal(sh, got[off:off + c])
    _no_device_errors()


# ---- with replacement --------------------------------------------------------

WR_CASES = [(1, 5), (4, 1000), (2, 3), (100, 100), (2 ** 24, 2 ** 20), (10 ** 9 + 7, 100003),
            (2 ** 45, 2 ** 18), (2 ** 20, 2 ** 22), (3, 50000)]


@pytest.mark.parametrize("N,n", WR_CASES)
def test_wr_full_compare(N, n):
    for seed in (2, 2 ** 64 - 1):
        got = _np(rs.sample_wr(N, n, seed))
        exp = O.sample_wr(N, n, seed)
        assert np.array_equal(got, exp), (N, n, seed)
    _no_device_errors()


# ---- Bernoulli -------------------------------------------------------------------

# chunk ranges r <= 2^16 (u16 buffers, 4 chunks per ticket), <= 2^24 (u32), above (u64)
BERN_CASES = [(2 ** 24, 0.01), (10 ** 6 + 17, 0.3), (2 ** 20, 1e-3), (1000, 0.999), (5, 0.5),
              (2 ** 26, 1e-5), (1000, 0.0), (1000, 1.0), (0, 0.5), (2 ** 30, 1e-6),
              (2 ** 40 + 3, 1e-9), (3 * 10 ** 8, 0.5),
              # fp64 skip candidates: u32 chunks (r <= 2^24), u64 arithmetic with
              # u32 positions (r <= 2^32), u64 positions (r > 2^32)
              (2 ** 32, 1e-4), (2 ** 37 + 5, 2 ** -16), (2 ** 50, 1e-9)]


@pytest.mark.parametrize("N,rho", BERN_CASES)
def test_bernoulli_full_compare(N, rho):
    for seed in (3, 0xDEADBEEF):
        got = _np(rs.bernoulli(N, rho, seed))
        exp = O.bernoulli(N, rho, seed)
        assert np.array_equal(got, exp), (N, rho, seed)
    _no_device_errors()


def test_bernoulli_cfg3b():
    N, rho = W.CFG3B["N"], W.CFG3B["rho"]
    got = _np(rs.bernoulli(N, rho, 1))
    exp = O.bernoulli(N, rho, 1)
    assert np.array_equal(got, exp)


def test_bernoulli_capacity_overflow_is_reported():
    o, cnt = rs.bernoulli(2 ** 20, 0.01, 5, capacity=100, return_count=True)
    exp = O.bernoulli(2 ** 20, 0.01, 5)
    assert int(cnt.item()) == exp.size
    assert np.array_equal(_np(o[:100]), exp[:100])


# ---- shards (Algorithm P): identical output for every p ----------------------------

@pytest.mark.parametrize("N,n,mode", [(2 ** 30, 2 ** 20, 0), (2 ** 26, 3 * 2 ** 24, 0),
                                      (2 ** 24, 2 ** 20, 1), (10 ** 7 + 1, 54321, 0)])
def test_shards_concatenate_to_full(N, n, mode):
    full = _np(rs.sample_wr(N, n, 9) if mode else rs.sample_wor(N, n, 9))
    for world in (2, 4, 8):
        parts = []
        for rank in range(world):
            f = rs.sample_wr_shard if mode else rs.sample_wor_shard
            parts.append(_np(f(N, n, 9, world, rank)))
        assert np.array_equal(np.concatenate(parts), full)


def test_bernoulli_shards_concatenate():
    N, rho = 2 ** 24, 0.02
    full = _np(rs.bernoulli(N, rho, 4))
    for world in (2, 8):
        parts = [_np(rs.bernoulli_shard(N, rho, 4, world, r)) for r in range(world)]
        assert np.array_equal(np.concatenate(parts), full)


# ---- full BASELINE sizes: sampled parity + properties ----------------------------

def _sampled_leaf_parity(out, N, n, seed, mode, nsample=48):
    D = O.plan(N, n, mode)[0]
    rng = np.random.default_rng(seed % 2**32)
    leaves = sorted(set([0, 1, (1 << D) - 1] + list(rng.integers(0, 1 << D, nsample))))
    for i in leaves:
        vals, off = O.leaf(N, n, seed, int(i), mode)
        got = _np(out[off: off + len(vals)])
        assert np.array_equal(got, vals), (i, off)


@pytest.mark.parametrize("cfg", ["CFG1", "HEADLINE"])
def test_full_size_wor(cfg):
    c = getattr(W, cfg)
    N, n, seed = c["N"], c["n"], c["seed"]
    out = rs.sample_wor(N, n, seed)
    torch.cuda.synchronize()
    assert out.numel() == n
    assert rs.validate(out, N, strict=True) == 0
    _sampled_leaf_parity(out, N, n, seed, O.MODE_WOR)
    # 2^16-bin uniformity on the device output (WOR variance factor ~1);
    # the output is sorted, so bin counts are differences of searchsorted
    edges = torch.arange(0, 2 ** 16 + 1, dtype=torch.int64, device=out.device) * (N // 2 ** 16)
    pos = torch.searchsorted(out.view(torch.int64), edges + 1)
    b = (pos[1:] - pos[:-1]).double()
    E = n / 2 ** 16
    chi2 = float(((b - E) ** 2 / E).sum())
    from scipy import stats
    assert stats.chi2.sf(chi2, 2 ** 16 - 1) > 1e-3
    _no_device_errors()
    del out
    torch.cuda.empty_cache()


def test_full_size_complement():
    c = W.CFG3A
    N, n, seed = c["N"], c["n"], c["seed"]
    out = rs.sample_wor(N, n, seed)
    assert rs.validate(out, N, strict=True) == 0
    _sampled_leaf_parity(out, N, n, seed, O.MODE_WOR, nsample=24)
    _no_device_errors()
    del out
    torch.cuda.empty_cache()


def test_full_size_wr():
    c = W.CFG4
    N, n, seed = c["N"], c["n"], c["seed"]
    out = rs.sample_wr(N, n, seed)
    assert rs.validate(out, N, strict=False) == 0
    _sampled_leaf_parity(out, N, n, seed, O.MODE_WR, nsample=24)
    _no_device_errors()
    del out
    torch.cuda.empty_cache()


def test_digest_matches_oracle_cfg0():
    N, n = W.CFG0["N"], W.CFG0["n"]
    out = rs.sample_wor(N, n, 1)
    assert rs.digest(out) == O.digest_range(N, n, 1)


def test_deterministic_repeat():
    a = rs.sample_wor(2 ** 40, 2 ** 22, 123)
    b = rs.sample_wor(2 ** 40, 2 ** 22, 123)
    assert torch.equal(a.view(torch.int64), b.view(torch.int64))


def test_host_buffer_call():
    N, n = 2 ** 30, 2 ** 20
    h = rs.sample_wor_host(N, n, 1)
    assert np.array_equal(h.numpy(), O.sample_wor(N, n, 1))


def test_workspace_variant():
    N, n = 2 ** 30, 2 ** 20
    wsb = rs.workspace_bytes(rs.MODE_WOR, N, n)
    ws = torch.empty(wsb, dtype=torch.uint8, device="cuda")
    out = torch.empty(n, dtype=torch.uint64, device="cuda")
    rs.sample_wor_ws(N, n, 1, 1, 0, out, ws)
    assert np.array_equal(_np(out), O.sample_wor(N, n, 1))
    with pytest.raises(rs.RSError):
        rs.sample_wor_ws(N, n, 1, 1, 0, out, ws[: wsb // 2])


# ---- NEXT-1: any node / leaf range of the tree (range-addressable sampling) ------

@pytest.mark.parametrize("N,n,mode", [(2 ** 30, 2 ** 20, 0), (2 ** 22, 3 * 2 ** 20, 0),
                                      (2 ** 24, 2 ** 20, 1), (10 ** 9 + 7, 100003, 0)])
def test_nodes_and_ranges(N, n, mode):
    full = _np(rs.sample_wr(N, n, 11) if mode else rs.sample_wor(N, n, 11))
    D = rs.plan(mode, N, n)[0]
    for d in sorted(set([0, 2, 5, D])):
        for i in sorted(set(i for i in [0, 1, (1 << d) // 2, (1 << d) - 1] if i < (1 << d))):
            cnt, off = rs.node_info(mode, N, n, 11, d, i)
            got = _np(rs.sample_node(mode, N, n, 11, d, i))
            assert got.size == cnt
            assert np.array_equal(got, full[off: off + cnt]), (d, i)
    for lo, hi in [(0, 1 << D), (3, 17), ((1 << D) // 3, (1 << D) - 5), (7, 8)]:
        got, off = rs.sample_range(mode, N, n, 11, lo, hi)
        assert np.array_equal(_np(got), full[off: off + got.numel()]), (lo, hi)


def test_host_buffer_batched_overlap():
    # > 2^26 values: the host path runs several node batches, copies overlapped
    N, n = 2 ** 40, 3 * 2 ** 26 + 12345
    h = rs.sample_wor_host(N, n, 5)
    d = rs.sample_wor(N, n, 5)
    assert torch.equal(h.view(torch.int64), d.cpu().view(torch.int64))
    _sampled_leaf_parity(d, N, n, 5, O.MODE_WOR, nsample=16)
    # the cached staging: a smaller call reuses it, a WR shard after a release
    # re-creates it
    assert np.array_equal(rs.sample_wor_host(2 ** 30, 2 ** 20, 1).numpy(), O.sample_wor(2 ** 30, 2 ** 20, 1))
    rs.release_cache()
    hw = rs.sample_shard_host(rs.MODE_WR, 2 ** 36, 2 ** 27, 3, 2, 1)
    dw = rs.sample_wr_shard(2 ** 36, 2 ** 27, 3, 2, 1)
    assert torch.equal(hw.view(torch.int64), dw.cpu().view(torch.int64))


# ---- NEXT-2: uneven universe over PEs ---------------------------------

@pytest.mark.parametrize("L,n", [([17, 3, 40, 0, 25, 9, 11, 30, 14, 22, 8, 31, 19], 50),
                                 ([2 ** 30, 3 * 2 ** 28, 12345, 2 ** 31], 2 ** 21),
                                 ([10 ** 6, 1, 5 * 10 ** 5, 7 * 10 ** 5 + 3], 10 ** 6)])
def test_uneven_local_samples(L, n):
    counts = rs.uneven_counts(L, n, 21)
    assert sum(counts) == n
    for pe in range(len(L)):
        vals, cnt = rs.uneven_local_sample(L, n, 21, pe)
        exp = O.sample_wor(L[pe], cnt, O.uneven_seed(21, pe))
        assert np.array_equal(_np(vals), exp), pe


# ---- NEXT-3: random graphs, decode fused into every store path --------------------

@pytest.mark.parametrize("V,m", [(4, 6), (100, 37), (1000, 4000), (3000, 3 * 10 ** 6),     # warp / bitmap / complement
                                 (2 ** 20 + 7, 2 ** 20), (70000, 2 ** 31)])
def test_gnm(V, m):
    got = _np(rs.gnm(V, m, 13))
    assert np.array_equal(got, O.gnm(V, m, 13)), (V, m)
    _no_device_errors()


def test_gnm_cta_path():
    rs.set_option(rs.OPT_LEAF_PATH, 1)
    try:
        got = _np(rs.gnm(5000, 10 ** 5, 2))
    finally:
        rs.set_option(rs.OPT_LEAF_PATH, 0)
    assert np.array_equal(got, O.gnm(5000, 10 ** 5, 2))


@pytest.mark.parametrize("V,p", [(5, 1.0), (1000, 0.01), (3000, 0.3), (2 ** 16, 1e-4)])
def test_gnp(V, p):
    got = _np(rs.gnp(V, p, 17))
    assert np.array_equal(got, O.gnp(V, p, 17)), (V, p)


# ---- NEXT-4: Algorithm B + repair (the comparison baseline) -----------------

ALGB_CASES = [(1, 1, 4.0), (10, 10, 4.0), (100, 95, 4.0), (1000, 100, 0.0), (2 ** 20, 2 ** 10, 4.0),
              (2 ** 30, 2 ** 20, 4.0), (2 ** 40, 3 * 10 ** 6, 2.0), (2 ** 48, 5000, 0.5)]


@pytest.mark.parametrize("N,n,slack", ALGB_CASES)
def test_algb(N, n, slack):
    for seed in (3, 2 ** 64 - 1):
        got, att = rs.sample_wor_algb(N, n, seed, slack=slack, return_attempts=True)
        exp, eatt = O.algb(N, n, seed, slack=slack)
        assert att == eatt, (N, n, seed)
        assert np.array_equal(_np(got), exp), (N, n, seed)
    _no_device_errors()


def test_algb_restarts_and_errors():
    # slack 0 restarts about half the time: the attempt counts and outputs
    # follow the oracle's seed_a sequence
    for seed in range(12):
        got, att = rs.sample_wor_algb(1000, 100, seed, slack=0.0, return_attempts=True)
        exp, eatt = O.algb(1000, 100, seed, slack=0.0)
        assert att == eatt and np.array_equal(_np(got), exp)
    assert rs.sample_wor_algb(50, 0, 1).numel() == 0
    N, n = 2 ** 30, 2 ** 16                      # caller workspace, and one too small
    ws = torch.empty(rs.algb_workspace_bytes(N, n), dtype=torch.uint8, device="cuda")
    got, att = rs.sample_wor_algb(N, n, 9, ws=ws, return_attempts=True)
    exp, eatt = O.algb(N, n, 9)
    assert att == eatt and np.array_equal(_np(got), exp)
    with pytest.raises(rs.RSError):
        rs.sample_wor_algb(N, n, 9, ws=ws[:1024])
    with pytest.raises(rs.RSError):
        rs.sample_wor_algb(10, 11, 1)
    with pytest.raises(rs.RSError):
        rs.sample_wor_algb(10, 5, 1, slack=-1.0)
    fails = 0
    for seed in range(40):          # one pass only: fails whenever n' < n
        try:
            rs.sample_wor_algb(1000, 100, seed, slack=0.0, max_attempts=1)
        except rs.RSError as e:
            assert "restart" in str(e)
            fails += 1
    assert 5 < fails < 35


def test_graphs_with_workspace():
    V, m, p = 5000, 10 ** 6, 0.05
    N = V * (V - 1) // 2
    ws = torch.empty(rs.workspace_bytes(rs.MODE_WOR, N, m, 0.0, 1), dtype=torch.uint8, device="cuda")
    assert np.array_equal(_np(rs.gnm(V, m, 4, ws=ws)), O.gnm(V, m, 4))
    ws = torch.empty(rs.workspace_bytes(rs.MODE_BERNOULLI, N, 0, p, 1), dtype=torch.uint8, device="cuda")
    assert np.array_equal(_np(rs.gnp(V, p, 4, ws=ws)), O.gnp(V, p, 4))
    with pytest.raises(rs.RSError):
        rs.gnm(V, m, 4, ws=ws[:16])


# ---- split deviates one by one (HYP/HRUA, BINV/BTRS on the device) ----------

DEV_CASES = [(16, 50, 100), (17, 10 ** 6, 2 * 10 ** 6), (1000, 2 ** 26, 2 ** 27), (1024, 2 ** 25 + 3, 2 ** 26 + 7),
             (5000, 3, 10 ** 4), (8192, 2 ** 40, 2 ** 41), (2 ** 20, 2 ** 45, 2 ** 46 + 1),
             (2 ** 32, 2 ** 47, 2 ** 48), (3 * 2 ** 30, 2 ** 31, 2 ** 32), (10 ** 5, 123456, 10 ** 6),
             (2 ** 33, 2 ** 61, 2 ** 62 - 5)]


@pytest.mark.parametrize("k,L,R", DEV_CASES)
def test_deviates_vs_oracle(k, L, R):
    cnt = 20000
    for kind, f in ((0, O.hgd_batch), (1, O.bin_batch)):
        if kind == 1 and k > 2 ** 40:
            continue
        exp = f(k, L, R, 77, 1, cnt)
        # thread per deviate, then lane groups of 32 and 8 (parallel iterations)
        for kk in (kind, kind + 2, kind + 4):
            got = _np(rs.deviates(kk, k, L, R, 77, 1, cnt))
            assert np.array_equal(got, exp), (kk, k, L, R, int(np.sum(got != exp)))


@pytest.mark.parametrize("tmax", [0, 1, 2])
def test_topup_fallback(tmax):
    # small leaf ranges: the *_tu kernels top the distinct set up draw by draw;
    # a low limit forces the full-round fallback -- same result either way
    rs.set_option(rs.OPT_TOPUP_MAX, tmax)
    try:
        for N, n in ((2 ** 30, 2 ** 20), (2 ** 26 + 12345, 2 ** 16 + 7)):
            got = _np(rs.sample_wor(N, n, 11))
            assert np.array_equal(got, O.sample_wor(N, n, 11)), (tmax, N, n)
        assert np.array_equal(_np(rs.gnm(70000, 2 ** 22, 5)), O.gnm(70000, 2 ** 22, 5))
    finally:
        rs.set_option(rs.OPT_TOPUP_MAX, 32)
    _no_device_errors()


# ---- device-side capacity failures are reported through the API ----

def test_capacity_overflow_returns_ecapacity():
    """A leaf the kernels cannot hold on chip must surface as RS_ECAPACITY from
    the synchronous calls, without rs_device_errors().  RS_OPT_LEAF_CAP caps
    the CTA leaf kernel at 64 draws, so cfg0's ~1024-value leaves overflow."""
    N, n = 2 ** 30, 2 ** 20
    rs.set_option(rs.OPT_LEAF_PATH, 1)
    rs.set_option(rs.OPT_LEAF_CAP, 64)
    try:
        with pytest.raises(rs.RSError, match="capacity"):
            rs.sample_checked(rs.MODE_WOR, N, n, 1)
        with pytest.raises(rs.RSError, match="capacity"):
            rs.sample_shard_host(rs.MODE_WOR, N, n, 1, 1, 0)
        with pytest.raises(rs.RSError, match="capacity"):
            rs.sample_checked(rs.MODE_WR, N, n, 1)
    finally:
        rs.set_option(rs.OPT_LEAF_CAP, 0)
        rs.set_option(rs.OPT_LEAF_PATH, 0)
        rs.device_errors(clear=True)
    # the same calls succeed (and match the oracle) with the default capacity
    got = rs.sample_checked(rs.MODE_WOR, N, n, 1)
    assert np.array_equal(_np(got), O.sample_wor(N, n, 1))
    assert rs.device_errors(clear=True) == 0


def test_host_stream_ring():
    """rs_sample_shard_host_stream with a host buffer smaller than the slice
    (two batches of ~2^25 values through a 2 x (2^25 + 2^20) ring): every
    value that reaches the ring is one of the sample's; with a buffer of the
    full size it equals rs_sample_shard_host."""
    N, n, seed = 2 ** 40, 2 ** 26 + 5, 3
    full = rs.sample_shard_host(rs.MODE_WOR, N, n, seed, 1, 0)
    big = torch.empty(n, dtype=torch.uint64, pin_memory=True)
    rs.sample_shard_host_stream(rs.MODE_WOR, N, n, seed, 1, 0, big)
    assert torch.equal(big.view(torch.int64), full.view(torch.int64))
    ring = torch.zeros(2 * (2 ** 25 + 2 ** 20), dtype=torch.uint64, pin_memory=True)
    rs.sample_shard_host_stream(rs.MODE_WOR, N, n, seed, 1, 0, ring)
    r = ring.view(torch.int64).numpy()
    v = r[r != 0]
    f = full.view(torch.int64).numpy()
    idx = np.minimum(np.searchsorted(f, v), f.size - 1)
    assert v.size > 2 ** 25 and np.array_equal(f[idx], v)
    with pytest.raises(rs.RSError):
        rs.sample_shard_host_stream(rs.MODE_WOR, N, n, seed, 1, 0, ring[:1000])
