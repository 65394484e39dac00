"""NEXT-3 pins: the oracle's edge decode is a bijection from
0..V(V-1)/2-1 onto the pairs u < v in lexicographic order (brute-force
enumeration, V <= 100, as SPEC S:591 asks), G(V, m) has m distinct edges and
G(V, p) each edge with probability p.  -m "not gpu"."""
from __future__ import annotations

import numpy as np
import pytest

import oracle as O


@pytest.mark.parametrize("V", [2, 3, 4, 5, 17, 64, 100])
def test_edge_decode_is_lexicographic_bijection(V):
    N = V * (V - 1) // 2
    got = O.edges(V, np.arange(1, N + 1, dtype=np.uint64))
    exp = np.array([(u << 32) | v for u in range(V) for v in range(u + 1, V)], dtype=np.uint64)
    assert np.array_equal(got, exp)


def test_edge_decode_large_v_endpoints():
    V = 2 ** 32 - 1
    N = V * (V - 1) // 2
    got = O.edges(V, [1, 2, V - 1, V, N - 1, N])
    exp = [(0 << 32) | 1, (0 << 32) | 2, (0 << 32) | (V - 1), (1 << 32) | 2,
           ((V - 3) << 32) | (V - 1), ((V - 2) << 32) | (V - 1)]
    assert [int(x) for x in got] == exp


def test_gnm_gnp_properties():
    V = 1000
    g = O.gnm(V, 5000, 3)
    assert g.size == 5000 and np.all(np.diff(g.astype(np.int64)) > 0)
    u, v = g >> np.uint64(32), g & np.uint64(0xFFFFFFFF)
    assert np.all(u < v) and np.all(v < V)
    assert np.array_equal(O.gnm(4, 6, 1), O.edges(4, np.arange(1, 7)))   # complete K4
    h = O.gnp(V, 0.01, 5)
    N = V * (V - 1) // 2
    z = (h.size - N * 0.01) / np.sqrt(N * 0.01 * 0.99)
    assert abs(z) < 4.5
