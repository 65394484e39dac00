"""CPU oracle for the divide-and-conquer sampler (arXiv 1610.05141).

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s ``cpu_baseline`` / ``--impl reference`` legs may import this
package.  The product path (``paper_1610_05141_b200``) never imports it and
shares no code with it; see ``oracle/rso.c`` for the algorithm and its pins.

This module is argument marshalling (ctypes + numpy) around ``librso.so``;
every step of the method is in ``rso.c``.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "rso.c")
_LIB = os.path.join(_HERE, "librso.so")

GCC_FLAGS = ["-O2", "-std=c11", "-Wall", "-ffp-contract=off", "-fno-fast-math",
             "-fPIC", "-shared", "-pthread"]

MODE_WOR, MODE_WR = 0, 1


def build(force: bool = False) -> str:
    """Compile librso.so with gcc (no FMA contraction, no fast-math)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + ".tmp"
        subprocess.check_call(["gcc", *GCC_FLAGS, "-o", tmp, _SRC, "-lm"])
        os.replace(tmp, _LIB)
    return _LIB


_lib = None


def lib():
    global _lib
    if _lib is None:
        build()
        L = C.CDLL(_LIB)
        u64, u32, dbl, i32 = C.c_uint64, C.c_uint32, C.c_double, C.c_int
        P64 = C.POINTER(C.c_uint64)
        P32 = C.POINTER(C.c_uint32)
        sig = {
            "rso_philox": (None, [P32, P32, P32]),
            "rso_u52": (dbl, [u32, u32]),
            "rso_draw": (u64, [u64, u32, u64, u64, u64]),
            "rso_lemire64_scan": (None, [u64, u64, u64, u64, P64]),
            "rso_log": (dbl, [dbl]),
            "rso_log1p": (dbl, [dbl]),
            "rso_stirlerr": (dbl, [dbl]),
            "rso_bd0": (dbl, [dbl, dbl]),
            "rso_ldbinom": (dbl, [dbl, dbl, dbl, dbl]),
            "rso_hgd_logratio": (dbl, [u64, u64, u64, u64, u64]),
            "rso_hgd": (u64, [u64, u64, u64, u64, u64]),
            "rso_bin": (u64, [u64, u64, u64, u64, u64]),
            "rso_geo": (dbl, [dbl, dbl]),
            "rso_node": (None, [u64, i32, u64, P64, P64, P64]),
            "rso_depth": (i32, [u64, u64]),
            "rso_tree_counts": (None, [u64, u64, u64, i32, i32, P64]),
            "rso_path": (None, [u64, u64, u64, i32, i32, u64, P64, P64]),
            "rso_digest": (u64, [P64, u64, u64]),
            "rso_sample_wor": (i32, [u64, u64, u64, P64, i32]),
            "rso_sample_wr": (i32, [u64, u64, u64, P64, i32]),
            "rso_digest_range": (i32, [u64, u64, u64, i32, i32, u64, u64, P64]),
            "rso_plan": (i32, [u64, u64, i32, C.POINTER(C.c_int), C.POINTER(C.c_int), P64]),
            "rso_leaf": (i32, [u64, u64, u64, i32, u64, P64, P64, P64]),
            "rso_leaf_size": (i32, [u64, u64, u64, i32, u64, P64, P64]),
            "rso_bern_depth": (i32, [u64, dbl]),
            "rso_bernoulli": (i32, [u64, dbl, u64, P64, u64, P64]),
            "rso_bern_chunk": (u64, [u64, dbl, u64, u64, P64]),
            "rso_shard_info": (i32, [u64, u64, u64, i32, i32, i32, P64, P64]),
            "rso_lemire32": (i32, [u32, u64, P64]),
            "rso_lemire32_hist": (u64, [u64, P32]),
            "rso_hgd_batch": (None, [u64, u64, u64, u64, u64, u64, P64]),
            "rso_bin_batch": (None, [u64, u64, u64, u64, u64, u64, P64]),
            "rso_small_samples": (None, [u64, u64, u64, u64, i32, P64]),
            "rso_digest_leaves_replay": (i32, [u64, u64, u64, i32, i32, u64, u64, P64, P64]),
            "rso_bern_chunks_digest": (i32, [u64, dbl, u64, u64, u64, P64, P64]),
            "rso_bern_chunks_digest_mt": (i32, [u64, dbl, u64, i32, u64, u64, P64, P64]),
            "rso_uneven_counts": (i32, [i32, P64, u64, u64, P64]),
            "rso_uneven_seed": (u64, [u64, u64]),
            "rso_edges": (None, [u64, P64, u64, P64]),
            "rso_algb": (i32, [u64, u64, u64, dbl, P64, C.c_uint32, C.POINTER(C.c_uint32)]),
        }
        for name, (res, args) in sig.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib


def _p64(a: np.ndarray):
    return a.ctypes.data_as(C.POINTER(C.c_uint64))


# ---- primitives -----------------------------------------------------------

def philox(ctr, key):
    c = (C.c_uint32 * 4)(*ctr)
    k = (C.c_uint32 * 2)(*key)
    o = (C.c_uint32 * 4)()
    lib().rso_philox(c, k, o)
    return tuple(o)


def u52(a, b):
    return lib().rso_u52(a, b)


def draw(seed, purpose, node_id, r, j):
    return lib().rso_draw(seed, purpose, node_id, r, j)


def log(x):
    return lib().rso_log(x)


def log1p(x):
    return lib().rso_log1p(x)


def stirlerr(n):
    return lib().rso_stirlerr(float(n))


def bd0(x, np_):
    return lib().rso_bd0(float(x), float(np_))


def ldbinom(x, n, p, q):
    return lib().rso_ldbinom(float(x), float(n), p, q)


def hgd_logratio(kp, g, R, K, M):
    return lib().rso_hgd_logratio(kp, g, R, K, M)


def hgd(k, L, R, seed, node_id):
    return lib().rso_hgd(k, L, R, seed, node_id)


def binom(k, L, R, seed, node_id):
    return lib().rso_bin(k, L, R, seed, node_id)


def geo(U, log1m_rho):
    return lib().rso_geo(U, log1m_rho)


def node(N, d, i):
    lo, R, L = C.c_uint64(), C.c_uint64(), C.c_uint64()
    lib().rso_node(N, d, i, C.byref(lo), C.byref(R), C.byref(L))
    return lo.value, R.value, L.value


def depth(m, n0=1024):
    return lib().rso_depth(m, n0)


def plan(N, n, mode=MODE_WOR):
    D, comp, m = C.c_int(), C.c_int(), C.c_uint64()
    lib().rso_plan(N, n, mode, C.byref(D), C.byref(comp), C.byref(m))
    return D.value, bool(comp.value), m.value


def tree_counts(N, m, seed, D, wr=False):
    cnt = np.zeros(1 << D, dtype=np.uint64)
    lib().rso_tree_counts(N, m, seed, D, int(wr), _p64(cnt))
    return cnt


def path(N, m, seed, d, i, wr=False):
    c, o = C.c_uint64(), C.c_uint64()
    lib().rso_path(N, m, seed, int(wr), d, i, C.byref(c), C.byref(o))
    return c.value, o.value


def digest(v: np.ndarray, base_index: int = 0) -> int:
    v = np.ascontiguousarray(v, dtype=np.uint64)
    return lib().rso_digest(_p64(v), v.size, base_index)


# ---- whole samples --------------------------------------------------------

def _check(st):
    if st != 0:
        raise ValueError(f"oracle status {st}")


def sample_wor(N, n, seed, nthreads=None):
    nthreads = nthreads or os.cpu_count() or 1
    out = np.zeros(n, dtype=np.uint64)
    _check(lib().rso_sample_wor(N, n, seed, _p64(out), nthreads))
    return out


def sample_wr(N, n, seed, nthreads=None):
    nthreads = nthreads or os.cpu_count() or 1
    out = np.zeros(n, dtype=np.uint64)
    _check(lib().rso_sample_wr(N, n, seed, _p64(out), nthreads))
    return out


def digest_range(N, n, seed, mode=MODE_WOR, leaf_lo=0, leaf_hi=2**64 - 1, nthreads=None):
    nthreads = nthreads or os.cpu_count() or 1
    d = C.c_uint64()
    _check(lib().rso_digest_range(N, n, seed, mode, nthreads, leaf_lo, leaf_hi, C.byref(d)))
    return d.value


def leaf(N, n, seed, i, mode=MODE_WOR):
    """(values, global_offset) of output leaf i, by path replay."""
    cnt, rng = C.c_uint64(), C.c_uint64()
    _check(lib().rso_leaf_size(N, n, seed, mode, i, C.byref(cnt), C.byref(rng)))
    buf = np.zeros(max(rng.value if cnt.value > 0 else 0, cnt.value, 1), dtype=np.uint64)
    c, off = C.c_uint64(), C.c_uint64()
    _check(lib().rso_leaf(N, n, seed, mode, i, _p64(buf), C.byref(c), C.byref(off)))
    return buf[: c.value].copy(), off.value


def bern_depth(N, rho):
    return lib().rso_bern_depth(N, rho)


def bernoulli(N, rho, seed, capacity=None):
    if capacity is None:
        capacity = int(N * rho + 10 * (N * rho * (1 - rho)) ** 0.5) + 64
        capacity = min(capacity, N)
    out = np.zeros(max(capacity, 1), dtype=np.uint64)
    cnt = C.c_uint64()
    st = lib().rso_bernoulli(N, rho, seed, _p64(out), capacity, C.byref(cnt))
    if st not in (0, 4):
        _check(st)
    if cnt.value > capacity:
        raise ValueError("bernoulli capacity exceeded")
    return out[: cnt.value].copy()


def bern_chunk(N, rho, seed, chunk):
    c = lib().rso_bern_chunk(N, rho, seed, chunk, None)
    buf = np.zeros(max(c, 1), dtype=np.uint64)
    lib().rso_bern_chunk(N, rho, seed, chunk, _p64(buf))
    return buf[:c].copy()


def shard_info(N, n, seed, world, rank, mode=MODE_WOR):
    c, o = C.c_uint64(), C.c_uint64()
    _check(lib().rso_shard_info(N, n, seed, mode, world, rank, C.byref(c), C.byref(o)))
    return c.value, o.value


# ---- test hooks -----------------------------------------------------------

def lemire32_hist(r):
    hist = np.zeros(r, dtype=np.uint32)
    acc = lib().rso_lemire32_hist(r, hist.ctypes.data_as(C.POINTER(C.c_uint32)))
    return hist, acc


def hgd_batch(k, L, R, seed, id0, count):
    out = np.zeros(count, dtype=np.uint64)
    lib().rso_hgd_batch(k, L, R, seed, id0, count, _p64(out))
    return out


def bin_batch(k, L, R, seed, id0, count):
    out = np.zeros(count, dtype=np.uint64)
    lib().rso_bin_batch(k, L, R, seed, id0, count, _p64(out))
    return out


def small_samples(N, n, s0, count, mode=MODE_WOR):
    out = np.zeros(count, dtype=np.uint64)
    lib().rso_small_samples(N, n, s0, count, mode, _p64(out))
    return out


def digest_leaves_replay(N, n, seed, mode, leaf_lo, leaf_hi, nthreads=None):
    """(digest, values) of output leaves [leaf_lo, leaf_hi) via path replay."""
    nthreads = nthreads or os.cpu_count() or 1
    d, v = C.c_uint64(), C.c_uint64()
    _check(lib().rso_digest_leaves_replay(N, n, seed, mode, nthreads, leaf_lo, leaf_hi,
                                          C.byref(d), C.byref(v)))
    return d.value, v.value


def bern_chunks_digest(N, rho, seed, c_lo, c_hi):
    d, v = C.c_uint64(), C.c_uint64()
    _check(lib().rso_bern_chunks_digest(N, rho, seed, c_lo, c_hi, C.byref(d), C.byref(v)))
    return d.value, v.value


def bern_digest(N, rho, seed, c_lo=0, c_hi=2**64 - 1, nthreads=None):
    """(digest, count) of Bernoulli chunks [c_lo, c_hi) with threads (digest
    indices start at 0 for chunk c_lo)."""
    nthreads = nthreads or os.cpu_count() or 1
    d, v = C.c_uint64(), C.c_uint64()
    _check(lib().rso_bern_chunks_digest_mt(N, rho, seed, nthreads, c_lo, c_hi, C.byref(d), C.byref(v)))
    return d.value, v.value


def lemire64_scan(r, v, w_lo, w_hi):
    """Test hook: (#accepted words -> v, #accepted -> other, #rejected) over [w_lo, w_hi)."""
    o = np.zeros(3, dtype=np.uint64)
    lib().rso_lemire64_scan(r, v, w_lo, w_hi, _p64(o))
    return tuple(int(x) for x in o)


def uneven_counts(L, n, seed):
    """Per-PE sample counts for an uneven universe."""
    Lv = np.ascontiguousarray(np.asarray(L, dtype=np.uint64))
    out = np.zeros(Lv.size, dtype=np.uint64)
    _check(lib().rso_uneven_counts(int(Lv.size), _p64(Lv), int(n), int(seed) % 2**64, _p64(out)))
    return out


def uneven_seed(seed, i):
    return int(lib().rso_uneven_seed(int(seed) % 2**64, int(i)))


def edges(V, values):
    """Packed (u << 32) | v edges of 1-based edge indices (NEXT-3)."""
    v = np.ascontiguousarray(np.asarray(values, dtype=np.uint64))
    out = np.zeros(v.size, dtype=np.uint64)
    lib().rso_edges(int(V), _p64(v), int(v.size), _p64(out))
    return out


def gnm(V, m, seed):
    return edges(V, sample_wor(V * (V - 1) // 2, m, seed))


def gnp(V, p, seed):
    return edges(V, bernoulli(V * (V - 1) // 2, p, seed))



def algb(N, n, seed, slack=4.0, max_attempts=1000):
    """NEXT-4: Algorithm B + repair (rso_algb): (sorted sample, attempts)."""
    out = np.zeros(max(int(n), 1), dtype=np.uint64)
    att = C.c_uint32()
    _check(lib().rso_algb(int(N), int(n), int(seed) % 2**64, float(slack), _p64(out),
                          int(max_attempts), C.byref(att)))
    return out[: int(n)].copy(), att.value
