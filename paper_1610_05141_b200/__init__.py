"""B200-native divide-and-conquer random sampling (arXiv 1610.05141).

Thin Python binding over ``librs.so`` (C ABI: ``include/rs.h``).  Argument
marshalling only: every step of the sampler runs in the CUDA kernels of
``csrc/``.  PyTorch is used for device memory and the current stream.  There
is no CPU fallback: if the library or a CUDA device is missing, calls raise.

    import torch, paper_1610_05141_b200 as rs
    out = rs.sample_wor(N=2**40, n=2**30, seed=1)       # torch.uint64 on cuda
"""
from __future__ import annotations

import ctypes as C
import os

import torch

from . import build as _build

__all__ = [
    "sample_wor", "sample_wr", "bernoulli", "bernoulli_capacity", "shard_info",
    "sample_wor_shard", "sample_wr_shard", "bernoulli_shard", "workspace_bytes",
    "sample_wor_host", "sample_shard_host", "digest", "validate", "plan", "device_errors", "launch_count",
    "timing_enable", "timing_read",
    "RSError", "MODE_WOR", "MODE_WR", "MODE_BERNOULLI", "lib", "LIB_PATH",
]

MODE_WOR, MODE_WR, MODE_BERNOULLI = 0, 1, 2
LIB_PATH = _build.LIB

_u64, _dbl, _int, _vp, _sz = C.c_uint64, C.c_double, C.c_int, C.c_void_p, C.c_size_t
_P64 = C.POINTER(C.c_uint64)

# name -> (restype, argtypes); mirrors include/rs.h
SIGNATURES = {
    "rs_sample_wor": (_int, [_u64, _u64, _u64, _vp, _vp]),
    "rs_sample_wr": (_int, [_u64, _u64, _u64, _vp, _vp]),
    "rs_bernoulli": (_int, [_u64, _dbl, _u64, _vp, _u64, _vp, _vp]),
    "rs_bernoulli_capacity": (_u64, [_u64, _dbl]),
    "rs_shard_info": (_int, [_u64, _u64, _u64, _int, _int, _int, _P64, _P64]),
    "rs_sample_wor_shard": (_int, [_u64, _u64, _u64, _int, _int, _vp, _vp]),
    "rs_sample_wr_shard": (_int, [_u64, _u64, _u64, _int, _int, _vp, _vp]),
    "rs_bernoulli_shard": (_int, [_u64, _dbl, _u64, _int, _int, _vp, _u64, _vp, _vp]),
    "rs_workspace_bytes": (_int, [_int, _u64, _u64, _dbl, _int, C.POINTER(_sz)]),
    "rs_sample_wor_ws": (_int, [_u64, _u64, _u64, _int, _int, _vp, _vp, _sz, _vp]),
    "rs_sample_wr_ws": (_int, [_u64, _u64, _u64, _int, _int, _vp, _vp, _sz, _vp]),
    "rs_bernoulli_ws": (_int, [_u64, _dbl, _u64, _int, _int, _vp, _u64, _vp, _vp, _sz, _vp]),
    "rs_sample_wor_host": (_int, [_u64, _u64, _u64, _vp, _vp]),
    "rs_sample_shard_host": (_int, [_int, _u64, _u64, _u64, _int, _int, _vp, _vp]),
    "rs_sample_shard_host_stream": (_int, [_int, _u64, _u64, _u64, _int, _int, _vp, _u64, _vp]),
    "rs_sample_checked": (_int, [_int, _u64, _u64, _u64, _int, _int, _vp, _vp]),
    "rs_digest": (_int, [_vp, _u64, _u64, _vp, _vp]),
    "rs_validate": (_int, [_vp, _u64, _u64, _int, _vp, _vp]),
    "rs_plan": (_int, [_int, _u64, _u64, _dbl, C.POINTER(_int), C.POINTER(_int), _P64]),
    "rs_device_errors": (_int, [_int, C.POINTER(C.c_uint)]),
    "rs_launch_count": (_u64, [_int]),
    "rs_set_option": (_int, [_int, _int]),
    "rs_node_info": (_int, [_int, _u64, _u64, _u64, _int, _u64, _P64, _P64]),
    "rs_uneven_counts": (_int, [_int, _P64, _u64, _u64, _P64]),
    "rs_uneven_seed": (_u64, [_u64, _u64]),
    "rs_gnm": (_int, [_u64, _u64, _u64, _vp, _vp, _sz, _vp]),
    "rs_gnp": (_int, [_u64, _dbl, _u64, _vp, _u64, _vp, _vp, _sz, _vp]),
    "rs_sample_wor_algb": (_int, [_u64, _u64, _u64, _dbl, C.c_uint32, _vp, C.POINTER(C.c_uint32), _vp, _sz, _vp]),
    "rs_algb_workspace_bytes": (_u64, [_u64, _u64, _dbl]),
    "rs_sample_node": (_int, [_int, _u64, _u64, _u64, _int, _u64, _vp, _vp]),
    "rs_timing_enable": (_int, [_int]),
    "rs_release_cache": (_int, []),
    "rs_deviates": (_int, [_int, _u64, _u64, _u64, _u64, _u64, _u64, _vp, _vp]),
    "rs_timing_read": (_int, [_int, C.POINTER(_dbl), _P64]),
    "rs_status_string": (C.c_char_p, [_int]),
    "rs_last_status": (_int, []),
    "rs_version": (C.c_char_p, []),
}


class RSError(RuntimeError):
    pass


_lib = None


def lib():
    """Load librs.so (building it if stale and nvcc is present)."""
    global _lib
    if _lib is None:
        override = os.environ.get("RS_LIB")      # dev: benchmark a variant build
        if override:
            L = C.CDLL(override)
            for name, (res, args) in SIGNATURES.items():
                f = getattr(L, name)
                f.restype = res
                f.argtypes = args
            _lib = L
            return _lib
        if not os.path.exists(LIB_PATH) or _build.stale():
            try:
                _build.build()
            except Exception as e:  # no silent fallback: the product needs the library
                if not os.path.exists(LIB_PATH):
                    raise ImportError(f"librs.so missing and build failed: {e}") from e
        L = C.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib


def _check(st: int):
    if st != 0:
        raise RSError(f"librs: {lib().rs_status_string(st).decode()} (status {st})")


def _stream(stream=None):
    if stream is None:
        stream = torch.cuda.current_stream()
    return C.c_void_p(stream.cuda_stream)


def _out(n: int, out, device):
    if out is None:
        return torch.empty(max(n, 1), dtype=torch.uint64, device=device)[:n]
    if (out.dtype not in (torch.uint64, torch.int64) or not out.is_cuda or out.numel() < n
            or not out.is_contiguous()):
        raise ValueError("out must be a contiguous cuda uint64 tensor with >= n elements")
    return out


def _host(n: int, out_host):
    """A host uint64 buffer of >= n elements (the C ABI writes n values)."""
    if out_host is None:
        return torch.empty(max(n, 1), dtype=torch.uint64, pin_memory=True)
    if (out_host.dtype not in (torch.uint64, torch.int64) or out_host.is_cuda
            or out_host.numel() < n or not out_host.is_contiguous()):
        raise ValueError("out_host must be a contiguous CPU uint64 tensor with >= n elements")
    return out_host


def _ptr(t):
    return C.c_void_p(t.data_ptr()) if t.numel() else C.c_void_p(0)


def _require_cuda():
    if not torch.cuda.is_available():
        raise RSError("librs: CUDA device required (no CPU fallback)")


# ---- sampling -------------------------------------------------------------

def sample_wor(N: int, n: int, seed: int, out=None, device="cuda", stream=None):
    """Sorted sample of n distinct integers of 1..N (uint64, on the device)."""
    _require_cuda()
    o = _out(n, out, device)
    _check(lib().rs_sample_wor(N, n, seed % 2**64, _ptr(o), _stream(stream)))
    return o[:n]


def sample_wr(N: int, n: int, seed: int, out=None, device="cuda", stream=None):
    """n iid uniform integers of 1..N, sorted with multiplicities."""
    _require_cuda()
    o = _out(n, out, device)
    _check(lib().rs_sample_wr(N, n, seed % 2**64, _ptr(o), _stream(stream)))
    return o[:n]


def bernoulli_capacity(N: int, rho: float) -> int:
    return int(lib().rs_bernoulli_capacity(N, rho))


def bernoulli(N: int, rho: float, seed: int, capacity=None, out=None, device="cuda",
              stream=None, return_count=False):
    """Each of 1..N independently with probability rho, ascending."""
    _require_cuda()
    cap = bernoulli_capacity(N, rho) if capacity is None else capacity
    o = _out(cap, out, device)
    cnt = torch.zeros(1, dtype=torch.uint64, device=o.device)
    _check(lib().rs_bernoulli(N, float(rho), seed % 2**64, _ptr(o), cap, _ptr(cnt), _stream(stream)))
    if return_count:
        return o, cnt
    c = int(cnt.item())
    if c > cap:
        raise RSError(f"bernoulli: {c} values exceed capacity {cap}; retry with a larger buffer")
    return o[:c]


def shard_info(N: int, n: int, seed: int, world: int, rank: int, mode: int = MODE_WOR):
    c, off = C.c_uint64(), C.c_uint64()
    _check(lib().rs_shard_info(N, n, seed % 2**64, mode, world, rank, C.byref(c), C.byref(off)))
    return c.value, off.value


def sample_wor_shard(N, n, seed, world, rank, out=None, device="cuda", stream=None):
    _require_cuda()
    cnt, _ = shard_info(N, n, seed, world, rank, MODE_WOR)
    o = _out(cnt, out, device)
    _check(lib().rs_sample_wor_shard(N, n, seed % 2**64, world, rank, _ptr(o), _stream(stream)))
    return o[:cnt]


def sample_wr_shard(N, n, seed, world, rank, out=None, device="cuda", stream=None):
    _require_cuda()
    cnt, _ = shard_info(N, n, seed, world, rank, MODE_WR)
    o = _out(cnt, out, device)
    _check(lib().rs_sample_wr_shard(N, n, seed % 2**64, world, rank, _ptr(o), _stream(stream)))
    return o[:cnt]


def bernoulli_shard(N, rho, seed, world, rank, capacity=None, out=None, device="cuda", stream=None,
                    return_count=False):
    _require_cuda()
    cap = bernoulli_capacity(N, rho) if capacity is None else capacity
    o = _out(cap, out, device)
    cnt = torch.zeros(1, dtype=torch.uint64, device=o.device)
    _check(lib().rs_bernoulli_shard(N, float(rho), seed % 2**64, world, rank, _ptr(o), cap,
                                    _ptr(cnt), _stream(stream)))
    if return_count:
        return o, cnt
    c = int(cnt.item())
    if c > cap:
        raise RSError("bernoulli_shard: capacity exceeded")
    return o[:c]


def workspace_bytes(mode: int, N: int, n: int = 0, rho: float = 0.0, world: int = 1) -> int:
    b = C.c_size_t()
    _check(lib().rs_workspace_bytes(mode, N, n, float(rho), world, C.byref(b)))
    return b.value


def _ws_out(mode, N, n, seed, world, rank, out):
    if out is None:
        raise ValueError("out is required (a cuda uint64 tensor of the shard's count)")
    cnt, _ = shard_info(N, n, seed, world, rank, mode)
    return _out(cnt, out, None)


def sample_wor_ws(N, n, seed, world, rank, out, ws, stream=None):
    out = _ws_out(MODE_WOR, N, n, seed, world, rank, out)
    _check(lib().rs_sample_wor_ws(N, n, seed % 2**64, world, rank, _ptr(out), _ptr(ws),
                                  ws.numel() * ws.element_size(), _stream(stream)))
    return out


def sample_wr_ws(N, n, seed, world, rank, out, ws, stream=None):
    out = _ws_out(MODE_WR, N, n, seed, world, rank, out)
    _check(lib().rs_sample_wr_ws(N, n, seed % 2**64, world, rank, _ptr(out), _ptr(ws),
                                 ws.numel() * ws.element_size(), _stream(stream)))
    return out


def bernoulli_ws(N, rho, seed, world, rank, out, capacity, count, ws, stream=None):
    _check(lib().rs_bernoulli_ws(N, float(rho), seed % 2**64, world, rank, _ptr(out), capacity,
                                 _ptr(count), _ptr(ws), ws.numel() * ws.element_size(),
                                 _stream(stream)))
    return out


def sample_wor_host(N: int, n: int, seed: int, out_host=None, stream=None):
    """rs_sample_wor into a host (ideally pinned) uint64 tensor."""
    _require_cuda()
    cnt, _ = shard_info(N, n, seed, 1, 0, MODE_WOR)
    out_host = _host(cnt, out_host)
    _check(lib().rs_sample_wor_host(N, n, seed % 2**64, _ptr(out_host), _stream(stream)))
    return out_host


def sample_shard_host(mode: int, N: int, n: int, seed: int, world: int, rank: int,
                      out_host=None, stream=None):
    """The rank's slice (WOR or WR) into a host (ideally pinned) tensor."""
    _require_cuda()
    cnt, _ = shard_info(N, n, seed, world, rank, mode)
    out_host = _host(cnt, out_host)
    _check(lib().rs_sample_shard_host(mode, N, n, seed % 2**64, world, rank, _ptr(out_host),
                                      _stream(stream)))
    return out_host[:cnt]


def sample_shard_host_stream(mode: int, N: int, n: int, seed: int, world: int, rank: int,
                             out_host, stream=None):
    """The rank's slice streamed device->host through a bounded host buffer
    (rs_sample_shard_host_stream: a two-slot ring when out_host is smaller
    than the slice)."""
    _require_cuda()
    if out_host is None or out_host.is_cuda or not out_host.is_contiguous() or \
            out_host.dtype not in (torch.uint64, torch.int64):
        raise ValueError("out_host must be a contiguous CPU uint64 tensor")
    _check(lib().rs_sample_shard_host_stream(mode, N, n, seed % 2**64, world, rank, _ptr(out_host),
                                             out_host.numel(), _stream(stream)))
    return out_host


def sample_checked(mode: int, N: int, n: int, seed: int, world: int = 1, rank: int = 0, out=None,
                   device="cuda", stream=None):
    """rs_sample_checked: the (shard of the) sample, synchronised, with the
    call's own capacity status (raises RSError on RS_ECAPACITY)."""
    _require_cuda()
    cnt, _ = shard_info(N, n, seed, world, rank, mode)
    o = _out(cnt, out, device)
    _check(lib().rs_sample_checked(mode, N, n, seed % 2**64, world, rank, _ptr(o), _stream(stream)))
    return o[:cnt]


def deviates(kind: int, k: int, L: int, R: int, seed: int, id0: int, count: int, stream=None):
    """The split tree's deviates for node ids id0..id0+count-1 (0 = HGD, 1 = BIN)."""
    _require_cuda()
    o = torch.empty(count, dtype=torch.uint64, device="cuda")
    _check(lib().rs_deviates(kind, k, L, R, seed % 2**64, id0, count, _ptr(o), _stream(stream)))
    return o


def release_cache():
    """Free the host-buffer calls' cached device staging (rs_release_cache)."""
    _check(lib().rs_release_cache())


# ---- validation helpers ---------------------------------------------------

def digest(v, base_index: int = 0, stream=None) -> int:
    acc = torch.zeros(1, dtype=torch.uint64, device=v.device)
    _check(lib().rs_digest(_ptr(v), v.numel(), base_index, _ptr(acc), _stream(stream)))
    return int(acc.item())


def validate(v, N: int, strict: bool = True, stream=None) -> int:
    bad = torch.zeros(1, dtype=torch.uint64, device=v.device)
    _check(lib().rs_validate(_ptr(v), v.numel(), N, int(strict), _ptr(bad), _stream(stream)))
    return int(bad.item())


def plan(mode: int, N: int, n: int = 0, rho: float = 0.0):
    d, c, m = C.c_int(), C.c_int(), C.c_uint64()
    _check(lib().rs_plan(mode, N, n, float(rho), C.byref(d), C.byref(c), C.byref(m)))
    return d.value, bool(c.value), m.value


def device_errors(clear: bool = True) -> int:
    f = C.c_uint()
    _check(lib().rs_device_errors(int(clear), C.byref(f)))
    return f.value


OPT_LEAF_PATH = 1
OPT_TOPUP_MAX = 2
OPT_LEAF_CAP = 3
OPT_SPLIT_COOP = 4
OPT_FUSED = 5
OPT_WARP_CAP = 6


def node_info(mode: int, N: int, n: int, seed: int, depth: int, index: int):
    """(count, global_offset) of split-tree node (depth, index) (host replay)."""
    c, off = C.c_uint64(), C.c_uint64()
    _check(lib().rs_node_info(int(mode), N, n, seed % 2**64, int(depth), int(index), C.byref(c),
                              C.byref(off)))
    return c.value, off.value


def sample_node(mode: int, N: int, n: int, seed: int, depth: int, index: int, out=None,
                device="cuda", stream=None):
    """The node's slice of the full WOR / WR output (device tensor)."""
    _require_cuda()
    cnt, _ = node_info(mode, N, n, seed, depth, index)
    o = _out(cnt, out, device)
    _check(lib().rs_sample_node(int(mode), N, n, seed % 2**64, int(depth), int(index), _ptr(o),
                                _stream(stream)))
    return o[:cnt]


def gnm(V: int, m: int, seed: int, out=None, ws=None, device="cuda", stream=None):
    """G(V, m): m distinct edges as packed (u << 32) | v, lexicographic order."""
    _require_cuda()
    o = _out(m, out, device)
    _check(lib().rs_gnm(V, m, seed % 2**64, _ptr(o), _ptr(ws) if ws is not None else None,
                        ws.numel() if ws is not None else 0, _stream(stream)))
    return o[:m]


def gnp(V: int, p: float, seed: int, capacity=None, out=None, ws=None, device="cuda", stream=None):
    """G(V, p): every edge with probability p, packed (u << 32) | v, sorted."""
    _require_cuda()
    N = V * (V - 1) // 2
    cap = bernoulli_capacity(N, p) if capacity is None else capacity
    o = _out(cap, out, device)
    cnt = torch.zeros(1, dtype=torch.uint64, device=o.device)
    _check(lib().rs_gnp(V, float(p), seed % 2**64, _ptr(o), cap, _ptr(cnt), _ptr(ws) if ws is not None else None,
                        ws.numel() if ws is not None else 0, _stream(stream)))
    c = int(cnt.item())
    if c > cap:
        raise RSError("gnp: capacity exceeded")
    return o[:c]


def algb_workspace_bytes(N: int, n: int, slack: float = 4.0) -> int:
    return int(lib().rs_algb_workspace_bytes(N, n, float(slack)))


def sample_wor_algb(N: int, n: int, seed: int, slack: float = 4.0, max_attempts: int = 1000,
                    out=None, ws=None, device="cuda", stream=None, return_attempts=False):
    """NEXT-4: Algorithm B + repair (the paper's B_GPU design, P:191-208,
    P:621-637) -- a uniform sorted n-subset of 1..N, NOT the same one as
    sample_wor.  Synchronous (n' goes to the host after each Bernoulli pass).
    ws: optional uint8 device tensor of algb_workspace_bytes(N, n, slack)."""
    _require_cuda()
    o = _out(n, out, device)
    att = C.c_uint32()
    _check(lib().rs_sample_wor_algb(N, n, seed % 2**64, float(slack), int(max_attempts), _ptr(o),
                                    C.byref(att), _ptr(ws) if ws is not None else None,
                                    ws.numel() if ws is not None else 0, _stream(stream)))
    return (o[:n], att.value) if return_attempts else o[:n]


def unpack_edges(e):
    """(u, v) int64 tensors of packed edges."""
    x = e.view(torch.int64)
    return x >> 32, x & 0xFFFFFFFF


def uneven_counts(L, n: int, seed: int):
    """Per-PE sample counts for PEs owning L[i] elements: a list."""
    p = len(L)
    La = (C.c_uint64 * p)(*[int(x) for x in L])
    out = (C.c_uint64 * p)()
    _check(lib().rs_uneven_counts(p, La, int(n), seed % 2**64, out))
    return [int(v) for v in out]


def uneven_seed(seed: int, pe: int) -> int:
    return int(lib().rs_uneven_seed(seed % 2**64, int(pe)))


def uneven_local_sample(L, n: int, seed: int, pe: int, device="cuda", stream=None):
    """PE pe's share of a uniform n-subset of the union of all PEs' elements:
    sorted local element indices (1-based) on the device, and its count."""
    cnt = uneven_counts(L, n, seed)[pe]
    return sample_wor(int(L[pe]), cnt, uneven_seed(seed, pe), device=device, stream=stream), cnt


def leaf_range_nodes(D: int, lo: int, hi: int):
    """Canonical decomposition of the leaf range [lo, hi) at depth D into
    maximal aligned dyadic nodes (depth, index), left to right."""
    out = []
    while lo < hi:
        size = lo & -lo if lo else 1 << D
        while size > hi - lo:
            size >>= 1
        d = D - (size.bit_length() - 1)
        out.append((d, lo >> (D - d)))
        lo += size
    return out


def sample_range(mode: int, N: int, n: int, seed: int, leaf_lo: int, leaf_hi: int, stream=None):
    """Leaves [leaf_lo, leaf_hi) of the full output -- any contiguous slice of
    the sorted sample, e.g. for larger-than-HBM samples in batches (NEXT-1).
    Returns (device tensor, global offset of its first value)."""
    D = plan(mode, N, n)[0]
    nodes = leaf_range_nodes(D, leaf_lo, leaf_hi)
    if not nodes:
        return torch.empty(0, dtype=torch.uint64, device="cuda"), 0
    parts = [sample_node(mode, N, n, seed, d, i, stream=stream) for d, i in nodes]
    return torch.cat(parts), node_info(mode, N, n, seed, *nodes[0])[1]


def set_option(option: int, value: int):
    """Test hook (rs_set_option): OPT_LEAF_PATH 0 = automatic, 1 = CTA kernels only."""
    _check(lib().rs_set_option(int(option), int(value)))


def launch_count(reset: bool = False) -> int:
    return int(lib().rs_launch_count(int(reset)))


TIMING_CLASSES = ("split", "leaf", "bernoulli", "other")


def timing_enable(on: bool = True):
    _check(lib().rs_timing_enable(int(on)))


def timing_read(reset: bool = True):
    """{class: (ms, launches)} accumulated since the last reset (CUDA events
    recorded on each call's launch stream)."""
    ms = (C.c_double * 4)()
    cnt = (C.c_uint64 * 4)()
    _check(lib().rs_timing_read(int(reset), ms, cnt))
    return {k: (ms[i], cnt[i]) for i, k in enumerate(TIMING_CLASSES)}
