"""The N > 1 host path on CPU: world_size 2 and 4 `gloo` process groups run
paper_1610_05141_b200.parallel.shard_offsets -- Algorithm P replay in librs
(host arithmetic) plus the one all-gather of counts -- and
check it against the independent oracle's per-rank replay and the invariants
(counts sum to n; offsets are the exclusive prefix).  -m "not gpu"."""
from __future__ import annotations

import os
import socket

import pytest
import torch.multiprocessing as mp

CASES = [(2 ** 48, 2 ** 32, 1, 0), (2 ** 40, 2 ** 30, 7, 0), (2 ** 36, 2 ** 32, 1, 1),
         (2 ** 32, 3 * 2 ** 30, 1, 0), (1000, 500, 3, 0), (12345, 6173, 5, 0), (7, 3, 2, 1)]


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, errq):
    try:
        import torch.distributed as dist
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        dist.init_process_group("gloo", rank=rank, world_size=world)
        import oracle as O
        from paper_1610_05141_b200 import parallel as P
        for N, n, seed, mode in CASES:
            cnt, off, allc = P.shard_offsets(N, n, seed, mode)
            ec, eo = O.shard_info(N, n, seed, world, rank, mode)
            assert (cnt, off) == (ec, eo), (N, n, seed, mode, rank, cnt, off, ec, eo)
            assert int(allc.sum()) == n
        # NEXT-2: all-gather of the L values, then the same count replay on every rank
        import paper_1610_05141_b200 as rs
        Lmine = [17, 3, 40, 25][rank % 4] * (rank + 1)
        allL = P.allgather_counts(Lmine)
        L = [int(v) for v in allL.tolist()]
        counts = rs.uneven_counts(L, sum(L) // 3, 9)
        assert counts == [int(v) for v in O.uneven_counts(L, sum(L) // 3, 9)]
        dist.destroy_process_group()
    except Exception as e:  # report to the parent
        errq.put(f"rank {rank}: {e!r}")


@pytest.mark.parametrize("world", [2, 4])
def test_shard_offsets_gloo(world):
    ctx = mp.get_context("spawn")
    errq = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, errq)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=240)
    errs = []
    while not errq.empty():
        errs.append(errq.get())
    assert not errs, errs
    assert all(p.exitcode == 0 for p in procs)
