"""parallel.sample / parallel.bernoulli / parallel.uneven_sample under a
world-size-2 gloo group whose ranks share cuda:0 -- -m gpu.  The ranks' kernels
never wait on each other (the only collective is gloo's all-gather of counts on
the host), so sharing one GPU is safe.  The concatenated rank slices must equal
the single-call sample (p-independence) and the offsets the
Algorithm P replay."""
from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    try:
        import torch
        import torch.distributed as dist
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        torch.cuda.set_device(0)
        dist.init_process_group("gloo", rank=rank, world_size=world)
        from paper_1610_05141_b200 import parallel as P
        import paper_1610_05141_b200 as rs
        a, off_a = P.sample(2 ** 30, 2 ** 20, 5, rs.MODE_WOR)
        b, off_b = P.sample(2 ** 24, 2 ** 20, 5, rs.MODE_WR)
        c, off_c = P.bernoulli(2 ** 24, 0.01, 5)
        u, cnt_u, L = P.uneven_sample(1000 * (rank + 1), 700, 5)
        torch.cuda.synchronize()
        q.put((rank, off_a, a.cpu().numpy(), off_b, b.cpu().numpy(), off_c, c.cpu().numpy(),
               cnt_u, u.cpu().numpy(), L))
        dist.barrier()
        dist.destroy_process_group()
    except Exception as e:
        q.put((rank, "error", repr(e)))


def test_parallel_gloo_two_ranks_on_one_gpu():
    import oracle as O
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = {}
    for _ in range(2):
        item = q.get(timeout=300)
        assert item[1] != "error", item
        res[item[0]] = item
    for p in procs:
        p.join(timeout=60)
    r0, r1 = res[0], res[1]
    assert r0[1] == 0 and r1[1] == r0[2].size
    assert np.array_equal(np.concatenate([r0[2], r1[2]]), O.sample_wor(2 ** 30, 2 ** 20, 5))
    assert r1[3] == r0[4].size
    assert np.array_equal(np.concatenate([r0[4], r1[4]]), O.sample_wr(2 ** 24, 2 ** 20, 5))
    assert r1[5] == r0[6].size
    assert np.array_equal(np.concatenate([r0[6], r1[6]]), O.bernoulli(2 ** 24, 0.01, 5))
    L = r0[9]
    assert L == [1000, 2000] and r1[9] == L
    counts = O.uneven_counts(L, 700, 5)
    assert r0[7] == counts[0] and r1[7] == counts[1]
