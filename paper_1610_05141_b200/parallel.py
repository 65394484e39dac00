"""Multi-GPU layer: Algorithm P over a torch.distributed process group.

Rank g of world p = 2^s (s <= 3) owns the dyadic range [floor(gN/p),
floor((g+1)N/p)) -- the paper's even partition made nested.  Its
sample count comes from replaying the s splits on its root path ("each PE
generates <= ceil(log p) hypergeometric random deviates") inside
librs (rs_shard_info, host arithmetic, no device).  The ONE collective is an
all-gather of the p per-rank counts (8 B each; NCCL over NVLink on the GPU
box, gloo in the CPU tests) whose exclusive prefix gives every rank its
global output offset; it is cross-checked against the replay.  The sample
itself never moves: communication is independent of n.

Argument marshalling and plumbing only -- every sampling step runs in librs.
"""
from __future__ import annotations

import torch
import torch.distributed as dist

from . import MODE_WOR, MODE_WR, bernoulli_shard, sample_wor_shard, sample_wr_shard, shard_info


def _group_info(group=None):
    return dist.get_world_size(group), dist.get_rank(group)


def _coll_device(group=None):
    """Device of the collective's tensors: the current GPU under NCCL, the
    host under gloo (gloo's all-gather takes CPU tensors)."""
    if dist.get_backend(group) == "nccl":
        return torch.device("cuda", torch.cuda.current_device())
    return torch.device("cpu")


def allgather_counts(local_count: int, group=None, device=None) -> torch.Tensor:
    """All-gather of one u64 count per rank (the path's only collective)."""
    world, _ = _group_info(group)
    dev = device if device is not None else torch.device("cpu")
    mine = torch.tensor([int(local_count)], dtype=torch.int64, device=dev)
    allc = torch.empty(world, dtype=torch.int64, device=dev)
    dist.all_gather_into_tensor(allc, mine, group=group)
    return allc


def shard_offsets(N: int, n: int, seed: int, mode: int = MODE_WOR, group=None, device=None):
    """(local_count, global_offset, all_counts) of this rank.  The replayed
    offset must equal the exclusive prefix of the all-gathered counts."""
    world, rank = _group_info(group)
    cnt, off = shard_info(N, n, seed, world, rank, mode)
    allc = allgather_counts(cnt, group, device)
    prefix = int(allc[:rank].sum().item())
    if prefix != off:
        raise RuntimeError(f"rank {rank}: all-gathered offset {prefix} != Algorithm P replay {off}")
    if int(allc.sum().item()) != n:
        raise RuntimeError(f"rank {rank}: counts sum to {int(allc.sum().item())}, expected n = {n}")
    return cnt, off, allc


def sample(N: int, n: int, seed: int, mode: int = MODE_WOR, group=None, stream=None):
    """This rank's slice of the world's sample (device tensor) and its global
    offset.  Identical for every world size when concatenated in rank order."""
    world, rank = _group_info(group)
    cnt, off, _ = shard_offsets(N, n, seed, mode, group, _coll_device(group))
    f = sample_wr_shard if mode == MODE_WR else sample_wor_shard
    return f(N, n, seed, world, rank, stream=stream), off


def bernoulli(N: int, rho: float, seed: int, group=None, stream=None):
    """This rank's Bernoulli slice and its global offset: counts are only known
    after generation, so the all-gather follows the kernel."""
    world, rank = _group_info(group)
    vals, cnt = bernoulli_shard(N, rho, seed, world, rank, stream=stream, return_count=True)
    c = int(cnt.item())
    if c > vals.numel():
        raise RuntimeError("bernoulli shard: capacity exceeded")
    allc = allgather_counts(c, group, _coll_device(group))
    return vals[:c], int(allc[:rank].sum().item())


def uneven_sample(L_local: int, n: int, seed: int, group=None, stream=None):
    """NEXT-2: every rank owns L_local elements; returns this
    rank's sorted local element indices (1-based, device) of a uniform
    n-subset of the union, plus (its count, all ranks' L).  The paper's
    binomial-tree messages become one all-gather of the L values; each rank
    then replays the whole count tree (rs_uneven_counts) -- every rank
    derives the same counts."""
    from . import uneven_local_sample
    world, rank = _group_info(group)
    allL = allgather_counts(L_local, group, _coll_device(group))
    L = [int(v) for v in allL.tolist()]
    vals, cnt = uneven_local_sample(L, n, seed, rank, stream=stream)
    return vals, cnt, L

