"""Frequency sharding of the EM path over GPUs.

Every stage except the V ("H") update is bin-local, so rank r owns the
contiguous, balanced bin range ``shard_bins(F, world, r)``; the only exchange
per iteration is the allreduce of the V-update numerator/denominator
(engine.cpp:125-133), done inside the library over NCCL (``dfm_comm_init``).
"""
from __future__ import annotations


def shard_bins(num_bins: int, world: int, rank: int):
    """Contiguous balanced partition: the first ``num_bins % world`` ranks get
    one extra bin.  Returns ``(f_begin, f_end)``."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("shard_bins: invalid world/rank")
    base, rem = divmod(num_bins, world)
    f0 = rank * base + min(rank, rem)
    return f0, f0 + base + (1 if rank < rem else 0)
