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


def fit_sharded_host(engines, iters: int):
    """Runs one EM fit over bin-shard Engines (each created with its
    ``f_begin/f_end``) in lockstep, summing the V-update numerator/denominator
    on the host where the GPU ranks use ncclAllReduce (same order of
    operations per shard).  Returns the global cost trace and the fallback
    count.  Used to verify the sharded decomposition on one device."""
    import numpy as np

    from . import _capi

    lib = _capi.load()
    nd = None
    for e in engines:
        _capi.check(lib.dfm_shard_begin(e.ctx, iters), "shard_begin")
    more = 1
    while more:
        parts = []
        for e in engines:
            buf = np.empty(2 * e.N * e.K * e.T)
            _capi.check(lib.dfm_shard_numden(e.ctx, buf.ctypes.data), "shard_numden")
            parts.append(buf)
        nd = parts[0].copy()
        for p in parts[1:]:
            nd += p
        for e in engines:
            more = _capi.check(lib.dfm_shard_advance(e.ctx, nd.ctypes.data), "shard_advance")
    cost = np.zeros(iters + 1)
    fb = 0
    for e in engines:
        local = np.empty(iters + 1)
        fb += _capi.check(lib.dfm_shard_end(e.ctx, local.ctypes.data), "shard_end")
        cost += local
    return cost, fb
