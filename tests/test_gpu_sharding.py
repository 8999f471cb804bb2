"""The product's frequency-sharded path driven from two processes (SURVEY.md
§8e): each rank owns one bin-shard context of the device engine (dfm_create
with its bin range) and runs the real kernels through the shard stepping API
(dfm_shard_begin / dfm_shard_numden / dfm_shard_advance / dfm_shard_end); the
one exchange per iteration - the V-update {num, den} sum over ranks,
engine.cpp:125-133 - goes through torch.distributed (gloo), where GPU ranks
use ncclAllReduce inside the library.  Both ranks share the one GPU of this
pool: their kernels never wait on each other (the exchange is on the host),
so this is a decomposition test, not a stand-in for multi-GPU timing."""
import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _rank_main(rank, world, port, x, sizes, init, iters, out):
    import sys

    sys.path.insert(0, ROOT)
    import torch
    import torch.distributed as dist

    import paper_2605_19388_b200 as dfm
    from paper_2605_19388_b200 import _capi
    from paper_2605_19388_b200.sharding import shard_bins

    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    F, T, M = x.shape
    N, _, K = init["T"].shape
    f0, f1 = shard_bins(F, world, rank)
    layout = dfm.BlockLayout(sizes)
    eng = dfm.Engine(F, T, layout, N, K, f_begin=f0, f_end=f1)
    eng.set_obs(np.ascontiguousarray(x[f0:f1]))
    eng.set_model(dfm.NmfModel(init["T"], init["V"]), init["w"], init["lam"])
    lib = _capi.load()
    _capi.check(lib.dfm_shard_begin(eng.ctx, iters), "shard_begin")
    more = 1
    buf = np.empty(2 * N * K * T)
    while more:
        _capi.check(lib.dfm_shard_numden(eng.ctx, buf.ctypes.data), "shard_numden")
        t = torch.from_numpy(buf.copy())
        dist.all_reduce(t)  # the one exchange per iteration
        nd = np.ascontiguousarray(t.numpy())
        more = _capi.check(lib.dfm_shard_advance(eng.ctx, nd.ctypes.data), "shard_advance")
    local = np.empty(iters + 1)
    fb = _capi.check(lib.dfm_shard_end(eng.ctx, local.ctypes.data), "shard_end")
    tc = torch.from_numpy(local.copy())
    dist.all_reduce(tc)  # cost partials reduced once at the end
    nmf, wb, lam = eng.get_model()
    maps = open("/proc/self/maps").read()
    out[rank] = dict(trace=tc.numpy().copy(), V=nmf.V, T=nmf.T[:, f0:f1], lam=lam[f0:f1],
                     w=[w[f0:f1] for w in wb], fb=fb, f0=f0, f1=f1,
                     native="libdfm_b200.so" in maps)
    eng.close()
    dist.destroy_process_group()


@pytest.mark.parametrize("sizes,N,K", [([4, 4, 4], 5, 16), ([2, 2], 3, 4)])
def test_two_process_product_shards_match_oracle(oracle, sizes, N, K):
    import torch
    import torch.multiprocessing as mp

    assert torch.cuda.is_available()
    F, T, iters = 37, 80, 12
    x = oracle.generate_mixture(1, F, T, sum(sizes), N, K, 31)
    init = oracle.random_init(F, T, sizes, N, K, 32)
    ref = oracle.run_engine(x, sizes, init, iters)
    mgr = mp.Manager()
    out = mgr.dict()
    port = _free_port()
    ctx = mp.get_context("spawn")
    procs = [ctx.Process(target=_rank_main, args=(r, 2, port, x, sizes, init, iters, out)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=300)
        assert p.exitcode == 0
    r0, r1 = out[0], out[1]
    assert r0["native"] and r1["native"], "each rank must run the product library"
    assert np.array_equal(r0["trace"], r1["trace"])
    c = r0["trace"]
    assert np.max(np.abs(c - ref["cost_trace"]) / np.abs(ref["cost_trace"])) < 1e-8
    assert np.all(c[1:] <= c[:-1] + 1e-9 * np.abs(c[:-1]))
    assert np.array_equal(r0["V"], r1["V"])  # V identical on every rank
    rel = lambda a, b: np.linalg.norm(a - b) / np.linalg.norm(b)
    assert rel(r0["V"], ref["V"]) < 1e-7
    assert rel(np.concatenate([r0["T"], r1["T"]], axis=1), ref["T"]) < 1e-7
    assert rel(np.concatenate([r0["lam"], r1["lam"]]), ref["lam"]) < 1e-7
    for l in range(len(sizes)):
        assert rel(np.concatenate([r0["w"][l], r1["w"][l]]), ref["w"][l]) < 1e-7
    assert r0["fb"] + r1["fb"] == ref["fallbacks"]
