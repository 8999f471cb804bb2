"""Multi-rank logic of the frequency-sharded EM path, on the CPU with gloo
(world_size 2): the oracle's bin-local stages run on each rank's shard and
the V-update numerator/denominator and the cost are allreduced, exactly as the
GPU ranks do over NCCL.  The sharded trajectory must match the
unsharded oracle engine."""
import os
import socket

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _sharded_oracle_fit(rank, world, port, x, sizes, init, iters, out):
    import sys

    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import torch
    import torch.distributed as dist

    import oracle
    from paper_2605_19388_b200.sharding import shard_bins

    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    F, T, M = x.shape
    f0, f1 = shard_bins(F, world, rank)
    xl = np.ascontiguousarray(x[f0:f1])
    Tm = np.ascontiguousarray(init["T"][:, f0:f1])
    V = init["V"].copy()
    lam = np.ascontiguousarray(init["lam"][f0:f1])
    w = [np.ascontiguousarray(b[f0:f1]) for b in init["w"]]
    offs = [int(v) for v in np.cumsum([0] + sizes[:-1])]

    def allreduce(a):
        t = torch.from_numpy(np.ascontiguousarray(a, dtype=np.float64))
        dist.all_reduce(t)
        return t.numpy()

    def power_P():
        P = np.zeros((f1 - f0, T, M))
        for l, o in enumerate(offs):
            P[:, :, o:o + sizes[l]] = oracle.decorrelate_block(xl, o, w[l])[1]
        return P

    def cost_now(P, h):
        local = oracle.power_term(P, h, lam) - T * sum(oracle.logdet_term(b) for b in w)
        return float(allreduce(np.array([local]))[0])

    h = oracle.spectrogram(Tm, V)
    eta = oracle.eta_from(h, lam)
    P = power_P()
    trace = [cost_now(P, h)]
    for _ in range(iters):
        for l, o in enumerate(offs):
            for mu in range(sizes[l]):
                w[l], _ = oracle.ip_sweep_column(xl, eta, o, w[l], mu)
        P = power_P()
        a, b = oracle.build_tv_weights(lam, P, eta)
        Tm = oracle.update_t(Tm, V, a, b)
        h = oracle.spectrogram(Tm, V)
        eta = oracle.eta_from(h, lam)
        a, b = oracle.build_tv_weights(lam, P, eta)
        nd = allreduce(oracle.update_v_partial(Tm, a, b, 0, f1 - f0))  # the one exchange
        V = oracle.update_v_apply(V, nd)
        h = oracle.spectrogram(Tm, V)
        eta = oracle.eta_from(h, lam)
        lam = oracle.update_lambda(lam, h, P, eta)
        eta = oracle.eta_from(h, lam)
        trace.append(cost_now(P, h))
    out[rank] = dict(trace=trace, V=V, T=Tm, lam=lam)
    dist.destroy_process_group()


def test_shard_bins_partition():
    from paper_2605_19388_b200.sharding import shard_bins

    for F in (1, 7, 257, 513, 1025):
        for world in (1, 2, 3, 4, 8):
            if world > F:
                continue
            parts = [shard_bins(F, world, r) for r in range(world)]
            assert parts[0][0] == 0 and parts[-1][1] == F
            assert all(parts[i][1] == parts[i + 1][0] for i in range(world - 1))
            sizes = [b - a for a, b in parts]
            assert max(sizes) - min(sizes) <= 1
    with pytest.raises(ValueError):
        shard_bins(10, 2, 2)


def test_two_rank_gloo_sharded_em_matches_unsharded(oracle):
    import torch.multiprocessing as mp

    F, T, sizes, N, K, iters = 9, 24, [2, 2], 3, 4, 6
    x = oracle.generate_mixture(1, F, T, sum(sizes), N, K, 3)
    init = oracle.random_init(F, T, sizes, N, K, 5)
    ref = oracle.run_engine(x, sizes, init, iters)
    mgr = mp.Manager()
    out = mgr.dict()
    port = _free_port()
    ctx = mp.get_context("spawn")
    procs = [ctx.Process(target=_sharded_oracle_fit, args=(r, 2, port, x, sizes, init, iters, out))
             for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=240)
        assert p.exitcode == 0
    t0, t1 = np.array(out[0]["trace"]), np.array(out[1]["trace"])
    assert np.array_equal(t0, t1)  # every rank sees the same global cost
    assert np.max(np.abs(t0 - ref["cost_trace"]) / np.abs(ref["cost_trace"])) < 1e-12
    assert np.array_equal(out[0]["V"], out[1]["V"])  # V identical on all ranks
    assert np.allclose(out[0]["V"], ref["V"], rtol=1e-11, atol=0)
    f0 = out[0]["T"].shape[1]
    assert np.allclose(np.concatenate([out[0]["T"], out[1]["T"]], axis=1), ref["T"], rtol=1e-11, atol=0)
    assert np.allclose(np.concatenate([out[0]["lam"], out[1]["lam"]]), ref["lam"], rtol=1e-11, atol=0)
    assert f0 == 5
