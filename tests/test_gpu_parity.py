"""GPU parity: the sm_100a kernels (through the C ABI) against the CPU oracle,
on the same seeded inputs, plus the reference's own known-answer tests run on
the device path.  Tolerances follow BASELINE.json's north_star:
  * cost (negative log-likelihood) trajectory within 1e-8 relative over the
    first 20 iterations,
  * separated STFTs within 1e-6 relative L2,
  * cost non-increase every iteration (1e-9 relative slack, as the reference's
    tests allow).
Per-step kernels are compared at 1e-10 (they differ from the oracle only in
floating-point summation order and FMA contraction).
"""
import os

import numpy as np
import pytest

import naive

pytestmark = pytest.mark.gpu

TRAJ_RTOL = 1e-8
STEP_RTOL = 1e-10


@pytest.fixture(scope="module")
def dfm():
    import torch

    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    import paper_2605_19388_b200 as m

    m._capi.load()
    return m


def _init_dict(init):
    return dict(T=init.nmf.T, V=init.nmf.V, lam=init.lambda0, w=init.w0)


def _rel(a, b):
    return np.linalg.norm(np.asarray(a) - np.asarray(b)) / max(np.linalg.norm(np.asarray(b)), 1e-300)


def _inst(oracle, F, T, M, N, K, seed, sizes=None):
    import paper_2605_19388_b200 as m

    x, Tm, V, lam, w = oracle.random_instance(F, T, M, N, K, seed)
    sizes = sizes or [M]
    blocks, o = [], 0
    for mb in sizes:
        blocks.append(np.ascontiguousarray(w[:, o:o + mb, o:o + mb]))
        o += mb
    layout = m.BlockLayout(sizes)
    init = m.InitBundle(layout, m.NmfModel(Tm, V), blocks, lam)
    return x, layout, init


# ------------------------------------------------------------ step kernels
def test_step_spectrogram_eta_decorrelate(dfm, oracle):
    x, layout, init = _inst(oracle, 5, 37, 4, 3, 5, 1, [2, 2])
    h = dfm.build_spectrogram(init.nmf)
    assert _rel(h, oracle.spectrogram(init.nmf.T, init.nmf.V)) < STEP_RTOL
    eta = dfm.compute_eta(init.nmf, init.lambda0)
    assert _rel(eta, oracle.eta_from(oracle.spectrogram(init.nmf.T, init.nmf.V), init.lambda0)) < STEP_RTOL
    y, P = dfm.decorrelate_blocks(x, layout, init.w0)
    for l, o in enumerate(layout.offsets):
        yr, Pr = oracle.decorrelate_block(x, o, init.w0[l])
        assert _rel(y[:, :, o:o + 2], yr) < STEP_RTOL
        assert _rel(P[:, :, o:o + 2], Pr) < STEP_RTOL


@pytest.mark.parametrize("sizes", [[3], [2, 3, 1], [4, 4], [12]])
def test_step_ip_column_matches_oracle(dfm, oracle, sizes):
    M = sum(sizes)
    x, layout, init = _inst(oracle, 6, 50, M, 2, 3, 7, sizes)
    eta = dfm.compute_eta(init.nmf, init.lambda0)
    for l, (o, mb) in enumerate(zip(layout.offsets, layout.sizes)):
        w_gpu = init.w0[l].copy()
        w_ref = init.w0[l].copy()
        for mu in range(mb):
            dfm.ip_update_block(x, eta, layout, l, w_gpu, mu)
            w_ref, _ = oracle.ip_sweep_column(x, eta, o, w_ref, mu)
        assert _rel(w_gpu, w_ref) < 1e-9


def test_step_ip_fallback_on_singular_system(dfm, oracle):
    # silent + duplicated channel (test_fastmnmf.cpp:377-404): Q singular -> pinv path
    x, layout, init = _inst(oracle, 3, 10, 4, 2, 2, 77)
    x[:, :, 1] = 0
    x[:, :, 3] = x[:, :, 2]
    eta = dfm.compute_eta(init.nmf, init.lambda0)
    w_gpu = init.w0[0].copy()
    w_ref = init.w0[0].copy()
    fb_gpu = fb_ref = 0
    for mu in range(4):
        fb_gpu += dfm.ip_update_w(x, eta, w_gpu, mu)
        w_ref, f = oracle.ip_sweep_column(x, eta, 0, w_ref, mu)
        fb_ref += f
    assert fb_gpu == fb_ref and fb_gpu > 0
    assert np.all(np.isfinite(w_gpu))
    assert _rel(w_gpu, w_ref) < 1e-8


def test_step_mm_updates_match_oracle(dfm, oracle):
    x, layout, init = _inst(oracle, 5, 23, 3, 2, 4, 23)
    P = np.abs(naive.decorrelate(x, init.w0[0])) ** 2
    for which in ("t", "v", "lambda"):
        nmf = init.nmf.copy()
        lam = init.lambda0.copy()
        eta = dfm.compute_eta(nmf, lam)
        eta_ref = eta.copy()
        if which == "t":
            dfm.mm_update_t(nmf, lam, P, eta)
            a, b = oracle.build_tv_weights(lam, P, eta_ref)
            ref = oracle.update_t(init.nmf.T, init.nmf.V, a, b)
            assert _rel(nmf.T, ref) < STEP_RTOL
        elif which == "v":
            dfm.mm_update_v(nmf, lam, P, eta)
            a, b = oracle.build_tv_weights(lam, P, eta_ref)
            ref = oracle.update_v(init.nmf.T, init.nmf.V, a, b)
            assert _rel(nmf.V, ref) < STEP_RTOL
        else:
            dfm.mm_update_lambda(nmf, lam, P, eta)
            ref = oracle.update_lambda(init.lambda0, oracle.spectrogram(init.nmf.T, init.nmf.V), P, eta_ref)
            assert _rel(lam, ref) < STEP_RTOL


def test_step_cost_matches_oracle_and_raises_on_singular(dfm, oracle):
    for seed in range(4):
        x, layout, init = _inst(oracle, 3, 9, 6, 2, 2, seed + 10, [2, 3, 1])
        spatial = dfm.BlockSpatialModel(layout, init.w0, init.lambda0)
        got = dfm.cost_dist(x, init.nmf, spatial)
        ref = oracle.cost_dist(x, [2, 3, 1], _init_dict(init))
        assert got == pytest.approx(ref, rel=1e-12)
    x, layout, init = _inst(oracle, 2, 4, 2, 1, 1, 3)
    init.w0[0][1] = 0
    with pytest.raises(dfm.SingularDemixerError):
        dfm.cost_full(x, init.nmf, dfm.SpatialModel(init.w0[0], init.lambda0))


def test_step_wiener_matches_oracle(dfm, oracle):
    x, layout, init = _inst(oracle, 4, 19, 6, 3, 2, 47, [2, 3, 1])
    spatial = dfm.BlockSpatialModel(layout, init.w0, init.lambda0)
    got = dfm.wiener_block(x, init.nmf, spatial).images
    ref = oracle.wiener_block(x, [2, 3, 1], _init_dict(init))
    assert _rel(got, ref) < 1e-12
    assert np.linalg.norm(got.sum(0) - x) <= 1e-9 * np.linalg.norm(x)


# ------------------------------------------------------------ fused engine
ENGINE_CASES = [
    # (F, T, sizes, N, K, iters)
    (7, 33, [2, 2], 3, 4, 20),
    (9, 41, [2, 3, 1], 2, 2, 20),
    (5, 64, [4, 4, 4], 5, 16, 20),
    (4, 30, [12], 5, 16, 20),
    (6, 25, [1, 1, 1], 3, 3, 20),
    # limits and ragged shapes: N = 8, K = 64, a 16-mic block, one bin /
    # one frame, odd frame counts that do not fill a tile
    (3, 17, [16], 8, 64, 10),
    (2, 5, [3, 5], 8, 32, 10),
    (1, 4, [2], 2, 3, 5),
    (11, 257, [4, 4], 6, 20, 10),
    (5, 130, [8, 8], 4, 9, 10),
]


@pytest.mark.parametrize("F,T,sizes,N,K,iters", ENGINE_CASES)
def test_engine_trajectory_matches_oracle(dfm, oracle, F, T, sizes, N, K, iters):
    layout = dfm.BlockLayout(sizes)
    x = dfm.generate_mixture(1, F, T, layout.total, N, K, 3)
    init = dfm.random_init(F, T, layout, N, K, 5)
    fit = dfm.fit_distributed(x, layout, init, iters, True)
    ref = oracle.run_engine(x, sizes, _init_dict(init), iters)
    c, r = fit.report.cost_trace, ref["cost_trace"]
    assert c.shape == (iters + 1,)
    assert np.max(np.abs(c - r) / np.abs(r)) < TRAJ_RTOL
    assert np.all(c[1:] <= c[:-1] + 1e-9 * np.abs(c[:-1]))
    assert fit.report.fallbacks == ref["fallbacks"]
    assert _rel(fit.models[0].T, ref["T"]) < 1e-7
    assert _rel(fit.models[0].V, ref["V"]) < 1e-7
    assert _rel(fit.spatial.Lambda, ref["lam"]) < 1e-7
    for a, b in zip(fit.spatial.W, ref["w"]):
        assert _rel(a, b) < 1e-7


@pytest.mark.parametrize("FT,TB,sizes", [(32, 32, [4, 4, 4]), (64, 64, [4, 4, 4]), (128, 128, [4, 4, 4]),
                                         (256, 32, [4, 4, 4]), (96, 64, [4, 4, 4]), (512, 128, [4, 4, 4]),
                                         (160, 128, [4, 4, 4]), (96, 128, [12]), (160, 64, [12]),
                                         (192, 128, [12])])
def test_engine_tilings_agree(dfm, oracle, FT, TB, sizes):
    F, T, N, K, iters = 11, 70, 5, 8, 10
    layout = dfm.BlockLayout(sizes)
    x = dfm.generate_mixture(1, F, T, layout.total, N, K, 9)
    init = dfm.random_init(F, T, layout, N, K, 2)
    with dfm.Engine(F, T, layout, N, K) as eng:
        eng.set_tiling(FT, TB)
        t = eng.tiling()
        assert (t["frame_tile"], t["pd_frames"]) == (FT, TB)
        eng.set_obs(x)
        eng.set_model(init.nmf, init.w0, init.lambda0)
        cost, _, _, _ = eng.fit(iters)
    ref = oracle.run_engine(x, sizes, _init_dict(init), iters)
    assert np.max(np.abs(cost - ref["cost_trace"]) / np.abs(ref["cost_trace"])) < TRAJ_RTOL


def test_engine_is_deterministic_and_l1_reduction(dfm, oracle):
    # test_fastmnmf.cpp:364-366 bitwise determinism; test_dist.cpp:166-182 L=1
    x, layout, init = _inst(oracle, 4, 14, 4, 2, 3, 61)
    a = dfm.fit_full(x, init, 25)
    b = dfm.fit_distributed(x, layout, init, 25, True)
    assert np.array_equal(a.report.cost_trace, b.report.cost_trace)
    assert np.array_equal(a.nmf.T, b.models[0].T) and np.array_equal(a.nmf.V, b.models[0].V)
    assert np.array_equal(a.spatial.W, b.spatial.W[0])
    c = dfm.fit_full(x, init, 25)
    assert np.array_equal(a.report.cost_trace, c.report.cost_trace)


def test_engine_zero_iterations_and_final_cost(dfm, oracle):
    # test_fastmnmf.cpp:351-375
    x, layout, init = _inst(oracle, 4, 12, 3, 2, 2, 55)
    f0 = dfm.fit_full(x, init, 0)
    assert f0.report.cost_trace.shape == (1,)
    assert f0.report.cost_trace[0] == pytest.approx(
        dfm.cost_full(x, init.nmf, dfm.SpatialModel(init.w0[0], init.lambda0)), rel=1e-12)
    a = dfm.fit_full(x, init, 30)
    assert a.report.wall_seconds.shape == (30,)
    final = dfm.cost_full(x, a.nmf, a.spatial)
    assert final == pytest.approx(a.report.cost_trace[-1], rel=1e-12)


@pytest.mark.parametrize("M", [4, 8])
def test_engine_adversarial_stays_finite(dfm, oracle, M):
    # test_fastmnmf.cpp:377-404 — exercises the device pinv fallback (M = 4:
    # the quad fast path; M = 8: the warp fast path with precomputed inverses)
    x, layout, init = _inst(oracle, 3, 10, M, 2, 2, 77)
    x[:, :, 1] = 0
    x[:, :, 3] = x[:, :, 2]
    fit = dfm.fit_full(x, init, 60)
    for a in (fit.nmf.T, fit.nmf.V, fit.spatial.Lambda):
        assert np.all(np.isfinite(a)) and a.min() >= dfm.kFloor
    assert np.all(np.isfinite(fit.spatial.W))
    assert not np.any(np.isnan(fit.report.cost_trace))
    assert fit.report.fallbacks > 0
    ref = oracle.run_engine(x, [M], _init_dict(init), 60)
    assert fit.report.fallbacks == ref["fallbacks"]
    c, r = fit.report.cost_trace, ref["cost_trace"]
    fin = np.isfinite(r)  # a singular W gives the reference's +inf cost
    assert np.array_equal(np.isfinite(c), fin) and np.array_equal(c[~fin], r[~fin])
    assert np.all(np.abs(c[fin] - r[fin]) <= 1e-6 * np.abs(r[fin]))


def test_engine_underdetermined_and_independent_mode(dfm, oracle):
    # test_dist.cpp:184-229
    x, layout, init = _inst(oracle, 3, 10, 4, 3, 2, 81, [2, 2])
    fit = dfm.fit_distributed(x, layout, init, 40, True)
    c = fit.report.cost_trace
    assert np.all(c[1:] <= c[:-1] + 1e-9 * np.abs(c[:-1]))
    x, layout, init = _inst(oracle, 3, 12, 5, 2, 2, 71, [3, 2])
    dist = fit_ind = dfm.fit_distributed(x, layout, init, 20, False)
    assert not dist.shared and len(dist.models) == 2
    for l in range(2):
        single = dfm.fit_single(dfm.extract_block(x, layout, l), dfm.slice_init(init, l), 20)
        assert np.array_equal(single.nmf.T, dist.models[l].T)
        assert np.array_equal(single.spatial.W, dist.spatial.W[l])
    final = dfm.cost_dist(x, fit_ind.models, fit_ind.spatial)
    assert final == pytest.approx(fit_ind.report.cost_trace[-1], rel=1e-10)


@pytest.mark.parametrize("sizes,N,K", [([2, 2], 3, 4), ([4, 4, 4], 5, 4), ([12], 5, 4), ([8, 3], 4, 4)])
def test_engine_wiener_matches_oracle_after_fit(dfm, oracle, sizes, N, K):
    """Engine.wiener on the static kernels (in-CTA (W^H)^-1 for blocks <= 4
    mics; the warp Gauss-Jordan inverse for the 12-mic block) and the generic
    kernel (8 + 3 mics)."""
    F, T = 8, 45
    layout = dfm.BlockLayout(sizes)
    # the BASELINE generator of configs 1-3 (rank-1 + diffuse source SCMs);
    # the rank-deficient config-0 generator on a 12-mic block is intrinsically
    # ill-conditioned, see test_wiener_drift_is_the_problems_own_sensitivity
    x = dfm.generate_mixture(1, F, T, layout.total, N, K, 1)
    init = dfm.random_init(F, T, layout, N, K, 2)
    with dfm.Engine(F, T, layout, N, K) as eng:
        eng.set_obs(x)
        eng.set_model(init.nmf, init.w0, init.lambda0)
        eng.fit(30)
        img = eng.wiener()
        nmf, wb, lam = eng.get_model()
    ref = oracle.run_engine(x, sizes, _init_dict(init), 30)
    ref_img = oracle.wiener_block(x, sizes, ref)
    assert _rel(img, ref_img) < 1e-6  # north_star: separated STFTs within 1e-6
    assert np.linalg.norm(img.sum(0) - x) <= 1e-9 * np.linalg.norm(x)
    with dfm.Engine(F, T, layout, N, K) as eng:
        eng.set_obs(x)
        eng.set_model(dfm.NmfModel(ref["T"], ref["V"]), [np.asarray(w) for w in ref["w"]], ref["lam"])
        img2 = eng.wiener()
    assert _rel(img2, ref_img) < 1e-10


def test_eval_callback_chunks_match_single_run(dfm, oracle):
    x, layout, init = _inst(oracle, 4, 16, 4, 2, 2, 91, [2, 2])
    seen = []
    opts = dfm.FitOptions(eval_every=5, on_eval=lambda s: seen.append((s.iteration, s.cost)))
    a = dfm.fit_distributed(x, layout, init, 15, True, opts)
    b = dfm.fit_distributed(x, layout, init, 15, True)
    assert [s[0] for s in seen] == [5, 10, 15]
    assert np.allclose(a.report.cost_trace, b.report.cost_trace, rtol=1e-13, atol=0)
    assert seen[-1][1] == a.report.cost_trace[-1]


@pytest.mark.parametrize("sizes,N,K", [([2, 2], 3, 4), ([4, 4, 4], 5, 16), ([12], 5, 16), ([4] * 8, 8, 32)])
def test_static_shape_kernels_match_generic_and_oracle(dfm, oracle, sizes, N, K):
    """The compile-time-shape k_bin instantiations (BASELINE configs 0-3) and
    the generic runtime-shape kernel both track the oracle."""
    F, T, iters = 9, 57, 12
    layout = dfm.BlockLayout(sizes)
    x = dfm.generate_mixture(1, F, T, layout.total, N, K, 4)
    init = dfm.random_init(F, T, layout, N, K, 8)
    ref = oracle.run_engine(x, sizes, _init_dict(init), iters)
    costs = []
    for generic in (0, 1):
        with dfm.Engine(F, T, layout, N, K) as eng:
            dfm._capi.check(eng.lib.dfm_force_generic(eng.ctx, generic))
            eng.set_obs(x)
            eng.set_model(init.nmf, init.w0, init.lambda0)
            cost, _, _, _ = eng.fit(iters)
            costs.append(cost)
            nmf, wb, lam = eng.get_model()
        assert np.max(np.abs(cost - ref["cost_trace"]) / np.abs(ref["cost_trace"])) < TRAJ_RTOL
        assert _rel(nmf.V, ref["V"]) < 1e-7 and _rel(lam, ref["lam"]) < 1e-7
    assert np.max(np.abs(costs[0] - costs[1]) / np.abs(costs[1])) < TRAJ_RTOL


@pytest.mark.parametrize("nshards", [2, 3])
def test_frequency_sharded_engine_matches_single_gpu(dfm, oracle, nshards):
    """SURVEY §8e on one device: bin-shard contexts run the real kernels in
    lockstep and exchange the V-update {num, den} on the host (the GPU ranks
    use ncclAllReduce).  The global trajectory and fitted model must match the
    unsharded engine and the oracle."""
    from paper_2605_19388_b200.sharding import fit_sharded_host, shard_bins

    F, T, sizes, N, K, iters = 17, 48, [4, 4, 4], 5, 16, 12
    layout = dfm.BlockLayout(sizes)
    x = dfm.generate_mixture(1, F, T, layout.total, N, K, 21)
    init = dfm.random_init(F, T, layout, N, K, 22)
    engines = []
    for r in range(nshards):
        f0, f1 = shard_bins(F, nshards, r)
        e = dfm.Engine(F, T, layout, N, K, f_begin=f0, f_end=f1)
        e.set_obs(x[f0:f1])
        e.set_model(init.nmf, init.w0, init.lambda0)
        engines.append(e)
    cost, fb = fit_sharded_host(engines, iters)
    ref = oracle.run_engine(x, sizes, _init_dict(init), iters)
    assert np.max(np.abs(cost - ref["cost_trace"]) / np.abs(ref["cost_trace"])) < TRAJ_RTOL
    # V is identical on every shard; T / Lambda / W of each shard's bins match the oracle
    Vs = [e.get_model()[0].V for e in engines]
    for v in Vs[1:]:
        assert np.array_equal(v, Vs[0])
    assert _rel(Vs[0], ref["V"]) < 1e-7
    for r, e in enumerate(engines):
        f0, f1 = shard_bins(F, nshards, r)
        nmf, wb, lam = e.get_model()
        assert _rel(nmf.T[:, f0:f1], ref["T"][:, f0:f1]) < 1e-7
        assert _rel(lam[f0:f1], ref["lam"][f0:f1]) < 1e-7
        e.close()


def test_binding_mirror_fit_is_monotone(dfm):
    # proj/python/tests/test_smoke.py:40-48 through the _fastmnmf mirror
    from paper_2605_19388_b200 import _fastmnmf

    rng = np.random.default_rng(3)
    x = (rng.standard_normal((16, 48, 4)) + 1j * rng.standard_normal((16, 48, 4))) / np.sqrt(2)
    report = _fastmnmf.fit_distributed(x, partition=[2, 2], n_sources=2, k_bases=4, iterations=15, seed=5)
    trace = np.asarray(report["cost_trace"])
    assert trace.shape == (16,)
    assert np.all(np.diff(trace) <= 1e-9 * np.abs(trace[:-1]))
    assert set(report) == {"cost_trace", "wall_seconds", "iterations", "stages"}
    full = _fastmnmf.fit_full(x, n_sources=2, k_bases=4, iterations=5, seed=1)
    assert len(full["cost_trace"]) == 6
    with pytest.raises(ValueError):
        _fastmnmf.fit_full(np.zeros((3, 4)), n_sources=2)


def test_fit_many_matches_individual_fits(dfm, oracle):
    # BASELINE config 4 path: independent mixtures fitted together (one
    # context and stream each, launches interleaved) give bitwise the results
    # of fitting each alone, and each trace matches the oracle
    F, T, N, K, sizes = 257, 200, 3, 4, [2, 2]
    engines, inits, xs = [], [], []
    for j in range(3):
        x = dfm.generate_mixture(0, F, T, 4, N, K, 700 + j)
        layout = dfm.BlockLayout(sizes)
        init = dfm.random_init(F, T, layout, N, K, 900 + j)
        e = dfm.Engine(F, T, layout, N, K)
        e.set_obs(x)
        e.set_model(init.nmf, init.w0, init.lambda0)
        engines.append(e)
        inits.append(init)
        xs.append(x)
    costs, secs, fb = dfm.fit_many(engines, 12)
    assert costs.shape == (3, 13) and secs > 0 and fb >= 0
    for j, (e, x, init) in enumerate(zip(engines, xs, inits)):
        nmf, w, lam = e.get_model()
        e2 = dfm.Engine(F, T, dfm.BlockLayout(sizes), N, K)
        e2.set_obs(x)
        e2.set_model(init.nmf, init.w0, init.lambda0)
        c2, _, _, _ = e2.fit(12)
        assert np.array_equal(costs[j], c2)
        nmf2, w2, lam2 = e2.get_model()
        assert np.array_equal(nmf.T, nmf2.T) and np.array_equal(nmf.V, nmf2.V) and np.array_equal(lam, lam2)
        r = oracle.run_engine(x, sizes, _init_dict(init), 12)
        assert _rel(costs[j], r["cost_trace"]) < TRAJ_RTOL
        assert np.all(np.diff(costs[j]) <= 1e-9 * np.abs(costs[j][:-1]))
        e.close()
        e2.close()


def test_nccl_collective_path_matches_single_gpu(dfm, oracle):
    # the frequency-sharded device path -- V-update {num, den} through
    # ncclAllReduce, k_vapply, a separate H = T V launch -- on a one-rank
    # communicator gives bitwise the single-GPU (fused, graph-replayed) fit
    import ctypes

    F, T, N, K, sizes = 40, 52, 3, 4, [2, 2]
    x = dfm.generate_mixture(0, F, T, 4, N, K, 81)
    layout = dfm.BlockLayout(sizes)
    init = dfm.random_init(F, T, layout, N, K, 82)
    runs = []
    for collective in (False, True):
        e = dfm.Engine(F, T, layout, N, K)
        if collective:
            buf = ctypes.create_string_buffer(128)
            dfm._capi.check(e.lib.dfm_nccl_get_unique_id(buf))
            e.comm_init(buf.raw, 1, 0)
            dfm._capi.check(e.lib.dfm_force_collective(e.ctx, 1))
        e.set_obs(x)
        e.set_model(init.nmf, init.w0, init.lambda0)
        cost, _, _, _ = e.fit(15)
        runs.append((cost, e.get_model()))
        e.close()
    (c0, (n0, w0, l0)), (c1, (n1, w1, l1)) = runs
    assert np.array_equal(c0, c1)
    assert np.array_equal(n0.T, n1.T) and np.array_equal(n0.V, n1.V) and np.array_equal(l0, l1)
    assert all(np.array_equal(a, b) for a, b in zip(w0, w1))
    maps = open("/proc/self/maps").read()
    assert "libnccl" in maps, "the collective path must have loaded NCCL"


def test_fit_reports_operation_counts(dfm, oracle):
    # test_bench.cpp:34-52 through the fits: full M=6 and distributed {2,2,2}
    # (shared and independent spectrograms count the same W-stage work)
    x, layout, init = _inst(oracle, 4, 16, 6, 2, 2, 17, [6])
    r = dfm.fit_full(x, init, 2).report
    assert r.ops["w_update"] == pytest.approx(4.0 * 2 * (6 ** 4 + 16.0 * 6 ** 3))
    x, layout, init = _inst(oracle, 4, 16, 6, 2, 2, 17, [2, 2, 2])
    for shared in (True, False):
        r = dfm.fit_distributed(x, layout, init, 2, shared).report
        assert r.ops["w_update"] == pytest.approx(4.0 * 2 * 3 * (2 ** 4 + 16.0 * 2 ** 3))


def _wiener_paths(dfm, x, T, V, lam, w_blocks, sizes):
    """Both device Wiener paths: the step kernel (wiener_block) and the engine
    context kernel (Engine.wiener, k_wiener_ctx incl. the in-CTA inverse)."""
    layout = dfm.BlockLayout(sizes)
    a = dfm.wiener_block(x, dfm.NmfModel(T, V), dfm.BlockSpatialModel(layout, w_blocks, lam)).images
    F, Tn, _ = x.shape
    e = dfm.Engine(F, Tn, layout, T.shape[0], T.shape[2])
    e.set_obs(x)
    e.set_model(dfm.NmfModel(T, V), w_blocks, lam)
    b = e.wiener()
    e.close()
    return a, b


def test_wiener_reference_cases_on_device(dfm, oracle):
    # test_wiener.cpp:39-141 on both device paths
    x, T, V, lam, w = oracle.random_instance(3, 6, 3, 1, 2, 1)  # single source passes through
    for s in _wiener_paths(dfm, x, T, V, lam, [w], [3]):
        assert np.linalg.norm(s[0] - x) <= 1e-12 * np.linalg.norm(x)
    x, T, V, lam, w = oracle.random_instance(2, 5, 3, 2, 2, 3)  # equal sources split in half
    T[1] = T[0]
    V[1] = V[0]
    lam[:, 1] = lam[:, 0]
    for s in _wiener_paths(dfm, x, T, V, lam, [w], [3]):
        for n in range(2):
            assert np.linalg.norm(s[n] - 0.5 * x) <= 1e-12 * np.linalg.norm(x)
    for seed in range(4):  # direct-covariance formula, completeness
        x, T, V, lam, w = oracle.random_instance(3, 7, 3, 2, 2, seed + 10)
        ref = naive.wiener_direct(x, T, V, lam, w)
        for s in _wiener_paths(dfm, x, T, V, lam, [w], [3]):
            for n in range(2):
                for i in range(3):
                    assert np.linalg.norm(s[n, i] - ref[n, i]) <= 1e-9 * (1 + np.linalg.norm(ref[n, i]))
            assert np.linalg.norm(s.sum(0) - x) <= 1e-9 * np.linalg.norm(x)
    x, T, V, lam, w = oracle.random_instance(3, 8, 4, 2, 2, 41)  # one block == full, bitwise
    full = dfm.wiener_full(x, dfm.NmfModel(T, V), dfm.SpatialModel(w, lam)).images
    blk = dfm.wiener_block(x, dfm.NmfModel(T, V), dfm.BlockSpatialModel(dfm.BlockLayout([4]), [w], lam)).images
    assert np.array_equal(full, blk)
    x, T, V, lam, w = oracle.random_instance(3, 8, 6, 2, 2, 47)  # per-block oracle
    sizes, o, wb = [2, 3, 1], 0, []
    for mb in sizes:
        wb.append(np.ascontiguousarray(w[:, o:o + mb, o:o + mb]))
        o += mb
    for s in _wiener_paths(dfm, x, T, V, lam, wb, sizes):
        o = 0
        for l, mb in enumerate(sizes):
            ref = naive.wiener_direct(x[:, :, o:o + mb], T, V, lam[:, :, o:o + mb], wb[l])
            for n in range(2):
                for i in range(3):
                    got = s[n, i, :, o:o + mb]
                    assert np.linalg.norm(got - ref[n, i]) <= 1e-9 * (1 + np.linalg.norm(ref[n, i]))
            o += mb
        assert np.linalg.norm(s.sum(0) - x) <= 1e-9 * np.linalg.norm(x)


def test_wiener_static_context_kernel_matches_step_kernel(dfm, oracle):
    # the config-1 static-shape context kernel (in-CTA (W^H)^-1, reciprocal
    # gains, per-warp staging) against the generic step kernel
    F, T, N, K, sizes = 21, 300, 5, 16, [4, 4, 4]
    layout = dfm.BlockLayout(sizes)
    x = dfm.generate_mixture(1, F, T, 12, N, K, 91)
    init = dfm.random_init(F, T, layout, N, K, 92)
    a, b = _wiener_paths(dfm, x, init.nmf.T, init.nmf.V, init.lambda0, init.w0, sizes)
    assert np.linalg.norm(a - b) <= 1e-12 * np.linalg.norm(a)
    assert np.linalg.norm(b.sum(0) - x) <= 1e-9 * np.linalg.norm(x)


def test_reconstruct_inverts_clean_images(dfm):
    # test_wiener.cpp:143-160
    from paper_2605_19388_b200 import stft as st

    cfg = st.StftConfig(8000.0, 256, 64)
    clean = np.random.default_rng(51).standard_normal((4096, 2))
    waves = st.reconstruct([st.stft_forward(clean, cfg)], cfg, 4096)
    assert len(waves) == 1
    sl = slice(256, 4096 - 256)
    assert np.linalg.norm(waves[0][sl] - clean[sl]) <= 1e-9 * np.linalg.norm(clean[sl])
    zero = st.reconstruct([np.zeros((129, 60, 2), complex)], cfg, 4096)
    assert not np.any(zero[0])
    X = st.stft_forward(clean, cfg)
    lin = st.reconstruct([2.0 * X, X], cfg, 4096)
    assert np.linalg.norm(lin[0] - 2.0 * lin[1]) <= 1e-12 * np.linalg.norm(lin[0])


def _perturbed(init_d, rel, seed):
    out = dict(init_d)
    rng = np.random.default_rng(seed)
    out["T"] = init_d["T"] * (1 + rel * rng.standard_normal(init_d["T"].shape))
    return out


def test_wiener_drift_is_the_problems_own_sensitivity(dfm, oracle):
    """The config-0 generator (rank-1 point sources, 1e-3 sensor noise) on a
    12-mic block with 45 frames leaves Q_mu with ~1e6 condition numbers: the
    oracle perturbed by 1e-14 relative in its initial T already moves the
    separated STFTs after 30 iterations by ~1e-5.  The device fit must stay
    within a small multiple of that intrinsic amplification (rounding-level
    differences, not an algorithmic drift); with the configs 1-3 generator the
    same shape meets 1e-6 (test_engine_wiener_matches_oracle_after_fit)."""
    F, T, sizes, N, K, iters = 8, 45, [12], 5, 4, 30
    layout = dfm.BlockLayout(sizes)
    x = dfm.generate_mixture(0, F, T, 12, N, K, 1)
    init = dfm.random_init(F, T, layout, N, K, 2)
    init_d = _init_dict(init)
    ref = oracle.run_engine(x, sizes, init_d, iters)
    ref_img = oracle.wiener_block(x, sizes, ref)
    spread = 0.0
    for seed in range(3):
        rp = oracle.run_engine(x, sizes, _perturbed(init_d, 1e-14, seed), iters)
        spread = max(spread, _rel(oracle.wiener_block(x, sizes, rp), ref_img))
    fit = dfm.fit_distributed(x, layout, init, iters, True)
    img = dfm.wiener_block(x, fit.models, fit.spatial).images
    dev = _rel(img, ref_img)
    print(f"device vs oracle {dev:.2e}; oracle vs 1e-14-perturbed oracle up to {spread:.2e}")
    assert spread > 1e-8  # the case is genuinely ill-conditioned
    assert dev <= 30 * spread


def _near_singular_mixture(oracle, F, T, sizes, N, K, seed, lo, hi):
    """BASELINE config-1 generator with channel pairs made nearly collinear,
    x_{p+1} = x_p + delta_f n, delta_f log-spaced over the bins: S = W^H Q_mu
    sweeps through the reference's 1e-6 LU residual threshold (engine.cpp:47-49)."""
    x = oracle.generate_mixture(1, F, T, sum(sizes), N, K, seed)
    rng = np.random.default_rng(seed)
    d = np.logspace(lo, hi, F)
    off = 0
    for mb in sizes:
        for p in range(0, mb - 1, 2):
            nz = (rng.standard_normal((F, T)) + 1j * rng.standard_normal((F, T))) * np.abs(x[:, :, off + p]).mean()
            x[:, :, off + p + 1] = x[:, :, off + p] + d[:, None] * nz
        off += mb
    return x


def _lu_residuals(oracle, x, init_d, sizes):
    """Per bin, the largest ||S u_LU - e_mu|| of the first IP sweep (numpy LU)."""
    h = oracle.spectrogram(init_d["T"], init_d["V"])
    eta = oracle.eta_from(h, init_d["lam"])
    F, T, _ = x.shape
    out = np.zeros(F)
    off = 0
    for b, mb in enumerate(sizes):
        for f in range(F):
            W = init_d["w"][b][f].copy()
            xb = x[f, :, off:off + mb]
            for mu in range(mb):
                w = 1 / np.maximum(eta[f, :, off + mu], 1e-6)
                Q = (xb.T * w) @ xb.conj() / T
                S = W.conj().T @ Q
                e = np.zeros(mb)
                e[mu] = 1
                u = np.linalg.solve(S, e)
                r = np.linalg.norm(S @ u - e)
                out[f] = max(out[f], r)
                if not np.all(np.isfinite(u)) or r > 1e-6:
                    u = np.linalg.pinv(S) @ e
                W[:, mu] = u / np.sqrt(max((u.conj() @ Q @ u).real, 1e-6))
        off += mb
    return out


@pytest.mark.parametrize("sizes,N,K", [([4, 4, 4], 5, 16), ([2, 2], 3, 4), ([12], 5, 16), ([8], 2, 2)])
def test_ip_branch_near_the_residual_threshold(dfm, oracle, sizes, N, K):
    """The fast IP paths (quad: static 4- and 2-mic blocks; warp: the 12-mic
    static and the generic 8-mic kernels) solve (W^H Q)^-1 e in another form
    than the reference's LU.  They are accepted only when every column's
    residual is under the 1e-8 guard band (kFastResid); otherwise the exact
    sweep applies the reference's LU predicate.  Near the threshold the
    reference's own decision is rounding-dependent: the oracle perturbed by
    1e-14 flips a few columns.  So: on every bin whose first sweep is stable
    under such perturbations (including bins that take the pinv branch), the
    device W equals the oracle's; over all bins the device's pinv count lies
    within the oracle's perturbation spread."""
    F, T = 64, 64
    x = _near_singular_mixture(oracle, F, T, sizes, N, K, 3, -8, -2)
    layout = dfm.BlockLayout(sizes)
    init = dfm.random_init(F, T, layout, N, K, 4)
    init_d = _init_dict(init)
    ref = oracle.run_engine(x, sizes, init_d, 1)
    stable = np.ones(F, bool)
    fbs = [ref["fallbacks"]]
    for seed, p in enumerate([1e-14, 1e-13, 1e-12]):
        rp = oracle.run_engine(x, sizes, _perturbed(init_d, p, seed), 1)
        fbs.append(rp["fallbacks"])
        for a, b in zip(ref["w"], rp["w"]):
            stable &= np.array([_rel(b[f], a[f]) < 1e-9 for f in range(F)])
    res = _lu_residuals(oracle, x, init_d, sizes)
    assert (stable & (res > 1e-6)).sum() >= 2, "the case must hold decision-stable pinv bins"
    fit = dfm.fit_distributed(x, layout, init, 1, True)
    spread = max(fbs) - min(fbs)
    assert min(fbs) - max(2, spread) <= fit.report.fallbacks <= max(fbs) + max(2, spread)
    for a, b in zip(fit.spatial.W, ref["w"]):
        for f in np.nonzero(stable)[0]:
            assert _rel(a[f], b[f]) < 1e-7, f"bin {f} (LU residual {res[f]:.1e})"



def test_two_cta_cluster_bins_match_oracle(dfm, oracle):
    """A shard with at most half as many bins as SMs runs every bin as a 2-CTA
    cluster (k_em_bin<..., CS=2>: half the frames each, partial sums through
    distributed shared memory).  The fit meets the north_star bar against the
    oracle: trajectory 1e-8 over 20 iterations, non-increasing cost, separated
    STFTs 1e-6; and the full-size context keeps one CTA per bin."""
    F, T, sizes, N, K, iters = 40, 160, [4, 4, 4], 5, 16, 20
    layout = dfm.BlockLayout(sizes)
    x = dfm.generate_mixture(1, F, T, layout.total, N, K, 31)
    init = dfm.random_init(F, T, layout, N, K, 32)
    e = dfm.Engine(F, T, layout, N, K)
    assert e.tiling()["ctas"] == 2 * F
    e.close()
    big = dfm.Engine(513, 626, layout, N, K)
    assert big.tiling()["ctas"] == 513
    big.close()
    fit = dfm.fit_distributed(x, layout, init, iters, True)
    ref = oracle.run_engine(x, sizes, _init_dict(init), iters)
    cost = fit.report.cost_trace
    assert np.max(np.abs(cost - ref["cost_trace"]) / np.abs(ref["cost_trace"])) < TRAJ_RTOL
    assert np.all(cost[1:] <= cost[:-1] + 1e-9 * np.abs(cost[:-1]))
    assert fit.report.fallbacks == ref["fallbacks"]
    img = dfm.wiener_block(x, fit.models, fit.spatial).images
    ref_img = oracle.wiener_block(x, sizes, ref)
    assert _rel(img, ref_img) < 1e-6


@pytest.mark.parametrize("K", [24, 16])
def test_v_update_frame_pair_kernel_matches_oracle(dfm, oracle, K):
    """k_vupd_mma<KT, 2> (16 frames per CTA, a lane loads frame pairs and KT
    consecutive bases) is selected for even T and K once its grid has two
    rounds of CTAs per SM: T = 1210 frames (even, not a multiple of 16: the
    last CTA is ragged) x 8 sources = 608 CTAs.  K = 24 leaves the fourth base
    tile half empty.  Trajectory against the oracle at the north_star bar and
    the fitted V within 1e-7."""
    F, T, sizes, N, iters = 12, 1210, [2, 2], 8, 6
    layout = dfm.BlockLayout(sizes)
    x = dfm.generate_mixture(1, F, T, layout.total, N, K, 41)
    init = dfm.random_init(F, T, layout, N, K, 42)
    fit = dfm.fit_distributed(x, layout, init, iters, True)
    ref = oracle.run_engine(x, sizes, _init_dict(init), iters)
    cost = fit.report.cost_trace
    assert np.max(np.abs(cost - ref["cost_trace"]) / np.abs(ref["cost_trace"])) < TRAJ_RTOL
    assert np.all(cost[1:] <= cost[:-1] + 1e-9 * np.abs(cost[:-1]))
    assert _rel(fit.models[0].V, ref["V"]) < 1e-7
    assert _rel(fit.models[0].T, ref["T"]) < 1e-7
