"""Pins the CPU oracle (oracle/dfm_oracle.c) against the reference's own
known-answer tests and invariants.  The reference cannot be
built here (no Eigen), so these ported checks ARE the parity pin.

Each test names the reference test it ports (paths under /root/reference/proj).
"""
import numpy as np
import pytest

import naive

FLOOR = 1e-6


# --------------------------------------------------------------------- rng
def test_splitmix64_published_vectors(oracle):
    # Vigna's splitmix64 reference output for state 0 (rng.hpp:13-18 restates it)
    s, out = 0, []
    for _ in range(4):
        v, s = oracle.splitmix64(s)
        out.append(v)
    assert out == [0xE220A8397B1DCDAF, 0x6E789E6AA1B965F4, 0x06C45D188009454F, 0xF88BB8A8724C81EC]


def test_rng_uniform_and_gaussian_properties(oracle):
    u = oracle.rng_draws(7, 200000, False)
    assert np.all((u >= 0) & (u < 1))
    assert abs(u.mean() - 0.5) < 5e-3
    g = oracle.rng_draws(7, 200000, True)
    assert abs(g.mean()) < 1e-2 and abs(g.std() - 1) < 1e-2
    # deterministic per seed, distinct across seeds (bench.cpp random_observations contract)
    assert np.array_equal(oracle.rng_draws(3, 10, True), oracle.rng_draws(3, 10, True))
    assert not np.array_equal(oracle.rng_draws(3, 10), oracle.rng_draws(4, 10))
    assert oracle.derive_seed(1, "a", 0) != oracle.derive_seed(1, "b", 0)
    assert oracle.derive_seed(1, "a", 0) != oracle.derive_seed(1, "a", 1)
    assert oracle.derive_seed(1, "a", 5) == oracle.derive_seed(1, "a", 5)


def test_random_observations_deterministic(oracle):
    a = oracle.random_observations(3, 5, 2, 9)
    b = oracle.random_observations(3, 5, 2, 9)
    c = oracle.random_observations(3, 5, 2, 10)
    assert np.array_equal(a, b) and not np.array_equal(a, c)


def test_random_init_ranges(oracle):
    m = oracle.random_init(5, 7, [2, 3], 2, 3, 11)
    assert m["T"].shape == (2, 5, 3) and m["V"].shape == (2, 3, 7) and m["lam"].shape == (5, 2, 5)
    assert m["T"].min() >= FLOOR and m["T"].max() < 1 + FLOOR
    assert m["lam"].min() >= 0.5 and m["lam"].max() < 1.5
    assert [w.shape for w in m["w"]] == [(5, 2, 2), (5, 3, 3)]
    # W = I + 0.3 (g + i g): diagonal centred at 1
    d = np.concatenate([np.diagonal(w, axis1=1, axis2=2).ravel() for w in m["w"]])
    assert abs(d.real.mean() - 1) < 0.3


# ------------------------------------------------------------- step stages
def test_decorrelate_identity_scaling_naive(oracle):
    # test_fastmnmf.cpp:69-85
    x, *_ = oracle.random_instance(3, 5, 3, 1, 1, 1)
    eye = np.tile(np.eye(3, dtype=complex), (3, 1, 1))
    y, _ = oracle.decorrelate_block(x, 0, eye)
    assert np.array_equal(y, x)
    y, _ = oracle.decorrelate_block(x, 0, 2 * eye)
    assert np.abs(y - 2 * x).max() < 1e-14
    rng = np.random.default_rng(0)
    w = rng.standard_normal((3, 3, 3)) + 1j * rng.standard_normal((3, 3, 3))
    y, P = oracle.decorrelate_block(x, 0, w)
    ref = naive.decorrelate(x, w)
    assert np.linalg.norm(y - ref) <= 1e-12 * np.linalg.norm(ref)
    assert np.allclose(P, np.abs(ref) ** 2, rtol=1e-12)


def test_eta_scalar_cases_and_floor(oracle):
    # test_fastmnmf.cpp:87-101
    one = np.ones((1, 1, 1))
    h = oracle.spectrogram(one, one)
    assert oracle.eta_from(h, one)[0, 0, 0] == 1.0
    T = np.full((1, 1, 1), 2.0); V = np.full((1, 1, 1), 3.0); lam = np.full((1, 1, 1), 0.5)
    assert oracle.eta_from(oracle.spectrogram(T, V), lam)[0, 0, 0] == pytest.approx(3.0)
    T[:] = 0.0
    assert oracle.eta_from(oracle.spectrogram(T, V), lam)[0, 0, 0] == FLOOR


def test_eta_matches_naive(oracle):
    # test_fastmnmf.cpp:103-112
    _, T, V, lam, _ = oracle.random_instance(3, 6, 3, 2, 2, 99)
    eta = oracle.eta_from(oracle.spectrogram(T, V), lam)
    ref = np.maximum(naive.eta_raw(T, V, lam), FLOOR)
    assert np.allclose(eta, ref, rtol=1e-12, atol=0)


def _cost_full(oracle, x, T, V, lam, w_full):
    return oracle.cost_dist(x, [x.shape[2]], dict(T=T, V=V, lam=lam, w=[w_full]))


def test_cost_scalar_zero_power_and_naive(oracle):
    # test_fastmnmf.cpp:114-136
    x = np.ones((1, 1, 1), dtype=complex)
    one = np.ones((1, 1, 1))
    assert _cost_full(oracle, x, one, one, one, np.ones((1, 1, 1), complex)) == pytest.approx(1.0)
    x, T, V, lam, w = oracle.random_instance(2, 4, 2, 1, 1, 5)
    x[:] = 0; T[:] = 1; V[:] = 1; lam[:] = 1
    det_term = -sum(4 * np.log(abs(np.linalg.det(w[i])) ** 2) for i in range(2))
    assert _cost_full(oracle, x, T, V, lam, w) == pytest.approx(det_term, rel=1e-10)
    for seed in range(8):
        x, T, V, lam, w = oracle.random_instance(3, 7, 3, 2, 2, seed)
        assert _cost_full(oracle, x, T, V, lam, w) == pytest.approx(naive.cost(x, T, V, lam, w), rel=1e-10)


def test_cost_singular_raises(oracle):
    # test_fastmnmf.cpp:143-149
    x, T, V, lam, w = oracle.random_instance(2, 4, 2, 1, 1, 3)
    w[1][:, 0] = 0; w[1][:, 1] = 0
    with pytest.raises(oracle.SingularDemixer):
        _cost_full(oracle, x, T, V, lam, w)


def test_ip_scalar_closed_form_and_white_fixed_point(oracle):
    # test_fastmnmf.cpp:151-173
    rng = np.random.default_rng(6)
    x = rng.standard_normal((2, 8, 1)) + 1j * rng.standard_normal((2, 8, 1))
    eta = np.ones((2, 8, 1))
    w, nfb = oracle.ip_sweep_column(x, eta, 0, np.ones((2, 1, 1), complex), 0)
    for i in range(2):
        q = np.sum(np.abs(x[i]) ** 2) / 8.0
        assert abs(w[i, 0, 0]) ** 2 == pytest.approx(1.0 / q, rel=1e-10)
    M = 3
    white = np.zeros((1, M, M), dtype=complex)
    white[0] = np.sqrt(M) * np.eye(M)
    weye = np.eye(M, dtype=complex)[None]
    for m in range(M):
        weye, _ = oracle.ip_sweep_column(white, np.ones((1, M, M)), 0, weye, m)
    assert np.linalg.norm(weye[0] - np.eye(M)) < 1e-12


def test_ip_normalisation(oracle):
    # test_fastmnmf.cpp:175-190
    x, T, V, lam, w = oracle.random_instance(3, 16, 3, 2, 2, 11)
    eta = oracle.eta_from(oracle.spectrogram(T, V), lam)
    for m in range(3):
        w, _ = oracle.ip_sweep_column(x, eta, 0, w, m)
    for i in range(3):
        for m in range(3):
            q = np.einsum("j,ja,jb->ab", 1 / np.maximum(eta[i, :, m], FLOOR), x[i], x[i].conj()) / 16
            quad = w[i, :, m].conj() @ q @ w[i, :, m]
            assert abs(quad.real - 1) <= 1e-9


def _mm_t(oracle, T, V, lam, P, eta):
    a, b = oracle.build_tv_weights(lam, P, eta)
    T = oracle.update_t(T, V, a, b)
    return T, oracle.eta_from(oracle.spectrogram(T, V), lam)


def _mm_v(oracle, T, V, lam, P, eta):
    a, b = oracle.build_tv_weights(lam, P, eta)
    V = oracle.update_v(T, V, a, b)
    return V, oracle.eta_from(oracle.spectrogram(T, V), lam)


def _mm_lambda(oracle, T, V, lam, P, eta):
    h = oracle.spectrogram(T, V)
    lam = oracle.update_lambda(lam, h, P, eta)
    return lam, oracle.eta_from(h, lam)


def _scalar(v):
    x = np.full((1, 1, 1), v, dtype=complex)
    one = np.ones((1, 1, 1))
    return x, one.copy(), one.copy(), one.copy()


def test_mm_scalar_reductions(oracle):
    # test_fastmnmf.cpp:192-218
    x, T, V, lam = _scalar(2.0)
    P = np.abs(x) ** 2
    eta = oracle.eta_from(oracle.spectrogram(T, V), lam)
    T, eta = _mm_t(oracle, T, V, lam, P, eta)
    assert T[0, 0, 0] == pytest.approx(2.0, rel=1e-12) and eta[0, 0, 0] == pytest.approx(2.0, rel=1e-12)
    x, T, V, lam = _scalar(3.0)
    eta = oracle.eta_from(oracle.spectrogram(T, V), lam)
    V, _ = _mm_v(oracle, T, V, lam, np.abs(x) ** 2, eta)
    assert V[0, 0, 0] == pytest.approx(3.0, rel=1e-12)
    x, T, V, lam = _scalar(4.0)
    eta = oracle.eta_from(oracle.spectrogram(T, V), lam)
    lam, _ = _mm_lambda(oracle, T, V, lam, np.abs(x) ** 2, eta)
    assert lam[0, 0, 0] == pytest.approx(4.0, rel=1e-12)


def test_mm_updates_match_naive(oracle):
    # test_fastmnmf.cpp:220-280
    x, T, V, lam, w = oracle.random_instance(3, 5, 3, 2, 2, 23)
    P = np.abs(naive.decorrelate(x, w)) ** 2
    eta = oracle.eta_from(oracle.spectrogram(T, V), lam)
    T1, _ = _mm_t(oracle, T, V, lam, P, eta)
    ref = naive.update_t(T, V, lam, P)
    assert np.linalg.norm(T1 - ref) <= 1e-11 * np.linalg.norm(ref)
    l1, _ = _mm_lambda(oracle, T, V, lam, P, eta)
    ref = naive.update_lambda(T, V, lam, P)
    assert np.linalg.norm(l1 - ref) <= 1e-11 * np.linalg.norm(ref)


def test_mm_exact_fit_fixed_point(oracle):
    # test_fastmnmf.cpp:282-303
    x, T, V, lam, w = oracle.random_instance(2, 5, 3, 2, 2, 31)
    eta = oracle.eta_from(oracle.spectrogram(T, V), lam)
    P = eta.copy()  # W = I, x = sqrt(eta)
    T1, eta = _mm_t(oracle, T, V, lam, P, eta)
    V1, eta = _mm_v(oracle, T1, V, lam, P, eta)
    l1, eta = _mm_lambda(oracle, T1, V1, lam, P, eta)
    assert np.abs(T1 - T).max() <= 1e-12 and np.abs(V1 - V).max() <= 1e-12
    assert np.abs(l1 - lam).max() <= 1e-12


def test_every_update_non_increasing(oracle):
    # test_fastmnmf.cpp:315-349
    rng = np.random.default_rng(100)
    for seed in range(12):
        F, Tn, M, N, K = (2 + rng.integers(3), 8 + rng.integers(8), 2 + rng.integers(3),
                          1 + rng.integers(3), 1 + rng.integers(3))
        x, T, V, lam, w = oracle.random_instance(int(F), int(Tn), int(M), int(N), int(K), seed)
        eta = oracle.eta_from(oracle.spectrogram(T, V), lam)
        cost = _cost_full(oracle, x, T, V, lam, w)

        def check(c_prev):
            c = _cost_full(oracle, x, T, V, lam, w)
            assert c <= c_prev + 1e-9 * abs(c_prev)
            return c

        for _ in range(3):
            for m in range(M):
                w, _ = oracle.ip_sweep_column(x, eta, 0, w, m)
                cost = check(cost)
            P = oracle.decorrelate_block(x, 0, w)[1]
            T, eta = _mm_t(oracle, T, V, lam, P, eta)
            cost = check(cost)
            V, eta = _mm_v(oracle, T, V, lam, P, eta)
            cost = check(cost)
            lam, eta = _mm_lambda(oracle, T, V, lam, P, eta)
            cost = check(cost)


def test_fit_zero_iters_determinism_monotone(oracle):
    # test_fastmnmf.cpp:351-375
    x, T, V, lam, w = oracle.random_instance(4, 12, 3, 2, 2, 55)
    init = dict(T=T, V=V, lam=lam, w=[w])
    r0 = oracle.run_engine(x, [3], init, 0)
    assert r0["cost_trace"].shape == (1,)
    assert r0["cost_trace"][0] == pytest.approx(_cost_full(oracle, x, T, V, lam, w), rel=1e-14)
    a = oracle.run_engine(x, [3], init, 30)
    b = oracle.run_engine(x, [3], init, 30)
    assert np.array_equal(a["cost_trace"], b["cost_trace"])
    c = a["cost_trace"]
    assert np.all(c[1:] <= c[:-1] + 1e-9 * np.abs(c[:-1]))
    assert a["wall_seconds"].shape == (30,)
    final = _cost_full(oracle, x, a["T"], a["V"], a["lam"], a["w"][0])
    assert final == pytest.approx(c[-1], rel=1e-12)


def test_fit_adversarial_stays_finite(oracle):
    # test_fastmnmf.cpp:377-404
    x, T, V, lam, w = oracle.random_instance(3, 10, 4, 2, 2, 77)
    x[:, :, 1] = 0
    x[:, :, 3] = x[:, :, 2]
    r = oracle.run_engine(x, [4], dict(T=T, V=V, lam=lam, w=[w]), 60)
    for k in ("T", "V", "lam"):
        assert np.all(np.isfinite(r[k])) and r[k].min() >= FLOOR
    assert np.all(np.isfinite(r["w"][0]))
    assert not np.any(np.isnan(r["cost_trace"]))
    assert r["fallbacks"] > 0  # the pinv path is exercised


def test_op_counts(oracle):
    # test_bench.cpp:34-52: w_update ops = bins*iters*(M^4 + J M^3) per block layout
    x = oracle.random_observations(4, 16, 6, 3)
    init = oracle.random_init(4, 16, [6], 2, 2, 3)
    r = oracle.run_engine(x, [6], init, 2)
    assert r["ops"]["w_update"] == pytest.approx(4.0 * 2 * (6 ** 4 + 16.0 * 6 ** 3))
    init = oracle.random_init(4, 16, [2, 2, 2], 2, 2, 3)
    r = oracle.run_engine(x, [2, 2, 2], init, 2)
    assert r["ops"]["w_update"] == pytest.approx(4.0 * 2 * 3 * (2 ** 4 + 16.0 * 2 ** 3))


# ------------------------------------------------------------ distributed
def _init_from(inst, sizes):
    x, T, V, lam, w = inst
    blocks, o = [], 0
    for mb in sizes:
        blocks.append(w[:, o:o + mb, o:o + mb].copy())
        o += mb
    return dict(T=T, V=V, lam=lam, w=blocks)


def test_cost_dist_one_block_equals_full(oracle):
    # test_dist.cpp:56-63
    inst = oracle.random_instance(3, 8, 4, 2, 2, 1)
    m = _init_from(inst, [4])
    assert oracle.cost_dist(inst[0], [4], m) == _cost_full(oracle, *inst)


def test_cost_dist_equals_assembled_full(oracle):
    # test_dist.cpp:65-79
    for seed in range(6):
        inst = oracle.random_instance(3, 9, 6, 2, 2, seed + 10)
        m = _init_from(inst, [2, 3, 1])
        a = oracle.cost_dist(inst[0], [2, 3, 1], m)
        b = _cost_full(oracle, inst[0], m["T"], m["V"], m["lam"], naive.block_diag_w(m["w"]))
        assert a == pytest.approx(b, rel=1e-10)


def test_cost_dist_zero_observations(oracle):
    # test_dist.cpp:81-95
    x, T, V, lam, w = oracle.random_instance(2, 5, 4, 1, 1, 3)
    x[:] = 0; T[:] = 1; V[:] = 1; lam[:] = 1
    m = _init_from((x, T, V, lam, w), [2, 2])
    expect = -sum(5 * np.log(abs(np.linalg.det(b[i])) ** 2) for b in m["w"] for i in range(2))
    assert oracle.cost_dist(x, [2, 2], m) == pytest.approx(expect, rel=1e-10)


def test_size_one_block_closed_form(oracle):
    # test_dist.cpp:110-122
    rng = np.random.default_rng(5)
    x = rng.standard_normal((2, 12, 3)) + 1j * rng.standard_normal((2, 12, 3))
    eta = np.ones((2, 12, 3))
    w, _ = oracle.ip_sweep_column(x, eta, 2, np.ones((2, 1, 1), complex), 0)
    for i in range(2):
        q = np.sum(np.abs(x[i, :, 2]) ** 2) / 12
        assert abs(w[i, 0, 0]) ** 2 == pytest.approx(1 / q, rel=1e-10)


def test_block_ip_sweep_non_increasing(oracle):
    # test_dist.cpp:124-140
    for seed in range(8):
        inst = oracle.random_instance(3, 12, 5, 2, 2, seed + 40)
        m = _init_from(inst, [3, 2])
        eta = oracle.eta_from(oracle.spectrogram(m["T"], m["V"]), m["lam"])
        cost = oracle.cost_dist(inst[0], [3, 2], m)
        offs = [0, 3]
        for l, mb in enumerate([3, 2]):
            for mu in range(mb):
                m["w"][l], _ = oracle.ip_sweep_column(inst[0], eta, offs[l], m["w"][l], mu)
                nxt = oracle.cost_dist(inst[0], [3, 2], m)
                assert nxt <= cost + 1e-9 * abs(cost)
                cost = nxt


def test_shared_two_subarray_scalar_mm(oracle):
    # test_dist.cpp:142-164
    x = np.array([[[2.0, 3.0]]], dtype=complex)
    T = np.ones((1, 1, 1)); V = np.ones((1, 1, 1))
    lam = np.array([[[1.0, 2.0]]])
    eta = oracle.eta_from(oracle.spectrogram(T, V), lam)
    assert eta[0, 0, 0] == 1.0 and eta[0, 0, 1] == 2.0
    T, _ = _mm_t(oracle, T, V, lam, np.abs(x) ** 2, eta)
    assert T[0, 0, 0] == pytest.approx(np.sqrt((4.0 + 4.5) / 2.0), rel=1e-12)


def test_locally_underdetermined_and_monotone(oracle):
    # test_dist.cpp:215-229, 251-261
    inst = oracle.random_instance(3, 10, 4, 3, 2, 81)
    r = oracle.run_engine(inst[0], [2, 2], _init_from(inst, [2, 2]), 40)
    assert np.all(np.isfinite(r["T"])) and r["T"].min() >= FLOOR
    c = r["cost_trace"]
    assert np.all(c[1:] <= c[:-1] + 1e-9 * np.abs(c[:-1]))


def test_v_update_sharded_sum_equals_full(oracle):
    # frequency-sharded partials + one allreduce == the unsharded update
    x, T, V, lam, w = oracle.random_instance(7, 9, 3, 2, 3, 5)
    P = np.abs(naive.decorrelate(x, w)) ** 2
    eta = oracle.eta_from(oracle.spectrogram(T, V), lam)
    a, b = oracle.build_tv_weights(lam, P, eta)
    full = oracle.update_v(T, V, a, b)
    nd = oracle.update_v_partial(T, a, b, 0, 3) + oracle.update_v_partial(T, a, b, 3, 7)
    shard = oracle.update_v_apply(V, nd)
    assert np.allclose(shard, full, rtol=1e-13, atol=0)


# ------------------------------------------------------------------ wiener
def _wiener_full(oracle, x, T, V, lam, w):
    return oracle.wiener_block(x, [x.shape[2]], dict(T=T, V=V, lam=lam, w=[w]))


def test_wiener_single_source_passthrough(oracle):
    # test_wiener.cpp:39-45
    x, T, V, lam, w = oracle.random_instance(3, 6, 3, 1, 2, 1)
    s = _wiener_full(oracle, x, T, V, lam, w)
    assert np.linalg.norm(s[0] - x) <= 1e-12 * np.linalg.norm(x)


def test_wiener_equal_split(oracle):
    # test_wiener.cpp:47-58
    x, T, V, lam, w = oracle.random_instance(2, 5, 3, 2, 2, 3)
    T[1] = T[0]; V[1] = V[0]; lam[:, 1] = lam[:, 0]
    s = _wiener_full(oracle, x, T, V, lam, w)
    for n in range(2):
        assert np.linalg.norm(s[n] - 0.5 * x) <= 1e-12 * np.linalg.norm(x)


def test_wiener_direct_formula_and_completeness(oracle):
    # test_wiener.cpp:60-82
    for seed in range(6):
        x, T, V, lam, w = oracle.random_instance(3, 7, 3, 2, 2, seed + 10)
        s = _wiener_full(oracle, x, T, V, lam, w)
        ref = naive.wiener_direct(x, T, V, lam, w)
        for n in range(2):
            for i in range(3):
                assert np.linalg.norm(s[n, i] - ref[n, i]) <= 1e-9 * (1 + np.linalg.norm(ref[n, i]))
    x, T, V, lam, w = oracle.random_instance(4, 9, 3, 3, 2, 21)
    s = _wiener_full(oracle, x, T, V, lam, w)
    assert np.linalg.norm(s.sum(0) - x) <= 1e-9 * np.linalg.norm(x)


def test_wiener_block_one_block_equals_full_and_per_block_oracle(oracle):
    # test_wiener.cpp:98-141
    inst = oracle.random_instance(3, 8, 6, 2, 2, 47)
    x, T, V, lam, w = inst
    m = _init_from(inst, [2, 3, 1])
    s = oracle.wiener_block(x, [2, 3, 1], m)
    o = 0
    for l, mb in enumerate([2, 3, 1]):
        ref = naive.wiener_direct(x[:, :, o:o + mb], T, V, lam[:, :, o:o + mb], m["w"][l])
        for n in range(2):
            for i in range(3):
                got = s[n, i, :, o:o + mb]
                assert np.linalg.norm(got - ref[n, i]) <= 1e-9 * (1 + np.linalg.norm(ref[n, i]))
        o += mb
    assert np.linalg.norm(s.sum(0) - x) <= 1e-9 * np.linalg.norm(x)


# ------------------------------------------------------------------ linalg
def test_lu_and_pinv_solves(oracle):
    rng = np.random.default_rng(4)
    for n in (1, 2, 4, 7, 12):
        S = rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n))
        e = np.zeros(n, complex); e[0] = 1
        assert np.allclose(oracle.lu_solve(S, e), np.linalg.solve(S, e), rtol=1e-10, atol=1e-12)
        assert np.allclose(oracle.pinv_solve(S, e), np.linalg.solve(S, e), rtol=1e-9, atol=1e-11)
        # rank deficient: pinv minimum-norm solution (hermlin.cpp:19-23; test_hermlin.cpp:73-87)
        if n > 1:
            G = rng.standard_normal((n, n - 1)) + 1j * rng.standard_normal((n, n - 1))
            S = G @ G.conj().T
            b = rng.standard_normal(n) + 1j * rng.standard_normal(n)
            assert np.allclose(oracle.pinv_solve(S, b), np.linalg.pinv(S) @ b, rtol=1e-8, atol=1e-9)
    z = np.zeros((3, 3), complex)
    assert np.array_equal(oracle.pinv_solve(z, np.ones(3, complex)), np.zeros(3, complex))
