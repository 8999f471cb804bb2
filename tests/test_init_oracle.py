"""Pins the C restatement of the initialisation pipeline (oracle/
dfm_init_oracle.c via oracle/init_oracle.py) against the reference's own
tests, test_init.cpp:44-418 and the GEVD cases of test_hermlin.cpp:98-138.
The reference's scenes are rebuilt with the same construction (two sources
active in disjoint 8-frame blocks, steering phases 0.3 + 0.11 i and + pi);
their random draws come from a seeded numpy generator."""
import itertools

import numpy as np
import pytest

import init_oracle as io


def two_source_scene(F, T, seed):
    # test_init.cpp:20-40
    rng = np.random.default_rng(seed)
    active = np.array([(j // 8) % 2 for j in range(T)])
    x = np.zeros((F, T, 2), dtype=np.complex128)
    for i in range(F):
        th = 0.3 + 0.11 * i
        a0 = np.array([1.0, np.exp(1j * th)])
        a1 = np.array([1.0, np.exp(1j * (th + np.pi))])
        for j in range(T):
            s = rng.standard_normal() + 1j * rng.standard_normal()
            x[i, j] = (a0 if active[j] == 0 else a1) * s
    return x, active


def random_tensor(F, T, M, rng):
    return rng.standard_normal((F, T, M)) + 1j * rng.standard_normal((F, T, M))


def random_hpd(m, rng):
    a = rng.standard_normal((m, m)) + 1j * rng.standard_normal((m, m))
    return a @ a.conj().T + m * np.eye(m)


def test_one_source_mask_is_all_ones():
    m = io.cluster_masks(random_tensor(3, 10, 2, np.random.default_rng(1)), 1, 7)
    assert np.array_equal(m, np.ones((3, 10, 1)))


def test_rows_sum_to_one_and_silent_bin_is_uniform():
    x = random_tensor(4, 12, 3, np.random.default_rng(2))
    x[2] = 0
    m = io.cluster_masks(x, 3, 11)
    assert np.allclose(m.sum(axis=2), 1.0, atol=1e-9)
    assert np.array_equal(m[2], np.full((12, 3), 1.0 / 3))


def test_fewer_frames_than_sources_is_rejected():
    with pytest.raises(ValueError, match="fewer frames than sources"):
        io.cluster_masks(random_tensor(2, 2, 2, np.random.default_rng(3)), 3, 1)


def test_separates_disjointly_active_sources():
    x, act = two_source_scene(12, 64, 3)
    m = io.cluster_masks(x, 2, 5)
    pur = []
    for i in range(12):
        lab = (m[i, :, 0] < m[i, :, 1]).astype(int)
        frac = np.mean(lab == act)
        pur.append(max(frac, 1 - frac))
    assert np.mean(pur) >= 0.9


def test_alignment_fixed_point_and_planted_swaps():
    _, act = two_source_scene(10, 48, 9)
    mask = np.zeros((10, 48, 2))
    for j in range(48):
        mask[:, j, act[j]] = 0.95
        mask[:, j, 1 - act[j]] = 0.05
    assert np.array_equal(io.align_frequency_permutations(mask), mask)
    # test_init.cpp:98-122: planted per-bin swaps are undone
    _, act = two_source_scene(40, 64, 13)
    mask = np.zeros((40, 64, 2))
    for j in range(64):
        mask[:, j, act[j]] = 0.9
        mask[:, j, 1 - act[j]] = 0.1
    rng = np.random.default_rng(17)
    scr = mask.copy()
    for i in range(40):
        if rng.random() < 0.5:
            scr[i] = scr[i][:, ::-1]
    al = io.align_frequency_permutations(scr)
    direct = sum(np.linalg.norm(al[i] - mask[i]) < 1e-12 for i in range(40))
    assert max(direct, 40 - direct) / 40 >= 0.95


def test_two_bin_swap_is_detected():
    act = np.array([1, 1, 0, 0, 1, 0], dtype=float)
    m = np.zeros((2, 6, 2))
    m[0, :, 0], m[0, :, 1] = act, 1 - act
    m[1, :, 0], m[1, :, 1] = 1 - act, act
    al = io.align_frequency_permutations(m)
    assert np.array_equal(al[0], al[1])


def test_subarray_permutations():
    # test_init.cpp:138-197
    rng = np.random.default_rng(23)
    F, T, N = 6, 32, 3
    base = rng.random((F, T, N))
    base /= base.sum(axis=2, keepdims=True)
    assert list(io.align_subarray_permutations([base, base])[1]) == [0, 1, 2]
    shifted = np.zeros_like(base)
    for n in range(N):
        shifted[:, :, (n + 1) % N] = base[:, :, n]
    p = io.align_subarray_permutations([base, shifted])[1]
    assert np.allclose(shifted[:, :, p], base, atol=1e-12)
    noisy = np.maximum(0.0, shifted + 0.05 * rng.standard_normal(shifted.shape))
    p = io.align_subarray_permutations([base, noisy])[1]
    flat = lambda m, n: m[:, :, n].reshape(-1)

    def pear(u, v):
        du, dv = u - u.mean(), v - v.mean()
        return du @ dv / (np.linalg.norm(du) * np.linalg.norm(dv))

    best, top = None, -1e300
    for perm in itertools.permutations(range(N)):
        s = sum(pear(flat(noisy, perm[n]), flat(base, n)) for n in range(N))
        if s > top:
            top, best = s, list(perm)
    assert list(p) == best


def test_best_permutation_rejects_more_than_eight_sources():
    with pytest.raises(ValueError, match="too many sources"):
        io.best_permutation(np.ones((4, 9)), np.ones((4, 9)))


def test_init_spectrogram_closed_forms():
    # test_init.cpp:226-254
    rng = np.random.default_rng(37)
    c = rng.standard_normal((2, 16, 1)) + 1j * rng.standard_normal((2, 16, 1))
    ones = [np.ones((2, 16, 1))]
    R = io.init_scm(c, [1], ones)
    h0 = io.init_spectrogram(c, [1], ones, R)
    for i in range(2):
        mp = np.sum(np.abs(c[i]) ** 2) / 16
        assert np.allclose(h0[i, :, 0], np.abs(c[i, :, 0]) ** 2 / mp, rtol=1e-4)
    cc = np.full((1, 12, 1), 0.7 - 0.2j)
    o = [np.ones((1, 12, 1))]
    assert np.allclose(io.init_spectrogram(cc, [1], o, io.init_scm(cc, [1], o)), 1.0, rtol=1e-4)
    cz = np.zeros((1, 8, 2), dtype=complex)
    o = [np.ones((1, 8, 1))]
    assert not np.any(io.init_spectrogram(cz, [2], o, io.init_scm(cz, [2], o)))


def test_masked_scm_matches_numpy():
    rng = np.random.default_rng(5)
    x = random_tensor(3, 20, 5, rng)
    masks = [rng.random((3, 20, 2)), rng.random((3, 20, 2))]
    R = io.init_scm(x, [2, 3], masks)
    for n in range(2):
        for f in range(3):
            c = x[f].copy()
            c[:, :2] *= masks[0][f, :, n][:, None]
            c[:, 2:] *= masks[1][f, :, n][:, None]
            assert np.allclose(R[n, f], c.T @ c.conj() / 20, atol=1e-13)


def test_is_nmf_rank_one_scalar_and_monotone():
    # test_init.cpp:256-305
    rng = np.random.default_rng(41)
    t, v = 0.5 + rng.random(6), 0.5 + rng.random(10)
    h0 = (t[:, None] * v[None, :])[:, :, None]
    Tm, V, tr, its = io.is_nmf(h0, 1, 1000, 3)
    assert tr[0][-1] <= 1e-6
    assert np.all(np.diff(tr[0]) <= 1e-9 * np.abs(tr[0][:-1]))
    assert np.allclose(Tm[0] @ V[0], t[:, None] * v[None, :], rtol=1e-3)
    Tm, V, _, _ = io.is_nmf(np.full((1, 1, 1), 2.5), 1, 50, 9)
    assert Tm[0, 0, 0] * V[0, 0, 0] == pytest.approx(2.5, rel=1e-3)
    h0 = 0.1 + np.random.default_rng(47).random((5, 12, 2))
    _, _, tr, _ = io.is_nmf(h0, 3, 200, 5)
    for s in tr:
        assert np.all(np.diff(s) <= 1e-9 * np.abs(s[:-1]))


def test_gevd_reference_cases():
    # test_hermlin.cpp:98-138
    w, d = io.gevd(np.diag([2.0, 3.0]).astype(complex), np.eye(2, dtype=complex))
    assert d[0] == pytest.approx(3.0) and d[1] == pytest.approx(2.0)
    assert abs(np.abs(w[:, 0]).max() - 1) < 1e-12 and abs(abs(w[1, 0]) - 1) < 1e-12 and abs(abs(w[0, 1]) - 1) < 1e-12
    a = random_hpd(3, np.random.default_rng(7))
    w, d = io.gevd(a, a)
    assert np.allclose(d, 1.0, atol=1e-10)
    assert np.linalg.norm(w.conj().T @ a @ w - np.eye(3)) < 1e-10
    for seed in range(20):
        rng = np.random.default_rng(seed)
        g = rng.standard_normal((4, 3)) + 1j * rng.standard_normal((4, 3))
        a = g @ g.conj().T
        b = random_hpd(4, rng)
        w, d = io.gevd(a, b)
        assert np.linalg.norm(w.conj().T @ b @ w - np.eye(4)) <= 1e-10
        waw = w.conj().T @ a @ w
        np.fill_diagonal(waw, 0)
        assert np.linalg.norm(waw) <= 1e-9 * np.linalg.norm(a)
        assert np.all(np.diff(d) <= 0)
    b = np.zeros((2, 2), dtype=complex)
    b[0, 0] = 1
    with pytest.raises(RuntimeError, match="not positive definite"):
        io.gevd(np.eye(2, dtype=complex), b)


def test_init_spatial_reference_cases():
    # test_init.cpp:307-393
    R = np.zeros((2, 1, 2, 2), dtype=complex)
    R[0, 0] = np.diag([2.0, 1.0])
    R[1, 0] = np.eye(2)
    w0, lam = io.init_spatial(R, [2])
    assert np.allclose(np.linalg.norm(w0[0][0], axis=0), 1.0, atol=1e-5)
    assert np.allclose(lam[0], [[2.0, 1.0], [1.0, 1.0]], atol=1e-5)
    for seed in range(5):
        rng = np.random.default_rng(seed)
        q, _ = np.linalg.qr(rng.standard_normal((3, 3)) + 1j * rng.standard_normal((3, 3)))
        e1, e2 = 0.5 + rng.random(3), 0.5 + rng.random(3)
        R = np.stack([q @ np.diag(e1) @ q.conj().T, q @ np.diag(e2) @ q.conj().T])[:, None]
        w0, lam = io.init_spatial(R, [3])
        w = w0[0][0]
        for n in range(2):
            d = w.conj().T @ R[n, 0] @ w
            sc = np.linalg.norm(d)
            np.fill_diagonal(d, 0)
            assert np.linalg.norm(d) <= 1e-6 * sc
        assert np.linalg.norm(w.conj().T @ R[1, 0] @ w - np.eye(3)) <= 1e-4
    rng = np.random.default_rng(53)
    R = np.stack([random_hpd(3, rng) for _ in range(3)])[:, None]
    w0, lam = io.init_spatial(R, [3])
    assert lam.min() >= 0 and np.all(np.isfinite(w0[0]))
    assert np.linalg.norm(w0[0][0].conj().T @ R[2, 0] @ w0[0][0] - np.eye(3)) <= 1e-4
    # block slicing agrees (test_init.cpp:369-393)
    rng = np.random.default_rng(59)
    R = np.zeros((2, 1, 5, 5), dtype=complex)
    for n in range(2):
        R[n, 0, :2, :2] = random_hpd(2, rng)
        R[n, 0, 2:, 2:] = random_hpd(3, rng)
    wb, lb = io.init_spatial(R, [2, 3])
    for l, (o, mb) in enumerate([(0, 2), (2, 3)]):
        ws, ls = io.init_spatial(np.ascontiguousarray(R[:, :, o:o + mb, o:o + mb]), [mb])
        assert np.array_equal(wb[l], ws[0]) and np.array_equal(lb[:, :, o:o + mb], ls)


def test_pipeline_is_deterministic_and_distributed_fills_blocks():
    # test_init.cpp:395-418
    x, _ = two_source_scene(8, 40, 61)
    a = io.init_full(x, 2, 3, 12345, nmf_iters=50)
    b = io.init_full(x, 2, 3, 12345, nmf_iters=50)
    c = io.init_full(x, 2, 3, 54321, nmf_iters=50)
    assert np.array_equal(a["T"], b["T"]) and np.array_equal(a["lambda0"], b["lambda0"])
    assert np.array_equal(a["w0"][0], b["w0"][0])
    assert not np.array_equal(a["T"], c["T"])
    assert a["T"].min() > 0 and a["lambda0"].min() >= 1e-6
    x2, _ = two_source_scene(8, 40, 67)
    rng = np.random.default_rng(71)
    x4 = np.concatenate([x2, x2 + 0.05 * (rng.standard_normal(x2.shape) + 1j * rng.standard_normal(x2.shape))], 2)
    d = io.init_distributed(x4, [2, 2], 2, 3, 77, nmf_iters=50)
    assert len(d["w0"]) == 2 and d["w0"][0].shape == (8, 2, 2) and d["lambda0"].shape == (8, 2, 4)
    assert d["T"].shape == (2, 8, 3) and d["lambda0"].min() >= 1e-6
