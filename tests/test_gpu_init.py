"""The device initialisation pipeline (csrc/dfm_init.cu + the host alignment)
against the oracle restatement (oracle/dfm_init_oracle.c) on the same seeded
inputs, plus the reference's own init tests (test_init.cpp) re-run on the
device path and an end-to-end separate() check.

Tolerances: the k-means masks, SCMs, ML spectrograms and the GEVD follow the
oracle's operation order and differ only by FMA contraction and the device's
exp / hypot (1e-10); IS-NMF sums its GEMMs on the FP64 tensor cores in
another order, so its divergence traces and factors are compared at 1e-7
relative over up to 1000 multiplicative iterations."""
import numpy as np
import pytest

import init_oracle as io
import oracle as orc

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def di():
    import torch

    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    import paper_2605_19388_b200.init as m

    return m


def two_source_scene(F, T, seed):
    rng = np.random.default_rng(seed)
    active = np.array([(j // 8) % 2 for j in range(T)])
    x = np.zeros((F, T, 2), dtype=np.complex128)
    for i in range(F):
        th = 0.3 + 0.11 * i
        a0, a1 = np.array([1.0, np.exp(1j * th)]), np.array([1.0, np.exp(1j * (th + np.pi))])
        for j in range(T):
            s = rng.standard_normal() + 1j * rng.standard_normal()
            x[i, j] = (a0 if active[j] == 0 else a1) * s
    return x, active


def _mix(F, T, M, N, K, seed):
    import paper_2605_19388_b200 as dfm

    return dfm.generate_mixture(0, F, T, M, N, K, seed)


@pytest.mark.parametrize("F,T,M,N,seed", [(12, 64, 2, 2, 3), (20, 80, 4, 3, 4), (16, 50, 3, 4, 5), (9, 30, 12, 5, 6)])
def test_device_masks_match_oracle(di, F, T, M, N, seed):
    x = _mix(F, T, M, N, 4, seed)
    x[F // 2] = 0  # a silent bin keeps the uniform mask
    a = di.cluster_masks(x, N, 1000 + seed)
    b = io.cluster_masks(x, N, 1000 + seed)
    assert a.shape == (F, T, N)
    assert np.allclose(a.sum(axis=2), 1.0, atol=1e-12)
    assert np.array_equal(a.argmax(axis=2), b.argmax(axis=2))
    assert np.max(np.abs(a - b)) <= 1e-10
    assert np.array_equal(a[F // 2], np.full((T, N), 1.0 / N))


def test_device_mask_reference_cases(di):
    rng = np.random.default_rng(1)
    x = rng.standard_normal((3, 10, 2)) + 1j * rng.standard_normal((3, 10, 2))
    assert np.array_equal(di.cluster_masks(x, 1, 7), np.ones((3, 10, 1)))
    with pytest.raises(ValueError, match="fewer frames than sources"):
        di.cluster_masks(x[:, :2], 3, 1)
    x, act = two_source_scene(12, 64, 3)  # test_init.cpp:65-82
    m = di.cluster_masks(x, 2, 5)
    pur = [max(np.mean((m[i, :, 0] < m[i, :, 1]) == act), 1 - np.mean((m[i, :, 0] < m[i, :, 1]) == act))
           for i in range(12)]
    assert np.mean(pur) >= 0.9


def test_device_scm_and_spectrogram_match_oracle(di):
    rng = np.random.default_rng(11)
    F, T, M, N, sizes = 7, 40, 5, 3, [2, 3]
    x = rng.standard_normal((F, T, M)) + 1j * rng.standard_normal((F, T, M))
    masks = [rng.random((F, T, N)) for _ in sizes]
    R, h0 = di._scm_spec(x, sizes, masks)
    Ro = io.init_scm(x, sizes, masks)
    ho = io.init_spectrogram(x, sizes, masks, Ro)
    assert np.linalg.norm(R - Ro) <= 1e-12 * np.linalg.norm(Ro)
    assert np.linalg.norm(h0 - ho) <= 1e-10 * np.linalg.norm(ho)
    # test_init.cpp:226-254 closed forms on the device
    c = rng.standard_normal((2, 16, 1)) + 1j * rng.standard_normal((2, 16, 1))
    h = di.init_spectrogram([c])
    for i in range(2):
        mp = np.sum(np.abs(c[i]) ** 2) / 16
        assert np.allclose(h[i, :, 0], np.abs(c[i, :, 0]) ** 2 / mp, rtol=1e-4)
    assert not np.any(di.init_spectrogram([np.zeros((1, 8, 2), complex)]))


@pytest.mark.parametrize("F,T,N,K,iters", [(20, 30, 2, 3, 200), (33, 41, 3, 5, 1000), (8, 12, 1, 2, 60)])
def test_device_is_nmf_matches_oracle(di, F, T, N, K, iters):
    h0 = 0.05 + np.random.default_rng(F).random((F, T, N)) ** 2
    tr = []
    model = di.itakura_saito_nmf(h0, K, iters, 77, tr)
    To, Vo, tro, its = io.is_nmf(h0, K, iters, 77)
    for n in range(N):
        assert abs(len(tr[n]) - len(tro[n])) <= 1
        L = min(len(tr[n]), len(tro[n]))
        assert np.allclose(tr[n][:L], tro[n][:L], rtol=1e-7)
        assert np.all(np.diff(tr[n]) <= 1e-9 * np.abs(tr[n][:-1]))
    rec = np.einsum("nfk,nkt->nft", model.T, model.V)
    reco = np.einsum("nfk,nkt->nft", To, Vo)
    assert np.linalg.norm(rec - reco) <= 1e-6 * np.linalg.norm(reco)


def test_device_is_nmf_reference_cases(di):
    rng = np.random.default_rng(41)  # test_init.cpp:256-280 rank-one
    t, v = 0.5 + rng.random(6), 0.5 + rng.random(10)
    tr = []
    m = di.itakura_saito_nmf((t[:, None] * v[None, :])[:, :, None], 1, 1000, 3, tr)
    assert tr[0][-1] <= 1e-6
    assert np.allclose(m.T[0] @ m.V[0], t[:, None] * v[None, :], rtol=1e-3)
    m = di.itakura_saito_nmf(np.full((1, 1, 1), 2.5), 1, 50, 9)  # :282-288
    assert m.T[0, 0, 0] * m.V[0, 0, 0] == pytest.approx(2.5, rel=1e-3)


def test_device_init_spatial_matches_oracle(di):
    import paper_2605_19388_b200 as dfm

    rng = np.random.default_rng(21)
    F, N, sizes = 9, 3, [4, 4, 4]
    M = sum(sizes)
    R = np.zeros((N, F, M, M), dtype=complex)
    for n in range(N):
        for f in range(F):
            g = rng.standard_normal((M, M + 2)) + 1j * rng.standard_normal((M, M + 2))
            R[n, f] = g @ g.conj().T / M
    R[N - 1, 3] = 0  # silent pair -> identity demixer
    w, lam = di.init_spatial(R, dfm.BlockLayout(sizes))
    wo, lamo = io.init_spatial(R, sizes)
    for a, b in zip(w, wo):
        assert np.max(np.abs(a - b)) <= 1e-9
    assert np.max(np.abs(lam - lamo) / lamo) <= 1e-9
    assert np.array_equal(w[0][3], np.eye(4))
    assert lam.min() >= 1e-6
    # test_init.cpp:344-367: w^H R_N w = I on the GEVD pair
    for b, o in enumerate([0, 4, 8]):
        for f in (0, 5):
            wb = w[b][f]
            Rb = R[N - 1, f][o:o + 4, o:o + 4] + 1e-6 * np.trace(R[N - 1, f][o:o + 4, o:o + 4]).real / 4 * np.eye(4)
            assert np.linalg.norm(wb.conj().T @ Rb @ wb - np.eye(4)) <= 1e-9


def test_device_pipeline_matches_oracle_and_fits(di):
    import paper_2605_19388_b200 as dfm

    F, T, sizes, N, K = 24, 60, [2, 2], 3, 4
    x = _mix(F, T, 4, N, K, 31)
    layout = dfm.BlockLayout(sizes)
    cfg = di.InitConfig(num_sources=N, k_bases=K, nmf_max_iters=300)
    b = di.init_distributed(x, layout, cfg, 12345)
    o = io.init_distributed(x, sizes, N, K, 12345, nmf_iters=300)
    assert np.max(np.abs(b.mask - o["masks"][0])) <= 1e-10
    assert np.linalg.norm(b.h0 - o["h0"]) <= 1e-9 * np.linalg.norm(o["h0"])
    assert np.max(np.abs(b.lambda0 - o["lambda0"]) / o["lambda0"]) <= 1e-8
    for a, c in zip(b.w0, o["w0"]):
        assert np.max(np.abs(a - c)) <= 1e-8
    rec = np.einsum("nfk,nkt->nft", b.nmf.T, b.nmf.V)
    reco = np.einsum("nfk,nkt->nft", o["T"], o["V"])
    assert np.linalg.norm(rec - reco) <= 1e-6 * np.linalg.norm(reco)
    # deterministic in the seed (test_init.cpp:395-412)
    b2 = di.init_distributed(x, layout, cfg, 12345)
    assert np.array_equal(b.nmf.T, b2.nmf.T) and np.array_equal(b.lambda0, b2.lambda0)
    b3 = di.init_distributed(x, layout, cfg, 54321)
    assert not np.array_equal(b.nmf.T, b3.nmf.T)
    # the EM fit from the device init is monotone and matches the fit from the oracle init
    fit = dfm.fit_distributed(x, layout, b, 25)
    oi = dfm.InitBundle(layout, dfm.NmfModel(o["T"], o["V"]), o["w0"], o["lambda0"])
    fo = dfm.fit_distributed(x, layout, oi, 25)
    ct, co = fit.report.cost_trace, fo.report.cost_trace
    assert np.all(np.diff(ct) <= 1e-9 * np.abs(ct[:-1]))
    assert np.max(np.abs(ct - co) / np.abs(co)) <= 1e-6


def test_separate_end_to_end():
    import paper_2605_19388_b200._fastmnmf as fm

    rng = np.random.default_rng(5)
    L, M = 8000, 4
    t = np.arange(L)
    s1 = np.sin(2 * np.pi * 440 * t / 8000) * (t % 2000 < 1000)
    s2 = rng.standard_normal(L) * (t % 2000 >= 1000)
    a = rng.standard_normal((2, M))
    mix = s1[:, None] * a[0] + s2[:, None] * a[1] + 1e-3 * rng.standard_normal((L, M))
    out = fm.separate(mix, 8000.0, "distributed", [2, 2], n_sources=2, k_bases=4, iterations=15, window_len=256,
                      hop_len=64, seed=3)
    assert len(out["sources"]) == 2 and out["sources"][0].shape == (L, M)
    tr = np.array(out["report"]["cost_trace"])
    assert len(tr) == 16 and np.all(np.diff(tr) <= 1e-9 * np.abs(tr[:-1]))
    # Wiener images add up to the mixture (wiener.cpp completeness) -> so do the waveforms
    tot = out["sources"][0] + out["sources"][1]
    sl = slice(256, L - 256)
    assert np.linalg.norm(tot[sl] - mix[sl]) <= 1e-8 * np.linalg.norm(mix[sl])
    full = fm.separate(mix, 8000.0, "full", n_sources=2, k_bases=4, iterations=5, window_len=256, hop_len=64)
    assert len(full["report"]["cost_trace"]) == 6
    x = fm.stft(mix, 8000.0, 256, 64)
    assert x.shape == (129, (L - 256) // 64 + 1, M)
    back = fm.istft(x, 8000.0, 256, 64, L)
    assert np.linalg.norm(back[sl] - mix[sl]) <= 1e-10 * np.linalg.norm(mix[sl])
