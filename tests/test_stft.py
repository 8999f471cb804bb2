"""STFT / inverse STFT (stft.cpp:74-141): the reference's own test cases
(test_stft.cpp:33-156) pin the oracle restatement (oracle/stft.py) on the
CPU; the device transforms (csrc/dfm_stft.cu through the C ABI) are then
compared with the oracle on the same seeded signals and re-run through the
same test cases on the GPU."""
import math

import numpy as np
import pytest

import stft as ost


def random_signal(length, channels, seed):
    return np.random.default_rng(seed).standard_normal((length, channels))


def interior_error(a, b, margin):
    da, db = a[margin:len(a) - margin], b[margin:len(b) - margin]
    return np.linalg.norm(da - db) / np.linalg.norm(da)


# ------------------------------------------------------------- oracle pins
def test_oracle_fft_matches_numpy():
    rng = np.random.default_rng(0)
    for n in (1, 2, 8, 64, 1024, 12, 7):
        a = rng.standard_normal(n) + 1j * rng.standard_normal(n)
        ref = np.fft.fft(a)
        assert np.linalg.norm(ost.fft(a) - ref) <= 1e-12 * max(1.0, np.linalg.norm(ref))
        assert np.linalg.norm(ost.fft(a, inverse=True) - np.fft.ifft(a)) <= 1e-12 * max(1.0, np.linalg.norm(a))


def test_oracle_silence_shapes_and_paper_parameters():
    # test_stft.cpp:33-51
    x = ost.stft_forward(np.zeros((16000, 2)), 4096, 1024)
    assert x.shape == (2049, (16000 - 4096) // 1024 + 1, 2) and not np.any(x)
    assert ost.num_frames(160000, 4096, 1024) == (160000 - 4096) // 1024 + 1


def test_oracle_bin_center_sinusoid_concentrates_energy():
    # test_stft.cpp:53-70
    n, hop, sr, b = 512, 128, 16000.0, 40
    t = np.arange(8192)
    s = np.sin(2 * math.pi * (b * sr / n) * t / sr)[:, None]
    p = np.abs(ost.stft_forward(s, n, hop)[:, :, 0]) ** 2
    assert np.all(p[b - 1:b + 2].sum(0) / p.sum(0) >= 0.99)


@pytest.mark.parametrize("n,hop,length,ch,seed,margin,tol", [
    (1024, 256, 8192, 3, 42, 1024, 1e-10),   # test_stft.cpp:72-78
    (12, 3, 240, 1, 3, 12, 1e-10),           # :140-147 non-power-of-two
])
def test_oracle_round_trip_interior(n, hop, length, ch, seed, margin, tol):
    s = random_signal(length, ch, seed)
    r = ost.stft_inverse(ost.stft_forward(s, n, hop), n, hop, length)
    assert interior_error(s, r, margin) <= tol


def test_oracle_tiny_window_zero_tensor_linearity_and_errors():
    s = (0.01 * np.arange(64))[:, None]  # test_stft.cpp:88-95
    assert interior_error(s, ost.stft_inverse(ost.stft_forward(s, 8, 2), 8, 2, 64), 8) <= 1e-12
    r = ost.stft_inverse(np.zeros((129, 10, 2), complex), 256, 64, 1000)  # :97-103
    assert r.shape == (1000, 2) and not np.any(r)
    s1, s2 = random_signal(2048, 2, 1), random_signal(2048, 2, 2)  # :105-115
    xa = ost.stft_forward(2.5 * s1 - 0.5 * s2, 256, 64)
    d = xa - 2.5 * ost.stft_forward(s1, 256, 64) + 0.5 * ost.stft_forward(s2, 256, 64)
    assert np.all(np.linalg.norm(d, axis=(1, 2)) <= 1e-12 * (1 + np.linalg.norm(xa, axis=(1, 2))))
    with pytest.raises(ValueError, match="shorter than one window"):  # :134-137
        ost.stft_forward(np.zeros((100, 1)), 256, 64)


# ------------------------------------------------------------- device path
gpu = pytest.mark.gpu


@pytest.fixture(scope="module")
def st():
    import torch

    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    import paper_2605_19388_b200.stft as m

    return m


@gpu
@pytest.mark.parametrize("n,hop,length,ch", [(1024, 256, 8192, 3), (256, 64, 2048, 2), (12, 3, 240, 2),
                                              (8, 2, 64, 1), (4096, 1024, 48000, 1), (1, 1, 5, 2), (100, 100, 1000, 1)])
def test_device_stft_matches_oracle(st, n, hop, length, ch):
    s = random_signal(length, ch, 11 + n)
    cfg = st.StftConfig(16000.0, n, hop)
    x = st.stft_forward(s, cfg)
    xo = ost.stft_forward(s, n, hop)
    assert x.shape == xo.shape
    assert np.linalg.norm(x - xo) <= 1e-12 * np.linalg.norm(xo)
    r = st.stft_inverse(x, cfg, length + 17)
    ro = ost.stft_inverse(xo, n, hop, length + 17)
    assert r.shape == ro.shape == (length + 17, ch)
    assert np.linalg.norm(r - ro) <= 1e-12 * max(np.linalg.norm(ro), 1e-300)
    if 2 * hop <= n:  # samples at the window's zeros need overlapping frames
        assert interior_error(s, r[:length], n) <= 1e-10


@gpu
def test_device_reference_cases(st):
    cfg = st.StftConfig(16000.0, 4096, 1024)  # test_stft.cpp:33-43
    assert st.stft_num_bins(cfg) == 2049
    x = st.stft_forward(np.zeros((16000, 2)), cfg)
    assert x.shape == (2049, (16000 - 4096) // 1024 + 1, 2) and not np.any(x)
    p = st.StftConfig.from_ms(16000.0, 256.0, 64.0)  # :45-51
    assert (p.window_len, p.hop_len) == (4096, 1024)
    assert st.stft_num_frames(p, 160000) == (160000 - 4096) // 1024 + 1
    s = random_signal(3 * 16000, 1, 7)  # :80-86 paper-parameter round trip
    r = st.stft_inverse(st.stft_forward(s, p), p, len(s))
    assert interior_error(s, r, 4096) <= 1e-10
    cfg = st.StftConfig(16000.0, 512, 128)  # :53-70 sinusoid
    t = np.arange(8192)
    pw = np.abs(st.stft_forward(np.sin(2 * math.pi * (40 * 16000.0 / 512) * t / 16000.0)[:, None], cfg)[:, :, 0]) ** 2
    assert np.all(pw[39:42].sum(0) / pw.sum(0) >= 0.99)
    z = st.stft_inverse(np.zeros((129, 10, 2), complex), st.StftConfig(8000.0, 256, 64), 1000)  # :97-103
    assert z.shape == (1000, 2) and not np.any(z)
    c = st.StftConfig(8000.0, 256, 64)  # :117-132 channel permutation energy
    s = random_signal(2048, 3, 9)
    e1 = np.sum(np.abs(st.stft_forward(s, c)) ** 2)
    e2 = np.sum(np.abs(st.stft_forward(s[:, [2, 0, 1]], c)) ** 2)
    assert e1 == pytest.approx(e2, rel=1e-12)


@gpu
def test_device_errors(st):
    import paper_2605_19388_b200 as dfm

    c = st.StftConfig(8000.0, 256, 64)
    with pytest.raises(dfm._capi.SignalTooShortError):
        st.stft_forward(np.zeros((100, 1)), c)
    with pytest.raises(ValueError, match="window_len >= hop_len"):
        st.stft_forward(np.zeros((1000, 1)), st.StftConfig(8000.0, 64, 128))
    bad = np.zeros((1000, 1))
    bad[5] = np.nan
    with pytest.raises(ValueError, match="non-finite"):
        st.stft_forward(bad, c)
    with pytest.raises(dfm.ShapeMismatchError, match="bin count"):
        st.stft_inverse(np.zeros((100, 3, 1), complex), c, 500)
