"""TEST INFRASTRUCTURE ONLY (checker, never shipped): numpy restatement of
the reference's STFT, src/stft.cpp:1-141, used to pin the device STFT
(csrc/dfm_stft.cu).

* fft: radix-2 with bit reversal and twiddles by the recurrence w *= wlen
  (stft.cpp:14-35) for power-of-two sizes; the plain DFT with the angle
  2 pi (k t mod n) / n otherwise (:37-50); inverse scaled by 1/n (:55-58).
* hann_window: periodic Hann (:63-68).
* stft_forward (:70-94) and stft_inverse (:96-139), including the
  window-square floor at half the full overlap.
"""
import math

import numpy as np

TWO_PI = 6.283185307179586476925286766559


def _fft_radix2(a, inverse):
    n = a.shape[-1]
    a = a.copy()
    j = 0
    for i in range(1, n):  # bit reversal (stft.cpp:17-22)
        bit = n >> 1
        while j & bit:
            j ^= bit
            bit >>= 1
        j ^= bit
        if i < j:
            a[..., [i, j]] = a[..., [j, i]]
    length = 2
    while length <= n:
        ang = (TWO_PI if inverse else -TWO_PI) / length
        wlen = complex(math.cos(ang), math.sin(ang))
        half = length // 2
        w = np.empty(half, dtype=np.complex128)
        cur = complex(1.0, 0.0)
        for k in range(half):  # w *= wlen, the reference's recurrence
            w[k] = cur
            cur = cur * wlen
        blk = a.reshape(a.shape[:-1] + (n // length, length))
        u = blk[..., :half].copy()
        v = blk[..., half:] * w
        blk[..., :half] = u + v
        blk[..., half:] = u - v
        a = blk.reshape(a.shape)
        length <<= 1
    return a


def _dft(a, inverse):
    n = a.shape[-1]
    k = np.arange(n)
    kt = (k[:, None] * k[None, :]) % n
    sign = 1.0 if inverse else -1.0
    ang = sign * TWO_PI * kt.astype(np.float64) / n
    e = np.cos(ang) + 1j * np.sin(ang)
    return a @ e.T


def fft(a, inverse=False):
    a = np.asarray(a, dtype=np.complex128)
    n = a.shape[-1]
    if n <= 1:
        return a.copy()
    out = _fft_radix2(a, inverse) if (n & (n - 1)) == 0 else _dft(a, inverse)
    if inverse:
        out = out * (1.0 / n)
    return out


def hann_window(n):
    t = np.arange(n, dtype=np.float64)
    return 0.5 - 0.5 * np.cos(2.0 * math.pi * t / n)


def num_frames(length, window, hop):
    return 0 if length < window else (length - window) // hop + 1


def stft_forward(signal, window, hop):
    """signal (len, M) -> X (F, T, M) complex."""
    s = np.asarray(signal, dtype=np.float64)
    if window < 1 or hop < 1 or hop > window:
        raise ValueError("stft_forward: need window_len >= hop_len >= 1")
    if not np.all(np.isfinite(s)):
        raise ValueError("stft_forward: non-finite samples")
    length, M = s.shape
    if length < window:
        raise ValueError("stft_forward: signal shorter than one window")
    T, F = num_frames(length, window, hop), window // 2 + 1
    w = hann_window(window)
    idx = np.arange(T)[:, None] * hop + np.arange(window)[None, :]
    frames = s[idx, :].transpose(2, 0, 1) * w  # (M, T, n)
    spec = fft(frames.astype(np.complex128))
    return np.ascontiguousarray(spec[..., :F].transpose(2, 1, 0))


def stft_inverse(x, window, hop, out_len):
    """X (F, T, M) -> (out_len, M)."""
    x = np.asarray(x, dtype=np.complex128)
    F, T, M = x.shape
    if F != window // 2 + 1:
        raise ValueError("stft_inverse: bin count does not match the config")
    w = hann_window(window)
    covered = (T - 1) * hop + window if T > 0 else 0
    acc_len = max(covered, out_len)
    acc = np.zeros((acc_len, M))
    den = np.zeros(acc_len)
    for m in range(M):
        for j in range(T):
            buf = np.empty(window, dtype=np.complex128)
            buf[:F] = x[:, j, m]
            for i in range(F, window):
                buf[i] = np.conj(buf[window - i])
            y = fft(buf, inverse=True)
            st = j * hop
            acc[st:st + window, m] += y.real * w
            if m == 0:
                den[st:st + window] += w * w
    den_floor = max(1e-12, 0.5 * den.max()) if acc_len else 1e-12
    out = np.zeros((out_len, M))
    n = min(out_len, covered)
    for t in range(n):
        if den[t] > 1e-12:
            out[t] = acc[t] / max(den[t], den_floor)
    return out
