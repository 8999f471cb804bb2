"""Hann-window STFT and weighted overlap-add inverse on the device (mirror of
include/fastmnmf/stft.hpp:8-40 and reconstruct, wiener.cpp:71-77), through
the C ABI (dfm_stft_*, csrc/dfm_stft.cu).

Shapes follow the rest of the package: signals are (samples, channels),
spectra are ObsTensor-shaped complex (F, T, M)."""
from __future__ import annotations

import math
from dataclasses import dataclass
from typing import List, Sequence

import numpy as np

from . import _capi
from ._capi import check


@dataclass
class StftConfig:
    """stft.hpp:8-21."""
    sample_rate: float = 16000.0
    window_len: int = 4096  # 256 ms at 16 kHz
    hop_len: int = 1024     # 64 ms at 16 kHz

    @staticmethod
    def from_ms(sample_rate: float, window_ms: float, hop_ms: float) -> "StftConfig":
        # std::lround: half away from zero
        rnd = lambda v: int(math.floor(v + 0.5)) if v >= 0 else -int(math.floor(-v + 0.5))
        return StftConfig(sample_rate, rnd(window_ms * 1e-3 * sample_rate), rnd(hop_ms * 1e-3 * sample_rate))


def stft_num_bins(cfg: StftConfig) -> int:
    return cfg.window_len // 2 + 1


def stft_num_frames(cfg: StftConfig, signal_len: int) -> int:
    return int(_capi.load().dfm_stft_num_frames(int(signal_len), cfg.window_len, cfg.hop_len))


def hann_window(n: int) -> np.ndarray:
    """Periodic Hann, zero at the first sample (stft.cpp:63-68)."""
    t = np.arange(n, dtype=np.float64)
    return 0.5 - 0.5 * np.cos(2.0 * math.pi * t / n)


def stft_forward(signal: np.ndarray, cfg: StftConfig, device: int = 0) -> np.ndarray:
    """One-sided spectrum per frame; frame j covers [j hop, j hop + window)."""
    s = np.asarray(signal, dtype=np.float64)
    if s.ndim == 1:
        s = s[:, None]
    length, M = s.shape
    sc = np.ascontiguousarray(s.T)  # Eigen col-major samples x channels
    T = max(stft_num_frames(cfg, length), 0)
    out = np.zeros((stft_num_bins(cfg), T, M), dtype=np.complex128)
    lib = _capi.load()
    check(lib.dfm_stft_forward(sc.ctypes.data_as(_capi.C.c_void_p), length, M, cfg.window_len, cfg.hop_len,
                               out.ctypes.data_as(_capi.C.c_void_p), device))
    return out


def stft_inverse(x: np.ndarray, cfg: StftConfig, out_len: int, device: int = 0) -> np.ndarray:
    """Weighted overlap-add inverse; (out_len, channels)."""
    x = np.ascontiguousarray(x, dtype=np.complex128)
    if x.ndim != 3:
        raise ValueError("stft_inverse: expected a complex (F, T, M) array")
    F, T, M = x.shape
    out = np.zeros((M, max(out_len, 0)))
    lib = _capi.load()
    check(lib.dfm_stft_inverse(x.ctypes.data_as(_capi.C.c_void_p) if x.size else None, F, T, M, cfg.window_len,
                               cfg.hop_len, int(out_len), out.ctypes.data_as(_capi.C.c_void_p) if out.size else None,
                               device))
    return np.ascontiguousarray(out.T)


def reconstruct(images: Sequence[np.ndarray], cfg: StftConfig, out_len: int) -> List[np.ndarray]:
    """wiener.cpp:71-77: the inverse STFT of every separated source image."""
    return [stft_inverse(img, cfg, out_len) for img in images]
