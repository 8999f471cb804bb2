"""Mirror of the reference's Python module ``_fastmnmf`` (proj/python/module.cpp)
running on the B200 engine:

  stft(samples, sample_rate, window_len, hop_len)                      module.cpp:135-141
  istft(x, sample_rate, window_len, hop_len, out_len)                  module.cpp:143-152
  fit_full(x, n_sources, k_bases=16, iterations=200, seed=0)            module.cpp:156-170
  fit_distributed(x, partition, n_sources, k_bases=16, iterations=200,
                  seed=0, share_spectrograms=True)                      module.cpp:172-188
  separate(samples, sample_rate, method, partition=[], n_sources=3,
           k_bases=16, iterations=200, window_len=4096, hop_len=1024,
           seed=0, share_spectrograms=True)                             module.cpp:88-125, 190-195

Same argument names, defaults and report dictionaries (``report_to_dict``,
module.cpp:72-84); the typed exceptions are re-exported under the binding's
names (module.cpp:132-134).  As in the reference, fit_full / fit_distributed
/ separate start from the initialisation pipeline (init_full /
init_distributed, init.cpp:428-472), which runs on the device here.  The
room simulation and SDR entry points are outside this build.
"""
from __future__ import annotations

import numpy as np

from . import fastmnmf as _f
from ._capi import NotPositiveDefiniteError, ShapeMismatchError, SingularDemixerError  # noqa: F401

ShapeMismatchError = ShapeMismatchError
SingularDemixerError = SingularDemixerError
NotPositiveDefiniteError = NotPositiveDefiniteError


def _report_to_dict(report: _f.FitReport) -> dict:
    return {
        "cost_trace": [float(v) for v in report.cost_trace],
        "wall_seconds": [float(v) for v in report.wall_seconds],
        "iterations": int(report.iterations),
        "stages": {k: float(v) for k, v in report.stages.items()},
    }


def _tensor(x) -> np.ndarray:
    arr = np.asarray(x)
    if arr.ndim != 3:
        raise ValueError("expected a complex array of shape (I, J, M)")
    return np.ascontiguousarray(arr, dtype=np.complex128)


def _init_cfg(n_sources: int, k_bases: int):
    from .init import InitConfig

    return InitConfig(num_sources=n_sources, k_bases=k_bases)


def stft(samples, sample_rate: float, window_len: int, hop_len: int) -> np.ndarray:
    """One-sided STFT; returns a complex array of shape (bins, frames, channels)."""
    from . import stft as _s

    return _s.stft_forward(np.asarray(samples, dtype=np.float64), _s.StftConfig(sample_rate, window_len, hop_len))


def istft(x, sample_rate: float, window_len: int, hop_len: int, out_len: int) -> np.ndarray:
    """Overlap-add inverse of stft()."""
    from . import stft as _s

    return _s.stft_inverse(np.asarray(x), _s.StftConfig(sample_rate, window_len, hop_len), out_len)


def fit_full(x, n_sources: int, k_bases: int = 16, iterations: int = 200, seed: int = 0) -> dict:
    """Full-array estimation; returns the fit report."""
    from .init import init_full

    x = _tensor(x)
    init = init_full(x, _init_cfg(n_sources, k_bases), seed)
    return _report_to_dict(_f.fit_full(x, init, iterations).report)


def fit_distributed(x, partition, n_sources: int, k_bases: int = 16, iterations: int = 200, seed: int = 0,
                    share_spectrograms: bool = True) -> dict:
    """Distributed estimation with block-diagonal spatial covariances."""
    from .init import init_distributed

    x = _tensor(x)
    layout = _f.BlockLayout(partition)
    init = init_distributed(x, layout, _init_cfg(n_sources, k_bases), seed)
    return _report_to_dict(_f.fit_distributed(x, layout, init, iterations, share_spectrograms).report)


def separate(samples, sample_rate: float, method: str, partition=(), n_sources: int = 3, k_bases: int = 16,
             iterations: int = 200, window_len: int = 4096, hop_len: int = 1024, seed: int = 0,
             share_spectrograms: bool = True) -> dict:
    """End-to-end separation of a (T, M) mixture (module.cpp:88-125): STFT,
    initialisation, EM fit, Wiener separation and inverse STFT; returns
    {"sources": [per-source (T, M) waveforms], "report": {...}}."""
    from . import stft as _s
    from .init import init_distributed, init_full

    sig = np.asarray(samples, dtype=np.float64)
    if sig.ndim == 1:
        sig = sig[:, None]
    cfg = _s.StftConfig(sample_rate, window_len, hop_len)
    x = _s.stft_forward(sig, cfg)
    icfg = _init_cfg(n_sources, k_bases)
    if method in ("full", "single"):
        init = init_full(x, icfg, seed)
        fit = _f.fit_full(x, init, iterations)
        images = _f.wiener_full(x, fit.nmf, fit.spatial)
    elif method == "distributed":
        layout = _f.BlockLayout(list(partition))
        init = init_distributed(x, layout, icfg, seed)
        fit = _f.fit_distributed(x, layout, init, iterations, share_spectrograms)
        images = _f.wiener_block(x, fit.models, fit.spatial)
    else:
        raise ValueError("method must be full, single or distributed")
    sources = _s.reconstruct(list(images.images), cfg, sig.shape[0])
    return {"sources": sources, "report": _report_to_dict(fit.report)}
