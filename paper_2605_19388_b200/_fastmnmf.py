"""Mirror of the reference's Python module ``_fastmnmf`` (proj/python/module.cpp)
for the entry points on the EM path, running on the B200 engine.

  fit_full(x, n_sources, k_bases=16, iterations=200, seed=0)            module.cpp:156-170
  fit_distributed(x, partition, n_sources, k_bases=16, iterations=200,
                  seed=0, share_spectrograms=True)                      module.cpp:172-188

Same argument names, defaults and report dictionaries (``report_to_dict``,
module.cpp:72-84); the typed exceptions are re-exported under the binding's
names (module.cpp:132-134).  One documented difference: the reference seeds
the fit with its CPU initialisation pipeline (init_full / init_distributed,
init.cpp:428-472), which is outside this path; here the
seed drives random_init (init.cpp:496-521), as the reference's own benchmark
does (bench.cpp:83-88).  The STFT, simulation and SDR entry points are out of
scope for this build.
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


def fit_full(x, n_sources: int, k_bases: int = 16, iterations: int = 200, seed: int = 0) -> dict:
    """Full-array estimation; returns the fit report."""
    x = _tensor(x)
    F, T, M = x.shape
    layout = _f.BlockLayout.full(M)
    init = _f.random_init(F, T, layout, n_sources, k_bases, seed)
    return _report_to_dict(_f.fit_full(x, init, iterations).report)


def fit_distributed(x, partition, n_sources: int, k_bases: int = 16, iterations: int = 200, seed: int = 0,
                    share_spectrograms: bool = True) -> dict:
    """Distributed estimation with block-diagonal spatial covariances."""
    x = _tensor(x)
    F, T, M = x.shape
    layout = _f.BlockLayout(partition)
    init = _f.random_init(F, T, layout, n_sources, k_bases, seed)
    return _report_to_dict(_f.fit_distributed(x, layout, init, iterations, share_spectrograms).report)
