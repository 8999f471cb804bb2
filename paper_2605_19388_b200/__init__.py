"""B200-native distributed-FastMNMF EM path (hand-written sm_100a kernels
behind the C ABI in include/dfm_b200.h).  See DESIGN.md."""
from . import _capi  # noqa: F401
from .fastmnmf import (  # noqa: F401
    BlockLayout, BlockSpatialModel, DeviceError, DistFit, Engine, FitOptions, FitReport, FitSnapshot,
    FullFit, InitBundle, NmfModel, NotPositiveDefiniteError, ShapeMismatchError, SingularDemixerError,
    SourceImages, SpatialModel, build_spectrogram, compute_eta, cost_dist, cost_full, decorrelate,
    decorrelate_blocks, extract_block, fit_distributed, fit_full, fit_single, generate_mixture,
    ip_update_block, ip_update_w, kFloor, mm_update_lambda, mm_update_t, mm_update_v, power_of,
    fit_many, random_init, random_observations, slice_init, trace_run, TraceResult, TraceRow, wiener_block,
    wiener_full)

from . import container, init, stft  # noqa: F401,E402
from ._capi import SignalTooShortError  # noqa: F401,E402

__all__ = [n for n in dir() if not n.startswith("_")]
