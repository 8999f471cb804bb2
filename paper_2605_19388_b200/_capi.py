"""ctypes binding of the C ABI in include/dfm_b200.h (libdfm_b200.so).

There is no fallback: if the CUDA library is missing or cannot be loaded the
import fails loudly, and every compute entry point raises when no CUDA
device is present.
"""
from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
# DFM_LIB: another build of the library (A/B timing experiments in tools/)
LIB_PATH = os.environ.get("DFM_LIB") or os.path.join(_HERE, "libdfm_b200.so")

_dp = C.POINTER(C.c_double)
_ip = C.POINTER(C.c_int)
_vp = C.c_void_p
_i = C.c_int
_d = C.c_double
_u64 = C.c_uint64
_sz = C.c_size_t
_cp = C.c_char_p

DFM_MAX_BLOCKS = 32


class FmnmHeader(C.Structure):
    """dfm_fmnm_header (include/dfm_b200.h): the FMNM v2 container header."""
    _fields_ = [("version", C.c_uint32), ("num_bins", C.c_uint32), ("num_frames", C.c_uint32),
                ("channels", C.c_uint32), ("n_sources", C.c_uint32), ("k_bases", C.c_uint32),
                ("n_blocks", C.c_uint32), ("sizes", C.c_uint32 * DFM_MAX_BLOCKS), ("shared", C.c_uint32),
                ("floor", C.c_double), ("seed", C.c_uint64), ("sample_rate", C.c_double),
                ("window_len", C.c_uint32), ("hop_len", C.c_uint32), ("iterations", C.c_uint32),
                ("n_models", C.c_uint32)]

# name: (restype, argtypes)
_SIGS = {
    "dfm_last_error": (C.c_char_p, []),
    "dfm_limits": (_i, [_ip, _ip, _ip, _ip]),
    "dfm_create": (_vp, [_i, _i, _i, _ip, _i, _i, _d, _i, _i, _i]),
    "dfm_destroy": (None, [_vp]),
    "dfm_local_bins": (_i, [_vp, _ip, _ip]),
    "dfm_set_obs": (_i, [_vp, _vp]),
    "dfm_set_model": (_i, [_vp, _vp, _vp, _vp, _vp]),
    "dfm_get_model": (_i, [_vp, _vp, _vp, _vp, _vp]),
    "dfm_set_model_native": (_i, [_vp, _vp, _vp, _vp, _vp]),
    "dfm_get_model_native": (_i, [_vp, _vp, _vp, _vp, _vp]),
    "dfm_comm_init": (_i, [_vp, _vp, _i, _i]),
    "dfm_nccl_get_unique_id": (_i, [_vp]),
    "dfm_fit": (_i, [_vp, _i, _vp, _vp, _vp]),
    "dfm_fit_many": (_i, [_vp, _i, _i, _vp, _vp]),
    "dfm_force_collective": (_i, [_vp, _i]),
    "dfm_fmnm_sizes": (_sz, [_vp, _vp, _vp, _vp, _vp]),
    "dfm_stft_num_frames": (_i, [_i, _i, _i]),
    "dfm_cluster_masks": (_i, [_vp, _i, _i, _i, _i, _u64, _i, _d, _i, _i, _vp, _i]),
    "dfm_align_frequency_permutations": (_i, [_vp, _i, _i, _i, _i, _i]),
    "dfm_align_subarray_permutations": (_i, [_vp, _i, _i, _i, _i, _vp]),
    "dfm_init_scm_spectrogram": (_i, [_vp, _i, _i, _i, _i, _i, _vp, _vp, _vp, _vp, _i]),
    "dfm_is_nmf": (_i, [_vp, _i, _i, _i, _i, _i, _u64, _vp, _vp, _vp, _vp, _i]),
    "dfm_init_spatial": (_i, [_vp, _i, _i, _i, _i, _vp, _vp, _vp, _i]),
    "dfm_init_pipeline": (_i, [_vp, _i, _i, _i, _vp, _i, _i, _u64, _i, _i, _d, _i, _i, _vp, _vp, _vp, _vp, _vp,
                               _vp, _i]),
    "dfm_stft_forward": (_i, [_vp, _i, _i, _i, _i, _vp, _i]),
    "dfm_stft_inverse": (_i, [_vp, _i, _i, _i, _i, _i, _i, _vp, _i]),
    "dfm_bench_stft": (_i, [_i, _i, _i, _i, _i, _vp, _vp, _i]),
    "dfm_fmnm_write": (_i, [_cp, _vp, _vp, _vp, _vp, _vp]),
    "dfm_fmnm_read_header": (_i, [_cp, _vp]),
    "dfm_fmnm_read": (_i, [_cp, _vp, _vp, _vp, _vp, _vp]),
    "dfm_bench_step_many": (_i, [_vp, _i, _vp]),
    "dfm_shard_begin": (_i, [_vp, _i]),
    "dfm_shard_numden": (_i, [_vp, _vp]),
    "dfm_shard_advance": (_i, [_vp, _vp]),
    "dfm_shard_end": (_i, [_vp, _vp]),
    "dfm_prime": (_i, [_vp]),
    "dfm_bench_step": (_i, [_vp]),
    "dfm_bench_split_step": (_i, [_vp]),
    "dfm_sync": (_i, [_vp]),
    "dfm_bench_last_ms": (_d, [_vp]),
    "dfm_bench_last_split": (_i, [_vp, _dp]),
    "dfm_launch_count": (C.c_longlong, [_vp]),
    "dfm_set_tiling": (_i, [_vp, _i, _i]),
    "dfm_get_tiling": (_i, [_vp, _ip, _ip, _ip, _ip, _ip]),
    "dfm_force_generic": (_i, [_vp, _i]),
    "dfm_debug_bits": (_i, [_vp, _i]),
    "dfm_cta_trace": (_i, [_vp, _i, _i, _vp]),
    "dfm_set_trace": (_i, [_vp, _i]),
    "dfm_get_trace": (_i, [_vp, _vp, _i]),
    "dfm_wiener": (_i, [_vp, _vp]),
    "dfm_bench_wiener": (_i, [_vp, _dp]),
    "dfm_step_spectrogram": (_i, [_i, _i, _i, _i, _vp, _vp, _vp]),
    "dfm_step_eta": (_i, [_i, _i, _i, _i, _vp, _vp, _d, _vp]),
    "dfm_step_decorrelate": (_i, [_i, _i, _i, _vp, _i, _i, _vp, _vp, _vp]),
    "dfm_step_ip_column": (_i, [_i, _i, _i, _vp, _vp, _i, _i, _vp, _i, _d]),
    "dfm_step_tv_weights": (_i, [_i, _i, _i, _i, _vp, _vp, _vp, _vp, _vp]),
    "dfm_step_update_t": (_i, [_i, _i, _i, _i, _vp, _vp, _vp, _vp, _d]),
    "dfm_step_update_v": (_i, [_i, _i, _i, _i, _vp, _vp, _vp, _vp, _d]),
    "dfm_step_update_lambda": (_i, [_i, _i, _i, _i, _vp, _vp, _vp, _vp, _d]),
    "dfm_step_power_term": (_i, [_i, _i, _i, _i, _vp, _vp, _vp, _d, _dp]),
    "dfm_step_logdet": (_i, [_i, _i, _vp, _dp]),
    "dfm_step_cost": (_i, [_i, _i, _i, _ip, _i, _i, _vp, _vp, _vp, _vp, _vp, _d, _dp]),
    "dfm_step_wiener": (_i, [_i, _i, _i, _ip, _i, _i, _vp, _vp, _vp, _vp, _vp, _d, _vp]),
    "dfm_derive_seed": (_u64, [_u64, C.c_char_p, _u64]),
    "dfm_random_init": (_i, [_i, _i, _i, _ip, _i, _i, _u64, _vp, _vp, _vp, _vp]),
    "dfm_random_observations": (_i, [_i, _i, _i, _u64, _vp]),
    "dfm_generate_mixture": (_i, [_i, _i, _i, _i, _i, _i, _u64, _vp]),
    "dfm_probe_fp64_tflops": (_d, [_i]),
    "dfm_l2_flush": (_i, [_i]),
}

DFM_OK = 0
DFM_ERR_SHAPE = -1
DFM_ERR_ARG = -2
DFM_ERR_SINGULAR = -3
DFM_ERR_CUDA = -4
DFM_ERR_NCCL = -5
DFM_ERR_UNSUPPORTED = -6
DFM_ERR_IO = -7
DFM_ERR_TOO_SHORT = -8


class ShapeMismatchError(ValueError):
    """fastmnmf::ShapeMismatch (include/fastmnmf/types.hpp:18-20)."""


class SingularDemixerError(RuntimeError):
    """fastmnmf::SingularDemixer (include/fastmnmf/types.hpp:24-26)."""


class NotPositiveDefiniteError(RuntimeError):
    """fastmnmf::NotPositiveDefinite (include/fastmnmf/types.hpp:21-23)."""


class SignalTooShortError(ValueError):
    """fastmnmf::SignalTooShort (include/fastmnmf/types.hpp:27-29)."""


class DeviceError(RuntimeError):
    """CUDA / NCCL failure (std::runtime_error in the reference's terms)."""


_lib = None


def load() -> C.CDLL:
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(
                f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
                "(the CUDA engine has no CPU fallback)")
        lib = C.CDLL(LIB_PATH)
        for name, (res, args) in _SIGS.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
    return _lib


def last_error() -> str:
    msg = load().dfm_last_error()
    return msg.decode() if msg else ""


def check(rc: int, what: str = "") -> int:
    if rc >= 0:
        return rc
    msg = f"{what}: {last_error()}" if what else last_error()
    if rc == DFM_ERR_SHAPE:
        raise ShapeMismatchError(msg)
    if rc == DFM_ERR_ARG:
        raise ValueError(msg)
    if rc == DFM_ERR_SINGULAR:
        raise SingularDemixerError(msg)
    if rc == DFM_ERR_UNSUPPORTED:
        raise NotImplementedError(msg)
    if rc == DFM_ERR_TOO_SHORT:
        raise SignalTooShortError(last_error())
    if rc == DFM_ERR_IO:  # std::runtime_error in the reference (io.cpp)
        raise RuntimeError(last_error())
    raise DeviceError(msg)


def exported_symbols():
    return list(_SIGS)
