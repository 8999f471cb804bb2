"""FMNM v2 model container, JSON debug dumps and CSV traces (mirror of
include/fastmnmf/io.hpp:12-64 / src/io.cpp).

The binary container is read and written by native host code behind the C
ABI (dfm_fmnm_*, csrc/dfm_io.cpp); this module converts between its payload
order (Eigen col-major, identical to dfm_set_model's buffers) and the math
shapes used everywhere else: T (N, F, K), V (N, K, T), Lambda (F, N, M),
W blocks (F, M_b, M_b).
"""
from __future__ import annotations

import ctypes as C
import json
from dataclasses import dataclass, field
from typing import List, Sequence, Tuple

import numpy as np

from . import _capi
from ._capi import check
from .fastmnmf import BlockLayout, FitReport, InitBundle, NmfModel, _c, _uc, _w_from_c, _w_to_c, kFloor

kModelFormatVersion = 2  # io.hpp:12 (v2 added layout and share mode)


@dataclass
class ModelConfig:
    """io.hpp:14-21."""
    n_sources: int = 0
    k_bases: int = 0
    iterations: int = 0
    floor: float = kFloor
    seed: int = 0
    sample_rate: float = 0.0
    window_len: int = 0
    hop_len: int = 0


@dataclass
class ModelDump:
    """io.hpp:23-30: one NmfModel when shared, one per block otherwise."""
    config: ModelConfig
    layout: BlockLayout
    shared: bool = True
    models: List[NmfModel] = field(default_factory=list)
    lam: np.ndarray = None               # (F, N, M)
    w: List[np.ndarray] = field(default_factory=list)  # [block] (F, M_b, M_b)

    def init_bundle(self) -> InitBundle:
        """The dumped state as an EM starting point (shared mode)."""
        return InitBundle(self.layout, self.models[0], [np.array(b) for b in self.w], np.array(self.lam))


def _header(dump: ModelDump) -> _capi.FmnmHeader:
    h = _capi.FmnmHeader()
    F = int(dump.lam.shape[0])
    n_src = int(dump.lam.shape[1]) if F else 0
    h.version = kModelFormatVersion
    h.num_bins = F
    h.num_frames = int(dump.models[0].V.shape[2]) if dump.models else 0
    h.channels = dump.layout.total
    h.n_sources = n_src
    h.k_bases = int(dump.config.k_bases)
    sizes = list(dump.layout.sizes)
    if len(sizes) > len(h.sizes):
        raise ValueError("save_model: too many blocks")
    h.n_blocks = len(sizes)
    for i, s in enumerate(sizes):
        h.sizes[i] = int(s)
    h.shared = 1 if dump.shared else 0
    h.floor = float(dump.config.floor)
    h.seed = int(dump.config.seed) & 0xFFFFFFFFFFFFFFFF
    h.sample_rate = float(dump.config.sample_rate)
    h.window_len = int(dump.config.window_len)
    h.hop_len = int(dump.config.hop_len)
    h.iterations = int(dump.config.iterations)
    h.n_models = len(dump.models)
    return h


def save_model(path: str, dump: ModelDump) -> None:
    """io.cpp:49-82."""
    lib = _capi.load()
    h = _header(dump)
    F, N, K = h.num_bins, h.n_sources, h.k_bases
    for m in dump.models:
        if m.T.shape != (N, F, K) or m.V.shape != (N, K, h.num_frames):
            raise ValueError("save_model: model shapes disagree with Lambda")
    T = np.concatenate([_c(m.T).reshape(-1) for m in dump.models]) if dump.models else np.zeros(0)
    V = np.concatenate([_c(m.V).reshape(-1) for m in dump.models]) if dump.models else np.zeros(0)
    lam = _c(dump.lam).reshape(-1)
    w = _w_to_c(dump.w).view(np.float64) if dump.w else np.zeros(0)
    # empty arrays still need valid pointers
    bufs = [np.ascontiguousarray(b) if b.size else np.zeros(1) for b in (T, V, lam, w)]
    check(lib.dfm_fmnm_write(path.encode(), C.byref(h), *[b.ctypes.data_as(C.c_void_p) for b in bufs]),
          "save_model")


def load_model(path: str) -> ModelDump:
    """io.cpp:84-135; raises RuntimeError with the reference's messages."""
    lib = _capi.load()
    h = _capi.FmnmHeader()
    check(lib.dfm_fmnm_read_header(path.encode(), C.byref(h)), "load_model")
    nt, nv, nl, nw = (C.c_size_t() for _ in range(4))
    lib.dfm_fmnm_sizes(C.byref(h), C.byref(nt), C.byref(nv), C.byref(nl), C.byref(nw))
    T = np.zeros(max(nt.value, 1))
    V = np.zeros(max(nv.value, 1))
    lam = np.zeros(max(nl.value, 1))
    w = np.zeros(max(nw.value, 1))
    check(lib.dfm_fmnm_read(path.encode(), C.byref(h), *[b.ctypes.data_as(C.c_void_p) for b in (T, V, lam, w)]),
          "load_model")
    F, J, M, N, K = h.num_bins, h.num_frames, h.channels, h.n_sources, h.k_bases
    sizes = [int(h.sizes[i]) for i in range(h.n_blocks)]
    cfg = ModelConfig(n_sources=N, k_bases=K, iterations=int(h.iterations), floor=float(h.floor),
                      seed=int(h.seed), sample_rate=float(h.sample_rate), window_len=int(h.window_len),
                      hop_len=int(h.hop_len))
    tper, vper = N * F * K, N * K * J
    models = [NmfModel(_uc(T[i * tper:(i + 1) * tper].reshape(N, K, F)),
                       _uc(V[i * vper:(i + 1) * vper].reshape(N, J, K))) for i in range(h.n_models)]
    lam_m = _uc(lam[:nl.value].reshape(F, M, N))
    wb = _w_from_c(w[:nw.value].view(np.complex128), F, sizes)
    return ModelDump(cfg, BlockLayout(sizes), bool(h.shared), models, lam_m, wb)


def _real_json(m: np.ndarray):
    return [[float(v) for v in row] for row in np.asarray(m)]


def _cplx_json(m: np.ndarray):
    return [[[float(v.real), float(v.imag)] for v in row] for row in np.asarray(m)]


def dump_model_json(path: str, dump: ModelDump) -> None:
    """io.cpp:163-191: the same content as nested JSON arrays (row-major
    matrices: T_n is F x K, V_n is K x T, Lambda per bin N x M, W per bin)."""
    c = dump.config
    j = {"format_version": kModelFormatVersion,
         "config": {"n_sources": c.n_sources, "k_bases": c.k_bases, "iterations": c.iterations,
                    "floor": c.floor, "seed": c.seed, "sample_rate": c.sample_rate,
                    "window_len": c.window_len, "hop_len": c.hop_len},
         "partition": list(dump.layout.sizes), "share_spectrograms": bool(dump.shared),
         "models": [{"T": [_real_json(t) for t in m.T], "V": [_real_json(v) for v in m.V]} for m in dump.models],
         "lambda": [_real_json(l) for l in dump.lam],
         "w": [[_cplx_json(wi) for wi in wb] for wb in dump.w]}
    with open(path, "w") as fh:
        json.dump(j, fh)


def dump_init_json(path: str, init: InitBundle, mask: np.ndarray = None, h0: np.ndarray = None) -> None:
    """io.cpp:193-210: audit dump of an initialisation bundle (mask (F, T, N)
    and h0 (F, T, N) when the caller has them)."""
    j = {"partition": list(init.layout.sizes), "num_sources": init.nmf.num_sources(), "k_bases": init.nmf.K}
    if mask is not None:
        j["mask"] = [_real_json(b) for b in mask]
    if h0 is not None:
        j["h0"] = [_real_json(b) for b in h0]
    j["lambda0"] = [_real_json(l) for l in init.lambda0]
    j["w0"] = [[_cplx_json(wi) for wi in wb] for wb in init.w0]
    j["t0"] = [_real_json(t) for t in init.nmf.T]
    j["v0"] = [_real_json(v) for v in init.nmf.V]
    with open(path, "w") as fh:
        json.dump(j, fh)


def _g17(v: float) -> str:
    return f"{v:.17g}"


def write_trace_csv(path: str, report: FitReport) -> None:
    """io.cpp:212-221: iteration, cost, wall_seconds (row 0 = initial cost)."""
    with open(path, "w") as fh:
        fh.write("iteration,cost,wall_seconds\n")
        for it, cost in enumerate(report.cost_trace):
            wall = 0.0 if it == 0 else float(report.wall_seconds[it - 1])
            fh.write(f"{it},{_g17(float(cost))},{_g17(wall)}\n")


def write_eval_trace_csv(path: str, rows: Sequence[Tuple[int, float, float, float]]) -> None:
    """io.cpp:223-231: iteration, cumulative_seconds, cost, mean_sdr_improvement."""
    with open(path, "w") as fh:
        fh.write("iteration,cumulative_seconds,cost,mean_sdr_improvement\n")
        for it, secs, cost, sdr in rows:
            fh.write(f"{int(it)},{_g17(secs)},{_g17(cost)},{_g17(sdr)}\n")
