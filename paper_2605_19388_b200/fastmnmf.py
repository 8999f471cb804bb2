"""Host-side mirror of the reference's public FastMNMF API on the B200 engine.

Same names, argument meaning and error behaviour as
/root/reference/proj/include/fastmnmf/{types,model,init,fastmnmf,dist,wiener}.hpp;
every computation runs in the sm_100a kernels of libdfm_b200.so through the
C ABI (include/dfm_b200.h).  There is no CPU fallback.

Array conventions ("math shapes" of the reference containers):
  x            (F, T, M) complex128   x[i, j, m] = ObsTensor::bins[i](m, j)
  NmfModel.T   (N, F, K)              T[n][i, k]  (NmfModel::T[n] is I x K)
  NmfModel.V   (N, K, T)              V[n][k, j]  (NmfModel::V[n] is K x J)
  Lambda       (F, N, M)              Lambda[i][n, m]
  W            (F, M, M) complex      SpatialModel::W[i]
  W blocks     list of (F, mb, mb)    BlockSpatialModel::W[l][i]
  eta, |y|^2   (F, T, M)              eta[i][j, m]
  h            (F, T, N)              spectrogram h[i][j, n]
The C ABI wants the reference's Eigen column-major storage, i.e. these
arrays with their last two axes swapped (``_c`` below).
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from typing import Callable, List, Optional, Sequence

import numpy as np

from . import _capi
from ._capi import (DeviceError, NotPositiveDefiniteError, ShapeMismatchError,  # noqa: F401
                    SingularDemixerError, check)

kFloor = 1e-6  # types.hpp:16


# ------------------------------------------------------------------ helpers
def _c(a: np.ndarray, dtype=np.float64) -> np.ndarray:
    return np.ascontiguousarray(np.swapaxes(np.asarray(a, dtype=dtype), -1, -2))


def _uc(a: np.ndarray) -> np.ndarray:
    return np.ascontiguousarray(np.swapaxes(a, -1, -2))


def _ptr(a: np.ndarray):
    assert a.flags.c_contiguous
    return a.ctypes.data_as(C.c_void_p)


def _ints(v: Sequence[int]):
    return (C.c_int * len(v))(*[int(s) for s in v])


def _obs(x) -> np.ndarray:
    x = np.ascontiguousarray(x, dtype=np.complex128)
    if x.ndim != 3:
        raise ShapeMismatchError("expected a complex array of shape (I, J, M)")
    return x


# --------------------------------------------------------------- core types
class BlockLayout:
    """Contiguous partition of the channel axis (types.hpp:63-88)."""

    def __init__(self, sizes: Sequence[int]):
        self.sizes = [int(s) for s in sizes]
        self.offsets = []
        self.total = 0
        for s in self.sizes:
            if s <= 0:
                raise ValueError("BlockLayout: block sizes must be positive")
            self.offsets.append(self.total)
            self.total += s

    @staticmethod
    def full(channels: int) -> "BlockLayout":
        return BlockLayout([channels])

    def num_blocks(self) -> int:
        return len(self.sizes)

    def global_index(self, block: int, mu: int) -> int:
        if block < 0 or block >= len(self.sizes) or mu < 0 or mu >= self.sizes[block]:
            raise IndexError("BlockLayout: (block, mu) out of range")
        return self.offsets[block] + mu

    def __eq__(self, other):
        return isinstance(other, BlockLayout) and self.sizes == other.sizes

    def __repr__(self):
        return f"BlockLayout({self.sizes})"


@dataclass
class NmfModel:
    """h_ijn = sum_k t_ikn v_kjn (model.hpp:14-26)."""
    T: np.ndarray  # (N, F, K)
    V: np.ndarray  # (N, K, T)

    @property
    def K(self) -> int:
        return int(self.T.shape[2])

    def num_sources(self) -> int:
        return int(self.T.shape[0])

    def num_bins(self) -> int:
        return int(self.T.shape[1])

    def num_frames(self) -> int:
        return int(self.V.shape[2])

    def copy(self) -> "NmfModel":
        return NmfModel(self.T.copy(), self.V.copy())


@dataclass
class SpatialModel:
    """Full-array spatial model (model.hpp:30-35)."""
    W: np.ndarray       # (F, M, M) complex
    Lambda: np.ndarray  # (F, N, M)

    def num_channels(self) -> int:
        return int(self.W.shape[1])


@dataclass
class BlockSpatialModel:
    """Block-diagonal spatial model (model.hpp:38-47)."""
    layout: BlockLayout
    W: List[np.ndarray]  # [block] (F, mb, mb) complex
    Lambda: np.ndarray   # (F, N, M)

    def assembled_w(self, bin_: int) -> np.ndarray:
        M = self.layout.total
        out = np.zeros((M, M), dtype=np.complex128)
        for l, o in enumerate(self.layout.offsets):
            mb = self.layout.sizes[l]
            out[o:o + mb, o:o + mb] = self.W[l][bin_]
        return out

    def block_model(self, block: int) -> SpatialModel:
        o, mb = self.layout.offsets[block], self.layout.sizes[block]
        return SpatialModel(self.W[block], np.ascontiguousarray(self.Lambda[:, :, o:o + mb]))


@dataclass
class FitReport:
    """model.hpp:69-81."""
    cost_trace: np.ndarray
    wall_seconds: np.ndarray
    iterations: int = 0
    stages: dict = field(default_factory=lambda: dict(w_update=0.0, mm_update=0.0, eta=0.0,
                                                      decorrelate=0.0))
    fallbacks: int = 0
    ops: dict = field(default_factory=lambda: dict(w_update=0.0, mm_update=0.0))  # OpCounts, model.hpp:60-67

    def total_seconds(self) -> float:
        return float(np.sum(self.wall_seconds))


@dataclass
class FitSnapshot:
    """model.hpp:84-93 (read-only view handed to on_eval)."""
    iteration: int
    cost: float
    elapsed_seconds: float
    layout: BlockLayout
    models: List[NmfModel]
    w_blocks: List[np.ndarray]
    Lambda: np.ndarray
    shared: bool = True


@dataclass
class FitOptions:
    """model.hpp:95-99."""
    floor: float = kFloor
    eval_every: int = 0
    on_eval: Optional[Callable[[FitSnapshot], None]] = None


@dataclass
class InitBundle:
    """init.hpp:69-77: the EM starting point (layout, nmf, w0, lambda0) plus,
    from the initialisation pipeline (paper_2605_19388_b200.init), the ML
    spectrograms h0 and the reference subarray's aligned soft mask."""
    layout: BlockLayout
    nmf: NmfModel
    w0: List[np.ndarray]   # [block] (F, mb, mb)
    lambda0: np.ndarray    # (F, N, M)
    h0: Optional[np.ndarray] = None    # (F, T, N)
    mask: Optional[np.ndarray] = None  # (F, T, N)


@dataclass
class FullFit:
    nmf: NmfModel
    spatial: SpatialModel
    report: FitReport


@dataclass
class DistFit:
    models: List[NmfModel]
    spatial: BlockSpatialModel
    report: FitReport
    shared: bool = True


@dataclass
class SourceImages:
    """wiener.hpp:14-19; images has shape (N, F, T, M)."""
    images: np.ndarray
    reference_mic: int = 0

    def num_sources(self) -> int:
        return int(self.images.shape[0])


# ------------------------------------------------------------ initialisation
def random_init(num_bins: int, num_frames: int, layout: BlockLayout, num_sources: int, k: int,
                seed: int) -> InitBundle:
    """init.cpp:496-521, bit-exact RNG streams (host runtime of libdfm_b200)."""
    lib = _capi.load()
    F, T, N, K, M = num_bins, num_frames, num_sources, k, layout.total
    Tc = np.empty((N, K, F)); Vc = np.empty((N, T, K)); lc = np.empty((F, M, N))
    wc = np.empty(sum(F * s * s for s in layout.sizes), dtype=np.complex128)
    check(lib.dfm_random_init(F, T, layout.num_blocks(), _ints(layout.sizes), N, K, seed,
                              _ptr(Tc), _ptr(Vc), _ptr(lc), _ptr(wc)), "random_init")
    return InitBundle(layout, NmfModel(_uc(Tc), _uc(Vc)), _w_from_c(wc, F, layout.sizes), _uc(lc))


def random_observations(num_bins: int, num_frames: int, num_channels: int, seed: int) -> np.ndarray:
    """bench.cpp:10-20."""
    x = np.empty((num_bins, num_frames, num_channels), dtype=np.complex128)
    check(_capi.load().dfm_random_observations(num_bins, num_frames, num_channels, seed, _ptr(x)))
    return x


def generate_mixture(kind: int, F: int, T: int, M: int, N: int, K: int, seed: int) -> np.ndarray:
    """Synthetic STFT-domain mixture of the BASELINE.json configs."""
    x = np.empty((F, T, M), dtype=np.complex128)
    check(_capi.load().dfm_generate_mixture(kind, F, T, M, N, K, seed, _ptr(x)))
    return x


def slice_init(init: InitBundle, block: int) -> InitBundle:
    """init.cpp:474-494."""
    o, mb = init.layout.offsets[block], init.layout.sizes[block]
    return InitBundle(BlockLayout.full(mb), init.nmf.copy(), [init.w0[block].copy()],
                      np.ascontiguousarray(init.lambda0[:, :, o:o + mb]))


def extract_block(x: np.ndarray, layout: BlockLayout, block: int) -> np.ndarray:
    """types.hpp:91-99."""
    if layout.total != x.shape[2]:
        raise ShapeMismatchError("extract_block: layout does not match channel count")
    o, mb = layout.offsets[block], layout.sizes[block]
    return np.ascontiguousarray(x[:, :, o:o + mb])


def _w_to_c(w_blocks: Sequence[np.ndarray]) -> np.ndarray:
    return np.concatenate([_c(w, np.complex128).reshape(-1) for w in w_blocks])


def _w_from_c(buf: np.ndarray, F: int, sizes: Sequence[int]) -> List[np.ndarray]:
    out, o = [], 0
    for mb in sizes:
        n = F * mb * mb
        out.append(_uc(buf[o:o + n].reshape(F, mb, mb)))
        o += n
    return out


# ------------------------------------------------------------ per-update API
def decorrelate(x: np.ndarray, w: np.ndarray) -> np.ndarray:
    """y_ij = W_i^H x_ij (fastmnmf.cpp:43-54); returns (F, T, M) complex."""
    x = _obs(x)
    F, T, M = x.shape
    w = np.asarray(w, dtype=np.complex128)
    if w.shape != (F, M, M):
        raise ShapeMismatchError("decorrelate: demixer size mismatch")
    y = np.zeros_like(x)
    check(_capi.load().dfm_step_decorrelate(F, T, M, _ptr(x), 0, M, _ptr(_c(w, np.complex128)),
                                            _ptr(y), None), "decorrelate")
    return y


def decorrelate_blocks(x: np.ndarray, layout: BlockLayout, w_blocks: Sequence[np.ndarray]):
    """Block-diagonal decorrelation (dist.cpp:9-18); returns (y, |y|^2)."""
    x = _obs(x)
    F, T, M = x.shape
    y = np.zeros_like(x)
    P = np.zeros((F, M, T))
    for l, (o, mb) in enumerate(zip(layout.offsets, layout.sizes)):
        check(_capi.load().dfm_step_decorrelate(F, T, M, _ptr(x), o, mb,
                                                _ptr(_c(w_blocks[l], np.complex128)), _ptr(y), _ptr(P)))
    return y, _uc(P)


def power_of(y: np.ndarray) -> np.ndarray:
    """|y_ijm|^2 (fastmnmf.cpp:56-61)."""
    return np.abs(y) ** 2


def build_spectrogram(model: NmfModel) -> np.ndarray:
    """fastmnmf.cpp:63-65 -> (F, T, N)."""
    N, F, K = model.T.shape
    T = model.V.shape[2]
    h = np.empty((F, N, T))
    check(_capi.load().dfm_step_spectrogram(F, T, N, K, _ptr(_c(model.T)), _ptr(_c(model.V)), _ptr(h)))
    return _uc(h)


def _eta_from(h: np.ndarray, lam: np.ndarray, floor: float) -> np.ndarray:
    F, T, N = h.shape
    M = lam.shape[2]
    eta = np.empty((F, M, T))
    check(_capi.load().dfm_step_eta(F, T, N, M, _ptr(_c(h)), _ptr(_c(lam)), floor, _ptr(eta)))
    return _uc(eta)


def compute_eta(model: NmfModel, lam: np.ndarray, floor: float = kFloor) -> np.ndarray:
    """fastmnmf.cpp:67-73 -> (F, T, M)."""
    return _eta_from(build_spectrogram(model), lam, floor)


def _cost(x, layout: BlockLayout, model: NmfModel, w_blocks, lam, floor) -> float:
    x = _obs(x)
    F, T, M = x.shape
    if layout.total != M:
        raise ShapeMismatchError("cost_dist: layout/channel mismatch")
    N, _, K = model.T.shape
    out = C.c_double()
    check(_capi.load().dfm_step_cost(F, T, layout.num_blocks(), _ints(layout.sizes), N, K, _ptr(x),
                                     _ptr(_c(model.T)), _ptr(_c(model.V)), _ptr(_c(lam)),
                                     _ptr(_w_to_c(w_blocks)), floor, C.byref(out)), "cost")
    return out.value


def cost_full(x: np.ndarray, model: NmfModel, spatial: SpatialModel, floor: float = kFloor) -> float:
    """fastmnmf.cpp:75-84; raises SingularDemixerError on a singular W."""
    return _cost(x, BlockLayout.full(_obs(x).shape[2]), model, [spatial.W], spatial.Lambda, floor)


def cost_dist(x: np.ndarray, models, spatial: BlockSpatialModel, floor: float = kFloor) -> float:
    """dist.cpp:20-43: shared model, or one NmfModel per block (independent)."""
    if isinstance(models, NmfModel):
        models = [models]
    if len(models) == 1:
        return _cost(x, spatial.layout, models[0], spatial.W, spatial.Lambda, floor)
    if len(models) != spatial.layout.num_blocks():
        raise ShapeMismatchError("cost_dist: one model per subarray expected")
    return sum(cost_full(extract_block(x, spatial.layout, l), models[l], spatial.block_model(l), floor)
               for l in range(spatial.layout.num_blocks()))


def ip_update_block(x, eta, layout: BlockLayout, block: int, w_block: np.ndarray, mu: int,
                    floor: float = kFloor) -> int:
    """dist.cpp:45-49 / engine.cpp:30-58: w_block (F, mb, mb) updated in place.
    Returns the number of bins that took the pinv fallback."""
    x = _obs(x)
    F, T, M = x.shape
    if w_block.dtype != np.complex128:
        raise TypeError("w_block must be complex128")
    off, mb = layout.offsets[block], layout.sizes[block]
    wc = _c(w_block, np.complex128)
    fb = check(_capi.load().dfm_step_ip_column(F, T, M, _ptr(x), _ptr(_c(eta)), off, mb, _ptr(wc), mu,
                                               floor), "ip_update_block")
    w_block[...] = _uc(wc)
    return fb


def ip_update_w(x, eta, w: np.ndarray, m: int, floor: float = kFloor) -> int:
    """fastmnmf.cpp:86-90: column m of every W_i (full array)."""
    return ip_update_block(x, eta, BlockLayout.full(_obs(x).shape[2]), 0, w, m, floor)


def _tv_weights(lam, pow_y, eta):
    F, N, M = lam.shape
    T = pow_y.shape[1]
    a = np.empty((N, T, F)); b = np.empty((N, T, F))
    check(_capi.load().dfm_step_tv_weights(F, T, N, M, _ptr(_c(lam)), _ptr(_c(pow_y)), _ptr(_c(eta)),
                                           _ptr(a), _ptr(b)))
    return a, b  # C layout (N, T, F)


def mm_update_t(model: NmfModel, lam, pow_y, eta: np.ndarray, floor: float = kFloor) -> None:
    """fastmnmf.cpp:92-99: T update, then eta refreshed in place."""
    N, F, K = model.T.shape
    T = model.V.shape[2]
    a, b = _tv_weights(lam, pow_y, eta)
    Tc = _c(model.T)
    check(_capi.load().dfm_step_update_t(F, T, N, K, _ptr(Tc), _ptr(_c(model.V)), _ptr(a), _ptr(b), floor))
    model.T = _uc(Tc)
    eta[...] = compute_eta(model, lam, floor)


def mm_update_v(model: NmfModel, lam, pow_y, eta: np.ndarray, floor: float = kFloor) -> None:
    """fastmnmf.cpp:101-108: V update (cross-bin reduction), eta refreshed."""
    N, F, K = model.T.shape
    T = model.V.shape[2]
    a, b = _tv_weights(lam, pow_y, eta)
    Vc = _c(model.V)
    check(_capi.load().dfm_step_update_v(F, T, N, K, _ptr(_c(model.T)), _ptr(Vc), _ptr(a), _ptr(b), floor))
    model.V = _uc(Vc)
    eta[...] = compute_eta(model, lam, floor)


def mm_update_lambda(model: NmfModel, lam: np.ndarray, pow_y, eta: np.ndarray,
                     floor: float = kFloor) -> None:
    """fastmnmf.cpp:110-116: Lambda update in place, eta refreshed."""
    F, N, M = lam.shape
    h = build_spectrogram(model)
    T = h.shape[1]
    lc = _c(lam)
    check(_capi.load().dfm_step_update_lambda(F, T, N, M, _ptr(lc), _ptr(_c(h)), _ptr(_c(pow_y)),
                                              _ptr(_c(eta)), floor))
    lam[...] = _uc(lc)
    eta[...] = _eta_from(h, lam, floor)


# ------------------------------------------------------------------- engine
class Engine:
    """Owns one device context (dfm_ctx): the resident state of
    detail::run_engine (engine.cpp:167-272) for bins [f_begin, f_end)."""

    def __init__(self, num_bins: int, num_frames: int, layout: BlockLayout, num_sources: int, k: int,
                 floor: float = kFloor, device: int = 0, f_begin: int = 0, f_end: Optional[int] = None):
        self.lib = _capi.load()
        self.F, self.T, self.layout, self.N, self.K = num_bins, num_frames, layout, num_sources, k
        self.floor = floor
        self.f_begin = f_begin
        self.f_end = num_bins if f_end is None else f_end
        self.ctx = self.lib.dfm_create(num_bins, num_frames, layout.num_blocks(), _ints(layout.sizes),
                                       num_sources, k, floor, device, self.f_begin, self.f_end)
        if not self.ctx:
            msg = _capi.last_error()
            if "floor" in msg or "negative" in msg:
                raise ValueError(msg)
            raise ShapeMismatchError(msg) if ("layout" in msg or "range" in msg or "dimension" in msg
                                              or "size" in msg) else DeviceError(msg)

    def close(self):
        if getattr(self, "ctx", None):
            self.lib.dfm_destroy(self.ctx)
            self.ctx = None

    def __del__(self):
        self.close()

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    @property
    def local_bins(self) -> int:
        return self.f_end - self.f_begin

    def set_obs(self, x_local: np.ndarray) -> None:
        x_local = _obs(x_local)
        if x_local.shape != (self.local_bins, self.T, self.layout.total):
            raise ShapeMismatchError("run_engine: observations do not match the engine shape")
        check(self.lib.dfm_set_obs(self.ctx, _ptr(x_local)), "set_obs")

    def set_model(self, nmf: NmfModel, w_blocks: Sequence[np.ndarray], lam: np.ndarray) -> None:
        N, F, K = nmf.T.shape
        if (N, F, K) != (self.N, self.F, self.K) or nmf.V.shape != (self.N, self.K, self.T):
            raise ShapeMismatchError("run_engine: init factor shapes do not match the observations")
        if len(w_blocks) != self.layout.num_blocks():
            raise ShapeMismatchError("run_engine: init has wrong number of demixer blocks")
        if lam.shape != (self.F, self.N, self.layout.total):
            raise ShapeMismatchError("run_engine: Lambda shape mismatch")
        # the context's device layouts (dfm_set_model_native): T (F, N, K),
        # V (N, K, T) and Lambda (F, N, M) are the math shapes up to one
        # transpose of T; W per bin is the blocks' col-major matrices
        f0, f1 = self.f_begin, self.f_end
        Tn = np.ascontiguousarray(np.asarray(nmf.T, dtype=np.float64)[:, f0:f1].transpose(1, 0, 2))
        Vn = np.ascontiguousarray(nmf.V, dtype=np.float64)
        ln = np.ascontiguousarray(np.asarray(lam, dtype=np.float64)[f0:f1])
        wn = np.ascontiguousarray(np.concatenate(
            [np.asarray(w, dtype=np.complex128)[f0:f1].transpose(0, 2, 1).reshape(f1 - f0, -1) for w in w_blocks],
            axis=1))
        check(self.lib.dfm_set_model_native(self.ctx, _ptr(Tn), _ptr(Vn), _ptr(ln), _ptr(wn)), "set_model")

    def get_model(self):
        """(NmfModel, W blocks, Lambda) in global shapes; a frequency shard
        fills its own bins [f_begin, f_end) (the others are zero)."""
        Fl, f0, f1 = self.local_bins, self.f_begin, self.f_end
        Tn = np.empty((Fl, self.N, self.K)); Vn = np.empty((self.N, self.K, self.T))
        ln = np.empty((Fl, self.N, self.layout.total))
        wn = np.empty((Fl, sum(s * s for s in self.layout.sizes)), dtype=np.complex128)
        check(self.lib.dfm_get_model_native(self.ctx, _ptr(Tn), _ptr(Vn), _ptr(ln), _ptr(wn)), "get_model")
        full = f0 == 0 and f1 == self.F
        T = np.zeros((self.N, self.F, self.K))
        T[:, f0:f1] = Tn.transpose(1, 0, 2)
        lam = ln if full else np.zeros((self.F, self.N, self.layout.total))
        if not full:
            lam[f0:f1] = ln
        wb, o = [], 0
        for mb in self.layout.sizes:
            blk = wn[:, o:o + mb * mb].reshape(Fl, mb, mb).transpose(0, 2, 1)
            if full:
                wb.append(np.ascontiguousarray(blk))
            else:
                g = np.zeros((self.F, mb, mb), dtype=np.complex128)
                g[f0:f1] = blk
                wb.append(g)
            o += mb * mb
        return NmfModel(T, Vn), wb, lam

    def comm_init(self, unique_id: bytes, nranks: int, rank: int) -> None:
        buf = C.create_string_buffer(bytes(unique_id), 128)
        check(self.lib.dfm_comm_init(self.ctx, buf, nranks, rank), "comm_init")

    def fit(self, iters: int):
        """Returns (cost_trace, wall_seconds, fallbacks)."""
        cost = np.zeros(iters + 1)
        wall = np.zeros(max(iters, 1))
        stages = np.zeros(4)
        fb = check(self.lib.dfm_fit(self.ctx, iters, _ptr(cost), _ptr(wall), _ptr(stages)), "fit")
        return cost, wall[:iters], stages, fb

    def wiener(self) -> np.ndarray:
        img = np.empty((self.N, self.local_bins, self.T, self.layout.total), dtype=np.complex128)
        check(self.lib.dfm_wiener(self.ctx, _ptr(img)), "wiener")
        return img

    def set_tiling(self, frame_tile: int = 0, pd_frames: int = 0) -> None:
        """Frame tile (threads per CTA) of the per-bin kernel and of k_pd; 0 = heuristic."""
        check(self.lib.dfm_set_tiling(self.ctx, frame_tile, pd_frames), "set_tiling")

    def tiling(self) -> dict:
        v = [C.c_int() for _ in range(5)]
        check(self.lib.dfm_get_tiling(self.ctx, *[C.byref(a) for a in v]))
        return dict(zip(("frame_tile", "pd_frames", "ctas", "threads", "smem_bytes"), [a.value for a in v]))

    def launches(self) -> int:
        return int(self.lib.dfm_launch_count(self.ctx))


def fit_many(engines: Sequence["Engine"], iters: int):
    """Fits independent mixtures together (BASELINE config 4): every engine
    (one mixture each, same device, observations and model already set) runs
    `iters` EM sweeps with their launches interleaved so their kernels overlap.
    Returns (cost_traces (n, iters+1), device seconds of the batch, fallbacks)."""
    engines = list(engines)
    if not engines:
        raise ValueError("fit_many: no engines")
    if iters < 0:
        raise ValueError("run_engine: negative iteration count")
    arr = (C.c_void_p * len(engines))(*[e.ctx for e in engines])
    cost = np.zeros((len(engines), iters + 1))
    secs = C.c_double(0.0)
    lib = engines[0].lib
    fb = check(lib.dfm_fit_many(arr, len(engines), iters, _ptr(cost), C.byref(secs)), "fit_many")
    return cost, secs.value, fb


def op_counts(F: int, T: int, sizes: Sequence[int], N: int, M: int, K: int, iters: int) -> dict:
    """The reference's analytic operation counters (OpCounts, engine.cpp:55-57,
    110-112, 121, 131, 146) for `iters` EM iterations:
      w_update  += F (T mb^2 + mb^3) per IP column, mb columns per block;
      mm_update += 2 F T N M per T/V weight build (two per iteration),
                   2 F K T per source for the T and for the V update,
                   2 N M T per bin for the Lambda update."""
    w = sum(mb * F * (float(T) * mb * mb + float(mb) ** 3) for mb in sizes)
    mm = 2 * (2.0 * F * T * N * M) + N * (2.0 * F * K * T) * 2 + F * (2.0 * N * M * T)
    return dict(w_update=iters * w, mm_update=iters * mm)


def _run_engine(x, layout: BlockLayout, init: InitBundle, iters: int, options: FitOptions):
    """detail::run_engine (engine.cpp:167-272) on the device."""
    x = _obs(x)
    F, T, M = x.shape
    if layout.total != M:
        raise ShapeMismatchError("run_engine: layout/channel mismatch")
    if len(init.w0) != layout.num_blocks():
        raise ShapeMismatchError("run_engine: init has wrong number of demixer blocks")
    if init.nmf.num_bins() != F or init.nmf.num_frames() != T:
        raise ShapeMismatchError("run_engine: init factor shapes do not match the observations")
    if iters < 0:
        raise ValueError("run_engine: negative iteration count")
    if not options.floor > 0:
        raise ValueError("run_engine: floor must be positive")
    eng = Engine(F, T, layout, init.nmf.num_sources(), init.nmf.K, options.floor)
    try:
        eng.set_obs(x)
        eng.set_model(init.nmf, init.w0, init.lambda0)
        every = options.eval_every if (options.eval_every > 0 and options.on_eval) else iters
        costs, walls, fb, done = [], [], 0, 0
        stages = np.zeros(4)
        while True:
            chunk = min(every, iters - done) if iters > 0 else 0
            c, w, st, f = eng.fit(chunk)
            costs.append(c if done == 0 else c[1:])
            walls.append(w)
            stages += st
            fb += f
            done += chunk
            if options.eval_every > 0 and options.on_eval and chunk > 0 and done % options.eval_every == 0:
                nmf, wb, lam = eng.get_model()
                options.on_eval(FitSnapshot(done, float(c[-1]), float(np.sum(np.concatenate(walls))),
                                            layout, [nmf], wb, lam, True))
            if done >= iters:
                break
        nmf, wb, lam = eng.get_model()
    finally:
        eng.close()
    report = FitReport(np.concatenate(costs), np.concatenate(walls) if walls else np.zeros(0), iters,
                       dict(w_update=stages[0], mm_update=stages[1], eta=stages[2], decorrelate=stages[3]),
                       fb, op_counts(F, T, layout.sizes, init.nmf.num_sources(), M, init.nmf.K, iters))
    return nmf, wb, lam, report


def fit_full(x, init: InitBundle, iters: int, options: Optional[FitOptions] = None) -> FullFit:
    """fastmnmf.cpp:118-128."""
    options = options or FitOptions()
    layout = BlockLayout.full(_obs(x).shape[2])
    nmf, wb, lam, rep = _run_engine(x, layout, init, iters, options)
    return FullFit(nmf, SpatialModel(wb[0], lam), rep)


def fit_single(x_subarray, init: InitBundle, iters: int, options: Optional[FitOptions] = None) -> FullFit:
    """fastmnmf.cpp:130-133."""
    return fit_full(x_subarray, init, iters, options)


def fit_distributed(x, layout: BlockLayout, init: InitBundle, iters: int, share_spectrograms: bool = True,
                    options: Optional[FitOptions] = None) -> DistFit:
    """dist.cpp:51-94: shared spectrograms run one engine over the block
    layout; independent mode runs fit_single per block on slice_init."""
    options = options or FitOptions()
    x = _obs(x)
    if layout.total != x.shape[2]:
        raise ShapeMismatchError("fit_distributed: layout/channel mismatch")
    if share_spectrograms:
        nmf, wb, lam, rep = _run_engine(x, layout, init, iters, options)
        return DistFit([nmf], BlockSpatialModel(layout, wb, lam), rep, True)
    F = x.shape[0]
    models, wbs = [], []
    lam = np.zeros((F, init.nmf.num_sources(), layout.total))
    cost = np.zeros(iters + 1)
    wall = np.zeros(iters)
    stages = dict(w_update=0.0, mm_update=0.0, eta=0.0, decorrelate=0.0)
    ops = dict(w_update=0.0, mm_update=0.0)
    fb = 0
    for l in range(layout.num_blocks()):
        fit = fit_single(extract_block(x, layout, l), slice_init(init, l), iters, options)
        models.append(fit.nmf)
        wbs.append(fit.spatial.W)
        o, mb = layout.offsets[l], layout.sizes[l]
        lam[:, :, o:o + mb] = fit.spatial.Lambda
        cost += fit.report.cost_trace
        wall += fit.report.wall_seconds
        for k in stages:
            stages[k] += fit.report.stages[k]
        for k in ops:  # dist.cpp:91
            ops[k] += fit.report.ops[k]
        fb += fit.report.fallbacks
    return DistFit(models, BlockSpatialModel(layout, wbs, lam), FitReport(cost, wall, iters, stages, fb, ops),
                   False)


# ------------------------------------------------------------------- wiener
def _wiener(x, layout: BlockLayout, model: NmfModel, w_blocks, lam, floor) -> np.ndarray:
    x = _obs(x)
    F, T, M = x.shape
    N, _, K = model.T.shape
    img = np.empty((N, F, T, M), dtype=np.complex128)
    check(_capi.load().dfm_step_wiener(F, T, layout.num_blocks(), _ints(layout.sizes), N, K, _ptr(x),
                                       _ptr(_c(model.T)), _ptr(_c(model.V)), _ptr(_c(lam)),
                                       _ptr(_w_to_c(w_blocks)), floor, _ptr(img)), "wiener")
    return img


def wiener_full(x, model: NmfModel, spatial: SpatialModel, floor: float = kFloor) -> SourceImages:
    """wiener.cpp:38-48."""
    x = _obs(x)
    if spatial.W.shape[0] != x.shape[0]:
        raise ShapeMismatchError("wiener_full: bin count mismatch")
    return SourceImages(_wiener(x, BlockLayout.full(x.shape[2]), model, [spatial.W], spatial.Lambda, floor))


def wiener_block(x, models, spatial: BlockSpatialModel, floor: float = kFloor) -> SourceImages:
    """wiener.cpp:50-69 (shared model or one model per block)."""
    x = _obs(x)
    if spatial.layout.total != x.shape[2]:
        raise ShapeMismatchError("wiener_block: layout/channel mismatch")
    if isinstance(models, NmfModel):
        models = [models]
    if len(models) == 1:
        return SourceImages(_wiener(x, spatial.layout, models[0], spatial.W, spatial.Lambda, floor))
    if len(models) != spatial.layout.num_blocks():
        raise ShapeMismatchError("wiener_block: one model per subarray expected")
    out = np.zeros((models[0].num_sources(),) + x.shape, dtype=np.complex128)
    for l in range(spatial.layout.num_blocks()):
        o, mb = spatial.layout.offsets[l], spatial.layout.sizes[l]
        sub = spatial.block_model(l)
        out[:, :, :, o:o + mb] = _wiener(extract_block(x, spatial.layout, l), BlockLayout.full(mb),
                                         models[l], [sub.W], sub.Lambda, floor)
    return SourceImages(out)


# ------------------------------------------------------------ tracing harness
@dataclass
class TraceRow:
    """sdr.hpp:50-55: one periodic evaluation of a running fit."""
    iteration: int = 0
    seconds: float = 0.0  # cumulative estimation time, evaluation excluded
    cost: float = 0.0
    mean_sdr_improvement: float = 0.0


@dataclass
class TraceResult:
    """sdr.hpp:57-60."""
    report: FitReport
    rows: List[TraceRow] = field(default_factory=list)


def trace_run(run_fit: Callable[[FitOptions], FitReport], score: Optional[Callable[[FitSnapshot], float]],
              eval_every: int, floor: float = kFloor) -> TraceResult:
    """sdr.cpp:158-177: runs an estimator with periodic snapshot scoring.

    ``run_fit`` maps FitOptions to a FitReport (e.g. ``lambda o:
    fit_distributed(x, layout, init, iters, options=o).report``); ``score`` maps
    a FitSnapshot to a number (the reference's SDR improvement, or any other
    figure of merit).  The snapshots are taken between graph-replayed chunks of
    ``eval_every`` iterations, so the device clock that fills ``seconds`` never
    runs while ``score`` does (the reference pauses its estimator clock).
    """
    out = TraceResult(report=FitReport(np.zeros(0), np.zeros(0)))
    options = FitOptions(floor=floor, eval_every=eval_every)
    if eval_every > 0 and score is not None:
        def on_eval(snap: FitSnapshot) -> None:
            out.rows.append(TraceRow(snap.iteration, snap.elapsed_seconds, snap.cost, float(score(snap))))
        options.on_eval = on_eval
    out.report = run_fit(options)
    return out
