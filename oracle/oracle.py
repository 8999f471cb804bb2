"""ctypes wrapper of the CPU oracle (oracle/dfm_oracle.c).

TEST INFRASTRUCTURE ONLY.  Imported by tests/, __graft_entry__.smoke() and
bench.py's cpu_baseline / ``--impl reference`` leg — never by the product
package ``paper_2605_19388_b200``.

Arrays use the "math shapes" of the reference containers (see
paper_2605_19388_b200/layout.py for the same convention):
  x     (F, T, M) complex   x[i, j, m] = ObsTensor.bins[i](m, j)
  T     (N, F, K)           T[n, i, k] = NmfModel.T[n](i, k)
  V     (N, K, T)           V[n, k, j] = NmfModel.V[n](k, j)
  lam   (F, N, M)           lam[i, n, m] = Lambda[i](n, m)
  w     list over blocks of (F, mb, mb) complex, w[b][i] = W_b[i]
  eta,P (F, T, M);  h (F, T, N);  a,b (N, F, T);  images (N, F, T, M)
The C side stores Eigen column-major order, i.e. the last two axes swapped
(x, y, images already match).
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "_build", "libdfm_oracle.so")
_lib = None

_dp = C.POINTER(C.c_double)
_ip = C.POINTER(C.c_int)


class SingularDemixer(RuntimeError):
    pass


def build() -> str:
    subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return _LIB_PATH


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            build()
        L = C.CDLL(_LIB_PATH)
        L.dfo_splitmix64.restype = C.c_uint64
        L.dfo_splitmix64.argtypes = [C.POINTER(C.c_uint64)]
        L.dfo_derive_seed.restype = C.c_uint64
        L.dfo_derive_seed.argtypes = [C.c_uint64, C.c_char_p, C.c_uint64]
        L.dfo_power_term.restype = C.c_double
        L.dfo_logdet_term.restype = C.c_double
        L.dfo_log_abs_det.restype = C.c_double
        L.dfo_rng_draws.argtypes = [C.c_uint64, C.c_int, C.c_int, _dp]
        L.dfo_random_init.argtypes = [C.c_int, C.c_int, C.c_int, _ip, C.c_int, C.c_int, C.c_uint64,
                                      _dp, _dp, _dp, _dp]
        L.dfo_random_instance.argtypes = [C.c_int] * 5 + [C.c_uint64] + [_dp] * 5
        L.dfo_random_observations.argtypes = [C.c_int] * 3 + [C.c_uint64, _dp]
        L.dfo_generate_mixture.argtypes = [C.c_int] * 6 + [C.c_uint64, _dp]
        L.dfo_run_engine.argtypes = [C.c_int, C.c_int, C.c_int, _dp, C.c_int, _ip, C.c_int, C.c_int,
                                     _dp, _dp, _dp, _dp, C.c_int, C.c_double, _dp, _dp, _dp, _dp]
        L.dfo_ip_sweep_column.argtypes = [C.c_int] * 3 + [_dp, _dp, C.c_int, C.c_int, _dp, C.c_int,
                                                          C.c_double]
        L.dfo_cost_dist.argtypes = [C.c_int] * 3 + [_dp, C.c_int, _ip, C.c_int, C.c_int, _dp, _dp,
                                                    _dp, _dp, C.c_double, _dp]
        L.dfo_wiener_block.argtypes = [C.c_int] * 3 + [_dp, C.c_int, _ip, C.c_int, C.c_int, _dp,
                                                       _dp, _dp, _dp, C.c_double, _dp]
        for name in ("dfo_update_t", "dfo_update_v", "dfo_update_lambda", "dfo_build_tv_weights",
                     "dfo_eta_from", "dfo_spectrogram", "dfo_power_term", "dfo_update_v_apply"):
            getattr(L, name).argtypes = None
        _lib = L
    return _lib


def set_threads(n: int) -> None:
    lib().dfo_set_threads(int(n))


# ----------------------------------------------------------------- helpers
def _p(a: np.ndarray):
    assert a.flags.c_contiguous
    return a.ctypes.data_as(_dp)


def _ints(v):
    arr = (C.c_int * len(v))(*[int(s) for s in v])
    return arr


def _d(v: float):
    return C.c_double(float(v))


def to_c(a: np.ndarray) -> np.ndarray:
    """math shape -> C-ABI (Eigen col-major) buffer: swap the last two axes."""
    return np.ascontiguousarray(np.swapaxes(a, -1, -2))


def from_c(a: np.ndarray) -> np.ndarray:
    return np.ascontiguousarray(np.swapaxes(a, -1, -2))


def _cplx(a: np.ndarray) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.complex128)


def w_to_c(w_blocks) -> np.ndarray:
    return np.concatenate([to_c(_cplx(wb)).reshape(-1) for wb in w_blocks])


def w_from_c(buf: np.ndarray, F: int, sizes) -> list:
    out, o = [], 0
    for mb in sizes:
        n = F * mb * mb
        out.append(from_c(buf[o:o + n].reshape(F, mb, mb)))
        o += n
    return out


# ------------------------------------------------------------------- rng
def splitmix64(state: int):
    s = C.c_uint64(state)
    v = lib().dfo_splitmix64(C.byref(s))
    return int(v), int(s.value)


def rng_draws(seed: int, n: int, gaussian: bool = False) -> np.ndarray:
    out = np.empty(n)
    lib().dfo_rng_draws(C.c_uint64(seed), n, int(gaussian), _p(out))
    return out


def derive_seed(seed: int, tag: str, index: int = 0) -> int:
    return int(lib().dfo_derive_seed(C.c_uint64(seed), tag.encode(), C.c_uint64(index)))


# ----------------------------------------------------------------- inits
def random_init(F, T, sizes, N, K, seed) -> dict:
    M = sum(sizes)
    Tc = np.empty((N, K, F)); Vc = np.empty((N, T, K)); lc = np.empty((F, M, N))
    wc = np.empty(sum(F * s * s for s in sizes), dtype=np.complex128)
    lib().dfo_random_init(F, T, len(sizes), _ints(sizes), N, K, C.c_uint64(seed), _p(Tc), _p(Vc),
                          _p(lc), wc.ctypes.data_as(_dp))
    return dict(T=from_c(Tc), V=from_c(Vc), lam=from_c(lc), w=w_from_c(wc, F, sizes))


def random_instance(F, T, M, N, K, seed):
    """testutil.hpp:61-79: returns (x, T, V, lam, w_full (F, M, M))."""
    x = np.empty((F, T, M), dtype=np.complex128)
    Tc = np.empty((N, K, F)); Vc = np.empty((N, T, K)); lc = np.empty((F, M, N))
    wc = np.empty((F, M, M), dtype=np.complex128)
    lib().dfo_random_instance(F, T, M, N, K, C.c_uint64(seed), x.ctypes.data_as(_dp), _p(Tc),
                              _p(Vc), _p(lc), wc.ctypes.data_as(_dp))
    return x, from_c(Tc), from_c(Vc), from_c(lc), from_c(wc)


def random_observations(F, T, M, seed) -> np.ndarray:
    x = np.empty((F, T, M), dtype=np.complex128)
    lib().dfo_random_observations(F, T, M, C.c_uint64(seed), x.ctypes.data_as(_dp))
    return x


def generate_mixture(kind, F, T, M, N, K, seed) -> np.ndarray:
    x = np.empty((F, T, M), dtype=np.complex128)
    lib().dfo_generate_mixture(kind, F, T, M, N, K, C.c_uint64(seed), x.ctypes.data_as(_dp))
    return x


# ------------------------------------------------------------ step functions
def spectrogram(T_, V_) -> np.ndarray:
    N, F, K = T_.shape
    Tn = V_.shape[2]
    h = np.empty((F, N, Tn))
    lib().dfo_spectrogram(F, Tn, N, K, _p(to_c(T_)), _p(to_c(V_)), _p(h))
    return from_c(h)


def eta_from(h, lam, floor=1e-6) -> np.ndarray:
    F, Tn, N = h.shape
    M = lam.shape[2]
    eta = np.empty((F, M, Tn))
    lib().dfo_eta_from(F, Tn, N, M, _p(to_c(h)), _p(to_c(lam)), _d(floor), _p(eta))
    return from_c(eta)


def decorrelate_block(x, off, wb):
    """Returns (y rows of the block (F, T, mb) complex, P (F, T, mb))."""
    F, Tn, M = x.shape
    mb = wb.shape[1]
    y = np.zeros((F, Tn, M), dtype=np.complex128)
    P = np.zeros((F, M, Tn))
    lib().dfo_decorrelate_block(F, Tn, M, x.ctypes.data_as(_dp), off, mb,
                                to_c(_cplx(wb)).ctypes.data_as(_dp), y.ctypes.data_as(_dp), _p(P))
    return y[:, :, off:off + mb], from_c(P)[:, :, off:off + mb]


def ip_sweep_column(x, eta, off, wb, mu, floor=1e-6):
    F, Tn, M = x.shape
    mb = wb.shape[1]
    wc = to_c(_cplx(wb))
    nfb = lib().dfo_ip_sweep_column(F, Tn, M, _cplx(x).ctypes.data_as(_dp), _p(to_c(eta)), off, mb,
                                    wc.ctypes.data_as(_dp), mu, _d(floor))
    return from_c(wc), int(nfb)


def build_tv_weights(lam, P, eta):
    F, N, M = lam.shape
    Tn = P.shape[1]
    a = np.empty((N, Tn, F)); b = np.empty((N, Tn, F))
    lib().dfo_build_tv_weights(F, Tn, N, M, _p(to_c(lam)), _p(to_c(P)), _p(to_c(eta)), _p(a), _p(b))
    return from_c(a), from_c(b)


def update_t(T_, V_, a, b, floor=1e-6):
    N, F, K = T_.shape
    Tn = V_.shape[2]
    Tc = to_c(T_)
    lib().dfo_update_t(F, Tn, N, K, _p(Tc), _p(to_c(V_)), _p(to_c(a)), _p(to_c(b)), _d(floor))
    return from_c(Tc)


def update_v(T_, V_, a, b, floor=1e-6):
    N, F, K = T_.shape
    Tn = V_.shape[2]
    Vc = to_c(V_)
    lib().dfo_update_v(F, Tn, N, K, _p(to_c(T_)), _p(Vc), _p(to_c(a)), _p(to_c(b)), _d(floor))
    return from_c(Vc)


def update_v_partial(T_, a, b, f0, f1):
    """Sum over bins [f0, f1) of the V-update numerator/denominator; returns
    an array (2, N, T, K) = {num, den} in C order."""
    N, F, K = T_.shape
    Tn = a.shape[2]
    nd = np.empty((2, N, Tn, K))
    lib().dfo_update_v_partial(F, f0, f1, Tn, N, K, _p(to_c(T_)), _p(to_c(a)), _p(to_c(b)), _p(nd))
    return nd


def update_v_apply(V_, numden, floor=1e-6):
    N, K, Tn = V_.shape
    Vc = to_c(V_)
    lib().dfo_update_v_apply(Tn, N, K, _p(Vc), _p(np.ascontiguousarray(numden)), _d(floor))
    return from_c(Vc)


def update_lambda(lam, h, P, eta, floor=1e-6):
    F, N, M = lam.shape
    Tn = h.shape[1]
    lc = to_c(lam)
    lib().dfo_update_lambda(F, Tn, N, M, _p(lc), _p(to_c(h)), _p(to_c(P)), _p(to_c(eta)), _d(floor))
    return from_c(lc)


def power_term(P, h, lam, floor=1e-6) -> float:
    F, N, M = lam.shape
    Tn = h.shape[1]
    return float(lib().dfo_power_term(F, Tn, N, M, _p(to_c(P)), _p(to_c(h)), _p(to_c(lam)), _d(floor)))


def logdet_term(wb) -> float:
    F, mb, _ = wb.shape
    return float(lib().dfo_logdet_term(F, mb, to_c(_cplx(wb)).ctypes.data_as(_dp)))


def lu_solve(S, e):
    mb = S.shape[0]
    u = np.empty(mb, dtype=np.complex128)
    lib().dfo_lu_solve(mb, to_c(_cplx(S)).ctypes.data_as(_dp), _cplx(e).ctypes.data_as(_dp),
                       u.ctypes.data_as(_dp))
    return u


def pinv_solve(S, e):
    mb = S.shape[0]
    u = np.empty(mb, dtype=np.complex128)
    lib().dfo_pinv_solve(mb, to_c(_cplx(S)).ctypes.data_as(_dp), _cplx(e).ctypes.data_as(_dp),
                         u.ctypes.data_as(_dp))
    return u


# ------------------------------------------------------------------ engine
def run_engine(x, sizes, init: dict, iters: int, floor: float = 1e-6) -> dict:
    """engine.cpp:167-272 on a copy of ``init``; returns the fitted model and report."""
    x = _cplx(x)
    F, Tn, M = x.shape
    N, _, K = init["T"].shape
    Tc = to_c(init["T"]); Vc = to_c(init["V"]); lc = to_c(init["lam"]); wc = w_to_c(init["w"])
    cost = np.empty(iters + 1); wall = np.empty(max(iters, 1)); stages = np.empty(4); ops = np.empty(2)
    nfb = lib().dfo_run_engine(F, Tn, M, x.ctypes.data_as(_dp), len(sizes), _ints(sizes), N, K,
                               _p(Tc), _p(Vc), _p(lc), wc.ctypes.data_as(_dp), iters, floor,
                               _p(cost), _p(wall), _p(stages), _p(ops))
    if nfb < 0:
        raise ValueError("run_engine: invalid arguments")
    return dict(T=from_c(Tc), V=from_c(Vc), lam=from_c(lc), w=w_from_c(wc, F, sizes),
                cost_trace=cost, wall_seconds=wall[:iters],
                stages=dict(zip(("w_update", "mm_update", "eta", "decorrelate"), stages)),
                ops=dict(w_update=ops[0], mm_update=ops[1]), fallbacks=nfb)


def cost_dist(x, sizes, model: dict, floor: float = 1e-6) -> float:
    x = _cplx(x)
    F, Tn, M = x.shape
    N, _, K = model["T"].shape
    out = C.c_double()
    rc = lib().dfo_cost_dist(F, Tn, M, x.ctypes.data_as(_dp), len(sizes), _ints(sizes), N, K,
                             _p(to_c(model["T"])), _p(to_c(model["V"])), _p(to_c(model["lam"])),
                             w_to_c(model["w"]).ctypes.data_as(_dp), floor, C.byref(out))
    if rc:
        raise SingularDemixer("cost_dist: singular demixing matrix")
    return out.value


def wiener_block(x, sizes, model: dict, floor: float = 1e-6) -> np.ndarray:
    x = _cplx(x)
    F, Tn, M = x.shape
    N, _, K = model["T"].shape
    img = np.empty((N, F, Tn, M), dtype=np.complex128)
    lib().dfo_wiener_block(F, Tn, M, x.ctypes.data_as(_dp), len(sizes), _ints(sizes), N, K,
                           _p(to_c(model["T"])), _p(to_c(model["V"])), _p(to_c(model["lam"])),
                           w_to_c(model["w"]).ctypes.data_as(_dp), floor, img.ctypes.data_as(_dp))
    return img
