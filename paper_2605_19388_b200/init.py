"""Initialisation pipeline (mirror of include/fastmnmf/init.hpp:10-111): k-means
soft masks with permutation alignment, masked spatial covariances, ML
spectrograms, the Itakura-Saito NMF warm start and the GEVD spatial start,
run on the device through the C ABI (csrc/dfm_init.cu; the alignment is host
code, csrc/dfm_align.cpp).

Shapes: x (F, T, M) complex; masks and h0 (F, T, N) with rows summing to one
(SoftMask); R (N, F, M, M); NmfModel T (N, F, K), V (N, K, T); Lambda
(F, N, M); W blocks (F, M_b, M_b)."""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from typing import List, Optional, Sequence

import numpy as np

from . import _capi
from ._capi import check
from .fastmnmf import BlockLayout, InitBundle, NmfModel, _c, _obs, _uc, _w_from_c


def _p(a: np.ndarray):
    assert a.flags.c_contiguous
    return a.ctypes.data_as(C.c_void_p)


@dataclass
class MaskOptions:
    """init.hpp:19-24."""
    kmeans_iters: int = 50
    softmax_temperature: float = 1.0
    align_neighborhood: int = 3
    align_rounds: int = 10


@dataclass
class InitConfig:
    """init.hpp:82-87."""
    num_sources: int = 3
    k_bases: int = 16
    nmf_max_iters: int = 1000
    mask_options: MaskOptions = field(default_factory=MaskOptions)


def cluster_masks(x: np.ndarray, num_sources: int, seed: int, options: MaskOptions = MaskOptions(),
                  device: int = 0) -> np.ndarray:
    """init.cpp:76-188: bin-wise k-means soft masks, then frequency alignment."""
    x = _obs(x)
    F, T, M = x.shape
    m = np.zeros((F, num_sources, T))
    check(_capi.load().dfm_cluster_masks(_p(x), F, T, M, num_sources, int(seed) & (2 ** 64 - 1),
                                         options.kmeans_iters, options.softmax_temperature,
                                         options.align_neighborhood, options.align_rounds, _p(m), device))
    return _uc(m)


def align_frequency_permutations(mask: np.ndarray, options: MaskOptions = MaskOptions()) -> np.ndarray:
    """init.cpp:190-221 (returns the aligned copy)."""
    m = _c(mask)
    F, N, T = m.shape
    check(_capi.load().dfm_align_frequency_permutations(_p(m), F, T, N, options.align_neighborhood,
                                                        options.align_rounds))
    return _uc(m)


def align_subarray_permutations(masks: Sequence[np.ndarray]) -> List[List[int]]:
    """init.cpp:223-250: perms[l][n] = source of mask l matched to source n of mask 0."""
    if len(masks) < 2:
        raise ValueError("align_subarray_permutations: need at least two subarrays")
    F, T, N = masks[0].shape
    for m in masks:
        if m.shape != (F, T, N):
            from ._capi import ShapeMismatchError
            raise ShapeMismatchError("align_subarray_permutations: mask shapes differ")
    buf = np.ascontiguousarray(np.stack([_c(m) for m in masks]))
    perms = np.zeros((len(masks), N), dtype=np.int32)
    check(_capi.load().dfm_align_subarray_permutations(_p(buf), len(masks), F, T, N, _p(perms)))
    return perms.tolist()


def permute_mask(mask: np.ndarray, permutation: Sequence[int]) -> np.ndarray:
    """init.cpp:252-256 (column gather)."""
    return np.ascontiguousarray(mask[:, :, list(permutation)])


def soft_mask_images(x: np.ndarray, mask: np.ndarray) -> List[np.ndarray]:
    """init.cpp:258-266: c_ijn = mask_ijn x_ij (the images add up to x)."""
    x = _obs(x)
    if mask.shape[:2] != x.shape[:2]:
        from ._capi import ShapeMismatchError
        raise ShapeMismatchError("soft_mask_images: mask does not match observations")
    return [x * mask[:, :, n][:, :, None] for n in range(mask.shape[2])]


def _scm_spec(x: np.ndarray, sizes: Sequence[int], masks: Sequence[np.ndarray], device: int = 0):
    x = _obs(x)
    F, T, M = x.shape
    N = masks[0].shape[2]
    mb = np.ascontiguousarray(np.stack([_c(m) for m in masks]))
    R = np.zeros((N, F, M, M), dtype=np.complex128)
    h0 = np.zeros((F, N, T))
    sz = np.ascontiguousarray(sizes, dtype=np.int32)
    check(_capi.load().dfm_init_scm_spectrogram(_p(x), F, T, M, N, len(sizes), _p(sz), _p(mb), _p(R), _p(h0),
                                                device))
    return _uc(R), _uc(h0)


def init_scm(images: Sequence[np.ndarray], device: int = 0) -> np.ndarray:
    """init.cpp:268-278: R_n,f = sum_t c c^H / T -> (N, F, M, M)."""
    out = []
    for img in images:
        F, T, M = img.shape
        R, _ = _scm_spec(img, [M], [np.ones((F, T, 1))], device)
        out.append(R[0])
    return np.stack(out)


def init_spectrogram(images: Sequence[np.ndarray], device: int = 0) -> np.ndarray:
    """init.cpp:280-304: h0 = max(Re(c^H (R + ridge)^-1 c) / M, 0) -> (F, T, N),
    with R = init_scm(images) recomputed on the device."""
    cols = []
    for img in images:
        F, T, M = img.shape
        _, h = _scm_spec(img, [M], [np.ones((F, T, 1))], device)
        cols.append(h[:, :, 0])
    return np.stack(cols, axis=2)


def itakura_saito_nmf(h0: np.ndarray, k: int, max_iters: int, seed: int, divergence_trace: Optional[list] = None,
                      device: int = 0) -> NmfModel:
    """init.cpp:306-372: per-source IS-NMF by multiplicative updates (all
    sources batched on the device).  divergence_trace, when a list, receives
    one divergence sequence per source."""
    hc = _c(h0)  # (F, N, T)
    F, N, T = hc.shape
    Tm = np.zeros((N, k, F))
    V = np.zeros((N, T, k))
    tr = np.zeros((N, max_iters + 1))
    its = np.zeros(N, dtype=np.int32)
    check(_capi.load().dfm_is_nmf(_p(hc), F, T, N, k, max_iters, int(seed) & (2 ** 64 - 1), _p(Tm), _p(V),
                                  _p(tr), _p(its), device))
    if divergence_trace is not None:
        for n in range(N):
            divergence_trace.append(tr[n, :its[n] + 1].copy())
    return NmfModel(_uc(Tm), _uc(V))


def init_spatial(r_init: np.ndarray, layout: BlockLayout, device: int = 0):
    """init.cpp:374-407 (+ the kFloor clamp): (w0 blocks, lambda0 (F, N, M))."""
    Rc = _c(r_init, np.complex128)
    N, F, M, _ = Rc.shape
    if N < 2:
        raise ValueError("init_spatial: needs at least two sources")
    sz = np.ascontiguousarray(layout.sizes, dtype=np.int32)
    w0 = np.zeros(sum(F * s * s for s in layout.sizes), dtype=np.complex128)
    lam = np.zeros((F, M, N))
    check(_capi.load().dfm_init_spatial(_p(Rc), F, M, N, len(layout.sizes), _p(sz), _p(w0), _p(lam), device))
    return _w_from_c(w0, F, layout.sizes), _uc(lam)


def _pipeline(x: np.ndarray, layout: BlockLayout, cfg: InitConfig, seed: int, device: int = 0) -> InitBundle:
    x = _obs(x)
    F, T, M = x.shape
    if layout.total != M:
        from ._capi import ShapeMismatchError
        raise ShapeMismatchError("init_distributed: layout/channel mismatch")
    N, K = cfg.num_sources, cfg.k_bases
    o = cfg.mask_options
    sz = np.ascontiguousarray(layout.sizes, dtype=np.int32)
    Tm = np.zeros((N, K, F))
    V = np.zeros((N, T, K))
    lam = np.zeros((F, M, N))
    w0 = np.zeros(sum(F * s * s for s in layout.sizes), dtype=np.complex128)
    h0 = np.zeros((F, N, T))
    mask = np.zeros((F, N, T))
    check(_capi.load().dfm_init_pipeline(_p(x), F, T, len(layout.sizes), _p(sz), N, K, int(seed) & (2 ** 64 - 1),
                                         cfg.nmf_max_iters, o.kmeans_iters, o.softmax_temperature,
                                         o.align_neighborhood, o.align_rounds, _p(Tm), _p(V), _p(lam), _p(w0),
                                         _p(h0), _p(mask), device))
    b = InitBundle(layout, NmfModel(_uc(Tm), _uc(V)), _w_from_c(w0, F, layout.sizes), _uc(lam))
    b.h0 = _uc(h0)
    b.mask = _uc(mask)
    return b


def init_full(x: np.ndarray, cfg: InitConfig, seed: int, device: int = 0) -> InitBundle:
    """init.cpp:431-436: one mask over all channels, full-array GEVD."""
    return _pipeline(x, BlockLayout([_obs(x).shape[2]]), cfg, seed, device)


def init_distributed(x: np.ndarray, layout: BlockLayout, cfg: InitConfig, seed: int, device: int = 0) -> InitBundle:
    """init.cpp:438-472: per-subarray masks aligned across subarrays,
    block-diagonal GEVD, shared IS-NMF warm start."""
    return _pipeline(x, layout, cfg, seed, device)
