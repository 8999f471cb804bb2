"""TEST INFRASTRUCTURE ONLY: Python face of the C restatement of the
reference's initialisation pipeline (oracle/dfm_init_oracle.c; src/init.cpp
and the GEVD of src/hermlin.cpp).  Math shapes: x (F, T, M) complex, masks
and h0 (F, T, N), R (N, F, M, M), T (N, F, K), V (N, K, T), Lambda (F, N, M),
W blocks (F, M_b, M_b)."""
import ctypes as C

import numpy as np

import oracle as _o

_dp = C.POINTER(C.c_double)
_ip = C.POINTER(C.c_int)


def _lib():
    L = _o.lib()
    if not getattr(L, "_init_sigs", False):
        L.dfo_cluster_masks.argtypes = [C.c_int] * 3 + [_dp, C.c_int, C.c_uint64, C.c_int, C.c_double, C.c_int,
                                                        C.c_int, _dp]
        L.dfo_align_subarray_permutations.argtypes = [C.c_int] * 4 + [_dp, _ip]
        L.dfo_align_frequency_permutations.argtypes = [C.c_int] * 3 + [_dp, C.c_int, C.c_int]
        L.dfo_best_permutation.argtypes = [C.c_int, C.c_int, _dp, _dp, _ip]
        L.dfo_init_scm.argtypes = [C.c_int] * 4 + [_dp, C.c_int, _ip, _dp, _dp]
        L.dfo_init_spectrogram.argtypes = [C.c_int] * 4 + [_dp, C.c_int, _ip, _dp, _dp, _dp]
        L.dfo_is_nmf.argtypes = [C.c_int] * 4 + [_dp, C.c_int, C.c_uint64, _dp, _dp, _dp, _ip]
        L.dfo_gevd.argtypes = [C.c_int, _dp, _dp, _dp, _dp]
        L.dfo_init_spatial.argtypes = [C.c_int] * 4 + [_ip, _dp, _dp, _dp]
        L._init_sigs = True
    return L


def _p(a):
    return a.ctypes.data_as(_dp)


def _ints(v):
    a = np.ascontiguousarray(v, dtype=np.int32)
    return a, a.ctypes.data_as(_ip)


def cluster_masks(x, N, seed, kmeans_iters=50, temp=1.0, nbhd=3, rounds=10):
    """init.cpp:76-188 (+ align_frequency_permutations) -> mask (F, T, N)."""
    x = np.ascontiguousarray(x, dtype=np.complex128)
    F, T, M = x.shape
    m = np.zeros((F, N, T))
    rc = _lib().dfo_cluster_masks(F, T, M, _p(x.view(np.float64)), N, C.c_uint64(seed), kmeans_iters, temp, nbhd,
                                  rounds, _p(m))
    if rc == -1:
        raise ValueError("cluster_masks: need at least one source")
    if rc == -2:
        raise ValueError("cluster_masks: fewer frames than sources")
    return _o.from_c(m)


def align_frequency_permutations(mask, nbhd=3, rounds=10):
    m = np.ascontiguousarray(_o.to_c(np.asarray(mask, dtype=np.float64)))
    F, N, T = m.shape
    _lib().dfo_align_frequency_permutations(F, T, N, _p(m), nbhd, rounds)
    return _o.from_c(m)


def best_permutation(cand, ref):
    """cand, ref: (L, N) -> permutation list (init.cpp:24-42)."""
    c = np.ascontiguousarray(np.asarray(cand, dtype=np.float64).T)
    r = np.ascontiguousarray(np.asarray(ref, dtype=np.float64).T)
    N, L = c.shape
    out, po = _ints(np.zeros(N))
    if _lib().dfo_best_permutation(L, N, _p(c), _p(r), po) != 0:
        raise ValueError("permutation alignment: too many sources for exhaustive search")
    return [int(v) for v in out]


def align_subarray_permutations(masks):
    """init.cpp:223-250: masks list of (F, T, N) -> perms (L, N)."""
    L = len(masks)
    F, T, N = masks[0].shape
    buf = np.ascontiguousarray(np.stack([_o.to_c(np.asarray(m, dtype=np.float64)) for m in masks]))
    perms, pp = _ints(np.zeros((L, N)))
    if _lib().dfo_align_subarray_permutations(L, F, T, N, _p(buf), pp) != 0:
        raise ValueError("align_subarray_permutations: need at least two subarrays")
    return perms.astype(int)


def _mask_stack(masks):
    return np.ascontiguousarray(np.stack([_o.to_c(np.asarray(m, dtype=np.float64)) for m in masks]))


def init_scm(x, sizes, masks):
    """init.cpp:268-278 with block b's channels masked by masks[b] -> R (N, F, M, M)."""
    x = np.ascontiguousarray(x, dtype=np.complex128)
    F, T, M = x.shape
    N = masks[0].shape[2]
    R = np.zeros((N, F, M, M), dtype=np.complex128)
    sz, ps = _ints(sizes)
    _lib().dfo_init_scm(F, T, M, N, _p(x.view(np.float64)), len(sizes), ps, _p(_mask_stack(masks)),
                        _p(R.view(np.float64)))
    return _o.from_c(R)


def init_spectrogram(x, sizes, masks, R):
    """init.cpp:280-304 -> h0 (F, T, N)."""
    x = np.ascontiguousarray(x, dtype=np.complex128)
    F, T, M = x.shape
    N = masks[0].shape[2]
    Rc = np.ascontiguousarray(_o.to_c(np.asarray(R, dtype=np.complex128)))
    h0 = np.zeros((F, N, T))
    sz, ps = _ints(sizes)
    _lib().dfo_init_spectrogram(F, T, M, N, _p(x.view(np.float64)), len(sizes), ps, _p(_mask_stack(masks)),
                                _p(Rc.view(np.float64)), _p(h0))
    return _o.from_c(h0)


def is_nmf(h0, K, max_iters, seed):
    """init.cpp:306-372 -> (T (N, F, K), V (N, K, T), traces, iterations)."""
    hc = np.ascontiguousarray(_o.to_c(np.asarray(h0, dtype=np.float64)))
    F, N, T = hc.shape
    Tm = np.zeros((N, K, F))
    V = np.zeros((N, T, K))
    tr = np.full((N, max_iters + 1), np.nan)
    its, pi = _ints(np.zeros(N))
    _lib().dfo_is_nmf(F, T, N, K, _p(hc), max_iters, C.c_uint64(seed), _p(Tm), _p(V), _p(tr), pi)
    traces = [tr[n, :its[n] + 1].copy() for n in range(N)]
    return _o.from_c(Tm), _o.from_c(V), traces, its.astype(int)


def gevd(A, B):
    """hermlin.cpp:25-53 -> (w (m, m), d (m,)) with A w = d B w, w^H B w = I."""
    A = np.ascontiguousarray(_o.to_c(np.asarray(A, dtype=np.complex128)))
    B = np.ascontiguousarray(_o.to_c(np.asarray(B, dtype=np.complex128)))
    m = A.shape[0]
    w = np.zeros((m, m), dtype=np.complex128)
    d = np.zeros(m)
    if _lib().dfo_gevd(m, _p(A.view(np.float64)), _p(B.view(np.float64)), _p(w.view(np.float64)), _p(d)) != 0:
        raise RuntimeError("gevd_joint_diag: B is not positive definite")
    return _o.from_c(w), d


def init_spatial(R, sizes):
    """init.cpp:374-407 (+ kFloor clamp) -> (w0 blocks, lambda0 (F, N, M))."""
    Rc = np.ascontiguousarray(_o.to_c(np.asarray(R, dtype=np.complex128)))
    N, F, M, _ = Rc.shape
    w0 = np.zeros(sum(F * s * s for s in sizes), dtype=np.complex128)
    lam = np.zeros((F, M, N))
    sz, ps = _ints(sizes)
    if _lib().dfo_init_spatial(F, M, N, len(sizes), ps, _p(Rc.view(np.float64)), _p(w0.view(np.float64)),
                               _p(lam)) != 0:
        raise ValueError("init_spatial: needs at least two sources")
    return _o.w_from_c(w0, F, sizes), _o.from_c(lam)


def extract_block(x, sizes, b):
    o = sum(sizes[:b])
    return np.ascontiguousarray(x[:, :, o:o + sizes[b]])


def init_distributed(x, sizes, N, K, seed, nmf_iters=1000, kmeans_iters=50, temp=1.0, nbhd=3, rounds=10):
    """init.cpp:440-472: per-block masks aligned to block 0, masked images,
    SCMs, ML spectrograms, IS-NMF warm start, block-diagonal GEVD."""
    masks = [cluster_masks(extract_block(x, sizes, b), N, _o.derive_seed(seed, "mask", b), kmeans_iters, temp,
                           nbhd, rounds) for b in range(len(sizes))]
    if len(sizes) > 1:
        perms = align_subarray_permutations(masks)
        masks = [masks[0]] + [masks[b][:, :, perms[b]] for b in range(1, len(sizes))]
    R = init_scm(x, sizes, masks)
    h0 = init_spectrogram(x, sizes, masks, R)
    Tm, V, traces, its = is_nmf(h0, K, nmf_iters, _o.derive_seed(seed, "is-nmf"))
    w0, lam = init_spatial(R, sizes)
    return dict(masks=masks, R=R, h0=h0, T=Tm, V=V, traces=traces, nmf_iters=its, w0=w0, lambda0=lam)


def init_full(x, N, K, seed, nmf_iters=1000, kmeans_iters=50, temp=1.0, nbhd=3, rounds=10):
    """init.cpp:431-436: one mask over all channels (layout = one block)."""
    M = x.shape[2]
    mask = cluster_masks(x, N, _o.derive_seed(seed, "mask"), kmeans_iters, temp, nbhd, rounds)
    R = init_scm(x, [M], [mask])
    h0 = init_spectrogram(x, [M], [mask], R)
    Tm, V, traces, its = is_nmf(h0, K, nmf_iters, _o.derive_seed(seed, "is-nmf"))
    w0, lam = init_spatial(R, [M])
    return dict(masks=[mask], R=R, h0=h0, T=Tm, V=V, traces=traces, nmf_iters=its, w0=w0, lambda0=lam)
