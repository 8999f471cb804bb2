"""TEST INFRASTRUCTURE ONLY (checker, never shipped): an independent
restatement of the reference's FMNM v2 model container, src/io.cpp:49-135,
in plain numpy/struct, used to cross-check the native reader/writer
(csrc/dfm_io.cpp) and to generate the golden container under tests/golden/.

Layout (little-endian): "FMNM", u32 version=2, u32 bins, u32 frames,
u32 channels, u32 sources, u32 k_bases, u32 n_blocks, u32 sizes[n_blocks],
u8 shared, f64 floor, u64 seed, f64 sample_rate, u32 window_len,
u32 hop_len, u32 iterations (io.cpp:60-73), u32 n_models, then per model
every T_n (bins x K, Eigen col-major) followed by every V_n (K x frames)
(io.cpp:75-79), Lambda per bin (sources x channels, :80), W per block per bin
(M_b x M_b complex, :81-82).
"""
import struct

import numpy as np

MAGIC = b"FMNM"
VERSION = 2


def write(path, cfg, sizes, shared, models, lam, w):
    """models: list of (T (N, F, K), V (N, K, J)); lam (F, N, M); w: [block] (F, mb, mb)."""
    F, N, M = lam.shape
    J = models[0][1].shape[2] if models else 0
    with open(path, "wb") as fh:
        fh.write(MAGIC)
        fh.write(struct.pack("<7I", VERSION, F, J, M, N, cfg["k_bases"], len(sizes)))
        fh.write(struct.pack(f"<{len(sizes)}I", *sizes))
        fh.write(struct.pack("<B", 1 if shared else 0))
        fh.write(struct.pack("<dQd3I", cfg["floor"], cfg["seed"], cfg["sample_rate"], cfg["window_len"],
                             cfg["hop_len"], cfg["iterations"]))
        fh.write(struct.pack("<I", len(models)))
        for T, V in models:
            for n in range(N):
                fh.write(np.asfortranarray(T[n]).tobytes(order="F"))
            for n in range(N):
                fh.write(np.asfortranarray(V[n]).tobytes(order="F"))
        for f in range(F):
            fh.write(np.asfortranarray(lam[f]).tobytes(order="F"))
        for wb in w:
            for f in range(F):
                fh.write(np.asfortranarray(wb[f]).astype(np.complex128).tobytes(order="F"))


def read(path):
    with open(path, "rb") as fh:
        buf = fh.read()
    if buf[:4] != MAGIC:
        raise RuntimeError(f"load_model: bad magic in {path}")
    o = 4
    (version,) = struct.unpack_from("<I", buf, o)
    o += 4
    if version != VERSION:
        raise RuntimeError("load_model: unsupported container version")
    F, J, M, N, K, nb = struct.unpack_from("<6I", buf, o)
    o += 24
    sizes = list(struct.unpack_from(f"<{nb}I", buf, o))
    o += 4 * nb
    if sum(sizes) != M:
        raise RuntimeError("load_model: layout mismatch")
    (shared,) = struct.unpack_from("<B", buf, o)
    o += 1
    floor, seed, sr, wl, hl, it = struct.unpack_from("<dQd3I", buf, o)
    o += 36
    (nm,) = struct.unpack_from("<I", buf, o)
    o += 4

    def take(count, dtype, shape):
        nonlocal o
        nbytes = count * np.dtype(dtype).itemsize
        if o + nbytes > len(buf):
            raise RuntimeError(f"load_model: truncated file {path}")
        a = np.frombuffer(buf, dtype=dtype, count=count, offset=o).reshape(shape, order="F")
        o += nbytes
        return np.array(a)

    models = []
    for _ in range(nm):
        T = np.stack([take(F * K, np.float64, (F, K)) for _ in range(N)]) if N else np.zeros((0, F, K))
        V = np.stack([take(K * J, np.float64, (K, J)) for _ in range(N)]) if N else np.zeros((0, K, J))
        models.append((T, V))
    lam = np.stack([take(N * M, np.float64, (N, M)) for _ in range(F)])
    w = [np.stack([take(mb * mb, np.complex128, (mb, mb)) for _ in range(F)]) for mb in sizes]
    cfg = dict(n_sources=N, k_bases=K, iterations=it, floor=floor, seed=seed, sample_rate=sr, window_len=wl,
               hop_len=hl)
    return cfg, sizes, bool(shared), models, lam, w
