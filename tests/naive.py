"""Explicit-loop numpy oracles kept independent of the C restatement, the way
the reference keeps naive_decorrelate / naive_eta / naive_cost / the naive
MM updates (test_fastmnmf.cpp:16-53, :226-280) and the direct-covariance
Wiener oracle (test_wiener.cpp:14-35).  Math shapes as in oracle/oracle.py."""
import numpy as np

FLOOR = 1e-6


def decorrelate(x, w):
    """y[i, j, m] = sum_a conj(w[i][a, m]) x[i, j, a]   (test_fastmnmf.cpp:16-26)"""
    return np.einsum("iam,ija->ijm", np.conj(w), x)


def block_diag_w(w_blocks):
    F = w_blocks[0].shape[0]
    M = sum(b.shape[1] for b in w_blocks)
    out = np.zeros((F, M, M), dtype=np.complex128)
    o = 0
    for b in w_blocks:
        mb = b.shape[1]
        out[:, o:o + mb, o:o + mb] = b
        o += mb
    return out


def spectrogram(T, V):
    return np.einsum("nik,nkj->ijn", T, V)


def eta_raw(T, V, lam):
    """test_fastmnmf.cpp:28-37 (unfloored)"""
    return np.einsum("ijn,inm->ijm", spectrogram(T, V), lam)


def cost(x, T, V, lam, w_full, floor=FLOOR):
    """test_fastmnmf.cpp:39-53"""
    y = decorrelate(x, w_full)
    e = eta_raw(T, V, lam)
    acc = np.sum(np.abs(y) ** 2 / np.maximum(e, floor)) + np.sum(np.log(np.maximum(e, 1e-300)))
    Tn = x.shape[1]
    for i in range(x.shape[0]):
        acc -= Tn * np.log(np.abs(np.linalg.det(w_full[i])) ** 2)
    return float(acc)


def update_t(T, V, lam, P, floor=FLOOR):
    """test_fastmnmf.cpp:234-252 (eta from the current model, floored)"""
    e = np.maximum(eta_raw(T, V, lam), floor)
    num = np.einsum("nkj,inm,ijm->nik", V, lam, P / e ** 2)
    den = np.einsum("nkj,inm,ijm->nik", V, lam, 1.0 / e)
    return np.maximum(T * np.sqrt(num / np.maximum(den, floor)), floor)


def update_lambda(T, V, lam, P, floor=FLOOR):
    """test_fastmnmf.cpp:254-276"""
    h = spectrogram(T, V)
    e = np.maximum(eta_raw(T, V, lam), floor)
    num = np.einsum("ijn,ijm->inm", h, P / e ** 2)
    den = np.einsum("ijn,ijm->inm", h, 1.0 / e)
    return np.maximum(lam * np.sqrt(num / np.maximum(den, floor)), floor)


def wiener_direct(x, T, V, lam, w_full):
    """test_wiener.cpp:14-35: c_n = h_n R_n (sum h R)^-1 x, R_n = W^-H diag(lam_n) W^-1"""
    F, Tn, M = x.shape
    N = T.shape[0]
    h = spectrogram(T, V)
    out = np.zeros((N, F, Tn, M), dtype=np.complex128)
    for i in range(F):
        winv = np.linalg.inv(w_full[i])
        R = [winv.conj().T @ np.diag(lam[i, n]) @ winv for n in range(N)]
        for j in range(Tn):
            tot = sum(h[i, j, n] * R[n] for n in range(N))
            ti = np.linalg.inv(tot)
            for n in range(N):
                out[n, i, j] = h[i, j, n] * R[n] @ ti @ x[i, j]
    return out
