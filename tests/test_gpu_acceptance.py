"""The reference's in-scope acceptance criteria (proj/tests/acceptance.cpp)
run on the device path.  SURVEY.md §2.1 marks criteria 1, 2, 3, 9 and 12 in
scope; 2 (L=1 bitwise), 3 (independent mode) and 9 (Wiener equivalence) are
in tests/test_gpu_parity.py (test_engine_is_deterministic_and_l1_reduction,
test_engine_underdetermined_and_independent_mode, test_wiener_reference_cases_
on_device).  Here:
  criterion 1  per-update monotonicity on 50 random instances, full-array and
               per-subarray IP (acceptance.cpp:57-152),
  criterion 7  runtime ordering single < distributed < full with
               distributed <= 0.6 x full and the MM-stage ratio in
               [0.5, 1.5] (acceptance.cpp:398-422; bench.cpp:75-103),
  criterion 12 recovery of model-sampled data (acceptance.cpp:628-704), with
               an STFT-domain image error in place of the SDR scorer (sdr.cpp
               is out of scope).
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

M64 = (1 << 64) - 1


class Rng:
    """rng.hpp:21-48 (splitmix64; next_below = next % n)."""

    def __init__(self, seed):
        self.s = seed & M64
        self.next_u64()

    def next_u64(self):
        self.s = (self.s + 0x9E3779B97F4A7C15) & M64
        z = self.s
        z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & M64
        z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & M64
        return z ^ (z >> 31)

    def next_below(self, n):
        return self.next_u64() % n

    def uniform(self):
        return (self.next_u64() >> 11) * 2.0 ** -53


@pytest.fixture(scope="module")
def dfm():
    import torch

    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    import paper_2605_19388_b200 as m

    m._capi.load()
    return m


def test_rng_matches_the_oracle(oracle):
    # the port above against the oracle's rng.hpp restatement
    r = Rng(1234)
    got = [r.uniform() for _ in range(8)]
    assert np.array_equal(np.array(got), oracle.rng_draws(1234, 8))


def _le(a, b):
    return a <= b + 1e-9 * abs(b)


def test_criterion1_per_update_monotonicity(dfm, oracle):
    for seed in range(50):
        dr = Rng(seed * 31 + 1)
        I = 2 + dr.next_below(7)
        J = 8 + dr.next_below(25)
        M = 2 + dr.next_below(5)
        N = 1 + dr.next_below(3)
        K = 1 + dr.next_below(3)
        x, Tm, V, lam, w = oracle.random_instance(I, J, M, N, K, seed)
        # full-array granular updates: IP columns, then t, v, Lambda (two sweeps)
        nmf = dfm.NmfModel(Tm.copy(), V.copy())
        W = w.copy()
        L = lam.copy()
        eta = dfm.compute_eta(nmf, L)
        cost = dfm.cost_full(x, nmf, dfm.SpatialModel(W, L))
        for _ in range(2):
            for m in range(M):
                dfm.ip_update_w(x, eta, W, m)
                nxt = dfm.cost_full(x, nmf, dfm.SpatialModel(W, L))
                assert _le(nxt, cost), f"full IP increased cost at seed {seed}"
                cost = nxt
            P = dfm.power_of(dfm.decorrelate(x, W))
            for what, upd in (("t", dfm.mm_update_t), ("v", dfm.mm_update_v), ("lambda", dfm.mm_update_lambda)):
                upd(nmf, L, P, eta)
                nxt = dfm.cost_full(x, nmf, dfm.SpatialModel(W, L))
                assert _le(nxt, cost), f"{what} increased cost at seed {seed}"
                cost = nxt
        # per-subarray IP columns on the block-diagonal model
        sr = Rng(seed * 17 + 3)
        sizes, left = [], M
        while left > 0:
            s = 1 + sr.next_below(min(left, 3))
            sizes.append(s)
            left -= s
        layout = dfm.BlockLayout(sizes)
        blocks, o = [], 0
        for mb in sizes:
            blocks.append(np.ascontiguousarray(w[:, o:o + mb, o:o + mb]))
            o += mb
        nmf = dfm.NmfModel(Tm.copy(), V.copy())
        spatial = dfm.BlockSpatialModel(layout, blocks, lam.copy())
        eta = dfm.compute_eta(nmf, spatial.Lambda)
        cost = dfm.cost_dist(x, nmf, spatial)
        for l, mb in enumerate(sizes):
            for mu in range(mb):
                dfm.ip_update_block(x, eta, layout, l, spatial.W[l], mu)
                nxt = dfm.cost_dist(x, nmf, spatial)
                assert _le(nxt, cost), f"block IP increased cost at seed {seed}"
                cost = nxt
    # 200-iteration traces stay monotone (full and distributed, fused engine)
    x, Tm, V, lam, w = oracle.random_instance(6, 24, 4, 2, 3, 999)
    init_f = dfm.InitBundle(dfm.BlockLayout([4]), dfm.NmfModel(Tm, V), [w], lam)
    tr = dfm.fit_full(x, init_f, 200).report.cost_trace
    assert np.all(tr[1:] <= tr[:-1] + 1e-9 * np.abs(tr[:-1]))
    init_d = dfm.InitBundle(dfm.BlockLayout([2, 2]), dfm.NmfModel(Tm, V),
                            [np.ascontiguousarray(w[:, :2, :2]), np.ascontiguousarray(w[:, 2:, 2:])], lam)
    tr = dfm.fit_distributed(x, dfm.BlockLayout([2, 2]), init_d, 200, True).report.cost_trace
    assert np.all(tr[1:] <= tr[:-1] + 1e-9 * np.abs(tr[:-1]))


def _bench_methods(dfm, F, T, N, K, partition, iters, repeats, seed):
    """bench.cpp:75-103 through the device fits: one warm-up run (1
    iteration) before every timed run; totals are the summed per-iteration
    device times (FitReport.total_seconds), stages averaged over repeats."""
    layout = dfm.BlockLayout(partition)
    x = dfm.random_observations(F, T, layout.total, seed)
    x1 = dfm.extract_block(x, layout, 0)
    init_full = dfm.random_init(F, T, dfm.BlockLayout([layout.total]), N, K, seed)
    init_dist = dfm.random_init(F, T, layout, N, K, seed)
    init_single = dfm.slice_init(init_dist, 0)
    runs = {
        "single": lambda n: dfm.fit_single(x1, init_single, n).report,
        "distributed": lambda n: dfm.fit_distributed(x, layout, init_dist, n, True).report,
        "full": lambda n: dfm.fit_full(x, init_full, n).report,
    }
    out = {}
    res = {k: [] for k in runs}
    for _ in range(repeats):
        for k, run in runs.items():
            run(1)
            res[k].append(run(iters))
    for k, reps in res.items():
        tot = np.array([r.total_seconds() for r in reps])
        stages = {s: np.mean([r.stages[s] for r in reps]) for s in reps[0].stages}
        out[k] = dict(mean=float(tot.mean()), se=float(tot.std(ddof=1) / np.sqrt(len(tot))), stages=stages)
    return out


def test_criterion7_runtime_ordering(dfm):
    r = _bench_methods(dfm, 96, 256, 3, 16, [4, 4, 4], 200, 3, 12345)
    s, d, f = r["single"]["mean"], r["distributed"]["mean"], r["full"]["mean"]
    mm_full = r["full"]["stages"]["mm_update"] + r["full"]["stages"]["eta"]
    mm_dist = r["distributed"]["stages"]["mm_update"] + r["distributed"]["stages"]["eta"]
    print(f"single {s:.4f} +- {r['single']['se']:.4f} s, distributed {d:.4f} +- {r['distributed']['se']:.4f} s, "
          f"full {f:.4f} +- {r['full']['se']:.4f} s (ratio {d / f:.3f}), MM-stage ratio {mm_dist / mm_full:.3f}; "
          f"stages {r['distributed']['stages']}")
    for k in r:  # every stage is measured, and the stages sum to about the fit's device time
        st = r[k]["stages"]
        assert all(v > 0 for v in st.values()), (k, st)
        assert 0.5 * r[k]["mean"] <= sum(st.values()) <= 1.2 * r[k]["mean"], (k, st, r[k]["mean"])
    assert s < d < f
    assert d <= 0.6 * f
    assert 0.5 <= mm_dist / mm_full <= 1.5


def _sample_model(rng, r, h):
    """c_n,i,j ~ CN(0, h[i, j, n] R_n,i) (mixsim.cpp:284-302 sample_model, in
    distribution): x = sum_n c_n."""
    N, F = len(r), len(r[0])
    T = h.shape[1]
    M = r[0][0].shape[0]
    imgs = np.zeros((N, F, T, M), dtype=np.complex128)
    for n in range(N):
        for i in range(F):
            Lc = np.linalg.cholesky(r[n][i])
            z = (rng.standard_normal((T, M)) + 1j * rng.standard_normal((T, M))) / np.sqrt(2)
            imgs[n, i] = np.sqrt(h[i, :, n])[:, None] * (z @ Lc.T)
    return imgs.sum(0), imgs


def test_criterion12_model_sampled_recovery(dfm):
    """Block-diagonal ground-truth model with temporally structured sources
    (acceptance.cpp:634-664), init_distributed, a 200-iteration distributed
    fit, Wiener separation: the final cost is below the initial one, and the
    separated images improve on the mixture (best permutation, all mics, STFT
    domain) on average over 10 seeds."""
    from paper_2605_19388_b200 import init as dinit

    F, T, N = 33, 300, 2  # 64-sample window, 16 hop at 8 kHz: 33 bins
    layout = dfm.BlockLayout([4, 4])
    gains = []
    for seed in range(10):
        rng = np.random.default_rng(7000 + seed)
        r = []
        for n in range(N):
            rn = []
            for i in range(F):
                R = np.zeros((8, 8), dtype=np.complex128)
                for o in (0, 4):
                    a = (rng.standard_normal(4) + 1j * rng.standard_normal(4)) / np.sqrt(2)
                    R[o:o + 4, o:o + 4] = np.outer(a, a.conj()) + 0.01 * np.eye(4)
                rn.append(R)
            r.append(rn)
        h = np.zeros((F, T, N))
        j = np.arange(T)
        for n in range(N):
            rate = 0.5 + 0.8 * n
            spectral = 0.2 + rng.uniform(size=F)
            env = 0.05 + (0.5 + 0.5 * np.sin(2 * np.pi * rate * j / 50.0 + n)) ** 2
            h[:, :, n] = spectral[:, None] * env[None, :]
        x, truth = _sample_model(np.random.default_rng(7700 + seed), r, h)
        init = dinit.init_distributed(x, layout, dinit.InitConfig(N, 4), seed)
        fit = dfm.fit_distributed(x, layout, init, 200, True)
        tr = fit.report.cost_trace
        assert tr[-1] <= tr[0], f"final cost above the initial cost at seed {seed}"
        est = dfm.wiener_block(x, fit.models, fit.spatial).images

        def snr(ref, e):
            return 10 * np.log10(np.sum(np.abs(ref) ** 2) / np.sum(np.abs(e - ref) ** 2))

        best = -np.inf
        for perm in ((0, 1), (1, 0)):
            g = np.mean([snr(truth[n], est[perm[n]]) - snr(truth[n], x) for n in range(N)])
            best = max(best, g)
        gains.append(best)
    print("image-domain improvement per seed (dB):", np.round(gains, 2))
    assert np.mean(gains) > 0.0
