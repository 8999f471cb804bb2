"""The north_star parity bar on every BASELINE.json configuration, at full size.

Each case starts the device engine and the CPU oracle from the SAME dumped
initial state: ``random_init`` (init.cpp:496-521, as the reference's own
benchmark does, bench.cpp:83-88) is written once as an FMNM v2 container by
the oracle's independent writer (oracle/fmnm.py, io.cpp:49-82) and read back
by the product's native reader (csrc/dfm_io.cpp) for the device and by the
oracle's reader for the CPU run.  The observations are the seeded BASELINE
generator (bit-exact between oracle and product, tests/test_capi_host.py).

Bar (BASELINE.json north_star):
  * cost (negative log-likelihood) trajectory within 1e-8 relative over the
    first 20 iterations,
  * cost non-increase every iteration (1e-9 relative slack, as the
    reference's tests allow: test_fastmnmf.cpp:315-349),
  * final separated STFTs (Wiener images, wiener.cpp:50-69) within 1e-6
    relative L2 of the oracle's images of the oracle's fit.

Parity with the reference itself is pinned through the oracle, which is
checked against the reference's known-answer tests (tests/test_oracle.py);
bitwise agreement with Eigen's GEMM/LU/COD is not pinnable here (Eigen is
absent and no reference test fixes it).
"""
import os

import numpy as np
import pytest

pytestmark = [pytest.mark.gpu, pytest.mark.slow]

TRAJ_RTOL = 1e-8
IMG_RTOL = 1e-6


@pytest.fixture(scope="module")
def dfm():
    import torch

    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    import paper_2605_19388_b200 as m

    m._capi.load()
    return m


def _rel(a, b):
    return np.linalg.norm(np.asarray(a) - np.asarray(b)) / max(np.linalg.norm(np.asarray(b)), 1e-300)


def _dumped_init(dfm, oracle, tmp_path, c, seed_init, tag):
    """random_init -> FMNM v2 (oracle writer) -> (product InitBundle, oracle dict)."""
    import fmnm

    F, T, N, K, sizes = c["F"], c["T"], c["N"], c["K"], c["sizes"]
    r = oracle.random_init(F, T, sizes, N, K, seed_init)
    path = str(tmp_path / f"init_{tag}.fmnm")
    cfg = dict(k_bases=K, floor=1e-6, seed=seed_init, sample_rate=16000.0, window_len=2 * (F - 1),
               hop_len=(F - 1) // 2, iterations=c["iters"])
    fmnm.write(path, cfg, sizes, True, [(r["T"], r["V"])], r["lam"], r["w"])
    dump = dfm.container.load_model(path)
    assert dump.layout.sizes == list(sizes) and dump.shared
    init = dump.init_bundle()
    _, osizes, _, models, lam, w = fmnm.read(path)
    ref_init = dict(T=models[0][0], V=models[0][1], lam=lam, w=w)
    # the two readers agree bit for bit on the dumped state
    assert np.array_equal(init.nmf.T, ref_init["T"]) and np.array_equal(init.nmf.V, ref_init["V"])
    assert np.array_equal(init.lambda0, ref_init["lam"])
    assert all(np.array_equal(a, b) for a, b in zip(init.w0, ref_init["w"]))
    return init, ref_init


def _bin_subset(model_like, sel):
    return dict(T=np.ascontiguousarray(model_like["T"][:, sel]), V=model_like["V"],
                lam=np.ascontiguousarray(model_like["lam"][sel]),
                w=[np.ascontiguousarray(w[sel]) for w in model_like["w"]])


def _check_fit(dfm, oracle, x, c, cost, model, ref, wiener_bins=None):
    """model: dict(T, V, lam, w) of the device fit; ref: the oracle's run_engine result."""
    r = ref["cost_trace"]
    n = min(21, len(r))
    rel = np.max(np.abs(cost[:n] - r[:n]) / np.abs(r[:n]))
    assert rel < TRAJ_RTOL, f"trajectory {rel:.3e} over the first {n - 1} iterations"
    assert np.all(cost[1:] <= cost[:-1] + 1e-9 * np.abs(cost[:-1])), "cost increased"
    sizes = c["sizes"]
    sel = slice(None) if wiener_bins is None else wiener_bins
    xs = np.ascontiguousarray(x[sel])
    mine = _bin_subset(model, sel)
    layout = dfm.BlockLayout(sizes)
    img = dfm.wiener_block(xs, [dfm.NmfModel(mine["T"], mine["V"])],
                           dfm.BlockSpatialModel(layout, mine["w"], mine["lam"])).images
    ref_img = oracle.wiener_block(xs, sizes, _bin_subset(ref, sel))
    e = _rel(img, ref_img)
    assert e < IMG_RTOL, f"separated STFTs {e:.3e}"
    assert np.linalg.norm(img.sum(0) - xs) <= 1e-9 * np.linalg.norm(xs)
    return rel, e


def _fit_device(dfm, x, c, init, iters):
    layout = dfm.BlockLayout(c["sizes"])
    fit = dfm.fit_distributed(x, layout, init, iters, True)
    model = dict(T=fit.models[0].T, V=fit.models[0].V, lam=fit.spatial.Lambda, w=list(fit.spatial.W))
    return fit.report.cost_trace, model, fit.report


@pytest.mark.parametrize("workload,iters,wiener_stride", [
    ("config0", 50, None),    # B=2 x 2 mics, N=3, F=257, T=200, K=4: its own 50 iterations
    ("config1", 200, None),   # B=3 x 4, N=5, F=513, T=626, K=16: 200 iterations
    ("config2", 200, None),   # the same mixture as one 12 x 12 block: 200 iterations
    ("config3", 20, 8),       # B=8 x 4, N=8, F=1025, T=2000, K=32: 20 iterations; Wiener on every 8th bin
])
def test_baseline_config_parity_from_dumped_init(dfm, oracle, tmp_path, workload, iters, wiener_stride):
    import bench

    oracle.set_threads(os.cpu_count() or 1)
    c = bench.CONFIGS[workload]
    M = sum(c["sizes"])
    x = oracle.generate_mixture(c["kind"], c["F"], c["T"], M, c["N"], c["K"], bench.SEED_X)
    init, ref_init = _dumped_init(dfm, oracle, tmp_path, c, bench.SEED_INIT, workload)
    cost, model, report = _fit_device(dfm, x, c, init, iters)
    ref = oracle.run_engine(x, c["sizes"], ref_init, iters)
    assert report.fallbacks == ref["fallbacks"]
    sel = None if wiener_stride is None else np.arange(0, c["F"], wiener_stride)
    rel, e = _check_fit(dfm, oracle, x, c, cost, model, ref, sel)
    print(f"{workload}: trajectory {rel:.2e}, separated STFTs {e:.2e}")


def test_baseline_config4_mixtures_through_fit_many(dfm, oracle, tmp_path):
    """Config 4 (independent config-1-shape mixtures, each from its own seed,
    100 iterations) through the batch path dfm_fit_many: every mixture meets
    the same bar as a single fit."""
    import bench

    oracle.set_threads(os.cpu_count() or 1)
    c = bench.CONFIGS["config4"]
    F, T, N, K, sizes, iters = c["F"], c["T"], c["N"], c["K"], c["sizes"], c["iters"]
    layout = dfm.BlockLayout(sizes)
    engines, cases = [], []
    for j in range(2):
        x = oracle.generate_mixture(c["kind"], F, T, sum(sizes), N, K, bench.SEED_X + j)
        init, ref_init = _dumped_init(dfm, oracle, tmp_path, c, bench.SEED_INIT + j, f"c4_{j}")
        e = dfm.Engine(F, T, layout, N, K)
        e.set_obs(x)
        e.set_model(init.nmf, init.w0, init.lambda0)
        engines.append(e)
        cases.append((x, ref_init))
    costs, secs, fb = dfm.fit_many(engines, iters)
    assert secs > 0
    for e, cst, (x, ref_init) in zip(engines, costs, cases):
        nmf, w, lam = e.get_model()
        ref = oracle.run_engine(x, sizes, ref_init, iters)
        _check_fit(dfm, oracle, x, c, cst, dict(T=nmf.T, V=nmf.V, lam=lam, w=w), ref)
        e.close()
