"""Phase breakdown of the fused bin kernel from its %globaltimer stamps.

  python tools/trace_bin.py [--workload config1] [--tiling G,CS]

Runs one steady-state EM step of the chosen BASELINE config with per-CTA
tracing on and prints, per phase, the mean/max duration over CTAs, the CTA
lifetime and how the CTAs spread over the kernel's span (waves)."""
import argparse
import ctypes
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

PHASES = ["A:lambda (tiles + reduce)", "B:cost+Q (tiles)", "B:Q-reduce", "IP", "C:T-weights"]


def main():
    import bench
    import paper_2605_19388_b200 as dfm

    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="config1")
    ap.add_argument("--tiling", default="")
    ap.add_argument("--generic", action="store_true")
    ap.add_argument("--no-flush", action="store_true")
    ap.add_argument("--dbg", type=int, default=0, help="timing experiments (results invalid)")
    ap.add_argument("--shards", type=int, default=1, help="trace the first of S frequency shards")
    args = ap.parse_args()
    c = bench.CONFIGS[args.workload]
    layout = dfm.BlockLayout(c["sizes"])
    F, T, N, K = c["F"], c["T"], c["N"], c["K"]
    x = dfm.generate_mixture(c["kind"], F, T, layout.total, N, K, bench.SEED_X)
    init = dfm.random_init(F, T, layout, N, K, bench.SEED_INIT)
    from paper_2605_19388_b200.sharding import shard_bins

    f0, f1 = shard_bins(F, args.shards, 0)
    x = np.ascontiguousarray(x[f0:f1])
    eng = dfm.Engine(F, T, layout, N, K, f_begin=f0, f_end=f1)
    lib = eng.lib
    if args.generic:
        dfm._capi.check(lib.dfm_force_generic(eng.ctx, 1))
    if args.tiling:
        ft, tb = (int(v) for v in args.tiling.split(","))
        eng.set_tiling(ft, tb)
    if args.dbg:
        dfm._capi.check(lib.dfm_debug_bits(eng.ctx, args.dbg))
    eng.set_obs(x)
    eng.set_model(init.nmf, init.w0, init.lambda0)
    dfm._capi.check(lib.dfm_prime(eng.ctx))
    for _ in range(3):
        dfm._capi.check(lib.dfm_bench_step(eng.ctx))
    n = dfm._capi.check(lib.dfm_set_trace(eng.ctx, 1))
    if not args.no_flush:
        dfm._capi.check(lib.dfm_l2_flush(0))
    dfm._capi.check(lib.dfm_bench_split_step(eng.ctx))
    ms = lib.dfm_bench_last_ms(eng.ctx)
    sp = (ctypes.c_double * 5)()
    lib.dfm_bench_last_split(eng.ctx, sp)
    buf = np.zeros(n, dtype=np.uint64)
    dfm._capi.check(lib.dfm_get_trace(eng.ctx, buf.ctypes.data_as(ctypes.c_void_p), n))
    tr = buf.reshape(-1, 16)[:, :6].astype(np.int64)
    t0 = tr[:, 0].min()
    tr = tr - t0
    d = np.diff(tr, axis=1) / 1e3  # us
    life = (tr[:, 5] - tr[:, 0]) / 1e3
    out = {"workload": args.workload, "tiling": eng.tiling(), "step_ms": ms,
           "kernels_ms": dict(zip(["k_em_bin", "k_tupd+h", "k_pdw", "k_vupd+H", "tail"], [round(v, 4) for v in sp])),
           "ctas": int(tr.shape[0]),
           "span_us": float(tr[:, 5].max() / 1e3), "cta_life_us_mean": float(life.mean()),
           "cta_life_us_max": float(life.max()),
           "phases_us_mean": {p: round(float(d[:, i].mean()), 3) for i, p in enumerate(PHASES)},
           "phases_us_max": {p: round(float(d[:, i].max()), 3) for i, p in enumerate(PHASES)}}
    starts = np.sort(tr[:, 0]) / 1e3
    chol = (buf.reshape(-1, 16)[:, 6].astype(np.int64) - t0 - tr[:, 3]) / 1e3
    if (buf.reshape(-1, 16)[:, 6] > 0).all():
        out["ip_cholesky_us_mean"] = round(float(chol.mean()), 3)
    cyc = buf.reshape(-1, 16)[:, 8].astype(np.float64)
    if cyc.max() > 0:
        out["ip_sweep_cycles_block0_mean"] = float(cyc.mean())
    slow = buf.reshape(-1, 16)[:, 7]
    out["ip_slow_path_blocks"] = int(slow.sum())
    out["ip_slow_path_bins"] = int((slow > 0).sum())
    out["start_percentiles_us"] = [round(float(np.percentile(starts, q)), 1) for q in (0, 10, 25, 50, 75, 90, 100)]
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
