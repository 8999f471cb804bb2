"""Per-kernel device times of one config's steady-state EM iteration
(stream-launched with events between the kernels), optionally under timing
experiments (dfm_debug_bits; results invalid):
  bit 0 no Lambda reduction, bit 1 no Q accumulation (k_em_bin),
  bit 2 no fused H = T V epilogues (k_tupd, k_vupd).

  python tools/split_bench.py [--workload config1] [--dbg BITS] [--steps 30]"""
import argparse
import ctypes
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="config1")
    ap.add_argument("--dbg", type=int, default=0)
    ap.add_argument("--steps", type=int, default=30)
    ap.add_argument("--tiling", default="", help="FT,TB (dfm_set_tiling)")
    args = ap.parse_args()
    import bench
    import paper_2605_19388_b200 as dfm

    lib = dfm._capi.load()
    c = bench.CONFIGS[args.workload]
    layout = dfm.BlockLayout(c["sizes"])
    x = dfm.generate_mixture(c["kind"], c["F"], c["T"], layout.total, c["N"], c["K"], bench.SEED_X)
    init = dfm.random_init(c["F"], c["T"], layout, c["N"], c["K"], bench.SEED_INIT)
    eng = dfm.Engine(c["F"], c["T"], layout, c["N"], c["K"])
    eng.set_obs(x)
    eng.set_model(init.nmf, init.w0, init.lambda0)
    if args.tiling:
        ft, tb = (int(v) for v in args.tiling.split(","))
        dfm._capi.check(lib.dfm_set_tiling(eng.ctx, ft, tb))
    dfm._capi.check(lib.dfm_prime(eng.ctx))
    if args.dbg:
        dfm._capi.check(lib.dfm_debug_bits(eng.ctx, args.dbg))
    rows, graph = [], []
    for i in range(args.steps + 3):
        dfm._capi.check(lib.dfm_l2_flush(0))
        dfm._capi.check(lib.dfm_bench_split_step(eng.ctx))
        sp = (ctypes.c_double * 5)()
        dfm._capi.check(lib.dfm_bench_last_split(eng.ctx, sp))
        if i >= 3:
            rows.append(list(sp))
        dfm._capi.check(lib.dfm_l2_flush(0))
        dfm._capi.check(lib.dfm_bench_step(eng.ctx))
        if i >= 3:
            graph.append(lib.dfm_bench_last_ms(eng.ctx))
    m = np.mean(np.array(rows), axis=0)
    out = {"workload": args.workload, "dbg": args.dbg, "graph_step_ms": float(np.mean(graph)),
           "split_ms": dict(zip(["k_em_bin", "k_tupd+h", "k_pdw", "k_vupd+H", "tail"], map(float, m)))}
    print(json.dumps(out))
    eng.close()


if __name__ == "__main__":
    main()
