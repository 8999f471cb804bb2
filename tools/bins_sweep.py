"""k_em_bin time against the number of bins (config-1 shape, 128-frame
tiles): how the kernel scales with bins per SM (148 SMs, 4 CTAs per SM).

  python tools/bins_sweep.py [bins ...] [--no-flush]"""
import ctypes
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import bench
    import paper_2605_19388_b200 as dfm

    c = bench.CONFIGS["config1"]
    layout = dfm.BlockLayout(c["sizes"])
    F, T, N, K = c["F"], c["T"], c["N"], c["K"]
    x = dfm.generate_mixture(c["kind"], F, T, layout.total, N, K, bench.SEED_X)
    init = dfm.random_init(F, T, layout, N, K, bench.SEED_INIT)
    flush = "--no-flush" not in sys.argv
    sweep = [int(v) for v in sys.argv[1:] if not v.startswith("--")] or [148, 296, 444, 481, 513]
    out = {}
    for nb in sweep:
        eng = dfm.Engine(F, T, layout, N, K, f_begin=0, f_end=nb)
        eng.set_tiling(128, 128)
        eng.set_obs(np.ascontiguousarray(x[:nb]))
        eng.set_model(init.nmf, init.w0, init.lambda0)
        lib = eng.lib
        dfm._capi.check(lib.dfm_prime(eng.ctx))
        for _ in range(3):
            dfm._capi.check(lib.dfm_bench_step(eng.ctx))
        sp = (ctypes.c_double * 5)()
        acc = np.zeros(5)
        for _ in range(10):
            if flush:
                dfm._capi.check(lib.dfm_l2_flush(0))
            dfm._capi.check(lib.dfm_bench_split_step(eng.ctx))
            lib.dfm_bench_last_split(eng.ctx, sp)
            acc += np.array(list(sp))
        out[nb] = [round(v / 10, 4) for v in acc]
        eng.close()
    print(json.dumps({"kernels_ms [em_bin, tupd, pdw, vupd, tail]": out}, indent=1))


if __name__ == "__main__":
    main()
