"""Device time per mixture-iteration of a batch of independent config-1
mixtures (dfm_bench_step_many: one graph replay per context, each on its own
stream) against the batch size.

  python tools/batch_scaling.py [sizes...]   default 1 2 4 8 16 64"""
import ctypes
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2605_19388_b200 as dfm  # noqa: E402

sizes = [int(v) for v in sys.argv[1:]] or [1, 2, 4, 8, 16, 64]
c = bench.CONFIGS["config1"]
layout = dfm.BlockLayout(c["sizes"])
F, T, N, K = c["F"], c["T"], c["N"], c["K"]
engines = []
for j in range(max(sizes)):
    x = dfm.generate_mixture(c["kind"], F, T, layout.total, N, K, bench.SEED_X + j)
    init = dfm.random_init(F, T, layout, N, K, bench.SEED_INIT + j)
    e = dfm.Engine(F, T, layout, N, K)
    e.set_obs(x)
    e.set_model(init.nmf, init.w0, init.lambda0)
    dfm._capi.check(e.lib.dfm_prime(e.ctx))
    engines.append(e)
lib = engines[0].lib
for b in sizes:
    arr = (ctypes.c_void_p * b)(*[e.ctx for e in engines[:b]])
    ms = []
    for i in range(8):
        dfm._capi.check(lib.dfm_l2_flush(0))
        v = ctypes.c_double()
        dfm._capi.check(lib.dfm_bench_step_many(arr, b, ctypes.byref(v)))
        if i >= 3:
            ms.append(v.value)
    m = float(np.median(ms))
    print(f"batch {b:3d}: {m:8.3f} ms per step, {1e3 * m / b:7.1f} us per mixture-iteration, "
          f"{b * F * T / (m * 1e-3):.3e} TF-bin*iter/s")
