"""Device time of the Wiener separation (dfm_bench_wiener) for a BASELINE
workload after a short fit: python tools/wiener_bench.py [config1]"""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2605_19388_b200 as dfm  # noqa: E402

w = sys.argv[1] if len(sys.argv) > 1 else "config1"
c = bench.CONFIGS[w]
layout = dfm.BlockLayout(c["sizes"])
x = dfm.generate_mixture(c["kind"], c["F"], c["T"], layout.total, c["N"], c["K"], bench.SEED_X)
init = dfm.random_init(c["F"], c["T"], layout, c["N"], c["K"], bench.SEED_INIT)
eng = dfm.Engine(c["F"], c["T"], layout, c["N"], c["K"])
eng.set_obs(x)
eng.set_model(init.nmf, init.w0, init.lambda0)
eng.fit(2)
v = ctypes.c_double()
for _ in range(4):
    dfm._capi.check(eng.lib.dfm_l2_flush(0))
    dfm._capi.check(eng.lib.dfm_bench_wiener(eng.ctx, ctypes.byref(v)))
    print(f"wiener {w}: {v.value * 1e3:.1f} us")
