import sys, numpy as np
sys.path.insert(0, '.'); sys.path.insert(0, 'oracle')
import paper_2605_19388_b200 as dfm, oracle
F, T, sizes, N, K, iters = 4, 30, [12], 5, 16, 4
layout = dfm.BlockLayout(sizes)
x = dfm.generate_mixture(1, F, T, layout.total, N, K, 3)
init = dfm.random_init(F, T, layout, N, K, 5)
ref = oracle.run_engine(x, sizes, dict(T=init.nmf.T, V=init.nmf.V, lam=init.lambda0, w=init.w0), iters)
print("ref", ref["cost_trace"])
for gen in (0, 1):
    for ft in (32, 128):
        with dfm.Engine(F, T, layout, N, K) as eng:
            dfm._capi.check(eng.lib.dfm_force_generic(eng.ctx, gen))
            eng.set_tiling(ft, 0)
            eng.set_obs(x); eng.set_model(init.nmf, init.w0, init.lambda0)
            c, _, _, fb = eng.fit(iters)
            print("generic", gen, "FT", ft, eng.tiling(), c, fb)
