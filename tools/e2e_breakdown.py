"""Host-side breakdown of bench.py's e2e step (config 1): pinned X in,
model in, fit(20), model out."""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2605_19388_b200 as dfm  # noqa: E402

c = bench.CONFIGS["config1"]
layout = dfm.BlockLayout(c["sizes"])
x = dfm.generate_mixture(1, c["F"], c["T"], 12, c["N"], c["K"], bench.SEED_X)
init = dfm.random_init(c["F"], c["T"], layout, c["N"], c["K"], bench.SEED_INIT)
xs = torch.from_numpy(np.ascontiguousarray(x)).pin_memory().numpy()
eng = dfm.Engine(c["F"], c["T"], layout, c["N"], c["K"])
for rep in range(4):
    t = [time.perf_counter()]
    eng.set_obs(xs); t.append(time.perf_counter())
    eng.set_model(init.nmf, init.w0, init.lambda0); t.append(time.perf_counter())
    eng.fit(200); t.append(time.perf_counter())
    eng.get_model(); t.append(time.perf_counter())
    d = np.diff(t) * 1e3
    print(f"set_obs {d[0]:.2f} ms ({xs.nbytes / d[0] / 1e6:.1f} GB/s)  set_model {d[1]:.2f}  fit(200) {d[2]:.2f}  "
          f"get_model {d[3]:.2f}  total {sum(d):.2f} ms")
