"""Stage timings of the device initialisation pipeline (init_distributed) for
a BASELINE workload: python tools/init_timing.py [config1]"""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2605_19388_b200 as dfm  # noqa: E402
from paper_2605_19388_b200 import init as di  # noqa: E402

w = sys.argv[1] if len(sys.argv) > 1 else "config1"
c = bench.CONFIGS[w]
layout = dfm.BlockLayout(c["sizes"])
x = dfm.generate_mixture(c["kind"], c["F"], c["T"], layout.total, c["N"], c["K"], bench.SEED_X)
di.init_distributed(x[:8], layout, di.InitConfig(c["N"], c["K"], 5), 1)  # warm-up


def tick(label, fn):
    t = time.perf_counter()
    r = fn()
    print(f"{label:40s} {1e3 * (time.perf_counter() - t):8.1f} ms")
    return r


b = tick("init_distributed (1000 IS-NMF iters)", lambda: di.init_distributed(x, layout, di.InitConfig(c["N"], c["K"], 1000), 19388))
o = 0
masks = []
for l, mb in enumerate(c["sizes"]):
    xb = np.ascontiguousarray(x[:, :, o:o + mb])
    masks.append(tick(f"cluster_masks block {l} (k-means + align)", lambda: di.cluster_masks(xb, c["N"], 7 + l)))
    o += mb
tick("align_subarray_permutations", lambda: di.align_subarray_permutations(masks))
R, h0 = tick("masked SCM + ML spectrograms", lambda: di._scm_spec(x, c["sizes"], masks))
tr = []
tick("IS-NMF (1000 iters max)", lambda: di.itakura_saito_nmf(h0, c["K"], 1000, 7, tr))
print("  IS-NMF iterations run:", [len(v) - 1 for v in tr])
tick("init_spatial (GEVD)", lambda: di.init_spatial(R, layout))
