"""Per-GPU EM step time of a frequency shard of a BASELINE workload, on one
GPU (the compute part of an N-GPU run; no collective):

  python tools/shard_bench.py [config1] [shards...]   e.g. 1 2 4 8
  DFM_COLLECTIVE=1 python tools/shard_bench.py ...     with the NCCL path on a
                                                       one-rank communicator"""
import ctypes
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2605_19388_b200 as dfm  # noqa: E402
from paper_2605_19388_b200.sharding import shard_bins  # noqa: E402

w = sys.argv[1] if len(sys.argv) > 1 else "config1"
shards = [int(v) for v in sys.argv[2:]] or [1, 2, 4, 8]
c = bench.CONFIGS[w]
layout = dfm.BlockLayout(c["sizes"])
F, T, N, K = c["F"], c["T"], c["N"], c["K"]
x = dfm.generate_mixture(c["kind"], F, T, layout.total, N, K, bench.SEED_X)
init = dfm.random_init(F, T, layout, N, K, bench.SEED_INIT)
for S in shards:
    f0, f1 = shard_bins(F, S, 0)
    eng = dfm.Engine(F, T, layout, N, K, f_begin=f0, f_end=f1)
    if os.environ.get("DFM_COLLECTIVE"):
        buf = ctypes.create_string_buffer(128)
        dfm._capi.check(eng.lib.dfm_nccl_get_unique_id(buf))
        eng.comm_init(buf.raw, 1, 0)
        dfm._capi.check(eng.lib.dfm_force_collective(eng.ctx, 1))
    eng.set_obs(np.ascontiguousarray(x[f0:f1]))
    eng.set_model(init.nmf, init.w0, init.lambda0)
    lib = eng.lib
    dfm._capi.check(lib.dfm_prime(eng.ctx))
    ms = []
    for i in range(30):
        dfm._capi.check(lib.dfm_l2_flush(0))
        dfm._capi.check(lib.dfm_bench_step(eng.ctx))
        if i >= 5:
            ms.append(lib.dfm_bench_last_ms(eng.ctx))
    sp = (ctypes.c_double * 5)()
    dfm._capi.check(lib.dfm_bench_split_step(eng.ctx))
    lib.dfm_bench_last_split(eng.ctx, sp)
    print(f"{w} shard 1/{S}: {f1 - f0} bins, tiling {eng.tiling()['frame_tile']}, step {np.median(ms):.4f} ms, "
          f"split {[round(v, 4) for v in sp]}")
    eng.close()
