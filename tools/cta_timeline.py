"""Per-CTA timelines of the EM step kernels (dfm_cta_trace): for each kernel
kind the launch span, the CTA durations (min / median / max), how many CTAs
each SM ran, and when the last CTA started -- separates per-CTA latency from
waves, imbalance and launch ramp.

  python tools/cta_timeline.py [--workload config1] [--steps 5]"""
import argparse
import ctypes
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
KINDS = {0: "k_tupd", 1: "k_pdw(setup)", 2: "k_vupd", 3: "k_em_bin"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="config1")
    ap.add_argument("--steps", type=int, default=5)
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
    dfm._capi.check(lib.dfm_prime(eng.ctx))
    cap = 1 << 16
    for k in KINDS:
        dfm._capi.check(lib.dfm_cta_trace(eng.ctx, k, cap, None))
    out = {}
    for i in range(args.steps):
        dfm._capi.check(lib.dfm_l2_flush(0))
        dfm._capi.check(lib.dfm_bench_step(eng.ctx))
    buf = np.zeros(3 * cap, dtype=np.uint64)
    t_first = None
    for k, name in KINDS.items():
        n = lib.dfm_cta_trace(eng.ctx, k, cap, buf.ctypes.data_as(ctypes.c_void_p))
        r = buf[:3 * n].reshape(n, 3).astype(np.int64)
        r = r[r[:, 1] > 0]
        if not len(r):
            continue
        t0 = r[:, 0].min()
        d = (r[:, 1] - r[:, 0]) / 1e3
        per_sm = np.bincount(r[:, 2].astype(int))
        out[name] = {"ctas": int(len(r)), "span_us": float((r[:, 1].max() - t0) / 1e3),
                     "cta_us_min_med_max": [float(d.min()), float(np.median(d)), float(d.max())],
                     "last_start_us": float((r[:, 0].max() - t0) / 1e3),
                     "first_end_us": float((r[:, 1].min() - t0) / 1e3),
                     "ctas_per_sm_max": int(per_sm.max()), "sms_used": int((per_sm > 0).sum()),
                     "start_abs": int(t0)}
    base = min(v["start_abs"] for v in out.values())
    for v in out.values():
        v["start_us"] = (v.pop("start_abs") - base) / 1e3
    print(json.dumps({"workload": args.workload, "kernels": out}, indent=1))
    eng.close()


if __name__ == "__main__":
    main()
