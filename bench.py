#!/usr/bin/env python
"""Benchmark of the B200-native distributed-FastMNMF EM iteration.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference]
                  [--workload config1|config0|config2|config3|config4] [--e2e-iters I]

A *step* is one steady-state EM iteration of BASELINE.json's config 1
(B=3 subarrays x M_b=4 mics, N=5 sources, F=513 bins, T=626 frames, K=16):
the fused bin kernel (finishes iteration i-1: Lambda update + cost; starts
iteration i: IP sweep, decorrelation, T update, V-update weights) followed by
the cross-bin V update.  Inputs are resident in HBM; X (61.7 MB) fits in the
126 MB L2, so L2 is FLUSHED (384 MB write, untimed) before every timed step.
Timing: CUDA events on the engine stream, summed over exactly K steps,
barrier + synchronize on both sides, max over ranks.

N > 1 (torchrun): frequency bins sharded over the ranks, one NCCL allreduce of
the V-update numerator/denominator per iteration (strong scaling).

--workload config4: 64 independent config-1 mixtures (seeds SEED_X + j,
SEED_INIT + j), mixtures sharded over the ranks with no communication; a step
is one EM iteration of every local mixture (one context per mixture, each on
its own stream, kernels of different mixtures overlapping).  The 64 contexts'
working sets (8.4 GB) exceed L2, so no flush is needed between steps.

--impl reference: the reference's CPU algorithm (oracle/ restatement; the
reference itself needs Eigen, absent here) on all host cores, rank 0 only.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CONFIGS = {
    "config0": dict(kind=0, F=257, T=200, sizes=[2, 2], N=3, K=4, iters=50),
    "config1": dict(kind=1, F=513, T=626, sizes=[4, 4, 4], N=5, K=16, iters=200),
    "config2": dict(kind=1, F=513, T=626, sizes=[12], N=5, K=16, iters=200),
    "config3": dict(kind=1, F=1025, T=2000, sizes=[4] * 8, N=8, K=32, iters=100),
    # 64 independent config-1 mixtures, each from its own seed, sharded over GPUs
    "config4": dict(kind=1, F=513, T=626, sizes=[4, 4, 4], N=5, K=16, iters=100, batch=64),
}
SEED_X, SEED_INIT = 2605, 19388
PAPER_CPU_TFBIN = 266.5e3  # BASELINE.md derived paper figure (other config/hardware), context only


def alg_bytes(c) -> float:
    """SURVEY.md §8(d) compulsory bytes per EM iteration."""
    F, T, N, K, M = c["F"], c["T"], c["N"], c["K"], sum(c["sizes"])
    S2 = sum(s * s for s in c["sizes"])
    return 16.0 * F * T * M + 2 * 8.0 * (F * K * N + K * T * N + F * N * M) + 2 * 16.0 * F * S2 + 32.0 * N * K * T


def alg_bytes_bin_kernel(c) -> float:
    """Compulsory bytes of the per-bin kernel k_em_bin: X once, Lambda and W
    read and written (its other traffic - H, the T-update weights, X re-reads
    from L2 - is intermediate, not algorithmic)."""
    F, T, N, K, M = c["F"], c["T"], c["N"], c["K"], sum(c["sizes"])
    S2 = sum(s * s for s in c["sizes"])
    return 16.0 * F * T * M + 16.0 * F * N * M + 32.0 * F * S2


def alg_flops(c) -> float:
    """SURVEY.md §8(d) algorithmic flops per EM iteration (FMA = 2)."""
    F, T, N, K, M = c["F"], c["T"], c["N"], c["K"], sum(c["sizes"])
    S2 = sum(s * s for s in c["sizes"])
    FTM = F * T * M
    f = F * T * sum(2 * m ** 3 + 5 * m ** 2 + 3 * m for m in c["sizes"])
    f += F * sum(m * (32.0 / 3 * m ** 3 + 24 * m ** 2) for m in c["sizes"])
    f += 8.0 * F * T * S2 + 3 * FTM
    f += 2.0 * F * T * (4 * N * M + 3 * M)
    f += 8.0 * N * F * K * T
    f += 4.0 * N * F * T * K
    f += 3 * (2.0 * F * T * N * M + FTM)
    f += 4.0 * F * T * N * M + 3 * FTM
    f += 4.0 * FTM
    return f


def peaks():
    p = dict(hbm_gbs=6540.5, source="fallback (MEASURED_PEAKS.json absent)")
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(path):
        with open(path) as fh:
            j = json.load(fh)
        p = dict(hbm_gbs=float(j["hbm_gbs"]), source="measured (MEASURED_PEAKS.json)")
    return p


class ClockSampler:
    """Samples SM clocks and throttle reasons via NVML during the timed region."""

    def __init__(self, device: int, period_s: float = 0.0005):
        self.device, self.period, self.samples, self.reasons = device, period_s, [], set()
        self.sample_now = lambda: None
        self.max_mhz = None
        self._stop = threading.Event()
        self._t = None

    def start(self):
        try:
            import pynvml as nv

            nv.nvmlInit()
            h = nv.nvmlDeviceGetHandleByIndex(self.device)
            self.max_mhz = nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM)
            names = {
                getattr(nv, "nvmlClocksEventReasonHwSlowdown", 0x8): "hw_slowdown",
                getattr(nv, "nvmlClocksEventReasonHwThermalSlowdown", 0x40): "hw_thermal_slowdown",
                getattr(nv, "nvmlClocksEventReasonSwThermalSlowdown", 0x20): "sw_thermal_slowdown",
                getattr(nv, "nvmlClocksEventReasonSwPowerCap", 0x4): "sw_power_cap",
                getattr(nv, "nvmlClocksEventReasonHwPowerBrakeSlowdown", 0x80): "hw_power_brake",
            }

            def once():
                try:
                    self.samples.append(nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM))
                    r = nv.nvmlDeviceGetCurrentClocksEventReasons(h)
                    for bit, name in names.items():
                        if r & bit:
                            self.reasons.add(name)
                except Exception:
                    pass

            self.sample_now = once  # also called by the timing loop itself (short regions)

            def run():
                while not self._stop.is_set():
                    once()
                    time.sleep(self.period)

            self._t = threading.Thread(target=run, daemon=True)
            self._t.start()
        except Exception as e:  # NVML unavailable: record why
            self.reasons.add(f"nvml_unavailable:{type(e).__name__}")
        return self

    def stop(self):
        self._stop.set()
        if self._t:
            self._t.join(timeout=1)
        med = statistics.median(self.samples) if self.samples else None
        return {"sm_mhz": med, "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons),
                "samples": len(self.samples)}


def pinned_copy(a: np.ndarray) -> np.ndarray:
    """A numpy view of page-locked host memory holding a copy of `a` (the
    caller's input buffer for the e2e measurement: H2D from pinned memory)."""
    import torch

    t = torch.empty(a.shape, dtype=torch.complex128 if np.iscomplexobj(a) else torch.float64, pin_memory=True)
    out = t.numpy()
    out[...] = a  # the view's base is the tensor, which keeps the pinned storage alive
    return out


def dist_setup():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def shard(F: int, world: int, rank: int):
    from paper_2605_19388_b200.sharding import shard_bins

    return shard_bins(F, world, rank)


def host_cpu() -> dict:
    """nproc and the CPU model of this host (BASELINE.md CPU baseline plan)."""
    model = "unknown"
    try:
        with open("/proc/cpuinfo") as fh:
            for line in fh:
                if line.startswith("model name"):
                    model = line.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    try:
        usable = len(os.sched_getaffinity(0))
    except AttributeError:
        usable = os.cpu_count() or 1
    return {"nproc": usable, "cpu_count": os.cpu_count() or 1, "model": model}


def cpu_protocol(workload: str, threads: int, steps: int, warmup: int, budget_s: float, mixture: int = 0) -> dict:
    """The reference's CPU algorithm (oracle/ C restatement of engine.cpp;
    the reference itself needs Eigen3, absent here) timed with the
    reference's protocol (bench.cpp:31-71): one untimed warm-up run, then the
    timed EM iterations split into repeats of >= 5 iterations (every repeat an
    independent run from the same dumped start, the per-iteration cost
    evaluation included as in engine.cpp:253), reported as mean +- SE over
    the repeats.  The sample is the first Fs bins of the workload's own
    mixture (every frame), Fs sized so the whole run fits `budget_s`.
    Inputs come from the oracle's restatement of the BASELINE generator and
    of random_init only: this process never loads the product library."""
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import oracle

    oracle.build()
    c = CONFIGS[workload]
    F, T, N, K, sizes = c["F"], c["T"], c["N"], c["K"], c["sizes"]
    oracle.set_threads(max(1, min(threads, 64)))
    x = oracle.generate_mixture(c["kind"], F, T, sum(sizes), N, K, SEED_X + mixture)
    init = oracle.random_init(F, T, sizes, N, K, SEED_INIT + mixture)
    sub = lambda Fs: dict(T=np.ascontiguousarray(init["T"][:, :Fs]), V=init["V"],
                          lam=np.ascontiguousarray(init["lam"][:Fs]),
                          w=[np.ascontiguousarray(w[:Fs]) for w in init["w"]])
    oracle.set_threads(threads)
    Fp = min(F, max(8, threads))
    r = oracle.run_engine(np.ascontiguousarray(x[:Fp]), sizes, sub(Fp), 1)
    per_bin_iter = max(float(np.sum(r["wall_seconds"])) / Fp, 1e-9)
    Fs = int(max(min(F, 8), min(F, budget_s / ((steps + max(warmup, 1)) * per_bin_iter))))
    xs = np.ascontiguousarray(x[:Fs])
    oracle.run_engine(xs, sizes, sub(Fs), max(warmup, 1))  # untimed warm-up run
    nrep = max(1, steps // 5)
    lens = [5] * (nrep - 1) + [steps - 5 * (nrep - 1)]
    per_rep, total = [], 0.0
    for it in lens:
        rr = oracle.run_engine(xs, sizes, sub(Fs), it)
        t = float(np.sum(rr["wall_seconds"]))
        total += t
        per_rep.append(Fs * T * it / t)
    mean = float(np.mean(per_rep))
    se = float(np.std(per_rep, ddof=1) / np.sqrt(len(per_rep))) if len(per_rep) > 1 else 0.0
    return {"value": Fs * T * steps / total, "unit": "TF-bin*iter/s", "mean": mean, "se": se,
            "repeats": len(per_rep), "iters_per_repeat": lens, "per_repeat": per_rep, "cores": threads,
            "kind": "port", "seconds_per_iter_sample": total / steps, "seconds_per_iter_full": total / steps * F / Fs,
            "sample": (f"oracle/ run_engine (C restatement of engine.cpp, OpenMP over bins) on the first {Fs} of {F} "
                       f"bins x {T} frames of the {workload} mixture; 1 warm-up run of {max(warmup, 1)} iteration(s), "
                       f"then {steps} timed iterations in {len(per_rep)} repeats; mean +- SE over the repeats"),
            "host": host_cpu()}


def cpu_protocol_subprocess(workload: str, threads: int, steps: int, warmup: int, budget_s: float,
                            mixture: int = 0) -> dict:
    """cpu_protocol in a fresh interpreter (numpy + oracle only): no torch
    OpenMP pool or CUDA context shares the cores, and the product library is
    never mapped, so the bench's baseline and the reference arm measure the
    same thing."""
    import subprocess

    spec = json.dumps(dict(workload=workload, threads=threads, steps=steps, warmup=warmup, budget_s=budget_s,
                           mixture=mixture))
    out = subprocess.run([sys.executable, os.path.abspath(__file__), "--cpu-worker", spec], check=True,
                         capture_output=True, text=True).stdout
    return json.loads(out.strip().splitlines()[-1])


def bench_config(workload: str, world: int) -> dict:
    """The workload's identity, identical in both arms' JSON lines."""
    c = CONFIGS[workload]
    out = {"workload": workload, **{k: c[k] for k in ("F", "T", "sizes", "N", "K", "iters")}}
    if "batch" in c:
        out["mixtures"] = c["batch"]
    out["gpus"] = world
    return out


def run_reference(args, c, world, rank):
    """--impl reference: the reference's CPU algorithm on all host threads,
    rank 0 only, in the reference's timing protocol (cpu_protocol).  Each
    step is one EM iteration over the sample bins of the workload."""
    if rank != 0:
        return None
    threads = host_cpu()["nproc"]
    budget = 120.0
    r = cpu_protocol_subprocess(args.workload, threads, args.steps, args.warmup, budget)
    value = r["value"]
    if "batch" in c:  # config 4: mixtures are independent; one mixture's rate is the per-mixture rate
        r["sample"] += " (config 4: one mixture; the batch rate is the same per TF-bin)"
    return {
        "metric": f"dFastMNMF EM TF-bin*iter/s (BASELINE {args.workload})", "value": value,
        "unit": "TF-bin*iter/s", "impl": "reference", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * r["seconds_per_iter_sample"], "higher_is_better": True,
        "scaling": "strong" if world > 1 else "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded STFT-domain mixture, BASELINE config generator)",
        "config": bench_config(args.workload, world),
        "cpu_baseline": {k: r[k] for k in ("value", "unit", "cores", "kind", "sample", "mean", "se", "repeats",
                                            "host")},
        "e2e": {"value": value, "unit": "TF-bin*iter/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "iter_per_s_full_config": value / (c["F"] * c["T"]),
    }


def init_measurement(c, x, local, cpu_sample=True):
    """The initialisation pipeline (init_distributed, init.cpp:438-472) for
    this workload: device wall time of one dfm_init_pipeline call (host X in,
    model out, IS-NMF up to 1000 iterations), and the oracle's CPU time on a
    bounded sample (all host threads; k-means/alignment/SCM/GEVD in full,
    IS-NMF timed over 20 iterations and reported per iteration)."""
    import paper_2605_19388_b200 as dfm
    from paper_2605_19388_b200 import init as dinit

    layout = dfm.BlockLayout(c["sizes"])
    cfg = dinit.InitConfig(num_sources=c["N"], k_bases=c["K"], nmf_max_iters=1000)
    dinit.init_distributed(x[:8], layout, dinit.InitConfig(c["N"], c["K"], 5), 1)  # warm-up (module load)
    t0 = time.perf_counter()
    b = dinit.init_distributed(x, layout, cfg, SEED_INIT)
    dev_s = time.perf_counter() - t0
    out = {"step": "init_distributed (k-means masks, alignment, SCM/h0, IS-NMF <= 1000 iters, GEVD) through "
                   "paper_2605_19388_b200.init, host X in / model out",
           "device_seconds": dev_s, "nmf_max_iters": 1000, "lambda0_min": float(b.lambda0.min())}
    if cpu_sample:
        sys.path.insert(0, os.path.join(ROOT, "oracle"))
        import oracle
        import init_oracle

        oracle.build()
        oracle.set_threads(os.cpu_count() or 1)
        t0 = time.perf_counter()
        init_oracle.init_distributed(x, c["sizes"], c["N"], c["K"], SEED_INIT, nmf_iters=0)
        t_rest = time.perf_counter() - t0
        h0 = b.h0
        t0 = time.perf_counter()
        init_oracle.is_nmf(h0, c["K"], 20, 7)
        t_nmf = (time.perf_counter() - t0) / 20
        out["cpu_baseline"] = {"kind": "port", "cores": os.cpu_count() or 1,
                               "seconds_without_nmf": t_rest, "seconds_per_nmf_iter": t_nmf,
                               "seconds_extrapolated_1000_iters": t_rest + 1000 * t_nmf,
                               "sample": "oracle/ init_distributed without IS-NMF in full + 20 IS-NMF iterations "
                                         "(OpenMP over sources/bins)"}
    return out


def run_batch(args, c, world, rank, local):
    """config 4: independent mixtures, one context each, no communication."""
    import ctypes

    import torch

    import paper_2605_19388_b200 as dfm

    lib = dfm._capi.load()
    layout = dfm.BlockLayout(c["sizes"])
    F, T, N, K, M = c["F"], c["T"], c["N"], c["K"], layout.total
    nb = args.batch or c["batch"]
    mine = list(range(rank, nb, world))
    engines, xs, inits = [], [], []
    for j in mine:
        x = dfm.generate_mixture(c["kind"], F, T, M, N, K, SEED_X + j)
        init = dfm.random_init(F, T, layout, N, K, SEED_INIT + j)
        e = dfm.Engine(F, T, layout, N, K, device=local)
        e.set_obs(x)
        e.set_model(init.nmf, init.w0, init.lambda0)
        dfm._capi.check(lib.dfm_prime(e.ctx))
        engines.append(e)
        xs.append(pinned_copy(x))  # the caller's pinned host arrays (contract: H2D from pinned memory)
        inits.append(init)
    arr = (ctypes.c_void_p * len(engines))(*[e.ctx for e in engines])

    def step():
        v = ctypes.c_double()
        dfm._capi.check(lib.dfm_bench_step_many(arr, len(engines), ctypes.byref(v)))
        return v.value

    pg = torch.distributed if world > 1 else None
    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    if pg:
        pg.barrier()
    launches0 = sum(e.launches() for e in engines)
    sampler = ClockSampler(local).start()
    t_ms = [step() for _ in range(args.steps)]
    clocks = sampler.stop()
    launches = sum(e.launches() for e in engines) - launches0
    total_ms = float(np.sum(t_ms))
    if pg:
        tt = torch.tensor([total_ms], dtype=torch.float64, device="cuda")
        pg.all_reduce(tt, op=pg.ReduceOp.MAX)
        total_ms = float(tt.item())
    ms_step = total_ms / args.steps
    value = nb * F * T * args.steps / (total_ms * 1e-3)
    # e2e: every local mixture's pinned host X + init in, e2e_iters EM sweeps
    # of the batch (dfm_fit_many), cost traces and fitted models out
    e2e_times = []
    for _ in range(2):
        if pg:
            pg.barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for e, x, init in zip(engines, xs, inits):
            e.set_obs(x)
            e.set_model(init.nmf, init.w0, init.lambda0)
        dfm.fit_many(engines, args.e2e_iters)
        for e in engines:
            e.get_model()
        dt = time.perf_counter() - t0
        if pg:
            tt = torch.tensor([dt], dtype=torch.float64, device="cuda")
            pg.all_reduce(tt, op=pg.ReduceOp.MAX)
            dt = float(tt.item())
        e2e_times.append(dt)
    e2e_dt = min(e2e_times)
    mbytes = (inits[0].nmf.T.nbytes + inits[0].nmf.V.nbytes + inits[0].lambda0.nbytes
              + sum(w.nbytes for w in inits[0].w0))
    h2d = len(engines) * (xs[0].nbytes + mbytes)
    d2h = len(engines) * (mbytes + 8 * (args.e2e_iters + 1))
    if rank != 0:
        for e in engines:
            e.close()
        return None
    pk = peaks()
    fp64_peak = float(lib.dfm_probe_fp64_tflops(local))
    fl = nb * alg_flops(c) / (ms_step * 1e-3) / 1e12
    ab = nb * alg_bytes(c)
    line = {
        "metric": f"dFastMNMF EM TF-bin*iter/s (BASELINE {args.workload})",
        "value": value, "unit": "TF-bin*iter/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": ms_step, "higher_is_better": True, "scaling": "strong" if world > 1 else "weak",
        "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded STFT-domain mixtures, BASELINE config generator, one seed per mixture)",
        "config": bench_config(args.workload, world),
        "l2": f"working set of {len(engines)} contexts (~131 MB each) exceeds L2 (no flush)",
        "parallelism": f"mixtures sharded x{world}" if world > 1 else "1 GPU, one stream per mixture",
        "iter_per_s": 1e3 / ms_step,
        "roofline": {"bound": "hbm", "achieved": ab / (ms_step * 1e-3) / 1e9, "peak": pk["hbm_gbs"], "unit": "GB/s",
                     "frac": ab / (ms_step * 1e-3) / 1e9 / pk["hbm_gbs"], "traffic": None,
                     "kernel": "whole iteration (all mixtures)", "alg_bytes_per_step": ab,
                     "peak_source": pk["source"]},
        "roofline_fp64": {"bound": "fp64", "achieved": fl, "peak": fp64_peak, "unit": "TFLOP/s",
                          "frac": fl / fp64_peak if fp64_peak > 0 else None,
                          "peak_source": "measured in this run (DFMA microbenchmark, dfm_probe_fp64_tflops)"},
        "e2e": {"value": nb * F * T * args.e2e_iters / e2e_dt, "unit": "TF-bin*iter/s",
                "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h),
                "step": f"set_obs/set_model of every mixture (pinned host X + init H2D), fit_many({args.e2e_iters}), "
                        "get_model of every mixture; best of 2", "seconds_per_step": e2e_dt},
        "gpu_launches": int(launches),
        "clocks": clocks,
    }
    if not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_protocol_subprocess(args.workload, 1, 15, 1, 20.0)
    for e in engines:
        e.close()
    return line


def main():
    if len(sys.argv) == 3 and sys.argv[1] == "--cpu-worker":  # cpu_protocol_subprocess
        spec = json.loads(sys.argv[2])
        print(json.dumps(cpu_protocol(**spec)), flush=True)
        return
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--workload", default="config1", choices=sorted(CONFIGS))
    ap.add_argument("--e2e-iters", type=int, default=0,
                    help="EM iterations per e2e call (default: the config's own iteration count, e.g. 200 for config 1)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--tiling", default="", help="FT,TB override: frame tile of the per-bin kernel and of k_pd")
    ap.add_argument("--batch", type=int, default=0, help="config4: number of mixtures (default 64)")
    ap.add_argument("--no-init", action="store_true", help="skip the initialisation-pipeline measurement")
    ap.add_argument("--spinup-ms", type=float, default=300.0,
                    help="untimed steps for this long before the warm-up (GPU out of its idle clocks)")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    c = CONFIGS[args.workload]
    if args.e2e_iters <= 0:  # one e2e call = one full fit of the BASELINE config
        args.e2e_iters = c["iters"]
    world, rank, local = dist_setup()

    if args.impl == "reference":
        line = run_reference(args, c, world, rank)
        if line is not None:
            print(json.dumps(line), flush=True)
        return

    import torch

    torch.cuda.set_device(local)
    pg = None
    if world > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        pg = dist
    if "batch" in c:
        line = run_batch(args, c, world, rank, local)
        if line is not None:
            print(json.dumps(line), flush=True)
        if pg:
            pg.destroy_process_group()
        return
    import paper_2605_19388_b200 as dfm

    lib = dfm._capi.load()
    layout = dfm.BlockLayout(c["sizes"])
    F, T, N, K, M = c["F"], c["T"], c["N"], c["K"], layout.total
    x = dfm.generate_mixture(c["kind"], F, T, M, N, K, SEED_X)
    init = dfm.random_init(F, T, layout, N, K, SEED_INIT)
    f0, f1 = shard(F, world, rank)

    eng = dfm.Engine(F, T, layout, N, K, device=local, f_begin=f0, f_end=f1)
    if args.tiling:
        g, cs = (int(v) for v in args.tiling.split(","))
        eng.set_tiling(g, cs)
    if world > 1:
        uid = torch.zeros(128, dtype=torch.uint8, device="cuda")
        if rank == 0:
            import ctypes

            buf = ctypes.create_string_buffer(128)
            dfm._capi.check(lib.dfm_nccl_get_unique_id(buf))
            uid.copy_(torch.frombuffer(bytearray(buf.raw), dtype=torch.uint8))
        pg.broadcast(uid, 0)
        eng.comm_init(bytes(uid.cpu().numpy().tobytes()), world, rank)
    eng.set_obs(np.ascontiguousarray(x[f0:f1]))
    eng.set_model(init.nmf, init.w0, init.lambda0)
    ctx = eng.ctx

    def step(split=False):
        import ctypes

        dfm._capi.check(lib.dfm_l2_flush(local))  # untimed: outside the step's events
        if split:  # stream launches with per-kernel events (breakdown only)
            dfm._capi.check(lib.dfm_bench_split_step(ctx))
            sp = (ctypes.c_double * 5)()
            dfm._capi.check(lib.dfm_bench_last_split(ctx, sp))
            return list(sp)
        dfm._capi.check(lib.dfm_bench_step(ctx))  # one CUDA-graph replay
        return lib.dfm_bench_last_ms(ctx)

    dfm._capi.check(lib.dfm_prime(ctx))
    # untimed spin-up before the W warm-up steps: the same steps for a fixed
    # wall time, so a GPU that was idle (fresh process, fresh box) has left its
    # idle clocks before anything is timed
    if pg:
        # sharded steps hold an allreduce: every rank must run the same number
        # of them, so the spin-up is a fixed count there, not a wall time
        for _ in range(100 if args.spinup_ms > 0 else 0):
            step()
    else:
        spin_until = time.perf_counter() + args.spinup_ms * 1e-3
        spin = 0
        while time.perf_counter() < spin_until and spin < 4000:
            step()
            spin += 1
    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    if pg:
        pg.barrier()
    torch.cuda.synchronize()
    launches0 = eng.launches()
    sampler = ClockSampler(local).start()
    t_ms = []
    for i in range(args.steps):
        t_ms.append(step())
        if i % 4 == 1:  # between steps (host side; the steps are timed on the device)
            sampler.sample_now()
    dfm._capi.check(lib.dfm_sync(ctx))
    torch.cuda.synchronize()
    clocks = sampler.stop()
    launches = eng.launches() - launches0
    # per-kernel breakdown from separate (untimed-for-value) stream-launched steps
    split = [step(split=True) for _ in range(min(20, args.steps))]
    total_ms = float(np.sum(t_ms))
    if pg:
        tt = torch.tensor([total_ms], dtype=torch.float64, device="cuda")
        pg.all_reduce(tt, op=pg.ReduceOp.MAX)
        total_ms = float(tt.item())
        pg.barrier()
    torch.cuda.synchronize()
    ms_step = total_ms / args.steps
    value = F * T * args.steps / (total_ms * 1e-3)

    # ---------------------------------------------------------------- e2e
    # one user call through the public API per e2e step: pinned host X +
    # init in (H2D), e2e_iters EM sweeps, cost trace + fitted model out (D2H).
    # The caller's X lives in pinned host memory (allocated once, untimed);
    # its H2D copy is inside every timed step
    xs = pinned_copy(np.ascontiguousarray(x[f0:f1]))
    h2d = xs.nbytes + (init.nmf.T.nbytes + init.nmf.V.nbytes + init.lambda0.nbytes
                       + sum(w.nbytes for w in init.w0)) * (f1 - f0) // F
    e2e_times = []
    for rep in range(3):
        if pg:
            pg.barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        eng.set_obs(xs)
        eng.set_model(init.nmf, init.w0, init.lambda0)
        eng.fit(args.e2e_iters)  # cost trace D2H (allreduced across ranks when sharded)
        eng.get_model()
        dt = time.perf_counter() - t0
        if pg:
            tt = torch.tensor([dt], dtype=torch.float64, device="cuda")
            pg.all_reduce(tt, op=pg.ReduceOp.MAX)
            dt = float(tt.item())
        e2e_times.append(dt)
    e2e_dt = min(e2e_times)
    d2h = (init.nmf.T.nbytes + init.nmf.V.nbytes + init.lambda0.nbytes
           + sum(w.nbytes for w in init.w0)) * (f1 - f0) // F + 8 * (args.e2e_iters + 1)
    e2e_value = F * T * args.e2e_iters / e2e_dt

    if rank != 0:
        if pg:
            pg.destroy_process_group()
        return

    # Wiener separation (wiener.cpp:50-69) on the fitted model: HBM-bound,
    # reads X once and writes N images (16 F T M (1 + N) bytes)
    import ctypes as _ct

    w_ms = []
    for _ in range(5):
        dfm._capi.check(lib.dfm_l2_flush(local))
        v = _ct.c_double()
        dfm._capi.check(lib.dfm_bench_wiener(ctx, _ct.byref(v)))
        w_ms.append(v.value)
    w_ms = float(np.median(w_ms[1:]))
    w_bytes = 16.0 * (f1 - f0) * T * M * (1 + N)
    # STFT / inverse STFT of this workload's shape (stft.cpp:74-141, the
    # steps either side of the path): window 2 (F - 1), hop window / 4,
    # T frames, M channels, signal resident on the device
    sa, sb = _ct.c_double(), _ct.c_double()
    n_win = 2 * (F - 1)
    hop = n_win // 4
    sig_len = (T - 1) * hop + n_win
    dfm._capi.check(lib.dfm_bench_stft(sig_len, M, n_win, hop, 5, _ct.byref(sa), _ct.byref(sb), local))
    x_bytes = 16.0 * F * T * M
    stft = {"window": n_win, "hop": hop, "frames": T, "channels": M, "forward_ms": sa.value,
            "inverse_ms": sb.value,
            "alg_bytes_forward": 8.0 * sig_len * M + x_bytes, "alg_bytes_inverse": x_bytes + 8.0 * sig_len * M,
            "forward_gbs": (8.0 * sig_len * M + x_bytes) / (sa.value * 1e-3) / 1e9,
            "inverse_gbs": (x_bytes + 8.0 * sig_len * M) / (sb.value * 1e-3) / 1e9}
    pk = peaks()
    split_avg = np.mean(np.array(split), axis=0)
    names = ["k_em_bin", "k_tupd+h", "k_pdw", "k_vupd+H", "tail"]
    dom = int(np.argmax(split_avg))
    bin_avg = float(split_avg[0])
    ab_bin = alg_bytes_bin_kernel(c) * (f1 - f0) / F
    achieved = ab_bin / (bin_avg * 1e-3) / 1e9
    fp64_peak = float(lib.dfm_probe_fp64_tflops(local))
    fl = alg_flops(c) / (ms_step * 1e-3) / 1e12
    traffic = None
    prof = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(prof):
        try:
            with open(prof) as fh:
                traffic = json.load(fh).get(args.workload, {}).get("k_em_bin_dram_bytes_per_launch")
        except Exception:
            traffic = None
    line = {
        "metric": f"dFastMNMF EM TF-bin*iter/s (BASELINE {args.workload})",
        "value": value, "unit": "TF-bin*iter/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": ms_step, "higher_is_better": True, "scaling": "strong" if world > 1 else "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded STFT-domain mixture, BASELINE config generator)",
        "config": bench_config(args.workload, world),
        "l2": "flushed before every timed step (384 MB write, untimed)",
        "parallelism": f"freq-shard x{world}" if world > 1 else "1 GPU",
        "tiling": eng.tiling(),
        "iter_per_s": 1e3 / ms_step,
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": pk["hbm_gbs"], "unit": "GB/s",
                     "frac": achieved / pk["hbm_gbs"], "traffic": traffic, "kernel": "k_em_bin",
                     "alg_bytes_per_launch": ab_bin, "kernel_ms": bin_avg, "peak_source": pk["source"]},
        "roofline_fp64": {"bound": "fp64", "achieved": fl, "peak": fp64_peak, "unit": "TFLOP/s",
                          "frac": fl / fp64_peak if fp64_peak > 0 else None,
                          "alg_flops_per_iter": alg_flops(c),
                          "peak_source": "measured in this run (DFMA microbenchmark, dfm_probe_fp64_tflops)"},
        "iteration_roofline": {"alg_bytes_per_iter": alg_bytes(c), "hbm_frac": alg_bytes(c) / (ms_step * 1e-3) / 1e9 / pk["hbm_gbs"]},
        "kernel_split_ms": {n: float(v) for n, v in zip(names, split_avg)},
        "wiener": {"step": "separation of the fitted model (after the e2e fit): k_wiener_ctx, its (W_b^H)^-1 "
                           "written by the fit's last bin launch (blocks <= 4 mics; else k_wh_inverse first)",
                   "ms": w_ms, "alg_bytes": w_bytes, "achieved_gbs": w_bytes / (w_ms * 1e-3) / 1e9,
                   "frac_hbm": w_bytes / (w_ms * 1e-3) / 1e9 / pk["hbm_gbs"]},
        "dominant_kernel": names[dom],
        "stft": stft,
        "e2e": {"value": e2e_value, "unit": "TF-bin*iter/s", "h2d_bytes_per_step": int(h2d),
                "d2h_bytes_per_step": int(d2h),
                "step": f"Engine.set_obs/set_model (pinned host X + init H2D), Engine.fit({args.e2e_iters}) "
                        "(cost trace D2H), Engine.get_model (model D2H); best of 3",
                "seconds_per_step": e2e_dt},
        "gpu_launches": int(launches),
        "clocks": clocks,
        "paper_cpu_tfbin_iter_per_s_other_config": PAPER_CPU_TFBIN,
    }
    if world == 1 and not args.no_init:
        line["init_pipeline"] = init_measurement(c, x, local, cpu_sample=not args.no_cpu_baseline)
    if world == 1 and not args.no_cpu_baseline:
        # the same protocol and sample as the reference arm: 1 thread (the
        # reference's and the paper's protocol) and every host core
        line["cpu_baseline"] = cpu_protocol_subprocess(args.workload, 1, 15, 1, 20.0)
        line["cpu_baseline_all_cores"] = cpu_protocol_subprocess(args.workload, host_cpu()["nproc"], 15, 1, 20.0)
    print(json.dumps(line), flush=True)
    eng.close()
    if pg:
        pg.destroy_process_group()


if __name__ == "__main__":
    main()
