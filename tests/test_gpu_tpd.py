"""The opt-in fused T update + pass D (k_tpd, csrc/dfm_tv.cu: one cluster of N
CTAs per bin tile, bulk-copy ring, DSMEM exchange of T_new) against the
oracle.  It is off in the product path (measured slower) and is
enabled per process with DFM_TPD=1, so each case runs in a subprocess."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

# one steady-state iteration is k_em_bin + k_tpd + k_vupd with the fused
# kernel (three launches), k_em_bin + k_tupd + k_pdw + k_vupd without it
COUNT = r"""
import numpy as np, bench, paper_2605_19388_b200 as dfm
c = bench.CONFIGS["config0"]
layout = dfm.BlockLayout(c["sizes"])
x = dfm.generate_mixture(c["kind"], c["F"], c["T"], layout.total, c["N"], c["K"], bench.SEED_X)
init = dfm.random_init(c["F"], c["T"], layout, c["N"], c["K"], bench.SEED_INIT)
e = dfm.Engine(c["F"], c["T"], layout, c["N"], c["K"])
e.set_obs(x); e.set_model(init.nmf, init.w0, init.lambda0)
dfm._capi.check(e.lib.dfm_prime(e.ctx))
n0 = e.launches(); dfm._capi.check(e.lib.dfm_bench_step(e.ctx)); print("LAUNCHES", e.launches() - n0)
"""


def _run(args, tpd):
    env = dict(os.environ)
    env.pop("DFM_TPD", None)
    if tpd:
        env["DFM_TPD"] = "1"
    return subprocess.run(args, cwd=ROOT, env=env, capture_output=True, text=True, timeout=1200)


def test_fused_kernel_is_selected_by_the_switch():
    on = _run([sys.executable, "-c", COUNT], True)
    off = _run([sys.executable, "-c", COUNT], False)
    assert on.returncode == 0 and off.returncode == 0, on.stderr + off.stderr
    n_on = int(on.stdout.split("LAUNCHES")[1])
    n_off = int(off.stdout.split("LAUNCHES")[1])
    assert n_on == n_off - 1, (n_on, n_off)


def test_fused_kernel_meets_the_parity_bar():
    """Configs 0 and 1 at the north_star bar (trajectory 1e-8 over 20
    iterations, non-increasing cost, separated STFTs 1e-6) from the dumped
    init, with k_tpd in place of k_tupd + k_pdw."""
    r = _run([sys.executable, "-m", "pytest", "-q", "-x", "-m", "gpu", "-p", "no:cacheprovider",
              "tests/test_gpu_baseline_parity.py", "-k", "config0 or config1"], True)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]
    assert "2 passed" in r.stdout, r.stdout[-2000:]
