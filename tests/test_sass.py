"""Static checks of the built sm_100a library (no GPU needed).

* No cp.async (SASS LDGSTS) addresses shared memory through a uniform
  register ([Rn + URm]): with the L2 cache-hint operand that form raises "an
  illegal instruction was encountered" on sm_100a (driver 580.159, CUDA 12.9;
  isolated by tools/ldgsts_probe.cu).  ptxas picks the form by itself, so the
  built library is checked.
* The library holds native sm_100a code: FP64 tensor-core DMMA and TMA bulk
  copies (UBLKCP) are present.
"""
import os
import re
import shutil
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(ROOT, "paper_2605_19388_b200", "libdfm_b200.so")


@pytest.fixture(scope="module")
def sass():
    tool = shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump"
    if not os.path.exists(LIB) or not os.path.exists(tool):
        pytest.skip("library or cuobjdump missing")
    return subprocess.run([tool, "-sass", LIB], capture_output=True, text=True, check=True).stdout


def test_no_uniform_register_shared_address_in_ldgsts(sass):
    bad, fn = [], "?"
    for line in sass.splitlines():
        m = re.search(r"Function : (\S+)", line)
        if m:
            fn = m.group(1)
        if "LDGSTS" in line and re.search(r"\[R\d+\+UR\d+", line):
            bad.append((fn, line.strip()))
    assert not bad, f"{len(bad)} LDGSTS with a uniform-register shared address, e.g. {bad[:2]}"


def test_native_tensor_core_and_tma_instructions(sass):
    assert "DMMA" in sass  # mma.sync.m8n8k4.f64 (FP64 tensor cores)
    assert "UBLKCP" in sass  # cp.async.bulk (TMA bulk copies)
    assert "sm_100a" in subprocess.run([shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump", "-lelf", LIB],
                                       capture_output=True, text=True).stdout
