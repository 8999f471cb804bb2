"""Instruction mix of every kernel in the built library, from its SASS:

  python tools/sass_summary.py [lib.so] > profiles/rNN/sass_summary.md

Per kernel: instruction count, registers, and the counts of the mnemonics
that identify the path -- DMMA (mma.sync.m8n8k4.f64, the FP64 tensor cores),
DFMA/DMUL/DADD (FP64 pipe), LDGSTS (cp.async), UBLKCP (cp.async.bulk, the TMA
bulk copy engine), SYNCS (mbarrier), LDG/STG, LDS/STS, SHFL, BAR, and
UCGABAR / cluster instructions."""
import collections
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
lib = sys.argv[1] if len(sys.argv) > 1 else os.path.join(ROOT, "paper_2605_19388_b200", "libdfm_b200.so")
cuobjdump = "/usr/local/cuda/bin/cuobjdump"
sass = subprocess.run([cuobjdump, "-sass", lib], capture_output=True, text=True, check=True).stdout
res = subprocess.run([cuobjdump, "-res-usage", lib], capture_output=True, text=True, check=True).stdout
regs = {}
fn = None
for line in res.splitlines():
    m = re.search(r"Function (\S+):", line)
    if m:
        fn = m.group(1)
    m = re.search(r"REG:(\d+).*SHARED:(\d+)", line)
    if m and fn:
        regs[fn] = (int(m.group(1)), int(m.group(2)))
COLS = ["DMMA", "DFMA", "DMUL", "DADD", "MUFU", "LDGSTS", "UBLKCP", "SYNCS", "LDG", "STG", "LDS", "STS", "SHFL", "BAR"]
mix = collections.defaultdict(collections.Counter)
fn = None
for line in sass.splitlines():
    m = re.search(r"Function : (\S+)", line)
    if m:
        fn = m.group(1)
        continue
    m = re.search(r"/\*[0-9a-f]{4,}\*/\s+(?:@!?U?P\d+\s+)?([A-Z0-9_]+)", line)
    if m and fn:
        op = m.group(1)
        mix[fn]["total"] += 1
        for c in COLS:
            if op == c or op.startswith(c + "."):
                mix[fn][c] += 1
        if "CGA" in op or op.startswith("UCGABAR"):
            mix[fn]["cluster"] += 1
demangle = subprocess.run(["c++filt"], input="\n".join(mix), capture_output=True, text=True).stdout.splitlines()
names = dict(zip(mix, demangle))
print("# SASS instruction mix of `libdfm_b200.so` (sm_100a), `tools/sass_summary.py`\n")
print("| kernel | instr | regs | static smem | " + " | ".join(COLS) + " | cluster |")
print("|---|---|---|---|" + "---|" * (len(COLS) + 1))
for f in sorted(mix, key=lambda k: -mix[k]["total"]):
    n = names.get(f, f).replace("(anonymous namespace)::", "")
    n = re.sub(r"\(.*", "", n).replace("void ", "").replace("dfm::", "")
    r = regs.get(f, (0, 0))
    print(f"| `{n}` | {mix[f]['total']} | {r[0]} | {r[1]} | " + " | ".join(str(mix[f][c]) for c in COLS) +
          f" | {mix[f]['cluster']} |")
tot = collections.Counter()
for f in mix:
    tot.update(mix[f])
print(f"\nLibrary totals: " + ", ".join(f"{c} {tot[c]}" for c in COLS) + f"; kernels {len(mix)}.")
print("No HMMA / IMMA / QMMA (the path is FP64: tcgen05 has no FP64 kind, so DMMA is the tensor-core path), "
      "no `LDGSTS` with a uniform-register shared address (tests/test_sass.py).")
