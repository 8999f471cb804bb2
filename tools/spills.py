"""Static local-memory (spill) report for one kernel of the library.

  python tools/spills.py [kernel-substring]   (default: k_em_binILi4ELi3ELi5ELi4)

Compiles dfm_engine.cu to a cubin with line info and lists the LDL/STL
instructions of the matching kernel per source line."""
import collections
import os
import re
import subprocess
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def main():
    pat = sys.argv[1] if len(sys.argv) > 1 else "k_em_binILi4ELi3ELi5ELi4"
    with tempfile.TemporaryDirectory() as d:
        cub = os.path.join(d, "e.cubin")
        subprocess.run(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
                        "-I", os.path.join(ROOT, "include"), "-cubin", "-o", cub,
                        os.path.join(ROOT, "paper_2605_19388_b200", "csrc", "dfm_engine.cu")], check=True)
        sass = subprocess.run(["nvdisasm", "-g", cub], capture_output=True, text=True, check=True).stdout
    on, loc = False, None
    cnt = collections.Counter()
    n = 0
    for line in sass.splitlines():
        if re.match(r"^//-+ \.text\.", line):
            on = pat in line
            continue
        if not on:
            continue
        m = re.search(r'//## File "([^"]+)", line (\d+)', line)
        if m:
            loc = f"{os.path.basename(m.group(1))}:{m.group(2)}"
            continue
        if re.search(r"\b(LDL|STL)\b", line):
            cnt[loc] += 1
            n += 1
    print(f"{n} local-memory instructions in kernels matching {pat!r}")
    for k, v in cnt.most_common(30):
        print(f"  {v:4d}  {k}")


if __name__ == "__main__":
    main()
